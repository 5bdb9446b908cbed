// 2-D grid-point decomposition of the transform's grid (SURVEY.md section 8f
// row 4): latitude bands x longitude segments, and the second transposition
// between it and the ring-pair (Fourier-side) distribution the FFTs need --
// the role of ecTrans's TRGTOL / TRLTOG [domain: IFS/ecTrans conventions;
// the reference has no transform code, SPEC.md:20].
//
// Layout.  With nA x nB = P ranks, latitude band a holds a contiguous range
// of global rings (north first), split where the cumulative point count
// crosses a / nA of the total; segment b of ring j holds its points
// k in [floor(N_j b / nB), floor(N_j (b + 1) / nB)).  Rank a nB + b stores, per
// field, the segments b of the rings of band a, rings ascending, points
// ascending.  The ring-pair layout of a rank (its FFT output / input) is its
// rings in ascending global order (local north rings, then their southern
// mirrors), full rings.
//
// Transposition.  Every rank builds, for every peer, the per-point index list
// of what it sends (ascending ring, then point) and where incoming points go
// (the same order on the other side); pack and unpack are gather / scatter
// kernels over [peer block][field][point] buffers, and the exchange is a
// grouped NCCL send/recv in the reference's rotated order (collectives.py:
// 85-86).  One pass per direction: ring -> grid point after fft_f2g, grid
// point -> ring before fft_g2f.
#include <algorithm>

#include "sht_internal.h"

namespace sht {

namespace {

// t -> (peer block, position inside it): P <= a few dozen, linear search.
__device__ __forceinline__ int find_block(const int64_t* __restrict__ displ, int P, int64_t t) {
  int d = 0;
  while (d + 1 < P && displ[d + 1] <= t) ++d;
  return d;
}

// buf[displ[d] nfld + f cnt[d] + i] = src[f src_ld + idx[t]],  t = displ[d] + i
__global__ void gp_pack(const double* __restrict__ src, int64_t src_ld, const int32_t* __restrict__ idx,
                        const int64_t* __restrict__ displ, int P, int64_t ntot, int nfld, double* __restrict__ buf) {
  const int f = blockIdx.y;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntot; t += (int64_t)gridDim.x * blockDim.x) {
    const int d = find_block(displ, P, t);
    const int64_t cnt = displ[d + 1] - displ[d];
    buf[displ[d] * nfld + f * cnt + (t - displ[d])] = src[f * src_ld + idx[t]];
  }
}

// dst[f dst_ld + idx[t]] = buf[displ[d] nfld + f cnt[d] + i]
__global__ void gp_unpack(const double* __restrict__ buf, const int32_t* __restrict__ idx,
                          const int64_t* __restrict__ displ, int P, int64_t ntot, int nfld, double* __restrict__ dst,
                          int64_t dst_ld) {
  const int f = blockIdx.y;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntot; t += (int64_t)gridDim.x * blockDim.x) {
    const int d = find_block(displ, P, t);
    const int64_t cnt = displ[d + 1] - displ[d];
    dst[f * dst_ld + idx[t]] = buf[displ[d] * nfld + f * cnt + (t - displ[d])];
  }
}

}  // namespace

void gp_bands(const std::vector<int>& nloen, int nA, std::vector<int>& band_lo) {
  const int ndgl = (int)nloen.size();
  int64_t tot = 0;
  for (int n : nloen) tot += n;
  band_lo.assign(nA + 1, ndgl);
  band_lo[0] = 0;
  int64_t cum = 0;
  int a = 1;
  for (int j = 0; j < ndgl && a < nA; ++j) {
    cum += nloen[j];
    while (a < nA && cum * nA >= tot * a) band_lo[a++] = j + 1;
  }
}

int gp_build(const std::vector<int>& nloen, const std::vector<int>& ring_rank, int P, int rank, int nA, int nB,
             GpLayout& L) {
  const int ndgl = (int)nloen.size();
  L = GpLayout{};
  L.nA = nA;
  L.nB = nB;
  gp_bands(nloen, nA, L.band_lo);
  std::vector<int> band(ndgl);
  for (int a = 0; a < nA; ++a)
    for (int j = L.band_lo[a]; j < L.band_lo[a + 1]; ++j) band[j] = a;
  auto seg = [&](int j, int b, int& k0, int& k1) {
    k0 = (int)((int64_t)nloen[j] * b / nB);
    k1 = (int)((int64_t)nloen[j] * (b + 1) / nB);
  };
  // my ring-layout offsets (rings ascending) and every GP rank's ring offsets
  std::vector<int64_t> ringoff(ndgl, -1);
  int64_t o = 0;
  for (int j = 0; j < ndgl; ++j)
    if (ring_rank[j] == rank) {
      ringoff[j] = o;
      o += nloen[j];
    }
  const int my_a = rank / nB, my_b = rank % nB;
  std::vector<int64_t> gpoff(ndgl, -1);
  o = 0;
  for (int j = L.band_lo[my_a]; j < L.band_lo[my_a + 1]; ++j) {
    int k0, k1;
    seg(j, my_b, k0, k1);
    gpoff[j] = o;
    o += k1 - k0;
  }
  L.npts_gp = o;
  // ring -> GP (send lists, indices into my ring layout), grouped by destination
  L.send_displ.assign(P + 1, 0);
  L.recv_displ.assign(P + 1, 0);
  L.send_idx.clear();
  L.recv_idx.clear();
  for (int d = 0; d < P; ++d) {
    L.send_displ[d] = (int64_t)L.send_idx.size();
    const int a = d / nB, b = d % nB;
    for (int j = L.band_lo[a]; j < L.band_lo[a + 1]; ++j) {
      if (ring_rank[j] != rank) continue;
      int k0, k1;
      seg(j, b, k0, k1);
      for (int k = k0; k < k1; ++k) L.send_idx.push_back((int32_t)(ringoff[j] + k));
    }
  }
  L.send_displ[P] = (int64_t)L.send_idx.size();
  // GP side: from each source s, the points of my band's rings owned by s, same order
  for (int s = 0; s < P; ++s) {
    L.recv_displ[s] = (int64_t)L.recv_idx.size();
    for (int j = L.band_lo[my_a]; j < L.band_lo[my_a + 1]; ++j) {
      if (ring_rank[j] != s) continue;
      int k0, k1;
      seg(j, my_b, k0, k1);
      for (int k = k0; k < k1; ++k) L.recv_idx.push_back((int32_t)(gpoff[j] + k - k0));
    }
  }
  L.recv_displ[P] = (int64_t)L.recv_idx.size();
  if (L.send_idx.size() > INT32_MAX || L.npts_gp > INT32_MAX) return SHT_ERR_CONFIG;
  return SHT_OK;
}

void gp_launch_pack(const double* src, int64_t src_ld, const int32_t* idx, const int64_t* displ, int P, int64_t ntot,
                    int nfld, double* buf, cudaStream_t s) {
  if (ntot <= 0) return;
  dim3 grid((unsigned)std::min<int64_t>((ntot + 255) / 256, 148 * 4), (unsigned)nfld);
  gp_pack<<<grid, 256, 0, s>>>(src, src_ld, idx, displ, P, ntot, nfld, buf);
}

void gp_launch_unpack(const double* buf, const int32_t* idx, const int64_t* displ, int P, int64_t ntot, int nfld,
                      double* dst, int64_t dst_ld, cudaStream_t s) {
  if (ntot <= 0) return;
  dim3 grid((unsigned)std::min<int64_t>((ntot + 255) / 256, 148 * 4), (unsigned)nfld);
  gp_unpack<<<grid, 256, 0, s>>>(buf, idx, displ, P, ntot, nfld, dst, dst_ld);
}

void gp_preload() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, gp_pack);
  cudaFuncGetAttributes(&a, gp_unpack);
}

}  // namespace sht

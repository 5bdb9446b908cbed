// Ring FFTs of the SH transform on sm_100a (K4 fft_g2f: grid -> Fourier,
// K5 fft_f2g: Fourier -> grid) on the variable-length octahedral rings.
//
// One CTA owns one ring PAIR (northern ring i and its southern mirror, same
// length N) for a range of fields, processed in batches of nb fields.  The
// two hemispheres of a field are packed into one complex sequence
// (z = x_N + i x_S), so every transform is a complex DFT of length N; the
// hemispheres are separated with Z_m / conj(Z_{N-m}) and combined at once
// into the parity rows.
//
// The DFT is an in-place "pencil" FFT in shared memory: L = R_0 R_1 ... R_{d-1}
// (d <= 4, R_j <= 16, or a prime <= 31); in step j every thread owns whole
// pencils of R_j points (stride S_j), loads them, runs a straight-line
// codelet (tools/gen_codelets.py) in registers, applies the step's twiddles
// (base twiddle from a 2-level table in shared memory, powers by recurrence)
// and writes them back to the same addresses.  No value crosses a barrier in
// registers and no second buffer is needed, so a 2576-point ring pair for one
// field needs 82 KB and two CTAs share an SM.  The decimation-in-time
// order leaves the spectrum digit-reversed (extraction reads it through
// dit_pos).  One prime factor 16 < p <= 127 becomes the last step, done as
// FP64 tensor-core GEMMs (dmma_prime_step).  Larger primes (or two of them)
// send the ring through whole-ring Bluestein (below), or, for rings too long
// for one CTA, make a prime factor p > 16 a Bluestein step (factor-local
// chirp-z): its DFT_p pencils are gathered G at a time into a work buffer,
// convolved with the chirp kernel by an inner pencil FFT of 13-smooth length
// Lp >= 2p-1 (DIT, kernel product fused into the last inner step, then the
// transposed steps that map digit-reversed back to natural order) and
// scattered back; the ring itself is never padded, so rings up to 8192 points
// (TCo1999) fit one CTA.
//
// Fusions: g2f scales by 1/N and combines the two hemispheres into the
// parity rows the Legendre GEMM consumes, S' = w_i (F_N + F_S) and
// A' = w_i (F_N - F_S) (Gaussian weight folded in).  f2g reads S, A rows and
// forms F_N = S + A, F_S = S - A while filling its FFT buffer.  Fourier rows
// are addressed through per-(ring, m) row pointers, so g2f stores straight
// into the m-owner's receive buffer (a peer GPU's memory over NVLink when the
// transposition runs peer-to-peer) and f2g reads this rank's receive buffer:
// pack/unpack and the transposition itself are fused.
//
// This header holds the device code; sht_fft.cu instantiates the kernels for
// the classic Fourier-row layout (plus the host planning), sht_fft_blk.cu for
// the field-blocked one (sht_internal.h), so the two compile in parallel.
#pragma once
#include <algorithm>
#include <cmath>
#include <complex>
#include <functional>

#include "sht_internal.h"

namespace sht {

namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 conjc(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // -i * a
__device__ __forceinline__ double2 mul_pi(double2 a) { return make_double2(-a.y, a.x); }  // +i * a

#include "fft_codelets.cuh"

__device__ __forceinline__ int fdiv(int x, uint64_t mag) { return (int)(((uint64_t)(unsigned)x * mag) >> 40); }

// Padded shared-memory slot of FFT point x: one spare slot per 16 points, so
// the contiguous pencils of the last step (stride R) spread over the banks.
__device__ __forceinline__ int px(int x) { return x + (x >> 4); }

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int V>
struct FftCfg {  // 1: 256 threads, 2 CTAs / SM; 3: rings past 100 KB, 512 threads, 1 CTA / SM
  static constexpr int kThreads = V == 3 ? 512 : 256;
  static constexpr int kMinBlocks = V == 1 ? 2 : 1;
  template <int R>
  static constexpr bool has() {
    return V == 2 ? true : (R <= 16);
  }
};

constexpr int kMaxAllSteps = 3 * kMaxSteps;  // ring steps + inner steps of up to two Bluestein steps

// W^e of a transform from its 2-level table at `base` (lo[64], hi[...]).
__device__ __forceinline__ double2 tw_at(const double2* __restrict__ twt, int base, int e) {
  return cmul(twt[base + 64 + (e >> 6)], twt[base + (e & 63)]);
}

// One pencil step over nseq sequences of length L (in place).  kFwd: DIT
// step (codelet, then twiddle); else transposed step (twiddle, then codelet).
// kPost: last DIT step of a Bluestein convolution fused with the first
// transposed step (same pencils, no twiddle): store DFT(conj(X * bhat)).
template <int R, int V, bool kFwd, bool kPost>
__device__ __forceinline__ void step_run(double2* __restrict__ buf, int nseq, int L, const FftStep& st, bool tw,
                                         const double2* __restrict__ twt, const double2* __restrict__ bhat) {
  constexpr int NT = FftCfg<V>::kThreads;
  const int np = st.np, S = st.S;
  const int total = nseq * np;
  for (int b = threadIdx.x; b < total; b += NT) {
    const int q = fdiv(b, st.mag_np);
    const int pp = b - q * np;
    const int blk = fdiv(pp, st.mag_S);
    const int s = pp - blk * S;
    const int i0 = q * L + blk * st.B + s;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = buf[px(i0 + r * S)];
    const bool twd = tw && s > 0;
    double2 w1 = make_double2(1.0, 0.0);
    if (twd) w1 = tw_at(twt, st.tw_base, s * st.tmul);
    if (!kFwd && twd) {
      double2 wr = w1;
      v[1] = cmul(v[1], w1);
#pragma unroll
      for (int r = 2; r < R; ++r) {
        wr = cmul(wr, w1);
        v[r] = cmul(v[r], wr);
      }
    }
    dft<R>(v);
    if (kFwd && twd) {
      double2 wr = w1;
      v[1] = cmul(v[1], w1);
#pragma unroll
      for (int r = 2; r < R; ++r) {
        wr = cmul(wr, w1);
        v[r] = cmul(v[r], wr);
      }
    }
    if (kPost) {  // last DIT step: S == 1, positions blk * R + r
      const double2* bh = bhat + blk * R;
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = conjc(cmul(v[r], __ldg(bh + r)));
      dft<R>(v);
#pragma unroll
      for (int r = 0; r < R; ++r) buf[px(i0 + r)] = v[r];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) buf[px(i0 + r * S)] = v[r];
    }
  }
  __syncthreads();
}

template <int V, bool kFwd, bool kPost>
__device__ __forceinline__ void step_dispatch(double2* buf, int nseq, int L, const FftStep& st, bool tw,
                                              const double2* __restrict__ twt, const double2* __restrict__ bhat) {
  switch (st.R) {
#define SHT_CASE(R)                                                                                  \
  case R:                                                                                            \
    if constexpr (FftCfg<V>::template has<R>()) step_run<R, V, kFwd, kPost>(buf, nseq, L, st, tw, twt, bhat); \
    break;
    SHT_CASE(2) SHT_CASE(3) SHT_CASE(4) SHT_CASE(5) SHT_CASE(6) SHT_CASE(7) SHT_CASE(8) SHT_CASE(9)
    SHT_CASE(10) SHT_CASE(11) SHT_CASE(12) SHT_CASE(13) SHT_CASE(14) SHT_CASE(15) SHT_CASE(16)
    default:
      if constexpr (V == 2) {
        switch (st.R) { SHT_CASE(17) SHT_CASE(19) SHT_CASE(23) SHT_CASE(29) SHT_CASE(31) default: break; }
      }
      break;
#undef SHT_CASE
  }
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// DMMA prime step: the DFT_p (p prime, 16 < p <= kMaxDmmaPrime) of every
// contiguous pencil of the last DIT step as FP64 tensor-core GEMMs (SASS
// DMMA.8x8x4), instead of padding the whole ring through Bluestein.  With
// t_j = x_j + x_{p-j}, u_j = x_j - x_{p-j} (j = 1..H, H = (p-1)/2):
//   A_k = sum_j cos(2 pi jk/p) t_j   (k = 0..H; A_0 = sum t_j),
//   B_k = sum_j sin(2 pi jk/p) u_j,
//   X_k = x_0 + A_k - i B_k,  X_{p-k} = x_0 + A_k + i B_k.
// Each warp owns groups of 4 pencils (8 real columns = one DMMA n-tile): it
// forms t/u in place, accumulates all (H+1) output rows of its group in
// registers (<= 8 row tiles x {cos, sin}), then overwrites the group -- no
// other warp touches those pencils, so a __syncwarp orders reads and writes.
// A operand: (cos, sin)(2 pi ((k j) mod p) / p) from a p-entry table in shared
// memory; B operand: t_j / u_j straight from the pencil.
template <int V>
__device__ void dmma_prime_step(double2* __restrict__ buf, int nseq, int L, const FftStep& st,
                                const double2* __restrict__ cs) {
  constexpr int NT = FftCfg<V>::kThreads;
  constexpr int kTiles = (kMaxDmmaPrime - 1) / 2 / 8 + 1;  // row tiles of k = 0..H
  const int p = st.R, H = (p - 1) >> 1;
  const int npen = st.np;  // pencils per sequence (L / p)
  const int tot = nseq * npen;
  const int ngrp = (tot + 3) >> 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntile = (H + 8) >> 3;
  const int nj = (H + 3) >> 2;
  const uint32_t magp = (1u << 20) / (uint32_t)p + 1;  // (x * magp) >> 20 == x / p for x < 2^20 / p
  auto pbase = [&](int pen) {                          // unpadded index of a pencil's point 0
    const int q = fdiv(pen, st.mag_np);
    return q * L + (pen - q * npen) * p;
  };
  for (int g = warp; g < ngrp; g += NT / 32) {
    // 1. t / u in place: pairs (pencil, j) over the lanes
    for (int idx = lane; idx < 4 * H; idx += 32) {
      const int pl = idx / H, j = idx - pl * H + 1;
      const int pen = 4 * g + pl;
      if (pen < tot) {
        const int b0 = pbase(pen);
        const double2 a = buf[px(b0 + j)], b = buf[px(b0 + p - j)];
        buf[px(b0 + j)] = cadd(a, b);
        buf[px(b0 + p - j)] = csub(a, b);
      }
    }
    __syncwarp();
    // 2. GEMMs: rows k = 8 t + (lane >> 2), columns (pencil, re/im)
    double acc[kTiles][2][2];
#pragma unroll
    for (int t = 0; t < kTiles; ++t) acc[t][0][0] = acc[t][0][1] = acc[t][1][0] = acc[t][1][1] = 0.0;
    const int bpen = 4 * g + (lane >> 3), bre = (lane >> 2) & 1;  // B fragment: column lane >> 2
    const bool bval = bpen < tot;
    const int bb0 = bval ? pbase(bpen) : 0;
    for (int js = 0; js < nj; ++js) {
      const int j = 4 * js + (lane & 3) + 1;  // B row and A column of this lane
      double bt = 0.0, bu = 0.0;
      if (bval && j <= H) {
        const double2 t = buf[px(bb0 + j)], u = buf[px(bb0 + p - j)];
        bt = bre ? t.y : t.x;
        bu = bre ? u.y : u.x;
      }
#pragma unroll
      for (int t = 0; t < kTiles; ++t) {
        if (t < ntile) {
          const int k = 8 * t + (lane >> 2);
          double ac = 0.0, as = 0.0;
          if (j <= H && k <= H) {
            const uint32_t x = (uint32_t)(k * j);
            const double2 w = cs[x - ((x * magp) >> 20) * p];
            ac = w.x;
            as = w.y;
          }
          dmma(acc[t][0][0], acc[t][0][1], ac, bt);
          dmma(acc[t][1][0], acc[t][1][1], as, bu);
        }
      }
    }
    // 3. outputs: this lane holds row k = 8 t + (lane >> 2) of pencil lane & 3
    const int open = 4 * g + (lane & 3);
    const bool oval = open < tot;
    const int ob0 = oval ? pbase(open) : 0;
    const double2 x0 = oval ? buf[px(ob0)] : make_double2(0.0, 0.0);
    __syncwarp();  // every lane has read its t / u / x0
    if (oval) {
#pragma unroll
      for (int t = 0; t < kTiles; ++t) {
        const int k = 8 * t + (lane >> 2);
        if (t < ntile && k <= H) {
          const double ax = acc[t][0][0], ay = acc[t][0][1], bx = acc[t][1][0], by = acc[t][1][1];
          buf[px(ob0 + k)] = make_double2(x0.x + ax + by, x0.y + ay - bx);
          if (k) buf[px(ob0 + p - k)] = make_double2(x0.x + ax - by, x0.y + ay + bx);
        }
      }
    }
    __syncwarp();
  }
  __syncthreads();
}

// Bluestein step: every DFT_R pencil (R prime > 31) of the nseq sequences is
// x -> w_k conj(conv(x w, conj w))_k, the convolution done by the inner pencil
// FFT of length Lp on G pencils at a time in the work buffer W.
template <int V>
__device__ void bluestein_step(double2* __restrict__ buf, double2* __restrict__ W, int nseq, int L,
                               const FftStep& st, bool tw, const FftStep* __restrict__ steps,
                               const double2* __restrict__ twt, const double2* __restrict__ tab) {
  constexpr int NT = FftCfg<V>::kThreads;
  const int R = st.R, S = st.S, Lp = st.Lp;
  const int total = nseq * st.np;
  const double2* chirp = tab + st.chirp_off;
  const double2* bhat = tab + st.bhat_off;
  for (int g0 = 0; g0 < total; g0 += st.G) {
    const int ng = min(st.G, total - g0);
    for (int idx = threadIdx.x; idx < ng * Lp; idx += NT) {
      const int g = fdiv(idx, st.mag_Lp), r = idx - g * Lp;
      double2 v = make_double2(0.0, 0.0);
      if (r < R) {
        const int pen = g0 + g;
        const int q = fdiv(pen, st.mag_np), pp = pen - q * st.np;
        const int blk = fdiv(pp, st.mag_S), s = pp - blk * S;
        v = cmul(buf[px(q * L + blk * st.B + s + r * S)], __ldg(chirp + r));
      }
      W[px(idx)] = v;
    }
    __syncthreads();
    for (int j = 0; j < st.ninner; ++j) {
      const FftStep& is = steps[st.inner0 + j];
      if (j == st.ninner - 1)
        step_dispatch<V, true, true>(W, ng, Lp, is, false, twt, bhat);
      else
        step_dispatch<V, true, false>(W, ng, Lp, is, true, twt, bhat);
    }
    for (int j = st.ninner - 2; j >= 0; --j)
      step_dispatch<V, false, false>(W, ng, Lp, steps[st.inner0 + j], true, twt, bhat);
    for (int idx = threadIdx.x; idx < ng * R; idx += NT) {
      const int g = fdiv(idx, st.mag_Rb), k = idx - g * R;
      const int pen = g0 + g;
      const int q = fdiv(pen, st.mag_np), pp = pen - q * st.np;
      const int blk = fdiv(pp, st.mag_S), s = pp - blk * S;
      double2 y = cmul(__ldg(chirp + k), conjc(W[px(g * Lp + k)]));
      if (tw && s > 0) y = cmul(y, tw_at(twt, st.tw_base, k * s * st.tmul));
      buf[px(q * L + blk * st.B + s + k * S)] = y;
    }
    __syncthreads();
  }
}

// In-place ring DFT of nseq sequences.  Direct / factor-local Bluestein: DIT
// steps, spectrum left digit-reversed.  Whole-ring Bluestein: chirp-
// premultiplied input of length L, DIT with conj(X bhat) fused into the last
// step, then the transposed steps: buf holds conj(conv) in natural order.
template <int V>
__device__ __forceinline__ void ring_dft(double2* buf, double2* W, int L, int nseq, const FftStep* steps, int nstep,
                                         const double2* __restrict__ twt, const double2* __restrict__ tab,
                                         bool ring_blue, const double2* __restrict__ bhat) {
  if (ring_blue) {
    for (int j = 0; j < nstep; ++j) {
      if (j == nstep - 1)
        step_dispatch<V, true, true>(buf, nseq, L, steps[j], false, twt, bhat);
      else
        step_dispatch<V, true, false>(buf, nseq, L, steps[j], true, twt, bhat);
    }
    for (int j = nstep - 2; j >= 0; --j) step_dispatch<V, false, false>(buf, nseq, L, steps[j], true, twt, bhat);
    return;
  }
  for (int j = 0; j < nstep; ++j) {
    if (steps[j].ptab >= 0)
      dmma_prime_step<V>(buf, nseq, L, steps[j], twt + steps[j].ptab);
    else if (steps[j].blue)
      bluestein_step<V>(buf, W, nseq, L, steps[j], j < nstep - 1, steps, twt, tab);
    else
      step_dispatch<V, true, false>(buf, nseq, L, steps[j], j < nstep - 1, twt, nullptr);
  }
}

// Chirp w_k = exp(-i pi k^2 / N) along a thread's walk k = k0, k0 + NT, ...
// (k0 < NT, NT = 256 or 512): w_{k+256} = w_k g_k, g_{k+256} = g_k h, with
// g_t (t < 256) and h from the arena right after the chirp table
// (fft_build_ring).  Two complex multiplies per 256 replace an L2 load per
// point; ~N/256 steps keep the drift at a few ulp.
struct ChirpWalk {
  double2 c, g, h;
  __device__ __forceinline__ ChirpWalk(const double2* __restrict__ chirp, int N, int k0) {
    c = k0 < N ? __ldg(chirp + k0) : make_double2(1.0, 0.0);
    g = __ldg(chirp + N + (k0 & 255));
    h = __ldg(chirp + N + 256);
    if (k0 >= 256) g = cmul(g, h);
  }
  template <int NT>
  __device__ __forceinline__ void step() {
    static_assert(NT == 256 || NT == 512, "ChirpWalk strides by 256 or 512");
#pragma unroll
    for (int i = 0; i < NT / 256; ++i) {
      c = cmul(c, g);
      g = cmul(g, h);
    }
  }
};

// Digit-reversed position of spectrum index k after the DIT steps.
__device__ __forceinline__ int dit_pos(int k, const FftStep* steps, int nstep) {
  int pos = 0;
#pragma unroll
  for (int j = 0; j < kMaxSteps; ++j) {
    if (j < nstep) {
      const int kq = fdiv(k, steps[j].mag_R);
      pos += (k - kq * steps[j].R) * steps[j].S;
      k = kq;
    }
  }
  return pos;
}

// Shared prologue: ring descriptor, steps (ring + inner) and the twiddle tables.
struct RingSmem {
  FftRing rg;
  FftWork wk;
  FftStep st[kMaxAllSteps];
  double2 tw[kTwMax];
};

__device__ __forceinline__ void load_ring(RingSmem& rs, const FftParams& p, int w) {
  if (threadIdx.x == 0) {
    rs.wk = p.work[w];
    rs.rg = p.rings[rs.wk.ring];
  }
  __syncthreads();
  if ((int)threadIdx.x < kMaxAllSteps) rs.st[threadIdx.x] = p.steps[rs.rg.step0 + threadIdx.x];
  for (int t = threadIdx.x; t < rs.rg.ntw; t += blockDim.x) rs.tw[t] = p.tw[rs.rg.tw_off + t];
  __syncthreads();
}

// Field slot f of a Fourier row (sht_internal.h): classic rows hold every
// field; field-blocked rows (p2p, P > 1) hold 64, the blocks bs apart.
template <bool kBlk>
__device__ __forceinline__ int64_t slot_off(int f, int64_t bs) {
  if constexpr (kBlk) return (f >> 6) * bs + (f & 63) * 4;
  return (int64_t)f * 4;
}

// ------------------------------------------------------------------ grid -> Fourier
template <int V, bool kBlk>
__global__ void __launch_bounds__(FftCfg<V>::kThreads, FftCfg<V>::kMinBlocks)
    fft_g2f_kernel(const FftParams p, int w0, const double* __restrict__ grid, double* __restrict__ four) {
  constexpr int NT = FftCfg<V>::kThreads;
  extern __shared__ __align__(16) double2 smc[];
  __shared__ RingSmem rs;
  load_ring(rs, p, w0 + blockIdx.x);
  const FftRing& rg = rs.rg;
  const int N = rg.n, L = rg.L, M = rg.mcap;
  double2* buf = smc;
  double2* W = smc + fft_slots((size_t)rg.nb * L);  // factor-local Bluestein work buffer
  const bool blue = rg.chirp_off >= 0;             // whole-ring Bluestein
  const double2* chirp = p.tw + (blue ? rg.chirp_off : 0);
  const double2* bhat = p.tw + (blue ? rg.bhat_off : 0);
  const double scale = 0.5 / N;
  const double w = rg.w;
  const int nbatch = (rs.wk.f1 - rs.wk.f0 + rg.nb - 1) / rg.nb;

  for (int t = 0; t < nbatch; ++t) {
    const int fb = rs.wk.f0 + t * rg.nb;
    const int nseq = min(rg.nb, rs.wk.f1 - fb);
    // grid -> smem (north -> .x, south -> .y), zero tail; Bluestein rings
    // apply the chirp on the way (register loads), the others use cp.async
    if (blue && nseq == 1) {  // one field: thread-strided k with the chirp walked in registers
      constexpr int U = 4;
      const double* src = grid + (int64_t)fb * p.grid_ld;
      ChirpWalk cw(chirp, N, threadIdx.x);
      for (int k0 = threadIdx.x; k0 < L; k0 += U * NT) {
        double xn[U], xs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = k0 + u * NT;
          xn[u] = xs[u] = 0.0;
          if (k < N && !(p.debug & 2)) {
            xn[u] = __ldcs(src + rg.goff_n + k);
            xs[u] = __ldcs(src + rg.goff_s + k);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = k0 + u * NT;
          if (k < N) {
            buf[px(k)] = cmul(make_double2(xn[u], xs[u]), cw.c);
            cw.step<NT>();
          } else if (k < L) {
            buf[px(k)] = make_double2(0.0, 0.0);
          }
        }
      }
    } else if (blue) {
      // 4 elements per thread and round, all 12 loads issued before the first use
      constexpr int U = 4;
      const int tot = nseq * L;
      for (int i0 = threadIdx.x; i0 < tot; i0 += U * NT) {
        double xn[U], xs[U];
        double2 c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = i0 + u * NT;
          const int q = fdiv(idx, rg.mag_L), n = idx - q * L;
          xn[u] = xs[u] = 0.0;
          c[u] = make_double2(0.0, 0.0);
          if (idx < tot && n < N && !(p.debug & 2)) {
            const double* src = grid + (int64_t)(fb + q) * p.grid_ld;
            xn[u] = __ldcs(src + rg.goff_n + n);
            xs[u] = __ldcs(src + rg.goff_s + n);
            c[u] = __ldg(chirp + n);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = i0 + u * NT;
          if (idx < tot) buf[px(idx)] = cmul(make_double2(xn[u], xs[u]), c[u]);
        }
      }
    } else {
      for (int idx = threadIdx.x; idx < nseq * L; idx += NT) {
        const int q = fdiv(idx, rg.mag_L), n = idx - q * L;
        double* dst = reinterpret_cast<double*>(buf + px(idx));
        if (n < N) {
          if (!(p.debug & 2)) {
            const double* src = grid + (int64_t)(fb + q) * p.grid_ld;
            cp_async8(dst, src + rg.goff_n + n);
            cp_async8(dst + 1, src + rg.goff_s + n);
          }
        } else {
          buf[px(idx)] = make_double2(0.0, 0.0);
        }
      }
      cp_async_commit();
      cp_async_wait<0>();
    }
    __syncthreads();
    if (!(p.debug & 1)) ring_dft<V>(buf, W, L, nseq, rs.st, rg.nstep, rs.tw, p.tw, blue, bhat);
    auto Z = [&](int q, int k) {  // k = m or N - m (pruned Bluestein: the latter at L - m)
      if (blue) return cmul(__ldg(chirp + k), conjc(buf[px(q * L + (k > M ? k + rg.shift : k))]));
      return buf[px(q * L + __ldg(p.ditpos + rg.dit_off + k))];
    };
    // one thread per (m, field): consecutive threads store consecutive 32-byte
    // field slots of one Fourier row
    if (blue && nseq == 1 && !(p.debug & 4)) {  // chirp walked along m; w_{N-m} = (-1)^N w_m
      const double sg = (N & 1) ? -1.0 : 1.0;
      ChirpWalk cw(chirp, N, threadIdx.x);
      for (int m = threadIdx.x; m <= M; m += NT) {
        const double2 zm = cmul(cw.c, conjc(buf[px(m)]));
        const double2 zn = m == 0 ? zm : cmul(make_double2(sg * cw.c.x, sg * cw.c.y), conjc(buf[px(N - m + rg.shift)]));
        cw.step<NT>();
        const double2 fn = make_double2((zm.x + zn.x) * scale, (zm.y - zn.y) * scale);  // F_N
        const double2 fs = make_double2((zm.y + zn.y) * scale, (zn.x - zm.x) * scale);  // F_S
        st_slot(p.rows_out[rg.yrow_off + m] + slot_off<kBlk>(fb, kBlk ? p.rows_out_bs[rg.yrow_off + m] : 0), w * (fn.x + fs.x), w * (fn.y + fs.y),
                w * (fn.x - fs.x), w * (fn.y - fs.y));
      }
      __syncthreads();
      continue;
    }
    #pragma unroll 4
    for (int idx = threadIdx.x; idx < nseq * (M + 1); idx += NT) {
      const int m = idx / nseq, q = idx - m * nseq;
      const double2 zm = Z(q, m);
      const double2 zn = Z(q, m == 0 ? 0 : N - m);
      const double2 fn = make_double2((zm.x + zn.x) * scale, (zm.y - zn.y) * scale);  // F_N
      const double2 fs = make_double2((zm.y + zn.y) * scale, (zn.x - zm.x) * scale);  // F_S
      if (p.debug & 4) continue;
      st_slot(p.rows_out[rg.yrow_off + m] + slot_off<kBlk>(fb + q, kBlk ? p.rows_out_bs[rg.yrow_off + m] : 0), w * (fn.x + fs.x), w * (fn.y + fs.y),
              w * (fn.x - fs.x), w * (fn.y - fs.y));
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ Fourier -> grid
template <int V, bool kBlk>
__global__ void __launch_bounds__(FftCfg<V>::kThreads, FftCfg<V>::kMinBlocks)
    fft_f2g_kernel(const FftParams p, int w0, const double* __restrict__ four, double* __restrict__ grid) {
  constexpr int NT = FftCfg<V>::kThreads;
  extern __shared__ __align__(16) double2 smc[];
  __shared__ RingSmem rs;
  load_ring(rs, p, w0 + blockIdx.x);
  const FftRing& rg = rs.rg;
  const int N = rg.n, L = rg.L, M = rg.mcap;
  double2* buf = smc;
  double2* W = smc + fft_slots((size_t)rg.nb * L);
  const bool blue = rg.chirp_off >= 0;
  const double2* chirp = p.tw + (blue ? rg.chirp_off : 0);
  const double2* bhat = p.tw + (blue ? rg.bhat_off : 0);
  const int nbatch = (rs.wk.f1 - rs.wk.f0 + rg.nb - 1) / rg.nb;

  for (int t = 0; t < nbatch; ++t) {
    const int fb = rs.wk.f0 + t * rg.nb;
    const int nseq = min(rg.nb, rs.wk.f1 - fb);
    // zero the bins no coefficient reaches: (M, N - M + shift) and [N + shift, L)
    const int gap = L - 2 * M - 1, gap1 = N - 2 * M - 1 + rg.shift;
    if (nseq == 1) {  // two plain ranges, no division
      for (int k = M + 1 + threadIdx.x; k <= M + gap1; k += NT) buf[px(k)] = make_double2(0.0, 0.0);
      for (int k = N + rg.shift + threadIdx.x; k < L; k += NT) buf[px(k)] = make_double2(0.0, 0.0);
    } else {
      for (int idx = threadIdx.x; idx < nseq * gap; idx += NT) {
        const int q = idx / gap, g = idx - q * gap;
        const int k = g < gap1 ? M + 1 + g : N + rg.shift + (g - gap1);
        buf[px(q * L + k)] = make_double2(0.0, 0.0);
      }
    }
    // Fourier rows -> conj(Z) at k = m and k = N - m, Z = F_N + i F_S
    // (one thread per (m, field): a row's 32-byte field slots are read once)
    if (blue && nseq == 1) {  // chirp walked along m; w_{N-m} = (-1)^N w_m
      const double sg = (N & 1) ? -1.0 : 1.0;
      ChirpWalk cw(chirp, N, threadIdx.x);
      constexpr int U = 3;  // all of a thread's row loads in flight at once (M + 1 <= 3 NT in one round)
      for (int m0 = threadIdx.x; m0 <= M; m0 += U * NT) {
        double2 S[U], A[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int m = m0 + u * NT;
          S[u] = A[u] = make_double2(0.0, 0.0);
          if (m <= M && !(p.debug & 2))
            ld_slot(p.rows_in[rg.yrow_off + m] + slot_off<kBlk>(fb, p.in_bs), S[u].x, S[u].y, A[u].x, A[u].y);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int m = m0 + u * NT;
          if (m > M) break;
          double2 fn = cadd(S[u], A[u]), fs = csub(S[u], A[u]);
          if (m == 0) {
            fn.y = 0.0;
            fs.y = 0.0;
          }
          buf[px(m)] = cmul(make_double2(fn.x - fs.y, -(fn.y + fs.x)), cw.c);
          if (m)
            buf[px(N - m + rg.shift)] =
                cmul(make_double2(fn.x + fs.y, fn.y - fs.x), make_double2(sg * cw.c.x, sg * cw.c.y));
          cw.step<NT>();
        }
      }
    } else
    #pragma unroll 4
    for (int idx = threadIdx.x; idx < nseq * (M + 1); idx += NT) {
      const int m = idx / nseq, q = idx - m * nseq;
      double2 S = make_double2(0.0, 0.0), A = S;
      if (!(p.debug & 2))
        ld_slot(p.rows_in[rg.yrow_off + m] + slot_off<kBlk>(fb + q, p.in_bs), S.x, S.y, A.x, A.y);
      double2 fn = cadd(S, A), fs = csub(S, A);
      if (m == 0) {
        fn.y = 0.0;
        fs.y = 0.0;
      }
      // conj(Z) at k = m (Z = F_N + i F_S) and at k = N - m (Z = conj(F_N) + i conj(F_S))
      double2 lo = make_double2(fn.x - fs.y, -(fn.y + fs.x));
      double2 hi = make_double2(fn.x + fs.y, fn.y - fs.x);
      if (blue) {
        lo = cmul(lo, __ldg(chirp + m));
        if (m) hi = cmul(hi, __ldg(chirp + N - m));
      }
      buf[px(q * L + m)] = lo;
      if (m) buf[px(q * L + N - m + rg.shift)] = hi;
    }
    __syncthreads();
    if (!(p.debug & 1)) ring_dft<V>(buf, W, L, nseq, rs.st, rg.nstep, rs.tw, p.tw, blue, bhat);
    if (blue && nseq == 1) {  // chirp walked along k
      ChirpWalk cw(chirp, N, threadIdx.x);
      double* g = grid + (int64_t)fb * p.grid_ld;
      for (int k = threadIdx.x; k < N; k += NT) {
        const double2 r = cmul(cw.c, conjc(buf[px(k ? k + rg.shift : 0)]));
        cw.step<NT>();
        if (p.debug & 4) continue;
        __stcs(g + rg.goff_n + k, r.x);
        __stcs(g + rg.goff_s + k, -r.y);
      }
    } else if (blue) {  // chirp loads of 4 elements in flight per thread
      constexpr int U = 4;
      const int tot = nseq * N;
      for (int i0 = threadIdx.x; i0 < tot; i0 += U * NT) {
        double2 c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = i0 + u * NT;
          const int q = fdiv(idx, rg.mag_N), k = idx - q * N;
          c[u] = idx < tot ? __ldg(chirp + k) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = i0 + u * NT;
          if (idx >= tot || (p.debug & 4)) continue;
          const int q = fdiv(idx, rg.mag_N), k = idx - q * N;
          const double2 r = cmul(c[u], conjc(buf[px(q * L + (k ? k + rg.shift : 0))]));
          double* g = grid + (int64_t)(fb + q) * p.grid_ld;
          __stcs(g + rg.goff_n + k, r.x);
          __stcs(g + rg.goff_s + k, -r.y);
        }
      }
    } else {  // (the per-ring position table measured no faster than dit_pos here)
      for (int idx = threadIdx.x; idx < nseq * N; idx += NT) {
        const int q = fdiv(idx, rg.mag_N), k = idx - q * N;
        const double2 r = buf[px(q * L + dit_pos(k, rs.st, rg.nstep))];
        if (p.debug & 4) continue;
        double* g = grid + (int64_t)(fb + q) * p.grid_ld;
        __stcs(g + rg.goff_n + k, r.x);
        __stcs(g + rg.goff_s + k, -r.y);
      }
    }
    __syncthreads();
  }
}

template <int V, bool kBlk>
void launch_one(bool g2f, const FftParams& p, int w0, int nw, const double* in, double* out, size_t smem,
                cudaStream_t s) {
  if (g2f) {
    cudaFuncSetAttribute(fft_g2f_kernel<V, kBlk>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fft_g2f_kernel<V, kBlk><<<nw, FftCfg<V>::kThreads, smem, s>>>(p, w0, in, out);
  } else {
    cudaFuncSetAttribute(fft_f2g_kernel<V, kBlk>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fft_f2g_kernel<V, kBlk><<<nw, FftCfg<V>::kThreads, smem, s>>>(p, w0, in, out);
  }
}

}  // namespace
}  // namespace sht

// Legendre side of the SH transform on sm_100a:
//   K3 leg_diag/leg_poly : associated-Legendre table P_n^m(mu_i) (X-number recurrence)
//   K1 leg_inv           : per-m parity-split FP64 GEMM, spectral -> Fourier (S/A rows)
//   K2 leg_dir           : per-m parity-split FP64 GEMM, Fourier (S/A rows) -> spectral
//
// FP64 tensor cores: tcgen05.mma has no f64 kind, so the
// GEMMs are built from warp-level DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4),
// the only FP64 tensor path on B200; measured issue peak 37.1 TFLOP/s at
// 1965 MHz (profiles/r01_probe_fp64.json).  Operands are staged HBM -> shared
// memory by 1-D bulk copies (TMA, cp.async.bulk -> SASS UBLKCP) completing on
// per-stage mbarriers (2 stages of 64 wavenumbers / 32 rings); fragments are
// read with 128-bit LDS; a persistent CTA per SM pulls tiles (m ascending,
// largest K first) from an atomic ticket and prefetches the next tile's
// operands under the current tile's epilogue.
//
// Parity split (SURVEY.md App. A "Hemispheric split"): for each m the S
// accumulator takes the even n-m and the A accumulator the odd n-m.  Both come
// out of the same smem tiles because P[ring][n] and spec[field][n][re,im] keep
// n contiguous: one 128-bit LDS yields the (S, A) pair of an operand fragment.
// The ring FFT kernels consume/produce S and A directly (north = S + A,
// south = S - A), so the Legendre kernels have no combine epilogue at all.
#include "sht_internal.h"

namespace sht {

namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// ---- bulk-copy (TMA 1-D, cp.async.bulk) + mbarrier helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-specialised pipeline: warps 0..7 consume (DMMA), warps 8.. produce (bulk
// copies; 4 warps in leg_inv, 1 in leg_dir).  kStages shared-memory stages, each with a "full" barrier (the
// producer's expect_tx arrival + the copies' transaction bytes) and an
// "empty" barrier (one arrival per consumer warp), so no CTA-wide barrier sits
// in the K loop and the copy issue is off the DMMA warps' path.  CTAs walk the
// wavenumber-major tile list with a static stride (tile = blockIdx.x + k *
// gridDim.x): the list starts with the largest K, so the interleave balances.
constexpr int kConsumers = 8;
constexpr int kInvProducers = 4;  // leg_inv: 4 producer warps share a stage's row copies
constexpr int kInvThreads = 32 * (kConsumers + kInvProducers);
constexpr int kDirThreads = 32 * (kConsumers + 1);
constexpr int kMaxStages = 4;

struct Pipe {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
};

// leg_inv's staged epilogue (p2p transport, tiles with rings owned by a peer):
// the consumers park the finished tile in a per-CTA slot of local HBM and
// move on; the pusher warp (the last producer warp) streams it to the ring
// owners over NVLink while the next tile's GEMM runs.  "staged" completes when
// the 8 consumer warps have written a slot, "freed" when the pusher has read it.
constexpr int64_t kStageDbl = (int64_t)kInvRings * kLegFields * 4;
struct StagePipe {
  uint64_t staged[kStageSlots];
  uint64_t freed[kStageSlots];
};

__device__ __forceinline__ void st_stage(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ void ld_stage(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p) : "memory");
}

template <int kStages>
__device__ __forceinline__ void pipe_init(Pipe& pp) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&pp.full[s], 1);
      mbar_init(&pp.empty[s], kConsumers);
    }
    fence_mbar_init();
  }
}

// ------------------------------------------------------------------ leg_inv
// 4 stages of 32 wavenumbers, the 128 row copies of a stage issued by 4
// producer warps (one warp could not issue them under a stage's DMMA work;
// 1 warp x 2 stages of 64: 8.63 ms, 4 warps x 4 x 32: 8.32 ms at TCo639)
constexpr int kInvStages = 4;
constexpr int kInvKcP = 32;                    // k-chunk (wavenumbers n) per stage
constexpr int kInvPStr = kInvKcP + 8;          // 72 doubles: P rows (== 8 mod 16 -> no LDS.128 conflicts)
constexpr int kInvSStr = 2 * kInvKcP + 2;      // 130 doubles: field rows of the spectral tile (== 2 mod 16)
constexpr int kInvPDbl = kInvRings * kInvPStr;
constexpr int kInvSDbl = kLegFields * kInvSStr;
constexpr int kInvStageDbl = kInvPDbl + kInvSDbl;

// Tile: rings r0..r0+63 (northern index) x fields f0..f0+63 of wavenumber lm.
// Consumer warp w: rings 32*(w&1).. , fields 16*(w>>1)..  -> 4 ring groups x 2
// field groups x {S.re, S.im, A.re, A.im} DMMA accumulators (64 doubles per thread).
struct InvTile {
  int lm, r0, f0, K, nk, kp, nrows, nf;
  const double* P;
  const double* S;
};

__device__ __forceinline__ InvTile inv_tile(const LegParams& p, const double* spec, int t) {
  InvTile c;
  const LegTile tile = p.tiles[t];
  c.lm = tile.lm;
  c.r0 = tile.r0;
  c.f0 = tile.f0;
  const int m = p.lm_m[c.lm];
  c.kp = p.lm_kp[c.lm];
  c.K = p.T - m + 1;
  c.nk = (c.K + kInvKcP - 1) / kInvKcP;
  c.nrows = min(kInvRings, p.nh - c.r0);
  c.nf = min(kLegFields, p.nfld - c.f0);
  c.P = p.ptab + p.lm_poff[c.lm] + (int64_t)(c.r0 - p.lm_i0[c.lm]) * c.kp;
  c.S = spec + 2 * p.lm_soff[c.lm];
  return c;
}

template <bool kStaged, bool kBlk>  // pusher epilogue; field-blocked Fourier rows (sht_internal.h)
__global__ void __launch_bounds__(kInvThreads, 1)
    leg_inv_kernel(const LegParams p, const double* __restrict__ spec, double* __restrict__ four) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) Pipe pp;
  __shared__ __align__(8) StagePipe sp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr bool staging = kStaged;  // p.stage != nullptr

  // stale operand slots must hold finite values (they meet zero P padding or
  // feed discarded accumulator rows)
  for (int i = tid; i < kInvStages * kInvStageDbl; i += kInvThreads) sm[i] = 0.0;
  pipe_init<kInvStages>(pp);
  if (staging && tid == 0) {
    for (int s = 0; s < kStageSlots; ++s) {
      mbar_init(&sp.staged[s], kConsumers);
      mbar_init(&sp.freed[s], 1);
    }
    fence_mbar_init();
  }
  fence_async_smem();
  __syncthreads();

  if (staging && warp == kConsumers + kInvProducers - 1) {  // ---- pusher
    int k = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      if (!p.tiles[t].pad) continue;
      const InvTile c = inv_tile(p, spec, t);
      const int slot = k & 1;
      mbar_wait(&sp.staged[slot], (k >> 1) & 1);
      ++k;
      const double* src = p.stage + ((int64_t)blockIdx.x * kStageSlots + slot) * kStageDbl;
      for (int r0 = 0; r0 < c.nrows; r0 += 4) {  // 8 slot loads in flight per lane
        double v[4][2][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int r = r0 + a, f = lane + 32 * b;
            if (r < c.nrows && f < c.nf)
              ld_stage(src + ((int64_t)r * kLegFields + f) * 4, v[a][b][0], v[a][b][1], v[a][b][2], v[a][b][3]);
          }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int r = r0 + a;
          if (r >= c.nrows) break;
          double* dst = p.ring_out[c.r0 + r] + (kBlk ? (c.f0 >> 6) * p.ring_bs[c.r0 + r] + (int64_t)c.lm * kRowDbl
                                                     : c.lm * p.row_ld + c.f0 * 4);
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int f = lane + 32 * b;
            if (f < c.nf) st_slot(dst + (int64_t)f * 4, v[a][b][0], v[a][b][1], v[a][b][2], v[a][b][3]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sp.freed[slot]);  // every load of the slot has returned
    }
    return;
  }

  if (warp >= kConsumers) {  // ---- producers: one bulk copy per P row / field row and k-chunk
    const int pw = warp - kConsumers;
    const int nprod = staging ? kInvProducers - 1 : kInvProducers;
    int st = 0;
    unsigned ph = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      const InvTile c = inv_tile(p, spec, t);
      for (int kc = 0; kc < c.nk; ++kc) {
        mbar_wait(&pp.empty[st], ph ^ 1);
        double* Ps = sm + st * kInvStageDbl;
        double* Ss = Ps + kInvPDbl;
        const int kcount = min(kInvKcP, c.K - kc * kInvKcP);
        if (pw == 0 && lane == 0) mbar_expect_tx(&pp.full[st], (unsigned)(c.nrows * kInvKcP * 8 + c.nf * kcount * 16));
        __syncwarp();
        for (int j = pw * 32 + lane; j < c.nrows + c.nf; j += 32 * nprod) {
          if (j < c.nrows)
            bulk_g2s(Ps + j * kInvPStr, c.P + (int64_t)j * c.kp + kc * kInvKcP, kInvKcP * 8, &pp.full[st]);
          else {
            const int f = j - c.nrows;
            bulk_g2s(Ss + f * kInvSStr, c.S + (int64_t)(c.f0 + f) * p.spec_ld + 2 * kc * kInvKcP, kcount * 16,
                     &pp.full[st]);
          }
        }
        if (++st == kInvStages) {
          st = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  // ---- consumers
  const int wr = warp & 1, wf = warp >> 1;
  const int lr = lane >> 2, lc = lane & 3;
  int st = 0;
  unsigned ph = 0;
  int ks = 0;  // staged tiles so far
  for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
    const InvTile c = inv_tile(p, spec, t);
    const bool staged = staging && p.tiles[t].pad;
    double acc[4][2][4][2];
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[g][h][q][0] = acc[g][h][q][1] = 0.0;
    // the tile's rings split evenly (in 8-ring groups) between the two ring
    // warps, so a ragged last tile costs ceil(rows / 16) groups, not min(4, ceil(rows / 8))
    const int rows = min(kInvRings, p.nh - c.r0);
    const int split = min(kInvRings / 2, ((rows + 1) / 2 + 7) & ~7);
    const int roff = wr ? split : 0;
    const int nrow = wr ? rows - min(split, rows) : min(split, rows);
    const bool active = nrow > 0 && (c.f0 + wf * 16 < p.nfld);
    // warp-uniform trims of the ragged edges: 8-ring groups, 8-field groups, 8-n sub-steps
    const int gmax = min(4, (nrow + 7) / 8);
    const int hmax = min(2, max(0, (p.nfld - c.f0 - wf * 16 + 7) / 8));
    // the epilogue's destination rows, fetched now so their latency hides under the K loop
    double* dst_row[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int ring = c.r0 + roff + g * 8 + (lane >> 2);
      dst_row[g] = (active && !staged && g < gmax && ring < p.nh)
                       ? p.ring_out[ring] + (kBlk ? (c.f0 >> 6) * p.ring_bs[ring] + (int64_t)c.lm * kRowDbl
                                                  : c.lm * p.row_ld + c.f0 * 4)
                       : nullptr;
    }

    for (int kc = 0; kc < c.nk; ++kc) {
      mbar_wait(&pp.full[st], ph);
      if (active) {
        const double* Ps = sm + st * kInvStageDbl + (roff + lr) * kInvPStr + 2 * lc;
        const double* Ss = sm + st * kInvStageDbl + kInvPDbl + (wf * 16 + lr) * kInvSStr + 4 * lc;
        const int smax = min(kInvKcP / 8, (c.K - kc * kInvKcP + 7) / 8);
#pragma unroll
        for (int sub = 0; sub < kInvKcP / 8; ++sub) {
          if (sub >= smax) break;
          double2 a[4], bs[2], ba[2];
#pragma unroll
          for (int g = 0; g < 4; ++g) a[g] = *reinterpret_cast<const double2*>(Ps + g * 8 * kInvPStr + sub * 8);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double* bp = Ss + h * 8 * kInvSStr + sub * 16;
            bs[h] = *reinterpret_cast<const double2*>(bp);
            ba[h] = *reinterpret_cast<const double2*>(bp + 2);
          }
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (g < gmax && h < hmax) {
                dmma(acc[g][h][0][0], acc[g][h][0][1], a[g].x, bs[h].x);
                dmma(acc[g][h][1][0], acc[g][h][1][1], a[g].x, bs[h].y);
                dmma(acc[g][h][2][0], acc[g][h][2][1], a[g].y, ba[h].x);
                dmma(acc[g][h][3][0], acc[g][h][3][1], a[g].y, ba[h].y);
              }
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&pp.empty[st]);  // this warp is done with stage st
      if (++st == kInvStages) {
        st = 0;
        ph ^= 1;
      }
    }
    // epilogue: each (ring, field) slot as one 256-bit store straight into the
    // ring owner's receive buffer (local, or a peer GPU over NVLink), or -- a
    // staged tile -- into this CTA's staging slot for the pusher; the producers
    // keep filling the next tile's stages meanwhile
    if (staged) {
      const int slot = ks & 1;
      mbar_wait(&sp.freed[slot], ((ks >> 1) & 1) ^ 1);  // the pusher has drained this slot's last tile
      ++ks;
      if (active && !(p.debug & 4)) {
        double* sdst = p.stage + ((int64_t)blockIdx.x * kStageSlots + slot) * kStageDbl;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int rl = roff + g * 8 + lr;
          if (g < gmax && c.r0 + rl < p.nh) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int fl = wf * 16 + h * 8 + 2 * lc + e;
                if (c.f0 + fl < p.nfld)
                  st_stage(sdst + ((int64_t)rl * kLegFields + fl) * 4, acc[g][h][0][e], acc[g][h][1][e],
                           acc[g][h][2][e], acc[g][h][3][e]);
              }
          }
        }
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sp.staged[slot]);
    } else if (active && !(p.debug & 4)) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int ring = c.r0 + roff + g * 8 + lr;
        if (g < gmax && ring < p.nh) {
          double* dst = dst_row[g];
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int fl = wf * 16 + h * 8 + 2 * lc + e;
              if (c.f0 + fl < p.nfld)
                st_slot(dst + fl * 4, acc[g][h][0][e], acc[g][h][1][e], acc[g][h][2][e], acc[g][h][3][e]);
            }
        }
      }
    }
  }
}

// ------------------------------------------------------------------ leg_dir
constexpr int kDirStages = 4;
constexpr int kDirKcR = 16;                    // k-chunk (rings) per stage
constexpr int kDirPStr = kDirN + 4;            // 132: P tile [ring][n]          (== 4 mod 16)
// B tile [ring][field][S.re, S.im, A.re, A.im]: row pitch a multiple of 128 B
// plus a per-ring 16-byte offset {0, 1, 4, 5}[ring % 4], so the 8 lanes of an
// LDS.128 phase (2 fields x 4 rings) hit 8 distinct bank groups
constexpr int kDirBStr = 4 * kLegFields + 16;  // 272 doubles = 17 x 128 B
__device__ __forceinline__ int dir_boff(int ring) { return 2 * ((ring & 1) + 4 * ((ring >> 1) & 1)); }
constexpr int kDirPDbl = kDirKcR * kDirPStr;
constexpr int kDirBDbl = kDirKcR * kDirBStr + 16;
constexpr int kDirStageDbl = kDirPDbl + kDirBDbl;

// Tile: n-m offsets n0..n0+127 (64 even-parity rows, 64 odd) x fields f0..f0+63.
// Consumer warp w: n 64*(w&1).. (4 groups of 8 (S,A) row pairs), fields 16*(w>>1)..
struct DirTile {
  int lm, n0, f0, K, i0, nrings, nk, kp, nf;
  const double* P;
};

__device__ __forceinline__ DirTile dir_tile(const LegParams& p, int t) {
  DirTile c;
  const LegTile tile = p.tiles[t];
  c.lm = tile.lm;
  c.n0 = tile.r0;
  c.f0 = tile.f0;
  const int m = p.lm_m[c.lm];
  c.i0 = p.lm_i0[c.lm];
  c.kp = p.lm_kp[c.lm];
  c.K = p.T - m + 1;
  c.nrings = p.nh - c.i0;
  c.nk = (c.nrings + kDirKcR - 1) / kDirKcR;
  c.nf = min(kLegFields, p.nfld - c.f0);
  c.P = p.ptab + p.lm_poff[c.lm];
  return c;
}

__global__ void __launch_bounds__(kDirThreads, 1)
    leg_dir_kernel(const LegParams p, const double* __restrict__ four, double* __restrict__ spec) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) Pipe pp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int i = tid; i < kDirStages * kDirStageDbl; i += kDirThreads) sm[i] = 0.0;
  pipe_init<kDirStages>(pp);
  fence_async_smem();
  __syncthreads();

  if (warp == kConsumers) {  // ---- producer: per ring of the chunk one P-row segment and one Fourier row
    int st = 0;
    unsigned ph = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      const DirTile c = dir_tile(p, t);
      const int pbytes = min(kDirN, c.kp - c.n0) * 8;
      for (int kc = 0; kc < c.nk; ++kc) {
        mbar_wait(&pp.empty[st], ph ^ 1);
        double* Ps = sm + st * kDirStageDbl;
        double* Bs = Ps + kDirPDbl;
        const int nr = min(kDirKcR, c.nrings - kc * kDirKcR);
        // rings past the end inside the last 4-ring k-step must contribute
        // zero; the expect_tx arrival (release) follows these stores
        for (int rr = nr; rr < ((nr + 3) & ~3); ++rr)
          for (int q = lane; q < kDirN; q += 32) Ps[rr * kDirPStr + q] = 0.0;
        __syncwarp();
        if (lane == 0) mbar_expect_tx(&pp.full[st], (unsigned)(nr * (pbytes + c.nf * 32)));
        __syncwarp();
        for (int j = lane; j < 2 * nr; j += 32) {
          const int rr = j >> 1;
          const int ring = kc * kDirKcR + rr;  // relative to i0
          if (j & 1)
            bulk_g2s(Bs + rr * kDirBStr + dir_boff(rr),
                     four + (c.f0 >> p.fsh) * p.xbs + (p.xbase[c.i0 + ring] + c.lm) * p.row_ld + (c.f0 & p.fmask) * 4,
                     c.nf * 32,
                     &pp.full[st]);
          else
            bulk_g2s(Ps + rr * kDirPStr, c.P + (int64_t)ring * c.kp + c.n0, pbytes, &pp.full[st]);
        }
        if (++st == kDirStages) {
          st = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  const int wn = warp & 1, wf = warp >> 1;
  const int lr = lane >> 2, lc = lane & 3;
  int st = 0;
  unsigned ph = 0;
  for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
    const DirTile c = dir_tile(p, t);
    double acc[4][2][4][2];
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[g][h][q][0] = acc[g][h][q][1] = 0.0;
    const bool active = (c.n0 + wn * 64 < c.K) && (c.f0 + wf * 16 < p.nfld);
    // warp-uniform trims: 16-n row-pair groups, 8-field groups, 4-ring k-steps
    const int gmax = min(4, max(0, (c.K - c.n0 - wn * 64 + 15) / 16));
    const int hmax = min(2, max(0, (p.nfld - c.f0 - wf * 16 + 7) / 8));

    for (int kc = 0; kc < c.nk; ++kc) {
      mbar_wait(&pp.full[st], ph);
      if (active) {
        const double* Ps = sm + st * kDirStageDbl + lc * kDirPStr + wn * 64 + 2 * lr;
        const double* Bs = sm + st * kDirStageDbl + kDirPDbl + lc * kDirBStr + dir_boff(lc) + 4 * (wf * 16 + lr);
        const int kmax = min(kDirKcR / 4, (c.nrings - kc * kDirKcR + 3) / 4);
#pragma unroll
        for (int ks = 0; ks < kDirKcR / 4; ++ks) {
          if (ks >= kmax) break;
          double2 a[4], bs[2], ba[2];
#pragma unroll
          for (int g = 0; g < 4; ++g)
            a[g] = *reinterpret_cast<const double2*>(Ps + ks * 4 * kDirPStr + 16 * g);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double* bp = Bs + ks * 4 * kDirBStr + 32 * h;
            bs[h] = *reinterpret_cast<const double2*>(bp);
            ba[h] = *reinterpret_cast<const double2*>(bp + 2);
          }
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (g < gmax && h < hmax) {
                dmma(acc[g][h][0][0], acc[g][h][0][1], a[g].x, bs[h].x);
                dmma(acc[g][h][1][0], acc[g][h][1][1], a[g].x, bs[h].y);
                dmma(acc[g][h][2][0], acc[g][h][2][1], a[g].y, ba[h].x);
                dmma(acc[g][h][3][0], acc[g][h][3][1], a[g].y, ba[h].y);
              }
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&pp.empty[st]);
      if (++st == kDirStages) {
        st = 0;
        ph ^= 1;
      }
    }

    if (active && !(p.debug & 4)) {
      const int64_t soff = 2 * p.lm_soff[c.lm];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int ns = c.n0 + wn * 64 + 2 * (g * 8 + lr);
        if (ns < c.K) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int f = c.f0 + wf * 16 + h * 8 + 2 * lc + e;
              if (f < p.nfld) {
                double2* d = reinterpret_cast<double2*>(spec + (int64_t)f * p.spec_ld + soff + 2 * ns);
                d[0] = make_double2(acc[g][h][0][e], acc[g][h][1][e]);
                if (ns + 1 < c.K) d[1] = make_double2(acc[g][h][2][e], acc[g][h][3][e]);
              }
            }
        }
      }
    }
  }
}

// ------------------------------------------------------------------ leg_poly
// X-number sectoral start values, one thread per northern ring walking m = 0..T.
// Operation order matches oracle/sht_oracle.py legendre_diag exactly (no FMA
// contraction), so the P table is bit-identical to the oracle's.
__global__ void leg_diag_kernel(int T, int nh, const double* __restrict__ sint, int nlm,
                                const int32_t* __restrict__ lm_m, double* __restrict__ dmant,
                                int32_t* __restrict__ dexp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nh) return;
  const double s = sint[i];
  const double two400 = 0x1p400, twom400 = 0x1p-400;
  double cur = 1.0 / sqrt(2.0);
  int e = 0;
  int lm = 0;
  if (lm < nlm && lm_m[lm] == 0) {
    dmant[(int64_t)lm * nh + i] = cur;
    dexp[(int64_t)lm * nh + i] = e;
    ++lm;
  }
  for (int m = 1; m <= T && lm < nlm; ++m) {
    const double fac = __dmul_rn(sqrt((2.0 * m + 1.0) / (2.0 * m)), s);
    cur = __dmul_rn(cur, fac);
    if (cur < twom400) {
      cur = __dmul_rn(cur, two400);
      e -= 400;
    }
    if (lm_m[lm] == m) {
      dmant[(int64_t)lm * nh + i] = cur;
      dexp[(int64_t)lm * nh + i] = e;
      ++lm;
    }
  }
}

__device__ __forceinline__ double eps_nm(int n, int m) {
  const double nn = (double)n;
  return sqrt(__ddiv_rn(__dsub_rn(__dmul_rn(nn, nn), (double)((int64_t)m * m)),
                        __dsub_rn(__dmul_rn(__dmul_rn(4.0, nn), nn), 1.0)));
}

// One thread per (local m, ring): three-term recurrence in n on the mantissa,
// shared per-ring exponent, renormalised by 2^-400 above 2^400.
// A warp's 32 rings produce 32 columns n at a time into a shared-memory tile,
// which the warp then stores row by row (one coalesced 256-byte segment per
// ring) -- a thread writing its own row (stride Kp) made every store
// instruction touch 32 rows.  eps(n, m) (a division and a square root) is the
// same for every ring: lane L computes it for column c0 + L of the chunk and
// the warp shares it by shuffles, instead of every ring recomputing it.  The
// arithmetic and its order are unchanged, so the table stays bit-identical to
// the oracle's.
constexpr int kPolyThreads = 128;
__global__ void __launch_bounds__(kPolyThreads)
    leg_poly_kernel(int T, int nh, int lm0, const int32_t* __restrict__ lm_m, const int32_t* __restrict__ lm_i0,
                    const int64_t* __restrict__ lm_poff, const int32_t* __restrict__ lm_kp,
                    const double* __restrict__ mu, const double* __restrict__ dmant, const int32_t* __restrict__ dexp,
                    double* __restrict__ ptab) {
  __shared__ double tile[kPolyThreads / 32][32][33];
  const int lm = lm0 + blockIdx.y;
  const int m = lm_m[lm];
  const int i0 = lm_i0[lm];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int ring0 = i0 + blockIdx.x * kPolyThreads + wp * 32;  // first ring of this warp
  if (ring0 >= nh) return;
  const int i = ring0 + lane;
  const bool live = i < nh;
  const int kp = lm_kp[lm], K = T - m + 1;
  double* rows = ptab + lm_poff[lm] + (int64_t)(ring0 - i0) * kp;
  const int nrow = min(32, nh - ring0);
  const double x = live ? mu[i] : 0.0;
  const double two400 = 0x1p400, twom400 = 0x1p-400;
  int e = live ? dexp[(int64_t)lm * nh + i] : 0;
  double q2 = live ? dmant[(int64_t)lm * nh + i] : 0.0;
  double q1 = 0.0, epsm1 = 0.0;
  double (*tl)[33] = tile[wp];
  for (int c0 = 0; c0 < kp; c0 += 32) {
    const double eps_l = (c0 + lane >= 1 && c0 + lane < K) ? eps_nm(m + c0 + lane, m) : 0.0;  // column c0 + lane
    for (int cc = 0; cc < 32; ++cc) {  // column c = n - m of this lane's ring
      const int c = c0 + cc;
      const double eps_c = __shfl_sync(0xffffffffu, eps_l, cc);
      double v = 0.0;  // zero padding beyond K (the scratch is reused in recompute mode)
      if (c == 0) {
        v = ldexp(q2, e);
      } else if (c == 1 && c < K) {
        q1 = __dmul_rn(__dmul_rn(sqrt(2.0 * m + 3.0), x), q2);
        epsm1 = eps_c;  // eps(m + 1, m)
        v = ldexp(q1, e);
      } else if (c < K) {
        const double epsn = eps_c;  // eps(m + c, m)
        double q = __ddiv_rn(__dsub_rn(__dmul_rn(x, q1), __dmul_rn(epsm1, q2)), epsn);
        if (fabs(q) > two400) {
          q = __dmul_rn(q, twom400);
          q1 = __dmul_rn(q1, twom400);
          e += 400;
        }
        q2 = q1;
        q1 = q;
        epsm1 = epsn;
        v = ldexp(q, e);
      }
      tl[lane][cc] = v;
    }
    __syncwarp();
    const int ncol = min(32, kp - c0);
    if (lane < ncol)
      for (int r = 0; r < nrow; ++r) rows[(int64_t)r * kp + c0 + lane] = tl[r][lane];
    __syncwarp();
  }
}

}  // namespace

size_t leg_inv_smem() { return (size_t)kInvStages * kInvStageDbl * sizeof(double); }
size_t leg_dir_smem() { return (size_t)kDirStages * kDirStageDbl * sizeof(double); }

void launch_leg_inv(const LegParams& p, const double* spec, double* four, int grid, cudaStream_t s) {
  // the attribute is per device: set it once for every device a plan runs on
  static uint64_t done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64 || !(done >> dev & 1)) {
    cudaFuncSetAttribute(leg_inv_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)leg_inv_smem());
    cudaFuncSetAttribute(leg_inv_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)leg_inv_smem());
    cudaFuncSetAttribute(leg_inv_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)leg_inv_smem());
    cudaFuncSetAttribute(leg_inv_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)leg_inv_smem());
    if (dev < 64) done |= 1ull << dev;
  }
  const bool blk = p.fsh == 6;
  auto k = p.stage ? (blk ? leg_inv_kernel<true, true> : leg_inv_kernel<true, false>)
                   : (blk ? leg_inv_kernel<false, true> : leg_inv_kernel<false, false>);
  k<<<grid, kInvThreads, leg_inv_smem(), s>>>(p, spec, four);
}

void launch_leg_dir(const LegParams& p, const double* four, double* spec, int grid, cudaStream_t s) {
  // the attribute is per device: set it once for every device a plan runs on
  static uint64_t done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64 || !(done >> dev & 1)) {
    cudaFuncSetAttribute(leg_dir_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)leg_dir_smem());
    if (dev < 64) done |= 1ull << dev;
  }
  leg_dir_kernel<<<grid, kDirThreads, leg_dir_smem(), s>>>(p, four, spec);
}

void leg_preload() {  // see fft_preload
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, leg_inv_kernel<false, false>);
  cudaFuncGetAttributes(&a, leg_inv_kernel<true, false>);
  cudaFuncGetAttributes(&a, leg_inv_kernel<false, true>);
  cudaFuncGetAttributes(&a, leg_inv_kernel<true, true>);
  cudaFuncGetAttributes(&a, leg_dir_kernel);
  cudaFuncGetAttributes(&a, leg_poly_kernel);
  cudaFuncGetAttributes(&a, leg_diag_kernel);
}

void launch_leg_diag(int T, int nh, int nlm, const int32_t* lm_m, const double* sint, double* dmant, int32_t* dexp,
                     cudaStream_t s) {
  if (nlm == 0) return;
  leg_diag_kernel<<<(nh + 127) / 128, 128, 0, s>>>(T, nh, sint, nlm, lm_m, dmant, dexp);
}

void launch_leg_poly(int T, int nh, int lm0, int lm1, const int32_t* lm_m, const int32_t* lm_i0,
                     const int64_t* lm_poff, const int32_t* lm_kp, const double* mu, const double* dmant,
                     const int32_t* dexp, double* ptab, cudaStream_t s) {
  if (lm1 <= lm0) return;
  dim3 grid((nh + kPolyThreads - 1) / kPolyThreads, lm1 - lm0);
  leg_poly_kernel<<<grid, kPolyThreads, 0, s>>>(T, nh, lm0, lm_m, lm_i0, lm_poff, lm_kp, mu, dmant, dexp, ptab);
}

}  // namespace sht

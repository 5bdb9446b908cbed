// Internal declarations shared by the host plan (sht_plan.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sht.h"

namespace sht {

#ifdef __CUDACC__
// One Fourier-row field slot {S.re, S.im, A.re, A.im} as a single 32-byte
// access (sm_100 256-bit LDG/STG): full sectors, also over NVLink when the
// row lives in a peer GPU's buffer.
__device__ __forceinline__ void st_slot(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
// (not volatile, no memory clobber: a read of data no kernel writes while it
// runs, so the compiler may batch several of them before their first use)
__device__ __forceinline__ void ld_slot(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
      : "l"(p));
}
#endif

// ---------------------------------------------------------------- error state
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define SHT_CUDA_TRY(expr)                                                                            \
  do {                                                                                               \
    cudaError_t _e = (expr);                                                                         \
    if (_e != cudaSuccess)                                                                           \
      return ::sht::fail(SHT_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));         \
  } while (0)

// ---------------------------------------------------------------- Legendre GEMM tiling
// leg_inv: CTA tile = 64 northern rings x 64 fields, k-chunk = 64 wavenumbers n.
// leg_dir: CTA tile = 128 wavenumbers n x 64 fields, k-chunk = 32 rings.
constexpr int kLegFields = 64;
constexpr int kInvRings = 64;
constexpr int kInvKc = 64;
constexpr int kDirN = 128;
constexpr int kDirKc = 32;
constexpr int kStageSlots = 2;  // leg_inv pusher epilogue: staging slots per CTA
// Fourier-row buffers (X, Y): field slot f (S.re, S.im, A.re, A.im) of row
// `row` sits at base + (f >> fsh) * bs + row * row_ld + (f & fmask) * 4.
// Classic layout (P = 1, NCCL): one row holds every field (row_ld = 4 nfld,
// fsh = 30).  Field-blocked layout (p2p, P > 1): [64-field block][row][64][4]
// (row_ld = kRowDbl, fsh = 6, bs = rows x kRowDbl): a ring's rows are 2 KB
// apart in each block, which keeps the remote footprint of the scattered
// NVLink row stores small (profiles/r02_transport_cliff.md).
constexpr int kRowDbl = kLegFields * 4;
constexpr int kPtabPad = 64;  // P-table rows are padded (with zeros) to a multiple of this

struct LegTile {  // one output tile of a Legendre GEMM
  int32_t lm;     // local wavenumber index
  int32_t r0;     // leg_inv: first northern ring; leg_dir: first n-m offset
  int32_t f0;     // first field
  int32_t pad;    // leg_inv with LegParams::stage: 1 if a ring of the tile is owned by a peer
};

struct LegParams {
  int T, nh, nfld;
  int nlm;                   // number of local wavenumbers
  const int32_t* lm_m;       // [nlm] m of each local wavenumber
  const int32_t* lm_i0;      // [nlm] first northern ring with M_i >= m
  const int64_t* lm_poff;    // [nlm] P-table offset (doubles) of (ring i0, n = m)
  const int32_t* lm_kp;      // [nlm] padded P-table row length
  const int64_t* lm_soff;    // [nlm] complex offset of (m, n = m) in the local spectral field
  int64_t spec_ld;           // doubles per local spectral field
  const int32_t* xbase;      // [nh] Fourier row of (ring i, lm = 0) in the m-side buffer (leg_dir)
  double* const* ring_out;   // [nh] leg_inv: row of (ring i, lm = 0), field block 0, in the ring owner's receive buffer
  const int64_t* ring_bs;    // [nh] field-block stride (doubles) of that buffer
  int64_t xbs;               // leg_dir: field-block stride of X
  int64_t row_ld;            // doubles between consecutive rows (of one field block)
  int fsh, fmask;            // field f -> block f >> fsh, slot f & fmask
  double* stage;             // leg_inv: [grid][2][64 rings][64 fields][4] staging slots of the
                             // pusher epilogue (p2p, P > 1), or nullptr
  const double* ptab;        // P table
  const LegTile* tiles;
  int ntiles;
  int* counter;              // persistent-scheduler ticket
  int debug;                 // profiling only (SHT_LEG_DEBUG): bit 0 skips operand loads, bit 1 skips DMMA
};

void launch_leg_inv(const LegParams& p, const double* spec, double* four, int grid, cudaStream_t s);
void launch_leg_dir(const LegParams& p, const double* four, double* spec, int grid, cudaStream_t s);
// P_m^m start values (X-numbers) of every local wavenumber on every ring.
void launch_leg_diag(int T, int nh, int nlm, const int32_t* lm_m, const double* sint, double* dmant, int32_t* dexp,
                     cudaStream_t s);
// P table rows of local wavenumbers [lm0, lm1) at ptab + lm_poff[lm].
void launch_leg_poly(int T, int nh, int lm0, int lm1, const int32_t* lm_m, const int32_t* lm_i0,
                     const int64_t* lm_poff, const int32_t* lm_kp, const double* mu, const double* dmant,
                     const int32_t* dexp, double* ptab, cudaStream_t s);
size_t leg_inv_smem();
void leg_preload();  // load every kernel of the file now (no lazy load inside a transform)
size_t leg_dir_smem();

// ---------------------------------------------------------------- ring FFTs
constexpr int kMaxSteps = 4;                       // pencil steps per transform (ring or Bluestein inner)
constexpr int kFftMaxLen = 8192;                   // longest ring one CTA handles
constexpr int kTwMax = 448;                        // per-ring twiddle-table entries (shared memory)
constexpr int kMaxAllStepsHost = 3 * 4;           // ring steps + inner steps of up to two Bluestein steps

// One step of the in-place "pencil" FFT of length L = R_0 R_1 ... R_{d-1}:
// blocks of length B = R_j S, each holding S pencils of R points at stride S.
// A Bluestein step (prime R > 31) computes its DFT_R pencils as chirp-z
// convolutions of length Lp in a work buffer, G pencils at a time, with the
// inner FFT steps inner0 .. inner0 + ninner - 1.
struct FftStep {
  int32_t R;           // pencil length (radix)
  int32_t S;           // pencil stride = B / R
  int32_t B;           // block length
  int32_t np;          // pencils per sequence = L / R
  int32_t tmul;        // twiddle W_B^(r s) = W^(r s tmul) of the owning transform's table
  int32_t tw_base;     // offset of that transform's 2-level table (lo[64], hi[...]) in the ring table
  uint64_t mag_S, mag_np, mag_R;  // multiply-shift (>> 40) divisors
  // Bluestein step only (blue != 0)
  int32_t blue, Lp, inner0, ninner, G;
  int32_t ptab;        // DMMA prime step (R prime, 17..kMaxDmmaPrime, last step): offset of the
                       // (cos, sin)(2 pi r / R) table in the ring table; -1 otherwise
  uint64_t mag_Lp, mag_Rb;  // divisors by Lp and by R
  int64_t chirp_off;   // w_r = exp(-pi i r^2 / R), r < R
  int64_t bhat_off;    // inner-FFT spectrum of the chirp kernel / Lp, digit-reversed for the inner plan
};

struct FftRing {       // one northern ring (and its southern mirror) on this rank
  int32_t n;           // points on the ring
  int32_t L;           // transform length: n, or the whole-ring Bluestein length
  int32_t mcap;        // M_i
  int32_t nstep;
  int32_t step0;       // first step in FftParams::steps
  int32_t nb;          // fields (= complex sequences, north + i south) per batch
  int32_t variant;
  int32_t wlen;        // Bluestein work-buffer length (complex), 0 if none
  uint64_t mag_N, mag_M1, mag_L;  // multiply-shift (>> 40) divisors for n, mcap + 1, L
  int64_t chirp_off;   // whole-ring Bluestein: chirp w_n (n < N) in the arena, -1 if none
  int64_t bhat_off;    // whole-ring Bluestein: kernel spectrum / L, digit-reversed
  int64_t goff_n;      // offset of the northern ring in the local grid field
  int64_t goff_s;      // offset of the southern ring in the local grid field
  int64_t yrow_off;    // offset into yrow[] of this ring's (M_i + 1) Fourier rows
  int64_t tw_off;      // arena offset of this ring's twiddle table (ntw entries)
  int64_t dit_off;     // offset of this ring's digit-reversed positions (N entries) in FftParams::ditpos, -1 if none
  int32_t ntw;
  int32_t shift;       // pruned whole-ring Bluestein: bins k > M of the spectrum sit at k + L - N (else 0)
  double w;            // Gaussian weight
};

struct FftWork {       // one CTA: fields [f0, f1) of one ring pair
  int32_t ring;
  int32_t f0;
  int32_t f1;
  int32_t pad;
};

struct FftParams {
  int nfld;
  int64_t grid_ld;           // doubles per local grid field
  const FftRing* rings;
  const FftStep* steps;
  const FftWork* work;
  const double2* tw;         // twiddle / chirp arena
  const int32_t* ditpos;     // per non-Bluestein ring: position of spectrum bin k after the DIT steps
  double* const* rows_out;   // g2f: Fourier row (field block 0) of (ring, m) in the m-owner's receive buffer
  const int64_t* rows_out_bs;    // its field-block stride (doubles)
  const double* const* rows_in;  // f2g: Fourier row (field block 0) of (ring, m) in this rank's receive buffer
  int64_t in_bs;                 // field-block stride of that buffer
  int fsh, fmask;                // field f -> block f >> fsh, slot f & fmask
  int debug;                 // profiling only (SHT_FFT_DEBUG): bit 0 skips the DFT steps
};

// Ring-FFT launch classes: 1 = 256 threads, <= 100 KB of shared memory
// (2 CTAs/SM); 3 = 512 threads, up to 212 KB (1 CTA/SM); 2 is unused.
constexpr int kFftVariants = 4;  // index 0 unused
void fft_preload();  // load every kernel of the file now (no lazy load inside a transform)
void fft_preload_blk();  // the field-blocked-layout kernels (sht_fft_blk.cu)
void launch_fft_blk(bool g2f, int variant, const FftParams& p, int w0, int nw, const double* in, double* out,
                    size_t smem, cudaStream_t s);
void launch_fft(bool g2f, int variant, const FftParams& p, int w0, int nw, const double* in, double* out,
                size_t smem, cudaStream_t s);

// Host plan of one ring length: steps (with Bluestein inner steps appended)
// and the ring's twiddle / chirp tables appended to the arena.
constexpr int kMaxDmmaPrime = 127;  // largest prime DFT done as FP64 tensor-core GEMMs (last step)
struct RingPlan {
  int variant = 1;
  int dprime = 0;              // a prime factor 17..kMaxDmmaPrime as a DMMA prime step (last step), else 0
  bool bluestein = false;      // a prime factor > kMaxDmmaPrime, or two prime factors > 16
  bool ring_blue = false;      // whole-ring Bluestein (transform length L fits one CTA)
  int L = 0;                   // transform length
  int mcap = -1;               // pruned whole-ring Bluestein (even n): only |k| <= mcap is kept,
  int shift = 0;               //   so L >= n + 2 mcap suffices; negative bins at L - |k| (shift = L - n)
  std::vector<int> radices;    // steps (factor-local Bluestein primes last)
  int wlen = 0;                // factor-local Bluestein: work buffer per pencil (Lp)
};
constexpr int kWholeBluesteinMax = 12288;  // longest whole-ring Bluestein transform (212 KB class: 1 CTA per SM)
constexpr int kWholeBluesteinPair = 6022;  // longest one whose buffer fits 100 KB (two CTAs per SM)
// mcap >= 0: the transform only needs / only feeds the wavenumbers |k| <= mcap
int fft_plan_ring(int n, RingPlan& rp, int mcap = -1);
// Appends the ring's steps (and inner steps) to `steps`, its tables to `arena`.
int fft_build_ring(int n, const RingPlan& rp, int G, std::vector<FftStep>& steps, std::vector<double2>& arena,
                   int64_t& tw_off, int& ntw, int64_t& chirp_off, int64_t& bhat_off);
// Position of DFT output k after the in-place DIT pencil FFT (digit reversal).
int fft_pos(int k, const std::vector<int>& radices);
// Shared-memory complex slots for n FFT points (one pad slot per 16 against bank conflicts).
__host__ __device__ inline size_t fft_slots(size_t n) { return n + n / 16 + 1; }
// Smallest 13-smooth length >= lo whose pencil plan has <= kMaxSteps steps.
int fft_bluestein_len(int lo, std::vector<int>& radices, int lmax);

// ---------------------------------------------------------------- 2-D grid-point layout (sht_gp.cu)
struct GpLayout {
  int nA = 0, nB = 0;                  // latitude bands x longitude segments (0: not set)
  std::vector<int> band_lo;            // [nA + 1] first global ring of every band
  int64_t npts_gp = 0;                 // grid-point-layout points of this rank per field
  std::vector<int32_t> send_idx;       // ring layout -> GP: my ring-layout index per point, by destination
  std::vector<int64_t> send_displ;     // [P + 1]
  std::vector<int32_t> recv_idx;       // my GP-layout index per incoming point, by source
  std::vector<int64_t> recv_displ;     // [P + 1]
};
void gp_bands(const std::vector<int>& nloen, int nA, std::vector<int>& band_lo);
int gp_build(const std::vector<int>& nloen, const std::vector<int>& ring_rank, int P, int rank, int nA, int nB,
             GpLayout& L);
void gp_launch_pack(const double* src, int64_t src_ld, const int32_t* idx, const int64_t* displ, int P, int64_t ntot,
                    int nfld, double* buf, cudaStream_t s);
void gp_launch_unpack(const double* buf, const int32_t* idx, const int64_t* displ, int P, int64_t ntot, int nfld,
                      double* dst, int64_t dst_ld, cudaStream_t s);
void gp_preload();

}  // namespace sht

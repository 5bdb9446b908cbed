// Internal declarations shared by the host plan (sht_plan.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sht.h"

namespace sht {

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
constexpr int kPtabPad = 64;  // P-table rows are padded (with zeros) to a multiple of this

struct LegTile {  // one output tile of a Legendre GEMM
  int32_t lm;     // local wavenumber index
  int32_t r0;     // leg_inv: first northern ring; leg_dir: first n-m offset
  int32_t f0;     // first field
  int32_t pad;
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
  const int32_t* xbase;      // [nh] Fourier row of (ring i, lm = 0) in the m-side buffer
  const double* ptab;        // P table
  const LegTile* tiles;
  int ntiles;
  int* counter;              // persistent-scheduler ticket
  int debug;                 // profiling only (SHT_LEG_DEBUG): bit 0 skips operand loads, bit 1 skips DMMA
};

void launch_leg_inv(const LegParams& p, const double* spec, double* four, int grid, cudaStream_t s);
void launch_leg_dir(const LegParams& p, const double* four, double* spec, int grid, cudaStream_t s);
void launch_leg_poly(int T, int nh, int nlm, const int32_t* lm_m, const int32_t* lm_i0, const int64_t* lm_poff,
                     const int32_t* lm_kp, const double* mu, const double* sint, double* dmant, int32_t* dexp,
                     double* ptab, cudaStream_t s);
size_t leg_inv_smem();
size_t leg_dir_smem();

// ---------------------------------------------------------------- ring FFTs
constexpr int kMaxPasses = 8;
constexpr int kFftMaxLen = 6912;   // longest transform one CTA handles (ping-pong buffers in smem)

struct FftPass {       // one Stockham pass of a ring plan
  int32_t radix;
  int32_t ns;          // span: product of the radices already applied
  int32_t nbf;         // butterflies per sequence = L / radix
  int32_t pad;
  uint64_t mag_nbf;    // multiply-shift (>> 40) divisors for nbf and ns
  uint64_t mag_ns;
  int32_t tstride;     // L / (ns radix): base twiddle of butterfly k is W_L^(k tstride)
  int32_t pad2;
};

constexpr int kTwLo = 64;                          // two-level twiddle table: W_L^e = hi[e / 64] lo[e % 64]
constexpr int kTwHi = (6912 + kTwLo - 1) / kTwLo;  // entries of hi for the longest transform

struct FftRing {       // one northern ring (and its southern mirror) on this rank
  int32_t n;           // points on the ring
  int32_t L;           // transform length (n, or the Bluestein length)
  int32_t mcap;        // M_i
  int32_t npass;
  int32_t pass0;       // first pass in FftParams::passes
  int32_t fp;          // field pairs per CTA
  int32_t nb;          // sequences per FFT batch
  int32_t pad;
  uint64_t mag_L, mag_N, mag_M1;  // multiply-shift (>> 40) divisors for L, n, mcap + 1
  int64_t chirp_off;   // Bluestein chirp w_n = exp(-pi i n^2 / N), n < N   (-1: none)
  int64_t bhat_off;    // Bluestein kernel spectrum / L                     (-1: none)
  int64_t goff_n;      // offset of the northern ring in the local grid field
  int64_t goff_s;      // offset of the southern ring in the local grid field
  int64_t yrow_off;    // offset into yrow[] of this ring's (M_i + 1) Fourier rows
  int64_t tw2_off;     // arena offset of lo[0..63] = W_L^e, then hi[h] = W_L^(64 h), h < ceil(L/64)
  double w;            // Gaussian weight
};

struct FftWork {       // one CTA of a ring-FFT launch
  int32_t ring;        // local ring index
  int32_t fp0;         // first field pair
};

struct FftParams {
  int nfld;
  int64_t grid_ld;           // doubles per local grid field
  const FftRing* rings;
  const FftPass* passes;
  const FftWork* work;
  const double2* tw;         // twiddle / chirp arena
  const int32_t* yrow;       // Fourier row of (ring, m)
  int debug;                 // profiling only (SHT_FFT_DEBUG): bit 0 skips the DFT passes
};

// Launch CTAs work[w0 .. w0+nw) of a ring-FFT class.  variant 0: radix <= 16,
// 256 threads, 2 CTAs/SM; 1: radix <= 16, 512 threads; 2: prime radices up to
// 31, 256 threads.  g2f: grid -> Fourier (in = grid), else Fourier -> grid.
void launch_fft(bool g2f, int variant, const FftParams& p, int w0, int nw, const double* in, double* out,
                size_t smem, cudaStream_t s);
// Complex values one in-place pass of `variant` can hold for these radices.
int fft_capacity(int variant, const std::vector<int>& radices);
// Plan for a ring of n points: mixed radix (composite <= 16, primes <= 31)
// when n factors over those, else Bluestein with a 13-smooth L >= 2n-1.
int fft_choose(int n, std::vector<int>& radices, int& L, bool& bluestein);
// Same with composite radices capped at `cap` (16, or 8 for the 1024-thread variant).
int fft_choose(int n, int cap, std::vector<int>& radices, int& L, bool& bluestein);
bool fft_needs_big(const std::vector<int>& radices);
void fft_passes(int L, const std::vector<int>& radices, std::vector<FftPass>& out, std::vector<double2>& arena,
                int64_t& tw2_off);

}  // namespace sht

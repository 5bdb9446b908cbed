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
#include "fft_kernels.cuh"

namespace sht {

// Loads every FFT kernel now (cudaFuncGetAttributes forces the lazy module
// load): a first launch inside a transform could otherwise block behind a
// kernel spinning on a dead peer.
void fft_preload() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, fft_g2f_kernel<1, false>);
  cudaFuncGetAttributes(&a, fft_f2g_kernel<1, false>);
  cudaFuncGetAttributes(&a, fft_g2f_kernel<3, false>);
  cudaFuncGetAttributes(&a, fft_f2g_kernel<3, false>);
  fft_preload_blk();
}

void launch_fft(bool g2f, int variant, const FftParams& p, int w0, int nw, const double* in, double* out,
                size_t smem, cudaStream_t s) {
  if (nw <= 0) return;
  if (p.fsh == 6) return launch_fft_blk(g2f, variant, p, w0, nw, in, out, smem, s);
  if (variant == 1) launch_one<1, false>(g2f, p, w0, nw, in, out, smem, s);
  if (variant == 3) launch_one<3, false>(g2f, p, w0, nw, in, out, smem, s);
}

// ------------------------------------------------------------------ host-side planning
static bool factor_primes(int n, int maxp, std::vector<int>& primes) {
  primes.clear();
  int m = n;
  for (int p = 2; p <= maxp && m > 1; ++p)
    while (m % p == 0) {
      primes.push_back(p);
      m /= p;
    }
  return m == 1;
}

// Pencil radices: primes > 16 alone, the rest multiplied into factors <= 16
// (first-fit decreasing), as few steps as possible.
static void group_pencils(const std::vector<int>& primes, std::vector<int>& radices) {
  radices.clear();
  std::vector<int> small;
  for (int p : primes) (p > 16 ? radices : small).push_back(p);
  std::sort(small.begin(), small.end(), std::greater<int>());
  std::vector<int> bins;
  for (int p : small) {
    bool placed = false;
    for (int& b : bins)
      if (b * p <= 16) {
        b *= p;
        placed = true;
        break;
      }
    if (!placed) bins.push_back(p);
  }
  radices.insert(radices.end(), bins.begin(), bins.end());
}

// Modelled cost of a Bluestein convolution of length L with pencil radices
// `rad` (forward DIT + transposed pass): per pencil the codelet's FP64
// instructions (SASS count of tools/gen_codelets.py output), the twiddle
// recurrence (8R - 8, every step but the last) and ~8 instructions of
// addressing / shared-memory traffic per point.
static int64_t bluestein_cost(int L, const std::vector<int>& rad) {
  static const int kCodelet[17] = {0, 0, 4, 12, 16, 36, 44, 66, 55, 88, 108, 150, 128, 204, 184, 200, 165};
  int64_t c = 0;
  const int n = (int)rad.size();
  for (int j = 0; j < n; ++j) {
    const int R = rad[j];
    const int64_t pen = L / R;
    c += pen * (2LL * kCodelet[R] + 16LL * R);
    if (j < n - 1) c += pen * 2LL * (8 * R - 8);
  }
  return c;
}

// Bluestein length for a convolution spanning `lo` lags: the 13-smooth
// length in [lo, min(lmax, 3 lo / 2)] with <= kMaxSteps pencil steps and the
// least modelled cost (a power-of-16 length often beats the shortest one);
// else the shortest such length up to min(lmax, 4 lo + 64); -1 if none.
int fft_bluestein_len(int lo, std::vector<int>& radices, int lmax) {
  std::vector<int> primes, rad;
  int best = -1;
  int64_t best_cost = 0;
  for (int cand = lo; cand <= std::min(lmax, lo + lo / 2); ++cand)
    if (factor_primes(cand, 13, primes)) {
      group_pencils(primes, rad);
      if ((int)rad.size() > kMaxSteps) continue;
      const int64_t c = bluestein_cost(cand, rad);
      if (best < 0 || c < best_cost) {
        best = cand;
        best_cost = c;
        radices = rad;
      }
    }
  if (best > 0) return best;
  for (int cand = lo; cand <= std::min(lmax, 4 * lo + 64); ++cand)
    if (factor_primes(cand, 13, primes)) {
      group_pencils(primes, radices);
      if ((int)radices.size() <= kMaxSteps) return cand;
    }
  return -1;
}

int fft_plan_ring(int n, RingPlan& rp, int mcap) {
  if (n < 2 || n > kFftMaxLen) return SHT_ERR_CONFIG;
  std::vector<int> primes, small, mid, big;
  factor_primes(n, n, primes);
  for (int p : primes) (p <= 16 ? small : p <= kMaxDmmaPrime ? mid : big).push_back(p);
  rp.variant = 1;
  rp.dprime = 0;
  rp.ring_blue = false;
  rp.L = n;
  rp.wlen = 0;
  rp.mcap = -1;
  rp.shift = 0;
  // direct: pencils <= 16 plus at most one prime 17..kMaxDmmaPrime as a DMMA
  // prime step (last), <= kMaxSteps steps in all
  if (big.empty() && mid.size() <= 1) {
    group_pencils(small, rp.radices);
    if (!mid.empty()) rp.radices.push_back(mid[0]);
    if (rp.radices.empty()) rp.radices.push_back(n);
    if ((int)rp.radices.size() <= kMaxSteps && (mid.empty() || rp.radices.size() >= 2)) {
      rp.bluestein = false;
      rp.dprime = mid.empty() ? 0 : mid[0];
      return SHT_OK;
    }
  }
  rp.bluestein = true;
  for (int p : mid) big.push_back(p);
  std::sort(big.begin(), big.end());
  {  // whole-ring Bluestein when the padded transform fits one CTA
    // Chirp-z convolution between n points and the 2 mcap + 1 kept bins
    // spans n + 2 mcap lags (the chirp is n-periodic for even n), not 2n - 1.
    const bool pruned = mcap >= 0 && n % 2 == 0 && n + 2 * mcap < 2 * n - 1;
    std::vector<int> rad;
    // prefer lengths that keep two CTAs per SM (<= 6022 points in 100 KB)
    const int lo = pruned ? n + 2 * mcap : 2 * n - 1;
    int L = fft_bluestein_len(lo, rad, kWholeBluesteinPair);
    if (L < 0) L = fft_bluestein_len(lo, rad, kWholeBluesteinMax);
    if (L > 0 && L <= kWholeBluesteinMax) {
      rp.ring_blue = true;
      rp.L = L;
      rp.radices = rad;
      if (pruned) {
        rp.mcap = mcap;
        rp.shift = L - n;
      }
      return SHT_OK;
    }
  }
  group_pencils(small, rp.radices);
  int maxLp = 0;
  for (int p : big) {
    rp.radices.push_back(p);  // factor-local Bluestein steps last (contiguous pencils)
    std::vector<int> inner;
    const int Lp = fft_bluestein_len(2 * p - 1, inner, kFftMaxLen);
    if (Lp < 0) return SHT_ERR_CONFIG;
    maxLp = std::max(maxLp, Lp);
  }
  rp.wlen = maxLp;  // per pencil; times G by the caller
  if (rp.radices.empty()) rp.radices.push_back(n);
  if ((int)rp.radices.size() > kMaxSteps || (int)big.size() > 2) return SHT_ERR_CONFIG;
  return SHT_OK;
}

int fft_pos(int k, const std::vector<int>& radices) {
  int S = 1;
  for (int R : radices) S *= R;
  int pos = 0;
  for (int R : radices) {
    S /= R;
    pos += (k % R) * S;
    k /= R;
  }
  return pos;
}

static void push_table(std::vector<double2>& arena, int L) {
  const long double two_pi = 6.283185307179586476925286766559005768L;
  auto W = [&](long long e) {
    const long double a = -two_pi * (long double)(e % L) / (long double)L;
    return make_double2((double)cosl(a), (double)sinl(a));
  };
  for (int e = 0; e < 64; ++e) arena.push_back(W(e));
  for (int h = 0; h < (L + 63) / 64; ++h) arena.push_back(W(64LL * h));
}

static FftStep make_step(int L, int B, int R, int tw_base) {
  FftStep st{};
  st.R = R;
  st.B = B;
  st.S = B / R;
  st.np = L / R;
  st.tmul = L / B;
  st.tw_base = tw_base;
  st.mag_S = ((uint64_t)1 << 40) / (uint64_t)st.S + 1;
  st.mag_np = ((uint64_t)1 << 40) / (uint64_t)st.np + 1;
  st.mag_R = ((uint64_t)1 << 40) / (uint64_t)R + 1;
  st.chirp_off = st.bhat_off = -1;
  st.ptab = -1;
  return st;
}

void dft_host(const std::vector<std::complex<long double>>& in, std::vector<std::complex<long double>>& out);

int fft_build_ring(int n, const RingPlan& rp, int G, std::vector<FftStep>& steps, std::vector<double2>& arena,
                   int64_t& tw_off, int& ntw, int64_t& chirp_off, int64_t& bhat_off) {
  typedef std::complex<long double> cld;
  const long double pi_ld = 3.14159265358979323846264338327950288L;
  const int L = rp.L;
  tw_off = (int64_t)arena.size();
  push_table(arena, L);  // ring (or whole-ring Bluestein) table at base 0
  const size_t first = steps.size();
  std::vector<FftStep> ring;
  int B = L;
  for (int R : rp.radices) {
    ring.push_back(make_step(L, B, R, 0));
    B /= R;
  }
  chirp_off = bhat_off = -1;
  if (rp.ring_blue) {
    ntw = (int)((int64_t)arena.size() - tw_off);
    std::vector<cld> chirp(n);
    for (int k = 0; k < n; ++k) {
      const long long qq = ((long long)k * k) % (2LL * n);
      const long double a = -pi_ld * (long double)qq / (long double)n;
      chirp[k] = cld(cosl(a), sinl(a));
    }
    chirp_off = (int64_t)arena.size();
    for (int k = 0; k < n; ++k) arena.push_back(make_double2((double)chirp[k].real(), (double)chirp[k].imag()));
    // ChirpWalk factors: g_t = exp(-i pi (512 t + 65536) / n), t < 256, then h = exp(-i pi 131072 / n)
    auto cis_n = [&](long long num) {
      const long double a = -pi_ld * (long double)(num % (2LL * n)) / (long double)n;
      return make_double2((double)cosl(a), (double)sinl(a));
    };
    for (int t = 0; t < 256; ++t) arena.push_back(cis_n(512LL * t + 65536LL));
    arena.push_back(cis_n(131072LL));
    // kernel b_j = conj(chirp_j) at lag j mod L: |j| < n, or (pruned)
    // j in [-(n + mcap - 1), mcap]
    std::vector<cld> b(L, cld(0)), bh;
    const long long jlo = rp.mcap >= 0 ? -(long long)(n + rp.mcap - 1) : -(long long)(n - 1);
    const long long jhi = rp.mcap >= 0 ? rp.mcap : n - 1;
    for (long long j = jlo; j <= jhi; ++j) {
      const long long qq = (j * j) % (2LL * n);
      const long double a = pi_ld * (long double)qq / (long double)n;
      b[(size_t)((j % L + L) % L)] = cld(cosl(a), sinl(a));
    }
    dft_host(b, bh);
    std::vector<double2> perm(L);
    for (int k = 0; k < L; ++k) {
      const cld v = bh[k] / (long double)L;
      perm[fft_pos(k, rp.radices)] = make_double2((double)v.real(), (double)v.imag());
    }
    bhat_off = (int64_t)arena.size();
    arena.insert(arena.end(), perm.begin(), perm.end());
    steps.insert(steps.end(), ring.begin(), ring.end());
    while (steps.size() < first + kMaxAllStepsHost) steps.push_back(FftStep{});
    return ntw > kTwMax ? SHT_ERR_CONFIG : SHT_OK;
  }
  // inner plans of the Bluestein steps (their tables follow the ring table)
  std::vector<FftStep> inner;
  std::vector<std::pair<size_t, std::vector<int>>> blue_inner;  // ring-step index, inner radices
  for (size_t j = 0; j < ring.size(); ++j) {
    FftStep& st = ring[j];
    if (st.R <= 16 || rp.dprime) continue;  // a direct plan's prime > 16 is its DMMA prime step
    std::vector<int> irad;
    const int Lp = fft_bluestein_len(2 * st.R - 1, irad, kFftMaxLen);
    const int base = (int)((int64_t)arena.size() - tw_off);
    push_table(arena, Lp);
    st.blue = 1;
    st.Lp = Lp;
    st.G = G;
    st.inner0 = (int)(rp.radices.size() + inner.size());
    st.ninner = (int)irad.size();
    st.mag_Lp = ((uint64_t)1 << 40) / (uint64_t)Lp + 1;
    st.mag_Rb = ((uint64_t)1 << 40) / (uint64_t)st.R + 1;
    int Bi = Lp;
    for (int Ri : irad) {
      inner.push_back(make_step(Lp, Bi, Ri, base));
      Bi /= Ri;
    }
    blue_inner.push_back({j, irad});
  }
  if (rp.dprime) {  // (cos, sin)(2 pi r / p) of the DMMA prime step, after the ring table
    const int P = rp.dprime;
    ring.back().ptab = (int)((int64_t)arena.size() - tw_off);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (int r = 0; r < P; ++r) {
      const long double a = two_pi * (long double)r / (long double)P;
      arena.push_back(make_double2((double)cosl(a), (double)sinl(a)));
    }
  }
  ntw = (int)((int64_t)arena.size() - tw_off);
  if (ntw > kTwMax || ring.size() + inner.size() > (size_t)kMaxAllStepsHost) return SHT_ERR_CONFIG;
  // chirp and kernel spectrum of each Bluestein step (global arena, offsets absolute)
  for (auto& bi : blue_inner) {
    FftStep& st = ring[bi.first];
    const int P = st.R, Lp = st.Lp;
    std::vector<cld> chirp(P);
    for (int r = 0; r < P; ++r) {
      const long long qq = ((long long)r * r) % (2LL * P);
      const long double a = -pi_ld * (long double)qq / (long double)P;
      chirp[r] = cld(cosl(a), sinl(a));
    }
    st.chirp_off = (int64_t)arena.size();
    for (int r = 0; r < P; ++r) arena.push_back(make_double2((double)chirp[r].real(), (double)chirp[r].imag()));
    std::vector<cld> b(Lp, cld(0)), bh;
    for (int r = 0; r < P; ++r) {
      b[r] = std::conj(chirp[r]);
      if (r) b[Lp - r] = std::conj(chirp[r]);
    }
    dft_host(b, bh);
    std::vector<double2> perm(Lp);
    for (int k = 0; k < Lp; ++k) {
      const cld v = bh[k] / (long double)Lp;
      perm[fft_pos(k, bi.second)] = make_double2((double)v.real(), (double)v.imag());
    }
    st.bhat_off = (int64_t)arena.size();
    arena.insert(arena.end(), perm.begin(), perm.end());
  }
  steps.insert(steps.end(), ring.begin(), ring.end());
  steps.insert(steps.end(), inner.begin(), inner.end());
  // pad so the device may always read kMaxAllSteps entries from step0
  while (steps.size() < first + kMaxAllStepsHost) steps.push_back(FftStep{});
  return SHT_OK;
}

}  // namespace sht

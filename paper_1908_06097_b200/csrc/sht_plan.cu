// Host side of libsht.so: plan construction (geometry, partition, buffer
// layouts, FFT plans, Legendre tile lists), the C-ABI of include/sht.h, and
// the NCCL grid<->spectral transposition.
//
// Data layout in HBM (per rank r, NFLD fields):
//   spectral  [nfld][2 * sum_{m in M_r} (T-m+1)]      m ascending, n ascending, re/im
//   grid      [nfld][sum_{i in R_r} 2 N_i]             local north rings asc, then their south mirrors
//   P table   per local m: [NDGLU(m) rings][Kp(m)]      Kp = roundup(T-m+1, 32), zero padded
//   Fourier   rows of nfld x {S.re, S.im, A.re, A.im}   one row per (ring pair i, m <= M_i)
//     X (m side, written by leg_inv / read by leg_dir):  [dest d][i in R_d][lm in M_r, m <= M_i]
//     Y (ring side, read by fft_f2g / written by fft_g2f): [src s][i in R_r][lm in M_s, m <= M_i]
//   so the per-destination block of X on rank r is exactly the per-source block
//   of Y on rank d, and the all-to-all is a plain grouped send/recv of
//   contiguous row ranges.  With one rank X and Y are the same buffer.
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>

#include "sht_internal.h"

namespace sht {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define SHT_NCCL_TRY(expr)                                                                           \
  do {                                                                                              \
    ncclResult_t _r = (expr);                                                                       \
    if (_r != ncclSuccess && _r != ncclInProgress) return ::sht::fail(SHT_ERR_COMM, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)

// Communication trace on stderr (SHT_DEBUG_COMM=1): failure-path diagnostics only.
static bool comm_debug() {
  static const bool d = getenv("SHT_DEBUG_COMM") != nullptr;
  return d;
}
#define SHT_COMM_LOG(...)                         \
  do {                                            \
    if (comm_debug()) {                           \
      fprintf(stderr, "[sht comm] " __VA_ARGS__); \
      fflush(stderr);                             \
    }                                             \
  } while (0)

// ------------------------------------------------------------------ geometry
// Gaussian nodes by Newton on theta in x87 extended precision.  The
// operation order is the one of oracle/sht_oracle.py gauss_nodes (numpy
// longdouble), so both round to the same doubles.
static void gauss_nodes_ld(int n, std::vector<double>& mu, std::vector<double>& sint, std::vector<double>& w) {
  typedef long double LD;
  const int nh = n / 2;
  const LD nld = (LD)n;
  const LD pi = 3.14159265358979323846264338327950288L;
  mu.resize(nh);
  sint.resize(nh);
  w.resize(nh);
  auto pn = [&](LD x, LD& p1o, LD& p0o) {
    LD p0 = 1.0L, p1 = x;
    for (int j = 2; j <= n; ++j) {
      const LD jl = (LD)j;
      const LD p2 = ((2.0L * jl - 1.0L) * x * p1 - (jl - 1.0L) * p0) / jl;
      p0 = p1;
      p1 = p2;
    }
    p1o = p1;
    p0o = p0;
  };
  for (int k = 1; k <= nh; ++k) {
    LD theta = pi * (4.0L * (LD)k - 1.0L) / (4.0L * nld + 2.0L);
    for (int it = 0; it < 8; ++it) {
      const LD x = cosl(theta);
      const LD s = sinl(theta);
      LD p1, p0;
      pn(x, p1, p0);
      const LD dp = nld * (x * p1 - p0) / (x * x - 1.0L);
      theta = theta + p1 / (s * dp);
    }
    const LD x = cosl(theta);
    const LD s = sinl(theta);
    LD p1, p0;
    pn(x, p1, p0);
    const LD ww = 2.0L * s * s / ((nld * p0) * (nld * p0));
    mu[k - 1] = (double)x;
    sint[k - 1] = (double)s;
    w[k - 1] = (double)ww;
  }
}

// Snake (boustrophedon) dealing of 0..n-1 over P ranks: 0,1,..,P-1,P-1,..,0,0,1,..
// Work per wavenumber, NDGLU(m)(T-m+1), and points per ring pair, 4i+20, are
// monotone, so the snake balances both.
static void snake(int n, int P, std::vector<int>& owner) {
  owner.resize(n);
  for (int k = 0; k < n; ++k) {
    const int blk = k / P, pos = k % P;
    owner[k] = (blk % 2 == 0) ? pos : P - 1 - pos;
  }
}

struct Geometry {
  int T = 0, ndgl = 0, nh = 0;
  std::vector<int> nloen;  // all rings
  std::vector<int> mcap;   // northern rings
};

static int make_geometry(int T, int ndgl, const int32_t* nloen, Geometry& g) {
  if (T < 1) return fail(SHT_ERR_CONFIG, "truncation must be >= 1");
  g.T = T;
  if (nloen == nullptr) {
    if (ndgl != 2 * (T + 1) && ndgl != 0)
      return fail(SHT_ERR_CONFIG, "octahedral grid needs ndgl == 2*(truncation+1)");
    g.ndgl = 2 * (T + 1);
    g.nloen.resize(g.ndgl);
    for (int i = 0; i <= T; ++i) {
      g.nloen[i] = 4 * (i + 1) + 16;
      g.nloen[g.ndgl - 1 - i] = g.nloen[i];
    }
  } else {
    if (ndgl < 2 || ndgl % 2) return fail(SHT_ERR_CONFIG, "ndgl must be even and >= 2");
    g.ndgl = ndgl;
    g.nloen.assign(nloen, nloen + ndgl);
    for (int j = 0; j < ndgl; ++j) {
      if (g.nloen[j] != g.nloen[ndgl - 1 - j])
        return fail(SHT_ERR_CONFIG, "nloen must be north/south symmetric");
      if (g.nloen[j] < 1) return fail(SHT_ERR_CONFIG, "nloen entries must be >= 1");
    }
  }
  g.nh = g.ndgl / 2;
  g.mcap.resize(g.nh);
  for (int i = 0; i < g.nh; ++i) {
    g.mcap[i] = std::min(T, (g.nloen[i] - 1) / 2);
    if (i > 0 && g.mcap[i] < g.mcap[i - 1])
      return fail(SHT_ERR_CONFIG, "ring wavenumber caps must be non-decreasing from pole to equator");
  }
  return SHT_OK;
}

// ------------------------------------------------------------------ host FFT (plan set-up only)
typedef std::complex<long double> cld;
static void dft_rec(const cld* in, int stride, cld* out, int n) {
  if (n == 1) {
    out[0] = in[0];
    return;
  }
  int p = 2;
  while (n % p) ++p;
  const int m = n / p;
  std::vector<cld> sub((size_t)n);
  for (int r = 0; r < p; ++r) dft_rec(in + (size_t)r * stride, stride * p, sub.data() + (size_t)r * m, m);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int k = 0; k < n; ++k) {
    cld acc = 0;
    for (int r = 0; r < p; ++r) {
      const long long e = ((long long)r * k) % n;
      const long double ang = -two_pi * (long double)e / (long double)n;
      acc += sub[(size_t)r * m + (k % m)] * cld(cosl(ang), sinl(ang));
    }
    out[k] = acc;
  }
}

void dft_host(const std::vector<cld>& in, std::vector<cld>& out) {
  out.resize(in.size());
  dft_rec(in.data(), 1, out.data(), (int)in.size());
}

// ------------------------------------------------------------------ plan
struct Phase {
  cudaEvent_t ev[10];
};

}  // namespace sht

struct sht_plan {
  sht::Geometry g;
  int nfld = 0, rank = 0, nranks = 1, flags = 0, nsm = 148;
  std::vector<double> mu, sint, w;
  std::vector<int> m_owner, ring_owner, lm_of_m;
  std::vector<int> my_m, my_rings;
  std::vector<int64_t> lm_soff;
  int64_t spec_ld = 0, grid_ld = 0;
  std::vector<int64_t> xoff, xrows, yoff, yrows;  // per peer, in rows
  int64_t xtot = 0, ytot = 0;
  std::vector<int64_t> xtot_of, ytot_of;         // every rank's X / Y row count (field-block strides)
  int nfb = 1;                                   // 64-field blocks of the Fourier-row buffers
  bool fblk = false;                             // field-blocked row layout (p2p, P > 1), else classic
  int64_t row_ld = 0;                            // doubles between consecutive rows (sht_internal.h)
  double work_leg = 0, work_fft = 0, work_a2a = 0;

  // device
  double* d_mu = nullptr;
  double* d_sint = nullptr;
  double* d_ptab = nullptr;
  int64_t ptab_len = 0;
  int32_t *d_lm_m = nullptr, *d_lm_i0 = nullptr, *d_lm_kp = nullptr, *d_xbase = nullptr;
  int64_t *d_lm_poff = nullptr, *d_lm_soff = nullptr;
  sht::LegTile *d_tiles_inv = nullptr, *d_tiles_dir = nullptr;
  int ntiles_inv = 0, ntiles_dir = 0;
  int* d_counter = nullptr;
  double* X = nullptr;
  double* Y = nullptr;
  sht::FftRing* d_rings = nullptr;
  sht::FftWork* d_work = nullptr;
  int fft_w0[sht::kFftVariants] = {}, fft_nw[sht::kFftVariants] = {};  // per ring-FFT kernel variant
  size_t fft_smem[sht::kFftVariants] = {};
  sht::FftStep* d_steps = nullptr;
  double2* d_tw = nullptr;
  int32_t* d_ditpos = nullptr;
  ncclComm_t comm = nullptr;
  bool have_events = false;
  cudaEvent_t ev[10];                      // ev[8], ev[9]: set-up timing
  static constexpr int kHist = 64;         // per-pair phase events of the last kHist pairs
  cudaEvent_t hist[kHist][12];             // (start, end) of inv_leg, inv_a2a, inv_fft, dir_fft, dir_a2a, dir_leg
  bool hist_inv[kHist] = {};               // set k holds the events of an inverse transform
  int hist_cur = 0, hist_done = 0;
  float setup_ms = 0.f;
  int fft_debug = 0;
  int leg_debug = 0;
  // SHT_FLAG_RECOMPUTE_LEGENDRE: the P table is regenerated chunk by chunk of
  // wavenumbers into a bounded scratch right before the GEMM tiles that use it
  struct Chunk {
    int lm0, lm1, ti0, ti1, td0, td1;
  };
  std::vector<Chunk> chunks;
  int64_t* d_lm_poff_rc = nullptr;   // chunk-relative P offsets
  double* d_dmant = nullptr;
  int32_t* d_dexp = nullptr;
  // transposition (SHT_TRANSPORT): "p2p" (default when every peer buffer can
  // be mapped) fuses it into the kernels -- leg_inv stores each ring's rows
  // into the ring owner's Y and fft_g2f stores each (ring, m) row into the m
  // owner's X, over NVLink peer memory -- leaving flag handshakes; "nccl" runs
  // grouped send/recv of the contiguous row blocks between the kernels.
  bool p2p = false;
  std::vector<double*> peer_x, peer_y;          // IPC mappings of the peers' X / Y (own at [rank])
  std::vector<uint32_t*> peer_flags;            // IPC mappings of the peers' flag words
  uint32_t* flagw = nullptr;                    // [4][P] written by the peers: kYArr, kXArr, kYFree, kXFree
  uint32_t** d_peer_flags = nullptr;
  uint32_t inv_epoch = 0, dir_epoch = 0;
  std::vector<int32_t> xbase;                   // host copy: X row of (ring, lm = 0)
  std::vector<int64_t> yrow;                    // per (local ring, m): row in this rank's Y
  std::vector<int32_t> orow_owner;              // per (local ring, m): owner of m
  std::vector<int64_t> orow;                    //   and the row in the owner's X
  std::vector<int64_t> yoff_at_owner;           // per ring owner d: row offset of block r in d's Y
  double** d_ring_out = nullptr;                // [nh] leg_inv destination row of (ring, lm = 0)
  double* d_stage = nullptr;                    // leg_inv pusher-epilogue staging slots (p2p, P > 1)
  int64_t* d_ring_bs = nullptr;                 // [nh] field-block stride of ring_out's buffer
  int64_t* d_rows_out_bs = nullptr;             // field-block stride of each rows_out row's buffer
  std::vector<sht::LegTile> h_tiles_inv;        // host copy of the leg_inv tile list
  double** d_rows_out = nullptr;                // fft_g2f destination row per (local ring, m)
  const double** d_rows_in = nullptr;           // fft_f2g source row per (local ring, m)
  // 2-D grid-point layout (sht_plan_set_gp_layout): the TRGTOL-style transposition
  sht::GpLayout gp;
  int32_t *d_gp_send_idx = nullptr, *d_gp_recv_idx = nullptr;
  int64_t *d_gp_send_displ = nullptr, *d_gp_recv_displ = nullptr;
  double *d_gridR = nullptr, *d_gp_buf0 = nullptr, *d_gp_buf1 = nullptr;
  // failure detection (nranks > 1): handshake error word in mapped host memory
  int32_t* h_err = nullptr;
  int32_t* d_err = nullptr;
  uint64_t timeout_ns = 60ull * 1000000000ull;  // SHT_COMM_TIMEOUT_MS (default 60 s)
  bool failed = false;                          // an error was reported: no collective teardown
  std::string fail_msg;
};

namespace sht {

// Local release of a plan (sht_plan_destroy): no collective.  With the p2p
// transport a peer may still store into this rank's buffers until it has
// passed the collective barrier of sht_plan_close, which a well-behaved
// caller runs first; without it the device is synchronised (this rank's own
// kernels are done) and the buffers are released.
static void free_plan(sht_plan* p) {
  if (!p) return;
  if (p->nranks > 1) cudaDeviceSynchronize();
  for (int d = 0; d < (int)p->peer_x.size(); ++d) {
    if (d == p->rank) continue;
    if (p->peer_x[d]) cudaIpcCloseMemHandle(p->peer_x[d]);
    if (p->peer_y[d]) cudaIpcCloseMemHandle(p->peer_y[d]);
    if (p->peer_flags[d]) cudaIpcCloseMemHandle(p->peer_flags[d]);
  }
  void* ptrs[] = {p->d_mu, p->d_sint, p->d_ptab, p->d_lm_m, p->d_lm_i0, p->d_lm_kp, p->d_xbase, p->d_lm_poff,
                  p->d_lm_soff, p->d_tiles_inv, p->d_tiles_dir, p->d_counter, p->X, p->d_steps, p->d_lm_poff_rc, p->d_dmant, p->d_dexp,
                  p->Y == p->X ? nullptr : p->Y, p->d_rings, p->d_work, p->d_tw, p->d_ditpos, p->flagw, p->d_peer_flags,
                  p->d_ring_out, p->d_rows_out, (void*)p->d_rows_in, p->d_gp_send_idx, p->d_gp_recv_idx,
                  p->d_gp_send_displ, p->d_gp_recv_displ, p->d_gridR, p->d_gp_buf0, p->d_gp_buf1, p->d_stage,
                  p->d_ring_bs, p->d_rows_out_bs};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (p->have_events) {
    for (auto& e : p->ev) cudaEventDestroy(e);
    for (auto& set : p->hist)
      for (auto& e : set) cudaEventDestroy(e);
  }
  if (p->h_err) cudaFreeHost(p->h_err);
  if (p->comm) {
    if (p->failed)
      ncclCommAbort(p->comm);  // a peer is gone: destroy would wait for it
    else
      ncclCommDestroy(p->comm);
  }
  delete p;
}

template <typename T>
static int upload(T** dst, const std::vector<T>& v) {
  const size_t bytes = std::max<size_t>(v.size(), 1) * sizeof(T);
  SHT_CUDA_TRY(cudaMalloc((void**)dst, bytes));
  if (!v.empty()) SHT_CUDA_TRY(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return SHT_OK;
}

// Ring-FFT cost model of one ring pair per field, in "bytes": 3 per complex
// element per pencil step (measured: ~2.9 ps per element-step vs ~0.94 ps per
// HBM byte on B200) plus the grid (16 N) and Fourier-row (32 (M+1)) traffic.
// Whole-ring Bluestein rings cost ~4x a smooth ring of the same length.
static int64_t ring_fft_cost(int n, int mcap) {
  RingPlan rp;
  if (fft_plan_ring(n, rp, mcap)) return 16LL * n;
  const int64_t ns = (int64_t)rp.radices.size();
  // a DMMA prime step of p costs ~p/16 radix-16 steps; factor-local Bluestein ~6
  const int64_t esteps = rp.ring_blue ? 2LL * rp.L * ns
                                      : (int64_t)n * (ns + (rp.bluestein ? 6 : rp.dprime / 16));
  return 3 * esteps + 16LL * n + 32LL * (mcap + 1);
}

// Wavenumbers: snake (balances the Legendre work NDGLU(m)(T-m+1), monotone in
// m).  Ring pairs: longest-processing-time first over the FFT cost model --
// the Bluestein rings are scattered irregularly in i, so a plain snake of the
// ring pairs left one rank ~12% more FFT time at P = 2.
static int build_partition(const Geometry& g, int P, std::vector<int>& m_owner, std::vector<int>& ring_owner) {
  if (P < 1) return fail(SHT_ERR_CONFIG, "nranks must be >= 1");
  // every rank must own at least one wavenumber and one ring pair, or its
  // local arrays are empty while its peers wait for it in the handshakes
  if (P > g.T + 1 || P > g.nh)
    return fail(SHT_ERR_CONFIG, "nranks (" + std::to_string(P) + ") exceeds min(truncation + 1, ndgl / 2) = " +
                                    std::to_string(std::min(g.T + 1, g.nh)));
  snake(g.T + 1, P, m_owner);
  std::vector<int64_t> cost(g.nh);
  std::vector<int> order(g.nh);
  for (int i = 0; i < g.nh; ++i) {
    cost[i] = ring_fft_cost(g.nloen[i], g.mcap[i]);
    order[i] = i;
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  std::vector<int64_t> load(P, 0);
  ring_owner.assign(g.nh, 0);
  for (int i : order) {
    int best = 0;
    for (int r = 1; r < P; ++r)
      if (load[r] < load[best]) best = r;
    ring_owner[i] = best;
    load[best] += cost[i];
  }
  return SHT_OK;
}

// ------------------------------------------------------------------ transposition
enum FlagSlot { kYArr = 0, kXArr = 1, kYFree = 2, kXFree = 3 };
constexpr double kP2PMaxBytes = 2.0 * (1 << 30);  // largest receive buffer for the classic row layout under p2p

// Handshake of the p2p transposition, one thread per peer t: publish
// `sig_v` in slot `sig_slot` of peer t's flag words (release, system scope:
// orders every store this GPU made before it in stream order, including the
// previous kernel's NVLink stores), then wait until peer t has published at
// least `wait_v` in slot `wait_slot` of ours (acquire).  The wait is bounded:
// after `timeout_ns` (SHT_COMM_TIMEOUT_MS) without the peer's flag the
// kernel records (peer + 1, slot) in the host-mapped error word and returns,
// and every later handshake of the plan returns at once, so a dead or
// desynchronised peer turns into SHT_ERR_COMM on the host instead of a hang
// (the reference's first-error abort, halo/router.py:124-126, 199-205).
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void flag_kernel(uint32_t* const* peer_flags, const uint32_t* flags, int P, int r, int sig_slot,
                            uint32_t sig_v, int wait_slot, uint32_t wait_v, uint64_t timeout_ns,
                            volatile int32_t* err) {
  const int t = threadIdx.x;
  if (t >= P || t == r) return;
  if (err[0] != 0) return;  // the plan already failed: drain the stream
  if (sig_slot >= 0) {
    __threadfence_system();
    uint32_t* a = peer_flags[t] + sig_slot * P + r;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(sig_v) : "memory");
  }
  if (wait_slot >= 0) {
    const uint32_t* a = flags + wait_slot * P + t;
    const uint64_t t0 = globaltimer_ns();
    for (int it = 0;; ++it) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
      if ((int32_t)(v - wait_v) >= 0) break;
      if ((it & 63) == 63) {
        if (err[0] != 0) return;
        if (globaltimer_ns() - t0 > timeout_ns) {
          atomicCAS((int32_t*)err, 0, (t + 1) * 16 + wait_slot);
          __threadfence_system();
          return;
        }
      }
      __nanosleep(128);
    }
  }
}

void flag_preload() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, flag_kernel);
}

static int flags_op(sht_plan* p, int sig_slot, uint32_t sig_v, int wait_slot, uint32_t wait_v, cudaStream_t s) {
  flag_kernel<<<1, 32 * ((p->nranks + 31) / 32), 0, s>>>(p->d_peer_flags, p->flagw, p->nranks, p->rank, sig_slot,
                                                          sig_v, wait_slot, wait_v, p->timeout_ns, p->d_err);
  SHT_CUDA_TRY(cudaGetLastError());
  return SHT_OK;
}

// Host-side view of the plan's communication health: the handshake error
// word (written by flag_kernel) and NCCL's asynchronous error state.
static int comm_check(sht_plan* p) {
  SHT_COMM_LOG("rank %d: comm_check\n", p->rank);
  if (p->failed) return fail(SHT_ERR_COMM, "the plan failed earlier (" + p->fail_msg + "); close it");
  if (p->h_err && p->h_err[0] != 0) {
    const int v = p->h_err[0];
    static const char* slot[] = {"rows-arrived (inverse)", "rows-arrived (direct)", "buffer-drained (inverse)",
                                 "buffer-drained (direct)"};
    return fail(SHT_ERR_COMM, "transposition handshake timed out after " + std::to_string(p->timeout_ns / 1000000) +
                                  " ms waiting for rank " + std::to_string(v / 16 - 1) + " (" + slot[(v % 16) & 3] +
                                  "); the peer is dead or desynchronised");
  }
  // (ncclCommGetAsyncError is polled only right after an NCCL call, in
  // nccl_settle: with a dead peer it can block inside NCCL's progress engine)
  return SHT_OK;
}

// The plan's communicator is non-blocking (ncclConfig_t::blocking = 0), so no
// NCCL call can hang the host on a dead peer: a call returns at once, maybe
// with ncclInProgress, and nccl_settle polls its completion with the plan's
// timeout, aborting the communicator when it expires.
static int nccl_settle(sht_plan* p, ncclResult_t rc, const char* what) {
  SHT_COMM_LOG("rank %d: %s returned %d\n", p->rank, what, (int)rc);
  if (rc != ncclSuccess && rc != ncclInProgress)
    return fail(SHT_ERR_COMM, std::string(what) + ": " + ncclGetErrorString(rc));
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    ncclResult_t st = ncclSuccess;
    if (ncclCommGetAsyncError(p->comm, &st) != ncclSuccess) st = ncclInternalError;
    if (st == ncclSuccess) return SHT_OK;
    if (st != ncclInProgress) {
      p->failed = true;
      p->fail_msg = std::string(what) + ": " + ncclGetErrorString(st);
      return fail(SHT_ERR_COMM, p->fail_msg);
    }
    const uint64_t el = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                            std::chrono::steady_clock::now() - t0).count();
    if (el > p->timeout_ns) {
      p->failed = true;
      SHT_COMM_LOG("rank %d: %s timed out, aborting the communicator\n", p->rank, what);
      ncclCommAbort(p->comm);
      SHT_COMM_LOG("rank %d: communicator aborted\n", p->rank);
      p->comm = nullptr;
      p->fail_msg = std::string(what) + " did not complete within " + std::to_string(p->timeout_ns / 1000000) +
                    " ms; communicator aborted";
      return fail(SHT_ERR_COMM, p->fail_msg);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// Waits for stream `s` with a bound: polls the stream, the handshake error
// word and NCCL's asynchronous error; on a peer failure or after
// `timeout_ns` the plan is marked failed (its NCCL communicator is aborted at
// destroy, so no later collective waits for the dead peer).
static int wait_stream(sht_plan* p, cudaStream_t s, uint64_t timeout_ns) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return fail(SHT_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(q));
    if (int rc = comm_check(p)) {
      p->failed = true;
      p->fail_msg = g_err;
      SHT_COMM_LOG("rank %d: handshake failure seen by the wait, aborting\n", p->rank);
      if (p->comm) ncclCommAbort(p->comm), p->comm = nullptr;
      return rc;
    }
    const uint64_t el = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                            std::chrono::steady_clock::now() - t0).count();
    if (el > timeout_ns) {
      p->failed = true;
      SHT_COMM_LOG("rank %d: wait timed out, aborting\n", p->rank);
      if (p->comm) ncclCommAbort(p->comm), p->comm = nullptr;
      SHT_COMM_LOG("rank %d: aborted\n", p->rank);
      p->fail_msg = "transform did not complete within " + std::to_string(timeout_ns / 1000000) +
                    " ms (a peer is dead or desynchronised); communicator aborted";
      return fail(SHT_ERR_COMM, p->fail_msg);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  if (int rc = comm_check(p)) {
    p->failed = true;
    p->fail_msg = g_err;
    return rc;
  }
  return SHT_OK;
}

// Collective teardown barrier (sht_plan_close): after it no peer stores into
// this rank's buffers any more.
static int close_barrier(sht_plan* p) {
  if (p->nranks < 2 || !p->comm || p->failed) return SHT_OK;
  SHT_CUDA_TRY(cudaDeviceSynchronize());
  cudaStream_t s;
  SHT_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int* d = nullptr;
  int rc = SHT_OK;
  if (cudaMalloc((void**)&d, sizeof(int)) != cudaSuccess) rc = fail(SHT_ERR_CUDA, "cudaMalloc (close barrier)");
  if (!rc) rc = nccl_settle(p, ncclAllReduce(d, d, 1, ncclInt, ncclSum, p->comm, s), "ncclAllReduce (close barrier)");
  if (!rc) rc = wait_stream(p, s, p->timeout_ns);
  if (d) cudaFree(d);
  cudaStreamDestroy(s);
  return rc;
}

// Chooses the transport and builds the row-pointer tables the kernels store
// through.  p2p: every rank exports X, Y and its flag words (CUDA IPC); the
// handles travel over the plan's NCCL communicator, and all ranks must map all
// peers or all fall back to NCCL send/recv.
static int build_transport(sht_plan* p) {
  const int P = p->nranks, r = p->rank;
  p->peer_x.assign(P, nullptr);
  p->peer_y.assign(P, nullptr);
  p->peer_flags.assign(P, nullptr);
  p->peer_x[r] = p->X;
  p->peer_y[r] = p->Y;
  if (P > 1) {
    // p2p unless SHT_TRANSPORT=nccl (or a rank cannot map its peers).  Where
    // the receive buffers the kernels store into over NVLink are large and
    // spread over >= 2 peers, the scattered remote row stores of the classic
    // row layout fall off a translation cliff (TCo1999 x 548 on 4 B200, 13 GB
    // per rank: fft_g2f 120 ms against 49 ms with local stores; 13 GB on 2
    // B200 showed none, profiles/r02_transport_cliff.md):
    // there the plan switches to the field-blocked row layout (fblk below).
    const char* tr = getenv("SHT_TRANSPORT");
    const double rbuf = (double)std::max(p->xtot, p->ytot) * (double)p->nfld * 32.0;
    const bool cliff = P >= 3 && rbuf > kP2PMaxBytes;
    const bool want = !(tr && std::string(tr) == "nccl");
    SHT_CUDA_TRY(cudaMalloc((void**)&p->flagw, 4 * P * sizeof(uint32_t)));
    SHT_CUDA_TRY(cudaMemset(p->flagw, 0, 4 * P * sizeof(uint32_t)));
    p->peer_flags[r] = p->flagw;
    SHT_CUDA_TRY(cudaHostAlloc((void**)&p->h_err, 4 * sizeof(int32_t), cudaHostAllocMapped));
    std::memset(p->h_err, 0, 4 * sizeof(int32_t));
    SHT_CUDA_TRY(cudaHostGetDevicePointer((void**)&p->d_err, p->h_err, 0));
    struct Rec {
      int32_t ok[16];
      cudaIpcMemHandle_t h[3];
    };
    Rec mine{};
    mine.ok[0] = want && cudaIpcGetMemHandle(&mine.h[0], p->X) == cudaSuccess &&
                 cudaIpcGetMemHandle(&mine.h[1], p->Y) == cudaSuccess &&
                 cudaIpcGetMemHandle(&mine.h[2], p->flagw) == cudaSuccess;
    mine.ok[1] = cliff;
    cudaGetLastError();
    Rec* d = nullptr;
    SHT_CUDA_TRY(cudaMalloc((void**)&d, (P + 1) * sizeof(Rec)));
    std::vector<Rec> all(P);
    auto exchange = [&]() -> int {
      SHT_CUDA_TRY(cudaMemcpy(d + P, &mine, sizeof(Rec), cudaMemcpyHostToDevice));
      if (int rc = nccl_settle(p, ncclAllGather(d + P, d, sizeof(Rec), ncclChar, p->comm, 0), "ncclAllGather (IPC handles)"))
        return rc;
      if (int rc = wait_stream(p, 0, p->timeout_ns)) return rc;
      SHT_CUDA_TRY(cudaMemcpy(all.data(), d, P * sizeof(Rec), cudaMemcpyDeviceToHost));
      return SHT_OK;
    };
    int rc = exchange();
    bool ok = rc == SHT_OK;
    for (int t = 0; t < P && ok; ++t) ok = all[t].ok[0] != 0;
    for (int t = 0; t < P && rc == SHT_OK; ++t) p->fblk = p->fblk || all[t].ok[1] != 0;  // any rank past the cliff
    if (ok) {  // map every peer, then agree that everybody could
      for (int t = 0; t < P && ok; ++t) {
        if (t == r) continue;
        void *x = nullptr, *y = nullptr, *f = nullptr;
        ok = cudaIpcOpenMemHandle(&x, all[t].h[0], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess &&
             cudaIpcOpenMemHandle(&y, all[t].h[1], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess &&
             cudaIpcOpenMemHandle(&f, all[t].h[2], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
        p->peer_x[t] = (double*)x;
        p->peer_y[t] = (double*)y;
        p->peer_flags[t] = (uint32_t*)f;
      }
      cudaGetLastError();
      mine.ok[0] = ok;
      rc = exchange();
      ok = rc == SHT_OK;
      for (int t = 0; t < P && ok; ++t) ok = all[t].ok[0] != 0;
    }
    cudaFree(d);
    if (rc) return rc;
    p->p2p = ok;
    if (!ok) {
      for (int t = 0; t < P; ++t) {
        if (t == r) continue;
        if (p->peer_x[t]) cudaIpcCloseMemHandle(p->peer_x[t]);
        if (p->peer_y[t]) cudaIpcCloseMemHandle(p->peer_y[t]);
        if (p->peer_flags[t]) cudaIpcCloseMemHandle(p->peer_flags[t]);
        p->peer_x[t] = p->peer_y[t] = nullptr;
        p->peer_flags[t] = nullptr;
      }
      cudaGetLastError();
    }
    if (int rc2 = upload(&p->d_peer_flags, p->peer_flags)) return rc2;
  }
  // row pointers: leg_inv's destination per ring, fft_g2f's per (ring, m), fft_f2g's source per (ring, m)
  const int nh = p->g.nh;
  // row layout: field-blocked where the p2p kernels' scattered remote row
  // stores would fall off the translation cliff (agreed above: any rank's
  // receive buffer > 2 GiB with >= 3 ranks; TCo1279 x 548 on 4 B200, 5.4 GB,
  // measured 73.3 ms classic vs 64.4 ms blocked on one box, 64.3 classic on
  // another; TCo639 x 548, 0.9 GB: 11.73 classic vs ~12.0 blocked); SHT_ROW_LAYOUT=classic|blocked
  // overrides (set it identically on every rank)
  p->fblk = p->p2p && p->fblk;
  if (const char* lay = getenv("SHT_ROW_LAYOUT")) p->fblk = std::string(lay) == "blocked";
  p->row_ld = p->fblk ? kRowDbl : (int64_t)p->nfld * 4;
  const int64_t ld = p->row_ld;
  auto bs = [&](int64_t rows) { return p->fblk ? rows * kRowDbl : (int64_t)0; };
  std::vector<double*> ring_out(nh), rows_out(p->yrow.size());
  std::vector<const double*> rows_in(p->yrow.size());
  std::vector<int64_t> ring_bs(nh), rows_out_bs(p->yrow.size());
  for (int i = 0; i < nh; ++i) {
    const int d = p->ring_owner[i];
    ring_out[i] = p->p2p ? p->peer_y[d] + (p->xbase[i] - p->xoff[d] + p->yoff_at_owner[d]) * ld
                         : p->X + (size_t)p->xbase[i] * ld;
    ring_bs[i] = bs(p->p2p ? p->ytot_of[d] : p->xtot);
  }
  for (size_t k = 0; k < p->yrow.size(); ++k) {
    const int t = p->orow_owner[k];
    rows_in[k] = p->Y + p->yrow[k] * ld;
    rows_out[k] = p->p2p ? p->peer_x[t] + p->orow[k] * ld : p->Y + p->yrow[k] * ld;
    rows_out_bs[k] = bs(p->p2p ? p->xtot_of[t] : p->ytot);
  }
  if (int rc = upload(&p->d_ring_out, ring_out)) return rc;
  if (int rc = upload(&p->d_ring_bs, ring_bs)) return rc;
  if (int rc = upload(&p->d_rows_out_bs, rows_out_bs)) return rc;
  // p2p: leg_inv tiles with a ring owned by a peer take the staged (pusher)
  // epilogue, so the NVLink stores leave the DMMA warps' path (SHT_LEG_STAGE=0: direct stores)
  const char* stg = getenv("SHT_LEG_STAGE");
  if (p->p2p && p->nranks > 1 && !(stg && std::string(stg) == "0") && p->ntiles_inv > 0) {
    std::vector<LegTile> ti = p->h_tiles_inv;
    bool any = false;
    for (auto& t : ti) {
      t.pad = 0;
      for (int i = t.r0; i < std::min(nh, t.r0 + kInvRings); ++i)
        if (p->ring_owner[i] != p->rank) t.pad = 1;
      any = any || t.pad;
    }
    if (any) {
      SHT_CUDA_TRY(cudaMemcpy(p->d_tiles_inv, ti.data(), ti.size() * sizeof(LegTile), cudaMemcpyHostToDevice));
      SHT_CUDA_TRY(cudaMalloc((void**)&p->d_stage, (size_t)p->nsm * kStageSlots * kInvRings * kLegFields * 4 * sizeof(double)));
    }
  }
  if (int rc = upload(&p->d_rows_out, rows_out)) return rc;
  if (int rc = upload(&p->d_rows_in, rows_in)) return rc;
  return SHT_OK;
}

static int build_plan(sht_plan* p, const void* nccl_id, bool dry_run = false) {
  const Geometry& g = p->g;
  const int T = g.T, nh = g.nh, P = p->nranks, r = p->rank, nfld = p->nfld;
  gauss_nodes_ld(g.ndgl, p->mu, p->sint, p->w);
  if (int rc = build_partition(g, P, p->m_owner, p->ring_owner)) return rc;

  std::vector<std::vector<int>> Mlist(P), Rlist(P);
  p->lm_of_m.assign(T + 1, 0);
  for (int m = 0; m <= T; ++m) {
    const int s = p->m_owner[m];
    p->lm_of_m[m] = (int)Mlist[s].size();
    Mlist[s].push_back(m);
  }
  for (int i = 0; i < nh; ++i) Rlist[p->ring_owner[i]].push_back(i);
  p->my_m = Mlist[r];
  p->my_rings = Rlist[r];
  const int nlm = (int)p->my_m.size();

  // c[s][i] = #{m in M_s : m <= M_i}
  std::vector<std::vector<int>> cnt(P, std::vector<int>(nh));
  for (int s = 0; s < P; ++s) {
    size_t k = 0;
    for (int i = 0; i < nh; ++i) {
      while (k < Mlist[s].size() && Mlist[s][k] <= g.mcap[i]) ++k;
      cnt[s][i] = (int)k;
    }
  }
  // X: [d][i in R_d][lm]
  std::vector<int32_t> xbase(nh, 0);
  p->xoff.assign(P, 0);
  p->xrows.assign(P, 0);
  int64_t cur = 0;
  for (int d = 0; d < P; ++d) {
    p->xoff[d] = cur;
    for (int i : Rlist[d]) {
      xbase[i] = (int32_t)cur;
      cur += cnt[r][i];
    }
    p->xrows[d] = cur - p->xoff[d];
  }
  p->xtot = cur;
  // Y: [s][i in R_r][lm_s]
  std::vector<std::vector<int64_t>> ybase(P, std::vector<int64_t>(nh, 0));
  p->yoff.assign(P, 0);
  p->yrows.assign(P, 0);
  cur = 0;
  for (int s = 0; s < P; ++s) {
    p->yoff[s] = cur;
    for (int i : Rlist[r]) {
      ybase[s][i] = cur;
      cur += cnt[s][i];
    }
    p->yrows[s] = cur - p->yoff[s];
  }
  p->ytot = cur;
  // where this rank's blocks sit in the peers' buffers (p2p transposition):
  // block r of ring owner d's Y, and block r of m owner t's X
  p->yoff_at_owner.assign(P, 0);
  std::vector<int64_t> xoff_at_owner(P, 0);
  for (int d = 0; d < P; ++d)
    for (int s2 = 0; s2 < r; ++s2)
      for (int i : Rlist[d]) p->yoff_at_owner[d] += cnt[s2][i];
  for (int t = 0; t < P; ++t)
    for (int d = 0; d < r; ++d)
      for (int i : Rlist[d]) xoff_at_owner[t] += cnt[t][i];
  p->xbase = xbase;
  if (p->xtot > INT32_MAX || p->ytot > INT32_MAX) return fail(SHT_ERR_CONFIG, "Fourier row count overflows int32");
  // every rank's buffer heights: the field-block strides of the peers' X / Y (p2p)
  p->nfb = (nfld + kLegFields - 1) / kLegFields;
  p->xtot_of.assign(P, 0);
  p->ytot_of.assign(P, 0);
  for (int t = 0; t < P; ++t)
    for (int i = 0; i < nh; ++i) p->xtot_of[t] += cnt[t][i];
  for (int d = 0; d < P; ++d)
    for (int s2 = 0; s2 < P; ++s2)
      for (int i : Rlist[d]) p->ytot_of[d] += cnt[s2][i];
  if (p->xtot_of[r] != p->xtot || p->ytot_of[r] != p->ytot) return fail(SHT_ERR_CONFIG, "row-count bookkeeping");

  // local spectral layout
  p->lm_soff.resize(nlm);
  int64_t so = 0;
  for (int lm = 0; lm < nlm; ++lm) {
    p->lm_soff[lm] = so;
    so += T - p->my_m[lm] + 1;
  }
  p->spec_ld = 2 * so;

  // P-table layout
  std::vector<int32_t> lm_i0(nlm), lm_kp(nlm), lm_m(p->my_m.begin(), p->my_m.end());
  std::vector<int64_t> lm_poff(nlm);
  int64_t po = 0;
  double leg_flops = 0;
  for (int lm = 0; lm < nlm; ++lm) {
    const int m = p->my_m[lm];
    const int i0 = (int)(std::lower_bound(g.mcap.begin(), g.mcap.end(), m) - g.mcap.begin());
    const int K = T - m + 1;
    lm_i0[lm] = i0;
    lm_kp[lm] = (K + kPtabPad - 1) / kPtabPad * kPtabPad;
    lm_poff[lm] = po;
    po += (int64_t)(nh - i0) * lm_kp[lm];
    leg_flops += 4.0 * nfld * (double)(nh - i0) * K;
  }
  p->ptab_len = po;
  p->work_leg = 2.0 * leg_flops;

  // Legendre tiles, wavenumber-major with m ascending (K = T-m+1 descending):
  // the persistent tile queue then runs the largest GEMMs first (LPT) and the
  // ~150 tiles in flight touch only 2-4 wavenumbers, whose P-table rows and
  // spectral / Fourier blocks stay resident in L2 across ring / n / field tiles.
  std::vector<LegTile> ti, td;
  for (int lm = 0; lm < nlm; ++lm) {
    const int K = T - p->my_m[lm] + 1;
    for (int r0 = lm_i0[lm]; r0 < nh; r0 += kInvRings)
      for (int f0 = 0; f0 < nfld; f0 += kLegFields) ti.push_back({lm, r0, f0, 0});
    for (int f0 = 0; f0 < nfld; f0 += kLegFields)
      for (int n0 = 0; n0 < K; n0 += kDirN) td.push_back({lm, n0, f0, 0});
  }
  p->ntiles_inv = (int)ti.size();
  p->ntiles_dir = (int)td.size();
  p->h_tiles_inv = ti;

  // grid layout + FFT plans
  const int nlr = (int)p->my_rings.size();
  std::vector<FftRing> rings(nlr);
  std::vector<double2> arena;
  std::vector<int32_t> ditpos;  // digit-reversed bin positions of the non-Bluestein rings
  p->yrow.clear();
  p->orow.clear();
  p->orow_owner.clear();
  int64_t go = 0;
  for (int lr = 0; lr < nlr; ++lr) {
    rings[lr].goff_n = go;
    go += g.nloen[p->my_rings[lr]];
  }
  for (int lr = nlr - 1; lr >= 0; --lr) {
    rings[lr].goff_s = go;
    go += g.nloen[p->my_rings[lr]];
  }
  p->grid_ld = go;
  // shared memory per CTA: variant 1 runs 2 CTAs/SM, variant 2 one
  const size_t budget[kFftVariants] = {0, 100 * 1024, 212 * 1024, 212 * 1024};
  std::vector<FftStep> steps;
  std::vector<int64_t> ring_cost(nlr, 0);
  int64_t nfour_local = 0;
  for (int lr = 0; lr < nlr; ++lr) {
    const int i = p->my_rings[lr];
    FftRing& R = rings[lr];
    R.n = g.nloen[i];
    R.mcap = g.mcap[i];
    R.w = p->w[i];
    nfour_local += 2 * (int64_t)(R.mcap + 1);
    RingPlan rp;
    if (fft_plan_ring(R.n, rp, R.mcap))
      return fail(SHT_ERR_CONFIG, "no FFT plan for ring length " + std::to_string(R.n));
    int variant = rp.variant;
    R.L = rp.L;
    R.shift = rp.shift;
    R.dit_off = -1;
    if (!rp.ring_blue) {
      R.dit_off = (int64_t)ditpos.size();
      for (int k = 0; k < R.n; ++k) ditpos.push_back((int32_t)fft_pos(k, rp.radices));
    }
    R.mag_N = ((uint64_t)1 << 40) / (uint64_t)R.n + 1;
    R.mag_M1 = ((uint64_t)1 << 40) / (uint64_t)(R.mcap + 1) + 1;
    R.mag_L = ((uint64_t)1 << 40) / (uint64_t)R.L + 1;
    R.yrow_off = (int64_t)p->yrow.size();
    for (int m = 0; m <= R.mcap; ++m) {
      const int s = p->m_owner[m];
      p->yrow.push_back(ybase[s][i] + p->lm_of_m[m]);
      p->orow_owner.push_back(s);
      p->orow.push_back(ybase[s][i] - p->yoff[s] + xoff_at_owner[s] + p->lm_of_m[m]);
    }
    // batch: nb fields (one complex sequence of N each, north + i south) as
    // many as fit; Bluestein rings add a work buffer of G pencils x Lp
    const int Lp = rp.wlen;
    auto smem = [&](int nb, int G) {
      return (fft_slots((size_t)nb * R.L) + (Lp ? fft_slots((size_t)G * Lp) : 0)) * sizeof(double2);
    };
    auto fit = [&](size_t bud, int& nb, int& G) {
      for (nb = std::min(nfld, 128); nb >= 1; --nb) {
        G = Lp ? std::min(8, (int)(((bud - std::min(bud, fft_slots((size_t)nb * R.L) * sizeof(double2))) /
                                    sizeof(double2) * 16 / 17) / std::max(1, Lp))) : 0;
        if ((Lp == 0 || G >= 1) && smem(nb, G) <= bud) return true;
      }
      return false;
    };
    int nb = 1, G = 0;
    if (!fit(budget[variant], nb, G)) {
      if (variant != 1 || !fit(budget[3], nb, G))
        return fail(SHT_ERR_CONFIG, "ring FFT does not fit in shared memory (N=" + std::to_string(R.n) + ")");
      variant = 3;  // one CTA per SM with more shared memory
    }
    if (fft_build_ring(R.n, rp, std::max(G, 1), steps, arena, R.tw_off, R.ntw, R.chirp_off, R.bhat_off))
      return fail(SHT_ERR_CONFIG, "FFT plan tables too large for ring length " + std::to_string(R.n));
    R.step0 = (int)steps.size() - kMaxAllStepsHost;
    R.nstep = (int)rp.radices.size();
    R.variant = variant;
    R.nb = nb;
    R.wlen = Lp * std::max(G, 1);
    p->fft_smem[variant] = std::max(p->fft_smem[variant], smem(nb, G));
    const int64_t esteps = rp.ring_blue ? 2LL * R.L * (int64_t)rp.radices.size()
                                        : (int64_t)R.n * ((int64_t)rp.radices.size() +
                                                          (rp.bluestein ? 6 : rp.dprime / 16));
    ring_cost[lr] = (int64_t)nfld * (esteps + 4LL * R.n);
  }
  // split every ring's fields over CTAs so each variant's launch has
  // ~6 CTAs per SM of balanced cost; largest first (LPT)
  std::vector<FftWork> work;
  {
    int nsm = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    for (int v = 1; v < kFftVariants; ++v) {
      int64_t tot = 0;
      for (int lr = 0; lr < nlr; ++lr)
        if (rings[lr].variant == v) tot += ring_cost[lr];
      std::vector<std::pair<int64_t, FftWork>> wl;
      const double target = std::max<double>(1.0, (double)tot / (6.0 * nsm));
      for (int lr = 0; lr < nlr; ++lr) {
        if (rings[lr].variant != v) continue;
        const int K = rings[lr].nb;
        const int maxsplit = (nfld + K - 1) / K;
        const int splits = std::max(1, std::min(maxsplit, (int)std::llround(ring_cost[lr] / target)));
        int chunk = (nfld + splits - 1) / splits;
        chunk = (chunk + K - 1) / K * K;
        for (int a = 0; a < nfld; a += chunk) {
          const int b = std::min(nfld, a + chunk);
          wl.push_back({ring_cost[lr] * (b - a) / nfld, {lr, a, b, 0}});
        }
      }
      std::stable_sort(wl.begin(), wl.end(), [](const std::pair<int64_t, FftWork>& x,
                                                const std::pair<int64_t, FftWork>& y) { return x.first > y.first; });
      p->fft_w0[v] = (int)work.size();
      p->fft_nw[v] = (int)wl.size();
      for (auto& x : wl) work.push_back(x.second);
    }
  }
  int64_t npts_local = go;
  p->work_fft = 2.0 * nfld * (8.0 * (double)npts_local + 16.0 * (double)nfour_local);
  int64_t sent = 0;
  for (int d = 0; d < P; ++d)
    if (d != r) sent += p->xrows[d];
  p->work_a2a = 2.0 * (double)sent * nfld * 32.0;

  if (dry_run) return SHT_OK;

  // ---- device side
  fft_preload();
  leg_preload();
  flag_preload();
  gp_preload();
  int dev = 0;
  SHT_CUDA_TRY(cudaGetDevice(&dev));
  SHT_CUDA_TRY(cudaDeviceGetAttribute(&p->nsm, cudaDevAttrMultiProcessorCount, dev));
  if (int rc = upload(&p->d_mu, p->mu)) return rc;
  if (int rc = upload(&p->d_sint, p->sint)) return rc;
  if (int rc = upload(&p->d_lm_m, lm_m)) return rc;
  if (int rc = upload(&p->d_lm_i0, lm_i0)) return rc;
  if (int rc = upload(&p->d_lm_kp, lm_kp)) return rc;
  if (int rc = upload(&p->d_lm_poff, lm_poff)) return rc;
  if (int rc = upload(&p->d_lm_soff, p->lm_soff)) return rc;
  if (int rc = upload(&p->d_xbase, xbase)) return rc;
  if (int rc = upload(&p->d_tiles_inv, ti)) return rc;
  if (int rc = upload(&p->d_tiles_dir, td)) return rc;
  if (int rc = upload(&p->d_rings, rings)) return rc;
  if (int rc = upload(&p->d_work, work)) return rc;
  if (int rc = upload(&p->d_steps, steps)) return rc;
  if (int rc = upload(&p->d_tw, arena)) return rc;
  if (int rc = upload(&p->d_ditpos, ditpos)) return rc;
  SHT_CUDA_TRY(cudaMalloc((void**)&p->d_counter, 4 * sizeof(int)));
  const size_t rowb = (size_t)p->nfb * kRowDbl * sizeof(double);  // one row in every field block
  SHT_CUDA_TRY(cudaMalloc((void**)&p->X, std::max<int64_t>(p->xtot, 1) * rowb));
  if (P == 1) {
    p->Y = p->X;
  } else {
    SHT_CUDA_TRY(cudaMalloc((void**)&p->Y, std::max<int64_t>(p->ytot, 1) * rowb));
  }
  for (auto& e : p->ev) SHT_CUDA_TRY(cudaEventCreate(&e));
  for (auto& set : p->hist)
    for (auto& e : set) SHT_CUDA_TRY(cudaEventCreate(&e));
  p->have_events = true;

  SHT_CUDA_TRY(cudaMalloc((void**)&p->d_dmant, std::max(1, nlm) * (size_t)nh * sizeof(double)));
  SHT_CUDA_TRY(cudaMalloc((void**)&p->d_dexp, std::max(1, nlm) * (size_t)nh * sizeof(int32_t)));
  SHT_CUDA_TRY(cudaEventRecord(p->ev[8], 0));
  launch_leg_diag(T, nh, nlm, p->d_lm_m, p->d_sint, p->d_dmant, p->d_dexp, 0);
  if (!(p->flags & SHT_FLAG_RECOMPUTE_LEGENDRE)) {
    SHT_CUDA_TRY(cudaMalloc((void**)&p->d_ptab, std::max<int64_t>(p->ptab_len, 1) * sizeof(double)));
    SHT_CUDA_TRY(cudaMemset(p->d_ptab, 0, std::max<int64_t>(p->ptab_len, 1) * sizeof(double)));
    launch_leg_poly(T, nh, 0, nlm, p->d_lm_m, p->d_lm_i0, p->d_lm_poff, p->d_lm_kp, p->d_mu, p->d_dmant, p->d_dexp,
                    p->d_ptab, 0);
  } else {
    // chunks of consecutive wavenumbers whose table fits the scratch budget
    int64_t budget = (int64_t)256 << 20;  // doubles (2 GB); SHT_RECOMPUTE_CHUNK_MB overrides (tests)
    if (const char* mb = getenv("SHT_RECOMPUTE_CHUNK_MB")) budget = std::max<int64_t>(1, atoll(mb)) << 17;
    std::vector<int64_t> rc(nlm);
    int64_t scratch = 0;
    for (int lm = 0; lm < nlm;) {
      sht_plan::Chunk ch{};
      ch.lm0 = lm;
      int64_t used = 0;
      while (lm < nlm) {
        const int64_t sz = (int64_t)(nh - lm_i0[lm]) * lm_kp[lm];
        if (used > 0 && used + sz > budget) break;
        rc[lm] = used;
        used += sz;
        ++lm;
      }
      ch.lm1 = lm;
      scratch = std::max(scratch, used);
      p->chunks.push_back(ch);
    }
    // tile ranges of each chunk (both tile lists are wavenumber-major)
    size_t a = 0, b = 0;
    for (auto& ch : p->chunks) {
      ch.ti0 = (int)a;
      while (a < ti.size() && ti[a].lm < ch.lm1) ++a;
      ch.ti1 = (int)a;
      ch.td0 = (int)b;
      while (b < td.size() && td[b].lm < ch.lm1) ++b;
      ch.td1 = (int)b;
    }
    if (int rc2 = upload(&p->d_lm_poff_rc, rc)) return rc2;
    SHT_CUDA_TRY(cudaMalloc((void**)&p->d_ptab, std::max<int64_t>(scratch, 1) * sizeof(double)));
    SHT_CUDA_TRY(cudaMemset(p->d_ptab, 0, std::max<int64_t>(scratch, 1) * sizeof(double)));
    p->ptab_len = scratch;
  }
  SHT_CUDA_TRY(cudaGetLastError());
  SHT_CUDA_TRY(cudaEventRecord(p->ev[9], 0));
  SHT_CUDA_TRY(cudaEventSynchronize(p->ev[9]));
  SHT_CUDA_TRY(cudaEventElapsedTime(&p->setup_ms, p->ev[8], p->ev[9]));

  if (P > 1) {
    if (!nccl_id) return fail(SHT_ERR_CONFIG, "nranks > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;  // never block the host on a dead peer (nccl_settle)
    const ncclResult_t irc = ncclCommInitRankConfig(&p->comm, P, id, r, &cfg);
    if (irc != ncclSuccess && irc != ncclInProgress)
      return fail(SHT_ERR_COMM, std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(irc));
    if (int rc = nccl_settle(p, ncclInProgress, "ncclCommInitRankConfig")) return rc;
  }
  return build_transport(p);
}

static LegParams leg_params(const sht_plan* p, const LegTile* tiles, int ntiles, int* counter,
                            const int64_t* poff = nullptr) {
  LegParams lp;
  lp.T = p->g.T;
  lp.nh = p->g.nh;
  lp.nfld = p->nfld;
  lp.nlm = (int)p->my_m.size();
  lp.lm_m = p->d_lm_m;
  lp.lm_i0 = p->d_lm_i0;
  lp.lm_poff = poff ? poff : p->d_lm_poff;
  lp.lm_kp = p->d_lm_kp;
  lp.lm_soff = p->d_lm_soff;
  lp.spec_ld = p->spec_ld;
  lp.xbase = p->d_xbase;
  lp.ring_out = p->d_ring_out;
  lp.stage = p->d_stage;
  lp.ring_bs = p->d_ring_bs;
  lp.xbs = p->fblk ? p->xtot * kRowDbl : 0;
  lp.row_ld = p->row_ld;
  lp.fsh = p->fblk ? 6 : 30;
  lp.fmask = p->fblk ? 63 : (1 << 30) - 1;
  lp.ptab = p->d_ptab;
  lp.tiles = tiles;
  lp.ntiles = ntiles;
  lp.counter = counter;
  lp.debug = p->leg_debug;
  return lp;
}

static FftParams fft_params(const sht_plan* p) {
  FftParams fp;
  fp.nfld = p->nfld;
  fp.grid_ld = p->grid_ld;
  fp.rings = p->d_rings;
  fp.steps = p->d_steps;
  fp.work = p->d_work;
  fp.tw = p->d_tw;
  fp.ditpos = p->d_ditpos;
  fp.rows_out = p->d_rows_out;
  fp.rows_in = p->d_rows_in;
  fp.rows_out_bs = p->d_rows_out_bs;
  fp.in_bs = p->fblk ? p->ytot * kRowDbl : 0;
  fp.fsh = p->fblk ? 6 : 30;
  fp.fmask = p->fblk ? 63 : (1 << 30) - 1;
  fp.debug = p->fft_debug;
  return fp;
}

// Grouped NCCL send/recv in the rotated order of the reference's
// ROTATED_CONCURRENT schedule (collectives.py:85-86: rank r issues to
// target (k + r) % P for k = 0..P-1).  The self block is a
// device copy.  from_x: X -> Y (inverse), else Y -> X (direct).
static int alltoall(sht_plan* p, bool from_x, cudaStream_t s) {
  const int P = p->nranks, r = p->rank;
  const size_t rowd = p->row_ld;
  const int nblk = p->fblk ? p->nfb : 1;
  const double* src = from_x ? p->X : p->Y;
  double* dst = from_x ? p->Y : p->X;
  const size_t sbs = (size_t)(from_x ? p->xtot : p->ytot) * rowd;  // field-block strides (blocked layout)
  const size_t dbs = (size_t)(from_x ? p->ytot : p->xtot) * rowd;
  const std::vector<int64_t>& soff = from_x ? p->xoff : p->yoff;
  const std::vector<int64_t>& srows = from_x ? p->xrows : p->yrows;
  const std::vector<int64_t>& doff = from_x ? p->yoff : p->xoff;
  const std::vector<int64_t>& drows = from_x ? p->yrows : p->xrows;
  if (srows[r] > 0)  // the self block of every field block
    SHT_CUDA_TRY(cudaMemcpy2DAsync(dst + doff[r] * rowd, dbs * sizeof(double), src + soff[r] * rowd,
                                   sbs * sizeof(double), srows[r] * rowd * sizeof(double), nblk,
                                   cudaMemcpyDeviceToDevice, s));
  if (p->failed || !p->comm) return comm_check(p);
  SHT_COMM_LOG("rank %d: all-to-all %s: group start\n", p->rank, from_x ? "X->Y" : "Y->X");
  SHT_NCCL_TRY(ncclGroupStart());
  for (int k = 1; k < P; ++k) {
    const int to = (r + k) % P, from = (r - k + P) % P;
    for (int b = 0; b < nblk; ++b) {  // one message per field block
      if (srows[to] > 0)
        SHT_NCCL_TRY(ncclSend(src + b * sbs + soff[to] * rowd, srows[to] * rowd, ncclDouble, to, p->comm, s));
      if (drows[from] > 0)
        SHT_NCCL_TRY(ncclRecv(dst + b * dbs + doff[from] * rowd, drows[from] * rowd, ncclDouble, from, p->comm, s));
    }
  }
  return nccl_settle(p, ncclGroupEnd(), "ncclGroupEnd (transposition)");
}

static int check_ptr(const void* q, const char* what) {
  if (!q) return fail(SHT_ERR_CONFIG, std::string(what) + " is NULL");
  if (reinterpret_cast<uintptr_t>(q) % 16) return fail(SHT_ERR_CONFIG, std::string(what) + " must be 16-byte aligned");
  return SHT_OK;
}

}  // namespace sht

using namespace sht;

extern "C" {

int sht_version(void) { return 100; }

const char* sht_last_error(void) { return g_err.c_str(); }

int sht_gauss_nodes(int ndgl, double* mu, double* sint, double* w) {
  if (ndgl < 2 || ndgl % 2) return fail(SHT_ERR_CONFIG, "ndgl must be even and >= 2");
  std::vector<double> a, b, c;
  gauss_nodes_ld(ndgl, a, b, c);
  if (mu) std::copy(a.begin(), a.end(), mu);
  if (sint) std::copy(b.begin(), b.end(), sint);
  if (w) std::copy(c.begin(), c.end(), w);
  return SHT_OK;
}

int sht_plan_validate(int truncation, int ndgl, const int32_t* nloen, int nfld, int nranks) {
  if (nfld < 1) return fail(SHT_ERR_CONFIG, "nfld must be >= 1");
  if (nranks < 1) return fail(SHT_ERR_CONFIG, "invalid nranks");
  for (int r = 0; r < nranks; ++r) {
    sht_plan* p = new sht_plan();
    p->nfld = nfld;
    p->rank = r;
    p->nranks = nranks;
    int rc = make_geometry(truncation, ndgl, nloen, p->g);
    if (!rc) rc = build_plan(p, nullptr, true);
    delete p;
    if (rc) return rc;
  }
  return SHT_OK;
}

int sht_partition(int truncation, int ndgl, const int32_t* nloen, int nranks, int32_t* m_owner, int32_t* ring_owner) {
  Geometry g;
  if (int rc = make_geometry(truncation, ndgl, nloen, g)) return rc;
  std::vector<int> mo, ro;
  if (int rc = build_partition(g, nranks, mo, ro)) return rc;
  if (m_owner) std::copy(mo.begin(), mo.end(), m_owner);
  if (ring_owner) std::copy(ro.begin(), ro.end(), ring_owner);
  return SHT_OK;
}

int sht_alltoall_rows(int truncation, int ndgl, const int32_t* nloen, int nranks, int64_t* rows) {
  Geometry g;
  if (int rc = make_geometry(truncation, ndgl, nloen, g)) return rc;
  std::vector<int> mo, ro;
  if (int rc = build_partition(g, nranks, mo, ro)) return rc;
  const int P = nranks;
  // rows[r][d] = sum over rings i of d of #{m of r : m <= M_i}
  std::vector<std::vector<int64_t>> cnt(P, std::vector<int64_t>(g.nh, 0));
  for (int i = 0; i < g.nh; ++i)
    for (int m = 0; m <= std::min(g.T, g.mcap[i]); ++m) cnt[mo[m]][i] += 1;
  if (rows) {
    for (int k = 0; k < P * P; ++k) rows[k] = 0;
    for (int i = 0; i < g.nh; ++i)
      for (int r = 0; r < P; ++r) rows[(int64_t)r * P + ro[i]] += cnt[r][i];
  }
  return SHT_OK;
}

int sht_alltoall_order(int nranks, int rank, int32_t* peers) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SHT_ERR_CONFIG, "invalid rank / nranks");
  for (int k = 0; k < nranks; ++k) peers[k] = (rank + k) % nranks;  // collectives.py:85-86
  return SHT_OK;
}

int sht_fft_plan_info(int n, int32_t* radices, int32_t* nstages, int32_t* fft_len, int32_t* bluestein) {
  RingPlan rp;
  if (n < 1) return fail(SHT_ERR_CONFIG, "ring length must be >= 1");
  if (fft_plan_ring(n, rp)) return fail(SHT_ERR_CONFIG, "no FFT plan for this length");
  if (radices)
    for (size_t k = 0; k < rp.radices.size() && k < 32; ++k) radices[k] = rp.radices[k];
  if (nstages) *nstages = (int32_t)rp.radices.size();
  if (fft_len) *fft_len = rp.L;
  if (bluestein) *bluestein = rp.bluestein ? 1 : 0;
  return SHT_OK;
}

int sht_nccl_get_unique_id(void* out128) {
  if (!out128) return fail(SHT_ERR_CONFIG, "out128 is NULL");
  ncclUniqueId id;
  SHT_NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return SHT_OK;
}

static sht_plan* new_plan(int nfld, int rank, int nranks, int flags) {
  sht_plan* p = new sht_plan();
  p->nfld = nfld;
  p->rank = rank;
  p->nranks = nranks;
  p->flags = flags;
  if (const char* dbg = getenv("SHT_FFT_DEBUG")) p->fft_debug = atoi(dbg);
  if (const char* dbg = getenv("SHT_LEG_DEBUG")) p->leg_debug = atoi(dbg);
  if (const char* to = getenv("SHT_COMM_TIMEOUT_MS"))
    p->timeout_ns = (uint64_t)std::max(1LL, atoll(to)) * 1000000ull;
  return p;
}

int sht_plan_create(int truncation, int ndgl, const int32_t* nloen, int nfld, int rank, int nranks,
                    const void* nccl_unique_id, int flags, sht_plan** out) {
  if (!out) return fail(SHT_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  if (nfld < 1) return fail(SHT_ERR_CONFIG, "nfld must be >= 1");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SHT_ERR_CONFIG, "invalid rank / nranks");
  sht_plan* p = new_plan(nfld, rank, nranks, flags);
  int rc = make_geometry(truncation, ndgl, nloen, p->g);
  if (!rc) rc = build_plan(p, nccl_unique_id);
  if (rc) {
    const std::string msg = g_err;
    free_plan(p);
    g_err = msg;
    return rc;
  }
  *out = p;
  return SHT_OK;
}

void sht_plan_destroy(sht_plan* plan) { free_plan(plan); }

int sht_plan_close(sht_plan* plan) {
  if (!plan) return SHT_OK;
  const int rc = close_barrier(plan);
  const std::string msg = g_err;
  free_plan(plan);
  g_err = msg;
  return rc;
}

int sht_wait(sht_plan* plan, void* stream, int timeout_ms) {
  if (!plan) return fail(SHT_ERR_CONFIG, "plan is NULL");
  const uint64_t to = timeout_ms > 0 ? (uint64_t)timeout_ms * 1000000ull : plan->timeout_ns;
  return wait_stream(plan, (cudaStream_t)stream, to);
}

int sht_local_layout(const sht_plan* p, int64_t* nspec_re, int64_t* npts, int32_t* m_list, int32_t* n_m,
                     int32_t* ring_list, int32_t* n_rings) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  if (nspec_re) *nspec_re = p->spec_ld;
  if (npts) *npts = p->grid_ld;
  if (m_list) std::copy(p->my_m.begin(), p->my_m.end(), m_list);
  if (n_m) *n_m = (int32_t)p->my_m.size();
  const int nl = (int)p->my_rings.size();
  if (ring_list) {
    for (int k = 0; k < nl; ++k) ring_list[k] = p->my_rings[k];
    for (int k = 0; k < nl; ++k) ring_list[nl + k] = p->g.ndgl - 1 - p->my_rings[nl - 1 - k];
  }
  if (n_rings) *n_rings = 2 * nl;
  return SHT_OK;
}

int sht_work(const sht_plan* p, double* lf, double* fb, double* ab) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  if (lf) *lf = p->work_leg;
  if (fb) *fb = p->work_fft;
  if (ab) *ab = p->work_a2a;
  return SHT_OK;
}

}  // extern "C"

namespace sht {

static void prof_ev(sht_plan* p, int k, cudaStream_t s) {
  if (p->flags & SHT_FLAG_PROFILE_PHASES) cudaEventRecord(p->hist[p->hist_cur][k], s);
}

static int phase_leg(sht_plan* p, bool inv, const double* in, double* out, cudaStream_t s) {
  prof_ev(p, inv ? 0 : 10, s);
  const LegTile* tiles = inv ? p->d_tiles_inv : p->d_tiles_dir;
  const int ntiles = inv ? p->ntiles_inv : p->ntiles_dir;
  int* counter = p->d_counter + (inv ? 0 : 1);
  auto launch = [&](const LegParams& lp, int n) {
    if (inv)
      launch_leg_inv(lp, in, p->X, std::min(p->nsm, n), s);
    else
      launch_leg_dir(lp, p->X, out, std::min(p->nsm, n), s);
  };
  if (p->chunks.empty()) {
    if (ntiles) {
      SHT_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(int), s));
      launch(leg_params(p, tiles, ntiles, counter), ntiles);
    }
  } else {
    for (const auto& ch : p->chunks) {  // regenerate the P rows of this chunk, then its GEMM tiles
      launch_leg_poly(p->g.T, p->g.nh, ch.lm0, ch.lm1, p->d_lm_m, p->d_lm_i0, p->d_lm_poff_rc, p->d_lm_kp,
                      p->d_mu, p->d_dmant, p->d_dexp, p->d_ptab, s);
      const int t0 = inv ? ch.ti0 : ch.td0, t1 = inv ? ch.ti1 : ch.td1;
      if (t1 > t0) {
        SHT_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(int), s));
        launch(leg_params(p, tiles + t0, t1 - t0, counter, p->d_lm_poff_rc), t1 - t0);
      }
    }
  }
  SHT_CUDA_TRY(cudaGetLastError());
  prof_ev(p, inv ? 1 : 11, s);
  return SHT_OK;
}

static int phase_a2a(sht_plan* p, bool inv, cudaStream_t s) {
  prof_ev(p, inv ? 2 : 8, s);
  if (p->p2p) {  // rows are already in place: publish "mine arrived", wait for everybody's
    const uint32_t e = inv ? p->inv_epoch : p->dir_epoch;
    if (int rc = flags_op(p, inv ? kYArr : kXArr, e, inv ? kYArr : kXArr, e, s)) return rc;
  } else if (p->nranks > 1) {
    if (int rc = alltoall(p, inv, s)) return rc;
  }
  prof_ev(p, inv ? 3 : 9, s);
  return SHT_OK;
}

static int phase_fft(sht_plan* p, bool inv, const double* in, double* out, cudaStream_t s) {
  prof_ev(p, inv ? 4 : 6, s);
  const FftParams fp = fft_params(p);
  for (int c = 1; c < kFftVariants; ++c) {
    if (inv)
      launch_fft(false, c, fp, p->fft_w0[c], p->fft_nw[c], nullptr, out, p->fft_smem[c], s);
    else
      launch_fft(true, c, fp, p->fft_w0[c], p->fft_nw[c], in, nullptr, p->fft_smem[c], s);
  }
  SHT_CUDA_TRY(cudaGetLastError());
  prof_ev(p, inv ? 5 : 7, s);
  return SHT_OK;
}

static void hist_advance(sht_plan* p, bool inv) {
  if (!(p->flags & SHT_FLAG_PROFILE_PHASES)) return;
  if (inv) {
    p->hist_inv[p->hist_cur] = true;
  } else {
    p->hist_cur = (p->hist_cur + 1) % sht_plan::kHist;
    p->hist_inv[p->hist_cur] = false;
    p->hist_done = std::min(p->hist_done + 1, sht_plan::kHist);
  }
}

}  // namespace sht

extern "C" {

// p2p transposition, per direction with epoch e: wait until every peer has
// drained the receive buffer this rank stores into (epoch e-1), run the
// producing kernel (its stores land in the peers' buffers), publish + wait
// "arrived" (phase_a2a), run the consuming kernel, publish "drained".
int sht_inv_trans(sht_plan* p, const double* spec, double* grid, void* stream) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  if (int rc = check_ptr(spec, "spec")) return rc;
  if (int rc = check_ptr(grid, "grid")) return rc;
  if (int rc = comm_check(p)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t e = ++p->inv_epoch;
  if (p->p2p)
    if (int rc = flags_op(p, -1, 0, kYFree, e - 1, s)) return rc;
  if (int rc = phase_leg(p, true, spec, nullptr, s)) return rc;
  if (int rc = phase_a2a(p, true, s)) return rc;
  if (int rc = phase_fft(p, true, nullptr, grid, s)) return rc;
  if (p->p2p)
    if (int rc = flags_op(p, kYFree, e, -1, 0, s)) return rc;
  hist_advance(p, true);
  return SHT_OK;
}

int sht_dir_trans(sht_plan* p, const double* grid, double* spec, void* stream) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  if (int rc = check_ptr(spec, "spec")) return rc;
  if (int rc = check_ptr(grid, "grid")) return rc;
  if (int rc = comm_check(p)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t e = ++p->dir_epoch;
  if (p->p2p)
    if (int rc = flags_op(p, -1, 0, kXFree, e - 1, s)) return rc;
  if (int rc = phase_fft(p, false, grid, nullptr, s)) return rc;
  if (int rc = phase_a2a(p, false, s)) return rc;
  if (int rc = phase_leg(p, false, nullptr, spec, s)) return rc;
  if (p->p2p)
    if (int rc = flags_op(p, kXFree, e, -1, 0, s)) return rc;
  hist_advance(p, false);
  return SHT_OK;
}

int sht_plan_set_gp_layout(sht_plan* p, int nA, int nB) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  if (nA < 1 || nB < 1 || nA * nB != p->nranks)
    return fail(SHT_ERR_CONFIG, "grid-point layout needs nA * nB == nranks");
  if (nA > p->g.ndgl) return fail(SHT_ERR_CONFIG, "more latitude bands than rings");
  for (int n : p->g.nloen)
    if (n < nB) return fail(SHT_ERR_CONFIG, "a ring has fewer points than longitude segments");
  if (p->gp.nA) return fail(SHT_ERR_CONFIG, "the grid-point layout is already set");
  std::vector<int> ring_rank(p->g.ndgl);
  for (int j = 0; j < p->g.ndgl; ++j) ring_rank[j] = p->ring_owner[std::min(j, p->g.ndgl - 1 - j)];
  if (gp_build(p->g.nloen, ring_rank, p->nranks, p->rank, nA, nB, p->gp))
    return fail(SHT_ERR_CONFIG, "grid-point layout too large");
  const size_t nf = (size_t)p->nfld;
  if (int rc = upload(&p->d_gp_send_idx, p->gp.send_idx)) return rc;
  if (int rc = upload(&p->d_gp_recv_idx, p->gp.recv_idx)) return rc;
  if (int rc = upload(&p->d_gp_send_displ, p->gp.send_displ)) return rc;
  if (int rc = upload(&p->d_gp_recv_displ, p->gp.recv_displ)) return rc;
  const size_t nb = std::max<size_t>(1, std::max(p->gp.send_idx.size(), p->gp.recv_idx.size())) * nf;
  SHT_CUDA_TRY(cudaMalloc((void**)&p->d_gridR, std::max<int64_t>(p->grid_ld, 1) * nf * sizeof(double)));
  SHT_CUDA_TRY(cudaMalloc((void**)&p->d_gp_buf0, nb * sizeof(double)));
  SHT_CUDA_TRY(cudaMalloc((void**)&p->d_gp_buf1, nb * sizeof(double)));
  return SHT_OK;
}

int sht_gp_layout(const sht_plan* p, int64_t* npts_gp, int32_t* band_lo, int32_t* band_hi, int32_t* segment,
                  int32_t* nsegments) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  if (!p->gp.nA) return fail(SHT_ERR_CONFIG, "no grid-point layout set (sht_plan_set_gp_layout)");
  const int a = p->rank / p->gp.nB, b = p->rank % p->gp.nB;
  if (npts_gp) *npts_gp = p->gp.npts_gp;
  if (band_lo) *band_lo = p->gp.band_lo[a];
  if (band_hi) *band_hi = p->gp.band_lo[a + 1];
  if (segment) *segment = b;
  if (nsegments) *nsegments = p->gp.nB;
  return SHT_OK;
}

}  // extern "C"

namespace sht {
// Grouped send/recv of [peer block][field][point] buffers in the rotated
// order (collectives.py:85-86); the self block is a device copy.
static int gp_exchange(sht_plan* p, const double* sbuf, const std::vector<int64_t>& sdispl, double* rbuf,
                       const std::vector<int64_t>& rdispl, cudaStream_t s) {
  const int P = p->nranks, r = p->rank;
  const int64_t nf = p->nfld;
  const int64_t self = sdispl[r + 1] - sdispl[r];
  if (self != rdispl[r + 1] - rdispl[r]) return fail(SHT_ERR_CONFIG, "grid-point layout self block mismatch");
  if (self)
    SHT_CUDA_TRY(cudaMemcpyAsync(rbuf + rdispl[r] * nf, sbuf + sdispl[r] * nf, self * nf * sizeof(double),
                                 cudaMemcpyDeviceToDevice, s));
  if (P == 1) return SHT_OK;
  if (p->failed || !p->comm) return comm_check(p);
  SHT_NCCL_TRY(ncclGroupStart());
  for (int k = 1; k < P; ++k) {
    const int to = (r + k) % P, from = (r - k + P) % P;
    const int64_t ns = sdispl[to + 1] - sdispl[to], nr = rdispl[from + 1] - rdispl[from];
    if (ns) SHT_NCCL_TRY(ncclSend(sbuf + sdispl[to] * nf, (size_t)(ns * nf), ncclDouble, to, p->comm, s));
    if (nr) SHT_NCCL_TRY(ncclRecv(rbuf + rdispl[from] * nf, (size_t)(nr * nf), ncclDouble, from, p->comm, s));
  }
  return nccl_settle(p, ncclGroupEnd(), "ncclGroupEnd (grid-point transposition)");
}
}  // namespace sht

extern "C" {

// inv_trans with the grid in the 2-D grid-point layout: the ring-pair grid
// goes through the plan's buffer, then ring -> grid point (TRLTOG role).
int sht_inv_trans_gp(sht_plan* p, const double* spec, double* grid_gp, void* stream) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  if (!p->gp.nA) return fail(SHT_ERR_CONFIG, "no grid-point layout set (sht_plan_set_gp_layout)");
  if (int rc = check_ptr(grid_gp, "grid")) return rc;
  if (p->nranks == 1) return sht_inv_trans(p, spec, grid_gp, stream);  // 1 x 1 layout == ring layout
  if (int rc = sht_inv_trans(p, spec, p->d_gridR, stream)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const GpLayout& L = p->gp;
  gp_launch_pack(p->d_gridR, p->grid_ld, p->d_gp_send_idx, p->d_gp_send_displ, p->nranks,
                 (int64_t)L.send_idx.size(), p->nfld, p->d_gp_buf0, s);
  if (int rc = gp_exchange(p, p->d_gp_buf0, L.send_displ, p->d_gp_buf1, L.recv_displ, s)) return rc;
  gp_launch_unpack(p->d_gp_buf1, p->d_gp_recv_idx, p->d_gp_recv_displ, p->nranks, (int64_t)L.recv_idx.size(),
                   p->nfld, grid_gp, L.npts_gp, s);
  SHT_CUDA_TRY(cudaGetLastError());
  return SHT_OK;
}

// dir_trans from the 2-D grid-point layout: grid point -> ring (TRGTOL role),
// then the ring-pair transform.
int sht_dir_trans_gp(sht_plan* p, const double* grid_gp, double* spec, void* stream) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  if (!p->gp.nA) return fail(SHT_ERR_CONFIG, "no grid-point layout set (sht_plan_set_gp_layout)");
  if (int rc = check_ptr(grid_gp, "grid")) return rc;
  if (p->nranks == 1) return sht_dir_trans(p, grid_gp, spec, stream);
  if (int rc = comm_check(p)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const GpLayout& L = p->gp;
  gp_launch_pack(grid_gp, L.npts_gp, p->d_gp_recv_idx, p->d_gp_recv_displ, p->nranks, (int64_t)L.recv_idx.size(),
                 p->nfld, p->d_gp_buf1, s);
  if (int rc = gp_exchange(p, p->d_gp_buf1, L.recv_displ, p->d_gp_buf0, L.send_displ, s)) return rc;
  gp_launch_unpack(p->d_gp_buf0, p->d_gp_send_idx, p->d_gp_send_displ, p->nranks, (int64_t)L.send_idx.size(),
                   p->nfld, p->d_gridR, p->grid_ld, s);
  SHT_CUDA_TRY(cudaGetLastError());
  return sht_dir_trans(p, p->d_gridR, spec, stream);
}

int sht_gp_bands(int truncation, int ndgl, const int32_t* nloen, int nA, int32_t* band_lo) {
  Geometry g;
  if (int rc = make_geometry(truncation, ndgl, nloen, g)) return rc;
  if (nA < 1 || nA > g.ndgl) return fail(SHT_ERR_CONFIG, "invalid number of latitude bands");
  std::vector<int> b;
  gp_bands(g.nloen, nA, b);
  if (band_lo) std::copy(b.begin(), b.end(), band_lo);
  return SHT_OK;
}

int sht_transport(const sht_plan* p, int* p2p) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  if (p2p) *p2p = (p->p2p ? 1 : 0) | (p->fblk ? 2 : 0);
  return SHT_OK;
}

int sht_kernel_launches(const sht_plan* p, int* per_pair) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  int fft = 0;
  for (int c = 1; c < kFftVariants; ++c) fft += p->fft_nw[c] > 0;
  const int leg = p->chunks.empty() ? (p->ntiles_inv > 0) + (p->ntiles_dir > 0) : 4 * (int)p->chunks.size();
  const int sync = p->p2p ? 6 : 0;  // flag handshakes (the NCCL path's kernels are NCCL's)
  if (per_pair) *per_pair = leg + 2 * fft + sync;
  return SHT_OK;
}

int sht_phase_ms(sht_plan* p, float* ms, int n) { return sht_phase_ms_avg(p, 1, ms, n); }

int sht_phase_ms_avg(sht_plan* p, int npairs, float* ms, int n) {
  if (!p) return fail(SHT_ERR_CONFIG, "plan is NULL");
  if (!(p->flags & SHT_FLAG_PROFILE_PHASES)) return fail(SHT_ERR_CONFIG, "plan was created without SHT_FLAG_PROFILE_PHASES");
  if (npairs < 1 || npairs > p->hist_done) return fail(SHT_ERR_CONFIG, "npairs must be in [1, completed pairs <= 64]");
  double v[7] = {p->setup_ms, 0, 0, 0, 0, 0, 0};
  for (int q = 1; q <= npairs; ++q) {
    const int slot = (p->hist_cur - q + sht_plan::kHist) % sht_plan::kHist;
    cudaEvent_t* e = p->hist[slot];
    SHT_CUDA_TRY(cudaEventSynchronize(e[11]));
    for (int k = 0; k < 6; ++k) {
      if (k < 3 && !p->hist_inv[slot]) continue;  // a direct transform without a preceding inverse
      float t = 0.f;
      SHT_CUDA_TRY(cudaEventElapsedTime(&t, e[2 * k], e[2 * k + 1]));
      v[k + 1] += t / npairs;
    }
  }
  for (int k = 0; k < n && k < 7; ++k) ms[k] = (float)v[k];
  return SHT_OK;
}

}  // extern "C"

// Ring FFTs of the SH transform on sm_100a (K4 fft_g2f: grid -> Fourier,
// K5 fft_f2g: Fourier -> grid) on the variable-length octahedral rings.
//
// One CTA owns one ring PAIR (northern ring i and its southern mirror, same
// length N) for a group of field pairs.  Two real fields are packed into one
// complex sequence (z = x_a + i x_b), so every transform is a complex DFT of
// length N; the pair is separated with Z_m / conj(Z_{N-m}).  The transform is
// a self-sorting Stockham FFT ping-ponging between two shared-memory buffers:
// in every radix stage a thread takes a butterfly, twiddles its R inputs
// (table W_L in global memory, L1-resident), runs a radix-R codelet (R in
// {2,3,4,5,7,8,11,13}) and writes the outputs; one barrier per stage.
// Rings whose length has a prime factor > 13 use Bluestein's algorithm with a
// 7-smooth length L >= 2N-1 (SURVEY.md section 7 discusses why factor-local
// Rader is the eventual target; this is the round-1 plan).
//
// Fusions: g2f scales by 1/N, and combines the two hemispheres into the
// parity rows the Legendre GEMM consumes, S' = w_i (F_N + F_S) and
// A' = w_i (F_N - F_S) (Gaussian weight folded in).  f2g reads S, A rows and
// forms F_N = S + A, F_S = S - A while filling its FFT buffer.  Fourier rows
// are addressed through yrow[] so the same kernels read/write the all-to-all
// receive/send buffers directly (pack/unpack fused).
#include "sht_internal.h"

namespace sht {

namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 conjc(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // -i * a
__device__ __forceinline__ double2 mul_pi(double2 a) { return make_double2(-a.y, a.x); }  // +i * a

// Forward DFT codelets (exp(-2 pi i jk / R)), in place.  Odd primes pair x_j with
// x_{R-j}: X_k = x0 + sum_j t_j cos(2 pi jk/R) - i u_j sin(2 pi jk/R), t = x_j + x_{R-j},
// u = x_j - x_{R-j}; constants are generated literals (correctly rounded doubles).
template <int R>
__device__ __forceinline__ void dft(double2 (&v)[R]);

template <>
__device__ __forceinline__ void dft<3>(double2 (&v)[3]) {
  const double2 t1 = cadd(v[1], v[2]), u1 = csub(v[1], v[2]);
  const double2 x0 = v[0];
  v[0] = make_double2(x0.x + t1.x, x0.y + t1.y);
  {
    const double rx = fma(t1.x, -0.5, x0.x);
    const double ry = fma(t1.y, -0.5, x0.y);
    const double ix = u1.x * 0.8660254037844386;
    const double iy = u1.y * 0.8660254037844386;
    v[1] = make_double2(rx + iy, ry - ix);
    v[2] = make_double2(rx - iy, ry + ix);
  }
}

template <>
__device__ __forceinline__ void dft<5>(double2 (&v)[5]) {
  const double2 t1 = cadd(v[1], v[4]), u1 = csub(v[1], v[4]);
  const double2 t2 = cadd(v[2], v[3]), u2 = csub(v[2], v[3]);
  const double2 x0 = v[0];
  v[0] = make_double2(x0.x + t1.x + t2.x, x0.y + t1.y + t2.y);
  {
    const double rx = fma(t2.x, -0.8090169943749475, fma(t1.x, 0.30901699437494745, x0.x));
    const double ry = fma(t2.y, -0.8090169943749475, fma(t1.y, 0.30901699437494745, x0.y));
    const double ix = fma(u2.x, 0.5877852522924731, u1.x * 0.9510565162951535);
    const double iy = fma(u2.y, 0.5877852522924731, u1.y * 0.9510565162951535);
    v[1] = make_double2(rx + iy, ry - ix);
    v[4] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t2.x, 0.30901699437494745, fma(t1.x, -0.8090169943749475, x0.x));
    const double ry = fma(t2.y, 0.30901699437494745, fma(t1.y, -0.8090169943749475, x0.y));
    const double ix = fma(u2.x, -0.9510565162951535, u1.x * 0.5877852522924731);
    const double iy = fma(u2.y, -0.9510565162951535, u1.y * 0.5877852522924731);
    v[2] = make_double2(rx + iy, ry - ix);
    v[3] = make_double2(rx - iy, ry + ix);
  }
}

template <>
__device__ __forceinline__ void dft<7>(double2 (&v)[7]) {
  const double2 t1 = cadd(v[1], v[6]), u1 = csub(v[1], v[6]);
  const double2 t2 = cadd(v[2], v[5]), u2 = csub(v[2], v[5]);
  const double2 t3 = cadd(v[3], v[4]), u3 = csub(v[3], v[4]);
  const double2 x0 = v[0];
  v[0] = make_double2(x0.x + t1.x + t2.x + t3.x, x0.y + t1.y + t2.y + t3.y);
  {
    const double rx = fma(t3.x, -0.9009688679024191, fma(t2.x, -0.2225209339563144, fma(t1.x, 0.6234898018587335, x0.x)));
    const double ry = fma(t3.y, -0.9009688679024191, fma(t2.y, -0.2225209339563144, fma(t1.y, 0.6234898018587335, x0.y)));
    const double ix = fma(u3.x, 0.4338837391175581, fma(u2.x, 0.9749279121818236, u1.x * 0.7818314824680298));
    const double iy = fma(u3.y, 0.4338837391175581, fma(u2.y, 0.9749279121818236, u1.y * 0.7818314824680298));
    v[1] = make_double2(rx + iy, ry - ix);
    v[6] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t3.x, 0.6234898018587335, fma(t2.x, -0.9009688679024191, fma(t1.x, -0.2225209339563144, x0.x)));
    const double ry = fma(t3.y, 0.6234898018587335, fma(t2.y, -0.9009688679024191, fma(t1.y, -0.2225209339563144, x0.y)));
    const double ix = fma(u3.x, -0.7818314824680298, fma(u2.x, -0.4338837391175581, u1.x * 0.9749279121818236));
    const double iy = fma(u3.y, -0.7818314824680298, fma(u2.y, -0.4338837391175581, u1.y * 0.9749279121818236));
    v[2] = make_double2(rx + iy, ry - ix);
    v[5] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t3.x, -0.2225209339563144, fma(t2.x, 0.6234898018587335, fma(t1.x, -0.9009688679024191, x0.x)));
    const double ry = fma(t3.y, -0.2225209339563144, fma(t2.y, 0.6234898018587335, fma(t1.y, -0.9009688679024191, x0.y)));
    const double ix = fma(u3.x, 0.9749279121818236, fma(u2.x, -0.7818314824680298, u1.x * 0.4338837391175581));
    const double iy = fma(u3.y, 0.9749279121818236, fma(u2.y, -0.7818314824680298, u1.y * 0.4338837391175581));
    v[3] = make_double2(rx + iy, ry - ix);
    v[4] = make_double2(rx - iy, ry + ix);
  }
}

template <>
__device__ __forceinline__ void dft<11>(double2 (&v)[11]) {
  const double2 t1 = cadd(v[1], v[10]), u1 = csub(v[1], v[10]);
  const double2 t2 = cadd(v[2], v[9]), u2 = csub(v[2], v[9]);
  const double2 t3 = cadd(v[3], v[8]), u3 = csub(v[3], v[8]);
  const double2 t4 = cadd(v[4], v[7]), u4 = csub(v[4], v[7]);
  const double2 t5 = cadd(v[5], v[6]), u5 = csub(v[5], v[6]);
  const double2 x0 = v[0];
  v[0] = make_double2(x0.x + t1.x + t2.x + t3.x + t4.x + t5.x, x0.y + t1.y + t2.y + t3.y + t4.y + t5.y);
  {
    const double rx = fma(t5.x, -0.9594929736144974, fma(t4.x, -0.6548607339452851, fma(t3.x, -0.14231483827328514, fma(t2.x, 0.41541501300188644, fma(t1.x, 0.8412535328311812, x0.x)))));
    const double ry = fma(t5.y, -0.9594929736144974, fma(t4.y, -0.6548607339452851, fma(t3.y, -0.14231483827328514, fma(t2.y, 0.41541501300188644, fma(t1.y, 0.8412535328311812, x0.y)))));
    const double ix = fma(u5.x, 0.28173255684142967, fma(u4.x, 0.7557495743542583, fma(u3.x, 0.9898214418809327, fma(u2.x, 0.9096319953545183, u1.x * 0.5406408174555976))));
    const double iy = fma(u5.y, 0.28173255684142967, fma(u4.y, 0.7557495743542583, fma(u3.y, 0.9898214418809327, fma(u2.y, 0.9096319953545183, u1.y * 0.5406408174555976))));
    v[1] = make_double2(rx + iy, ry - ix);
    v[10] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t5.x, 0.8412535328311812, fma(t4.x, -0.14231483827328514, fma(t3.x, -0.9594929736144974, fma(t2.x, -0.6548607339452851, fma(t1.x, 0.41541501300188644, x0.x)))));
    const double ry = fma(t5.y, 0.8412535328311812, fma(t4.y, -0.14231483827328514, fma(t3.y, -0.9594929736144974, fma(t2.y, -0.6548607339452851, fma(t1.y, 0.41541501300188644, x0.y)))));
    const double ix = fma(u5.x, -0.5406408174555976, fma(u4.x, -0.9898214418809327, fma(u3.x, -0.28173255684142967, fma(u2.x, 0.7557495743542583, u1.x * 0.9096319953545183))));
    const double iy = fma(u5.y, -0.5406408174555976, fma(u4.y, -0.9898214418809327, fma(u3.y, -0.28173255684142967, fma(u2.y, 0.7557495743542583, u1.y * 0.9096319953545183))));
    v[2] = make_double2(rx + iy, ry - ix);
    v[9] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t5.x, -0.6548607339452851, fma(t4.x, 0.8412535328311812, fma(t3.x, 0.41541501300188644, fma(t2.x, -0.9594929736144974, fma(t1.x, -0.14231483827328514, x0.x)))));
    const double ry = fma(t5.y, -0.6548607339452851, fma(t4.y, 0.8412535328311812, fma(t3.y, 0.41541501300188644, fma(t2.y, -0.9594929736144974, fma(t1.y, -0.14231483827328514, x0.y)))));
    const double ix = fma(u5.x, 0.7557495743542583, fma(u4.x, 0.5406408174555976, fma(u3.x, -0.9096319953545183, fma(u2.x, -0.28173255684142967, u1.x * 0.9898214418809327))));
    const double iy = fma(u5.y, 0.7557495743542583, fma(u4.y, 0.5406408174555976, fma(u3.y, -0.9096319953545183, fma(u2.y, -0.28173255684142967, u1.y * 0.9898214418809327))));
    v[3] = make_double2(rx + iy, ry - ix);
    v[8] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t5.x, 0.41541501300188644, fma(t4.x, -0.9594929736144974, fma(t3.x, 0.8412535328311812, fma(t2.x, -0.14231483827328514, fma(t1.x, -0.6548607339452851, x0.x)))));
    const double ry = fma(t5.y, 0.41541501300188644, fma(t4.y, -0.9594929736144974, fma(t3.y, 0.8412535328311812, fma(t2.y, -0.14231483827328514, fma(t1.y, -0.6548607339452851, x0.y)))));
    const double ix = fma(u5.x, -0.9096319953545183, fma(u4.x, 0.28173255684142967, fma(u3.x, 0.5406408174555976, fma(u2.x, -0.9898214418809327, u1.x * 0.7557495743542583))));
    const double iy = fma(u5.y, -0.9096319953545183, fma(u4.y, 0.28173255684142967, fma(u3.y, 0.5406408174555976, fma(u2.y, -0.9898214418809327, u1.y * 0.7557495743542583))));
    v[4] = make_double2(rx + iy, ry - ix);
    v[7] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t5.x, -0.14231483827328514, fma(t4.x, 0.41541501300188644, fma(t3.x, -0.6548607339452851, fma(t2.x, 0.8412535328311812, fma(t1.x, -0.9594929736144974, x0.x)))));
    const double ry = fma(t5.y, -0.14231483827328514, fma(t4.y, 0.41541501300188644, fma(t3.y, -0.6548607339452851, fma(t2.y, 0.8412535328311812, fma(t1.y, -0.9594929736144974, x0.y)))));
    const double ix = fma(u5.x, 0.9898214418809327, fma(u4.x, -0.9096319953545183, fma(u3.x, 0.7557495743542583, fma(u2.x, -0.5406408174555976, u1.x * 0.28173255684142967))));
    const double iy = fma(u5.y, 0.9898214418809327, fma(u4.y, -0.9096319953545183, fma(u3.y, 0.7557495743542583, fma(u2.y, -0.5406408174555976, u1.y * 0.28173255684142967))));
    v[5] = make_double2(rx + iy, ry - ix);
    v[6] = make_double2(rx - iy, ry + ix);
  }
}

template <>
__device__ __forceinline__ void dft<13>(double2 (&v)[13]) {
  const double2 t1 = cadd(v[1], v[12]), u1 = csub(v[1], v[12]);
  const double2 t2 = cadd(v[2], v[11]), u2 = csub(v[2], v[11]);
  const double2 t3 = cadd(v[3], v[10]), u3 = csub(v[3], v[10]);
  const double2 t4 = cadd(v[4], v[9]), u4 = csub(v[4], v[9]);
  const double2 t5 = cadd(v[5], v[8]), u5 = csub(v[5], v[8]);
  const double2 t6 = cadd(v[6], v[7]), u6 = csub(v[6], v[7]);
  const double2 x0 = v[0];
  v[0] = make_double2(x0.x + t1.x + t2.x + t3.x + t4.x + t5.x + t6.x, x0.y + t1.y + t2.y + t3.y + t4.y + t5.y + t6.y);
  {
    const double rx = fma(t6.x, -0.970941817426052, fma(t5.x, -0.7485107481711011, fma(t4.x, -0.3546048870425356, fma(t3.x, 0.12053668025532305, fma(t2.x, 0.5680647467311558, fma(t1.x, 0.8854560256532099, x0.x))))));
    const double ry = fma(t6.y, -0.970941817426052, fma(t5.y, -0.7485107481711011, fma(t4.y, -0.3546048870425356, fma(t3.y, 0.12053668025532305, fma(t2.y, 0.5680647467311558, fma(t1.y, 0.8854560256532099, x0.y))))));
    const double ix = fma(u6.x, 0.23931566428755777, fma(u5.x, 0.6631226582407952, fma(u4.x, 0.9350162426854148, fma(u3.x, 0.992708874098054, fma(u2.x, 0.8229838658936564, u1.x * 0.46472317204376856)))));
    const double iy = fma(u6.y, 0.23931566428755777, fma(u5.y, 0.6631226582407952, fma(u4.y, 0.9350162426854148, fma(u3.y, 0.992708874098054, fma(u2.y, 0.8229838658936564, u1.y * 0.46472317204376856)))));
    v[1] = make_double2(rx + iy, ry - ix);
    v[12] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t6.x, 0.8854560256532099, fma(t5.x, 0.12053668025532305, fma(t4.x, -0.7485107481711011, fma(t3.x, -0.970941817426052, fma(t2.x, -0.3546048870425356, fma(t1.x, 0.5680647467311558, x0.x))))));
    const double ry = fma(t6.y, 0.8854560256532099, fma(t5.y, 0.12053668025532305, fma(t4.y, -0.7485107481711011, fma(t3.y, -0.970941817426052, fma(t2.y, -0.3546048870425356, fma(t1.y, 0.5680647467311558, x0.y))))));
    const double ix = fma(u6.x, -0.46472317204376856, fma(u5.x, -0.992708874098054, fma(u4.x, -0.6631226582407952, fma(u3.x, 0.23931566428755777, fma(u2.x, 0.9350162426854148, u1.x * 0.8229838658936564)))));
    const double iy = fma(u6.y, -0.46472317204376856, fma(u5.y, -0.992708874098054, fma(u4.y, -0.6631226582407952, fma(u3.y, 0.23931566428755777, fma(u2.y, 0.9350162426854148, u1.y * 0.8229838658936564)))));
    v[2] = make_double2(rx + iy, ry - ix);
    v[11] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t6.x, -0.7485107481711011, fma(t5.x, 0.5680647467311558, fma(t4.x, 0.8854560256532099, fma(t3.x, -0.3546048870425356, fma(t2.x, -0.970941817426052, fma(t1.x, 0.12053668025532305, x0.x))))));
    const double ry = fma(t6.y, -0.7485107481711011, fma(t5.y, 0.5680647467311558, fma(t4.y, 0.8854560256532099, fma(t3.y, -0.3546048870425356, fma(t2.y, -0.970941817426052, fma(t1.y, 0.12053668025532305, x0.y))))));
    const double ix = fma(u6.x, 0.6631226582407952, fma(u5.x, 0.8229838658936564, fma(u4.x, -0.46472317204376856, fma(u3.x, -0.9350162426854148, fma(u2.x, 0.23931566428755777, u1.x * 0.992708874098054)))));
    const double iy = fma(u6.y, 0.6631226582407952, fma(u5.y, 0.8229838658936564, fma(u4.y, -0.46472317204376856, fma(u3.y, -0.9350162426854148, fma(u2.y, 0.23931566428755777, u1.y * 0.992708874098054)))));
    v[3] = make_double2(rx + iy, ry - ix);
    v[10] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t6.x, 0.5680647467311558, fma(t5.x, -0.970941817426052, fma(t4.x, 0.12053668025532305, fma(t3.x, 0.8854560256532099, fma(t2.x, -0.7485107481711011, fma(t1.x, -0.3546048870425356, x0.x))))));
    const double ry = fma(t6.y, 0.5680647467311558, fma(t5.y, -0.970941817426052, fma(t4.y, 0.12053668025532305, fma(t3.y, 0.8854560256532099, fma(t2.y, -0.7485107481711011, fma(t1.y, -0.3546048870425356, x0.y))))));
    const double ix = fma(u6.x, -0.8229838658936564, fma(u5.x, -0.23931566428755777, fma(u4.x, 0.992708874098054, fma(u3.x, -0.46472317204376856, fma(u2.x, -0.6631226582407952, u1.x * 0.9350162426854148)))));
    const double iy = fma(u6.y, -0.8229838658936564, fma(u5.y, -0.23931566428755777, fma(u4.y, 0.992708874098054, fma(u3.y, -0.46472317204376856, fma(u2.y, -0.6631226582407952, u1.y * 0.9350162426854148)))));
    v[4] = make_double2(rx + iy, ry - ix);
    v[9] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t6.x, -0.3546048870425356, fma(t5.x, 0.8854560256532099, fma(t4.x, -0.970941817426052, fma(t3.x, 0.5680647467311558, fma(t2.x, 0.12053668025532305, fma(t1.x, -0.7485107481711011, x0.x))))));
    const double ry = fma(t6.y, -0.3546048870425356, fma(t5.y, 0.8854560256532099, fma(t4.y, -0.970941817426052, fma(t3.y, 0.5680647467311558, fma(t2.y, 0.12053668025532305, fma(t1.y, -0.7485107481711011, x0.y))))));
    const double ix = fma(u6.x, 0.9350162426854148, fma(u5.x, -0.46472317204376856, fma(u4.x, -0.23931566428755777, fma(u3.x, 0.8229838658936564, fma(u2.x, -0.992708874098054, u1.x * 0.6631226582407952)))));
    const double iy = fma(u6.y, 0.9350162426854148, fma(u5.y, -0.46472317204376856, fma(u4.y, -0.23931566428755777, fma(u3.y, 0.8229838658936564, fma(u2.y, -0.992708874098054, u1.y * 0.6631226582407952)))));
    v[5] = make_double2(rx + iy, ry - ix);
    v[8] = make_double2(rx - iy, ry + ix);
  }
  {
    const double rx = fma(t6.x, 0.12053668025532305, fma(t5.x, -0.3546048870425356, fma(t4.x, 0.5680647467311558, fma(t3.x, -0.7485107481711011, fma(t2.x, 0.8854560256532099, fma(t1.x, -0.970941817426052, x0.x))))));
    const double ry = fma(t6.y, 0.12053668025532305, fma(t5.y, -0.3546048870425356, fma(t4.y, 0.5680647467311558, fma(t3.y, -0.7485107481711011, fma(t2.y, 0.8854560256532099, fma(t1.y, -0.970941817426052, x0.y))))));
    const double ix = fma(u6.x, -0.992708874098054, fma(u5.x, 0.9350162426854148, fma(u4.x, -0.8229838658936564, fma(u3.x, 0.6631226582407952, fma(u2.x, -0.46472317204376856, u1.x * 0.23931566428755777)))));
    const double iy = fma(u6.y, -0.992708874098054, fma(u5.y, 0.9350162426854148, fma(u4.y, -0.8229838658936564, fma(u3.y, 0.6631226582407952, fma(u2.y, -0.46472317204376856, u1.y * 0.23931566428755777)))));
    v[6] = make_double2(rx + iy, ry - ix);
    v[7] = make_double2(rx - iy, ry + ix);
  }
}

template <>
__device__ __forceinline__ void dft<2>(double2 (&v)[2]) {
  const double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <>
__device__ __forceinline__ void dft<4>(double2 (&v)[4]) {
  const double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
  const double2 s13 = cadd(v[1], v[3]), d13 = csub(v[1], v[3]);
  v[0] = cadd(s02, s13);
  v[2] = csub(s02, s13);
  v[1] = cadd(d02, mul_mi(d13));
  v[3] = cadd(d02, mul_pi(d13));
}

template <>
__device__ __forceinline__ void dft<8>(double2 (&v)[8]) {
  constexpr double h = 0.70710678118654752440;
  double2 e[4] = {v[0], v[2], v[4], v[6]};
  double2 o[4] = {v[1], v[3], v[5], v[7]};
  dft<4>(e);
  dft<4>(o);
  // o_k *= exp(-2 pi i k / 8)
  o[1] = make_double2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
  o[2] = mul_mi(o[2]);
  o[3] = make_double2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = cadd(e[k], o[k]);
    v[k + 4] = csub(e[k], o[k]);
  }
}

// One Stockham radix-R stage (out of place, in -> out) over nseq sequences of
// length L in shared memory; span Ns = product of the radices already applied.
template <int R>
__device__ __forceinline__ void stage(const double2* __restrict__ in, double2* __restrict__ out, int L, int nseq,
                                      int Ns, const double2* __restrict__ W) {
  const int nbf = L / R;
  const int total = nseq * nbf;
  const int tstride = nbf / Ns;  // L / (Ns R)
  for (int b = threadIdx.x; b < total; b += kFftThreads) {
    const int s = b / nbf;
    const int j = b - s * nbf;
    const double2* ip = in + s * L + j;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = ip[r * nbf];
    const int k = j % Ns;
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(W + r * k * tstride));
    }
    dft<R>(v);
    double2* op = out + s * L + (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) op[r * Ns] = v[r];
  }
  __syncthreads();
}

// Forward DFT of nseq sequences of length L held in a (caller synced); b is
// scratch of the same size.  Returns the buffer holding the result.
__device__ double2* fft_run(double2* a, double2* b, int L, int nseq, const FftRing& rg,
                            const double2* __restrict__ W) {
  int Ns = 1;
  for (int s = 0; s < rg.nstage; ++s) {
    switch (rg.radix[s]) {
      case 2: stage<2>(a, b, L, nseq, Ns, W); Ns *= 2; break;
      case 3: stage<3>(a, b, L, nseq, Ns, W); Ns *= 3; break;
      case 4: stage<4>(a, b, L, nseq, Ns, W); Ns *= 4; break;
      case 5: stage<5>(a, b, L, nseq, Ns, W); Ns *= 5; break;
      case 7: stage<7>(a, b, L, nseq, Ns, W); Ns *= 7; break;
      case 8: stage<8>(a, b, L, nseq, Ns, W); Ns *= 8; break;
      case 11: stage<11>(a, b, L, nseq, Ns, W); Ns *= 11; break;
      case 13: stage<13>(a, b, L, nseq, Ns, W); Ns *= 13; break;
      default: break;
    }
    double2* t = a;
    a = b;
    b = t;
  }
  return a;
}

// Bluestein: X = FFT(a); X <- conj(X * bhat); FFT again.  Returns the result buffer.
__device__ double2* bluestein_run(double2* a, double2* b, int L, int nseq, const FftRing& rg,
                                  const double2* __restrict__ W, const double2* __restrict__ bhat) {
  double2* x = fft_run(a, b, L, nseq, rg, W);
  for (int idx = threadIdx.x; idx < nseq * L; idx += kFftThreads) {
    const int k = idx % L;
    x[idx] = conjc(cmul(x[idx], __ldg(bhat + k)));
  }
  __syncthreads();
  return fft_run(x, x == a ? b : a, L, nseq, rg, W);
}

// ------------------------------------------------------------------ grid -> Fourier
__global__ void __launch_bounds__(kFftThreads, 1)
    fft_g2f_kernel(const FftParams p, int w0, const double* __restrict__ grid, double* __restrict__ four) {
  extern __shared__ __align__(16) double2 smc[];
  const FftWork wk = p.work[w0 + blockIdx.x];
  const FftRing rg = p.rings[wk.ring];
  const int N = rg.n, L = rg.L, M = rg.mcap;
  const int npairs = (p.nfld + 1) / 2;
  const int nfp = min(rg.fp, npairs - wk.fp0);
  const int nseq = 2 * nfp;
  const int ncol = 2 * nfp;  // staged fields
  double2* buf = smc;                          // ping
  double2* buf2 = smc + (size_t)rg.nb * L;     // pong
  double2* stg = buf2 + (size_t)rg.nb * L;     // [side][m][field]
  const double2* W = p.tw + rg.tw_off;
  const bool blue = rg.chirp_off >= 0;
  const double2* chirp = p.tw + (blue ? rg.chirp_off : 0);
  const double2* bhat = p.tw + (blue ? rg.bhat_off : 0);
  const double scale = 0.5 / N;

  for (int q0 = 0; q0 < nseq; q0 += rg.nb) {
    const int nq = min(rg.nb, nseq - q0);
    for (int idx = threadIdx.x; idx < nq * L; idx += kFftThreads) {
      const int ql = idx / L, n = idx - ql * L;
      const int q = q0 + ql;
      const int side = q / nfp, pr = q - side * nfp;
      double2 z = make_double2(0.0, 0.0);
      if (n < N) {
        const int fa = 2 * (wk.fp0 + pr);
        const int64_t go = (side ? rg.goff_s : rg.goff_n) + n;
        z.x = grid[(int64_t)fa * p.grid_ld + go];
        if (fa + 1 < p.nfld) z.y = grid[(int64_t)(fa + 1) * p.grid_ld + go];
        if (blue) z = cmul(z, __ldg(chirp + n));
      }
      buf[idx] = z;
    }
    __syncthreads();
    const double2* res = blue ? bluestein_run(buf, buf2, L, nq, rg, W, bhat) : fft_run(buf, buf2, L, nq, rg, W);
    for (int idx = threadIdx.x; idx < nq * (M + 1); idx += kFftThreads) {
      const int ql = idx / (M + 1), m = idx - ql * (M + 1);
      const int q = q0 + ql;
      const int side = q / nfp, pr = q - side * nfp;
      const int k2 = (m == 0) ? 0 : N - m;
      double2 zm = res[ql * L + m], zn = res[ql * L + k2];
      if (blue) {
        zm = cmul(__ldg(chirp + m), conjc(zm));
        zn = cmul(__ldg(chirp + k2), conjc(zn));
      }
      const double2 fa = make_double2((zm.x + zn.x) * scale, (zm.y - zn.y) * scale);
      const double2 fb = make_double2((zm.y + zn.y) * scale, (zn.x - zm.x) * scale);
      double2* st = stg + ((size_t)side * (M + 1) + m) * ncol + 2 * pr;
      st[0] = fa;
      st[1] = fb;
    }
    __syncthreads();
  }

  const int nf = min(ncol, p.nfld - 2 * wk.fp0);
  const double w = rg.w;
  const int64_t rowd = (int64_t)p.nfld * 4;
  for (int idx = threadIdx.x; idx < (M + 1) * nf; idx += kFftThreads) {
    const int m = idx / nf, f = idx - m * nf;
    const double2 a = stg[(size_t)m * ncol + f];
    const double2 b = stg[((size_t)(M + 1) + m) * ncol + f];
    const int64_t row = p.yrow[rg.yrow_off + m];
    double2* d = reinterpret_cast<double2*>(four + row * rowd + (int64_t)(2 * wk.fp0 + f) * 4);
    d[0] = make_double2(w * (a.x + b.x), w * (a.y + b.y));
    d[1] = make_double2(w * (a.x - b.x), w * (a.y - b.y));
  }
}

// ------------------------------------------------------------------ Fourier -> grid
__global__ void __launch_bounds__(kFftThreads, 1)
    fft_f2g_kernel(const FftParams p, int w0, const double* __restrict__ four, double* __restrict__ grid) {
  extern __shared__ __align__(16) double2 smc[];
  const FftWork wk = p.work[w0 + blockIdx.x];
  const FftRing rg = p.rings[wk.ring];
  const int N = rg.n, L = rg.L, M = rg.mcap;
  const int npairs = (p.nfld + 1) / 2;
  const int nfp = min(rg.fp, npairs - wk.fp0);
  const int nseq = 2 * nfp;
  const int ncol = 2 * nfp;
  double2* buf = smc;                          // ping
  double2* buf2 = smc + (size_t)rg.nb * L;     // pong
  double2* stgS = buf2 + (size_t)rg.nb * L;    // [m][field]
  double2* stgA = stgS + (size_t)(M + 1) * ncol;
  const double2* W = p.tw + rg.tw_off;
  const bool blue = rg.chirp_off >= 0;
  const double2* chirp = p.tw + (blue ? rg.chirp_off : 0);
  const double2* bhat = p.tw + (blue ? rg.bhat_off : 0);
  const int nf = min(ncol, p.nfld - 2 * wk.fp0);
  const int64_t rowd = (int64_t)p.nfld * 4;

  for (int idx = threadIdx.x; idx < (M + 1) * ncol; idx += kFftThreads) {
    const int m = idx / ncol, f = idx - m * ncol;
    double2 s = make_double2(0.0, 0.0), a = s;
    if (f < nf) {
      const int64_t row = p.yrow[rg.yrow_off + m];
      const double2* src = reinterpret_cast<const double2*>(four + row * rowd + (int64_t)(2 * wk.fp0 + f) * 4);
      s = src[0];
      a = src[1];
    }
    stgS[idx] = s;
    stgA[idx] = a;
  }
  __syncthreads();

  for (int q0 = 0; q0 < nseq; q0 += rg.nb) {
    const int nq = min(rg.nb, nseq - q0);
    for (int idx = threadIdx.x; idx < nq * L; idx += kFftThreads) {
      const int ql = idx / L, k = idx - ql * L;
      const int q = q0 + ql;
      const int side = q / nfp, pr = q - side * nfp;
      double2 z = make_double2(0.0, 0.0);
      int m = -1;
      bool lo = true;
      if (k <= M) {
        m = k;
      } else if (k < N && k >= N - M) {
        m = N - k;
        lo = false;
      }
      if (m >= 0) {
        const size_t o = (size_t)m * ncol + 2 * pr;
        const double2 sa = stgS[o], aa = stgA[o], sb = stgS[o + 1], ab = stgA[o + 1];
        double2 fa = side ? csub(sa, aa) : cadd(sa, aa);
        double2 fb = side ? csub(sb, ab) : cadd(sb, ab);
        if (m == 0) {
          fa.y = 0.0;
          fb.y = 0.0;
        }
        // Z = Fa + i Fb (low half) or conj(Fa) + i conj(Fb) (mirror half); feed conj(Z)
        z = lo ? make_double2(fa.x - fb.y, -(fa.y + fb.x)) : make_double2(fa.x + fb.y, fa.y - fb.x);
        if (blue) z = cmul(z, __ldg(chirp + k));
      }
      buf[idx] = z;
    }
    __syncthreads();
    const double2* res = blue ? bluestein_run(buf, buf2, L, nq, rg, W, bhat) : fft_run(buf, buf2, L, nq, rg, W);
    for (int idx = threadIdx.x; idx < nq * N; idx += kFftThreads) {
      const int ql = idx / N, k = idx - ql * N;
      const int q = q0 + ql;
      const int side = q / nfp, pr = q - side * nfp;
      double2 r = res[ql * L + k];
      if (blue) r = cmul(__ldg(chirp + k), conjc(r));
      const int fa = 2 * (wk.fp0 + pr);
      const int64_t go = (side ? rg.goff_s : rg.goff_n) + k;
      grid[(int64_t)fa * p.grid_ld + go] = r.x;
      if (fa + 1 < p.nfld) grid[(int64_t)(fa + 1) * p.grid_ld + go] = -r.y;
    }
    __syncthreads();
  }
}

}  // namespace

void launch_fft_g2f(const FftParams& p, int w0, int nw, const double* grid, double* four, size_t smem,
                    cudaStream_t s) {
  if (nw <= 0) return;
  cudaFuncSetAttribute(fft_g2f_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fft_g2f_kernel<<<nw, kFftThreads, smem, s>>>(p, w0, grid, four);
}

void launch_fft_f2g(const FftParams& p, int w0, int nw, const double* four, double* grid, size_t smem,
                    cudaStream_t s) {
  if (nw <= 0) return;
  cudaFuncSetAttribute(fft_f2g_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fft_f2g_kernel<<<nw, kFftThreads, smem, s>>>(p, w0, four, grid);
}

int fft_capacity(const std::vector<int>& radices) {
  (void)radices;
  return kFftMaxLen;
}

static bool factor_radices(int n, const int* allowed, int nallowed, std::vector<int>& radices) {
  radices.clear();
  int m = n;
  int twos = 0;
  while (m % 2 == 0) {
    m /= 2;
    ++twos;
  }
  for (int a = 0; a < nallowed; ++a) {
    const int p = allowed[a];
    while (m % p == 0) {
      radices.push_back(p);
      m /= p;
    }
  }
  if (m != 1) return false;
  std::vector<int> pw;
  while (twos >= 3) {
    pw.push_back(8);
    twos -= 3;
  }
  if (twos == 2) pw.push_back(4);
  if (twos == 1) pw.push_back(2);
  radices.insert(radices.begin(), pw.begin(), pw.end());
  return true;
}

int fft_choose(int n, std::vector<int>& radices, int& L, bool& bluestein) {
  static const int direct[] = {3, 5, 7, 11, 13};
  static const int smooth[] = {3, 5, 7};
  if (n >= 1 && factor_radices(n, direct, 5, radices) && (int)radices.size() <= kMaxStages &&
      fft_capacity(radices) >= n) {
    L = n;
    bluestein = false;
    return 0;
  }
  bluestein = true;
  for (int cand = 2 * n - 1; cand < 8 * n + 64; ++cand) {
    if (factor_radices(cand, smooth, 3, radices) && (int)radices.size() <= kMaxStages &&
        fft_capacity(radices) >= cand) {
      L = cand;
      return 0;
    }
  }
  return SHT_ERR_CONFIG;
}

}  // namespace sht

// Ring-FFT kernels for the field-blocked Fourier-row layout (p2p transposition
// past the remote-store translation cliff, sht_internal.h); the device code is
// fft_kernels.cuh, shared with sht_fft.cu.
#include "fft_kernels.cuh"

namespace sht {

void fft_preload_blk() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, fft_g2f_kernel<1, true>);
  cudaFuncGetAttributes(&a, fft_f2g_kernel<1, true>);
  cudaFuncGetAttributes(&a, fft_g2f_kernel<3, true>);
  cudaFuncGetAttributes(&a, fft_f2g_kernel<3, true>);
}

void launch_fft_blk(bool g2f, int variant, const FftParams& p, int w0, int nw, const double* in, double* out,
                    size_t smem, cudaStream_t s) {
  if (variant == 1) launch_one<1, true>(g2f, p, w0, nw, in, out, smem, s);
  if (variant == 3) launch_one<3, true>(g2f, p, w0, nw, in, out, smem, s);
}

}  // namespace sht

// DMMA feed probe: what rate does the Legendre inner-loop shape reach?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
// MODE 0: constant fragments, 32 accumulators; MODE 1: fragments from smem (8 LDS.128 per 32 DMMA)
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(double* out, int iters) {
  extern __shared__ __align__(16) double sm[];
  for (int i = threadIdx.x; i < 8192; i += 256) sm[i] = 1.0 + i * 1e-6;
  __syncthreads();
  double acc[4][2][4][2] = {};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* Ps = sm + ((warp & 1) * 32 + (lane >> 2)) * 40 + 2 * (lane & 3);
  const double* Ss = sm + 2560 + ((warp >> 1) * 16 + (lane >> 2)) * 66 + 4 * (lane & 3);
  double2 a[4], bs[2], ba[2];
  for (int g = 0; g < 4; ++g) a[g] = make_double2(1.0 + g, 2.0);
  for (int h = 0; h < 2; ++h) { bs[h] = make_double2(0.5, 0.25); ba[h] = make_double2(0.125, 1.5); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int sub = 0; sub < 4; ++sub) {
      if (MODE == 1) {
#pragma unroll
        for (int g = 0; g < 4; ++g) a[g] = *reinterpret_cast<const double2*>(Ps + g * 8 * 40 + sub * 8);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double* bp = Ss + h * 8 * 66 + sub * 16;
          bs[h] = *reinterpret_cast<const double2*>(bp);
          ba[h] = *reinterpret_cast<const double2*>(bp + 2);
        }
      }
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          dmma(acc[g][h][0][0], acc[g][h][0][1], a[g].x, bs[h].x);
          dmma(acc[g][h][1][0], acc[g][h][1][1], a[g].x, bs[h].y);
          dmma(acc[g][h][2][0], acc[g][h][2][1], a[g].y, ba[h].x);
          dmma(acc[g][h][3][0], acc[g][h][3][1], a[g].y, ba[h].y);
        }
    }
    if (MODE == 2) __syncthreads();
  }
  double s = 0;
  for (int g = 0; g < 4; ++g) for (int h = 0; h < 2; ++h) for (int q = 0; q < 4; ++q) s += acc[g][h][q][0] + acc[g][h][q][1];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 256);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    kern<<<sms, 256, 65536>>>(out, 10); if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: launch failed %s\n", name, cudaGetErrorString(cudaGetLastError())); return; }
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); kern<<<sms, 256, 65536>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    double flops = 2.0 * 256 * 128 * (double)iters * 8 * sms;
    printf("%s: %.2f TFLOP/s\n", name, flops / best / 1e9);
  };
  run(k<0>, "const-frag 32acc");
  run(k<1>, "smem-frag 32acc");
  run(k<2>, "smem-frag? no: const + barrier per 128");
  return 0;
}

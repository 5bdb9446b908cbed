// FP64 peak probe for B200 (sm_100a): DMMA.8x8x4 and DFMA issue throughput.
// Used once to fix the Legendre roofline denominator (recorded in profiles/).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void mma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double x) {
  double c[NACC][2];
#pragma unroll
  for (int j = 0; j < NACC; ++j) { c[j][0] = 0; c[j][1] = 0; }
  double a = x + threadIdx.x, b = x * 0.5 + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) mma884(c[j][0], c[j][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double x) {
  double c[NACC];
#pragma unroll
  for (int j = 0; j < NACC; ++j) c[j] = threadIdx.x + j;
  double a = x, b = 1.0 - 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) c[j] = fma(c[j], b, a);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 32 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int tpb : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      dmma_loop<8><<<blocks, tpb>>>(out, 100, 1.0);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0); dmma_loop<8><<<blocks, tpb>>>(out, iters, 1.0); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double flops = 2.0 * 256 * 8 * (double)iters * (tpb / 32) * blocks;  // 256 FMA per warp-DMMA
      printf(", \"dmma_tpb%d_bps%d_tflops\": %.3f", tpb, bps, flops / best / 1e9);
    }
  }
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * 2;
    dfma_loop<8><<<blocks, tpb>>>(out, 100, 1.0);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_loop<8><<<blocks, tpb>>>(out, iters, 1.0); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * (double)iters * tpb * blocks;
    printf(", \"dfma_tpb%d_tflops\": %.3f", tpb, flops / best / 1e9);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf(", \"clock_khz_attr\": %d}\n", clk);
  return 0;
}

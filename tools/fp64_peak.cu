// FP64 pipe microbenchmark behind DESIGN.md's Black-Scholes analysis:
// DFMA throughput (8 independent chains per thread, full occupancy) and
// DFMA latency (one dependent chain, one warp).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void thr(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}

__global__ void lat(double* out, int iters, double a, double b, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (x == 12345.678) out[0] = x;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  const int iters = 1 << 14, block = 256, grid = sms * 8;
  thr<<<grid, block>>>(out, 16, 0.999, 1e-3);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  thr<<<grid, block>>>(out, iters, 0.999, 1e-3);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  double n = (double)grid * block * iters * 8;
  printf("DFMA throughput: %.3f T DFMA/s = %.1f TFLOP/s fp64 (%d SMs, %.0f DFMA/clk/SM at %d MHz)\n",
         n / ms / 1e9, 2 * n / ms / 1e9, sms, n / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  lat<<<1, 32>>>(out, iters, 0.999, 1e-3, cyc);
  cudaDeviceSynchronize();
  long long c = 0; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent-chain latency: %.2f cycles\n", (double)c / iters);
  return 0;
}

// L2 reduction-throughput microbenchmark: how many scattered 8-byte
// red.global.add operations per second B200 sustains, by target-array size
// and operand type, with no other memory traffic (indices come from a hash
// in registers).  This is the ceiling of a vecmerger histogram whose bins do
// not fit in shared memory (C5: 1M f64 bins, one RED per row).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_peak tools/red_peak.cu
//   ./tools/red_peak
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

template <int KIND>   // 0 f64 add, 1 u64 add, 2 f32 add
__global__ void __launch_bounds__(256) k_red(void* bins, uint64_t nbins, uint64_t per_thread) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t h = mix(t + 1);
  for (uint64_t i = 0; i < per_thread; ++i) {
    h = mix(h + i);
    const uint64_t b = h % nbins;
    if (KIND == 0) atomicAdd((double*)bins + b, 1.0);
    else if (KIND == 1) atomicAdd((unsigned long long*)bins + b, 1ULL);
    else atomicAdd((float*)bins + b, 1.0f);
  }
}

// same REDs with streaming loads of 16 B per RED (the histogram's shape)
__global__ void __launch_bounds__(256) k_red_stream(double* bins, uint64_t nbins, const int64_t* idx, const double* w,
                                                    uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t b = __ldcs(idx + i);
    atomicAdd(bins + b, __ldcs(w + i));
  }
}

__global__ void k_fill(int64_t* p, uint64_t n, uint64_t nb) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = (int64_t)(mix(i * 0x9E3779B97F4A7C15ULL + 7) % nb);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* bins;
  const uint64_t maxb = 1ULL << 27;   // 1 GiB of 8-byte bins
  cudaMalloc(&bins, maxb * 8);
  cudaMemset(bins, 0, maxb * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const unsigned grid = sms * 8;
  const uint64_t per = 256;
  const double ops = (double)grid * 256 * per;
  const char* kn[3] = {"f64", "u64", "f32"};
  for (uint64_t nb : {1ULL << 10, 1ULL << 17, 1000000ULL, 1ULL << 23, 1ULL << 27}) {
    for (int kind = 0; kind < 3; ++kind) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        if (kind == 0) k_red<0><<<grid, 256>>>(bins, nb, per);
        else if (kind == 1) k_red<1><<<grid, 256>>>(bins, nb, per);
        else k_red<2><<<grid, 256>>>(bins, nb, per);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("red %s bins=%llu (%.1f MB): %.3e RED/s (%.3f ms)\n", kn[kind], (unsigned long long)nb,
             nb * (kind == 2 ? 4.0 : 8.0) / 1e6, ops / (best * 1e-3), best);
    }
  }
  // the histogram shape: 1e9 rows (idx i64, w f64) into 1M f64 bins
  const uint64_t n = 1000000000ULL, nb = 1000000ULL;
  int64_t* idx;
  double* w;
  if (cudaMalloc(&idx, n * 8) == cudaSuccess && cudaMalloc(&w, n * 8) == cudaSuccess) {
    cudaMemset(w, 0, n * 8);
    k_fill<<<sms * 8, 256>>>(idx, n, nb);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k_red_stream<<<sms * 8, 256>>>((double*)bins, nb, idx, w, n);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("hist-shape 1e9 rows -> 1M f64 bins: %.3f ms, %.3e RED/s, %.0f GB/s of input\n", best, n / (best * 1e-3),
           n * 16.0 / (best * 1e-3) / 1e9);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}


// Scattered 64-bit atomic throughput into shared memory: the CTA's own
// (local ATOMS) vs the distributed shared memory of an 8-CTA cluster
// (remote, through map_shared_rank), with no other traffic.  The question
// behind it: can a dictmerger region table held in a cluster's shared memory
// aggregate faster than the L2-resident table (one probe + one RED per row,
// ~1.3e11 L2 ops/s, profiles/red_peak_r02.txt)?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_peak tools/dsmem_peak.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

constexpr int SLOTS = 4096;   // 32 KB of u64 counters per CTA

template <bool REMOTE>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512) k_atoms(uint64_t iters, unsigned long long* sink) {
  __shared__ unsigned long long tab[SLOTS];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) tab[i] = 0;
  cl.sync();
  uint64_t h = mix(blockIdx.x * 1024ULL + threadIdx.x + 1);
  for (uint64_t i = 0; i < iters; ++i) {
    h = mix(h + i);
    const unsigned slot = (unsigned)(h >> 3) & (SLOTS - 1);
    if (REMOTE) {
      unsigned long long* p = cl.map_shared_rank(&tab[slot], (unsigned)(h & 7));
      atomicAdd(p, 1ULL);
    } else {
      atomicAdd(&tab[slot], 1ULL);
    }
  }
  cl.sync();
  if (threadIdx.x == 0) atomicAdd(sink, tab[0]);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t iters = 2048;
  for (int remote = 0; remote < 2; ++remote) {
    for (int bpsm : {1, 2, 3}) {
      const unsigned grid = (unsigned)(sms / 8 * 8 * bpsm);
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        if (remote) k_atoms<true><<<grid, 512>>>(iters, sink);
        else k_atoms<false><<<grid, 512>>>(iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      const double ops = (double)grid * 512 * iters;
      printf("%s smem atomicAdd u64, %u CTAs (%d/SM): %.3e ops/s (%.3f ms)  %s\n", remote ? "cluster (DSMEM)" : "local",
             grid, bpsm, ops / (best * 1e-3), best, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

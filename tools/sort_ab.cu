// A/B microbenchmark: the library's onesweep radix sort (wg_radix.cuh)
// against cub::DeviceRadixSort::SortPairs on the same (u64 key, u64 value)
// pairs -- C4b's shape: 200M rows, keys scrambled over 64 bits, sorted on a
// 32-bit window.  Not part of the product (CUB is used only here).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sort_ab tools/sort_ab.cu
#include <cub/cub.cuh>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>
namespace { 
#include "../paper_1709_06416_b200/csrc/wg_radix.cuh"
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void gen(uint64_t* k, uint64_t* v, uint64_t n, uint64_t nkeys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ULL + 12345;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL; z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL; z ^= z >> 31;
    uint64_t key = z % nkeys;
    key = key * 0x9E3779B97F4A7C15ULL; key ^= key >> 29;
    k[i] = key; v[i] = i;
  }
}

template <typename K, typename V>
int ours(const K* kin, const V* vin, K* kA, K* kB, V* vA, V* vB, uint32_t n, int begin, int end, cudaStream_t s) {
  const int npass = (end - begin + 7) / 8;
  #ifndef AB_ITEMS
#define AB_ITEMS 8
#endif
  constexpr int ITEMS = AB_ITEMS, TILE = 512 * ITEMS;
  constexpr int SMEM = wgr::onesweep_smem<K, V, ITEMS>();
  cudaFuncSetAttribute(wgr::k_onesweep<K, V, V, V, wgr::VCopy, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const uint64_t tiles = (n + TILE - 1) / TILE;
  static uint32_t* hist = nullptr; static unsigned long long* status = nullptr;
  if (!hist) { cudaMalloc(&hist, 9 * 256 * 4); cudaMalloc(&status, tiles * 256 * 8); }
  cudaMemsetAsync(hist, 0, (npass * 256 + npass) * 4, s);
  wgr::k_radix_hist<K><<<148 * 16, 256, 0, s>>>(kin, n, begin, end, npass, hist);
  wgr::k_radix_offsets<<<npass, 256, 0, s>>>(hist);
  const K* ki = kin; const V* vi = vin;
  for (int p = 0; p < npass; ++p) {
    const bool toA = ((npass - 1 - p) & 1) == 0;
    K* ko = toA ? kA : kB; V* vo = toA ? vA : vB;
    const int shift = begin + 8 * p, wb = std::min(8, end - shift);
    cudaMemsetAsync(status, 0, tiles * 256 * 8, s);
    wgr::k_onesweep<K, V, V, V, wgr::VCopy, ITEMS><<<(unsigned)tiles, 512, SMEM, s>>>(ki, vi, ko, vo, n, shift, (1u << wb) - 1u,
                                                                  hist + p * 256, status, hist + npass * 256 + p, 0);
    ki = ko; vi = vo;
  }
  return 0;
}

int main(int argc, char** argv) {
  uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 200000000ULL;
  int begin = argc > 2 ? atoi(argv[2]) : 32, end = argc > 3 ? atoi(argv[3]) : 64;
  uint64_t *k0, *v0, *kA, *kB, *vA, *vB;
  CK(cudaMalloc(&k0, n * 8)); CK(cudaMalloc(&v0, n * 8)); CK(cudaMalloc(&kA, n * 8)); CK(cudaMalloc(&kB, n * 8));
  CK(cudaMalloc(&vA, n * 8)); CK(cudaMalloc(&vB, n * 8));
  gen<<<148 * 16, 256>>>(k0, v0, n, 10000000ULL);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms_ours = 1e9, ms_cub = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a, s);
    ours<uint64_t, uint64_t>(k0, v0, kA, kB, vA, vB, (uint32_t)n, begin, end, s);
    cudaEventRecord(b, s); CK(cudaEventSynchronize(b));
    float t; cudaEventElapsedTime(&t, a, b); ms_ours = std::min(ms_ours, t);
  }
  CK(cudaGetLastError());
  // keep our result for the check
  std::vector<uint64_t> hk(n), hv(n);
  cudaMemcpy(hk.data(), kA, n * 8, cudaMemcpyDeviceToHost); cudaMemcpy(hv.data(), vA, n * 8, cudaMemcpyDeviceToHost);
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, k0, kB, v0, vB, (int)n, begin, end, s);
  void* dt; CK(cudaMalloc(&dt, temp));
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a, s);
    cub::DeviceRadixSort::SortPairs(dt, temp, k0, kB, v0, vB, (int)n, begin, end, s);
    cudaEventRecord(b, s); CK(cudaEventSynchronize(b));
    float t; cudaEventElapsedTime(&t, a, b); ms_cub = std::min(ms_cub, t);
  }
  std::vector<uint64_t> ck(n), cv(n);
  cudaMemcpy(ck.data(), kB, n * 8, cudaMemcpyDeviceToHost); cudaMemcpy(cv.data(), vB, n * 8, cudaMemcpyDeviceToHost);
  bool same = ck == hk && cv == hv;
  const int npass = (end - begin + 7) / 8;
  double bytes = (double)n * 16 * 2 * npass;
  printf("{\"n\": %llu, \"bits\": [%d, %d], \"passes\": %d, \"ours_ms\": %.3f, \"cub_ms\": %.3f, "
         "\"ours_pass_GBs\": %.1f, \"cub_pass_GBs\": %.1f, \"identical\": %s}\n",
         (unsigned long long)n, begin, end, npass, ms_ours, ms_cub, bytes / ms_ours / 1e6, bytes / ms_cub / 1e6,
         same ? "true" : "false");
  return same ? 0 : 2;
}

// weldgpu.cu -- libweldgpu.so: the C-ABI under the Weld-IR GPU executor.
//
// Owns the device, one execution stream, a stream-ordered buffer pool, the
// device error word, NVRTC compilation of generated loop kernels (sm_100a,
// -fmad=false) and their launch, plus the fixed-function kernels every
// builder's result() needs (table init/compaction, order-preserving key
// transforms, stable radix sort, gathers, run heads) and the synthetic
// column generators used by the benchmark.
//
// Every entry point is `extern "C"`, returns 0 on success and -1 on failure
// with the message in wg_last_error() (thread-local).  Declarations and the
// reference interface each one replaces are in include/weldgpu.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>
#include <nccl.h>   // types only: libnccl.so.2 is dlopen()ed at wg_nccl_init
#include <dlfcn.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/weldgpu.h"

namespace {

thread_local std::string g_err;
std::mutex g_mu;
bool g_inited = false;
int g_device = -1;
cudaStream_t g_stream = nullptr;      // current stream (every call below enqueues here)
cudaStream_t g_streams[3] = {nullptr, nullptr, nullptr};  // 0 compute, 1 host->device, 2 device->host
int g_sm_count = 0;
int64_t* g_err_word = nullptr;      // device {code, info}
int64_t* g_err_host = nullptr;      // pinned mirror
int64_t g_sync_err[2] = {0, 0};     // error word captured by wg_dict_finish_small's sync
uint64_t g_live = 0, g_peak = 0;    // device bytes handed out by wg_alloc
std::mutex g_acct_mu;
std::unordered_map<void*, uint64_t> g_sizes;       // live blocks -> rounded size
std::multimap<uint64_t, void*> g_free;             // cached blocks by size
uint64_t g_cached = 0;
// Blocks freed while more than one stream may be in flight (the streaming
// host-input path selects the copy streams) are not reused until every
// stream has drained (wg_sync_all): a copy still pending on stream 1/2
// must not race with a new owner on stream 0.
bool g_multi = false;
std::vector<std::pair<uint64_t, void*>> g_deferred;
static void release_deferred() {   // caller holds g_acct_mu, every stream drained
  for (auto& kv : g_deferred) {
    g_free.emplace(kv.first, kv.second);
    g_cached += kv.first;
  }
  g_deferred.clear();
}


int fail(const std::string& msg) {
  g_err = msg;
  return -1;
}

// ---- per-launch device timing (wg_prof_*) ----------------------------------
// When enabled, every kernel this library launches -- fixed-function
// kernels and NVRTC loop kernels alike -- is bracketed by a pair of CUDA
// events on the stream it is launched on, tagged with the kernel's name.
// bench.py reads the records back to find the dominant kernel and the
// whole-step kernel time (no profiler attached, no extra synchronisation
// inside the step).
struct ProfRec { const char* name; cudaEvent_t a, b; };
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_prof_free;
std::mutex g_prof_mu;
std::unordered_map<uint64_t, std::string> g_fn_names;   // CUfunction -> kernel name

cudaEvent_t prof_event() {
  if (!g_prof_free.empty()) { cudaEvent_t e = g_prof_free.back(); g_prof_free.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  const char* name;
  cudaEvent_t a = nullptr;
  explicit ProfScope(const char* n) : name(n) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    a = prof_event();
    cudaEventRecord(a, g_stream);
  }
  ~ProfScope() {
    if (!a) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t b = prof_event();
    cudaEventRecord(b, g_stream);
    g_prof.push_back({name, a, b});
  }
};
#define WG_PROF(name) ProfScope wg_prof_scope_(name)

// Driver API entry points are resolved through cudart at wg_init() so the
// library loads (for symbol checks and NVRTC compile checks) on hosts with
// no GPU driver at all.
typedef CUresult (*PFN_GetErrorString)(CUresult, const char**);
typedef CUresult (*PFN_ModuleLoadData)(CUmodule*, const void*);
typedef CUresult (*PFN_ModuleGetFunction)(CUfunction*, CUmodule, const char*);
typedef CUresult (*PFN_LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                     unsigned, CUstream, void**, void**);
typedef CUresult (*PFN_Occupancy)(int*, CUfunction, int, size_t);
typedef CUresult (*PFN_FuncSetAttribute)(CUfunction, CUfunction_attribute, int);
PFN_GetErrorString p_cuGetErrorString = nullptr;
PFN_ModuleLoadData p_cuModuleLoadData = nullptr;
PFN_ModuleGetFunction p_cuModuleGetFunction = nullptr;
PFN_LaunchKernel p_cuLaunchKernel = nullptr;
PFN_Occupancy p_cuOccupancyMaxActiveBlocksPerMultiprocessor = nullptr;
PFN_FuncSetAttribute p_cuFuncSetAttribute = nullptr;

template <typename F>
bool resolve(const char* name, F* out) {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fp, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !fp)
    return false;
  *out = reinterpret_cast<F>(fp);
  return true;
}

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      return fail(std::string(#x) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

#define CKD(x)                                                                         \
  do {                                                                                 \
    CUresult r_ = (x);                                                                 \
    if (r_ != CUDA_SUCCESS) {                                                          \
      const char* s_ = nullptr;                                                        \
      if (p_cuGetErrorString) p_cuGetErrorString(r_, &s_);                                                       \
      return fail(std::string(#x) + ": " + (s_ ? s_ : "unknown driver error"));         \
    }                                                                                  \
  } while (0)

#define CKN(x)                                                                         \
  do {                                                                                 \
    nvrtcResult r_ = (x);                                                              \
    if (r_ != NVRTC_SUCCESS) return fail(std::string(#x) + ": " + nvrtcGetErrorString(r_)); \
  } while (0)

#define NEED_INIT() \
  do { if (!g_inited) return fail("weldgpu: wg_init() has not been called"); } while (0)

inline unsigned grid_for(uint64_t n, unsigned block) {
  uint64_t g = (n + block - 1) / block;
  uint64_t cap = (uint64_t)(g_sm_count > 0 ? g_sm_count : 148) * 16;
  if (g > cap) g = cap;
  if (g == 0) g = 1;
  return (unsigned)g;
}

#include "wg_radix.cuh"

// ---------------------------------------------------------------------------
// Fixed-function kernels.

__global__ void k_table_init(uint64_t* table, uint64_t nslots, int slot_words, const uint64_t* pattern_dev) {
  __shared__ uint64_t pat[64];
  if (threadIdx.x < (unsigned)slot_words) pat[threadIdx.x] = pattern_dev[threadIdx.x];
  __syncthreads();
  uint64_t total = nslots * (uint64_t)slot_words;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < total; w += (uint64_t)gridDim.x * blockDim.x)
    table[w] = pat[w % slot_words];
}

// Compact occupied slots to SoA word arrays (order is irrelevant: results
// are sorted by key afterwards).  mode 1: claim word is the key (EMPTY =
// all ones); mode 2: claim word is a state word (2 = full).
__global__ void k_table_compact(const uint64_t* table, uint64_t nslots, int slot_words, int mode,
                                uint64_t** out_words, int nout, unsigned long long* counter) {
  // one output reservation per CTA iteration (block scan of occupancy)
  __shared__ unsigned s_w[32];
  __shared__ unsigned long long s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < nslots; base += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s = base + threadIdx.x;
    bool occ = false;
    if (s < nslots) {
      uint64_t w0 = table[s * slot_words];
      occ = (mode == 1) ? (w0 != 0xffffffffffffffffULL) : (w0 == 2ULL);
    }
    unsigned m = __ballot_sync(0xffffffffu, occ);
    if (lane == 0) s_w[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned tot = 0;
      for (int w = 0; w < nw; ++w) { unsigned c = s_w[w]; s_w[w] = tot; tot += c; }
      s_base = tot ? atomicAdd(counter, (unsigned long long)tot) : 0ULL;
    }
    __syncthreads();
    if (occ) {
      uint64_t dst = s_base + s_w[warp] + __popc(m & ((1u << lane) - 1u));
      int first = (mode == 1) ? 0 : 1;
      for (int k = 0; k < nout; ++k) out_words[k][dst] = table[s * slot_words + first + k];
    }
    __syncthreads();
  }
}

// The sentinel-key slot (mode 1) sits at index nslots; occupied when its
// claim word was CAS'ed from EMPTY to 0.
__global__ void k_table_compact_sentinel(const uint64_t* table, uint64_t nslots, int slot_words,
                                         uint64_t** out_words, int nout, unsigned long long* counter) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const uint64_t* s = table + nslots * slot_words;
  if (s[0] == 0ULL) {
    uint64_t dst = atomicAdd(counter, 1ULL);
    out_words[0][dst] = 0xffffffffffffffffULL;
    for (int k = 1; k < nout; ++k) out_words[k][dst] = s[k];
  }
}

// Order-preserving u64 transform of a typed column (order_key,
// builders.py:496-507): signed ints flip the sign bit; floats use the
// IEEE total-order trick with every NaN mapped above +inf; -0.0 == 0.0.
// kind: 0 bool(u8) 1 i32 2 i64 3 f32 4 f64 ; src elements are `kind`-typed.
__global__ void k_order_key(const void* src, int kind, uint64_t n, const uint32_t* perm, uint64_t* dst) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t j = perm ? perm[i] : i;
    uint64_t k;
    switch (kind) {
      case 0: k = ((const uint8_t*)src)[j]; break;
      case 1: k = (uint64_t)(int64_t)((const int32_t*)src)[j] ^ 0x8000000000000000ULL; break;
      case 2: k = (uint64_t)((const int64_t*)src)[j] ^ 0x8000000000000000ULL; break;
      default: {
        double v = (kind == 3) ? (double)((const float*)src)[j] : ((const double*)src)[j];
        if (v != v) { k = 0xffffffffffffffffULL; break; }
        if (v == 0.0) v = 0.0;
        uint64_t b = (uint64_t)__double_as_longlong(v);
        k = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
        if (k == 0xffffffffffffffffULL) k = 0xfffffffffffffffeULL;  // keep NaN strictly last
      }
    }
    dst[i] = k;
  }
}

// ---- row partitioning for the multi-GPU combine --------------------------
// dest(row) = number of splitters <= order_key(key[row]) (range partition
// of the first key leaf: equal keys always meet on one rank, and rank-order
// concatenation of the per-rank results is globally sorted).
__device__ __forceinline__ uint64_t okey_at(const void* src, int kind, uint64_t j) {
  switch (kind) {
    case 0: return ((const uint8_t*)src)[j];
    case 1: return (uint64_t)(int64_t)((const int32_t*)src)[j] ^ 0x8000000000000000ULL;
    case 2: return (uint64_t)((const int64_t*)src)[j] ^ 0x8000000000000000ULL;
    default: {
      double v = (kind == 3) ? (double)((const float*)src)[j] : ((const double*)src)[j];
      if (v != v) return 0xffffffffffffffffULL;
      if (v == 0.0) v = 0.0;
      uint64_t b = (uint64_t)__double_as_longlong(v);
      uint64_t k = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
      return k == 0xffffffffffffffffULL ? 0xfffffffffffffffeULL : k;
    }
  }
}

#define WG_PART_MAX 64
struct PartSpec {
  int G, nsplit, ncols, kind;
  const void* key;
  uint64_t split[WG_PART_MAX];
  const void* in[16];
  void* out[16];
  int width[16];
};

__device__ __forceinline__ int part_dest(const PartSpec& p, uint64_t row) {
  const uint64_t k = okey_at(p.key, p.kind, row);
  int lo = 0, hi = p.nsplit;   // first splitter > k
  while (lo < hi) { const int m = (lo + hi) >> 1; if (p.split[m] <= k) lo = m + 1; else hi = m; }
  return lo;
}

// per-tile destination counts: cnt[d * ntiles + t]
__global__ void __launch_bounds__(256) k_part_count(PartSpec p, uint64_t n, uint32_t* cnt, uint32_t ntiles) {
  __shared__ uint32_t c[WG_PART_MAX];
  if (threadIdx.x < WG_PART_MAX) c[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t t0 = (uint64_t)blockIdx.x * 4096;
  for (int i = threadIdx.x; i < 4096; i += 256) {
    const uint64_t r = t0 + i;
    if (r < n) atomicAdd(&c[part_dest(p, r)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < p.G) cnt[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = c[threadIdx.x];
}

// one CTA per destination: exclusive scan of its per-tile counts (in
// place), the destination's total into tot[d]
__global__ void __launch_bounds__(1024) k_part_scan(uint32_t* cnt, uint32_t ntiles, uint64_t* tot) {
  __shared__ uint32_t ws[32];
  __shared__ uint64_t carry;
  uint32_t* c = cnt + (uint64_t)blockIdx.x * ntiles;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t b = 0; b < ntiles; b += 1024) {
    const uint32_t i = b + threadIdx.x;
    const uint32_t v = i < ntiles ? c[i] : 0;
    uint32_t x = v;
    for (int s = 1; s < 32; s <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, x, s); if (lane >= s) x += y; }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    uint32_t before = 0, all = 0;
    for (int j = 0; j < 32; ++j) { if (j < w) before += ws[j]; all += ws[j]; }
    const uint64_t base = carry;
    if (i < ntiles) c[i] = (uint32_t)(base + before + x - v);
    __syncthreads();
    if (threadIdx.x == 0) carry = base + all;
    __syncthreads();
  }
  if (threadIdx.x == 0) tot[blockIdx.x] = carry;
}

// stable scatter of every column: rows keep their input order inside each
// destination segment (warp rounds of 32 consecutive rows, ballot ranks)
__global__ void __launch_bounds__(256) k_part_scatter(PartSpec p, uint64_t n, const uint32_t* cnt, uint32_t ntiles,
                                                      const uint64_t* tot) {
  constexpr int ITEMS = 16;
  __shared__ uint32_t wc[8][WG_PART_MAX];
  __shared__ uint64_t base[WG_PART_MAX];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < 8 * WG_PART_MAX; i += 256) (&wc[0][0])[i] = 0;
  if (tid < p.G) {
    uint64_t b = 0;
    for (int d = 0; d < tid; ++d) b += tot[d];
    base[tid] = b + cnt[(uint64_t)tid * ntiles + blockIdx.x];
  }
  __syncthreads();
  const uint64_t wrow = (uint64_t)blockIdx.x * 4096 + (uint64_t)w * 512 + lane;
  int dd[ITEMS];
  uint32_t rk[ITEMS];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t r = wrow + i * 32;
    const int d = r < n ? part_dest(p, r) : WG_PART_MAX;
    unsigned pm = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 7; ++b) {
      const bool bit = (d >> b) & 1;
      const unsigned bm = __ballot_sync(0xffffffffu, bit);
      pm &= bit ? bm : ~bm;
    }
    const uint32_t below = __popc(pm & lt);
    const uint32_t prev = d < WG_PART_MAX ? wc[w][d] : 0u;
    __syncwarp();
    if (d < WG_PART_MAX && below == 0) wc[w][d] = prev + __popc(pm);
    __syncwarp();
    dd[i] = d;
    rk[i] = prev + below;
  }
  __syncthreads();
  if (tid < p.G) {   // warp offsets within the tile's segment of each destination
    uint32_t run = 0;
    for (int j = 0; j < 8; ++j) { const uint32_t c = wc[j][tid]; wc[j][tid] = run; run += c; }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int d = dd[i];
    if (d >= WG_PART_MAX) continue;
    const uint64_t src = wrow + i * 32;
    const uint64_t dst = base[d] + wc[w][d] + rk[i];
    for (int c = 0; c < p.ncols; ++c) {
      switch (p.width[c]) {
        case 1: ((uint8_t*)p.out[c])[dst] = ((const uint8_t*)p.in[c])[src]; break;
        case 4: ((uint32_t*)p.out[c])[dst] = ((const uint32_t*)p.in[c])[src]; break;
        default: ((uint64_t*)p.out[c])[dst] = ((const uint64_t*)p.in[c])[src]; break;
      }
    }
  }
}

__global__ void k_iota_u32(uint32_t* dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = (uint32_t)i;
}

template <typename T>
__global__ void k_gather(const T* src, const uint32_t* perm, T* dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}

// Narrow/widen an 8-byte word column into a typed column (table words to
// i32/f32/u8 results and back).
__global__ void k_narrow(const uint64_t* src, void* dst, int width, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v = src[i];
    if (width == 8) ((uint64_t*)dst)[i] = v;
    else if (width == 4) ((uint32_t*)dst)[i] = (uint32_t)v;
    else ((uint8_t*)dst)[i] = (uint8_t)v;
  }
}
__global__ void k_widen(const void* src, uint64_t* dst, int width, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v;
    if (width == 8) v = ((const uint64_t*)src)[i];
    else if (width == 4) v = ((const uint32_t*)src)[i];
    else v = ((const uint8_t*)src)[i];
    dst[i] = v;
  }
}

// Segment heads over sorted multi-word keys: flag[i] = (i == 0) || key(i) != key(i-1).
// ---------------------------------------------------------------------------
// Counter-based synthetic columns: h = splitmix64(seed ^
// (col << 56) ^ row); u = (h >> 11) * 2^-53; ints = lo + h mod span.
__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// dist: 0 int uniform [lo, lo+span) ; 1 float lo + u*(hi-lo) ; 2 float (lo + h mod span) / div
//       3 key scatter: sm64(lo + h mod span) as i64 (distinct keys spread over i64)
//       4 categorical over up to 8 (value, cumulative-probability) pairs (for Q1 flags)
struct GenSpec {
  int dist; int width; uint64_t seed; uint64_t col; int64_t lo; uint64_t span; double flo, fhi, div;
  double cum[8]; int64_t vals[8]; int ncat;
};
__global__ void k_gen(void* dst, uint64_t n, uint64_t row0, GenSpec g) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = sm64(g.seed ^ (g.col << 56) ^ (row0 + i));
    double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
    if (g.dist == 0 || g.dist == 3 || g.dist == 4) {
      int64_t v;
      if (g.dist == 0) v = g.lo + (int64_t)(h % g.span);
      else if (g.dist == 3) v = (int64_t)sm64((uint64_t)(g.lo + (int64_t)(h % g.span)));
      else {
        v = g.vals[g.ncat - 1];
        for (int c = 0; c < g.ncat; ++c) if (u < g.cum[c]) { v = g.vals[c]; break; }
      }
      if (g.width == 8) ((int64_t*)dst)[i] = v; else ((int32_t*)dst)[i] = (int32_t)v;
    } else {
      // explicit round-to-nearest ops: no FMA contraction, so numpy reproduces it bit for bit
      double v = (g.dist == 1) ? __dadd_rn(g.flo, __dmul_rn(u, __dsub_rn(g.fhi, g.flo)))
                               : __ddiv_rn((double)(g.lo + (int64_t)(h % g.span)), g.div);
      if (g.width == 8) ((double*)dst)[i] = v; else ((float*)dst)[i] = (float)v;
    }
  }
}

// Multiply a float column elementwise by another in place (k = s * U(0.9, 1.1)).
__global__ void k_mul_inplace(double* a, const double* b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = __dmul_rn(a[i], b[i]);
}

__global__ void k_flush(uint4* buf, uint64_t n16, uint32_t salt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
    buf[i] = make_uint4((uint32_t)i, salt, (uint32_t)(i >> 32), salt ^ 0x5a5a5a5a);
}


// ---- groupbuilder finalisation (single integer key leaf) -------------------
// After a stable radix sort on key bits [shift, 64), rows of one bucket
// (equal high bits) may still be out of order in the low bits.  Record the
// positions where order breaks inside a bucket; only those buckets get a
// stable insertion sort (most buckets hold a single distinct key).
__global__ void k_disorder(const uint64_t* k, uint64_t n, int shift, uint32_t* pos, unsigned long long* npos,
                           uint64_t cap) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i0 = 1;
  if ((((uintptr_t)k) & 31) == 0) {
    // rows 4q..4q+3 against their predecessors: one 256-bit load + the row before
    const uint64_t n4 = n / 4;
    for (uint64_t q = tid; q < n4; q += stride) {
      uint64_t c[5];
      asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(c[1]), "=l"(c[2]), "=l"(c[3]), "=l"(c[4]) : "l"(k + 4 * q));
      c[0] = q ? k[4 * q - 1] : c[1];
#pragma unroll
      for (int j = 1; j <= 4; ++j) {
        if ((c[j - 1] >> shift) == (c[j] >> shift) && c[j - 1] > c[j]) {
          unsigned long long p = atomicAdd(npos, 1ULL);
          if (p < cap) pos[p] = (uint32_t)(4 * q + j - 1);
        }
      }
    }
    i0 = n4 * 4 > 1 ? n4 * 4 : 1;
  }
  for (uint64_t i = i0 + tid; i < n; i += stride) {
    uint64_t a = k[i - 1], b = k[i];
    if ((a >> shift) == (b >> shift) && a > b) {
      unsigned long long q = atomicAdd(npos, 1ULL);
      if (q < cap) pos[q] = (uint32_t)i;
    }
  }
}

// One thread per recorded disorder position: find the bucket's start (bucket
// membership -- equal bits [shift, 64) -- is unaffected by reordering inside
// the bucket, so the walk is race-free) and claim the bucket through a bit
// in `claimed`; the single owner stable-insertion-sorts it.
__global__ void k_fix_buckets(uint64_t* k, uint64_t* v, uint64_t n, int shift, const uint32_t* pos, uint64_t npos,
                              int cap, int* too_long, unsigned* claimed) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < npos; q += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t i = pos[q];
    uint64_t top = k[i] >> shift;
    uint64_t s = i;
    while (s > 0 && (k[s - 1] >> shift) == top) --s;
    if (atomicOr(&claimed[s >> 5], 1u << (s & 31)) & (1u << (s & 31))) continue;
    uint64_t e = i + 1;
    while (e < n && (k[e] >> shift) == top) ++e;
    if (e - s > (uint64_t)cap) { *too_long = 1; continue; }
    for (uint64_t a = s + 1; a < e; ++a) {
      uint64_t kk = k[a], vv = v[a];
      uint64_t b = a;
      while (b > s && k[b - 1] > kk) { k[b] = k[b - 1]; v[b] = v[b - 1]; --b; }
      k[b] = kk; v[b] = vv;
    }
  }
}

// 32-bit sort keys: w = okey - base (every key's varying bits fit in 32)
__global__ void k_key_u32(const uint64_t* ok, uint64_t n, uint64_t base, uint32_t* w) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    w[i] = (uint32_t)(ok[i] - base);
}

// offsets[j] = starts[j]; offsets[K] = n; ukeys[j] = inverse order key.
template <typename KT>
__global__ void k_group_out(const uint32_t* starts, uint64_t K, uint64_t n, const KT* sk, uint64_t kmin,
                            int kind, int64_t* offs, void* ukeys) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j <= K; j += (uint64_t)gridDim.x * blockDim.x) {
    if (j == K) { offs[K] = (int64_t)n; continue; }
    uint64_t s = starts[j];
    offs[j] = (int64_t)s;
    uint64_t w = (uint64_t)sk[s] + kmin;
    if (kind == 0) ((uint8_t*)ukeys)[j] = (uint8_t)w;
    else if (kind == 1) ((int32_t*)ukeys)[j] = (int32_t)(int64_t)(w ^ 0x8000000000000000ULL);
    else ((int64_t*)ukeys)[j] = (int64_t)(w ^ 0x8000000000000000ULL);
  }
}

// ---- small dictmerger result (DictMergerState.result, builders.py:380-392,
// entries sorted by order_key builders.py:496-507) in ONE launch: collect the
// occupied slots, order them by the key's order-key tuple (bitonic sort in
// shared memory), and write typed key / value columns.  For results of up to
// WG_SMALL_DICT entries (TPC-H style group counts) this replaces
// compaction + per-leaf radix sorts + gathers (and their host round trips).
#define WG_SMALL_DICT 4096
struct SmallDictDesc {
  int nkl, nvl, mode, nw, sw, kbase;
  int kword[8], kshift[8], kwidth[8], kkind[8];
  int vkind[16];
  void* out[24];
};

__device__ __forceinline__ uint64_t wg_leaf_okey(uint64_t bits, int kind) {
  switch (kind) {
    case 0: return bits & 0xffULL;
    case 1: return (uint64_t)(int64_t)(int32_t)(uint32_t)bits ^ 0x8000000000000000ULL;
    case 2: return bits ^ 0x8000000000000000ULL;
    default: {
      double v = (kind == 3) ? (double)__int_as_float((int)(uint32_t)bits) : __longlong_as_double((long long)bits);
      if (v != v) return 0xffffffffffffffffULL;
      if (v == 0.0) v = 0.0;
      uint64_t b = (uint64_t)__double_as_longlong(v);
      uint64_t k = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
      return k == 0xffffffffffffffffULL ? 0xfffffffffffffffeULL : k;
    }
  }
}

__device__ __forceinline__ void wg_store_leaf(void* col, uint64_t i, uint64_t bits, int kind) {
  switch (kind) {
    case 0: ((uint8_t*)col)[i] = (uint8_t)bits; break;
    case 1: case 3: ((uint32_t*)col)[i] = (uint32_t)bits; break;
    default: ((uint64_t*)col)[i] = bits;
  }
}

__global__ void __launch_bounds__(1024) k_dict_finish_small(const uint64_t* table, uint64_t nslots, SmallDictDesc d,
                                                            const unsigned long long* counters,
                                                            unsigned long long* count_out) {
  __shared__ uint32_t s_idx[WG_SMALL_DICT];
  __shared__ unsigned s_n;
  extern __shared__ uint64_t s_ok[];      // [WG_SMALL_DICT * nkl] order keys
  // merges spilled past the table (counters[1]) must be replayed first
  if (counters && counters[1] != 0ULL) { if (threadIdx.x == 0) *count_out = ~0ULL; return; }
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  const uint64_t total = nslots + (d.mode == 1 ? 1 : 0);
  for (uint64_t s = threadIdx.x; s < total; s += blockDim.x) {
    const uint64_t w0 = table[s * d.sw];
    const bool occ = (s == nslots) ? (w0 == 0ULL) : (d.mode == 1 ? w0 != 0xffffffffffffffffULL : w0 == 2ULL);
    if (occ) {
      const unsigned e = atomicAdd(&s_n, 1u);
      if (e < WG_SMALL_DICT) s_idx[e] = (uint32_t)s;
    }
  }
  __syncthreads();
  const unsigned n = s_n;
  if (threadIdx.x == 0) *count_out = n;
  if (n > WG_SMALL_DICT) return;             // the host takes the general path
  unsigned np = 1;
  while (np < n) np <<= 1;
  for (unsigned e = threadIdx.x; e < np; e += blockDim.x) {
    if (e >= n) { s_idx[e] = 0xffffffffu; continue; }
    const uint64_t s = s_idx[e];
    for (int l = 0; l < d.nkl; ++l) {
      uint64_t w;
      if (d.mode == 1) w = (s == nslots) ? 0xffffffffffffffffULL : table[s * d.sw];
      else w = table[s * d.sw + 1 + d.kword[l]];
      const uint64_t bits = d.kwidth[l] == 64 ? (w >> d.kshift[l]) : ((w >> d.kshift[l]) & ((1ULL << d.kwidth[l]) - 1));
      s_ok[(uint64_t)e * d.nkl + l] = wg_leaf_okey(bits, d.kkind[l]);
    }
  }
  __syncthreads();
  // bitonic sort of entry positions; the key tuple travels with its entry
  for (unsigned k = 2; k <= np; k <<= 1) {
    for (unsigned j = k >> 1; j > 0; j >>= 1) {
      for (unsigned i = threadIdx.x; i < np; i += blockDim.x) {
        const unsigned l = i ^ j;
        if (l <= i) continue;
        const bool up = (i & k) == 0;
        // compare entries i and l (padding sorts last)
        int c = 0;
        const bool pi = s_idx[i] == 0xffffffffu, pl = s_idx[l] == 0xffffffffu;
        if (pi || pl) c = (pi == pl) ? 0 : (pi ? 1 : -1);
        else
          for (int q = 0; q < d.nkl && !c; ++q) {
            const uint64_t a = s_ok[(uint64_t)i * d.nkl + q], b = s_ok[(uint64_t)l * d.nkl + q];
            c = a < b ? -1 : (a > b ? 1 : 0);
          }
        if ((c > 0) == up && c != 0) {
          const uint32_t t = s_idx[i]; s_idx[i] = s_idx[l]; s_idx[l] = t;
          for (int q = 0; q < d.nkl; ++q) {
            const uint64_t u = s_ok[(uint64_t)i * d.nkl + q];
            s_ok[(uint64_t)i * d.nkl + q] = s_ok[(uint64_t)l * d.nkl + q];
            s_ok[(uint64_t)l * d.nkl + q] = u;
          }
        }
      }
      __syncthreads();
    }
  }
  for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t s = s_idx[i];
    for (int l = 0; l < d.nkl; ++l) {
      uint64_t w;
      if (d.mode == 1) w = (s == nslots) ? 0xffffffffffffffffULL : table[s * d.sw];
      else w = table[s * d.sw + 1 + d.kword[l]];
      const uint64_t bits = d.kwidth[l] == 64 ? (w >> d.kshift[l]) : ((w >> d.kshift[l]) & ((1ULL << d.kwidth[l]) - 1));
      wg_store_leaf(d.out[l], i, bits, d.kkind[l]);
    }
    for (int f = 0; f < d.nvl; ++f) wg_store_leaf(d.out[d.nkl + f], i, table[s * d.sw + d.kbase + f], d.vkind[f]);
  }
}

// order key of element j of a typed integer/bool column (kind 0/1/2)
__device__ __forceinline__ uint64_t wg_okey_col(const void* src, int kind, uint64_t j) {
  switch (kind) {
    case 0: return ((const uint8_t*)src)[j];
    case 1: return (uint64_t)(int64_t)((const int32_t*)src)[j] ^ 0x8000000000000000ULL;
    default: return (uint64_t)((const int64_t*)src)[j] ^ 0x8000000000000000ULL;
  }
}

// Order keys of a key column, their min/max (mm[0..1]) and, when vals is
// given, the min/max of the 8-byte values' flipped bits v ^ 2^63 (mm[4..5]:
// the payload-narrowing test of the sort).
// With `spec`, also the 256-bin counts of the four top bytes of the order key
// (bits 32..63): the radix histogram of a sort over the top 32 of 64 varying
// bits, taken in the same read (used when min/max confirm that window).
__global__ void k_okey_minmax(const void* keys, int kind, uint64_t n, unsigned long long* mm, uint64_t* ok,
                              const uint64_t* vals, uint32_t* spec) {
  __shared__ uint32_t sh[4][256];
  if (spec) {
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
  }
  uint64_t lo = ~0ULL, hi = 0, vlo = ~0ULL, vhi = 0;
  uint64_t i0 = 0;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
  if (kind == 2 && ((((uintptr_t)keys) | ((uintptr_t)ok) | ((uintptr_t)vals)) & 31) == 0) {
    // 8-byte keys: four rows per thread with 256-bit loads/stores (sm_100)
    const uint64_t n4 = n / 4;
    for (uint64_t q = tid; q < n4; q += stride) {
      uint64_t k[4];
      asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(k[0]), "=l"(k[1]), "=l"(k[2]), "=l"(k[3]) : "l"((const uint64_t*)keys + 4 * q));
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        k[c] ^= 0x8000000000000000ULL;
        lo = k[c] < lo ? k[c] : lo;
        hi = k[c] > hi ? k[c] : hi;
        if (spec) {
#pragma unroll
          for (int d = 0; d < 4; ++d) atomicAdd(&sh[d][(unsigned)(k[c] >> (32 + 8 * d)) & 255u], 1u);
        }
      }
      asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(ok + 4 * q), "l"(k[0]), "l"(k[1]), "l"(k[2]), "l"(k[3])
                   : "memory");
      if (vals) {
        uint64_t w[4];
        asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(vals + 4 * q));
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint64_t x = w[c] ^ (1ULL << 63);
          vlo = x < vlo ? x : vlo;
          vhi = x > vhi ? x : vhi;
        }
      }
    }
    i0 = n4 * 4;
  }
  for (uint64_t i = i0 + tid; i < n; i += stride) {
    const uint64_t v = wg_okey_col(keys, kind, i);
    ok[i] = v;
    if (spec) {
#pragma unroll
      for (int d = 0; d < 4; ++d) atomicAdd(&sh[d][(unsigned)(v >> (32 + 8 * d)) & 255u], 1u);
    }
    lo = v < lo ? v : lo;
    hi = v > hi ? v : hi;
    if (vals) {
      const uint64_t w = __ldcs(vals + i) ^ (1ULL << 63);
      vlo = w < vlo ? w : vlo;
      vhi = w > vhi ? w : vhi;
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    uint64_t a = __shfl_xor_sync(0xffffffffu, lo, d), b = __shfl_xor_sync(0xffffffffu, hi, d);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
    a = __shfl_xor_sync(0xffffffffu, vlo, d);
    b = __shfl_xor_sync(0xffffffffu, vhi, d);
    vlo = a < vlo ? a : vlo;
    vhi = b > vhi ? b : vhi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
    if (vals) { atomicMin(mm + 4, vlo); atomicMax(mm + 5, vhi); }
  }
  if (spec) {
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) {
      const uint32_t c = (&sh[0][0])[i];
      if (c) atomicAdd(spec + i, c);
    }
  }
}

// order keys relative to the minimum (same order, fewer varying bits)
__global__ void k_sub_min(uint64_t* ok, uint64_t n, uint64_t kmin) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    ok[i] -= kmin;
}
// offsets of a vector of fixed-length vectors: dst[j] = j * step
__global__ void k_iota_i64(int64_t* dst, uint64_t n, int64_t step) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = (int64_t)i * step;
}
// exclusive scan of n i64 counts by one CTA (tile offsets of the two-pass
// order-preserving appender schedule); *total = sum
__global__ void __launch_bounds__(1024) k_exscan_i64(const int64_t* src, int64_t* dst, uint64_t n, int64_t* total) {
  __shared__ int64_t s_w[32];
  __shared__ int64_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t base = 0; base < n; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const int64_t x = i < n ? src[i] : 0;
    int64_t incl = x;
    for (int d = 1; d < 32; d <<= 1) { const int64_t o = __shfl_up_sync(0xffffffffu, incl, d); if (lane >= d) incl += o; }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = s_w[lane], wi = w;
      for (int d = 1; d < 32; d <<= 1) { const int64_t o = __shfl_up_sync(0xffffffffu, wi, d); if (lane >= d) wi += o; }
      s_w[lane] = wi - w;
    }
    __syncthreads();
    const int64_t carry = s_carry;
    if (i < n) dst[i] = carry + s_w[warp] + incl - x;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = carry + s_w[31] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = s_carry;
}
// The canonical +0.0 key of a float dictionary column becomes -0.0 (the
// first-inserted key object, builders.py:346-351).
__global__ void k_neg_zero(void* col, uint64_t n, int width) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (width == 8) { uint64_t* c = (uint64_t*)col; if (c[i] == 0) c[i] = 0x8000000000000000ULL; }
    else { uint32_t* c = (uint32_t*)col; if (c[i] == 0) c[i] = 0x80000000U; }
  }
}
// Reallocation accounting of an unhinted vecbuilder (builders.py:256-272):
// coff[c] = output position where chunk c of the launch starts (coff[0] = 0),
// *total = the launch's appends.  A segment of k appends starts at capacity
// 16 and doubles while full: cap(k) = 16 << dbl(k), dbl(k) = ceil(log2(k)) - 4
// for k > 16.  out[0..1] += sum dbl / sum cap over the interior chunks
// 1..nch-2; out[2], out[3] = appends of the first and last chunk (segments a
// neighbouring launch of the same loop may share; the host folds those).
__global__ void k_seg_stats(const int64_t* coff, uint64_t nch, const int64_t* total, unsigned long long* out) {
  unsigned long long d = 0, c = 0;
  const int64_t tot = *total;
  for (uint64_t i = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < nch; i += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t k = coff[i + 1] - coff[i];
    if (k > 0) {
      const int db = k <= 16 ? 0 : (64 - __clzll((unsigned long long)(k - 1))) - 4;
      d += (unsigned long long)db;
      c += 16ULL << db;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if ((threadIdx.x & 31) == 0 && (d | c)) { atomicAdd(out, d); atomicAdd(out + 1, c); }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[2] = (unsigned long long)((nch > 1 ? coff[1] : tot) - coff[0]);
    out[3] = (unsigned long long)(nch > 1 ? tot - coff[nch - 1] : 0);
  }
}
}  // namespace

// ===========================================================================
extern "C" {

const char* wg_last_error(void) { return g_err.c_str(); }

int wg_version(void) { return 1; }

int wg_device_count(int* n) {
  CK(cudaGetDeviceCount(n));
  return 0;
}

int wg_init(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_inited) {
    if (device == g_device) return 0;
    return fail("weldgpu: already initialised on a different device");
  }
  CK(cudaSetDevice(device));
  CK(cudaFree(0));
  if (!resolve("cuGetErrorString", &p_cuGetErrorString) || !resolve("cuModuleLoadData", &p_cuModuleLoadData) ||
      !resolve("cuModuleGetFunction", &p_cuModuleGetFunction) || !resolve("cuLaunchKernel", &p_cuLaunchKernel) ||
      !resolve("cuOccupancyMaxActiveBlocksPerMultiprocessor", &p_cuOccupancyMaxActiveBlocksPerMultiprocessor) ||
      !resolve("cuFuncSetAttribute", &p_cuFuncSetAttribute))
    return fail("weldgpu: could not resolve CUDA driver entry points");
  for (int i = 0; i < 3; ++i) CK(cudaStreamCreateWithFlags(&g_streams[i], cudaStreamNonBlocking));
  g_stream = g_streams[0];
  CK(cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, device));
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;  // temporaries (sort scratch) use the stream-ordered pool
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  CK(cudaMalloc((void**)&g_err_word, 64));
  CK(cudaMemset(g_err_word, 0, 64));
  CK(cudaMallocHost((void**)&g_err_host, 64));
  g_device = device;
  g_inited = true;
  return 0;
}

int wg_sm_count(int* n) { NEED_INIT(); *n = g_sm_count; return 0; }

int wg_stream(uint64_t* s) { NEED_INIT(); *s = (uint64_t)(uintptr_t)g_stream; return 0; }

int wg_sync(void) { NEED_INIT(); CK(cudaStreamSynchronize(g_stream)); return 0; }

// ---- buffer manager --------------------------------------------------------
// Caching allocator.  Everything runs on one stream, so a freed block can
// be handed to the next request immediately: stream order guarantees the
// previous user's kernels finished before the new user's start.  Blocks
// are rounded (pow2 below 2 MiB, 2 MiB multiples above) and a request
// reuses any cached block up to 2x its size.  cudaMalloc runs only when
// the cache cannot serve a request (and on OOM the cache is released and
// the request retried).
int wg_alloc(uint64_t bytes, uint64_t* dptr) {
  NEED_INIT();
  uint64_t b = bytes ? bytes : 1;
  if (b < (2ULL << 20)) {
    uint64_t r = 256;
    while (r < b) r <<= 1;
    b = r;
  } else {
    b = (b + (2ULL << 20) - 1) & ~((2ULL << 20) - 1);
  }
  void* p = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_acct_mu);
    auto it = g_free.lower_bound(b);
    if (it != g_free.end() && it->first <= 2 * b) {
      p = it->second;
      b = it->first;
      g_free.erase(it);
      g_cached -= b;
    }
  }
  if (!p) {
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
      cudaGetLastError();
      for (int i = 0; i < 3; ++i) CK(cudaStreamSynchronize(g_streams[i]));
      {
        std::lock_guard<std::mutex> lk(g_acct_mu);
        release_deferred();
        for (auto& kv : g_free) cudaFree(kv.second);
        g_free.clear();
        g_cached = 0;
      }
      CK(cudaMalloc(&p, b));
    }
  }
  *dptr = (uint64_t)(uintptr_t)p;
  // WELDGPU_POISON=1: every block handed out is filled with 0xA5 bytes, so a
  // kernel that relies on zeroed memory fails deterministically in tests
  static const int poison = getenv("WELDGPU_POISON") && getenv("WELDGPU_POISON")[0] == '1';
  if (poison) CK(cudaMemsetAsync(p, 0xA5, b, g_stream));
  std::lock_guard<std::mutex> lk(g_acct_mu);
  g_live += b;
  if (g_live > g_peak) g_peak = g_live;
  g_sizes[p] = b;
  return 0;
}

int wg_free(uint64_t dptr) {
  NEED_INIT();
  if (!dptr) return 0;
  void* p = (void*)(uintptr_t)dptr;
  std::lock_guard<std::mutex> lk(g_acct_mu);
  auto it = g_sizes.find(p);
  if (it == g_sizes.end()) return fail("wg_free: unknown device pointer");
  g_live -= it->second;
  if (g_multi) g_deferred.emplace_back(it->second, p);
  else {
    g_free.emplace(it->second, p);
    g_cached += it->second;
  }
  g_sizes.erase(it);
  return 0;
}


int wg_mem_trim(void) {
  NEED_INIT();
  for (int i = 0; i < 3; ++i) CK(cudaStreamSynchronize(g_streams[i]));
  std::lock_guard<std::mutex> lk(g_acct_mu);
  release_deferred();
  for (auto& kv : g_free) cudaFree(kv.second);
  g_free.clear();
  g_cached = 0;
  return 0;
}

int wg_mem_stats(uint64_t* live, uint64_t* peak) {
  std::lock_guard<std::mutex> lk(g_acct_mu);
  *live = g_live;
  *peak = g_peak;
  return 0;
}

int wg_mem_reset_peak(void) {
  std::lock_guard<std::mutex> lk(g_acct_mu);
  g_peak = g_live;
  return 0;
}

int wg_memset(uint64_t dptr, int value, uint64_t bytes) {
  NEED_INIT();
  if (!bytes) return 0;
  WG_PROF("memset");
  CK(cudaMemsetAsync((void*)(uintptr_t)dptr, value, bytes, g_stream));
  return 0;
}

int wg_h2d(uint64_t dst, const void* src, uint64_t bytes) {
  NEED_INIT();
  if (!bytes) return 0;
  CK(cudaMemcpyAsync((void*)(uintptr_t)dst, src, bytes, cudaMemcpyHostToDevice, g_stream));
  return 0;
}

int wg_d2h(void* dst, uint64_t src, uint64_t bytes) {
  NEED_INIT();
  if (!bytes) return 0;
  CK(cudaMemcpyAsync(dst, (const void*)(uintptr_t)src, bytes, cudaMemcpyDeviceToHost, g_stream));
  CK(cudaStreamSynchronize(g_stream));
  return 0;
}

int wg_d2h_async(void* dst, uint64_t src, uint64_t bytes) {
  NEED_INIT();
  if (!bytes) return 0;
  CK(cudaMemcpyAsync(dst, (const void*)(uintptr_t)src, bytes, cudaMemcpyDeviceToHost, g_stream));
  return 0;
}

int wg_d2d(uint64_t dst, uint64_t src, uint64_t bytes) {
  NEED_INIT();
  if (!bytes) return 0;
  WG_PROF("memcpy_d2d");
  CK(cudaMemcpyAsync((void*)(uintptr_t)dst, (const void*)(uintptr_t)src, bytes, cudaMemcpyDeviceToDevice, g_stream));
  return 0;
}

int wg_host_alloc(uint64_t bytes, void** p) {
  NEED_INIT();
  CK(cudaMallocHost(p, bytes ? bytes : 1));
  return 0;
}

int wg_host_free(void* p) {
  NEED_INIT();
  CK(cudaFreeHost(p));
  return 0;
}

int wg_host_register(void* p, uint64_t bytes) {
  NEED_INIT();
  CK(cudaHostRegister(p, bytes, cudaHostRegisterDefault));
  return 0;
}

int wg_host_unregister(void* p) {
  NEED_INIT();
  CK(cudaHostUnregister(p));
  return 0;
}

// ---- device error word -----------------------------------------------------
int wg_error_ptr(uint64_t* p) { NEED_INIT(); *p = (uint64_t)(uintptr_t)g_err_word; return 0; }

int wg_read_error(int64_t* code, int64_t* info) {
  NEED_INIT();
  CK(cudaMemcpyAsync(g_err_host, g_err_word, 16, cudaMemcpyDeviceToHost, g_stream));
  CK(cudaStreamSynchronize(g_stream));
  *code = g_err_host[0];
  *info = g_err_host[1];
  if (g_err_host[0] != 0) CK(cudaMemsetAsync(g_err_word, 0, 16, g_stream));
  return 0;
}

// A result read-back and the error-word check in one synchronisation (the
// common tail of an evaluate(): a merger's slot, then "did any kernel raise").
int wg_d2h_checked(void* dst, uint64_t src, uint64_t bytes, int64_t* code, int64_t* info) {
  NEED_INIT();
  if (bytes) CK(cudaMemcpyAsync(dst, (const void*)(uintptr_t)src, bytes, cudaMemcpyDeviceToHost, g_stream));
  CK(cudaMemcpyAsync(g_err_host, g_err_word, 16, cudaMemcpyDeviceToHost, g_stream));
  CK(cudaStreamSynchronize(g_stream));
  *code = g_err_host[0];
  *info = g_err_host[1];
  if (g_err_host[0] != 0) CK(cudaMemsetAsync(g_err_word, 0, 16, g_stream));
  return 0;
}

// ---- NVRTC compile + module cache -----------------------------------------
int wg_compile(const char* src, const char* name, int nheaders, const char* const* header_srcs,
               const char* const* header_names, int nopts, const char* const* opts,
               uint64_t* module_out, char* log_buf, uint64_t log_cap) {
  NEED_INIT();
  nvrtcProgram prog;
  CKN(nvrtcCreateProgram(&prog, src, name, nheaders, header_srcs, header_names));
  nvrtcResult rc = nvrtcCompileProgram(prog, nopts, opts);
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  std::string log(log_size, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &log[0]);
  if (log_buf && log_cap) {
    size_t n = log.size() < log_cap - 1 ? log.size() : log_cap - 1;
    memcpy(log_buf, log.data(), n);
    log_buf[n] = 0;
  }
  if (rc != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return fail(std::string("nvrtc compile failed: ") + nvrtcGetErrorString(rc) + "\n" + log);
  }
  size_t cubin_size = 0;
  CKN(nvrtcGetCUBINSize(prog, &cubin_size));
  std::vector<char> cubin(cubin_size);
  CKN(nvrtcGetCUBIN(prog, cubin.data()));
  nvrtcDestroyProgram(&prog);
  CUmodule mod;
  CKD(p_cuModuleLoadData(&mod, cubin.data()));
  *module_out = (uint64_t)(uintptr_t)mod;
  return 0;
}

// Compile only (no device needed): used by the CPU test-suite and build() to
// prove every generated kernel compiles for sm_100a.  Returns the cubin size.
int wg_compile_check(const char* src, const char* name, int nheaders, const char* const* header_srcs,
                     const char* const* header_names, int nopts, const char* const* opts,
                     uint64_t* cubin_bytes, char* log_buf, uint64_t log_cap) {
  nvrtcProgram prog;
  CKN(nvrtcCreateProgram(&prog, src, name, nheaders, header_srcs, header_names));
  nvrtcResult rc = nvrtcCompileProgram(prog, nopts, opts);
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  std::string log(log_size, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &log[0]);
  if (log_buf && log_cap) {
    size_t n = log.size() < log_cap - 1 ? log.size() : log_cap - 1;
    memcpy(log_buf, log.data(), n);
    log_buf[n] = 0;
  }
  if (rc != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return fail(std::string("nvrtc compile failed: ") + nvrtcGetErrorString(rc) + "\n" + log);
  }
  size_t cubin_size = 0;
  CKN(nvrtcGetCUBINSize(prog, &cubin_size));
  nvrtcDestroyProgram(&prog);
  *cubin_bytes = cubin_size;
  return 0;
}

// PTX of a program (the executor's constant-pool pass rewrites it before the
// driver JIT compiles it for the device): *ptx_size is the PTX length + 1; a
// NULL / too-small buffer just reports the size.
int wg_compile_ptx(const char* src, const char* name, int nheaders, const char* const* header_srcs,
                   const char* const* header_names, int nopts, const char* const* opts, char* ptx_out,
                   uint64_t ptx_cap, uint64_t* ptx_size, char* log_buf, uint64_t log_cap) {
  nvrtcProgram prog;
  CKN(nvrtcCreateProgram(&prog, src, name, nheaders, header_srcs, header_names));
  nvrtcResult rc = nvrtcCompileProgram(prog, nopts, opts);
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  std::string log(log_size, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &log[0]);
  if (log_buf && log_cap) {
    size_t n = log.size() < log_cap - 1 ? log.size() : log_cap - 1;
    memcpy(log_buf, log.data(), n);
    log_buf[n] = 0;
  }
  if (rc != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return fail(std::string("nvrtc compile failed: ") + nvrtcGetErrorString(rc) + "\n" + log);
  }
  size_t n = 0;
  CKN(nvrtcGetPTXSize(prog, &n));
  *ptx_size = n;
  if (ptx_out && ptx_cap >= n) CKN(nvrtcGetPTX(prog, ptx_out));
  nvrtcDestroyProgram(&prog);
  return 0;
}

// Load a module image (cubin, or PTX text that the driver JIT-compiles).
int wg_module_load(const char* image, uint64_t* module_out) {
  NEED_INIT();
  CUmodule mod;
  CKD(p_cuModuleLoadData(&mod, image));
  *module_out = (uint64_t)(uintptr_t)mod;
  return 0;
}

int wg_module_function(uint64_t module, const char* name, uint64_t* fn) {
  NEED_INIT();
  CUfunction f;
  CKD(p_cuModuleGetFunction(&f, (CUmodule)(uintptr_t)module, name));
  *fn = (uint64_t)(uintptr_t)f;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_fn_names[*fn] = name;
  return 0;
}

int wg_occupancy(uint64_t fn, int block, int dyn_smem, int* blocks_per_sm) {
  NEED_INIT();
  if (dyn_smem > 0)  // opt in to exactly the requested dynamic shared memory (static + dynamic <= 227 KB)
    CKD(p_cuFuncSetAttribute((CUfunction)(uintptr_t)fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, dyn_smem));
  CKD(p_cuOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, (CUfunction)(uintptr_t)fn, block, (size_t)dyn_smem));
  return 0;
}

int wg_launch(uint64_t fn, uint32_t grid, uint32_t block, uint32_t dyn_smem, const void* params, uint64_t params_size) {
  NEED_INIT();
  CUfunction f = (CUfunction)(uintptr_t)fn;
  if (dyn_smem > 0)
    CKD(p_cuFuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)dyn_smem));
  size_t sz = (size_t)params_size;
  void* extra[] = {CU_LAUNCH_PARAM_BUFFER_POINTER, const_cast<void*>(params), CU_LAUNCH_PARAM_BUFFER_SIZE, &sz,
                   CU_LAUNCH_PARAM_END};
  const char* pname = "nvrtc_kernel";
  if (g_prof_on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    auto it = g_fn_names.find(fn);
    if (it != g_fn_names.end()) pname = it->second.c_str();
  }
  WG_PROF(pname);
  CKD(p_cuLaunchKernel(f, grid, 1, 1, block, 1, 1, dyn_smem, (CUstream)g_stream, nullptr, extra));
  return 0;
}

// ---- builder finalisation helpers -------------------------------------------
int wg_table_init(uint64_t table, uint64_t nslots, int slot_words, const uint64_t* pattern) {
  NEED_INIT();
  if (slot_words < 1 || slot_words > 64) return fail("wg_table_init: slot_words out of range");
  uint64_t* pat = nullptr;
  CK(cudaMallocAsync((void**)&pat, 64 * 8, g_stream));
  CK(cudaMemcpyAsync(pat, pattern, slot_words * 8, cudaMemcpyHostToDevice, g_stream));
  uint64_t total = nslots * (uint64_t)slot_words;
  { WG_PROF("k_table_init"); k_table_init<<<grid_for(total, 256), 256, 0, g_stream>>>((uint64_t*)(uintptr_t)table, nslots, slot_words, pat); }
  CK(cudaGetLastError());
  CK(cudaFreeAsync(pat, g_stream));
  return 0;
}

int wg_table_compact(uint64_t table, uint64_t nslots, int slot_words, int mode, const uint64_t* out_words,
                     int nout, uint64_t* count_out) {
  NEED_INIT();
  uint64_t** d_out = nullptr;
  unsigned long long* d_cnt = nullptr;
  CK(cudaMallocAsync((void**)&d_out, sizeof(uint64_t*) * (nout + 1), g_stream));
  CK(cudaMallocAsync((void**)&d_cnt, 8, g_stream));
  CK(cudaMemcpyAsync(d_out, out_words, sizeof(uint64_t) * nout, cudaMemcpyHostToDevice, g_stream));
  CK(cudaMemsetAsync(d_cnt, 0, 8, g_stream));
  { WG_PROF("k_table_compact"); k_table_compact<<<grid_for(nslots, 256), 256, 0, g_stream>>>((const uint64_t*)(uintptr_t)table, nslots,
                                                                slot_words, mode, d_out, nout, d_cnt); }
  CK(cudaGetLastError());
  if (mode == 1) {
    { WG_PROF("k_table_compact_sentinel"); k_table_compact_sentinel<<<1, 32, 0, g_stream>>>((const uint64_t*)(uintptr_t)table, nslots, slot_words, d_out,
                                                     nout, d_cnt); }
    CK(cudaGetLastError());
  }
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, d_cnt, 8, cudaMemcpyDeviceToHost, g_stream));
  CK(cudaStreamSynchronize(g_stream));
  CK(cudaFreeAsync(d_out, g_stream));
  CK(cudaFreeAsync(d_cnt, g_stream));
  *count_out = h;
  return 0;
}

// Small dictmerger result in one launch (see k_dict_finish_small).  key_desc:
// 4 ints per key leaf (word, shift, width, kind); val_kinds: one per value
// field; outs: nkl + nvl typed device columns of capacity >= the entry
// count.  *count_out receives the number of entries; when it exceeds
// WG_SMALL_DICT nothing is written and the caller uses the general path.
int wg_dict_finish_small(uint64_t table, uint64_t nslots, int slot_words, int mode, int nw, int nkl,
                         const int* key_desc, int nvl, const int* val_kinds, const uint64_t* outs,
                         uint64_t counters, uint64_t* count_out) {
  NEED_INIT();
  if (nkl > 6 || nvl > 16) return fail("wg_dict_finish_small: too many key/value leaves");
  SmallDictDesc d;
  memset(&d, 0, sizeof(d));
  d.nkl = nkl; d.nvl = nvl; d.mode = mode; d.nw = nw; d.sw = slot_words;
  d.kbase = mode == 1 ? 1 : 1 + nw;
  for (int l = 0; l < nkl; ++l) {
    d.kword[l] = key_desc[4 * l]; d.kshift[l] = key_desc[4 * l + 1];
    d.kwidth[l] = key_desc[4 * l + 2]; d.kkind[l] = key_desc[4 * l + 3];
  }
  for (int f = 0; f < nvl; ++f) d.vkind[f] = val_kinds[f];
  for (int i = 0; i < nkl + nvl; ++i) d.out[i] = (void*)(uintptr_t)outs[i];
  unsigned long long* d_cnt = (unsigned long long*)g_err_word + 2;   // scratch word next to the error word
  const int smem = WG_SMALL_DICT * nkl * 8;
  static bool attr_set = false;
  if (!attr_set) {
    CK(cudaFuncSetAttribute(k_dict_finish_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * WG_SMALL_DICT * 8));
    attr_set = true;
  }
  { WG_PROF("k_dict_finish_small"); k_dict_finish_small<<<1, 1024, smem, g_stream>>>((const uint64_t*)(uintptr_t)table, nslots, d,
                                                   (const unsigned long long*)(uintptr_t)counters, d_cnt); }
  CK(cudaGetLastError());
  // the entry count and the error word (its neighbour) in one copy and one
  // synchronisation; the error word is kept for wg_last_sync_error
  CK(cudaMemcpyAsync(g_err_host + 4, g_err_word, 24, cudaMemcpyDeviceToHost, g_stream));
  CK(cudaStreamSynchronize(g_stream));
  *count_out = (uint64_t)g_err_host[6];
  g_sync_err[0] = g_err_host[4];
  g_sync_err[1] = g_err_host[5];
  if (g_sync_err[0] != 0) CK(cudaMemsetAsync(g_err_word, 0, 16, g_stream));
  return 0;
}

// The error word as read by the last synchronising call that captures it
// (wg_dict_finish_small), then forgotten: the host needs no second copy.
int wg_last_sync_error(int64_t* code, int64_t* info) {
  *code = g_sync_err[0];
  *info = g_sync_err[1];
  g_sync_err[0] = g_sync_err[1] = 0;
  return 0;
}

int wg_order_key(uint64_t src, int kind, uint64_t n, uint64_t perm, uint64_t dst) {
  NEED_INIT();
  if (!n) return 0;
  { WG_PROF("k_order_key"); k_order_key<<<grid_for(n, 256), 256, 0, g_stream>>>((const void*)(uintptr_t)src, kind, n,
                                                       (const uint32_t*)(uintptr_t)perm, (uint64_t*)(uintptr_t)dst); }
  CK(cudaGetLastError());
  return 0;
}

int wg_neg_zero(uint64_t col, uint64_t n, int width) {
  NEED_INIT();
  if (!n) return 0;
  { WG_PROF("k_neg_zero"); k_neg_zero<<<grid_for(n, 256), 256, 0, g_stream>>>((void*)(uintptr_t)col, n, width); }
  CK(cudaGetLastError());
  return 0;
}

int wg_seg_stats(uint64_t coff, uint64_t nch, uint64_t total, uint64_t out) {
  NEED_INIT();
  CK(cudaMemsetAsync((void*)(uintptr_t)out, 0, 2 * sizeof(uint64_t), g_stream));
  const unsigned grid = nch > 2 ? grid_for(nch - 2, 256) : 1;
  { WG_PROF("k_seg_stats"); k_seg_stats<<<grid, 256, 0, g_stream>>>((const int64_t*)(uintptr_t)coff, nch,
                                         (const int64_t*)(uintptr_t)total, (unsigned long long*)(uintptr_t)out); }
  CK(cudaGetLastError());
  return 0;
}

int wg_exclusive_scan_i64(uint64_t src, uint64_t dst, uint64_t n, uint64_t total) {
  NEED_INIT();
  { WG_PROF("k_exscan_i64"); k_exscan_i64<<<1, 1024, 0, g_stream>>>((const int64_t*)(uintptr_t)src, (int64_t*)(uintptr_t)dst, n,
                                         (int64_t*)(uintptr_t)total); }
  CK(cudaGetLastError());
  return 0;
}

int wg_iota_i64(uint64_t dst, uint64_t n, int64_t step) {
  NEED_INIT();
  if (!n) return 0;
  { WG_PROF("k_iota_i64"); k_iota_i64<<<grid_for(n, 256), 256, 0, g_stream>>>((int64_t*)(uintptr_t)dst, n, step); }
  CK(cudaGetLastError());
  return 0;
}

int wg_iota_u32(uint64_t dst, uint64_t n) {
  NEED_INIT();
  if (!n) return 0;
  { WG_PROF("k_iota_u32"); k_iota_u32<<<grid_for(n, 256), 256, 0, g_stream>>>((uint32_t*)(uintptr_t)dst, n); }
  CK(cudaGetLastError());
  return 0;
}

}  // extern "C"

namespace {

// Stable LSD radix sort of (key, value) pairs over key bits [begin_bit,
// end_bit) with the onesweep kernels of wg_radix.cuh.  The first pass reads
// (kin, vin); the result lands in (kA, vA); (kB, vB) are ping-pong scratch.
// Stability is what makes multi-field lexicographic sorts (last field first)
// and order-preserving grouping correct.
template <typename K, typename VI, typename VS, typename VO, typename CV>
int onesweep_pass(const K* ki, const VI* vi, K* ko, VO* vo, uint64_t n, int shift, int wbits, const uint32_t* gofs,
                  unsigned long long* status, uint32_t* ctr, uint64_t vbase) {
  constexpr int ITEMS = 8, TILE = 512 * ITEMS;
  constexpr int SMEM = wgr::onesweep_smem<K, VS, ITEMS>();
  static bool attr_set = false;   // per template instance
  if (!attr_set) {
    CK(cudaFuncSetAttribute(wgr::k_onesweep<K, VI, VS, VO, CV, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    attr_set = true;
  }
  const uint64_t tiles = (n + TILE - 1) / TILE;
  CK(cudaMemsetAsync(status, 0, tiles * wgr::RADIX * 8, g_stream));
  { WG_PROF("k_onesweep"); wgr::k_onesweep<K, VI, VS, VO, CV, ITEMS><<<(unsigned)tiles, 512, SMEM, g_stream>>>(
      ki, vi, ko, vo, (uint32_t)n, shift, (1u << wbits) - 1u, gofs, status, ctr, vbase); }
  CK(cudaGetLastError());
  return 0;
}

// Radix histogram of the top 32 of 64 order-key bits taken by k_okey_minmax
// (wg_group_finish1 sets it around its sort when that is the sort's window).
static const uint32_t* g_pre_hist = nullptr;

// Histogram + offsets of every pass; *status sized for the tiles of a pass.
template <typename K>
int radix_prologue(const K* kin, uint64_t n, int begin_bit, int end_bit, int npass, uint32_t** hist,
                   unsigned long long** status) {
  const uint64_t tiles = (n + 4095) / 4096;
  CK(cudaMallocAsync((void**)hist, (npass * wgr::RADIX + npass) * 4, g_stream));
  CK(cudaMemsetAsync(*hist, 0, (npass * wgr::RADIX + npass) * 4, g_stream));
  CK(cudaMallocAsync((void**)status, tiles * wgr::RADIX * 8, g_stream));
  if (g_pre_hist && sizeof(K) == 8 && npass == 4 && begin_bit == 32 && end_bit == 64)
    CK(cudaMemcpyAsync(*hist, g_pre_hist, 4 * wgr::RADIX * 4, cudaMemcpyDeviceToDevice, g_stream));
  else { WG_PROF("k_radix_hist"); wgr::k_radix_hist<K><<<grid_for(n, 256), 256, 0, g_stream>>>(kin, n, begin_bit, end_bit, npass, *hist); }
  { WG_PROF("k_radix_offsets"); wgr::k_radix_offsets<<<npass, wgr::RADIX, 0, g_stream>>>(*hist); }
  return 0;
}

template <typename K, typename V>
int radix_sort(const K* kin, const V* vin, K* kA, K* kB, V* vA, V* vB, uint64_t n, int begin_bit, int end_bit) {
  if (n > 0xffffffffULL) return fail("radix sort: more than 2^32 items");
  if (!n) return 0;
  const int npass = end_bit > begin_bit ? (end_bit - begin_bit + 7) / 8 : 0;
  if (npass == 0) {
    if ((const void*)kA != (const void*)kin) CK(cudaMemcpyAsync(kA, kin, n * sizeof(K), cudaMemcpyDeviceToDevice, g_stream));
    if ((const void*)vA != (const void*)vin) CK(cudaMemcpyAsync(vA, vin, n * sizeof(V), cudaMemcpyDeviceToDevice, g_stream));
    return 0;
  }
  uint32_t* hist;
  unsigned long long* status;
  if (radix_prologue<K>(kin, n, begin_bit, end_bit, npass, &hist, &status)) return -1;
  uint32_t* ctr = hist + npass * wgr::RADIX;
  const K* ki = kin;
  const V* vi = vin;
  for (int p = 0; p < npass; ++p) {
    const bool toA = ((npass - 1 - p) & 1) == 0;
    K* ko = toA ? kA : kB;
    V* vo = toA ? vA : vB;
    const int shift = begin_bit + 8 * p;
    const int wbits = end_bit - shift < 8 ? end_bit - shift : 8;
    if (onesweep_pass<K, V, V, V, wgr::VCopy>(ki, vi, ko, vo, n, shift, wbits, hist + p * wgr::RADIX, status, ctr + p, 0))
      return -1;
    ki = ko;
    vi = vo;
  }
  CK(cudaFreeAsync(status, g_stream));
  CK(cudaFreeAsync(hist, g_stream));
  return 0;
}

// The same sort with a narrowed payload: 8-byte values whose flipped bits
// (v ^ 2^63) lie in [vbase, vbase + 2^32) travel as u32 offsets (t0/t1
// scratch, n words each) -- 12 instead of 16 bytes per row per pass for u64
// keys.  Needs at least two passes; the result lands in (kA, vout).
template <typename K>
int radix_sort_narrow(const K* kin, const uint64_t* vin, K* kA, K* kB, uint64_t* vout, uint32_t* t0, uint32_t* t1,
                      uint64_t n, int begin_bit, int end_bit, uint64_t vbase) {
  if (n > 0xffffffffULL) return fail("radix sort: more than 2^32 items");
  const int npass = end_bit > begin_bit ? (end_bit - begin_bit + 7) / 8 : 0;
  if (npass < 2) return fail("radix_sort_narrow: needs two passes or more");
  uint32_t* hist;
  unsigned long long* status;
  if (radix_prologue<K>(kin, n, begin_bit, end_bit, npass, &hist, &status)) return -1;
  uint32_t* ctr = hist + npass * wgr::RADIX;
  const K* ki = kin;
  const uint32_t* ti = nullptr;
  for (int p = 0; p < npass; ++p) {
    const bool toA = ((npass - 1 - p) & 1) == 0;
    K* ko = toA ? kA : kB;
    uint32_t* to = (p & 1) ? t1 : t0;
    const int shift = begin_bit + 8 * p;
    const int wbits = end_bit - shift < 8 ? end_bit - shift : 8;
    int rc;
    if (p == 0)
      rc = onesweep_pass<K, uint64_t, uint32_t, uint32_t, wgr::VNarrow>(ki, vin, ko, to, n, shift, wbits, hist, status, ctr, vbase);
    else if (p == npass - 1)
      rc = onesweep_pass<K, uint32_t, uint32_t, uint64_t, wgr::VWiden>(ki, ti, ko, vout, n, shift, wbits, hist + p * wgr::RADIX,
                                                                       status, ctr + p, vbase);
    else
      rc = onesweep_pass<K, uint32_t, uint32_t, uint32_t, wgr::VCopy>(ki, ti, ko, to, n, shift, wbits, hist + p * wgr::RADIX,
                                                                      status, ctr + p, 0);
    if (rc) return -1;
    ki = ko;
    ti = to;
  }
  CK(cudaFreeAsync(status, g_stream));
  CK(cudaFreeAsync(hist, g_stream));
  return 0;
}

// Run starts of sorted keys (u32 positions) and their count (host).
template <typename EQ>
int run_heads(EQ eq, uint64_t n, uint32_t* starts, uint64_t* count) {
  if (!n) { *count = 0; return 0; }
  constexpr int ITEMS = 16, TILE = 256 * ITEMS;
  const uint64_t tiles = (n + TILE - 1) / TILE;
  unsigned long long* st;
  CK(cudaMallocAsync((void**)&st, tiles * 8 + 16, g_stream));
  CK(cudaMemsetAsync(st, 0, tiles * 8 + 16, g_stream));
  unsigned long long* total = st + tiles;
  uint32_t* ctr = (uint32_t*)(st + tiles + 1);
  { WG_PROF("k_run_heads"); wgr::k_run_heads<EQ, ITEMS><<<(unsigned)tiles, 256, 0, g_stream>>>(eq, n, starts, st, ctr, total); }
  CK(cudaGetLastError());
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, total, 8, cudaMemcpyDeviceToHost, g_stream));
  CK(cudaStreamSynchronize(g_stream));
  CK(cudaFreeAsync(st, g_stream));
  *count = h;
  return 0;
}

}  // namespace

extern "C" {

int wg_sort_pairs(uint64_t keys_in, uint64_t vals_in, uint64_t keys_out, uint64_t vals_out, uint64_t n,
                  int begin_bit, int end_bit) {
  NEED_INIT();
  if (!n) return 0;
  if (n > 0xffffffffULL) return fail("wg_sort_pairs: more than 2^32 items");
  uint64_t* kB;
  uint32_t* vB;
  CK(cudaMallocAsync((void**)&kB, n * 8, g_stream));
  CK(cudaMallocAsync((void**)&vB, n * 4, g_stream));
  int rc = radix_sort<uint64_t, uint32_t>((const uint64_t*)(uintptr_t)keys_in, (const uint32_t*)(uintptr_t)vals_in,
                                          (uint64_t*)(uintptr_t)keys_out, kB, (uint32_t*)(uintptr_t)vals_out, vB, n,
                                          begin_bit, end_bit);
  CK(cudaFreeAsync(kB, g_stream));
  CK(cudaFreeAsync(vB, g_stream));
  return rc;
}

int wg_gather(uint64_t src, uint64_t perm, uint64_t dst, uint64_t n, int width) {
  NEED_INIT();
  if (!n) return 0;
  unsigned g = grid_for(n, 256);
  const uint32_t* pm = (const uint32_t*)(uintptr_t)perm;
  switch (width) {
    case 8: { WG_PROF("k_gather"); k_gather<uint64_t><<<g, 256, 0, g_stream>>>((const uint64_t*)(uintptr_t)src, pm, (uint64_t*)(uintptr_t)dst, n); } break;
    case 4: { WG_PROF("k_gather"); k_gather<uint32_t><<<g, 256, 0, g_stream>>>((const uint32_t*)(uintptr_t)src, pm, (uint32_t*)(uintptr_t)dst, n); } break;
    case 1: { WG_PROF("k_gather"); k_gather<uint8_t><<<g, 256, 0, g_stream>>>((const uint8_t*)(uintptr_t)src, pm, (uint8_t*)(uintptr_t)dst, n); } break;
    default: return fail("wg_gather: width must be 1, 4 or 8");
  }
  CK(cudaGetLastError());
  return 0;
}

int wg_narrow(uint64_t src, uint64_t dst, int width, uint64_t n) {
  NEED_INIT();
  if (!n) return 0;
  { WG_PROF("k_narrow"); k_narrow<<<grid_for(n, 256), 256, 0, g_stream>>>((const uint64_t*)(uintptr_t)src, (void*)(uintptr_t)dst, width, n); }
  CK(cudaGetLastError());
  return 0;
}

int wg_widen(uint64_t src, uint64_t dst, int width, uint64_t n) {
  NEED_INIT();
  if (!n) return 0;
  { WG_PROF("k_widen"); k_widen<<<grid_for(n, 256), 256, 0, g_stream>>>((const void*)(uintptr_t)src, (uint64_t*)(uintptr_t)dst, width, n); }
  CK(cudaGetLastError());
  return 0;
}

// Positions where a new key run starts in sorted multi-word keys; returns
// the run starts (u32) and their count.
int wg_run_starts(const uint64_t* key_words, int kw, uint64_t n, uint64_t starts_out, uint64_t* nruns) {
  NEED_INIT();
  if (!n) { *nruns = 0; return 0; }
  if (n > 0xffffffffULL) return fail("wg_run_starts: more than 2^32 items");
  uint64_t** d_words = nullptr;
  CK(cudaMallocAsync((void**)&d_words, sizeof(uint64_t*) * kw, g_stream));
  CK(cudaMemcpyAsync(d_words, key_words, sizeof(uint64_t) * kw, cudaMemcpyHostToDevice, g_stream));
  int rc = run_heads(wgr::EqWords{(const uint64_t* const*)d_words, kw}, n, (uint32_t*)(uintptr_t)starts_out, nruns);
  CK(cudaFreeAsync(d_words, g_stream));
  return rc;
}

// GroupBuilderState.result (builders.py:478-493) for one integer/bool key
// leaf and one value leaf: a stable sort of the appended {key, value} rows
// by key, then run starts -> (sorted unique keys, offsets[K+1], values in
// per-key input order).  Only the key bits that vary are sorted: a stable
// radix sort on the top 32 varying bits, then a stable insertion sort
// inside the (small) buckets; skewed data falls back to a full radix sort.
static bool g_group_u32 = getenv("WELDGPU_GROUP_U32") == nullptr || getenv("WELDGPU_GROUP_U32")[0] != '0';
static bool g_group_narrow = getenv("WELDGPU_GROUP_NARROW") == nullptr || getenv("WELDGPU_GROUP_NARROW")[0] != '0';
static bool g_group_spec_hist = getenv("WELDGPU_GROUP_SPEC_HIST") == nullptr || getenv("WELDGPU_GROUP_SPEC_HIST")[0] != '0';

int wg_group_finish1(uint64_t keys, int key_kind, uint64_t vals, int val_width, uint64_t n, uint64_t ukeys_out,
                     uint64_t offs_out, uint64_t vals_out, uint64_t* K_out) {
  NEED_INIT();
  if (n > 0xffffffffULL) return fail("wg_group_finish1: more than 2^32 rows");
  if (key_kind > 2) return fail("wg_group_finish1: integer or bool keys only");
  if (n == 0) {
    CK(cudaMemsetAsync((void*)(uintptr_t)offs_out, 0, 8, g_stream));
    *K_out = 0;
    return 0;
  }
  unsigned g = grid_for(n, 256);
  // Order keys (one fused pass with the min/max reduction) and 64-bit
  // values, stably radix-sorted on the top 32 varying bits; rows whose keys
  // share those bits are ordered by the bucket fix-up.
  // (Sorting (32-bit window, row index) pairs halves the bytes per radix pass
  // but the value/key gather afterwards is a random permutation -- 11 ms at
  // 200M rows on B200 vs 4.5 ms saved; carrying the payload through the
  // passes is cheaper.)
  uint64_t *k0, *kA, *kB, *v0, *vA, *vB;
  unsigned long long* mm;
  int* flag;
  const bool own_v0 = val_width != 8;
  CK(cudaMallocAsync((void**)&k0, n * 8, g_stream));
  if (own_v0) CK(cudaMallocAsync((void**)&v0, n * 8, g_stream)); else v0 = (uint64_t*)(uintptr_t)vals;
  CK(cudaMallocAsync((void**)&kA, n * 8, g_stream));
  CK(cudaMallocAsync((void**)&kB, n * 8, g_stream));
  CK(cudaMallocAsync((void**)&vB, n * 8, g_stream));
  // the last radix pass writes the values straight into vals_out when they are 8 bytes wide
  if (own_v0) CK(cudaMallocAsync((void**)&vA, n * 8, g_stream)); else vA = (uint64_t*)(uintptr_t)vals_out;
  CK(cudaMallocAsync((void**)&mm, 48 + 4 * 256 * 4, g_stream));
  flag = (int*)(mm + 2);
  uint32_t* spec = g_group_spec_hist && key_kind == 2 ? (uint32_t*)(mm + 6) : nullptr;
  uint64_t init[6] = {~0ULL, 0ULL, 0ULL, 0ULL, ~0ULL, 0ULL};
  CK(cudaMemcpyAsync(mm, init, 48, cudaMemcpyHostToDevice, g_stream));
  if (spec) CK(cudaMemsetAsync(spec, 0, 4 * 256 * 4, g_stream));
  const bool try_narrow = !own_v0 && g_group_narrow;
  { WG_PROF("k_okey_minmax"); k_okey_minmax<<<g, 256, 0, g_stream>>>((const void*)(uintptr_t)keys, key_kind, n, mm, k0,
                                                                   try_narrow ? v0 : nullptr, spec); }
  if (own_v0) { WG_PROF("k_widen"); k_widen<<<g, 256, 0, g_stream>>>((const void*)(uintptr_t)vals, v0, val_width, n); }
  unsigned long long hmm[6];
  CK(cudaMemcpyAsync(hmm, mm, 48, cudaMemcpyDeviceToHost, g_stream));
  CK(cudaStreamSynchronize(g_stream));
  // values narrow to u32 offsets when their flipped bits span < 2^32
  const bool narrow = try_narrow && hmm[5] - hmm[4] <= 0xffffffffULL;
  const uint64_t vbase = hmm[4];
  const uint64_t diff = hmm[0] ^ hmm[1], span = hmm[1] - hmm[0];
  int vbits = diff ? 64 - __builtin_clzll(diff) : 1;   // bits above vbits are equal in every key
  const int rbits = span ? 64 - __builtin_clzll(span) : 1;
  uint64_t kbase = 0;
  if (rbits + 8 <= vbits) {
    // a narrow range straddling a high bit (e.g. keys around 0): sort
    // (okey - min) -- one extra pass, several radix passes saved
    { WG_PROF("k_sub_min"); k_sub_min<<<g, 256, 0, g_stream>>>(k0, n, hmm[0]); }
    kbase = hmm[0];
    vbits = rbits;
  }
  const int begin_bit = vbits > 32 ? vbits - 32 : 0;
  uint32_t* starts;
  CK(cudaMallocAsync((void**)&starts, n * 4, g_stream));
  uint64_t hK = 0;
  if (begin_bit == 0 && g_group_u32) {
    // every key's varying bits fit in 32: sort (u32 key, u64 value) pairs --
    // 12 instead of 16 bytes per row per radix pass -- and rebuild the keys
    // from the common high bits
    const uint64_t lowmask = vbits >= 64 ? ~0ULL : ((1ULL << vbits) - 1);
    const uint64_t sub = kbase ? 0ULL : (hmm[0] & ~lowmask);   // k0 already holds okey - kbase when kbase != 0
    const uint64_t recon = kbase ? kbase : sub;
    uint32_t* w0 = (uint32_t*)kB;
    uint32_t* wA = (uint32_t*)kA;
    uint32_t* wB = w0 + n;                                      // kB holds w0 and wB (2 x 4n bytes)
    { WG_PROF("k_key_u32"); k_key_u32<<<g, 256, 0, g_stream>>>(k0, n, sub, w0); }
    if (narrow && vbits > 8) {
      if (radix_sort_narrow<uint32_t>(w0, v0, wA, wB, vA, (uint32_t*)vB, (uint32_t*)vB + n, n, 0, vbits, vbase)) return -1;
    } else if (radix_sort<uint32_t, uint64_t>(w0, v0, wA, wB, vA, vB, n, 0, vbits)) return -1;
    if (run_heads(wgr::EqU32{wA}, n, starts, &hK)) return -1;
    { WG_PROF("k_group_out"); k_group_out<uint32_t><<<grid_for(hK + 1, 256), 256, 0, g_stream>>>(
        starts, hK, n, wA, recon, key_kind, (int64_t*)(uintptr_t)offs_out, (void*)(uintptr_t)ukeys_out); }
  } else {
    g_pre_hist = (spec && kbase == 0) ? spec : nullptr;   // the window is bits 32..63 exactly when vbits == 64
    int rc_;
    if (narrow && vbits - begin_bit > 8)
      rc_ = radix_sort_narrow<uint64_t>(k0, v0, kA, kB, vA, (uint32_t*)vB, (uint32_t*)vB + n, n, begin_bit, vbits, vbase);
    else
      rc_ = radix_sort<uint64_t, uint64_t>(k0, v0, kA, kB, vA, vB, n, begin_bit, vbits);
    g_pre_hist = nullptr;
    if (rc_) return -1;
    if (begin_bit > 0) {
      uint64_t cap = n / 8 + 1024;
      uint32_t* pos = starts;             // scratch until the run starts are computed
      unsigned long long* npos = mm + 3;
      CK(cudaMemsetAsync(npos, 0, 8, g_stream));
      CK(cudaMemsetAsync(flag, 0, 4, g_stream));
      { WG_PROF("k_disorder"); k_disorder<<<g, 256, 0, g_stream>>>(kA, n, begin_bit, pos, npos, cap); }
      unsigned long long hn = 0;
      CK(cudaMemcpyAsync(&hn, npos, 8, cudaMemcpyDeviceToHost, g_stream));
      CK(cudaStreamSynchronize(g_stream));
      int hflag = hn > cap;
      if (!hflag && hn) {
        unsigned* claimed;
        CK(cudaMallocAsync((void**)&claimed, (n / 32 + 1) * 4, g_stream));
        CK(cudaMemsetAsync(claimed, 0, (n / 32 + 1) * 4, g_stream));
        { WG_PROF("k_fix_buckets"); k_fix_buckets<<<grid_for(hn, 128), 128, 0, g_stream>>>(kA, vA, n, begin_bit, pos, hn, 512,
                                                                                             flag, claimed); }
        CK(cudaFreeAsync(claimed, g_stream));
        CK(cudaMemcpyAsync(&hflag, flag, 4, cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
      }
      if (hflag) {
        // skewed buckets: a full stable sort of every varying bit (sorting
        // only the low bits now would undo the order of the high ones; ties
        // keep the current -- input -- order of each key's rows)
        uint64_t *kt, *vt;
        CK(cudaMallocAsync((void**)&kt, n * 8, g_stream));
        CK(cudaMallocAsync((void**)&vt, n * 8, g_stream));
        CK(cudaMemcpyAsync(kt, kA, n * 8, cudaMemcpyDeviceToDevice, g_stream));
        CK(cudaMemcpyAsync(vt, vA, n * 8, cudaMemcpyDeviceToDevice, g_stream));
        if (radix_sort<uint64_t, uint64_t>(kt, vt, kA, kB, vA, vB, n, 0, vbits)) return -1;
        CK(cudaFreeAsync(kt, g_stream));
        CK(cudaFreeAsync(vt, g_stream));
      }
    }
    if (run_heads(wgr::EqU64{kA}, n, starts, &hK)) return -1;
    { WG_PROF("k_group_out"); k_group_out<uint64_t><<<grid_for(hK + 1, 256), 256, 0, g_stream>>>(
        starts, hK, n, kA, kbase, key_kind, (int64_t*)(uintptr_t)offs_out, (void*)(uintptr_t)ukeys_out); }
  }
  if (own_v0) { WG_PROF("k_narrow"); k_narrow<<<g, 256, 0, g_stream>>>(vA, (void*)(uintptr_t)vals_out, val_width, n); }
  CK(cudaGetLastError());
  CK(cudaFreeAsync(starts, g_stream));
  CK(cudaFreeAsync(mm, g_stream));
  CK(cudaFreeAsync(k0, g_stream));
  if (own_v0) { CK(cudaFreeAsync(v0, g_stream)); CK(cudaFreeAsync(vA, g_stream)); }
  CK(cudaFreeAsync(kA, g_stream));
  CK(cudaFreeAsync(kB, g_stream));
  CK(cudaFreeAsync(vB, g_stream));
  *K_out = hK;
  return 0;
}

// ---- synthetic data + measurement helpers ----------------------------------
int wg_gen_column(uint64_t dst, uint64_t n, uint64_t row0, int dist, int width, uint64_t seed, uint64_t col,
                  int64_t lo, uint64_t span, double flo, double fhi, double div, int ncat, const double* cum,
                  const int64_t* vals) {
  NEED_INIT();
  if (!n) return 0;
  GenSpec g;
  memset(&g, 0, sizeof(g));
  g.dist = dist; g.width = width; g.seed = seed; g.col = col; g.lo = lo; g.span = span ? span : 1;
  g.flo = flo; g.fhi = fhi; g.div = div; g.ncat = ncat;
  if (ncat > 8) return fail("wg_gen_column: at most 8 categories");
  for (int c = 0; c < ncat; ++c) { g.cum[c] = cum[c]; g.vals[c] = vals[c]; }
  { WG_PROF("k_gen"); k_gen<<<grid_for(n, 256), 256, 0, g_stream>>>((void*)(uintptr_t)dst, n, row0, g); }
  CK(cudaGetLastError());
  return 0;
}

int wg_mul_inplace_f64(uint64_t a, uint64_t b, uint64_t n) {
  NEED_INIT();
  if (!n) return 0;
  { WG_PROF("k_mul_inplace"); k_mul_inplace<<<grid_for(n, 256), 256, 0, g_stream>>>((double*)(uintptr_t)a, (const double*)(uintptr_t)b, n); }
  CK(cudaGetLastError());
  return 0;
}

int wg_flush_l2(uint64_t buf, uint64_t bytes, uint32_t salt) {
  NEED_INIT();
  uint64_t n16 = bytes / 16;
  { WG_PROF("k_flush"); k_flush<<<grid_for(n16, 512), 512, 0, g_stream>>>((uint4*)(uintptr_t)buf, n16, salt); }
  CK(cudaGetLastError());
  return 0;
}

int wg_event_create(uint64_t* ev) {
  NEED_INIT();
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  *ev = (uint64_t)(uintptr_t)e;
  return 0;
}

int wg_event_record(uint64_t ev) {
  NEED_INIT();
  CK(cudaEventRecord((cudaEvent_t)(uintptr_t)ev, g_stream));
  return 0;
}

int wg_event_elapsed_ms(uint64_t start, uint64_t stop, float* ms) {
  NEED_INIT();
  CK(cudaEventSynchronize((cudaEvent_t)(uintptr_t)stop));
  CK(cudaEventElapsedTime(ms, (cudaEvent_t)(uintptr_t)start, (cudaEvent_t)(uintptr_t)stop));
  return 0;
}

// Copy/compute overlap for host-resident inputs: select which of the three
// streams subsequent calls enqueue on, and order streams with events.
// (Buffers handed between streams must stay alive until the consumer's
// event; the caching allocator is only stream-ordered on stream 0.)
int wg_stream_select(int which) {
  NEED_INIT();
  if (which < 0 || which > 2) return fail("wg_stream_select: stream 0, 1 or 2");
  g_stream = g_streams[which];
  if (which != 0) {
    std::lock_guard<std::mutex> lk(g_acct_mu);
    g_multi = true;
  }
  return 0;
}

int wg_stream_wait_event(uint64_t ev) {
  NEED_INIT();
  CK(cudaStreamWaitEvent(g_stream, (cudaEvent_t)(uintptr_t)ev, 0));
  return 0;
}

int wg_sync_all(void) {
  NEED_INIT();
  for (int i = 0; i < 3; ++i) CK(cudaStreamSynchronize(g_streams[i]));
  {
    std::lock_guard<std::mutex> lk(g_acct_mu);
    if (g_stream == g_streams[0]) g_multi = false;
    release_deferred();
  }
  return 0;
}

// ---- per-launch timing ---------------------------------------------------------
int wg_prof_enable(int on) {
  NEED_INIT();
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (on) {
    for (auto& r : g_prof) { g_prof_free.push_back(r.a); g_prof_free.push_back(r.b); }
    g_prof.clear();
  }
  g_prof_on = on != 0;
  return 0;
}

int wg_prof_count(int* n) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  *n = (int)g_prof.size();
  return 0;
}

int wg_prof_record(int i, char* name, int cap, float* ms) {
  NEED_INIT();
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (i < 0 || i >= (int)g_prof.size()) return fail("wg_prof_record: index out of range");
  const ProfRec& r = g_prof[i];
  CK(cudaEventSynchronize(r.b));
  CK(cudaEventElapsedTime(ms, r.a, r.b));
  if (name && cap > 0) {
    strncpy(name, r.name, cap - 1);
    name[cap - 1] = 0;
  }
  return 0;
}

int wg_event_destroy(uint64_t ev) {
  NEED_INIT();
  CK(cudaEventDestroy((cudaEvent_t)(uintptr_t)ev));
  return 0;
}


// ---- multi-GPU: row partitioning + NCCL (libnccl.so.2, dlopen'ed) ---------
// The combine step of row-partitioned evaluation.  The
// reference folds its per-chunk partials at result()
// (builders.py:314-328, 380-392, 435-450, 478-493); across GPUs the partials
// are exchanged with these collectives on the library's stream.
int wg_partition(uint64_t key_col, int key_kind, const uint64_t* splitters, int nsplit, int ncols,
                 const uint64_t* cols_in, const uint64_t* cols_out, const int* widths, uint64_t n,
                 uint64_t* counts_out) {
  NEED_INIT();
  if (nsplit + 1 > WG_PART_MAX) return fail("wg_partition: at most 64 destinations");
  if (ncols > 16) return fail("wg_partition: at most 16 columns");
  if (n > 0xffffffffULL) return fail("wg_partition: more than 2^32 rows");
  const int G = nsplit + 1;
  if (n == 0) { for (int d = 0; d < G; ++d) counts_out[d] = 0; return 0; }
  PartSpec p;
  memset(&p, 0, sizeof(p));
  p.G = G; p.nsplit = nsplit; p.ncols = ncols; p.kind = key_kind;
  p.key = (const void*)(uintptr_t)key_col;
  for (int i = 0; i < nsplit; ++i) p.split[i] = splitters[i];
  for (int c = 0; c < ncols; ++c) {
    p.in[c] = (const void*)(uintptr_t)cols_in[c];
    p.out[c] = (void*)(uintptr_t)cols_out[c];
    p.width[c] = widths[c];
    if (widths[c] != 1 && widths[c] != 4 && widths[c] != 8) return fail("wg_partition: column width must be 1, 4 or 8");
  }
  const uint32_t ntiles = (uint32_t)((n + 4095) / 4096);
  uint32_t* cnt;
  uint64_t* tot;
  CK(cudaMallocAsync((void**)&cnt, (uint64_t)G * ntiles * 4, g_stream));
  CK(cudaMallocAsync((void**)&tot, G * 8, g_stream));
  { WG_PROF("k_part_count"); k_part_count<<<ntiles, 256, 0, g_stream>>>(p, n, cnt, ntiles); }
  { WG_PROF("k_part_scan"); k_part_scan<<<G, 1024, 0, g_stream>>>(cnt, ntiles, tot); }
  { WG_PROF("k_part_scatter"); k_part_scatter<<<ntiles, 256, 0, g_stream>>>(p, n, cnt, ntiles, tot); }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(counts_out, tot, G * 8, cudaMemcpyDeviceToHost, g_stream));
  CK(cudaStreamSynchronize(g_stream));
  CK(cudaFreeAsync(cnt, g_stream));
  CK(cudaFreeAsync(tot, g_stream));
  return 0;
}

}  // extern "C"

namespace {
struct Nccl {
  void* h = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
} g_nccl;

int nccl_load() {
  if (g_nccl.h) return 0;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(std::string("wg_nccl: cannot load libnccl.so.2: ") + dlerror());
#define WG_NSYM(f)                                                              \
  g_nccl.f = reinterpret_cast<decltype(g_nccl.f)>(dlsym(h, "nccl" #f));          \
  if (!g_nccl.f) return fail("wg_nccl: libnccl.so.2 lacks nccl" #f);
  WG_NSYM(GetUniqueId) WG_NSYM(CommInitRank) WG_NSYM(CommDestroy) WG_NSYM(AllGather) WG_NSYM(AllReduce)
  WG_NSYM(Send) WG_NSYM(Recv) WG_NSYM(GroupStart) WG_NSYM(GroupEnd) WG_NSYM(GetErrorString)
#undef WG_NSYM
  g_nccl.h = h;
  return 0;
}
}  // namespace

#define CKNC(x)                                                                        \
  do {                                                                                 \
    ncclResult_t r_ = (x);                                                             \
    if (r_ != ncclSuccess) return fail(std::string(#x) + ": " + g_nccl.GetErrorString(r_)); \
  } while (0)
#define NEED_NCCL() \
  do { if (!g_nccl.comm) return fail("wg_nccl: wg_nccl_init() has not been called"); } while (0)

extern "C" {

int wg_nccl_unique_id(char* out, int cap) {
  if (cap < (int)sizeof(ncclUniqueId)) return fail("wg_nccl_unique_id: buffer smaller than 128 bytes");
  if (nccl_load()) return -1;
  ncclUniqueId id;
  CKNC(g_nccl.GetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return 0;
}

int wg_nccl_init(int rank, int world, const char* id_bytes) {
  NEED_INIT();
  if (nccl_load()) return -1;
  if (g_nccl.comm) return fail("wg_nccl_init: already initialised");
  ncclUniqueId id;
  memcpy(&id, id_bytes, sizeof(id));
  CKNC(g_nccl.CommInitRank(&g_nccl.comm, world, id, rank));
  g_nccl.rank = rank;
  g_nccl.world = world;
  return 0;
}

int wg_nccl_finalize(void) {
  if (!g_nccl.comm) return 0;
  CK(cudaStreamSynchronize(g_stream));
  CKNC(g_nccl.CommDestroy(g_nccl.comm));
  g_nccl.comm = nullptr;
  return 0;
}

int wg_nccl_allgather(uint64_t send, uint64_t recv, uint64_t bytes) {
  NEED_INIT(); NEED_NCCL();
  WG_PROF("ncclAllGather");
  CKNC(g_nccl.AllGather((const void*)(uintptr_t)send, (void*)(uintptr_t)recv, bytes, ncclUint8, g_nccl.comm, g_stream));
  return 0;
}

// kind: KIND_CODE (1 i32, 2 i64, 3 f32, 4 f64); op: 0 sum 1 prod 2 min 3 max
int wg_nccl_allreduce(uint64_t send, uint64_t recv, uint64_t count, int kind, int op) {
  NEED_INIT(); NEED_NCCL();
  ncclDataType_t t;
  switch (kind) {
    case 1: t = ncclInt32; break;
    case 2: t = ncclInt64; break;
    case 3: t = ncclFloat32; break;
    case 4: t = ncclFloat64; break;
    default: return fail("wg_nccl_allreduce: unsupported kind");
  }
  const ncclRedOp_t ops[4] = {ncclSum, ncclProd, ncclMin, ncclMax};
  if (op < 0 || op > 3) return fail("wg_nccl_allreduce: unsupported op");
  WG_PROF("ncclAllReduce");
  CKNC(g_nccl.AllReduce((const void*)(uintptr_t)send, (void*)(uintptr_t)recv, count, t, ops[op], g_nccl.comm, g_stream));
  return 0;
}

// Grouped point-to-point: an all-to-all-v of one or more columns is one
// group of sends and receives (NCCL has no alltoallv).
int wg_nccl_sendrecv(int nsend, const uint64_t* send_ptr, const uint64_t* send_bytes, const int* send_peer,
                     int nrecv, const uint64_t* recv_ptr, const uint64_t* recv_bytes, const int* recv_peer) {
  NEED_INIT(); NEED_NCCL();
  WG_PROF("ncclSendRecv");
  CKNC(g_nccl.GroupStart());
  for (int i = 0; i < nsend; ++i)
    if (send_bytes[i]) CKNC(g_nccl.Send((const void*)(uintptr_t)send_ptr[i], send_bytes[i], ncclUint8, send_peer[i], g_nccl.comm, g_stream));
  for (int i = 0; i < nrecv; ++i)
    if (recv_bytes[i]) CKNC(g_nccl.Recv((void*)(uintptr_t)recv_ptr[i], recv_bytes[i], ncclUint8, recv_peer[i], g_nccl.comm, g_stream));
  CKNC(g_nccl.GroupEnd());
  return 0;
}

}  // extern "C"

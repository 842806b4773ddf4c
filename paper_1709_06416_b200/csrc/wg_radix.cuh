// wg_radix.cuh -- hand-written sm_100a sorting and run-compaction kernels for
// the keyed builders' result() (included by weldgpu.cu).
//
//   * onesweep stable LSD radix sort of (key, value) pairs, 8-bit digits:
//       GroupBuilderState.result   builders.py:478-493  (stable by key)
//       DictMergerState.result     builders.py:380-392  (sorted by order_key)
//       order_key                  builders.py:496-507
//       ToVec / Sort               run.py:723-747
//     One upfront histogram pass counts every digit of every pass; then each
//     pass is ONE kernel: a CTA claims a tile (atomic counter, so every
//     predecessor is already resident), ranks its keys with warp-level
//     ballot multisplit (stable: rows are ranked in input order), publishes
//     its per-digit counts and resolves its per-digit global offsets by a
//     decoupled look-back over the predecessor tiles (one thread per digit),
//     then scatters keys and values through shared memory so consecutive
//     threads write consecutive addresses of each digit's run.
//   * single-pass run-head compaction (sorted keys -> run start positions),
//     the "unique keys" step of the same result() functions.
//
// Status words of both look-backs: [63:62] flag (0 = not ready, 1 = tile
// aggregate, 2 = inclusive prefix), [61:0] count.
#pragma once

namespace wgr {


constexpr int RADIX = 256;
constexpr unsigned long long ST_AGG = 1ULL << 62;
constexpr unsigned long long ST_INC = 2ULL << 62;
constexpr unsigned long long ST_CNT = (1ULL << 62) - 1;

__device__ __forceinline__ unsigned long long ld_vol(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_vol(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift, uint32_t mask) {
  return (uint32_t)(k >> shift) & mask;
}

// Counts of every digit of every pass: hist[p * 256 + d], passes of 8 bits
// starting at begin_bit (the last pass may be narrower, up to end_bit).
template <typename K>
__global__ void __launch_bounds__(256) k_radix_hist(const K* __restrict__ keys, uint64_t n, int begin_bit, int end_bit,
                                                    int npass, uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[8][RADIX];
  for (int i = threadIdx.x; i < 8 * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  int shifts[8];
  uint32_t masks[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    shifts[p] = begin_bit + 8 * p;
    const int w = min(8, end_bit - shifts[p]);
    masks[p] = w > 0 ? ((1u << w) - 1u) : 0u;
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const K k = keys[i];
#pragma unroll
    for (int p = 0; p < 8; ++p)
      if (p < npass) atomicAdd(&sh[p][digit_of(k, shifts[p], masks[p])], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * RADIX; i += blockDim.x) {
    const uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// Exclusive scan of each pass's 256 digit counts (one CTA per pass), in place.
__global__ void __launch_bounds__(RADIX) k_radix_offsets(uint32_t* hist) {
  __shared__ uint32_t warp_tot[RADIX / 32];
  uint32_t* h = hist + blockIdx.x * RADIX;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t c = h[t];
  uint32_t x = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  uint32_t base = 0;
  for (int j = 0; j < w; ++j) base += warp_tot[j];
  h[t] = base + x - c;
}

// One onesweep pass over a tile of TILE = BLOCK * ITEMS rows (BLOCK = 512:
// 16 warps; threads 0..255 own one digit each for the scans and the
// look-back).  Rows of a warp are ITEMS rounds of 32 consecutive rows,
// ranked round by round with match_any -> stable.  Keys and values are both
// loaded before the ranking (their loads overlap it), staged in shared
// memory at their tile rank, and written out together: consecutive threads
// write consecutive addresses of each digit's run.
// Dynamic shared memory: onesweep_smem<K, V, ITEMS>().
template <typename K, typename V, int ITEMS>
constexpr int onesweep_smem() {
  return 512 * ITEMS * (int)(sizeof(K) + sizeof(V)) + (512 / 32) * RADIX * 2;
}

// Payload conversions of a pass (value in -> staged -> value out).  Narrowed
// payloads: 8-byte values whose order-flipped bits (v ^ 2^63) span less than
// 2^32 travel the middle passes as u32 offsets from their minimum.
struct VCopy {
  template <typename T> __device__ static T in(T v, uint64_t) { return v; }
  template <typename T> __device__ static T out(T v, uint64_t) { return v; }
};
struct VNarrow {   // first pass: u64 in, u32 staged and out
  __device__ static uint32_t in(uint64_t v, uint64_t base) { return (uint32_t)((v ^ (1ULL << 63)) - base); }
  __device__ static uint32_t out(uint32_t v, uint64_t) { return v; }
};
struct VWiden {    // last pass: u32 in and staged, u64 out
  __device__ static uint32_t in(uint32_t v, uint64_t) { return v; }
  __device__ static uint64_t out(uint32_t v, uint64_t base) { return ((uint64_t)v + base) ^ (1ULL << 63); }
};

template <typename K, typename VI, typename VS, typename VO, typename CV, int ITEMS>
__global__ void __launch_bounds__(512, 2)
k_onesweep(const K* __restrict__ kin, const VI* __restrict__ vin, K* __restrict__ kout, VO* __restrict__ vout,
           uint32_t n, int shift, uint32_t dmask, const uint32_t* __restrict__ gofs, unsigned long long* status,
           uint32_t* tile_ctr, uint64_t vbase) {
  using V = VS;
  constexpr int BLOCK = 512, WARPS = BLOCK / 32, TILE = BLOCK * ITEMS;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  K* s_k = reinterpret_cast<K*>(s_dyn);
  V* s_v = reinterpret_cast<V*>(s_dyn + TILE * sizeof(K));
  uint16_t (*s_wh)[RADIX] = reinterpret_cast<uint16_t (*)[RADIX]>(s_dyn + TILE * (sizeof(K) + sizeof(V)));
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_dbase[RADIX];       // global position of the digit's run minus its tile-local start
  __shared__ uint32_t s_wtot[RADIX / 32];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = tid; i < WARPS * RADIX / 2; i += BLOCK) reinterpret_cast<uint32_t*>(&s_wh[0][0])[i] = 0u;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * (uint32_t)TILE;
  const uint32_t wbase = base + (uint32_t)w * (32 * ITEMS);

  K k[ITEMS];
  V v[ITEMS];
  uint32_t dr[ITEMS];   // digit << 16 | rank (digit RADIX = row past the end)
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t row = wbase + i * 32 + lane;
    const bool ok = row < n;
    k[i] = ok ? kin[row] : (K)0;
    v[i] = ok ? CV::in(vin[row], vbase) : (V)0;
  }
  const unsigned lt = lanemask_lt();
  // peer masks of every round first (independent, pipelined), then the
  // per-warp counter updates in round order (stable ranks)
  unsigned peers[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t row = wbase + i * 32 + lane;
    const uint32_t d = row < n ? digit_of(k[i], shift, dmask) : (uint32_t)RADIX;
    {
      // peers = lanes with the same digit: one ballot per digit bit (bit 8
      // marks rows past the end).  Measured faster than __match_any_sync on
      // B200 (sort_ab: 8.41 vs 9.47 ms for 4 passes over 200M pairs).
      unsigned pm = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 9; ++b) {
        const bool bit = (d >> b) & 1u;
        const unsigned bm = __ballot_sync(0xffffffffu, bit);
        pm &= bit ? bm : ~bm;
      }
      peers[i] = pm;
    }
    dr[i] = d << 16;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t d = dr[i] >> 16;
    const uint32_t below = __popc(peers[i] & lt);
    const uint32_t prev = d < RADIX ? s_wh[w][d] : 0u;
    __syncwarp();
    if (d < RADIX && below == 0) s_wh[w][d] = (uint16_t)(prev + __popc(peers[i]));
    __syncwarp();
    dr[i] |= prev + below;
  }
  __syncthreads();

  uint32_t excl = 0;
  if (tid < RADIX) {
    // digit tid: counts over the warps (-> exclusive per-warp offsets), tile total
    uint32_t tot = 0;
#pragma unroll
    for (int j = 0; j < WARPS; ++j) {
      const uint32_t c = s_wh[j][tid];
      s_wh[j][tid] = (uint16_t)tot;
      tot += c;
    }
    unsigned long long* my = status + (uint64_t)tile * RADIX + tid;
    if (tile == 0) st_vol(my, ST_INC | tot);
    else st_vol(my, ST_AGG | tot);
    // tile-local start of each digit's run: exclusive scan of tot over digits
    uint32_t x = tot;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, s);
      if (lane >= s) x += y;
    }
    if (lane == 31) s_wtot[w] = x;
    if (tile > 0) {
      // look back 4 predecessors per round trip
      const unsigned long long* p = my - RADIX;
      int64_t j = (int64_t)tile - 1;
      uint64_t acc = 0;
      while (true) {
        unsigned long long sv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) sv[q] = (j - q >= 0) ? ld_vol(p - q * RADIX) : ST_INC;
        int adv = 0;
        bool done = false;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (done || adv < q) continue;
          const unsigned long long f = sv[q] & ~ST_CNT;
          if (f == 0) continue;              // not published yet: retry from here
          acc += sv[q] & ST_CNT;
          adv = q + 1;
          done = f == ST_INC;
        }
        if (done) break;
        p -= adv * RADIX;
        j -= adv;
      }
      st_vol(my, ST_INC | (acc + tot));
      excl = (uint32_t)acc;
    }
    s_dbase[tid] = x - tot;   // inclusive-exclusive within the warp; completed below
  }
  __syncthreads();
  if (tid < RADIX) {
    uint32_t lstart = s_dbase[tid];
    for (int j = 0; j < w; ++j) lstart += s_wtot[j];
    s_dbase[tid] = gofs[tid] + excl - lstart;
#pragma unroll
    for (int j = 0; j < WARPS; ++j) s_wh[j][tid] = (uint16_t)(s_wh[j][tid] + lstart);
  }
  __syncthreads();

  // keys and values -> shared memory in tile order (by digit, stable)
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t d = dr[i] >> 16;
    if (d < RADIX) {
      const uint32_t r = (dr[i] & 0xffffu) + s_wh[w][d];
      s_k[r] = k[i];
      s_v[r] = v[i];
    }
  }
  __syncthreads();
  const uint32_t nvalid = (n - base) < (uint32_t)TILE ? (n - base) : (uint32_t)TILE;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t idx = i * BLOCK + tid;
    if (idx < nvalid) {
      const K kk = s_k[idx];
      const uint32_t dst = s_dbase[digit_of(kk, shift, dmask)] + idx;
      kout[dst] = kk;
      vout[dst] = CV::out(s_v[idx], vbase);
    }
  }
}

// Run heads of sorted keys -> starts[] (u32 positions, ascending), count.
// One pass: per-tile head counts, a block scan and a decoupled look-back
// over tiles (one warp), then ordered writes.  eq(i) says row i continues
// the run of row i-1.
struct EqU64 {
  const uint64_t* k;
  __device__ bool operator()(uint64_t i) const { return k[i] == k[i - 1]; }
};
struct EqU32 {
  const uint32_t* k;
  __device__ bool operator()(uint64_t i) const { return k[i] == k[i - 1]; }
};
struct EqWords {
  const uint64_t* const* w;
  int kw;
  __device__ bool operator()(uint64_t i) const {
    for (int j = 0; j < kw; ++j)
      if (w[j][i] != w[j][i - 1]) return false;
    return true;
  }
};

template <typename EQ, int ITEMS>
__global__ void __launch_bounds__(256) k_run_heads(EQ eq, uint64_t n, uint32_t* __restrict__ starts,
                                                   unsigned long long* status, uint32_t* tile_ctr,
                                                   unsigned long long* total) {
  constexpr int BLOCK = 256, WARPS = BLOCK / 32, TILE = BLOCK * ITEMS;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_w[WARPS];
  __shared__ unsigned long long s_excl;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  // warp w: ITEMS rounds of 32 consecutive rows (coalesced loads)
  const uint64_t wrow = tile * TILE + (uint64_t)w * (32 * ITEMS) + lane;
  unsigned m[ITEMS];
  uint32_t cnt = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t r = wrow + i * 32;
    const bool h = r < n && (r == 0 || !eq(r));
    m[i] = __ballot_sync(0xffffffffu, h);
    cnt += __popc(m[i]);
  }
  if (lane == 0) s_w[w] = cnt;
  __syncthreads();
  uint32_t before = 0, agg = 0;
#pragma unroll
  for (int j = 0; j < WARPS; ++j) {
    if (j < w) before += s_w[j];
    agg += s_w[j];
  }
  if (w == 0) {
    unsigned long long excl = 0;
    unsigned long long* my = status + tile;
    if (tile == 0) {
      if (lane == 0) st_vol(my, ST_INC | agg);
    } else {
      if (lane == 0) st_vol(my, ST_AGG | agg);
      int64_t t = (int64_t)tile - 1;
      while (true) {
        const int64_t idx = t - lane;
        const unsigned long long sv = idx >= 0 ? ld_vol(status + idx) : ST_INC;
        const unsigned long long f = sv & ~ST_CNT;
        const unsigned inc = __ballot_sync(0xffffffffu, f == ST_INC);
        const int first = inc ? __ffs(inc) - 1 : 32;
        const unsigned nr = __ballot_sync(0xffffffffu, f == 0 && lane < first);
        if (nr) continue;
        unsigned long long x = lane <= first ? (sv & ST_CNT) : 0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
        excl += x;
        if (inc) break;
        t -= 32;
      }
      if (lane == 0) st_vol(my, ST_INC | (excl + agg));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  uint64_t o = s_excl + before;
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (m[i] >> lane & 1u) starts[o + __popc(m[i] & lt)] = (uint32_t)(wrow + i * 32);
    o += __popc(m[i]);
  }
  if (tile == (n + TILE - 1) / TILE - 1 && tid == 0) *total = s_excl + agg;
}

}  // namespace wgr

// weld_device.cuh -- device-side building blocks for NVRTC-generated loop kernels.
//
// Every generated kernel (paper_1709_06416_b200/codegen.py) is this header plus
// one fused loop body.  The header carries:
//   * the reference's exact scalar semantics (wrapping ints, truncating
//     division with a DivideByZero error word, NaN-aware min/max, wrapping
//     float->int casts, per-op f32 rounding via -fmad=false);
//   * merge folds and their *internal* identities (see wg_ident_*);
//   * block reductions for merger partials, the single-pass decoupled
//     look-back tile scan for order-preserving appenders, and the
//     open-addressing hash table for dictmerger.
//
// Reference semantics cited against /root/reference/pkg/src/weldmill:
//   ints wrap              engine/run.py:395-437
//   float ops              engine/run.py:440-464
//   casts                  engine/run.py:503-528
//   merge folds            engine/builders.py:121-174
//   identities             types.py:185-192
// This file is compiled at run time by NVRTC for sm_100a (no host code here).
#pragma once

typedef long long i64;
typedef unsigned long long u64;
typedef int i32;
typedef unsigned int u32;
typedef unsigned char u8;

#define WG_INF __longlong_as_double(0x7ff0000000000000LL)
#define WG_NAN __longlong_as_double(0x7ff8000000000000LL)
#define WG_INFF __int_as_float(0x7f800000)
#define WG_NANF __int_as_float(0x7fc00000)

// ---------------------------------------------------------------------------
// Error word: first writer wins.  Layout {i64 code, i64 info}.
enum {
  WG_OK = 0,
  WG_ERR_DIVZERO = 1,       // DivideByZero        run.py:411-425
  WG_ERR_LOOKUP_OOB = 2,    // IndexOutOfBounds    run.py:693-700
  WG_ERR_VECMERGER_OOB = 3, // IndexOutOfBounds    builders.py:413-417
  WG_ERR_KEY_NOT_FOUND = 4, // KeyNotFound         run.py:704-710
  WG_ERR_INTERNAL = 5,
  WG_ERR_REMZERO = 6,       // DivideByZero (remainder)
  WG_ERR_ITER_LIMIT = 7,    // IterationLimit      run.py:680-684
  WG_ERR_EXTERN = 8,        // EvalError("extern ... failed: math domain/range error")  run.py:841-844
  WG_ERR_ZIP = 9,           // ZipLengthMismatch   run.py:935-940 (nested loops)
  WG_ERR_STRIDE = 10,       // EvalError (stride < 1)  run.py:921-924 (nested loops)
};

__device__ __forceinline__ void wg_raise(i64* err, i64 code, i64 info) {
  if (atomicCAS((u64*)err, 0ULL, (u64)code) == 0ULL) {
    ((volatile i64*)err)[1] = info;
  }
}

// count_evals (run.py:544-557): one node evaluation per active lane.  All
// lanes reaching this statement bump the same counter, so the warp's active
// lanes are counted with one atomic by the lowest of them.
__device__ __forceinline__ void wg_count(unsigned long long* c) {
  const unsigned m = __activemask();
  if ((threadIdx.x & 31) == (unsigned)(__ffs(m) - 1)) atomicAdd(c, (unsigned long long)__popc(m));
}

// ---------------------------------------------------------------------------
// Integer arithmetic: wraps at the width (computed unsigned, no UB).
__device__ __forceinline__ i64 wg_add_i64(i64 a, i64 b) { return (i64)((u64)a + (u64)b); }
__device__ __forceinline__ i64 wg_sub_i64(i64 a, i64 b) { return (i64)((u64)a - (u64)b); }
__device__ __forceinline__ i64 wg_mul_i64(i64 a, i64 b) { return (i64)((u64)a * (u64)b); }
__device__ __forceinline__ i64 wg_neg_i64(i64 a) { return (i64)(0ULL - (u64)a); }
__device__ __forceinline__ i32 wg_add_i32(i32 a, i32 b) { return (i32)((u32)a + (u32)b); }
__device__ __forceinline__ i32 wg_sub_i32(i32 a, i32 b) { return (i32)((u32)a - (u32)b); }
__device__ __forceinline__ i32 wg_mul_i32(i32 a, i32 b) { return (i32)((u32)a * (u32)b); }
__device__ __forceinline__ i32 wg_neg_i32(i32 a) { return (i32)(0U - (u32)a); }

// Truncating division / remainder; a zero divisor raises DivideByZero and
// yields 0 (the host raises after the launch).  MIN / -1 wraps like the
// reference's arbitrary-precision quotient followed by wrap().
__device__ __forceinline__ i64 wg_div_i64(i64 a, i64 b, i64* err) {
  if (b == 0) { wg_raise(err, WG_ERR_DIVZERO, 0); return 0; }
  if (b == -1) return wg_neg_i64(a);
  return a / b;
}
__device__ __forceinline__ i64 wg_rem_i64(i64 a, i64 b, i64* err) {
  if (b == 0) { wg_raise(err, WG_ERR_REMZERO, 0); return 0; }
  if (b == -1) return 0;
  return a % b;
}
__device__ __forceinline__ i32 wg_div_i32(i32 a, i32 b, i64* err) {
  if (b == 0) { wg_raise(err, WG_ERR_DIVZERO, 0); return 0; }
  if (b == -1) return wg_neg_i32(a);
  return a / b;
}
__device__ __forceinline__ i32 wg_rem_i32(i32 a, i32 b, i64* err) {
  if (b == 0) { wg_raise(err, WG_ERR_REMZERO, 0); return 0; }
  if (b == -1) return 0;
  return a % b;
}

// ---------------------------------------------------------------------------
// Float semantics.  min prefers a number over NaN; max propagates NaN
// (builders.py:133-152).  -0.0 vs 0.0 follow the reference's `<=`/`>=`.
__device__ __forceinline__ double wg_min_f64(double a, double b) {
  if (a != a) return b;
  if (b != b) return a;
  return a <= b ? a : b;
}
__device__ __forceinline__ double wg_max_f64(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a >= b ? a : b;
}
__device__ __forceinline__ float wg_min_f32(float a, float b) {
  if (a != a) return b;
  if (b != b) return a;
  return a <= b ? a : b;
}
__device__ __forceinline__ float wg_max_f32(float a, float b) {
  if (a != a) return a;
  if (b != b) return b;
  return a >= b ? a : b;
}
// Binary-op min/max on ints: `b if b < a else a` (run.py:435-436).
__device__ __forceinline__ i64 wg_min_i64(i64 a, i64 b) { return b < a ? b : a; }
__device__ __forceinline__ i64 wg_max_i64(i64 a, i64 b) { return b > a ? b : a; }
__device__ __forceinline__ i32 wg_min_i32(i32 a, i32 b) { return b < a ? b : a; }
__device__ __forceinline__ i32 wg_max_i32(i32 a, i32 b) { return b > a ? b : a; }

// Float remainder: NaN for a zero divisor, NaN operands, or infinite a;
// otherwise C fmod (exact, so no f32 re-rounding is needed).
__device__ __forceinline__ double wg_rem_f64(double a, double b) {
  if (b == 0.0 || a != a || b != b || isinf(a)) return WG_NAN;
  return fmod(a, b);
}
__device__ __forceinline__ float wg_rem_f32(float a, float b) {
  if (b == 0.0f || a != a || b != b || isinf(a)) return WG_NANF;
  return (float)fmod((double)a, (double)b);
}

// ---------------------------------------------------------------------------
// Casts (run.py:503-528).  float->int: NaN -> 0, +-inf saturate, finite
// values truncate then wrap modulo 2^width (CUDA's cvt saturates instead).
__device__ __forceinline__ i64 wg_f64_to_i64(double v) {
  if (v != v) return 0;
  if (v == WG_INF) return 0x7fffffffffffffffLL;
  if (v == -WG_INF) return (i64)0x8000000000000000ULL;
  double t = trunc(v);
  if (t >= -9223372036854775808.0 && t < 9223372036854775808.0) return (i64)t;
  // |t| >= 2^63: t is a multiple of 2^11, so fmod and the shift are exact.
  double r = fmod(t, 18446744073709551616.0);
  if (r < 0) r += 18446744073709551616.0;
  return (i64)(u64)r;
}
__device__ __forceinline__ i32 wg_f64_to_i32(double v) {
  if (v != v) return 0;
  if (v == WG_INF) return 0x7fffffff;
  if (v == -WG_INF) return (i32)0x80000000U;
  double t = trunc(v);
  if (t >= -9223372036854775808.0 && t < 9223372036854775808.0) return (i32)(u32)(u64)(i64)t;
  double r = fmod(t, 4294967296.0);
  return (i32)(u32)(u64)(i64)r;
}
__device__ __forceinline__ i64 wg_f32_to_i64(float v) { return wg_f64_to_i64((double)v); }
__device__ __forceinline__ i32 wg_f32_to_i32(float v) { return wg_f64_to_i32((double)v); }
// int -> f32 goes through f64 first, like f32_round(float(v)) (types.py:177).
__device__ __forceinline__ float wg_i64_to_f32(i64 v) { return (float)(double)v; }

// ---------------------------------------------------------------------------
// Merge folds.  A fold starts from an *internal* identity that is an exact
// no-op for every input, so a slot can be pre-initialised:
//   f +   : -0.0   (-0.0 + x == x for all x, including +-0.0)
//   f *   : 1.0
//   f min : NaN    (wg_min_f64 prefers the other side)
//   f max : -inf
//   int   : 0, 1, MAX, MIN
// The reference starts from the first merged value (builders.py:304-306) and
// yields identity_value (types.py:185-192) for an empty merger; a per-slot
// "merged" flag restores that at finalisation.
template <typename T> struct WgAdd { static __device__ __forceinline__ T f(T a, T b) { return a + b; } };
template <> struct WgAdd<i64> { static __device__ __forceinline__ i64 f(i64 a, i64 b) { return wg_add_i64(a, b); } };
template <> struct WgAdd<i32> { static __device__ __forceinline__ i32 f(i32 a, i32 b) { return wg_add_i32(a, b); } };
template <typename T> struct WgMul { static __device__ __forceinline__ T f(T a, T b) { return a * b; } };
template <> struct WgMul<i64> { static __device__ __forceinline__ i64 f(i64 a, i64 b) { return wg_mul_i64(a, b); } };
template <> struct WgMul<i32> { static __device__ __forceinline__ i32 f(i32 a, i32 b) { return wg_mul_i32(a, b); } };
template <typename T> struct WgMin { static __device__ __forceinline__ T f(T a, T b) { return a <= b ? a : b; } };
template <> struct WgMin<double> { static __device__ __forceinline__ double f(double a, double b) { return wg_min_f64(a, b); } };
template <> struct WgMin<float> { static __device__ __forceinline__ float f(float a, float b) { return wg_min_f32(a, b); } };
template <typename T> struct WgMax { static __device__ __forceinline__ T f(T a, T b) { return a >= b ? a : b; } };
template <> struct WgMax<double> { static __device__ __forceinline__ double f(double a, double b) { return wg_max_f64(a, b); } };
template <> struct WgMax<float> { static __device__ __forceinline__ float f(float a, float b) { return wg_max_f32(a, b); } };

// ---------------------------------------------------------------------------
// 64-bit value punning for partial/slot storage (every slot field is 8 bytes).
template <typename T> __device__ __forceinline__ u64 wg_to_bits(T v);
template <> __device__ __forceinline__ u64 wg_to_bits<double>(double v) { return (u64)__double_as_longlong(v); }
template <> __device__ __forceinline__ u64 wg_to_bits<float>(float v) { return (u64)(u32)__float_as_int(v); }
template <> __device__ __forceinline__ u64 wg_to_bits<i64>(i64 v) { return (u64)v; }
template <> __device__ __forceinline__ u64 wg_to_bits<i32>(i32 v) { return (u64)(u32)v; }
template <> __device__ __forceinline__ u64 wg_to_bits<bool>(bool v) { return v ? 1ULL : 0ULL; }
template <typename T> __device__ __forceinline__ T wg_from_bits(u64 b);
template <> __device__ __forceinline__ double wg_from_bits<double>(u64 b) { return __longlong_as_double((i64)b); }
template <> __device__ __forceinline__ float wg_from_bits<float>(u64 b) { return __int_as_float((int)(u32)b); }
template <> __device__ __forceinline__ i64 wg_from_bits<i64>(u64 b) { return (i64)b; }
template <> __device__ __forceinline__ i32 wg_from_bits<i32>(u64 b) { return (i32)(u32)b; }
template <> __device__ __forceinline__ bool wg_from_bits<bool>(u64 b) { return b != 0; }

// ---------------------------------------------------------------------------
// Block-wide fold of one value (plus the merged flag) in a fixed tree
// order; result valid in thread 0.  Lanes without data hold `ident`, the
// fold's internal identity, so padding is an exact no-op.  smem >= 32.
template <typename T, typename OP>
__device__ __forceinline__ void wg_block_fold(T& v, int& has, T ident, T* smem_v, int* smem_h) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    T o = __shfl_down_sync(0xffffffffu, v, d);
    int oh = __shfl_down_sync(0xffffffffu, has, d);
    v = OP::f(v, o);
    has |= oh;
  }
  __syncthreads();
  if (lane == 0) { smem_v[warp] = v; smem_h[warp] = has; }
  __syncthreads();
  if (warp == 0) {
    v = (lane < nw) ? smem_v[lane] : ident;
    has = (lane < nw) ? smem_h[lane] : 0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      T o = __shfl_down_sync(0xffffffffu, v, d);
      int oh = __shfl_down_sync(0xffffffffu, has, d);
      v = OP::f(v, o);
      has |= oh;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Block-wide exclusive scan of one i64 count per thread.  Returns the
// exclusive prefix; *total receives the block aggregate (all threads).
__device__ __forceinline__ i64 wg_block_exclusive_scan(i64 x, i64* smem /* >= 33 */, i64* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  i64 incl = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    i64 o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  __syncthreads();
  if (lane == 31) smem[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    i64 w = (lane < nw) ? smem[lane] : 0;
    i64 wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      i64 o = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += o;
    }
    if (lane < nw) smem[lane] = wi - w;  // exclusive warp offsets
    if (lane == nw - 1) smem[32] = wi;
  }
  __syncthreads();
  *total = smem[32];
  return smem[warp] + incl - x;
}

// ---------------------------------------------------------------------------
// Single-pass decoupled look-back (Merrill & Garland).  status[t] packs a
// 2-bit flag over a 62-bit count: 0 = not ready, 1 = aggregate, 2 = prefix.
// Tiles are claimed in launch order through an atomic counter, so every
// predecessor of a tile is held by a running block: spinning is safe.
#define WG_ST_AGG (1ULL << 62)
#define WG_ST_PRE (2ULL << 62)
#define WG_ST_MASK ((1ULL << 62) - 1)

__device__ __forceinline__ u64 wg_ld_volatile(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wg_st_volatile(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Called by warp 0 only.  Returns the exclusive prefix of `tile`.  Each
// look-back step inspects a window of 32 x WG_LB_PER predecessors (lane L
// covers distances 4L..4L+3), so the inclusive-prefix front moves 4x faster
// than a one-status-per-lane window -- with ~600 tiles in flight that front
// is what bounds a scan's throughput.
#ifndef WG_LB_PER
#define WG_LB_PER 1
#endif
#ifndef WG_LB_SLEEP
#define WG_LB_SLEEP 0
#endif
__device__ __forceinline__ i64 wg_lookback_core(u64* status, i64 tile, i64 aggregate);
__device__ __forceinline__ i64 wg_lookback(u64* status, i64 tile, i64 aggregate) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) wg_st_volatile(status, WG_ST_PRE | (u64)aggregate);
    return 0;
  }
  if (lane == 0) wg_st_volatile(status + tile, WG_ST_AGG | (u64)aggregate);
  return wg_lookback_core(status, tile, aggregate);
}
// The look-back proper (tile > 0, its aggregate already published): each
// lane reads WG_LB_PER consecutive predecessors per round trip.
__device__ __forceinline__ i64 wg_lookback_core(u64* status, i64 tile, i64 aggregate) {
  const int lane = threadIdx.x & 31;
  i64 excl = 0;
  i64 t = tile - 1;
  while (true) {
    u64 s[WG_LB_PER];
    int qp = WG_LB_PER;   // first prefix entry among this lane's span
#pragma unroll
    for (int q = 0; q < WG_LB_PER; ++q) {
      const i64 idx = t - (i64)(lane * WG_LB_PER + q);
      s[q] = (idx >= 0) ? wg_ld_volatile(status + idx) : WG_ST_PRE;
    }
#pragma unroll
    for (int q = WG_LB_PER - 1; q >= 0; --q) if ((s[q] >> 62) == 2) qp = q;
    bool xb = false;      // a not-ready entry before this lane's first prefix
#pragma unroll
    for (int q = 0; q < WG_LB_PER; ++q) if (q < qp && (s[q] >> 62) == 0) xb = true;
    const unsigned mp = __ballot_sync(0xffffffffu, qp < WG_LB_PER);
    const int first = mp ? __ffs(mp) - 1 : 32;        // lane holding the nearest prefix
    const unsigned mx = __ballot_sync(0xffffffffu, xb);
    const unsigned upto = (first >= 31) ? 0xffffffffu : ((2u << first) - 1u);
    if (mx & upto) {  // a needed predecessor has not published yet: back off, retry
#if WG_LB_SLEEP > 0
      __nanosleep(WG_LB_SLEEP);
#endif
      continue;
    }
    i64 val = 0;
    if (lane <= first) {
      const int lim = (lane == first) ? qp : WG_LB_PER - 1;
#pragma unroll
      for (int q = 0; q < WG_LB_PER; ++q) if (q <= lim) val += (i64)(s[q] & WG_ST_MASK);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) val += __shfl_xor_sync(0xffffffffu, val, d);
    excl += val;
    if (mp) break;
    t -= 32 * WG_LB_PER;
  }
  if (lane == 0) wg_st_volatile(status + tile, WG_ST_PRE | (u64)(excl + aggregate));
  return excl;
}

// Warp-specialised scan schedule (codegen SCAN_WS): the compute warps
// (threads [0, nthreads)) publish each tile's aggregate as soon as it is
// counted and move on; one extra warp resolves the tile's exclusive prefix
// later (the aggregate is already in status[tile]) and publishes the
// inclusive prefix.
__device__ __forceinline__ void wg_bar_group(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
// Block-wide exclusive scan over the compute group only (named barrier 1).
__device__ __forceinline__ i64 wg_group_exclusive_scan(i64 x, i64* smem /* >= 33 */, i64* total, int nthreads) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = nthreads >> 5;
  i64 incl = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    i64 o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  wg_bar_group(nthreads);
  if (lane == 31) smem[warp] = incl;
  wg_bar_group(nthreads);
  if (warp == 0) {
    i64 w = (lane < nw) ? smem[lane] : 0;
    i64 wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      i64 o = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += o;
    }
    if (lane < nw) smem[lane] = wi - w;
    if (lane == nw - 1) smem[32] = wi;
  }
  wg_bar_group(nthreads);
  *total = smem[32];
  return smem[warp] + incl - x;
}
__device__ __forceinline__ void wg_publish_aggregate(u64* status, i64 tile, i64 aggregate) {
  wg_st_volatile(status + tile, (tile == 0 ? WG_ST_PRE : WG_ST_AGG) | (u64)aggregate);
}
// The look-back of wg_lookback for a tile whose aggregate is already
// published (whole warp; returns the exclusive prefix).
__device__ __forceinline__ i64 wg_lookback_resolve(u64* status, i64 tile, i64 aggregate) {
  if (tile == 0) return 0;
  return wg_lookback_core(status, tile, aggregate);
}

// ---------------------------------------------------------------------------
// Atomic folds into 8-byte slots (dictmerger values, vecmerger bins).
template <typename T> __device__ __forceinline__ void wg_atomic_add(T* p, T v);
template <> __device__ __forceinline__ void wg_atomic_add<double>(double* p, double v) { atomicAdd(p, v); }
template <> __device__ __forceinline__ void wg_atomic_add<float>(float* p, float v) { atomicAdd(p, v); }
template <> __device__ __forceinline__ void wg_atomic_add<i64>(i64* p, i64 v) { atomicAdd((u64*)p, (u64)v); }
template <> __device__ __forceinline__ void wg_atomic_add<i32>(i32* p, i32 v) { atomicAdd(p, v); }

template <typename T, typename OP>
__device__ __forceinline__ void wg_atomic_cas_fold(T* p, T v);
template <typename OP>
__device__ __forceinline__ void wg_atomic_cas_fold_f64(double* p, double v) {
  u64* a = (u64*)p;
  u64 old = *(volatile u64*)a, assumed;
  do {
    assumed = old;
    double nv = OP::f(__longlong_as_double((i64)assumed), v);
    u64 nb = (u64)__double_as_longlong(nv);
    if (nb == assumed) return;
    old = atomicCAS(a, assumed, nb);
  } while (old != assumed);
}
template <typename OP>
__device__ __forceinline__ void wg_atomic_cas_fold_f32(float* p, float v) {
  u32* a = (u32*)p;
  u32 old = *(volatile u32*)a, assumed;
  do {
    assumed = old;
    float nv = OP::f(__int_as_float((int)assumed), v);
    u32 nb = (u32)__float_as_int(nv);
    if (nb == assumed) return;
    old = atomicCAS(a, assumed, nb);
  } while (old != assumed);
}
template <typename OP>
__device__ __forceinline__ void wg_atomic_cas_fold_i64(i64* p, i64 v) {
  u64* a = (u64*)p;
  u64 old = *(volatile u64*)a, assumed;
  do {
    assumed = old;
    u64 nb = (u64)OP::f((i64)assumed, v);
    if (nb == assumed) return;
    old = atomicCAS(a, assumed, nb);
  } while (old != assumed);
}
template <typename OP>
__device__ __forceinline__ void wg_atomic_cas_fold_i32(i32* p, i32 v) {
  u32* a = (u32*)p;
  u32 old = *(volatile u32*)a, assumed;
  do {
    assumed = old;
    u32 nb = (u32)OP::f((i32)assumed, v);
    if (nb == assumed) return;
    old = atomicCAS(a, assumed, nb);
  } while (old != assumed);
}

// op codes: 0 '+', 1 '*', 2 min, 3 max
template <int OPC, typename T> struct WgAtomicFold;
template <typename T> struct WgAtomicFold<0, T> { static __device__ __forceinline__ void f(T* p, T v) { wg_atomic_add<T>(p, v); } };
template <> struct WgAtomicFold<1, double> { static __device__ __forceinline__ void f(double* p, double v) { wg_atomic_cas_fold_f64<WgMul<double>>(p, v); } };
template <> struct WgAtomicFold<1, float> { static __device__ __forceinline__ void f(float* p, float v) { wg_atomic_cas_fold_f32<WgMul<float>>(p, v); } };
template <> struct WgAtomicFold<1, i64> { static __device__ __forceinline__ void f(i64* p, i64 v) { wg_atomic_cas_fold_i64<WgMul<i64>>(p, v); } };
template <> struct WgAtomicFold<1, i32> { static __device__ __forceinline__ void f(i32* p, i32 v) { wg_atomic_cas_fold_i32<WgMul<i32>>(p, v); } };
template <> struct WgAtomicFold<2, double> { static __device__ __forceinline__ void f(double* p, double v) { wg_atomic_cas_fold_f64<WgMin<double>>(p, v); } };
template <> struct WgAtomicFold<2, float> { static __device__ __forceinline__ void f(float* p, float v) { wg_atomic_cas_fold_f32<WgMin<float>>(p, v); } };
template <> struct WgAtomicFold<2, i64> { static __device__ __forceinline__ void f(i64* p, i64 v) { atomicMin((long long*)p, (long long)v); } };
template <> struct WgAtomicFold<2, i32> { static __device__ __forceinline__ void f(i32* p, i32 v) { atomicMin(p, v); } };
template <> struct WgAtomicFold<3, double> { static __device__ __forceinline__ void f(double* p, double v) { wg_atomic_cas_fold_f64<WgMax<double>>(p, v); } };
template <> struct WgAtomicFold<3, float> { static __device__ __forceinline__ void f(float* p, float v) { wg_atomic_cas_fold_f32<WgMax<float>>(p, v); } };
template <> struct WgAtomicFold<3, i64> { static __device__ __forceinline__ void f(i64* p, i64 v) { atomicMax((long long*)p, (long long)v); } };
template <> struct WgAtomicFold<3, i32> { static __device__ __forceinline__ void f(i32* p, i32 v) { atomicMax(p, v); } };

// Shared-memory variants (same semantics, smem addresses).
template <int OPC, typename T> __device__ __forceinline__ void wg_smem_fold(T* p, T v) { WgAtomicFold<OPC, T>::f(p, v); }

// sm_100 has no native 64-bit shared-memory atomic add (it is a CAS spin
// loop).  Integer + splits into two native 32-bit adds: the low word's old
// value tells each adder whether its low half carried, and the carries sum
// to the number of low-word wraps, so the 64-bit total is exact.
__device__ __forceinline__ void wg_smem_add_i64(i64* p, i64 v) {
  unsigned* w = reinterpret_cast<unsigned*>(p);
  const u64 uv = (u64)v;
  const unsigned lo = (unsigned)uv, hi = (unsigned)(uv >> 32);
  const unsigned old = atomicAdd(w, lo);
  const unsigned up = hi + ((unsigned)(old + lo) < old ? 1u : 0u);
  if (up) atomicAdd(w + 1, up);
}
template <int OPC, typename T> struct WgSmemFold { static __device__ __forceinline__ void f(T* p, T v) { WgAtomicFold<OPC, T>::f(p, v); } };
template <> struct WgSmemFold<0, i64> { static __device__ __forceinline__ void f(i64* p, i64 v) { wg_smem_add_i64(p, v); } };

// ---------------------------------------------------------------------------
// Hash table for dictmerger / group ids.  Keys are packed into KW 64-bit
// words.  KW == 1 uses the key word itself as the claim word with an EMPTY
// sentinel; the (rare) key equal to the sentinel lives in slot `cap`.
// Slot layout (AoS, 8-byte fields): [key words][value fields].
#define WG_EMPTY_KEY 0xffffffffffffffffULL

__device__ __forceinline__ u64 wg_mix64(u64 x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// Insert-or-find a one-word key.  Returns the slot index, or -1 when
// WG_MAX_PROBE consecutive slots are taken by other keys: the caller spills
// the merge to the overflow list and the host grows the table and replays
// it.  `claims` counts keys this thread inserted (summed per CTA into the
// table's distinct-key counter at kernel end -- no contended global
// counter on the insert path).
#define WG_MAX_PROBE 128
// Probe read of a single-word key slot: an L2 (cg) load.  A slot moves from
// EMPTY to its key exactly once (CAS), so a stale EMPTY only costs a failed
// CAS that returns the key; no system-scope (volatile) load is needed.
#ifndef WG_PROBE_VOLATILE
#define WG_PROBE_LD(p) __ldcg((const unsigned long long*)(p))
#else
#define WG_PROBE_LD(p) (*(volatile u64*)(p))
#endif
__device__ __forceinline__ i64 wg_ht_find1(u64* table, int slot_words, u64 mask, u64 key, int& claims) {
  if (key == WG_EMPTY_KEY) {
    // Dedicated slot for the sentinel value (claim word EMPTY -> 0).
    u64* s = table + (mask + 1) * (u64)slot_words;
    u64 prev = atomicCAS((unsigned long long*)s, WG_EMPTY_KEY, 0ULL);
    if (prev == WG_EMPTY_KEY) claims++;
    return (i64)(mask + 1);
  }
  u64 h = wg_mix64(key) & mask;
#pragma unroll 1
  for (int probe = 0; probe < WG_MAX_PROBE; ++probe) {
    u64* s = table + h * (u64)slot_words;
    u64 cur = WG_PROBE_LD(s);
    if (cur == key) return (i64)h;
    if (cur == WG_EMPTY_KEY) {
      u64 prev = atomicCAS((unsigned long long*)s, WG_EMPTY_KEY, key);
      if (prev == WG_EMPTY_KEY) { claims++; return (i64)h; }
      if (prev == key) return (i64)h;
    }
    h = (h + 1) & mask;
  }
  return -1;
}

// Multi-word keys: word 0 of the slot is a state word (0 empty, 1 busy,
// 2 full) followed by KW key words.
__device__ __forceinline__ i64 wg_ht_findN(u64* table, int slot_words, u64 mask, const u64* key, int kw,
                                            int& claims) {
  u64 hh = 0x9e3779b97f4a7c15ULL;
  for (int k = 0; k < kw; ++k) hh = wg_mix64(hh ^ key[k]) + 0x9e3779b97f4a7c15ULL * (u64)(k + 1);
  u64 h = hh & mask;
#pragma unroll 1
  for (int probe = 0; probe < WG_MAX_PROBE; ++probe) {
    u64* s = table + h * (u64)slot_words;
    u64 st = *(volatile u64*)s;
    if (st == 0) {
      u64 prev = atomicCAS((unsigned long long*)s, 0ULL, 1ULL);
      if (prev == 0) {
        for (int k = 0; k < kw; ++k) ((volatile u64*)s)[1 + k] = key[k];
        __threadfence();
        atomicExch((unsigned long long*)s, 2ULL);
        claims++;
        return (i64)h;
      }
      st = prev;
    }
    while (st == 1) st = *(volatile u64*)s;  // another thread is writing the key
    bool eq = true;
    for (int k = 0; k < kw; ++k) if (((volatile u64*)s)[1 + k] != key[k]) { eq = false; break; }
    if (eq) return (i64)h;
    h = (h + 1) & mask;
  }
  return -1;
}

// order_key (builders.py:496-507) of one key leaf as an unsigned 64-bit
// integer: signed ints ordered, floats in IEEE total order with -0.0 == 0.0
// and every NaN after +inf.  Dictionary probes compare these.
template <typename T> __device__ __forceinline__ u64 wg_okey(T v);
template <> __device__ __forceinline__ u64 wg_okey<bool>(bool v) { return v ? 1ULL : 0ULL; }
template <> __device__ __forceinline__ u64 wg_okey<i32>(i32 v) { return (u64)(i64)v ^ 0x8000000000000000ULL; }
template <> __device__ __forceinline__ u64 wg_okey<i64>(i64 v) { return (u64)v ^ 0x8000000000000000ULL; }
template <> __device__ __forceinline__ u64 wg_okey<double>(double v) {
  if (v != v) return 0xffffffffffffffffULL;
  if (v == 0.0) v = 0.0;
  const u64 b = (u64)__double_as_longlong(v);
  const u64 k = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
  return k == 0xffffffffffffffffULL ? 0xfffffffffffffffeULL : k;
}
template <> __device__ __forceinline__ u64 wg_okey<float>(float v) { return wg_okey<double>((double)v); }

// First row (loop index) merging a -0.0 (z[1]) / +0.0 (z[0]) key into a
// one-float-field dictmerger: the reference keeps the first-inserted key
// object of the pair -0.0 == 0.0 (Python dict semantics).
__device__ __forceinline__ void wg_zero_row(unsigned long long* z, bool neg, i64 row) {
  unsigned long long* w = z + (neg ? 1 : 0);
  if ((unsigned long long)row < *(volatile unsigned long long*)w) atomicMin(w, (unsigned long long)row);
}

// Canonical key words.  -0.0 and 0.0 are one dictionary key in the
// reference (Python dict semantics); they map to the same word here.
// Every NaN is one key too: the NaNs a program produces (0.0 / 0.0, inf -
// inf, ...) are one float object in the reference and compare as one key.
__device__ __forceinline__ u64 wg_key_f64(double v) {
  return v == 0.0 ? 0ULL : (v != v ? 0x7ff8000000000000ULL : (u64)__double_as_longlong(v));
}
__device__ __forceinline__ u64 wg_key_f32(float v) {
  return v == 0.0f ? 0ULL : (v != v ? 0x7fc00000ULL : (u64)(u32)__float_as_int(v));
}

// ---------------------------------------------------------------------------
#ifndef WG_LD256
#define WG_LD256 1
#endif
#ifndef WG_ST256
#define WG_ST256 1
#endif
// 256-bit vector ld/st need PTX 8.8 (CUDA 12.9); an older NVRTC (e.g. torch's
// bundled 12.8, when torch loaded its libnvrtc first) gets the 16-byte path.
#if !defined(__CUDACC_VER_MAJOR__) || __CUDACC_VER_MAJOR__ < 12 || (__CUDACC_VER_MAJOR__ == 12 && __CUDACC_VER_MINOR__ < 9)
#undef WG_LD256
#define WG_LD256 0
#undef WG_ST256
#define WG_ST256 0
#endif
// Contiguous per-thread column access (ITEMS consecutive elements): 32-byte
// (sm_100 LDG.256 / STG.256) or 16-byte
// vector loads/stores when the address allows, streaming cache hints so the
// single-use column traffic does not evict hash tables or bins from L2.
template <typename T, int N>
__device__ __forceinline__ void wg_load_contig(const T* __restrict__ src, T (&dst)[N]) {
  constexpr int B = N * (int)sizeof(T);
  const unsigned long long a = (unsigned long long)src;
#if WG_LD256
  // sm_100 256-bit loads: each lane reads whole 32-byte sectors
  if constexpr (B % 32 == 0) {
    if ((a & 31) == 0) {
#pragma unroll
      for (int c = 0; c < B / 32; ++c) {
        unsigned long long* d = reinterpret_cast<unsigned long long*>(&dst[0]) + 4 * c;
        asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(d[0]), "=l"(d[1]), "=l"(d[2]), "=l"(d[3]) : "l"(src + c * (32 / (int)sizeof(T))));
      }
      return;
    }
  }
#endif
  if constexpr (B % 16 == 0) {
    if ((a & 15) == 0) {
#pragma unroll
      for (int c = 0; c < B / 16; ++c) reinterpret_cast<uint4*>(&dst[0])[c] = __ldcs(reinterpret_cast<const uint4*>(src) + c);
      return;
    }
  }
  if constexpr (B % 8 == 0) {
    if ((a & 7) == 0) {
#pragma unroll
      for (int c = 0; c < B / 8; ++c) reinterpret_cast<uint2*>(&dst[0])[c] = __ldcs(reinterpret_cast<const uint2*>(src) + c);
      return;
    }
  }
  if constexpr (B % 4 == 0) {
    if ((a & 3) == 0) {
#pragma unroll
      for (int c = 0; c < B / 4; ++c) reinterpret_cast<unsigned*>(&dst[0])[c] = __ldcs(reinterpret_cast<const unsigned*>(src) + c);
      return;
    }
  }
#pragma unroll
  for (int q = 0; q < N; ++q) dst[q] = src[q];
}

template <typename T, int N>
__device__ __forceinline__ void wg_store_contig(T* __restrict__ dst, const T (&src)[N]) {
  constexpr int B = N * (int)sizeof(T);
  const unsigned long long a = (unsigned long long)dst;
#if WG_ST256
  if constexpr (B % 32 == 0) {
    if ((a & 31) == 0) {
#pragma unroll
      for (int c = 0; c < B / 32; ++c) {
        const unsigned long long* d = reinterpret_cast<const unsigned long long*>(&src[0]) + 4 * c;
        asm volatile("st.global.cs.v4.u64 [%0], {%1,%2,%3,%4};"
                     :: "l"(dst + c * (32 / (int)sizeof(T))), "l"(d[0]), "l"(d[1]), "l"(d[2]), "l"(d[3]) : "memory");
      }
      return;
    }
  }
#endif
  if constexpr (B % 16 == 0) {
    if ((a & 15) == 0) {
#pragma unroll
      for (int c = 0; c < B / 16; ++c) __stcs(reinterpret_cast<uint4*>(dst) + c, reinterpret_cast<const uint4*>(&src[0])[c]);
      return;
    }
  }
  if constexpr (B % 8 == 0) {
    if ((a & 7) == 0) {
#pragma unroll
      for (int c = 0; c < B / 8; ++c) __stcs(reinterpret_cast<uint2*>(dst) + c, reinterpret_cast<const uint2*>(&src[0])[c]);
      return;
    }
  }
#pragma unroll
  for (int q = 0; q < N; ++q) dst[q] = src[q];
}

// Shared-memory table probe with a caller-chosen probe limit.
__device__ __forceinline__ int wg_sht_findp(u64* t, int sw, int mask, u64 key, int max_probe) {
  if (key == WG_EMPTY_KEY) return -1;
  int h = (int)(wg_mix64(key) & (u64)mask);
#pragma unroll 1
  for (int probe = 0; probe < max_probe; ++probe) {
    u64* s = t + (u64)h * sw;
    u64 cur = *(volatile u64*)s;
    if (cur == key) return h;
    if (cur == WG_EMPTY_KEY) {
      u64 prev = atomicCAS((unsigned long long*)s, WG_EMPTY_KEY, key);
      if (prev == WG_EMPTY_KEY || prev == key) return h;
    }
    h = (h + 1) & mask;
  }
  return -1;
}

// Per-CTA shared-memory table (privatised dictmerger level 1) for one-word
// keys.  Bounded probing: a miss with no free slot returns -1 and the
// caller merges straight into the global table instead.
__device__ __forceinline__ int wg_sht_find1(u64* t, int sw, int mask, u64 key) {
  if (key == WG_EMPTY_KEY) return -1;
  int h = (int)(wg_mix64(key) & (u64)mask);
#pragma unroll 1
  for (int probe = 0; probe < 8; ++probe) {
    u64* s = t + (u64)h * sw;
    u64 cur = *(volatile u64*)s;
    if (cur == key) return h;
    if (cur == WG_EMPTY_KEY) {
      u64 prev = atomicCAS((unsigned long long*)s, WG_EMPTY_KEY, key);
      if (prev == WG_EMPTY_KEY || prev == key) return h;
    }
    h = (h + 1) & mask;
  }
  return -1;
}

// ---------------------------------------------------------------------------
// Deferred dictmerger merges (codegen: one pending merge per item, processed
// after the item loop while the warp is converged).

// Butterfly fold over the full warp; every lane receives the result.
template <typename T, typename OP>
__device__ __forceinline__ T wg_warp_allfold(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = OP::f(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

__device__ __forceinline__ u64 wg_ht_home(u64 key, u64 mask) { return wg_mix64(key) & mask; }

// Probe continuation for one-word keys given the home slot h and the word
// already loaded from it (lets callers issue the first probe of several
// rows before resolving any: memory-level parallelism for tables >> L2).
__device__ __forceinline__ i64 wg_ht_resolve1(u64* table, int slot_words, u64 mask, u64 key, u64 h, u64 cur,
                                               int& claims) {
  if (key == WG_EMPTY_KEY) return wg_ht_find1(table, slot_words, mask, key, claims);
#pragma unroll 1
  for (int probe = 0; probe < WG_MAX_PROBE; ++probe) {
    u64* s = table + h * (u64)slot_words;
    if (cur == key) return (i64)h;
    if (cur == WG_EMPTY_KEY) {
      u64 prev = atomicCAS((unsigned long long*)s, WG_EMPTY_KEY, key);
      if (prev == WG_EMPTY_KEY) { claims++; return (i64)h; }
      if (prev == key) return (i64)h;
    }
    h = (h + 1) & mask;
    cur = WG_PROBE_LD(table + h * (u64)slot_words);
  }
  return -1;
}

// ---------------------------------------------------------------------------
// Bulk-async column streaming (cp.async.bulk on the TMA engine + mbarrier).
__device__ __forceinline__ unsigned wg_saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wg_mbar_init(u64* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(wg_saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void wg_fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void wg_fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void wg_mbar_expect_tx(u64* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(wg_saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wg_bulk_g2s(void* dst, const void* src, unsigned bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(wg_saddr(dst)),
      "l"(src), "r"(bytes), "r"(wg_saddr(bar))
      : "memory");
}
__device__ __forceinline__ void wg_mbar_arrive(u64* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(wg_saddr(bar)) : "memory");
}
__device__ __forceinline__ void wg_mbar_wait(u64* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra WAIT_%=;\n}" ::"r"(
          wg_saddr(bar)),
      "r"(phase)
      : "memory");
}
// Shared-memory counterpart of wg_load_contig (stage -> registers).
template <typename T, int N>
__device__ __forceinline__ void wg_lds_contig(const T* src, T (&dst)[N]) {
  constexpr int B = N * (int)sizeof(T);
  if constexpr (B % 16 == 0) {
#pragma unroll
    for (int c = 0; c < B / 16; ++c) reinterpret_cast<uint4*>(&dst[0])[c] = reinterpret_cast<const uint4*>(src)[c];
  } else if constexpr (B % 8 == 0) {
#pragma unroll
    for (int c = 0; c < B / 8; ++c) reinterpret_cast<uint2*>(&dst[0])[c] = reinterpret_cast<const uint2*>(src)[c];
  } else if constexpr (B % 4 == 0) {
#pragma unroll
    for (int c = 0; c < B / 4; ++c) reinterpret_cast<unsigned*>(&dst[0])[c] = reinterpret_cast<const unsigned*>(src)[c];
  } else {
#pragma unroll
    for (int q = 0; q < N; ++q) dst[q] = src[q];
  }
}


// erf from a piecewise polynomial table (tools/gen_erf_table.py): one
// 80-byte row per 1/16 of |x| in [0, 6), degree-10 polynomial in
// w = 16|x| - k with a split constant term; c1..c5 in f64, the tail c6..c10
// in f32 (evaluated with FFMA).  <= 0.5 ulp table error and 11 FP64
// operations instead of libdevice's ~43 (24-term polynomial + exp).  The
// table is copied into shared memory at kernel entry (wg_erf_tab_init) and a
// row is five 16-byte loads; the 20-word stride spreads rows over all eight
// 16-byte bank groups.
#include "wg_erf_table.h"
__shared__ __align__(16) unsigned wg_erf_s[WG_ERF_ROWS * WG_ERF_STRIDE];
__device__ __forceinline__ void wg_erf_tab_init() {
  for (int q = threadIdx.x; q < WG_ERF_ROWS * WG_ERF_STRIDE; q += blockDim.x) wg_erf_s[q] = WG_ERF_TAB[q];
}
__device__ __forceinline__ double wg_erf_tab(double x) {
  const double a = fabs(x);
  const double ac = (a < 6.0) ? a : 6.0;                     // NaN -> 6.0 (fixed below)
  const double sh = fma(ac, 16.0, 6755399441055744.0);       // round(16a) + 1.5*2^52
  const int k = __double2loint(sh);
  const double w = fma(ac, 16.0, -(sh - 6755399441055744.0)); // exact, in [-1/2, 1/2]
  const uint4* r = reinterpret_cast<const uint4*>(wg_erf_s + k * WG_ERF_STRIDE);
  const uint4 u0 = r[0], u1 = r[1], u2 = r[2], u3 = r[3], u4 = r[4];
  const float wf = (float)w;
  const float t = fmaf(fmaf(fmaf(fmaf(__uint_as_float(u4.z), wf, __uint_as_float(u4.y)), wf, __uint_as_float(u4.x)),
                            wf, __uint_as_float(u3.w)), wf, __uint_as_float(u3.z));
  double q = fma((double)t, w, __hiloint2double((int)u2.w, (int)u2.z));   // c5
  q = fma(q, w, __hiloint2double((int)u2.y, (int)u2.x));                  // c4
  q = fma(q, w, __hiloint2double((int)u1.w, (int)u1.z));                  // c3
  q = fma(q, w, __hiloint2double((int)u1.y, (int)u1.x));                  // c2
  q = fma(q, w, __hiloint2double((int)u0.w, (int)u0.z));                  // c1
  double res = __hiloint2double((int)u3.y, (int)u3.x) + fma(q, w, __hiloint2double((int)u0.y, (int)u0.x));
  res = (a >= 5.9215871957945) ? 1.0 : res;                  // erf rounds to 1 beyond here
  res = (a != a) ? x : res;
  return copysign(res, x);
}

// log from a 128-row shared-memory table (tools/gen_log_table.py): x = 2^k z,
// row i = top 7 bits of bits(x) - OFF, r = z invc_i - 1 (|r| <= 2^-8, one fma),
// log x = k ln2 + logc_i + log1p(r) with the large sums compensated; <= 1 ulp
// (checked against mpmath by the generator and tests/test_gpu_math.py), 20
// FP64 operations and no reciprocal iteration (libdevice: ~30 + MUFU.RCP64H).
#include "wg_log_table.h"
__shared__ __align__(16) double wg_log_s[2 * WG_LOG_ROWS];
__shared__ double wg_log_lo_s[WG_LOG_ROWS];
__device__ __forceinline__ void wg_log_tab_init() {
  for (int q = threadIdx.x; q < 2 * WG_LOG_ROWS; q += blockDim.x) wg_log_s[q] = __longlong_as_double((long long)WG_LOG_TAB[q]);
  for (int q = threadIdx.x; q < WG_LOG_ROWS; q += blockDim.x) wg_log_lo_s[q] = __longlong_as_double((long long)WG_LOG_LO[q]);
}
__device__ __forceinline__ double wg_log_tab(double x) {
  unsigned long long ix = (unsigned long long)__double_as_longlong(x);
  int hi = (int)(ix >> 32);
  int kadj = 0;
  if (__builtin_expect(hi < 0x00100000, 0)) {           // subnormal, zero or negative
    x *= 18014398509481984.0;                           // 2^54
    ix = (unsigned long long)__double_as_longlong(x);
    hi = (int)(ix >> 32);
    kadj = -54;
  }
  if (__builtin_expect((unsigned)(hi - 1) > 0x7FEFFFFEu, 0)) {   // <= 0, inf, nan
    const double inf = __longlong_as_double(0x7FF0000000000000LL);
    return (ix << 1) == 0 ? -inf : fma(x, inf, inf);
  }
  const unsigned long long tmp = ix - WG_LOG_OFF;
  const int i = (int)(tmp >> 45) & (WG_LOG_ROWS - 1);
  const int k = (int)((long long)tmp >> 52) + kadj;
  const double z = __longlong_as_double((long long)(ix - (tmp & 0xFFF0000000000000ULL)));
  const double2 ic = reinterpret_cast<const double2*>(wg_log_s)[i];
  const double r = fma(z, ic.x, -1.0);
  const double kd = __hiloint2double(0x43300000, k ^ 0x80000000) - __hiloint2double(0x43300000, 0x80000000);
  const double l2hi = __longlong_as_double((long long)WG_LOG_LN2HI);
  const double t1 = fma(kd, l2hi, ic.y);
  const double e1 = fma(kd, l2hi, -t1) + ic.y;
  const double t2 = t1 + r;
  const double e2 = (t1 - t2) + r;
  const double lo = fma(kd, __longlong_as_double((long long)WG_LOG_LN2LO), wg_log_lo_s[i]) + (e1 + e2);
  double q = fma(1.0 / 7.0, r, -1.0 / 6.0);
  q = fma(q, r, 1.0 / 5.0);
  q = fma(q, r, -0.25);
  q = fma(q, r, 1.0 / 3.0);
  q = fma(q, r, -0.5);
  return t2 + (lo + (r * r) * q);
}

// exp from a 64-entry shared-memory table of 2^(j/64) (tools/gen_exp_table.py):
// k = round(64 x / ln2), r = x - k ln2/64 (Cody-Waite), exp(r) - 1 to r^6,
// result 2^(k>>6) (T_hi + (T_lo + T_hi p)); <= 1 ulp, 12 FP64 operations
// with a 9-deep chain (libdevice: 15, 15 deep).  Near over/underflow the
// scaling is split in two steps, as libdevice does.
#include "wg_exp_table.h"
__shared__ __align__(16) double wg_exp_s[2 * WG_EXP_N];
__device__ __forceinline__ void wg_exp_tab_init() {
  for (int q = threadIdx.x; q < 2 * WG_EXP_N; q += blockDim.x) wg_exp_s[q] = __longlong_as_double((long long)WG_EXP_TAB[q]);
}
__device__ __forceinline__ double wg_exp_tab(double x) {
  const double sh = fma(x, __longlong_as_double((long long)WG_EXP_INVL), 6755399441055744.0);
  const int k = __double2loint(sh);
  const double kf = sh - 6755399441055744.0;
  double r = fma(kf, -__longlong_as_double((long long)WG_EXP_L2HI), x);
  r = fma(kf, -__longlong_as_double((long long)WG_EXP_L2LO), r);
  const double2 t = reinterpret_cast<const double2*>(wg_exp_s)[k & (WG_EXP_N - 1)];
  const int e = k >> 6;
  double q = fma(1.0 / 720.0, r, 1.0 / 120.0);
  q = fma(q, r, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  const double p = fma(r * r, q, r);
  const double y = t.x + fma(t.x, p, t.y);
  double res = __hiloint2double(__double2hiint(y) + (e << 20), __double2loint(y));
  const int ahi = __double2hiint(x) & 0x7fffffff;
  if (__builtin_expect(ahi >= 0x4086232B, 0)) {          // |x| >= 708.39: over/underflow or subnormal
    res = (x < 0.0) ? 0.0 : x + __longlong_as_double(0x7FF0000000000000LL);
    if (ahi < 0x40874911) {                             // |x| <~ 745.1332 (glibc's smallest subnormal result): scale in two steps
      const int e1 = e / 2;
      const double y1 = __hiloint2double(__double2hiint(y) + (e1 << 20), __double2loint(y));
      res = y1 * __hiloint2double(((e - e1) << 20) + 0x3FF00000, 0);
    }
  }
  return res;
}

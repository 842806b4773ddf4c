"""The hand-written onesweep radix sort and run-head compaction
(csrc/wg_radix.cuh) behind the keyed builders' result():

  wg_sort_pairs     order_key sort of dict / sort() keys (builders.py:496-507,
                    run.py:723-747): stable, any bit window
  wg_run_starts     run heads of sorted multi-word keys
  wg_group_finish1  GroupBuilderState.result (builders.py:478-493): sorted
                    unique keys, offsets, values in per-key input order

Each is checked bit-exactly against numpy's stable sort (kind="stable") on
edge sizes around the 4096-row tile, skewed and constant keys, and every
code path of wg_group_finish1 (u32 window, 64-bit window + bucket fix-up,
skewed-bucket full re-sort, narrow range straddling zero, 4-byte values)."""
import ctypes
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [1, 2, 255, 4095, 4096, 4097, 100_003, 1 << 20]


def _dev(a):
    from paper_1709_06416_b200 import runtime as rt
    a = np.ascontiguousarray(a)
    b = rt.alloc(max(a.nbytes, 1))
    if a.nbytes:
        rt.h2d(b.ptr, a.ctypes.data, a.nbytes)
    return b


def _host(b, n, dt):
    from paper_1709_06416_b200 import runtime as rt
    out = np.empty(n, dtype=dt)
    if n:
        rt.d2h(out.ctypes.data, b.ptr, out.nbytes)
    return out


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("window", [(0, 64), (0, 8), (8, 40), (60, 64), (0, 13)])
def test_sort_pairs_stable(n, window):
    from paper_1709_06416_b200 import runtime as rt
    rng = np.random.default_rng(n * 131 + window[0])
    k = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    if n > 1000:
        k[: n // 3] = k[n // 2]        # a heavy duplicate run
    v = np.arange(n, dtype=np.uint32)
    lo, hi = window
    kd, vd = _dev(k), _dev(v)
    ko, vo = rt.alloc(8 * n), rt.alloc(4 * n)
    rt.call("wg_sort_pairs", kd.ptr, vd.ptr, ko.ptr, vo.ptr, n, lo, hi)
    sub = (k >> np.uint64(lo)) & np.uint64((1 << (hi - lo)) - 1 if hi - lo < 64 else 0xFFFFFFFFFFFFFFFF)
    order = np.argsort(sub, kind="stable")
    np.testing.assert_array_equal(_host(vo, n, np.uint32), v[order])
    np.testing.assert_array_equal(_host(ko, n, np.uint64), k[order])
    # inputs untouched
    np.testing.assert_array_equal(_host(kd, n, np.uint64), k)


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("kw", [1, 2])
def test_run_starts(n, kw):
    from paper_1709_06416_b200 import runtime as rt
    rng = np.random.default_rng(n + kw)
    words = [np.sort(rng.integers(0, max(2, n // 7), n)).astype(np.uint64)]
    if kw == 2:
        words.append(rng.integers(0, 2, n).astype(np.uint64))
        order = np.lexsort([words[1], words[0]])
        words = [w[order] for w in words]
    bufs = [_dev(w) for w in words]
    starts = rt.alloc(4 * n)
    nr = ctypes.c_uint64(0)
    ptrs = (ctypes.c_uint64 * kw)(*[b.ptr for b in bufs])
    rt.call("wg_run_starts", ptrs, kw, n, starts.ptr, ctypes.byref(nr))
    same = np.ones(n, dtype=bool)
    same[0] = False
    for w in words:
        same[1:] &= w[1:] == w[:-1]
    want = np.flatnonzero(~same).astype(np.uint32)
    assert nr.value == want.size
    np.testing.assert_array_equal(_host(starts, nr.value, np.uint32), want)


def _group(keys, vals):
    """wg_group_finish1 -> (unique keys, offsets, values)."""
    from paper_1709_06416_b200 import runtime as rt
    from paper_1709_06416_b200.irtypes import KIND_CODE, I32, I64, BOOL
    kind = {np.dtype(np.int64): I64, np.dtype(np.int32): I32, np.dtype(np.uint8): BOOL}[keys.dtype]
    n = keys.size
    kd, vd = _dev(keys), _dev(vals)
    uk, offs, vo = rt.alloc(max(n, 1) * keys.itemsize), rt.alloc(8 * (n + 1)), rt.alloc(max(n, 1) * vals.itemsize)
    K = ctypes.c_uint64(0)
    rt.call("wg_group_finish1", kd.ptr, KIND_CODE[kind], vd.ptr, vals.itemsize, n, uk.ptr, offs.ptr, vo.ptr,
            ctypes.byref(K))
    K = K.value
    return _host(uk, K, keys.dtype), _host(offs, K + 1, np.int64), _host(vo, n, vals.dtype)


def _group_want(keys, vals):
    order = np.argsort(keys, kind="stable")
    sk = keys[order]
    n = keys.size
    if n == 0:
        return sk, np.zeros(1, dtype=np.int64), vals
    head = np.ones(n, dtype=bool)
    head[1:] = sk[1:] != sk[:-1]
    st = np.flatnonzero(head)
    return sk[st], np.r_[st, n].astype(np.int64), vals[order]


CASES = {
    # 10M-style scrambled 64-bit keys: 64-bit window + bucket fix-up
    "scrambled64": lambda rng, n: (rng.integers(0, max(1, n // 20), n).astype(np.uint64)
                                   * np.uint64(0x9E3779B97F4A7C15)).view(np.int64),
    # ids < 2^32 apart: u32 window path
    "ids": lambda rng, n: rng.integers(0, max(1, n // 20), n).astype(np.int64),
    # narrow range around zero: okey - min path
    "around_zero": lambda rng, n: rng.integers(-1000, 1000, n).astype(np.int64),
    # one key
    "constant": lambda rng, n: np.full(n, -7, dtype=np.int64),
    "i32": lambda rng, n: rng.integers(-(1 << 31), (1 << 31) - 1, n).astype(np.int32),
    "bool": lambda rng, n: rng.integers(0, 2, n).astype(np.uint8),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("n", [0, 1, 4097, 300_001])
@pytest.mark.parametrize("vdt", [np.int64, np.int32])
def test_group_finish(case, n, vdt):
    rng = np.random.default_rng(zlib.crc32(f"{case}{n}".encode()))
    keys = CASES[case](rng, n)
    vals = rng.integers(-(1 << 31), (1 << 31) - 1, n).astype(vdt)
    got = _group(keys, vals)
    want = _group_want(keys, vals)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)


def test_group_finish_skewed_buckets_full_resort():
    """Keys that agree on their top 32 varying bits in large buckets whose
    low bits are disordered: the bucket fix-up overflows (bucket > 512 rows)
    and the full stable re-sort runs."""
    rng = np.random.default_rng(5)
    n = 200_000
    hi = rng.integers(0, 4, n).astype(np.int64) << np.int64(50)
    lo = rng.integers(0, 1 << 18, n).astype(np.int64)
    keys = hi | lo
    vals = np.arange(n, dtype=np.int64)
    got = _group(keys, vals)
    want = _group_want(keys, vals)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)

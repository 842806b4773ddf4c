"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's builder semantics for the five
benchmark programs (paper_1709_06416_b200/workloads.py), used to check the
GPU executor at sizes the reference engine cannot reach in seconds.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker -- never as the thing measured or
shipped.

Pinned: tests/test_oracle.py checks every function here against
tests/golden/configs.json, which holds outputs of the reference engine
itself (weldmill.engine.evaluate, /root/reference/pkg/src/weldmill/engine/
run.py:1008) on the same generator rows (tests/golden/make_golden.py).

Semantics restated (reference file:line):
  merger fold, f64 '+'           engine/builders.py:286-328, 121-163
  vecbuilder order               engine/builders.py:274-283
  dictmerger keyed fold + sort   engine/builders.py:331-392, 496-507
  groupbuilder per-key order     engine/builders.py:453-493
  vecmerger fold-at-index        engine/builders.py:395-450
  tovec                          engine/run.py:737-747
"""
from __future__ import annotations

import numpy as np


def q6(c):
    """result(for({shipdate, discount, quantity, price}, merger[f64,+], ...))"""
    sd, disc, qty, price = c["shipdate"], c["discount"], c["quantity"], c["price"]
    mask = (sd >= 8766) & (sd < 9131) & (disc >= 0.05) & (disc <= 0.07) & (qty < 24.0)
    return float(np.sum(np.where(mask, price * disc, 0.0)))


def blackscholes(c):
    """Two vecbuilder[f64] appends per row, in row order (builders.py:274-283)."""
    from scipy.special import erf
    s, k, t, r, v = c["s"], c["k"], c["t"], c["r"], c["v"]
    sq = np.sqrt(t)
    d1 = (np.log(s / k) + (r + 0.5 * v * v) * t) / (v * sq)
    d2 = d1 - v * sq
    df = np.exp(0.0 - r * t)
    nd1 = 0.5 * (1.0 + erf(d1 * 0.7071067811865476))
    nd2 = 0.5 * (1.0 + erf(d2 * 0.7071067811865476))
    call = s * nd1 - k * df * nd2
    put = k * df * (1.0 - nd2) - s * (1.0 - nd1)
    return call, put


def q1(c):
    """dictmerger[{i32,i32},{f64 x5, i64},+] then tovec (sorted by key)."""
    mask = c["shipdate"] <= 10471
    rf = c["returnflag"][mask].astype(np.int64)
    ls = c["linestatus"][mask].astype(np.int64)
    qty = c["quantity"][mask]
    price = c["price"][mask]
    disc = c["discount"][mask]
    tax = c["tax"][mask]
    key = rf * (1 << 32) + ls
    uk, inv = np.unique(key, return_inverse=True)
    dp = price * (1.0 - disc)
    ch = price * (1.0 - disc) * (1.0 + tax)
    out = []
    for j, kk in enumerate(uk):
        m = inv == j
        out.append(((int(kk >> 32), int(kk & 0xFFFFFFFF)),
                    (float(qty[m].sum()), float(price[m].sum()), float(dp[m].sum()), float(ch[m].sum()),
                     float(disc[m].sum()), int(m.sum()))))
    return out


def dict_sum(c):
    """dictmerger[i64,i64,+] then tovec: exact integer sums per key, key order.
    Returns (keys, sums) arrays."""
    k, v = c["k"], c["v"]
    order = np.argsort(k, kind="stable")
    ks = k[order]
    vs = v[order]
    if ks.size == 0:
        return ks, vs
    starts = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
    sums = np.add.reduceat(vs, starts)
    return ks[starts], sums


def group(c):
    """groupbuilder[i64,i64] then tovec: keys sorted; values per key in input
    order.  Returns (keys, offsets, values)."""
    k, v = c["k"], c["v"]
    order = np.argsort(k, kind="stable")
    ks = k[order]
    vs = v[order]
    if ks.size == 0:
        return ks, np.zeros(1, dtype=np.int64), vs
    starts = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
    offs = np.r_[starts, ks.size].astype(np.int64)
    return ks[starts], offs, vs


def hist(c):
    """vecmerger[f64,+](bins): bins[idx] += w, bounds-checked."""
    idx, w, bins = c["idx"], c["w"], c["bins"]
    if idx.size and (idx.min() < 0 or idx.max() >= bins.size):
        raise IndexError("vecmerger index out of range")
    return bins + np.bincount(idx, weights=w, minlength=bins.size)


def filt(c):
    """filter(v, x > 0): vecbuilder appends in row order (builders.py:274-283)."""
    v = c["v"]
    return v[v > 0]


def map3(c):
    """map(v, x * 3 + 1) with i64 wraparound (run.py:395-405)."""
    with np.errstate(over="ignore"):
        return c["v"] * np.int64(3) + np.int64(1)


ORACLES = {"q6": q6, "blackscholes": blackscholes, "q1": q1, "dict": dict_sum, "group": group, "hist": hist,
           "filter": filt, "map": map3}


def as_reference_payload(name, out):
    """Oracle output in the reference's payload form (lists/tuples)."""
    if name == "q6":
        return out
    if name == "blackscholes":
        return [out[0].tolist(), out[1].tolist()]
    if name == "q1":
        return [[list(k), list(v)] for k, v in out]
    if name == "dict":
        return [[int(a), int(b)] for a, b in zip(*out)]
    if name == "group":
        ks, offs, vs = out
        return [[int(kk), vs[offs[j]:offs[j + 1]].tolist()] for j, kk in enumerate(ks)]
    if name == "hist":
        return [[i, x] for i, x in enumerate(out.tolist()) if x != 0.0]
    if name in ("filter", "map"):
        return out.tolist()
    raise KeyError(name)

"""The benchmark programs (BASELINE.json ``configs``)
and their counter-based synthetic columns.

Each input column is a pure function of (seed, column id, row):
    h = splitmix64(seed ^ (col << 56) ^ row),  u = (h >> 11) * 2^-53
so any row range can be generated independently on the host (numpy, for the
oracle and parity tests) or on the device (libweldgpu wg_gen_column, for
full-size runs), and both produce identical bits.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _ref  # noqa: F401
from weldmill.optim import OptLevel, optimize
from weldmill.parser import parse, parse_type_text
from weldmill.sugar import expand
from weldmill.typecheck import check_linearity, infer
from weldmill.types import F64, Function, Scalar

SEED = 20261017
MASK = np.uint64(0xFFFFFFFFFFFFFFFF)


@dataclass
class ColSpec:
    name: str
    ty: str           # "i32" | "i64" | "f64"
    dist: int         # 0 int uniform, 1 float uniform, 2 int/div, 3 key scatter, 4 categorical
    col: int
    lo: int = 0
    span: int = 1
    flo: float = 0.0
    fhi: float = 1.0
    div: float = 1.0
    cum: tuple = ()
    vals: tuple = ()
    mul_by: str = ""  # multiply elementwise by another column (Black-Scholes strike)


@dataclass
class Workload:
    name: str
    title: str
    program: str
    columns: list
    n: int
    bytes_per_row: int
    out_bytes: object          # callable n -> algorithmic result bytes
    externs: tuple = ()
    opt: str = "O3"
    extra_inputs: dict = field(default_factory=dict)  # name -> (type text, n) zero vectors
    dtype: str = "f64"


Q6_PROGRAM = ("result(for({shipdate, discount, quantity, price}, merger[f64, +], (b, i, x) => "
              "if (x.0 >= 8766 && x.0 < 9131 && x.1 >= 0.05 && x.1 <= 0.07 && x.2 < 24.0, "
              "merge(b, x.3 * x.1), b)))")

BS_PROGRAM = ("result(for({s, k, t, r, v}, {vecbuilder[f64], vecbuilder[f64]}, (b, i, x) => "
              "sq := call(sqrt, x.2); "
              "d1 := (call(log, x.0 / x.1) + (x.3 + 0.5 * x.4 * x.4) * x.2) / (x.4 * sq); "
              "d2 := d1 - x.4 * sq; "
              "df := call(exp, 0.0 - x.3 * x.2); "
              "nd1 := 0.5 * (1.0 + call(erf, d1 * 0.7071067811865476)); "
              "nd2 := 0.5 * (1.0 + call(erf, d2 * 0.7071067811865476)); "
              "{merge(b.0, x.0 * nd1 - x.1 * df * nd2), merge(b.1, x.1 * df * (1.0 - nd2) - x.0 * (1.0 - nd1))}))")

Q1_PROGRAM = ("tovec(result(for({returnflag, linestatus, quantity, price, discount, tax, shipdate}, "
              "dictmerger[{i32, i32}, {f64, f64, f64, f64, f64, i64}, +], (b, i, x) => "
              "if (x.6 <= 10471, merge(b, {{x.0, x.1}, {x.2, x.3, x.3 * (1.0 - x.4), "
              "x.3 * (1.0 - x.4) * (1.0 + x.5), x.4, 1}}), b))))")

DICT_PROGRAM = "tovec(result(for({k, v}, dictmerger[i64, i64, +], (b, i, x) => merge(b, {x.0, x.1}))))"
GROUP_PROGRAM = "tovec(result(for({k, v}, groupbuilder[i64, i64], (b, i, x) => merge(b, {x.0, x.1}))))"
HIST_PROGRAM = "result(for({idx, w}, vecmerger[f64, +](bins), (b, i, x) => merge(b, {x.0, x.1})))"
# Appender scans measured on their own: an order-preserving
# filter (scan schedule: decoupled look-back) and a size-hinted map (DIRECT).
FILTER_PROGRAM = "filter(v, (x) => x > 0)"
MAP_PROGRAM = "map(v, (x) => x * 3 + 1)"

_Q1_CUM = (0.25, 0.26, 0.75, 1.0)

WORKLOADS = {
    "q6": Workload(
        "q6", "TPC-H Q6 filter+map+merger[f64,+]", Q6_PROGRAM,
        [ColSpec("shipdate", "i32", 0, 0, lo=8036, span=10561 - 8036 + 1),
         ColSpec("discount", "f64", 2, 1, lo=0, span=11, div=100.0),
         ColSpec("quantity", "f64", 2, 2, lo=1, span=50, div=1.0),
         ColSpec("price", "f64", 2, 3, lo=90000, span=10494950 - 90000 + 1, div=100.0)],
        n=1_000_000, bytes_per_row=28, out_bytes=lambda n: 8),
    "blackscholes": Workload(
        "blackscholes", "Black-Scholes via two appenders", BS_PROGRAM,
        [ColSpec("s", "f64", 1, 0, flo=10.0, fhi=100.0),
         ColSpec("k", "f64", 1, 1, flo=0.9, fhi=1.1, mul_by="s"),
         ColSpec("t", "f64", 1, 2, flo=0.1, fhi=2.0),
         ColSpec("r", "f64", 1, 3, flo=0.01, fhi=0.05),
         ColSpec("v", "f64", 1, 4, flo=0.1, fhi=0.5)],
        n=64 * 1024 * 1024, bytes_per_row=56, out_bytes=lambda n: 0,
        externs=("sqrt", "log", "exp", "erf"), opt="none"),
    "q1": Workload(
        "q1", "TPC-H Q1 dictmerger (4 groups)", Q1_PROGRAM,
        [ColSpec("returnflag", "i32", 4, 0, cum=_Q1_CUM, vals=(0, 1, 1, 2)),
         ColSpec("linestatus", "i32", 4, 0, cum=_Q1_CUM, vals=(0, 0, 1, 0)),
         ColSpec("quantity", "f64", 2, 2, lo=1, span=50, div=1.0),
         ColSpec("price", "f64", 2, 3, lo=90000, span=10494950 - 90000 + 1, div=100.0),
         ColSpec("discount", "f64", 2, 1, lo=0, span=11, div=100.0),
         ColSpec("tax", "f64", 2, 5, lo=0, span=9, div=100.0),
         ColSpec("shipdate", "i32", 0, 6, lo=8036, span=10561 - 8036 + 1)],
        n=60_000_000, bytes_per_row=44, out_bytes=lambda n: 4 * 56),
    "dict": Workload(
        "dict", "high-cardinality dictmerger[i64,i64,+] (10M keys)", DICT_PROGRAM,
        [ColSpec("k", "i64", 3, 0, lo=0, span=10_000_000),
         ColSpec("v", "i64", 0, 1, lo=-1000, span=2001)],
        n=200_000_000, bytes_per_row=16, out_bytes=lambda n: 10_000_000 * 16, dtype="i64"),
    "group": Workload(
        "group", "high-cardinality groupbuilder[i64,i64] (10M keys)", GROUP_PROGRAM,
        [ColSpec("k", "i64", 3, 0, lo=0, span=10_000_000),
         ColSpec("v", "i64", 0, 1, lo=-1000, span=2001)],
        n=200_000_000, bytes_per_row=16, out_bytes=lambda n: 10_000_000 * 16 + n * 8, dtype="i64"),
    "hist": Workload(
        "hist", "vecmerger[f64,+] histogram into 1M bins", HIST_PROGRAM,
        [ColSpec("idx", "i64", 0, 0, lo=0, span=1_000_000),
         ColSpec("w", "f64", 1, 1, flo=0.0, fhi=1.0)],
        n=1_000_000_000, bytes_per_row=16, out_bytes=lambda n: 16_000_000,
        extra_inputs={"bins": ("vec[f64]", 1_000_000)}),
    "filter": Workload(
        "filter", "appender scan: order-preserving filter over i64 (~50% selectivity)", FILTER_PROGRAM,
        [ColSpec("v", "i64", 0, 0, lo=-1000, span=2001)],
        n=500_000_000, bytes_per_row=8, out_bytes=lambda n: n * 4, dtype="i64"),
    "map": Workload(
        "map", "appender scan: size-hinted map over i64", MAP_PROGRAM,
        [ColSpec("v", "i64", 0, 0, lo=-1000, span=2001)],
        n=500_000_000, bytes_per_row=16, out_bytes=lambda n: 0, dtype="i64"),
}


def input_types(wl: Workload):
    env = {c.name: parse_type_text(f"vec[{c.ty}]") for c in wl.columns}
    for name, (tt, _) in wl.extra_inputs.items():
        env[name] = parse_type_text(tt)
    return env


def compile_program(wl: Workload, program=None):
    """Front end (reference): parse -> expand -> infer -> linearity -> optimize.
    Black-Scholes types its externs and skips the optimizer (BASELINE.md:
    any firing pass on a call(...) program crashes the recheck)."""
    env = input_types(wl)
    for name in wl.externs:
        env[name] = Function((Scalar(F64),), Scalar(F64))
    typed = infer(expand(parse(program or wl.program)), env)
    check_linearity(typed)
    level = OptLevel.none() if wl.opt == "none" else None
    return optimize(typed, level)[0]


def externs_for(wl: Workload):
    import math
    return {name: getattr(math, name) for name in wl.externs}


# ---------------------------------------------------------------------------
# host generator (numpy; identical bits to k_gen in libweldgpu)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def host_column(c: ColSpec, n: int, row0: int = 0, seed: int = SEED, cols=None):
    rows = np.arange(row0, row0 + n, dtype=np.uint64)
    h = splitmix64(np.uint64(seed) ^ (np.uint64(c.col) << np.uint64(56)) ^ rows)
    u = (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    if c.dist == 0:
        v = np.int64(c.lo) + (h % np.uint64(c.span)).astype(np.int64)
    elif c.dist == 3:
        v = splitmix64((np.int64(c.lo) + (h % np.uint64(c.span)).astype(np.int64)).astype(np.uint64)).view(np.int64)
    elif c.dist == 4:
        v = np.full(n, c.vals[-1], dtype=np.int64)
        done = np.zeros(n, dtype=bool)
        for cum, val in zip(c.cum, c.vals):
            hit = (~done) & (u < cum)
            v[hit] = val
            done |= hit
    elif c.dist == 1:
        v = c.flo + u * (c.fhi - c.flo)
    else:
        v = (np.int64(c.lo) + (h % np.uint64(c.span)).astype(np.int64)).astype(np.float64) / c.div
    if c.mul_by and cols is not None:
        v = v * cols[c.mul_by]
    dt = {"i32": np.int32, "i64": np.int64, "f64": np.float64}[c.ty]
    return np.ascontiguousarray(v.astype(dt))


def host_columns(wl: Workload, n: int, row0: int = 0, seed: int = SEED):
    out = {}
    for c in wl.columns:
        out[c.name] = host_column(c, n, row0, seed, out)
    for name, (tt, m) in wl.extra_inputs.items():
        out[name] = np.zeros(m, dtype=np.float64)
    return out


# ---------------------------------------------------------------------------
# device generator


def device_columns(wl: Workload, n: int, row0: int = 0, seed: int = SEED):
    from . import runtime as rt
    from .columns import Col, dvec_from_cols
    from weldmill.types import Vec
    out = {}
    for c in wl.columns:
        kind = c.ty
        col = Col.alloc(kind, n)
        width = 4 if kind == "i32" else 8
        ncat = len(c.cum)
        cum = (ctypes.c_double * 8)(*(list(c.cum) + [0.0] * (8 - ncat)))
        vals = (ctypes.c_int64 * 8)(*(list(c.vals) + [0] * (8 - ncat)))
        rt.call("wg_gen_column", col.ptr, n, row0, c.dist, width, seed, c.col, c.lo, c.span, c.flo, c.fhi, c.div,
                ncat, cum, vals)
        if c.mul_by:
            rt.call("wg_mul_inplace_f64", col.ptr, out[c.mul_by].cols[0].ptr, n)
        out[c.name] = dvec_from_cols(Scalar(kind), n, [col])
    for name, (tt, m) in wl.extra_inputs.items():
        col = Col.alloc("f64", m)
        rt.memset(col.ptr, 0, 8 * m)
        out[name] = dvec_from_cols(Scalar("f64"), m, [col])
    return out


def algorithmic_bytes(wl: Workload, n: int) -> int:
    """Compulsory bytes per launch: column reads + results."""
    extra = 0
    if wl.name == "hist":
        extra = 2 * 8 * 1_000_000  # init read + bins written
        return n * wl.bytes_per_row + extra
    if wl.name in ("blackscholes", "map"):
        return n * wl.bytes_per_row
    if wl.name == "filter":
        return n * 8 + n * 4          # read every row, write the ~50% kept (8 B each)
    if wl.name in ("dict", "group"):
        distinct = min(n, 10_000_000)
        out = distinct * 16 + (n * 8 if wl.name == "group" else 0)
        return n * wl.bytes_per_row + out
    return n * wl.bytes_per_row + wl.out_bytes(n)

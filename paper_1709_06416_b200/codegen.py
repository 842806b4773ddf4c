"""Lower one fused outer ``for`` loop to an sm_100a CUDA kernel.

Replaces the reference's closure compiler and loop runner
(/root/reference/pkg/src/weldmill/engine/run.py:560-983): instead of one
Python closure per IR node executed per row, the loop body becomes straight
C++ inside a hand-written kernel skeleton, compiled once by NVRTC.

Kernel skeleton (one CTA = 256 threads; a tile = 256 x ITEMS iterations,
each thread owning ITEMS *consecutive* iterations so every column is read
with 16-byte vector loads):

  * static schedule  -- grid-stride over tiles with a persistent grid of
    (#SM x occupancy) CTAs; used when no builder needs ordered output.
  * scan schedule    -- tiles claimed through an atomic counter; each tile
    runs the body once to *count* appends per thread (phase A, which also
    performs every order-insensitive merge), computes the tile's output
    offset with a block scan + single-pass decoupled look-back, then runs
    the body again to *store* appends (phase B).  Column values stay in
    registers between the phases, so HBM traffic is read-once.

Per builder (reference state classes in engine/builders.py):
  merger      (:286-328) per-thread register fold -> block tree fold ->
              per-CTA partial -> last CTA folds partials in fixed order
  vecbuilder  (:231-283) DIRECT(k) when every path merges exactly k values
              (out[i*k + c], vector stores); otherwise SCAN(M) above
  groupbuilder(:453-493) appended {key, value} pairs in iteration order;
              result() stable-sorts by key (builders_dev.py)
  dictmerger  (:331-392) open-addressing table in HBM, key claim by CAS,
              per-field atomic fold; shared-memory privatised table for
              low-cardinality keys (strategy local/shared)
  vecmerger   (:395-450) bounds-checked atomic fold at index; shared-memory
              privatised bins when they fit (strategy local/shared)
"""
from __future__ import annotations

import math
import re
import struct as _struct
from dataclasses import dataclass, field

from . import _ref  # noqa: F401
from weldmill.expr import (
    BinaryOp, BitSelect, Broadcast, CastScalar, ExternCall, FieldAccess, For, Ident, If, Lambda, Len, Let,
    Literal, Lookup, MakeStruct, MakeVector, Merge, NewBuilder, Result, UnaryOp,
)

from .irtypes import (
    BOOL, CTYPE, F32, F64, FLOAT_KINDS, I32, I64, INT_KINDS, OPCODE, OPSTRUCT, SIZE, STYPE, Builder, DeviceUnsupported,
    Dict, DictMerger, Function, GroupBuilder, Merger, Scalar, Simd, Struct, Vec, VecBuilder, VecMerger, identity_value,
    internal_identity, leaves,
)

W = 4  # SIMD_WIDTH (types.py:15)
BLOCK = 256
BLOCK_DEFAULT = int(__import__("os").environ.get("WELDGPU_BLOCK", str(BLOCK)))

import os as _os

# Tuning knobs (defaults chosen from ncu measurements).
PREFETCH = _os.environ.get("WELDGPU_PREFETCH", "1") == "1"
MINBLOCKS = int(_os.environ.get("WELDGPU_MINBLOCKS", "0"))
ITEMS_OVERRIDE = int(_os.environ.get("WELDGPU_ITEMS", "0"))
DEFER_DICT = _os.environ.get("WELDGPU_DEFER_DICT", "1") == "1"
AGG_MAX_GROUPS = int(_os.environ.get("WELDGPU_AGG_GROUPS", "8"))
REGCACHE = int(_os.environ.get("WELDGPU_REGCACHE", "4"))
PIPE = _os.environ.get("WELDGPU_PIPE", "1") == "1"
STAGE_SCAN = _os.environ.get("WELDGPU_STAGE_SCAN", "1") == "1"
LB_PER = int(_os.environ.get("WELDGPU_LB_PER", "1"))
LB_SLEEP = int(_os.environ.get("WELDGPU_LB_SLEEP", "64"))
# scan schedule: claim the next tile during the current tile's store phase
# instead of at the top of the next iteration (one barrier and one exposed
# atomic round trip less per tile)
SCAN_EARLY_CLAIM = _os.environ.get("WELDGPU_SCAN_EARLY_CLAIM", "1") == "1"
SCAN_MINBLOCKS = int(_os.environ.get("WELDGPU_SCAN_MINBLOCKS", "4"))   # in 256-thread CTAs per SM
PART_ITEMS = int(_os.environ.get("WELDGPU_PART_ITEMS", "8"))
PIPE_STAGES = int(_os.environ.get("WELDGPU_PIPE_STAGES", "4"))
# warp-specialised scan schedule: the compute warps publish each tile's
# aggregate and stage its appends, one extra warp resolves the look-back and
# stores the tile; WS_NBUF staging buffers decouple the two
SCAN_WS = _os.environ.get("WELDGPU_SCAN_WS", "1") == "1"
WS_NBUF = int(_os.environ.get("WELDGPU_WS_NBUF", "2"))
# 256-bit (sm_100) per-thread column loads / stores in wg_load_contig / wg_store_contig
LD256 = int(_os.environ.get("WELDGPU_LD256", "1"))
ST256 = int(_os.environ.get("WELDGPU_ST256", "1"))
WS_MINB = int(_os.environ.get("WELDGPU_WS_MINB", "3"))
WS_BLOCK = int(_os.environ.get("WELDGPU_WS_BLOCK", "384"))     # compute threads (+ the store warp)
WS_ITEMS = int(_os.environ.get("WELDGPU_WS_ITEMS", "8"))
PIPE_NOGUARD = _os.environ.get("WELDGPU_PIPE_NOGUARD", "1") == "1"
PIPE_MAX_STAGES = 8
PIPE_SMEM_BUDGET = int(_os.environ.get("WELDGPU_PIPE_SMEM", str(48 * 1024)))

# Extern names recognised as device intrinsics (the reference resolves
# `call(name, ...)` through a host registry, run.py:832-846).
EXTERN_F64 = {
    "exp": "exp", "log": "log", "sqrt": "sqrt", "erf": "erf", "erfc": "erfc", "sin": "sin", "cos": "cos",
    "tan": "tan", "tanh": "tanh", "sinh": "sinh", "cosh": "cosh", "asin": "asin", "acos": "acos",
    "atan": "atan", "fabs": "fabs", "log1p": "log1p", "expm1": "expm1", "log2": "log2", "log10": "log10",
    "cbrt": "cbrt", "exp2": "exp2", "atan2": "atan2", "pow": "pow", "hypot": "hypot", "copysign": "copysign",
    "fmod": "fmod",
}
EXTERN_IDS = {name: q for q, name in enumerate(sorted(EXTERN_F64))}


def _extern_checks(name, a, r):
    """C conditions under which Python's math.<name> raises for these
    arguments / this result: [(condition, 1 if OverflowError else 0)]."""
    x = a[0]
    y = a[1] if len(a) > 1 else None
    fin = lambda v: f"isfinite({v})"   # noqa: E731
    if name in ("exp", "exp2", "expm1", "sinh", "cosh"):
        return [(f"isinf({r}) && {fin(x)}", 1)]
    if name in ("log", "log2", "log10"):
        return [(f"{x} <= 0.0", 0)]
    if name == "log1p":
        return [(f"{x} <= -1.0", 0)]
    if name == "sqrt":
        return [(f"{x} < 0.0", 0)]
    if name in ("sin", "cos", "tan"):
        return [(f"isinf({x})", 0)]
    if name in ("asin", "acos"):
        return [(f"fabs({x}) > 1.0", 0)]
    if name == "pow":
        return [(f"(isnan({r}) && !isnan({x}) && !isnan({y})) || ({x} == 0.0 && {y} < 0.0 && {fin(y)})", 0),
                (f"isinf({r}) && {fin(x)} && {fin(y)} && {x} != 0.0", 1)]
    if name == "hypot":
        return [(f"isinf({r}) && {fin(x)} && {fin(y)}", 1)]
    if name == "fmod":
        return [(f"({y} == 0.0 && !isnan({x})) || (isinf({x}) && !isnan({y}))", 0)]
    return []


# static shared-memory bytes of each table-driven math function
# (weld_device.cuh: wg_erf_s 97 x 20 u32, wg_log_s + wg_log_lo_s 3 x 128 f64,
# wg_exp_s 2 x 64 f64)
TAB_BYTES = {"wg_erf_tab": 97 * 20 * 4, "wg_log_tab": 3 * 128 * 8, "wg_exp_tab": 2 * 64 * 8}


def _table_bytes(body):
    from weldmill.expr import walk
    fns = {EXTERN_F64.get(n.name) for n in walk(body) if isinstance(n, ExternCall)}
    return sum(TAB_BYTES.get(f, 0) for f in fns)


def extern_error_text(info):
    """Message of the EvalError a device extern failure raises (the
    reference: f"extern {name!r} failed: {exc}", run.py:843-844)."""
    names = sorted(EXTERN_F64)
    name = names[info // 2] if 0 <= info // 2 < len(names) else "?"
    return f"extern {name!r} failed: math {'range' if info % 2 else 'domain'} error"


# WELDGPU_MATH: "tab" (default) -- erf, log and exp from shared-memory
# tables (weld_device.cuh wg_erf_tab / wg_log_tab / wg_exp_tab: 11, 20 and
# 12 FP64 ops instead of libdevice's ~43, ~30 and 15); "taberf" -- erf only;
# "libdevice" -- CUDA's own.
MATH = _os.environ.get("WELDGPU_MATH", "tab")
if MATH == "tab":
    EXTERN_F64.update({"erf": "wg_erf_tab", "log": "wg_log_tab", "exp": "wg_exp_tab"})
elif MATH == "taberf":
    EXTERN_F64.update({"erf": "wg_erf_tab"})


# ---------------------------------------------------------------------------
# Values during code generation


class S:
    """A scalar C expression of an IR scalar kind."""
    __slots__ = ("c", "kind")

    def __init__(self, c, kind):
        self.c = c
        self.kind = kind


class T:
    """A struct value: tuple of field values."""
    __slots__ = ("items",)

    def __init__(self, items):
        self.items = list(items)


class Lanes:
    """A simd value: W lane scalars."""
    __slots__ = ("lanes", "kind")

    def __init__(self, lanes, kind):
        self.lanes = list(lanes)
        self.kind = kind


class VRef:
    """A loop-invariant device vector visible inside the body."""
    __slots__ = ("cols", "n", "elem")

    def __init__(self, cols, n, elem):
        self.cols = cols  # C pointer expressions, one per leaf
        self.n = n        # C expression for the length
        self.elem = elem


class DRef:
    """A loop-invariant finalised dictionary visible inside the body: key
    leaf columns sorted by order_key (builders.py:496-507), value leaf
    columns (dictmerger) or offsets + value columns (groupbuilder)."""
    __slots__ = ("kcols", "vcols", "offs", "n", "kty", "vty")

    def __init__(self, kcols, vcols, offs, n, kty, vty):
        self.kcols, self.vcols, self.offs, self.n, self.kty, self.vty = kcols, vcols, offs, n, kty, vty


class SVec:
    """A small vector literal built inside the body (registers)."""
    __slots__ = ("items", "elem", "node")

    def __init__(self, items, elem, node=None):
        self.items = list(items)
        self.elem = elem
        self.node = node


class BRef:
    """A reference to a builder (outer, by id) or a body-local merger."""
    __slots__ = ("b",)

    def __init__(self, b):
        self.b = b


class BTuple:
    __slots__ = ("items",)

    def __init__(self, items):
        self.items = list(items)


# ---------------------------------------------------------------------------
# Loop specification handed over by the executor


@dataclass
class IterSpec:
    elem: object          # element IR type (flat)
    simd: bool
    strided: bool         # explicit start/stride window (non-contiguous)
    kinds: list = field(default_factory=list)
    aligned: bool = True  # every column pointer 16-byte aligned (bulk copies)


@dataclass(eq=False)
class BSpec:
    """One outer builder as seen by the kernel."""
    bid: int
    kind: object                  # weldmill BuilderKind
    mode: str = ""                # vec/group: direct | scan | none ; dict/vecm: global | smem
    k: int = 0                    # direct: appends per iteration; scan: max appends per iteration
    extra: dict = field(default_factory=dict)


@dataclass
class Param:
    name: str
    ctype: str
    key: tuple


@dataclass
class KernelPlan:
    source: str
    name: str
    params: list
    schedule: str                 # static | scan
    items: int
    block: int
    smem: int
    builders: list
    scan_bids: list
    merger_bids: list
    key: str = ""
    pipe_stage_bytes: int = 0
    count_nodes: list = field(default_factory=list)   # count_evals: loop-local node ordinals
    stat_nodes: list = field(default_factory=list)    # ("alloc" | "trav", node): body EvalStats events
    lit_nodes: dict = field(default_factory=dict)     # nested appender bid -> ids of literals it keeps
    seg_bids: list = field(default_factory=list)      # unhinted scan appenders with chunk offsets
    threads: int = 0                                  # launch block size (block + the store warp under SCAN_WS)


def _hex_f64(v):
    b = _struct.unpack("<Q", _struct.pack("<d", v))[0]
    return f"__longlong_as_double(0x{b:016x}LL)"


def _hex_f32(v):
    b = _struct.unpack("<I", _struct.pack("<f", v))[0]
    return f"__int_as_float(0x{b:08x})"


def c_literal(kind, v):
    if kind == BOOL:
        return "true" if v else "false"
    if kind == I64:
        return f"((i64)0x{v & 0xFFFFFFFFFFFFFFFF:016x}ULL)"
    if kind == I32:
        return f"((i32)0x{v & 0xFFFFFFFF:08x}U)"
    if kind == F64:
        return _hex_f64(float(v))
    return _hex_f32(float(v))


def key_layout(kinds):
    """Pack key leaves into 64-bit words: list of (word, shift, width)."""
    out = []
    word, pos = 0, 0
    for k in kinds:
        w = 64 if SIZE[k] == 8 else (32 if SIZE[k] == 4 else 8)
        if pos + w > 64:
            word += 1
            pos = 0
        out.append((word, pos, w))
        pos += w
    return out, word + 1


# ---------------------------------------------------------------------------


class Gen:
    def __init__(self, loop: For, iters, bstruct, captures, externs, strategy, items=None):
        self.loop = loop
        self.iters = iters
        self.bstruct = bstruct      # nested tuple/BSpec mirroring the builders value
        self.captures = captures    # name -> (IR type, runtime value)
        self.externs = externs
        self.strategy = strategy
        self.params = []
        self.pnames = set()
        self.lines = []
        self.ind = 1
        self.ntmp = 0
        self.phase = "A"
        self.local_mergers = []
        self.bspecs = []
        self._collect(bstruct)
        self.items = items
        # count_evals (EngineConfig.count_evals, run.py:544-557): every node
        # evaluation in phase A bumps a per-node device counter; the host
        # maps these loop-local ordinals back to the program's nodes
        self.counting = False
        self.count_nodes = []
        self._count_ord = {}
        # EvalStats events inside the body: literal vectors materialised
        # ("alloc") and nested loops that read at least one element ("trav")
        self.stat_nodes = []
        self._stat_ord = {}
        self.lit_nodes = {}

    # -- helpers -----------------------------------------------------------
    def _collect(self, bs):
        if isinstance(bs, BSpec):
            self.bspecs.append(bs)
        else:
            for x in bs:
                self._collect(x)

    def param(self, name, ctype, key):
        if name not in self.pnames:
            self.pnames.add(name)
            self.params.append(Param(name, ctype, key))
        return f"p.{name}"

    def emit(self, line):
        self.lines.append("  " * self.ind + line)

    def tmp(self, prefix="t"):
        self.ntmp += 1
        return f"{prefix}{self.ntmp}"

    def let(self, kind, expr):
        name = self.tmp()
        self.emit(f"const {CTYPE[kind]} {name} = {expr};")
        return S(name, kind)

    # -- expressions -------------------------------------------------------
    def stat(self, what, e, cond=None):
        if self.phase != "A":
            return
        k = self._stat_ord.get((what, id(e)))
        if k is None:
            k = self._stat_ord[(what, id(e))] = len(self.stat_nodes)
            self.stat_nodes.append((what, e))
        self.param("scnt", "unsigned long long*", ("scnt",))
        self.emit(f"wg_count(p.scnt + {k});" if cond is None else f"if ({cond}) wg_count(p.scnt + {k});")

    def ex(self, e, env):
        m = getattr(self, "ex_" + type(e).__name__, None)
        if m is None:
            raise DeviceUnsupported(f"{type(e).__name__} inside a loop body is not lowered to the device")
        if self.counting and self.phase == "A":
            k = self._count_ord.get(id(e))
            if k is None:
                k = self._count_ord[id(e)] = len(self.count_nodes)
                self.count_nodes.append(e)
            self.emit(f"wg_count(p.cnt + {k});")
        return m(e, env)

    def ex_Literal(self, e, env):
        kind = e.ty.kind
        v = e.value
        if kind == F32:
            from .irtypes import f32_round
            v = f32_round(float(v))
        return S(c_literal(kind, v), kind)

    def ex_Ident(self, e, env):
        if e.name in env:
            return env[e.name]
        raise DeviceUnsupported(f"unbound name {e.name!r} in loop body")

    def ex_Let(self, e, env):
        v = self.ex(e.value, env)
        env2 = dict(env)
        env2[e.name] = v
        return self.ex(e.body, env2)

    def ex_MakeStruct(self, e, env):
        vals = [self.ex(x, env) for x in e.items]
        if any(isinstance(v, (BRef, BTuple)) for v in vals):
            return BTuple(vals)
        return T(vals)

    def ex_FieldAccess(self, e, env):
        b = self.ex(e.base, env)
        if isinstance(b, (T, BTuple)):
            return b.items[e.ordinal]
        raise DeviceUnsupported("field access on a non-struct value")

    def ex_MakeVector(self, e, env):
        items = [self.ex(x, env) for x in e.items]
        # the reference materialises every literal it evaluates (run.py:781-789):
        # an allocation per execution, counted for EvalStats
        self.stat("alloc", e)
        return SVec(items, e.ty.elem, e)

    def ex_Broadcast(self, e, env):
        v = self.ex(e.value, env)
        return Lanes([S(v.c, v.kind)] * W, v.kind)

    def _binop_c(self, op, kind, a, b):
        if op in ("==", "!=", "<", "<=", ">", ">="):
            return f"({a} {op} {b})"
        if kind == BOOL:
            if op == "&":
                return f"({a} && {b})"
            if op == "|":
                return f"({a} || {b})"
            raise DeviceUnsupported(f"operator {op} over bool")
        if kind in INT_KINDS:
            sfx = "i64" if kind == I64 else "i32"
            if op in ("+", "-", "*"):
                return f"wg_{ {'+': 'add', '-': 'sub', '*': 'mul'}[op]}_{sfx}({a}, {b})"
            if op == "/":
                return f"wg_div_{sfx}({a}, {b}, p.err)"
            if op == "%":
                return f"wg_rem_{sfx}({a}, {b}, p.err)"
            if op in ("&", "|"):
                return f"(({CTYPE[kind]})({a} {op} {b}))"
            if op in ("min", "max"):
                return f"wg_{op}_{sfx}({a}, {b})"
        else:
            sfx = "f64" if kind == F64 else "f32"
            if op in ("+", "-", "*", "/"):
                return f"({a} {op} {b})"
            if op == "%":
                return f"wg_rem_{sfx}({a}, {b})"
            if op in ("min", "max"):
                return f"wg_{op}_{sfx}({a}, {b})"
        raise DeviceUnsupported(f"operator {op} over {kind}")

    def ex_BinaryOp(self, e, env):
        op = e.op
        if op in ("&&", "||"):
            a = self.ex(e.lhs, env)
            name = self.tmp()
            self.emit(f"bool {name} = {a.c};")
            self.emit(f"if ({'' if op == '&&' else '!'}{name}) {{")
            self.ind += 1
            b = self.ex(e.rhs, env)
            self.emit(f"{name} = {b.c};")
            self.ind -= 1
            self.emit("}")
            return S(name, BOOL)
        a = self.ex(e.lhs, env)
        b = self.ex(e.rhs, env)
        lt = e.lhs.ty
        if isinstance(lt, Simd):
            rk = BOOL if op in ("==", "!=", "<", "<=", ">", ">=") else lt.kind
            return Lanes([self.let(rk, self._binop_c(op, lt.kind, x.c, y.c)) for x, y in zip(a.lanes, b.lanes)], rk)
        rk = BOOL if op in ("==", "!=", "<", "<=", ">", ">=") else lt.kind
        return self.let(rk, self._binop_c(op, lt.kind, a.c, b.c))

    def ex_UnaryOp(self, e, env):
        v = self.ex(e.operand, env)
        t = e.operand.ty

        def one(x, kind):
            if e.op == "!":
                return self.let(BOOL, f"(!{x.c})")
            if kind in FLOAT_KINDS:
                return self.let(kind, f"(-{x.c})")
            return self.let(kind, f"wg_neg_{'i64' if kind == I64 else 'i32'}({x.c})")

        if isinstance(t, Simd):
            return Lanes([one(x, t.kind) for x in v.lanes], t.kind)
        return one(v, t.kind)

    def _cast_c(self, src, dst, a):
        if src == dst:
            return a
        if dst in INT_KINDS:
            d = "i64" if dst == I64 else "i32"
            if src == F64:
                return f"wg_f64_to_{d}({a})"
            if src == F32:
                return f"wg_f32_to_{d}({a})"
            if src == BOOL:
                return f"(({CTYPE[dst]})({a} ? 1 : 0))"
            if dst == I32:
                return f"((i32)(u32)(u64)({a}))"
            return f"((i64)({a}))"
        if dst == F64:
            if src == BOOL:
                return f"({a} ? 1.0 : 0.0)"
            return f"((double)({a}))"
        if dst == F32:
            if src == BOOL:
                return f"({a} ? 1.0f : 0.0f)"
            if src == I64:
                return f"wg_i64_to_f32({a})"
            if src == I32:
                return f"((float)(double)({a}))"
            return f"((float)({a}))"
        raise DeviceUnsupported(f"cast {src} -> {dst}")

    def ex_CastScalar(self, e, env):
        v = self.ex(e.value, env)
        src = e.value.ty
        if isinstance(src, Simd):
            return Lanes([self.let(e.kind, self._cast_c(src.kind, e.kind, x.c)) for x in v.lanes], e.kind)
        return self.let(e.kind, self._cast_c(src.kind, e.kind, v.c))

    ext_calls = 0
    tabs = frozenset()

    def ex_ExternCall(self, e, env):
        self.ext_calls += 1
        if e.name not in self.externs:
            from weldmill.errors import ExternCallUnknown
            raise ExternCallUnknown(f"no extern function {e.name!r} registered")
        fn = EXTERN_F64.get(e.name)
        if fn is None:
            from weldmill.errors import ExternCallUnknown
            raise ExternCallUnknown(f"extern {e.name!r} has no device implementation")
        reg = self.externs[e.name]
        if reg is not None and reg is not getattr(math, e.name, None):
            # the reference calls whatever callable is registered (run.py:
            # 836-844); only the math module's own functions have a device
            # implementation -- anything else is not silently replaced
            raise DeviceUnsupported(f"extern {e.name!r} is bound to {reg!r}, not math.{e.name}; "
                                    "only the math module's functions run on the device")
        args = [self.let(F64, f"(double)({a.c})") for a in self.ex_args(e.args, env)]
        rk = e.ty.kind
        cargs = ", ".join(a.c for a in args)
        if fn.endswith("_tab"):
            self.tabs = self.tabs | {fn}    # kernel prologue copies the table to shared memory
        r = self.let(F64, f"{fn}({cargs})")
        # Python's math raises where C returns NaN/inf (ValueError "math
        # domain error", OverflowError "math range error"); the reference
        # turns that into EvalError (run.py:841-844) -- so does the device
        chk = _extern_checks(e.name, [a.c for a in args], r.c)
        for cond, rng in chk:
            self.emit(f"if ({cond}) wg_raise(p.err, WG_ERR_EXTERN, {2 * EXTERN_IDS[e.name] + rng});")
        if rk == F64:
            return r
        if rk == F32:
            return self.let(F32, f"((float){r.c})")
        raise DeviceUnsupported(f"extern {e.name} returning {rk}")

    def ex_args(self, args, env):
        return [self.ex(a, env) for a in args]

    def _select(self, c, a, b):
        if isinstance(a, S):
            return self.let(a.kind, f"({c} ? {a.c} : {b.c})")
        if isinstance(a, T):
            return T([self._select(c, x, y) for x, y in zip(a.items, b.items)])
        if isinstance(a, Lanes):
            return Lanes([self._select(c, x, y) for x, y in zip(a.lanes, b.lanes)], a.kind)
        raise DeviceUnsupported("select over non-scalar values")

    def ex_BitSelect(self, e, env):
        c = self.ex(e.cond, env)
        a = self.ex(e.on_true, env)
        b = self.ex(e.on_false, env)
        if isinstance(c, Lanes):
            return Lanes([self.let(a.kind, f"({ci.c} ? {x.c} : {y.c})")
                          for ci, x, y in zip(c.lanes, a.lanes, b.lanes)], a.kind)
        return self._select(c.c, a, b)

    def _declare_like(self, v, ty):
        """Declare mutable temps shaped like IR type ty."""
        if isinstance(ty, Scalar):
            n = self.tmp()
            self.emit(f"{CTYPE[ty.kind]} {n} = {c_literal(ty.kind, 0)};")
            return S(n, ty.kind)
        if isinstance(ty, Struct):
            return T([self._declare_like(None, f) for f in ty.fields])
        if isinstance(ty, Simd):
            return Lanes([self._declare_like(None, Scalar(ty.kind)) for _ in range(W)], ty.kind)
        raise DeviceUnsupported(f"conditional value of type {ty}")

    def _assign(self, dst, src):
        if isinstance(dst, S):
            self.emit(f"{dst.c} = {src.c};")
        elif isinstance(dst, T):
            for d, s in zip(dst.items, src.items):
                self._assign(d, s)
        else:
            for d, s in zip(dst.lanes, src.lanes):
                self._assign(d, s)

    def ex_If(self, e, env):
        c = self.ex(e.cond, env)
        if isinstance(e.ty, Builder) or _is_builder_struct(e.ty):
            self.emit(f"if ({c.c}) {{")
            self.ind += 1
            r = self.ex(e.on_true, env)
            self.ind -= 1
            self.emit("} else {")
            self.ind += 1
            self.ex(e.on_false, env)
            self.ind -= 1
            self.emit("}")
            return r
        out = self._declare_like(None, e.ty)
        self.emit(f"if ({c.c}) {{")
        self.ind += 1
        self._assign(out, self.ex(e.on_true, env))
        self.ind -= 1
        self.emit("} else {")
        self.ind += 1
        self._assign(out, self.ex(e.on_false, env))
        self.ind -= 1
        self.emit("}")
        return out

    def ex_Iterate(self, e, env):
        """iterate(init, update) inside a loop body (run.py:668-686): a
        device while-loop; IterationLimit after EngineConfig.max_iterations
        steps without the continue flag dropping."""
        lam = e.update
        if not isinstance(lam, Lambda) or len(lam.params) != 1:
            raise DeviceUnsupported("iterate update must be a one-parameter lambda literal")
        init = self.ex(e.init, env)
        state = self._declare_like(None, e.ty)
        self._assign(state, init)
        limit = self.param("maxit", "i64", ("maxit",))
        steps = self.tmp("it")
        self.emit(f"for (i64 {steps} = 1;; ++{steps}) {{")
        self.ind += 1
        env2 = dict(env)
        env2[lam.params[0].name] = state
        r = self.ex(lam.body, env2)
        if not isinstance(r, T) or len(r.items) != 2:
            raise DeviceUnsupported("iterate update must return {state, continue}")
        nxt = self._declare_like(None, e.ty)
        self._assign(nxt, r.items[0])
        go = self.let(BOOL, r.items[1].c)
        self._assign(state, nxt)
        self.emit(f"if (!{go.c}) break;")
        self.emit(f"if ({steps} >= {limit}) {{ wg_raise(p.err, WG_ERR_ITER_LIMIT, {steps}); break; }}")
        self.ind -= 1
        self.emit("}")
        return state

    def ex_Len(self, e, env):
        v = self.ex(e.coll, env)
        if isinstance(v, VRef):
            return S(v.n, I64)
        if isinstance(v, SVec):
            return S(c_literal(I64, len(v.items)), I64)
        if isinstance(v, DRef):
            return S(v.n, I64)
        raise DeviceUnsupported("len() of this value inside a loop body")

    def _load_elem(self, vref, idx_c):
        ks = leaves(vref.elem)
        vals = []
        for col, k in zip(vref.cols, ks):
            ld = f"{col}[{idx_c}]"
            vals.append(self.let(k, f"({ld} != 0)" if k == BOOL else ld))
        return _shape(vref.elem, vals)

    def ex_Lookup(self, e, env):
        coll = self.ex(e.coll, env)
        idx = self.ex(e.index, env)
        if isinstance(coll, VRef):
            ty = coll.elem
            out = self._declare_like(None, ty)
            ix = idx.c
            self.emit(f"if ((u64)({ix}) >= (u64)({coll.n})) {{ wg_raise(p.err, WG_ERR_LOOKUP_OOB, {ix}); }} else {{")
            self.ind += 1
            self._assign(out, self._load_elem(coll, ix))
            self.ind -= 1
            self.emit("}")
            return out
        if isinstance(coll, SVec):
            out = self._declare_like(None, coll.elem)
            self.emit(f"switch ({idx.c}) {{")
            for j, item in enumerate(coll.items):
                self.emit(f"case {j}: {{")
                self.ind += 1
                self._assign(out, item)
                self.emit("break; }")
                self.ind -= 1
            self.emit(f"default: wg_raise(p.err, WG_ERR_LOOKUP_OOB, {idx.c});")
            self.emit("}")
            return out
        if isinstance(coll, DRef):
            return self._dict_probe(coll, idx)
        raise DeviceUnsupported("lookup into this collection inside a loop body")

    def _dict_probe(self, d, key):
        """Hash-join probe (run.py:702-712): lower_bound over the entries'
        order-key tuples (they are sorted by it), KeyNotFound on a miss.
        Float keys compare through the canonical order key (-0.0 == 0.0,
        NaN after +inf), matching Python dict equality for the reference's
        key domain."""
        kks = leaves(d.kty)
        kv = _flat(key)
        oks = [self.let(I64, f"(i64)wg_okey<{CTYPE[k]}>({v.c})") for v, k in zip(kv, kks)]
        lo, hi, pos = self.tmp("lo"), self.tmp("hi"), self.tmp("pos")
        self.emit(f"i64 {lo} = 0, {hi} = {d.n};")
        self.emit(f"while ({lo} < {hi}) {{")
        self.ind += 1
        mid = self.tmp("m")
        self.emit(f"const i64 {mid} = ({lo} + {hi}) >> 1;")
        # entry < key  (lexicographic over the leaves' order keys)
        conds = []
        for l, (col, k) in enumerate(zip(d.kcols, kks)):
            e_ok = f"(u64)wg_okey<{CTYPE[k]}>(({CTYPE[k]}){col}[{mid}])"
            conds.append((e_ok, f"(u64){oks[l].c}"))
        less = self.tmp("lt")
        self.emit(f"bool {less} = false;")
        expr = ""
        for l in reversed(range(len(conds))):
            a, b = conds[l]
            expr = f"({a} < {b})" if not expr else f"(({a} < {b}) || (({a} == {b}) && {expr}))"
        self.emit(f"{less} = {expr};")
        self.emit(f"if ({less}) {lo} = {mid} + 1; else {hi} = {mid};")
        self.ind -= 1
        self.emit("}")
        found = " && ".join(f"((u64)wg_okey<{CTYPE[k]}>(({CTYPE[k]}){col}[{lo}]) == (u64){ok.c})"
                            for col, k, ok in zip(d.kcols, kks, oks))
        self.emit(f"const bool {pos} = ({lo} < {d.n}) && {found};")
        self.emit(f"if (!{pos}) wg_raise(p.err, WG_ERR_KEY_NOT_FOUND, 0);")
        j = self.let(I64, f"({pos} ? {lo} : (i64)0)")
        if d.offs is not None:
            # groupbuilder result: the key's value vector is a slice
            b0 = self.let(I64, f"({pos} ? {d.offs}[{j.c}] : (i64)0)")
            b1 = self.let(I64, f"({pos} ? {d.offs}[{j.c} + 1] : (i64)0)")
            return VRef([f"({c} + {b0.c})" for c in d.vcols], f"({b1.c} - {b0.c})", d.vty.elem)
        vks = leaves(d.vty)
        vals = [self.let(k, f"({pos} ? ({col}[{j.c}] != 0) : false)" if k == BOOL else
                         f"({pos} ? {col}[{j.c}] : ({CTYPE[k]})0)") for col, k in zip(d.vcols, vks)]
        return _shape(d.vty, vals)

    # -- builders ------------------------------------------------------------
    def ex_NewBuilder(self, e, env):
        kind = e.kind
        if isinstance(kind, Merger):
            lm = _LocalMerger(self, kind)
            self.local_mergers.append(lm)
            return BRef(lm)
        raise DeviceUnsupported(f"{kind} created inside a loop body")

    def ex_Result(self, e, env):
        b = self.ex(e.builder, env)
        if isinstance(b, BRef) and isinstance(b.b, _LocalMerger):
            return b.b.result()
        raise DeviceUnsupported("result() of an outer builder inside a loop body")

    def ex_Merge(self, e, env):
        bref = self.ex(e.builder, env)
        v = self.ex(e.value, env)
        if not isinstance(bref, BRef):
            raise DeviceUnsupported("merge into a non-builder")
        b = bref.b
        if isinstance(b, _LocalMerger):
            b.merge(v)
        else:
            self.merge(b, v, e.value.ty)
        return bref

    def ex_For(self, e, env):
        """A loop nested in the body: runs sequentially per thread (the
        reference runs nested loops inside the parent's chunk, run.py:952-956)."""
        datas = [self.ex(it.data, env) for it in e.iters]
        for it in e.iters:
            if it.simd:
                raise DeviceUnsupported("simditer in a nested loop")
        bval = self.ex(e.builders, env)
        lam = e.func
        if not isinstance(lam, Lambda):
            raise DeviceUnsupported("nested loop body must be a lambda")
        pb, pi, px = (p.name for p in lam.params)
        if all(isinstance(d, SVec) for d in datas):
            if any(it.start is not None for it in e.iters):
                raise DeviceUnsupported("windowed iteration over a vector literal")
            n = len(datas[0].items)
            if any(len(d.items) != n for d in datas):
                from weldmill.errors import ZipLengthMismatch
                raise ZipLengthMismatch("zipped iterations disagree")
            if n:
                self.stat("trav", e)
            for j in range(n):
                elem = datas[0].items[j] if len(datas) == 1 else T([d.items[j] for d in datas])
                env2 = dict(env)
                env2.update({pb: bval, pi: S(c_literal(I64, j), I64), px: elem})
                self.ex(lam.body, env2)
            return bval
        if all(isinstance(d, VRef) for d in datas):
            if self._counts_outer(lam.body, env, {pb: bval}):
                # data-dependent append counts: fine for scan-mode appenders
                # (counted in phase A, written in phase B, sized by a pre-pass)
                cnt_ = merge_counts(lam.body, {**_benv_from(env), pb: bval})
                if any(isinstance(b, BSpec) and isinstance(b.kind, (VecBuilder, GroupBuilder)) and mx > 0
                       and b.mode != "scan" for b, (mn, mx) in cnt_.items()):
                    raise DeviceUnsupported("appends inside a data-dependent nested loop into a non-scan builder")
            # per-iter counts with the reference's checks, in its order
            # (run.py:915-940): stride >= 1 (EvalError), window inside the
            # vector (IndexOutOfBounds), then equal zipped counts
            # (ZipLengthMismatch).  A failed check raises through the error
            # word and runs the nested loop zero times (no out-of-range reads).
            cnt = self.tmp("n")
            starts, strides, cs = [], [], []
            ok = self.tmp("ok")
            self.emit(f"bool {ok} = true;")
            for k, (it, d) in enumerate(zip(e.iters, datas)):
                if it.start is not None:
                    s = self.let(I64, self.ex(it.start, env).c).c
                    en = self.let(I64, self.ex(it.end, env).c).c
                    st = self.let(I64, self.ex(it.stride, env).c).c
                    self.emit(f"if ({ok} && {st} < 1) {{ wg_raise(p.err, WG_ERR_STRIDE, {st}); {ok} = false; }}")
                    self.emit(f"if ({ok} && !(0 <= {s} && {s} <= {en} && {en} <= {d.n})) "
                              f"{{ wg_raise(p.err, WG_ERR_LOOKUP_OOB, {s}); {ok} = false; }}")
                    c = self.let(I64, f"({ok} ? (({en} - {s} + {st} - 1) / {st}) : 0)").c
                else:
                    s, st, c = "0", "1", self.let(I64, d.n).c
                starts.append(s)
                strides.append(st)
                if k > 0:
                    self.emit(f"if ({ok} && {c} != {cs[0]}) {{ wg_raise(p.err, WG_ERR_ZIP, {c}); {ok} = false; }}")
                cs.append(c)
            self.emit(f"const i64 {cnt} = {ok} ? {cs[0]} : 0;")
            self.stat("trav", e, f"{cnt} > 0")
            j = self.tmp("j")
            self.emit(f"for (i64 {j} = 0; {j} < {cnt}; ++{j}) {{")
            self.ind += 1
            elems = [self._load_elem(d, f"({s} + {j} * {st})") for d, s, st in zip(datas, starts, strides)]
            elem = elems[0] if len(elems) == 1 else T(elems)
            env2 = dict(env)
            env2.update({pb: bval, pi: S(j, I64), px: elem})
            self.ex(lam.body, env2)
            self.ind -= 1
            self.emit("}")
            return bval
        raise DeviceUnsupported("nested loop over this kind of vector")

    def _counts_outer(self, body, env, benv):
        try:
            cnt = merge_counts(body, {**_benv_from(env), **benv})
        except DeviceUnsupported:
            return True
        return any(mx > 0 for b, (mn, mx) in cnt.items() if isinstance(b, BSpec)
                   and isinstance(b.kind, (VecBuilder, GroupBuilder)))

    # -- outer builder merges ----------------------------------------------
    def merge(self, b: BSpec, v, vty):
        kind = b.kind
        if isinstance(v, Lanes):
            for lane in v.lanes:
                self.merge(b, lane, Scalar(v.kind))
            return
        if isinstance(kind, Merger):
            if self.phase != "A":
                return
            vals = _flat(v)
            ks = leaves(kind.elem)
            for f, (x, k) in enumerate(zip(vals, ks)):
                self.emit(f"m{b.bid}_{f} = {OPSTRUCT[kind.op]}<{CTYPE[k]}>::f(m{b.bid}_{f}, {x.c});")
            self.emit(f"m{b.bid}_h = 1;")
            return
        if isinstance(kind, (VecBuilder, GroupBuilder)):
            ks = b.extra["kinds"]
            vals = _flat(v) if not b.extra.get("nested") else None
            if b.mode == "direct" and b.extra.get("nested"):
                if self.phase != "A":
                    return
                if not isinstance(v, SVec):
                    raise DeviceUnsupported(f"vecbuilder[{kind.elem}] of a non-literal vector")
                if v.node is not None:
                    self.lit_nodes.setdefault(b.bid, set()).add(id(v.node))
                L = len(v.items)
                if b.extra.setdefault("nested_len", L) != L:
                    raise DeviceUnsupported(f"vecbuilder[{kind.elem}] of vectors with different lengths")
                for q, item in enumerate(v.items):
                    for f, (x, k) in enumerate(zip(_flat(item), ks)):
                        val = f"(u8)({x.c})" if k == BOOL else x.c
                        col = self.param(f"a{b.bid}_{f}", f"{STYPE[k]}*", ("b", b.bid, "col", f))
                        self.emit(f"{col}[(li * {b.k} + c{b.bid}) * {L} + {q}] = {val};")
                self.emit(f"c{b.bid} += 1;")
                return
            if b.mode == "direct":
                if self.phase != "A":
                    return
                if b.extra.get("buffered"):
                    for f, (x, k) in enumerate(zip(vals, ks)):
                        val = f"(u8)({x.c})" if k == BOOL else x.c
                        self.emit(f"o{b.bid}_{f}[j * {b.k} + c{b.bid}] = {val};")
                else:
                    for f, (x, k) in enumerate(zip(vals, ks)):
                        val = f"(u8)({x.c})" if k == BOOL else x.c
                        col = self.param(f"a{b.bid}_{f}", f"{STYPE[k]}*", ("b", b.bid, "col", f))
                        self.emit(f"{col}[li * {b.k} + c{b.bid}] = {val};")
                self.emit(f"c{b.bid} += 1;")
                return
            if b.mode == "scan":
                if self.phase in ("A", "count"):
                    self.emit(f"cnt{b.bid} += 1;")
                else:
                    for f, (x, k) in enumerate(zip(vals, ks)):
                        val = f"(u8)({x.c})" if k == BOOL else x.c
                        col = self.param(f"a{b.bid}_{f}", f"{STYPE[k]}*", ("b", b.bid, "col", f))
                        if b.extra.get("staged"):
                            self.emit(f"s_ap{b.bid}_{f}[wpos{b.bid}] = {val};")
                        else:
                            self.emit(f"{col}[wpos{b.bid}] = {val};")
                    self.emit(f"wpos{b.bid} += 1;")
                return
            raise DeviceUnsupported(f"appender mode {b.mode}")
        if isinstance(kind, DictMerger):
            if self.phase != "A":
                return
            self._dict_merge(b, v)
            return
        if isinstance(kind, VecMerger):
            if self.phase != "A":
                return
            idx, val = v.items
            vals = _flat(val)
            ks = leaves(kind.elem)
            n = self.param(f"v{b.bid}_len", "i64", ("b", b.bid, "len"))
            self.emit(f"if ((u64)({idx.c}) >= (u64)({n})) {{ wg_raise(p.err, WG_ERR_VECMERGER_OOB, {idx.c}); }} else {{")
            self.ind += 1
            opc = OPCODE[kind.op]
            for f, (x, k) in enumerate(zip(vals, ks)):
                if b.mode == "smem":
                    self.emit(f"wg_smem_fold<{opc}, {CTYPE[k]}>((({CTYPE[k]}*)(s_vm{b.bid} + {f} * {b.extra['nbins']})) + {idx.c}, {x.c});")
                else:
                    col = self.param(f"v{b.bid}_{f}", f"{CTYPE[k]}*", ("b", b.bid, "col", f))
                    self.emit(f"WgAtomicFold<{opc}, {CTYPE[k]}>::f({col} + {idx.c}, {x.c});")
            self.ind -= 1
            self.emit("}")
            return
        raise DeviceUnsupported(f"merge into {kind}")

    def _key_words(self, kinds, vals):
        lay, nw = key_layout(kinds)
        words = [self.tmp("kw") for _ in range(nw)]
        for w in words:
            self.emit(f"u64 {w} = 0;")
        for (wi, sh, width), x, k in zip(lay, vals, kinds):
            if k == I64:
                bits = f"(u64)({x.c})"
            elif k == I32:
                bits = f"(u64)(u32)({x.c})"
            elif k == F64:
                bits = f"wg_key_f64({x.c})"
            elif k == F32:
                bits = f"wg_key_f32({x.c})"
            else:
                bits = f"(u64)({x.c} ? 1 : 0)"
            self.emit(f"{words[wi]} |= ({bits}) << {sh};")
        return words

    def _dict_merge(self, b, v):
        kind = b.kind
        key, val = v.items
        kks = leaves(kind.key)
        vks = leaves(kind.value)
        if len(kks) == 1 and kks[0] in (F32, F64):
            x = _flat(key)[0].c
            zr = self.param(f"d{b.bid}_zrow", "unsigned long long*", ("b", b.bid, "zrow"))
            neg = f"(__double_as_longlong({x}) < 0)" if kks[0] == F64 else f"(__float_as_int({x}) < 0)"
            self.emit(f"if ({x} == 0) wg_zero_row({zr}, {neg}, i);")
        words = self._key_words(kks, _flat(key))
        if b.extra.get("deferred"):
            # one pending merge per item; applied after the item loop
            self.emit(f"dkf{b.bid}[j] = true; dkk{b.bid}[j] = {words[0]};")
            for f, x in enumerate(_flat(val)):
                self.emit(f"dkv{b.bid}_{f}[j] = {x.c};")
            return
        vals = _flat(val)
        nw = len(words)
        opc = OPCODE[kind.op]
        sw = b.extra["slot_words"]
        kbase = 1 if nw == 1 else 1 + nw
        table = self.param(f"d{b.bid}_table", "u64*", ("b", b.bid, "table"))
        mask = self.param(f"d{b.bid}_mask", "u64", ("b", b.bid, "mask"))
        count = self.param(f"d{b.bid}_count", "unsigned long long*", ("b", b.bid, "count"))
        slot = self.tmp("sl")
        self.emit("{")
        self.ind += 1
        R = b.extra.get("regcache", 0)
        if R and nw == 1:
            # level 0: per-thread register cache (hits fold with no memory traffic)
            op = OPSTRUCT[kind.op]
            kc = words[0]

            def fold(r):
                return " ".join(f"rv{b.bid}_{r}_{f} = {op}<{CTYPE[k]}>::f(rv{b.bid}_{r}_{f}, {x.c});"
                                for f, (x, k) in enumerate(zip(vals, vks)))
            hit = self.tmp("hit")
            self.emit(f"bool {hit} = true;")
            chain = " else ".join(f"if (rk{b.bid}_{r} == {kc}) {{ {fold(r)} }}" for r in range(R))
            claim = " else ".join(f"if (rk{b.bid}_{r} == WG_EMPTY_KEY) {{ rk{b.bid}_{r} = {kc}; {fold(r)} }}"
                                  for r in range(R))
            # the sentinel-valued key bypasses the cache (an unclaimed slot
            # holds the sentinel too and would absorb its merges)
            self.emit(f"if ({kc} == WG_EMPTY_KEY) {{ {hit} = false; }} else {chain} else {{ {claim} else {{ {hit} = false; }} }}")
            self.emit(f"if (!{hit}) {{")
            self.ind += 1
        if b.mode == "smem" and nw == 1:
            # Privatised first level: per-CTA table in shared memory.
            ssl = self.tmp("ss")
            self.emit(f"const int {ssl} = wg_sht_find1(s_dk{b.bid}, {sw}, {b.extra['smem_slots'] - 1}, {words[0]});")
            self.emit(f"if ({ssl} >= 0) {{")
            self.ind += 1
            for f, (x, k) in enumerate(zip(vals, vks)):
                self.emit(f"wg_smem_fold<{opc}, {CTYPE[k]}>(({CTYPE[k]}*)(s_dk{b.bid} + (u64){ssl} * {sw} + {kbase + f}), {x.c});")
            self.ind -= 1
            self.emit("} else {")
            self.ind += 1
        if nw == 1:
            self.emit(f"const i64 {slot} = wg_ht_find1({table}, {sw}, {mask}, {words[0]}, wg_claims{b.bid});")
        else:
            arr = self.tmp("ka")
            self.emit(f"const u64 {arr}[{nw}] = {{{', '.join(words)}}};")
            self.emit(f"const i64 {slot} = wg_ht_findN({table}, {sw}, {mask}, {arr}, {nw}, wg_claims{b.bid});")
        self.emit(f"if ({slot} >= 0) {{")
        self.ind += 1
        for f, (x, k) in enumerate(zip(vals, vks)):
            self.emit(f"WgAtomicFold<{opc}, {CTYPE[k]}>::f(({CTYPE[k]}*)({table} + (u64){slot} * {sw} + {kbase + f}), {x.c});")
        self.ind -= 1
        self.emit("} else {")
        self.ind += 1
        ocount = self.param(f"d{b.bid}_ocount", "unsigned long long*", ("b", b.bid, "ocount"))
        ocap = self.param(f"d{b.bid}_ocap", "u64", ("b", b.bid, "ocap"))
        self.emit(f"const u64 o_ = atomicAdd({ocount}, 1ULL);")
        self.emit(f"if (o_ < {ocap}) {{")
        self.ind += 1
        for wi, w in enumerate(words):
            col = self.param(f"d{b.bid}_ok{wi}", "u64*", ("b", b.bid, "okey", wi))
            self.emit(f"{col}[o_] = {w};")
        for f, (x, k) in enumerate(zip(vals, vks)):
            col = self.param(f"d{b.bid}_ov{f}", "u64*", ("b", b.bid, "oval", f))
            self.emit(f"{col}[o_] = wg_to_bits<{CTYPE[k]}>({x.c});")
        self.ind -= 1
        self.emit("} else { wg_raise(p.err, WG_ERR_INTERNAL, 1); }")
        self.ind -= 1
        self.emit("}")
        if b.mode == "smem" and nw == 1:
            self.ind -= 1
            self.emit("}")
        if R and nw == 1:
            self.ind -= 1
            self.emit("}")
        self.ind -= 1
        self.emit("}")


class _LocalMerger:
    """A merger created inside the body: a sequential register fold."""

    def __init__(self, g: Gen, kind: Merger):
        self.g = g
        self.kind = kind
        self.ks = leaves(kind.elem)
        self.names = [g.tmp("lm") for _ in self.ks]
        self.has = g.tmp("lmh")
        for n, k in zip(self.names, self.ks):
            g.emit(f"{CTYPE[k]} {n} = {c_literal(k, internal_identity(kind.op, k))};")
        g.emit(f"int {self.has} = 0;")

    def merge(self, v):
        if isinstance(v, Lanes):
            for lane in v.lanes:
                self.merge(lane)
            return
        for n, x, k in zip(self.names, _flat(v), self.ks):
            self.g.emit(f"{n} = {OPSTRUCT[self.kind.op]}<{CTYPE[k]}>::f({n}, {x.c});")
        self.g.emit(f"{self.has} = 1;")

    def result(self):
        vals = []
        for n, k in zip(self.names, self.ks):
            ident = c_literal(k, identity_value(self.kind.op, k))
            vals.append(self.g.let(k, f"({self.has} ? {n} : {ident})"))
        return _shape(self.kind.elem, vals)


def _flat(v):
    if isinstance(v, S):
        return [v]
    if isinstance(v, T):
        out = []
        for x in v.items:
            out.extend(_flat(x))
        return out
    raise DeviceUnsupported("expected a scalar or struct value")


def _shape(ty, vals):
    it = iter(vals)

    def go(t):
        if isinstance(t, Scalar):
            return next(it)
        return T([go(f) for f in t.fields])

    try:
        return go(ty)
    finally:
        del go


def _is_builder_struct(t):
    return isinstance(t, Struct) and all(isinstance(f, Builder) or _is_builder_struct(f) for f in t.fields)


def _benv_from(env):
    return {k: v for k, v in env.items() if isinstance(v, (BRef, BTuple))}


# ---------------------------------------------------------------------------
# Static merge-count analysis: per outer builder, (min, max) scalar appends
# per iteration over all control paths.


INF = math.inf


def _add(a, b):
    out = dict(a)
    for k, (mn, mx) in b.items():
        x = out.get(k, (0, 0))
        out[k] = (x[0] + mn, x[1] + mx)
    return out


def _branch(a, b):
    out = {}
    for k in set(a) | set(b):
        x = a.get(k, (0, 0))
        y = b.get(k, (0, 0))
        out[k] = (min(x[0], y[0]), max(x[1], y[1]))
    return out


def _bref(e, benv):
    """Resolve a builder-typed expression to BRef/BTuple plus its counts."""
    if isinstance(e, Ident):
        return benv.get(e.name), {}
    if isinstance(e, FieldAccess):
        base, c = _bref(e.base, benv)
        if isinstance(base, BTuple):
            return base.items[e.ordinal], c
        return None, c
    if isinstance(e, Merge):
        r, c = _bref(e.builder, benv)
        n = W if isinstance(e.value.ty, Simd) else 1
        if isinstance(r, BRef):
            c = _add(c, {r.b: (n, n)})
        return r, c
    if isinstance(e, If):
        rt_, ct = _bref(e.on_true, benv)
        _, cf = _bref(e.on_false, benv)
        return rt_, _branch(ct, cf)
    if isinstance(e, Let):
        if isinstance(e.value.ty, Builder) or _is_builder_struct(e.value.ty):
            r, c = _bref(e.value, benv)
            r2, c2 = _bref(e.body, {**benv, e.name: r})
            return r2, _add(c, c2)
        return _bref(e.body, benv)
    if isinstance(e, MakeStruct):
        items, c = [], {}
        for x in e.items:
            r, cx = _bref(x, benv)
            items.append(r)
            c = _add(c, cx)
        return BTuple(items), c
    if isinstance(e, For):
        r, c = _bref(e.builders, benv)
        lam = e.func
        pb = lam.params[0].name
        _, cb = _bref(lam.body, {**benv, pb: r})
        data = e.iters[0].data
        if isinstance(data, MakeVector) and all(it.start is None for it in e.iters):
            n = len(data.items)
            cb = {k: (mn * n, mx * n) for k, (mn, mx) in cb.items()}
        else:
            cb = {k: (0, INF if mx > 0 else 0) for k, (mn, mx) in cb.items()}
        return r, _add(c, cb)
    if isinstance(e, NewBuilder):
        return BRef(object()), {}
    return None, {}


def merge_counts(body, benv):
    _, c = _bref(body, benv)
    return c


# ---------------------------------------------------------------------------
# Kernel assembly


def choose_items(iters):
    row = 0
    for it in iters:
        row += sum(SIZE[k] for k in it.kinds) * (W if it.simd else 1)
    row = max(row, 1)
    items = 128 // row
    p = 1
    while p * 2 <= items:
        p *= 2
    return max(2, min(8, p))


def generate(loop: For, iters, bstruct, captures, externs, strategy, name="wg_loop", items=None,
             count_only=False, counting=False) -> KernelPlan:
    g = Gen(loop, iters, bstruct, captures, externs, strategy)
    g.counting = counting and not count_only
    lam = loop.func
    if not isinstance(lam, Lambda):
        raise DeviceUnsupported("loop function must be a lambda literal")
    pb, pi, px = (p.name for p in lam.params)

    BLOCK = BLOCK_DEFAULT
    ITEMS = items or ITEMS_OVERRIDE or choose_items(iters)
    if not (items or ITEMS_OVERRIDE) and any(isinstance(b.kind, DictMerger) for b in g.bspecs):
        ITEMS = min(ITEMS, 2)   # deferred merges + register caches are register-hungry
    for b in g.bspecs:
        if b.extra.get("part"):
            # the tile's records are staged in dynamic shared memory; larger
            # tiles mean longer per-partition runs and fewer global
            # reservations per row
            rec = 8 + 8 * len(leaves(b.kind.value)) + 2
            ITEMS = PART_ITEMS
            while ITEMS > 1 and BLOCK * ITEMS * rec > 96 * 1024:
                ITEMS //= 2
    if not (items or ITEMS_OVERRIDE) and PIPE and not any(b.extra.get("part") for b in g.bspecs):
        # keep >= 2 pipeline stages inside the shared-memory budget
        row = sum(SIZE[k] * (W if it.simd else 1) for it in iters for k in it.kinds)
        while ITEMS > 1 and 2 * BLOCK * ITEMS * row > PIPE_SMEM_BUDGET:
            ITEMS //= 2
    g.items = ITEMS

    # builders value seen by the body
    def bref_of(bs):
        if isinstance(bs, BSpec):
            return BRef(bs)
        return BTuple([bref_of(x) for x in bs])

    bval = bref_of(bstruct)

    # captured values
    env = {}
    for cname, (cty, cval) in captures.items():
        env[cname] = _capture_val(g, cname, cty, cval)

    # appender modes from the static merge counts
    counts = merge_counts(lam.body, {pb: bval})
    for b in g.bspecs:
        mn, mx = counts.get(b, (0, 0))
        b.extra["maxm"] = mx
        if isinstance(b.kind, DictMerger) and mx <= 1 and key_layout(leaves(b.kind.key))[1] == 1:
            if b.extra.get("lowcard"):
                # low cardinality: inline register cache in front of the shared table
                if REGCACHE and len(leaves(b.kind.value)) <= 8:
                    b.extra["regcache"] = REGCACHE
            elif DEFER_DICT:
                # high / unknown cardinality: deferred merges, batched HBM probes
                b.extra["deferred"] = True
        if isinstance(b.kind, (VecBuilder, GroupBuilder)):
            if isinstance(b.kind, VecBuilder) and isinstance(b.kind.elem, Vec):
                # vecbuilder[vec[T]]: child leaves; the per-merge length is
                # fixed by the merged vector literals (set in Gen.merge)
                if not is_flat_type(b.kind.elem.elem):
                    raise DeviceUnsupported(f"vecbuilder[{b.kind.elem}] (doubly nested) on the device")
                b.extra["kinds"] = leaves(b.kind.elem.elem)
                b.extra["nested"] = True
            elif isinstance(b.kind, VecBuilder):
                b.extra["kinds"] = leaves(b.kind.elem)
            else:
                b.extra["kinds"] = leaves(b.kind.key) + leaves(b.kind.value)
            if b.extra.get("nested") and not (mn == mx and mx > 0) and mx != 0:
                raise DeviceUnsupported(f"vecbuilder[{b.kind.elem}] with data-dependent append counts")
            if mx == 0:
                b.mode, b.k = "none", 0
            elif mn == mx:
                b.mode, b.k = "direct", int(mn)
                b.extra["buffered"] = ITEMS * b.k <= 32 and not b.extra.get("nested")
            elif mx < INF:
                b.mode, b.k = "scan", int(mx)
            else:
                # appends inside a data-dependent nested loop (flatmap): the
                # scan schedule counts them in phase A and stores them in
                # phase B; the executor sizes the output with a count-only
                # pre-pass of the same body (generate(count_only=True))
                b.mode, b.k = "scan", None
                b.extra["unbounded"] = True

    scan_bs = [b for b in g.bspecs if b.mode == "scan"]
    if scan_bs and not (items or ITEMS_OVERRIDE):
        # larger tiles for look-back kernels: half as many tiles to resolve
        ITEMS = min(16, ITEMS * 2)
        g.items = ITEMS
        for b in g.bspecs:
            if b.mode == "direct":
                b.extra["buffered"] = ITEMS * b.k <= 32 and not b.extra.get("nested")
    # order-preserving appenders stage their tile output in shared memory so
    # the global stores are contiguous per tile (coalesced)
    staged_bytes = 0
    for b in scan_bs:
        b.extra["staged"] = False
    if scan_bs and STAGE_SCAN and all(b.k is not None for b in scan_bs):
        need = sum(BLOCK * ITEMS * b.k * SIZE[k] for b in scan_bs for k in b.extra["kinds"])
        # static shared memory is capped at 48 KB per kernel: the staging
        # buffers share it with the math tables the body's externs copy in
        if need <= min(40 * 1024, 46 * 1024 - _table_bytes(lam.body)):
            for b in scan_bs:
                b.extra["staged"] = True
            staged_bytes = need

    # warp-specialised scan schedule: appenders only (every builder of the
    # loop a scan appender with at most k merges per row), staged in dynamic
    # shared memory
    ws = bool(SCAN_WS and scan_bs and not count_only and all(b.mode == "scan" for b in g.bspecs)
              and all(b.k is not None for b in scan_bs) and ITEMS <= 32
              and not any(b.extra.get("segstats") == "fine" for b in scan_bs))
    if ws and not (items or ITEMS_OVERRIDE):
        ITEMS = min(ITEMS, WS_ITEMS)
        g.items = ITEMS
    if ws and "WELDGPU_BLOCK" not in _os.environ:
        BLOCK = WS_BLOCK
    ws_need = sum(BLOCK * ITEMS * b.k * SIZE[k] for b in scan_bs for k in b.extra["kinds"]) if ws else 0
    if ws and WS_NBUF * ws_need > 160 * 1024:
        ws = False
    if ws:
        for b in scan_bs:
            b.extra["staged"] = True
        staged_bytes = 0

    merger_bs = [b for b in g.bspecs if isinstance(b.kind, Merger)]
    schedule = "scan" if scan_bs else "static"

    # element loads ----------------------------------------------------------
    g.param("n", "i64", ("n",))
    g.param("idx0", "i64", ("idx0",))
    g.param("err", "i64*", ("err",))
    loads = []  # (array name, stype, kind, count_per_item, iter index, leaf)
    for k, it in enumerate(iters):
        per = W if it.simd else 1
        for l, kk in enumerate(it.kinds):
            col = g.param(f"it{k}_{l}", f"const {STYPE[kk]}*", ("itcol", k, l))
            loads.append((f"x{k}_{l}", STYPE[kk], kk, per, k, l, col))
        if it.strided:
            g.param(f"it{k}_start", "i64", ("itstart", k))
            g.param(f"it{k}_stride", "i64", ("itstride", k))

    if g.counting:
        g.param("cnt", "unsigned long long*", ("cnt",))
    seg_bs = [b for b in scan_bs if b.extra.get("segstats")] if not count_only else []
    if seg_bs:
        # chunk-start output positions of unhinted appenders (the
        # reference's per-(step, chunk) segments, builders.py:256-272)
        g.param("cgrain", "i64", ("cgrain",))
        g.param("cgmask", "i64", ("cgmask",))
        g.param("cbase", "i64", ("cbase",))
        for b in seg_bs:
            g.param(f"a{b.bid}_coff", "i64*", ("b", b.bid, "coff"))

    def elem_val(k, it):
        """Element value of iter k at item j (C arrays indexed by j)."""
        vals = []
        for (arr, st, kk, per, kk_i, l, col) in loads:
            if kk_i != k:
                continue
            if it.simd:
                lanes = [S(f"({arr}[j * {W} + {q}] != 0)" if kk == BOOL else f"{arr}[j * {W} + {q}]", kk)
                         for q in range(W)]
                vals.append(Lanes(lanes, kk))
            else:
                vals.append(S(f"({arr}[j] != 0)" if kk == BOOL else f"{arr}[j]", kk))
        if it.simd:
            return vals[0]
        return _shape(it.elem, vals)

    # body, phase A -----------------------------------------------------------
    def body_env():
        e = dict(env)
        elems = [elem_val(k, it) for k, it in enumerate(iters)]
        e[px] = elems[0] if len(elems) == 1 else T(elems)
        e[pi] = S("i", I64)
        e[pb] = bval
        return e

    if count_only:
        return _count_plan(g, lam, body_env, loads, iters, ITEMS, BLOCK, scan_bs, name)

    g.lines = []
    g.ind = 3
    g.phase = "A"
    for b in g.bspecs:
        if b.mode == "direct":
            g.emit(f"int c{b.bid} = 0;")
    g.ex(lam.body, body_env())
    body_a = g.lines
    body_b = []
    if scan_bs:
        g.lines = []
        g.ind = 3
        g.phase = "B"
        g.ex(lam.body, body_env())
        body_b = g.lines

    # builder params / smem -------------------------------------------------
    for b in merger_bs:
        g.param(f"m{b.bid}_part", "u64*", ("b", b.bid, "part"))
        g.param(f"m{b.bid}_slot", "u64*", ("b", b.bid, "slot"))
        g.param(f"m{b.bid}_init", "i64", ("b", b.bid, "init"))
        g.param(f"m{b.bid}_mirror", "u64*", ("b", b.bid, "mirror"))
    if merger_bs:
        g.param("ticket", "unsigned int*", ("ticket",))
    for b in g.bspecs:
        if b.mode == "direct":
            for f, kk in enumerate(b.extra["kinds"]):
                g.param(f"a{b.bid}_{f}", f"{STYPE[kk]}*", ("b", b.bid, "col", f))
        if b.mode == "scan":
            g.param(f"a{b.bid}_status", "u64*", ("b", b.bid, "status"))
            g.param(f"a{b.bid}_total", "i64*", ("b", b.bid, "total"))
    if schedule == "scan":
        g.param("tilectr", "unsigned long long*", ("tilectr",))

    smem_decls = []
    smem_init = []
    smem_flush = []
    dyn_smem = 0
    for b in g.bspecs:
        if isinstance(b.kind, VecMerger) and b.mode == "smem":
            nb = b.extra["nbins"]
            ks = leaves(b.kind.elem)
            off = dyn_smem // 8
            smem_decls.append(f"u64* s_vm{b.bid} = wg_dyn_smem + {off};")
            dyn_smem += nb * len(ks) * 8
            opc = OPCODE[b.kind.op]
            for f, kk in enumerate(ks):
                ident = c_literal(kk, internal_identity(b.kind.op, kk))
                smem_init.append(f"for (int q = threadIdx.x; q < {nb}; q += {BLOCK}) (({CTYPE[kk]}*)(s_vm{b.bid} + {f * nb}))[q] = {ident};")
                col = g.param(f"v{b.bid}_{f}", f"{CTYPE[kk]}*", ("b", b.bid, "col", f))
                smem_flush.append(
                    f"for (int q = threadIdx.x; q < {nb}; q += {BLOCK}) {{ const {CTYPE[kk]} v_ = (({CTYPE[kk]}*)(s_vm{b.bid} + {f * nb}))[q]; "
                    f"if (wg_to_bits<{CTYPE[kk]}>(v_) != wg_to_bits<{CTYPE[kk]}>({ident})) WgAtomicFold<{opc}, {CTYPE[kk]}>::f({col} + q, v_); }}")
        if isinstance(b.kind, DictMerger) and b.extra.get("part"):
            # hash-partitioned dictmerger: the tile's records, sorted by partition
            B = b.bid
            V_ = len(leaves(b.kind.value))
            T_ = BLOCK * ITEMS
            off = dyn_smem // 8
            smem_decls.append(f"u64* s_rk{B} = wg_dyn_smem + {off};"
                              + "".join(f" u64* s_rv{B}_{f} = wg_dyn_smem + {off + T_ * (1 + f)};" for f in range(V_))
                              + f" unsigned short* s_rp{B} = (unsigned short*)(wg_dyn_smem + {off + T_ * (1 + V_)});")
            dyn_smem += T_ * 8 * (1 + V_) + ((T_ * 2 + 7) // 8) * 8
        if isinstance(b.kind, DictMerger) and b.mode == "smem":
            ns = b.extra["smem_slots"]
            sw = b.extra["slot_words"]
            off = dyn_smem // 8
            smem_decls.append(f"u64* s_dk{b.bid} = wg_dyn_smem + {off};")
            dyn_smem += ns * sw * 8
            pat = b.extra["pattern"]
            smem_init.append(f"for (int q = threadIdx.x; q < {ns * sw}; q += {BLOCK}) {{ const int w_ = q % {sw}; "
                             f"s_dk{b.bid}[q] = {_pattern_switch(pat)}; }}")
            table = g.param(f"d{b.bid}_table", "u64*", ("b", b.bid, "table"))
            mask = g.param(f"d{b.bid}_mask", "u64", ("b", b.bid, "mask"))
            count = g.param(f"d{b.bid}_count", "unsigned long long*", ("b", b.bid, "count"))
            ocount = g.param(f"d{b.bid}_ocount", "unsigned long long*", ("b", b.bid, "ocount"))
            ocap = g.param(f"d{b.bid}_ocap", "u64", ("b", b.bid, "ocap"))
            vks = leaves(b.kind.value)
            opc = OPCODE[b.kind.op]
            fl = [f"for (int q = threadIdx.x; q < {ns}; q += {BLOCK}) {{",
                  f"  const u64 k_ = s_dk{b.bid}[(u64)q * {sw}];",
                  "  if (k_ == WG_EMPTY_KEY) continue;",
                  f"  const i64 sl_ = wg_ht_find1({table}, {sw}, {mask}, k_, wg_claims{b.bid});",
                  "  if (sl_ >= 0) {"]
            for f, kk in enumerate(vks):
                fl.append(f"    WgAtomicFold<{opc}, {CTYPE[kk]}>::f(({CTYPE[kk]}*)({table} + (u64)sl_ * {sw} + {1 + f}), "
                          f"*({CTYPE[kk]}*)(s_dk{b.bid} + (u64)q * {sw} + {1 + f}));")
            fl.append("  } else {")
            fl.append(f"    const u64 o_ = atomicAdd({ocount}, 1ULL);")
            fl.append(f"    if (o_ < {ocap}) {{")
            okc = g.param(f"d{b.bid}_ok0", "u64*", ("b", b.bid, "okey", 0))
            fl.append(f"      {okc}[o_] = k_;")
            for f, kk in enumerate(vks):
                col = g.param(f"d{b.bid}_ov{f}", "u64*", ("b", b.bid, "oval", f))
                fl.append(f"      {col}[o_] = s_dk{b.bid}[(u64)q * {sw} + {1 + f}];")
            fl.append("    } else { wg_raise(p.err, WG_ERR_INTERNAL, 1); }")
            fl.append("  }")
            fl.append("}")
            smem_flush.append("\n    ".join(fl))

    ws_off = 0
    ws_boff = {}
    if ws:
        ws_off = (dyn_smem + 127) // 128 * 128
        o_ = 0
        for b in scan_bs:
            for f, kk in enumerate(b.extra["kinds"]):
                ws_boff[(b.bid, f)] = o_
                o_ += (BLOCK * ITEMS * b.k * SIZE[kk] + 15) // 16 * 16
        ws_buf = o_
        dyn_smem = ws_off + WS_NBUF * ws_buf

    # bulk-async column pipeline (static schedule, contiguous 16B-aligned
    # columns).  The stage count is a launch parameter: the executor picks
    # the most stages that do not lower the kernel's occupancy.
    # Scan kernels use it too: with a persistent, fully resident grid the
    # static round-robin tile order is a valid look-back order.
    pipe = bool(PIPE and not scan_bs and loads
                and all((not it.strided) and it.aligned for it in iters))
    pipe_off = pipe_stage_bytes = 0
    pipe_col_off = []
    if pipe:
        off = 0
        for (arr, st, kk, per, k, l, col) in loads:
            pipe_col_off.append(off)
            off += (BLOCK * ITEMS * per * SIZE[kk] + 127) // 128 * 128
        pipe_stage_bytes = off
        pipe_off = (dyn_smem + 127) // 128 * 128
        if pipe_off + 2 * off > 200 * 1024:
            pipe = False
        else:
            g.param("pipe_stages", "i64", ("pipe_stages",))
    pipe_stages = "PIPE_S"

    deferred_lines = {b.bid: _deferred_dict_lines(g, b) for b in g.bspecs if b.extra.get("deferred")}
    regcache_flush = {b.bid: _regcache_flush_lines(g, b) for b in g.bspecs if b.extra.get("regcache")}

    # ---- assemble ----------------------------------------------------------
    src = []
    src.append(f"#define WG_LD256 {LD256}")
    src.append(f"#define WG_ST256 {ST256}")
    src.append(f"#define WG_LB_PER {LB_PER}")
    src.append(f"#define WG_LB_SLEEP {LB_SLEEP}")
    src.append('#include "weld_device.cuh"')
    src.append(f"#define BLOCK {BLOCK}")
    src.append(f"#define ITEMS {ITEMS}")
    if ws:
        src.append(f"#define WS_NBUF {WS_NBUF}")
    src.append("#define TILE (BLOCK * ITEMS)")
    src.append("struct Params {")
    for p_ in g.params:
        src.append(f"  {p_.ctype} {p_.name};")
    src.append("};")
    minb = MINBLOCKS
    if scan_bs and not MINBLOCKS and SCAN_MINBLOCKS:
        # scan schedule: resident CTAs hide each other's look-back waits;
        # capping registers buys CTAs (filter: 78 -> 64 registers, 3 -> 4
        # CTAs of 256 threads per SM)
        minb = SCAN_MINBLOCKS * 256 // BLOCK
    lb = f"BLOCK, {minb}" if minb else "BLOCK"
    if ws:
        lb = f"BLOCK + 32, {WS_MINB}" if WS_MINB else "BLOCK + 32"
    src.append(f'extern "C" __global__ void __launch_bounds__({lb}) {name}(const Params p) {{')
    src.append("  extern __shared__ __align__(16) u64 wg_dyn_smem[];")
    for t in sorted(g.tabs):
        smem_init.append(f"{t}_init();")
    src.extend("  " + d for d in smem_decls)
    src.extend("  " + d for d in smem_init)
    if smem_init:
        src.append("  __syncthreads();")
    for b in merger_bs:
        for f, kk in enumerate(leaves(b.kind.elem)):
            src.append(f"  {CTYPE[kk]} m{b.bid}_{f} = {c_literal(kk, internal_identity(b.kind.op, kk))};")
        src.append(f"  int m{b.bid}_h = 0;")
    dict_bs = [b for b in g.bspecs if isinstance(b.kind, DictMerger)]
    for b in dict_bs:
        src.append(f"  int wg_claims{b.bid} = 0;")
        src.extend(b.extra.get("smem_decl", []))
        if b.extra.get("regcache"):
            src.extend(_regcache_decl(b, b.extra["regcache"]))
    src.append("  const i64 n = p.n;")
    src.append("  const i64 ntiles = (n + TILE - 1) / TILE;")
    if ws:
        src.append("  __shared__ i64 s_scan[33];")
        src.append("  __shared__ i64 s_wtile;")
        src.append("  __shared__ i64 s_btile[WS_NBUF];")
        src.append(f"  __shared__ i64 s_bagg[WS_NBUF][{len(scan_bs)}];")
        if seg_bs:
            src.append(f"  __shared__ i64 s_bci[WS_NBUF][BLOCK];")
            src.append(f"  __shared__ int s_bcp[WS_NBUF][{len(seg_bs)}][BLOCK];")
        src.append("  __shared__ __align__(8) u64 wg_full[WS_NBUF], wg_empty[WS_NBUF];")
    elif scan_bs:
        src.append("  __shared__ i64 s_scan[33];")
        src.append(f"  __shared__ i64 s_toff[{len(scan_bs)}];")
        src.append("  __shared__ i64 s_tile[2];")
        for b in scan_bs:
            if b.extra["staged"]:
                for f, kk in enumerate(b.extra["kinds"]):
                    src.append(f"  __shared__ __align__(16) {STYPE[kk]} s_ap{b.bid}_{f}[TILE * {b.k}];")
    def load_lines(tvar, suffix, ind):
        out = [f"{ind}{{ const i64 lt0_ = {tvar} * TILE + (i64)threadIdx.x * ITEMS; const bool lfull_ = (lt0_ + ITEMS <= n);"]
        for (arr, st, kk, per, k, l, col) in loads:
            cnt = f"ITEMS * {per}" if per > 1 else "ITEMS"
            a = arr + suffix
            if iters[k].strided:
                out.append(f"{ind}  for (int q = 0; q < ITEMS; ++q) {{ const i64 li_ = lt0_ + q; "
                           f"{a}[q] = (li_ < n) ? {col}[p.it{k}_start + li_ * p.it{k}_stride] : ({st})0; }}")
            else:
                out.append(f"{ind}  if (lfull_) wg_load_contig<{st}, {cnt}>({col} + lt0_ * {per}, {a});")
                out.append(f"{ind}  else {{ for (int q = 0; q < {cnt}; ++q) {{ const i64 e_ = lt0_ * {per} + q; "
                           f"{a}[q] = (e_ < n * {per}) ? {col}[e_] : ({st})0; }} }}")
        out.append(f"{ind}}}")
        return out

    def ws_lines():
        """Warp-specialised scan schedule.  Threads [0, BLOCK) claim tiles in
        order, count, scan, publish the tile aggregate at once and stage the
        tile's appends in buffer it % WS_NBUF; the extra warp [BLOCK,
        BLOCK + 32) resolves each staged tile's look-back, stores it and frees
        the buffer.  A slow predecessor stalls only the store warp while the
        compute warps fill the other buffer(s)."""
        def bufptrs(ind, bvar):
            out = []
            for b in scan_bs:
                for f, kk in enumerate(b.extra["kinds"]):
                    out.append(f"{ind}{STYPE[kk]}* const s_ap{b.bid}_{f} = ({STYPE[kk]}*)((char*)wg_dyn_smem + {ws_off} + "
                               f"(u64){bvar} * {ws_buf} + {ws_boff[(b.bid, f)]});")
            return out
        out = ["  if (threadIdx.x == 0) {",
               "    for (int b_ = 0; b_ < WS_NBUF; ++b_) { wg_mbar_init(&wg_full[b_], 1); wg_mbar_init(&wg_empty[b_], 1); }",
               "    wg_fence_mbar_init();",
               "  }",
               "  __syncthreads();",
               "  if (threadIdx.x >= BLOCK) {",
               "    // look-back + store warp",
               "    const int lane_ = threadIdx.x & 31;",
               "    for (i64 it_ = 0; ; ++it_) {",
               "      const int bf_ = (int)(it_ % WS_NBUF);",
               "      wg_mbar_wait(&wg_full[bf_], (unsigned)((it_ / WS_NBUF) & 1));",
               "      const i64 tile = s_btile[bf_];",
               "      if (tile < 0) break;"]
        out += bufptrs("      ", "bf_")
        for si, b in enumerate(scan_bs):
            out.append(f"      {{ const i64 agg_ = s_bagg[bf_][{si}];")
            out.append(f"        const i64 pre_ = wg_lookback_resolve(p.a{b.bid}_status, tile, agg_);")
            out.append(f"        if (lane_ == 0 && tile == ntiles - 1) *p.a{b.bid}_total = pre_ + agg_;")
            for f, kk in enumerate(b.extra["kinds"]):
                out.append(f"        for (i64 q = lane_; q < agg_; q += 32) __stcs(p.a{b.bid}_{f} + pre_ + q, s_ap{b.bid}_{f}[q]);")
            if b in seg_bs:
                sj = seg_bs.index(b)
                out.append(f"        for (int q = lane_; q < BLOCK; q += 32) {{ const int lp_ = s_bcp[bf_][{sj}][q];"
                           f" if (lp_ >= 0) p.a{b.bid}_coff[s_bci[bf_][q]] = pre_ + lp_; }}")
            out.append("      }")
        out += ["      __syncwarp();",
                "      if (lane_ == 0) wg_mbar_arrive(&wg_empty[bf_]);",
                "    }",
                "    return;",
                "  }",
                "  if (threadIdx.x == 0) s_wtile = (i64)atomicAdd(p.tilectr, 1ULL);",
                "  wg_bar_group(BLOCK);",
                "  for (i64 it_ = 0; ; ++it_) {",
                "    const int bf_ = (int)(it_ % WS_NBUF);",
                # (claiming the next tile during phase B instead: 1.59 vs 1.46 ms --
                # a claimed-but-unpublished tile stalls every later look-back)
                "    if (it_ > 0) { if (threadIdx.x == 0) s_wtile = (i64)atomicAdd(p.tilectr, 1ULL); wg_bar_group(BLOCK); }",
                "    const i64 tile = s_wtile;",
                "    if (tile >= ntiles) {",
                "      if (threadIdx.x == 0) {",
                "        if (it_ >= WS_NBUF) wg_mbar_wait(&wg_empty[bf_], (unsigned)(((it_ / WS_NBUF) - 1) & 1));",
                "        s_btile[bf_] = -1;",
                "        wg_mbar_arrive(&wg_full[bf_]);",
                "      }",
                "      break;",
                "    }"]
        out += decl_lines("", "    ")
        out += load_lines("tile", "", "    ")
        out.append("    const i64 t0 = tile * TILE + (i64)threadIdx.x * ITEMS;")
        out.append("    const bool full = (t0 + ITEMS <= n);")
        for b in scan_bs:
            out.append(f"    i64 cnt{b.bid} = 0;")
        if seg_bs:
            out.append("    int j0a_ = -1;")
            out.append("    { i64 r_ = (p.cgmask >= 0) ? ((p.cbase + t0) & p.cgmask) : ((p.cbase + t0) % p.cgrain);")
            out.append("      r_ = r_ ? p.cgrain - r_ : 0; if (r_ < ITEMS && t0 + r_ < n) j0a_ = (int)r_; }")
            for b in seg_bs:
                out.append(f"    int c0s{b.bid} = -1;")
        out.append("#pragma unroll")
        out.append("    for (int j = 0; j < ITEMS; ++j) {")
        out.append("      const i64 li = t0 + j;")
        if seg_bs:
            out.append("      if (j == j0a_) { " + " ".join(f"c0s{b.bid} = (int)cnt{b.bid};" for b in seg_bs) + " }")
        out.append("      if (li < n) {")
        out.append("        const i64 i = p.idx0 + li;")
        out.extend(body_a)
        out.append("      }")
        out.append("    }")
        for si, b in enumerate(scan_bs):
            out.append(f"    i64 agg{b.bid};")
            out.append(f"    i64 wpos{b.bid} = wg_group_exclusive_scan(cnt{b.bid}, s_scan, &agg{b.bid}, BLOCK);")
            out.append(f"    if (threadIdx.x == 0) wg_publish_aggregate(p.a{b.bid}_status, tile, agg{b.bid});")
        out.append("    if (it_ >= WS_NBUF) wg_mbar_wait(&wg_empty[bf_], (unsigned)(((it_ / WS_NBUF) - 1) & 1));")
        out += bufptrs("    ", "bf_")
        if seg_bs:
            out.append("    {")
            out.append("      const i64 sgn_ = (j0a_ >= 0) ? j0a_ : 0;")
            out.append("      const i64 g0_ = p.cbase + t0 + sgn_;")
            out.append("      s_bci[bf_][threadIdx.x] = (p.cgmask >= 0) ? ((g0_ >> __popcll(p.cgmask)) - (p.cbase >> __popcll(p.cgmask)))"
                       " : (g0_ / p.cgrain - p.cbase / p.cgrain);")
            for sj, b in enumerate(seg_bs):
                out.append(f"      s_bcp[bf_][{sj}][threadIdx.x] = (c0s{b.bid} >= 0) ? (int)(wpos{b.bid} + c0s{b.bid}) : -1;")
            out.append("    }")
        out.append("#pragma unroll")
        out.append("    for (int j = 0; j < ITEMS; ++j) {")
        out.append("      const i64 li = t0 + j;")
        out.append("      if (li < n) {")
        out.append("        const i64 i = p.idx0 + li;")
        out.extend(body_b)
        out.append("      }")
        out.append("    }")
        out.append("    wg_bar_group(BLOCK);")
        out.append("    if (threadIdx.x == 0) {")
        out.append("      s_btile[bf_] = tile;")
        for si, b in enumerate(scan_bs):
            out.append(f"      s_bagg[bf_][{si}] = agg{b.bid};")
        out.append("      wg_mbar_arrive(&wg_full[bf_]);")
        out.append("    }")
        out.append("  }")
        return out

    def decl_lines(suffix, ind):
        return [f"{ind}alignas(16) {st} {arr}{suffix}[{'ITEMS * %d' % per if per > 1 else 'ITEMS'}];"
                for (arr, st, kk, per, k, l, col) in loads]

    def tile_body(mid=None, claim=False, guard=True):
        """Everything a thread does for one tile once its columns are in
        registers (x arrays): body, buffered stores, deferred dict merges,
        and for scan appenders the block scan + look-back + store phase."""
        out = []
        out.append("    const i64 t0 = tile * TILE + (i64)threadIdx.x * ITEMS;")
        out.append("    const bool full = (t0 + ITEMS <= n);")
        for b in g.bspecs:
            if b.mode == "direct" and b.extra.get("buffered"):
                for f, kk in enumerate(b.extra["kinds"]):
                    out.append(f"    alignas(16) {STYPE[kk]} o{b.bid}_{f}[ITEMS * {b.k}];")
            if b.mode == "scan":
                out.append(f"    i64 cnt{b.bid} = 0;")
            if b.extra.get("deferred"):
                out.append(f"    bool dkf{b.bid}[ITEMS]; u64 dkk{b.bid}[ITEMS];")
                out.append(f"#pragma unroll\n    for (int q = 0; q < ITEMS; ++q) dkf{b.bid}[q] = false;")
                for f, kk in enumerate(leaves(b.kind.value)):
                    out.append(f"    {CTYPE[kk]} dkv{b.bid}_{f}[ITEMS];")
        seg_coarse = seg_bs and not (ITEMS > 32 or any(b.extra.get("segstats") == "fine" for b in seg_bs))
        if seg_coarse:
            # the (at most one) item of this thread that starts a grain-wide
            # chunk; phase A notes the thread-local append count there
            out.append("    int j0a_ = -1;")
            out.append("    { i64 r_ = (p.cgmask >= 0) ? ((p.cbase + t0) & p.cgmask) : ((p.cbase + t0) % p.cgrain);")
            out.append("      r_ = r_ ? p.cgrain - r_ : 0; if (r_ < ITEMS && t0 + r_ < n) j0a_ = (int)r_; }")
            for b in seg_bs:
                out.append(f"    int c0s{b.bid} = -1;")
        out.append("#pragma unroll")
        out.append("    for (int j = 0; j < ITEMS; ++j) {")
        out.append("      const i64 li = t0 + j;")
        if seg_coarse:
            out.append("      if (j == j0a_) { " + " ".join(f"c0s{b.bid} = (int)cnt{b.bid};" for b in seg_bs) + " }")
        out.append("      if (li < n) {" if guard else "      {")
        out.append("        const i64 i = p.idx0 + li;")
        out.extend(body_a)
        out.append("      }")
        out.append("    }")
        for b in g.bspecs:
            if b.mode == "direct" and b.extra.get("buffered"):
                for f, kk in enumerate(b.extra["kinds"]):
                    col = f"p.a{b.bid}_{f}"
                    out.append(f"    if (full) wg_store_contig<{STYPE[kk]}, ITEMS * {b.k}>({col} + t0 * {b.k}, o{b.bid}_{f});")
                    out.append(f"    else {{ for (int q = 0; q < ITEMS * {b.k}; ++q) if (t0 * {b.k} + q < n * {b.k}) "
                               f"{col}[t0 * {b.k} + q] = o{b.bid}_{f}[q]; }}")
        for b in g.bspecs:
            if b.extra.get("deferred"):
                out.extend(deferred_lines[b.bid])
        if scan_bs:
            for si, b in enumerate(scan_bs):
                out.append(f"    i64 agg{b.bid};")
                out.append(f"    i64 wpos{b.bid} = wg_block_exclusive_scan(cnt{b.bid}, s_scan, &agg{b.bid});")
                out.append("    if (threadIdx.x < 32) {")
                out.append(f"      const i64 pre_ = wg_lookback(p.a{b.bid}_status, tile, agg{b.bid});")
                out.append(f"      if (threadIdx.x == 0) {{ s_toff[{si}] = pre_; if (tile == ntiles - 1) *p.a{b.bid}_total = pre_ + agg{b.bid}; }}")
                out.append("    }")
            out.append("    __syncthreads();")
            out.extend(mid or [])
            for si, b in enumerate(scan_bs):
                if not b.extra["staged"]:
                    out.append(f"    wpos{b.bid} += s_toff[{si}];")
            fine = ITEMS > 32 or any(b.extra.get("segstats") == "fine" for b in seg_bs)
            if seg_bs:
                # first item of this thread that starts a grain-wide chunk
                out.append("    i64 sgn_ = (p.cgmask >= 0) ? ((p.cbase + t0) & p.cgmask) : ((p.cbase + t0) % p.cgrain);")
                out.append("    sgn_ = sgn_ ? p.cgrain - sgn_ : 0;")
            if seg_bs and not fine:
                # grain >= ITEMS: at most one chunk start per thread; phase A
                # noted the thread-local append count there (c0s), so the
                # slot is written once, before phase B
                out.append(f"    if (c0s{seg_bs[0].bid} >= 0) {{")
                out.append("      const i64 g0_ = p.cbase + t0 + sgn_;")
                out.append("      const i64 ci0_ = (p.cgmask >= 0) ? ((g0_ >> __popcll(p.cgmask)) - (p.cbase >> __popcll(p.cgmask)))"
                           " : (g0_ / p.cgrain - p.cbase / p.cgrain);")
                for b in seg_bs:
                    si = scan_bs.index(b)
                    pos = f"wpos{b.bid} + s_toff[{si}]" if b.extra["staged"] else f"wpos{b.bid}"
                    out.append(f"      p.a{b.bid}_coff[ci0_] = {pos} + c0s{b.bid};")
                out.append("    }")
            out.append("#pragma unroll")
            out.append("    for (int j = 0; j < ITEMS; ++j) {")
            out.append("      const i64 li = t0 + j;")
            out.append("      if (li < n) {")
            out.append("        const i64 i = p.idx0 + li;")
            if seg_bs and fine:
                out.append("        if (j == sgn_) {")
                out.append("          const i64 ci_ = (p.cbase + li) / p.cgrain - p.cbase / p.cgrain;")
                for b in seg_bs:
                    si = scan_bs.index(b)
                    pos = f"wpos{b.bid} + s_toff[{si}]" if b.extra["staged"] else f"wpos{b.bid}"
                    out.append(f"          p.a{b.bid}_coff[ci_] = {pos};")
                out.append("          sgn_ += p.cgrain;")
                out.append("        }")
            out.extend(body_b)
            out.append("      }")
            out.append("    }")
            if any(b.extra["staged"] for b in scan_bs):
                out.append("    __syncthreads();")
                if claim:
                    # claim the next tile now: the atomic's latency overlaps
                    # the store phase, and the tile is unstarted only briefly
                    out.append("    i64 nclaim_ = 0; if (threadIdx.x == 0) nclaim_ = (i64)atomicAdd(p.tilectr, 1ULL);")
                for si, b in enumerate(scan_bs):
                    if not b.extra["staged"]:
                        continue
                    for f, kk in enumerate(b.extra["kinds"]):
                        out.append(f"    for (int q = threadIdx.x; q < (int)agg{b.bid}; q += BLOCK) "
                                   f"__stcs(p.a{b.bid}_{f} + s_toff[{si}] + q, s_ap{b.bid}_{f}[q]);")
                if claim:
                    out.append("    if (threadIdx.x == 0) s_tile[0] = nclaim_;")
                out.append("    __syncthreads();")
            elif claim:
                out.append("    if (threadIdx.x == 0) s_tile[0] = (i64)atomicAdd(p.tilectr, 1ULL);")
                out.append("    __syncthreads();")
        return out

    if ws:
        src.extend(ws_lines())
    elif scan_bs:
        # Dynamic tiles, claimed in order through an atomic counter (so every
        # predecessor a tile's look-back waits on is held by a running CTA).
        if SCAN_EARLY_CLAIM:
            src.append("  if (threadIdx.x == 0) s_tile[0] = (i64)atomicAdd(p.tilectr, 1ULL);")
            src.append("  __syncthreads();")
            src.append("  while (true) {")
        else:
            src.append("  while (true) {")
            src.append("    if (threadIdx.x == 0) s_tile[0] = (i64)atomicAdd(p.tilectr, 1ULL);")
            src.append("    __syncthreads();")
        src.append("    const i64 tile = s_tile[0];")
        src.append("    if (tile >= ntiles) break;")
        src.extend(decl_lines("", "    "))
        src.extend(load_lines("tile", "", "    "))
        src.extend(tile_body(claim=SCAN_EARLY_CLAIM))
        src.append("  }")
    elif pipe:
        # Bulk-async (TMA engine) column streaming: every full tile's column
        # chunks are copied HBM -> shared memory by cp.async.bulk, PIPE_STAGES
        # tiles ahead of the consumer, completion tracked by one mbarrier per
        # stage.  Bytes in flight no longer depend on registers/occupancy.
        src.append(f"  u64* wg_stage = wg_dyn_smem + {pipe_off // 8};")
        src.append("  const int PIPE_S = (int)p.pipe_stages;")
        src.append(f"  __shared__ __align__(8) u64 wg_bar[{PIPE_MAX_STAGES}];")
        src.append("  const i64 nfull = n / TILE;")
        src.append("  const i64 nmy = (nfull > (i64)blockIdx.x) ? (nfull - 1 - (i64)blockIdx.x) / gridDim.x + 1 : 0;")
        src.append("  if (threadIdx.x == 0) {")
        src.append(f"    for (int s_ = 0; s_ < {pipe_stages}; ++s_) wg_mbar_init(&wg_bar[s_], 1);")
        src.append("    wg_fence_mbar_init();")
        src.append("  }")
        src.append("  __syncthreads();")
        issue = ["      const i64 itile_ = (i64)blockIdx.x + k_ * gridDim.x;",
                 f"      u64* st_ = wg_stage + (u64)(k_ % {pipe_stages}) * {pipe_stage_bytes // 8};",
                 f"      wg_mbar_expect_tx(&wg_bar[k_ % {pipe_stages}], {pipe_stage_bytes});"]
        for (arr, st, kk, per, k, l, col), off in zip(loads, pipe_col_off):
            nb = BLOCK * ITEMS * per * SIZE[kk]
            issue.append(f"      wg_bulk_g2s((char*)st_ + {off}, {col} + itile_ * TILE * {per}, {nb}, &wg_bar[k_ % {pipe_stages}]);")
        src.append("  if (threadIdx.x == 0) {")
        src.append(f"    for (i64 k_ = 0; k_ < {pipe_stages} && k_ < nmy; ++k_) {{")
        src.extend(issue)
        src.append("    }")
        src.append("  }")
        src.append("  for (i64 kk_ = 0; kk_ < nmy; ++kk_) {")
        src.append("    const i64 tile = (i64)blockIdx.x + kk_ * gridDim.x;")
        src.append(f"    wg_mbar_wait(&wg_bar[kk_ % {pipe_stages}], (unsigned)((kk_ / {pipe_stages}) & 1));")
        src.extend(decl_lines("", "    "))
        src.append(f"    {{ const char* sg_ = (const char*)(wg_stage + (u64)(kk_ % {pipe_stages}) * {pipe_stage_bytes // 8});")
        for (arr, st, kk, per, k, l, col), off in zip(loads, pipe_col_off):
            cnt = f"ITEMS * {per}" if per > 1 else "ITEMS"
            src.append(f"      wg_lds_contig<{st}, {cnt}>((const {st}*)(sg_ + {off}) + threadIdx.x * {cnt}, {arr}); ")
        src.append("    }")
        src.append("    __syncthreads();")
        src.append(f"    if (threadIdx.x == 0 && kk_ + {pipe_stages} < nmy) {{")
        src.append("      wg_fence_proxy_async();")
        src.append(f"      const i64 k_ = kk_ + {pipe_stages};")
        src.extend("  " + x for x in issue)
        src.append("    }")
        # full tiles only: the per-row bound check is dropped (Black-Scholes
        # 0.910 -> 0.893 ms, Q1 0.481 -> 0.461) except for simd bodies,
        # where it measured slower (map 1.33 -> 1.46 ms)
        src.extend(tile_body(guard=not (PIPE_NOGUARD and not any(it.simd for it in iters))))
        src.append("  }")
        # the partial last tile (if any) through plain loads
        src.append("  if (nfull * TILE < n && (nfull % gridDim.x) == (i64)blockIdx.x) {")
        src.append("    const i64 tile = nfull;")
        src.extend(decl_lines("", "    "))
        src.extend(load_lines("tile", "", "    "))
        src.extend(tile_body())
        src.append("  }")
    elif PREFETCH:
        # register double buffering: the next tile's columns are in flight
        # while the current tile computes
        src.extend(decl_lines("", "  "))
        src.append("  i64 tile = blockIdx.x;")
        src.append("  if (tile < ntiles)")
        src.extend(load_lines("tile", "", "  "))
        src.append("  for (; tile < ntiles; tile += gridDim.x) {")
        src.extend(decl_lines("_nx", "    "))
        src.append("    const i64 ntile_ = tile + gridDim.x;")
        src.append("    if (ntile_ < ntiles)")
        src.extend(load_lines("ntile_", "_nx", "    "))
        src.extend(tile_body())
        for (arr, st, kk, per, k, l, col) in loads:
            cnt = f"ITEMS * {per}" if per > 1 else "ITEMS"
            src.append(f"#pragma unroll\n    for (int q = 0; q < {cnt}; ++q) {arr}[q] = {arr}_nx[q];")
        src.append("  }")
    else:
        src.append("  for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {")
        src.extend(decl_lines("", "    "))
        src.extend(load_lines("tile", "", "    "))
        src.extend(tile_body())
        src.append("  }")
    # epilogue: register caches, then shared-memory tables
    for b in g.bspecs:
        if b.extra.get("regcache"):
            src.extend(regcache_flush[b.bid])
        src.extend(b.extra.get("epilogue", []))
    if smem_flush:
        src.append("  __syncthreads();")
        src.extend("  " + fl for fl in smem_flush)
    # epilogue: distinct-key counts (one atomic per warp)
    for b in dict_bs:
        src.append(f"  {{ int c_ = wg_claims{b.bid};")
        src.append("#pragma unroll\n    for (int d = 16; d > 0; d >>= 1) c_ += __shfl_xor_sync(0xffffffffu, c_, d);")
        src.append(f"    if ((threadIdx.x & 31) == 0 && c_) atomicAdd(p.d{b.bid}_count, (unsigned long long)c_); }}")
    # epilogue: mergers
    if merger_bs:
        src.append("  __shared__ u64 s_red[32];")
        src.append("  __shared__ int s_redh[32];")
        src.append("  __shared__ int s_last;")
        for b in merger_bs:
            ks = leaves(b.kind.elem)
            F = len(ks)
            for f, kk in enumerate(ks):
                ct = CTYPE[kk]
                ident = c_literal(kk, internal_identity(b.kind.op, kk))
                src.append(f"  {{ int h_ = m{b.bid}_h; wg_block_fold<{ct}, {OPSTRUCT[b.kind.op]}<{ct}>>(m{b.bid}_{f}, h_, {ident}, ({ct}*)s_red, s_redh);")
                src.append(f"    if (threadIdx.x == 0) {{ p.m{b.bid}_part[(u64)blockIdx.x * {F + 1} + {f}] = wg_to_bits<{ct}>(m{b.bid}_{f});"
                           f" if ({f} == 0) p.m{b.bid}_part[(u64)blockIdx.x * {F + 1} + {F}] = (u64)h_; }} }}")
        # only thread 0 wrote this CTA's partials: it alone fences them
        # before taking the ticket (a CTA-wide fence stalled every warp)
        src.append("  if (threadIdx.x == 0) { __threadfence(); s_last = (atomicAdd(p.ticket, 1u) == gridDim.x - 1); }")
        src.append("  __syncthreads();")
        src.append("  if (s_last) {")
        src.append("    __threadfence();")
        for b in merger_bs:
            ks = leaves(b.kind.elem)
            F = len(ks)
            for f, kk in enumerate(ks):
                ct = CTYPE[kk]
                op = f"{OPSTRUCT[b.kind.op]}<{ct}>"
                ident = c_literal(kk, internal_identity(b.kind.op, kk))
                src.append(f"    {{ {ct} a_ = {ident}; int h_ = 0;")
                src.append(f"      for (unsigned q = threadIdx.x; q < gridDim.x; q += BLOCK) {{"
                           f" a_ = {op}::f(a_, wg_from_bits<{ct}>(__ldcg(p.m{b.bid}_part + (u64)q * {F + 1} + {f})));"
                           f" h_ |= (int)__ldcg(p.m{b.bid}_part + (u64)q * {F + 1} + {F}); }}")
                src.append(f"      wg_block_fold<{ct}, {op}>(a_, h_, {ident}, ({ct}*)s_red, s_redh);")
                # first launch into this merger writes the slot (no host-side init copy)
                src.append(f"      if (threadIdx.x == 0) {{ if (p.m{b.bid}_init) {{ p.m{b.bid}_slot[{f}] = wg_to_bits<{ct}>(a_);"
                           f" if ({f} == 0) p.m{b.bid}_slot[{F}] = (u64)h_; }}"
                           f" else if (h_) {{ p.m{b.bid}_slot[{f}] = wg_to_bits<{ct}>({op}::f(wg_from_bits<{ct}>(p.m{b.bid}_slot[{f}]), a_));"
                           f" p.m{b.bid}_slot[{F}] = 1; }} }} }}")
        # pinned host mirror of each slot plus the error word: the host reads
        # the result after a stream sync, with no copy-engine round trip
        src.append("    __syncthreads();")
        src.append("    if (threadIdx.x == 0) {")
        src.append("      const u64 e0_ = __ldcg((const u64*)p.err), e1_ = __ldcg((const u64*)p.err + 1);")
        for b in merger_bs:
            F = len(leaves(b.kind.elem))
            src.append(f"      if (p.m{b.bid}_mirror) {{ for (int f_ = 0; f_ <= {F}; ++f_) p.m{b.bid}_mirror[f_] = p.m{b.bid}_slot[f_];"
                       f" p.m{b.bid}_mirror[{F + 1}] = e0_; p.m{b.bid}_mirror[{F + 2}] = e1_; }}")
        src.append("      *p.ticket = 0;")
        src.append("    }")
        src.append("  }")
    src.append("}")
    source = "\n".join(src) + "\n"
    plan = KernelPlan(source=source, name=name, params=g.params, schedule=schedule, items=ITEMS, block=BLOCK,
                      smem=dyn_smem, builders=g.bspecs, scan_bids=[b.bid for b in scan_bs],
                      merger_bids=[b.bid for b in merger_bs], threads=BLOCK + 32 if ws else BLOCK)
    plan.pipe_stage_bytes = pipe_stage_bytes if pipe else 0
    plan.count_nodes = g.count_nodes
    plan.stat_nodes = g.stat_nodes
    plan.lit_nodes = {bid: set(v) for bid, v in g.lit_nodes.items()}
    plan.seg_bids = [b.bid for b in seg_bs]
    return plan


def _count_plan(g, lam, body_env, loads, iters, ITEMS, BLOCK, scan_bs, name):
    """Count-only pre-pass for appenders with data-dependent append counts
    (flatmap): runs the body with every merge disabled except the scan
    appenders' counters and adds the totals into one word per builder."""
    g.lines = []
    g.ind = 3
    g.phase = "count"
    g.ex(lam.body, body_env())
    body = g.lines
    unb = [b for b in scan_bs if b.extra.get("unbounded")]
    for b in unb:
        g.param(f"ct{b.bid}_total", "unsigned long long*", ("b", b.bid, "ctotal"))
    src = ['#include "weld_device.cuh"', f"#define BLOCK {BLOCK}", f"#define ITEMS {ITEMS}",
           "#define TILE (BLOCK * ITEMS)", "struct Params {"]
    src += [f"  {p_.ctype} {p_.name};" for p_ in g.params]
    src += ["};", f'extern "C" __global__ void __launch_bounds__(BLOCK) {name}(const Params p) {{',
            "  const i64 n = p.n;", "  const i64 ntiles = (n + TILE - 1) / TILE;"]
    if g.tabs:
        src.append("  " + " ".join(f"{t}_init();" for t in sorted(g.tabs)) + " __syncthreads();")
    src += [f"  i64 tc{b.bid} = 0;" for b in unb]
    src.append("  for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {")
    for (arr, st, kk, per, k, l, col) in loads:
        cnt = f"ITEMS * {per}" if per > 1 else "ITEMS"
        src.append(f"    alignas(16) {st} {arr}[{cnt}];")
    src.append("    { const i64 lt0_ = tile * TILE + (i64)threadIdx.x * ITEMS; const bool lfull_ = (lt0_ + ITEMS <= n);")
    for (arr, st, kk, per, k, l, col) in loads:
        cnt = f"ITEMS * {per}" if per > 1 else "ITEMS"
        if iters[k].strided:
            src.append(f"      for (int q = 0; q < ITEMS; ++q) {{ const i64 li_ = lt0_ + q; "
                       f"{arr}[q] = (li_ < n) ? {col}[p.it{k}_start + li_ * p.it{k}_stride] : ({st})0; }}")
        else:
            src.append(f"      if (lfull_) wg_load_contig<{st}, {cnt}>({col} + lt0_ * {per}, {arr});")
            src.append(f"      else {{ for (int q = 0; q < {cnt}; ++q) {{ const i64 e_ = lt0_ * {per} + q; "
                       f"{arr}[q] = (e_ < n * {per}) ? {col}[e_] : ({st})0; }} }}")
    src.append("    }")
    src.append("    const i64 t0 = tile * TILE + (i64)threadIdx.x * ITEMS;")
    src += [f"    i64 cnt{b.bid} = 0;" for b in scan_bs]
    src.append("#pragma unroll")
    src.append("    for (int j = 0; j < ITEMS; ++j) {")
    src.append("      const i64 li = t0 + j;")
    src.append("      if (li < n) {")
    src.append("        const i64 i = p.idx0 + li;")
    src.extend(body)
    src.append("      }")
    src.append("    }")
    src += [f"    tc{b.bid} += cnt{b.bid};" for b in unb]
    src.append("  }")
    for b in unb:
        src.append(f"  {{ i64 c_ = tc{b.bid};")
        src.append("    for (int d = 16; d > 0; d >>= 1) c_ += __shfl_xor_sync(0xffffffffu, c_, d);")
        src.append(f"    if ((threadIdx.x & 31) == 0 && c_) atomicAdd(p.ct{b.bid}_total, (unsigned long long)c_); }}")
    src.append("}")
    plan = KernelPlan(source="\n".join(src) + "\n", name=name, params=g.params, schedule="count", items=ITEMS,
                      block=BLOCK, smem=0, builders=g.bspecs, scan_bids=[b.bid for b in scan_bs], merger_bids=[])
    plan.pipe_stage_bytes = 0
    return plan


def is_flat_type(t):
    if isinstance(t, Scalar):
        return True
    if isinstance(t, Struct):
        return all(is_flat_type(f) for f in t.fields)
    return False


def _dict_params(g, b):
    vks = leaves(b.kind.value)
    P = dict(
        table=g.param(f"d{b.bid}_table", "u64*", ("b", b.bid, "table")),
        mask=g.param(f"d{b.bid}_mask", "u64", ("b", b.bid, "mask")),
        count=g.param(f"d{b.bid}_count", "unsigned long long*", ("b", b.bid, "count")),
        ocount=g.param(f"d{b.bid}_ocount", "unsigned long long*", ("b", b.bid, "ocount")),
        ocap=g.param(f"d{b.bid}_ocap", "u64", ("b", b.bid, "ocap")),
        okey=g.param(f"d{b.bid}_ok0", "u64*", ("b", b.bid, "okey", 0)),
        ovals=[g.param(f"d{b.bid}_ov{f}", "u64*", ("b", b.bid, "oval", f)) for f in range(len(vks))],
    )
    return P


def _regcache_decl(b, R):
    vks = leaves(b.kind.value)
    out = []
    for r in range(R):
        out.append(f"  u64 rk{b.bid}_{r} = WG_EMPTY_KEY;")
        for f, kk in enumerate(vks):
            out.append(f"  {CTYPE[kk]} rv{b.bid}_{r}_{f} = {c_literal(kk, internal_identity(b.kind.op, kk))};")
    return out


def _regcache_lines(b, R, ind="    "):
    """Level 0: a per-thread cache of R (key, value) slots in registers.
    Hits and first claims fold with no memory traffic at all; misses keep
    their pending flag for the shared/global levels."""
    kind = b.kind
    vks = leaves(kind.value)
    B = b.bid
    op = OPSTRUCT[kind.op]

    def fold(r):
        return " ".join(f"rv{B}_{r}_{f} = {op}<{CTYPE[kk]}>::f(rv{B}_{r}_{f}, dkv{B}_{f}[j]);"
                        for f, kk in enumerate(vks))

    # the sentinel-valued key (all ones) never enters the cache: an unclaimed
    # slot holds the sentinel too and would absorb its merges
    L = [f"{ind}#pragma unroll", f"{ind}for (int j = 0; j < ITEMS; ++j) {{",
         f"{ind}  if (!dkf{B}[j]) continue;", f"{ind}  const u64 k_ = dkk{B}[j];",
         f"{ind}  if (k_ == WG_EMPTY_KEY) continue;"]
    chain = []
    for r in range(R):
        chain.append(f"if (rk{B}_{r} == k_) {{ {fold(r)} }}")
    claim = []
    for r in range(R):
        claim.append(f"if (rk{B}_{r} == WG_EMPTY_KEY) {{ rk{B}_{r} = k_; {fold(r)} }}")
    L.append(f"{ind}  " + " else ".join(chain) + " else { " + " else ".join(claim) + " else { continue; } }")
    L.append(f"{ind}  dkf{B}[j] = false;")
    L.append(f"{ind}}}")
    return L


def _warpagg_lines(b, ind, flag, key, vals, outvals, glob, limit):
    """Fold lanes that merge the same key with a warp butterfly; the group
    leader applies the aggregate to the per-CTA shared-memory table.  Sets
    `glob` for lanes whose (aggregated) merge still needs the global table."""
    kind = b.kind
    vks = leaves(kind.value)
    sw = b.extra["slot_words"]
    ns = b.extra["smem_slots"]
    opc = OPCODE[kind.op]
    B = b.bid
    L = [f"{ind}{{",
         f"{ind}  const bool f_ = {flag}; const u64 k_ = {key};",
         f"{ind}  {glob} = f_;",
         f"{ind}  const unsigned fl_ = __ballot_sync(0xffffffffu, f_);",
         f"{ind}  const unsigned peers_ = __match_any_sync(0xffffffffu, k_) & fl_;",
         f"{ind}  const bool lead_ = f_ && ((__ffs(peers_) - 1) == lane_);",
         f"{ind}  const unsigned leaders_ = __ballot_sync(0xffffffffu, lead_);",
         f"{ind}  if (fl_ != 0 && __popc(leaders_) <= {limit}) {{"]
    for f, kk in enumerate(vks):
        L.append(f"{ind}    {outvals[f]} = {vals[f]};")
    L.append(f"{ind}    unsigned todo_ = leaders_;")
    L.append(f"{ind}    while (todo_) {{")
    L.append(f"{ind}      const int ld_ = __ffs(todo_) - 1; todo_ &= todo_ - 1;")
    L.append(f"{ind}      const unsigned grp_ = __shfl_sync(0xffffffffu, peers_, ld_);")
    L.append(f"{ind}      const bool in_ = (grp_ >> lane_) & 1u;")
    for f, kk in enumerate(vks):
        ct = CTYPE[kk]
        ident = c_literal(kk, internal_identity(kind.op, kk))
        L.append(f"{ind}      {{ const {ct} r_ = wg_warp_allfold<{ct}, {OPSTRUCT[kind.op]}<{ct}>>(in_ ? {vals[f]} : {ident});"
                 f" if (lane_ == ld_) {outvals[f]} = r_; }}")
    L.append(f"{ind}    }}")
    L.append(f"{ind}    {glob} = false;")
    L.append(f"{ind}    if (lead_) {{")
    L.append(f"{ind}      const int ss_ = wg_sht_find1(s_dk{B}, {sw}, {ns - 1}, k_);")
    L.append(f"{ind}      if (ss_ >= 0) {{")
    for f, kk in enumerate(vks):
        ct = CTYPE[kk]
        L.append(f"{ind}        wg_smem_fold<{opc}, {ct}>(({ct}*)(s_dk{B} + (u64)ss_ * {sw} + {1 + f}), {outvals[f]});")
    L.append(f"{ind}      }} else {{ {glob} = true; }}")
    L.append(f"{ind}    }}")
    L.append(f"{ind}  }} else {{")
    for f, kk in enumerate(vks):
        L.append(f"{ind}    {outvals[f]} = {vals[f]};")
    L.append(f"{ind}  }}")
    L.append(f"{ind}}}")
    return L


def _global_insert_lines(b, P, ind, flag, key, vals):
    kind = b.kind
    vks = leaves(kind.value)
    sw = b.extra["slot_words"]
    opc = OPCODE[kind.op]
    B = b.bid
    L = [f"{ind}if ({flag}) {{",
         f"{ind}  const i64 sl_ = wg_ht_find1({P['table']}, {sw}, {P['mask']}, {key}, wg_claims{B});"]
    L += _global_apply_lines(b, P, ind + "  ", key, vals)
    L.append(f"{ind}}}")
    return L


def _global_apply_lines(b, P, ind, key, vals):
    kind = b.kind
    vks = leaves(kind.value)
    sw = b.extra["slot_words"]
    opc = OPCODE[kind.op]
    L = [f"{ind}if (sl_ >= 0) {{"]
    for f, kk in enumerate(vks):
        ct = CTYPE[kk]
        L.append(f"{ind}  WgAtomicFold<{opc}, {ct}>::f(({ct}*)({P['table']} + (u64)sl_ * {sw} + {1 + f}), {vals[f]});")
    L.append(f"{ind}}} else {{")
    L.append(f"{ind}  const u64 o_ = atomicAdd({P['ocount']}, 1ULL);")
    L.append(f"{ind}  if (o_ < {P['ocap']}) {{ {P['okey']}[o_] = {key};")
    for f, kk in enumerate(vks):
        L.append(f"{ind}    {P['ovals'][f]}[o_] = wg_to_bits<{CTYPE[kk]}>({vals[f]});")
    L.append(f"{ind}  }} else {{ wg_raise(p.err, WG_ERR_INTERNAL, 1); }}")
    L.append(f"{ind}}}")
    return L


def dict_agg_source(kind, slot_words, S, pbits, name="wg_dagg"):
    """Second kernel of the partitioned dictmerger: insert the bucketed
    records into the HBM table in partition order (grid-stride over the
    partition-major bucket array), so the CTAs' working set is a few
    L2-resident table regions instead of the whole table."""
    vks = leaves(kind.value)
    V = len(vks)
    opc = OPCODE[kind.op]
    L = ['#include "weld_device.cuh"', "#define BLOCK 256", "struct Params {",
         "  u64* pk;"] + [f"  u64* pv{f};" for f in range(V)] + [
        "  unsigned long long* pcount; u64 pcap; u64 nparts;",
        "  u64* table; u64 mask; unsigned long long* count; unsigned long long* ocount; u64 ocap;",
        "  u64* ok0;"] + [f"  u64* ov{f};" for f in range(V)] + ["  i64* err;", "};",
        f'extern "C" __global__ void __launch_bounds__(BLOCK) {name}(const Params p) {{',
        "  int wg_claims = 0;",
        "  const u64 total = p.nparts * p.pcap;",
        "  for (u64 idx = blockIdx.x * (u64)BLOCK + threadIdx.x; idx < total; idx += (u64)gridDim.x * BLOCK) {",
        "    const u64 part = idx / p.pcap, r = idx - part * p.pcap;",
        "    if (r >= p.pcount[part]) continue;",
        "    const u64 k_ = p.pk[idx];"]
    for f, kk in enumerate(vks):
        L.append(f"    const {CTYPE[kk]} v{f}_ = wg_from_bits<{CTYPE[kk]}>(p.pv{f}[idx]);")
    L.append(f"    const i64 sl_ = wg_ht_find1(p.table, {slot_words}, p.mask, k_, wg_claims);")
    L += _agg_apply(vks, opc, slot_words, "    ", "k_", [f"v{f}_" for f in range(V)])
    L.append("  }")
    L.append("  { int c_ = wg_claims;")
    L.append("    for (int d = 16; d > 0; d >>= 1) c_ += __shfl_xor_sync(0xffffffffu, c_, d);")
    L.append("    if ((threadIdx.x & 31) == 0 && c_) atomicAdd(p.count, (unsigned long long)c_); }")
    L.append("}")
    return "\n".join(L) + "\n", 0


def _agg_apply(vks, opc, slot_words, ind, key, vals):
    L = [f"{ind}if (sl_ >= 0) {{"]
    for f, kk in enumerate(vks):
        ct = CTYPE[kk]
        L.append(f"{ind}  WgAtomicFold<{opc}, {ct}>::f(({ct}*)(p.table + (u64)sl_ * {slot_words} + {1 + f}), {vals[f]});")
    L.append(f"{ind}}} else {{")
    L.append(f"{ind}  const u64 o_ = atomicAdd(p.ocount, 1ULL);")
    L.append(f"{ind}  if (o_ < p.ocap) {{ p.ok0[o_] = {key};")
    for f, kk in enumerate(vks):
        L.append(f"{ind}    p.ov{f}[o_] = wg_to_bits<{CTYPE[kk]}>({vals[f]});")
    L.append(f"{ind}  }} else {{ wg_raise(p.err, WG_ERR_INTERNAL, 1); }}")
    L.append(f"{ind}}}")
    return L


def to_bits_c(kind, v):
    from .irtypes import to_bits
    return to_bits(kind, v)


def _deferred_dict_lines(g, b):
    """Apply the tile's pending dictmerger merges with the warp converged.

    Level 0: per-thread register cache (REGCACHE slots).  Level 1 (smem
    mode): lanes merging the same key are folded with a warp butterfly and
    only the group leader touches the per-CTA shared-memory table; warps
    seeing more than AGG_MAX_GROUPS distinct keys skip aggregation.  Level 2:
    every merge still pending goes to the global table with the first probe
    of all ITEMS rows issued up front (memory-level parallelism for tables
    far larger than L2)."""
    kind = b.kind
    vks = leaves(kind.value)
    sw = b.extra["slot_words"]
    P = _dict_params(g, b)
    B = b.bid
    R = b.extra.get("regcache", 0)
    L = ["    {", "      const int lane_ = threadIdx.x & 31;"]
    if R:
        L += _regcache_lines(b, R, "      ")
    if b.mode == "smem":
        L.append("#pragma unroll")
        L.append("      for (int j = 0; j < ITEMS; ++j) {")
        outv = [f"a{f}_" for f in range(len(vks))]
        for f, kk in enumerate(vks):
            L.append(f"        {CTYPE[kk]} a{f}_;")
        L.append("        bool g_;")
        L += _warpagg_lines(b, "        ", f"dkf{B}[j]", f"dkk{B}[j]", [f"dkv{B}_{f}[j]" for f in range(len(vks))],
                            outv, "g_", AGG_MAX_GROUPS)
        L.append(f"        dkf{B}[j] = g_;")
        for f, kk in enumerate(vks):
            L.append(f"        dkv{B}_{f}[j] = a{f}_;")
        L.append("      }")
        L.append("    }")
        return L
    if b.extra.get("part"):
        # Partitioned mode (cardinality >> L2).  Partition = the region of the
        # HBM table a key's home slot falls in (pbits top bits of the slot
        # index), so a second kernel that inserts the buckets in partition
        # order touches one L2-resident region at a time.  Records are
        # ranked per partition in shared memory so each tile issues one
        # global atomic per non-empty partition (not one per record).
        NP = 1 << b.extra["pbits"]
        pcount = g.param(f"d{B}_pcount", "unsigned long long*", ("b", B, "pcount"))
        pcap = g.param(f"d{B}_pcap", "u64", ("b", B, "pcap"))
        pshift = g.param(f"d{B}_pshift", "u64", ("b", B, "pshift"))
        pk = g.param(f"d{B}_pk", "u64*", ("b", B, "pk"))
        pvs = [g.param(f"d{B}_pv{f}", "u64*", ("b", B, "pv", f)) for f in range(len(vks))]
        V = len(vks)
        # (shared arrays are declared once at kernel scope: this block can be
        # emitted twice -- main tile loop and tail tile)
        decl = [f"  __shared__ unsigned s_ph{B}[{NP}], s_po{B}[{NP}];", f"  __shared__ u64 s_pb{B}[{NP}];",
                f"  __shared__ i64 s_sc{B}[33];"]
        b.extra["smem_decl"] = decl
        L.append(f"      unsigned pp_[ITEMS], pr_[ITEMS];")
        L.append(f"      for (int q = threadIdx.x; q < {NP}; q += BLOCK) s_ph{B}[q] = 0u;")
        L.append("      __syncthreads();")
        L.append("#pragma unroll")
        L.append("      for (int j = 0; j < ITEMS; ++j) {")
        L.append(f"        if (!dkf{B}[j]) continue;")
        L.append(f"        pp_[j] = (unsigned)((wg_mix64(dkk{B}[j]) & {P['mask']}) >> {pshift});")
        L.append(f"        pr_[j] = atomicAdd(&s_ph{B}[pp_[j]], 1u);")
        L.append("      }")
        L.append("      __syncthreads();")
        # tile-local counting sort by partition: exclusive offsets + one global
        # reservation per non-empty partition
        L.append(f"      {{ i64 tot_; for (int q0 = 0; q0 < {NP}; q0 += BLOCK) {{ const int q = q0 + threadIdx.x;")
        L.append(f"          const unsigned c_ = (q < {NP}) ? s_ph{B}[q] : 0u;")
        L.append(f"          const i64 ex_ = wg_block_exclusive_scan((i64)c_, s_sc{B}, &tot_);")
        L.append(f"          if (q < {NP}) {{ s_po{B}[q] = (unsigned)ex_ + (q0 ? s_po{B}[q0 - 1] + s_ph{B}[q0 - 1] : 0u);"
                 f" if (c_) s_pb{B}[q] = atomicAdd({pcount} + q, (unsigned long long)c_); }}")
        L.append("          __syncthreads(); } }")
        L.append("#pragma unroll")
        L.append("      for (int j = 0; j < ITEMS; ++j) {")
        L.append(f"        if (!dkf{B}[j]) continue;")
        L.append(f"        const unsigned lp_ = s_po{B}[pp_[j]] + pr_[j];")
        L.append(f"        s_rk{B}[lp_] = dkk{B}[j]; s_rp{B}[lp_] = (unsigned short)pp_[j];")
        for f, kk in enumerate(vks):
            L.append(f"        s_rv{B}_{f}[lp_] = wg_to_bits<{CTYPE[kk]}>(dkv{B}_{f}[j]);")
        L.append(f"        dkf{B}[j] = false;")
        L.append("      }")
        L.append("      __syncthreads();")
        # coalesced bucket writes: consecutive threads -> consecutive slots of
        # one partition's run
        L.append(f"      {{ const unsigned m_ = s_po{B}[{NP - 1}] + s_ph{B}[{NP - 1}];")
        L.append("        for (unsigned t_ = threadIdx.x; t_ < m_; t_ += BLOCK) {")
        L.append(f"          const unsigned pq_ = s_rp{B}[t_];")
        L.append(f"          const u64 pos_ = s_pb{B}[pq_] + (t_ - s_po{B}[pq_]);")
        L.append(f"          if (pos_ < {pcap}) {{")
        L.append(f"            const u64 at_ = (u64)pq_ * {pcap} + pos_;")
        L.append(f"            __stcs({pk} + at_, s_rk{B}[t_]);")
        for f in range(V):
            L.append(f"            __stcs({pvs[f]} + at_, s_rv{B}_{f}[t_]);")
        L.append("          } else {")
        L.append(f"            const u64 k_ = s_rk{B}[t_];")
        for f, kk in enumerate(vks):
            L.append(f"            const {CTYPE[kk]} v{f}_ = wg_from_bits<{CTYPE[kk]}>(s_rv{B}_{f}[t_]);")
        L.append(f"            const i64 sl_ = wg_ht_find1({P['table']}, {sw}, {P['mask']}, k_, wg_claims{B});")
        L += _global_apply_lines(b, P, "            ", "k_", [f"v{f}_" for f in range(V)])
        L.append("          }")
        L.append("        }")
        L.append("      }")
        L.append("      __syncthreads();")
    # global table: issue every first probe, then resolve
    L.append(f"      u64 h_[ITEMS], c_[ITEMS];")
    L.append("#pragma unroll")
    L.append(f"      for (int j = 0; j < ITEMS; ++j) {{ h_[j] = wg_ht_home(dkk{B}[j], {P['mask']}); "
             f"c_[j] = dkf{B}[j] ? WG_PROBE_LD({P['table']} + h_[j] * {sw}) : 0ULL; }}")
    L.append("#pragma unroll")
    L.append("      for (int j = 0; j < ITEMS; ++j) {")
    L.append(f"        if (!dkf{B}[j]) continue;")
    L.append(f"        const i64 sl_ = wg_ht_resolve1({P['table']}, {sw}, {P['mask']}, dkk{B}[j], h_[j], c_[j], wg_claims{B});")
    L += _global_apply_lines(b, P, "        ", f"dkk{B}[j]", [f"dkv{B}_{f}[j]" for f in range(len(vks))])
    L.append("      }")
    L.append("    }")
    return L


def _regcache_flush_lines(g, b):
    """Kernel epilogue: drain the register caches (warp-aggregated into the
    shared table in smem mode, else straight to the global table)."""
    R = b.extra.get("regcache", 0)
    if not R:
        return []
    vks = leaves(b.kind.value)
    P = _dict_params(g, b)
    B = b.bid
    L = ["  {", "    const int lane_ = threadIdx.x & 31;"]
    for r in range(R):
        vals = [f"rv{B}_{r}_{f}" for f in range(len(vks))]
        flag = f"(rk{B}_{r} != WG_EMPTY_KEY)"
        L.append("    {")
        if b.mode == "smem":
            outv = [f"a{f}_" for f in range(len(vks))]
            for f, kk in enumerate(vks):
                L.append(f"      {CTYPE[kk]} a{f}_;")
            L.append("      bool g_;")
            L += _warpagg_lines(b, "      ", flag, f"rk{B}_{r}", vals, outv, "g_", 32)
            L += _global_insert_lines(b, P, "      ", "g_", f"rk{B}_{r}", outv)
        else:
            L += _global_insert_lines(b, P, "      ", flag, f"rk{B}_{r}", vals)
        L.append("    }")
    L.append("  }")
    return L


def _pattern_switch(pat):
    """C expression selecting the init word for slot word index w_."""
    expr = f"0x{pat[-1] & 0xFFFFFFFFFFFFFFFF:016x}ULL"
    for i in range(len(pat) - 2, -1, -1):
        expr = f"(w_ == {i} ? 0x{pat[i] & 0xFFFFFFFFFFFFFFFF:016x}ULL : {expr})"
    return expr


def _capture_val(g: Gen, name, ty, val):
    """Bind a loop-invariant value from the enclosing scope as kernel params."""
    safe = "".join(ch if ch.isalnum() else "_" for ch in name)

    def go(t, v, path):
        tag = safe + "".join(f"_{q}" for q in path)
        if isinstance(t, Scalar):
            ct = {BOOL: "i64", I32: "i64", I64: "i64", F32: "double", F64: "double"}[t.kind]
            pn = g.param(f"c_{tag}", ct, ("cap", name) + tuple(path))
            if t.kind == BOOL:
                return S(f"({pn} != 0)", BOOL)
            if t.kind == I32:
                return S(f"((i32){pn})", I32)
            if t.kind == F32:
                return S(f"((float){pn})", F32)
            return S(pn, t.kind)
        if isinstance(t, Struct):
            return T([go(f, None, path + (i,)) for i, f in enumerate(t.fields)])
        if isinstance(t, Vec):
            ks = leaves(t.elem)
            cols = [g.param(f"c_{tag}_c{l}", f"const {STYPE[k]}*", ("capcol", name) + tuple(path) + (l,))
                    for l, k in enumerate(ks)]
            nn = g.param(f"c_{tag}_n", "i64", ("caplen", name) + tuple(path))
            return VRef(cols, nn, t.elem)
        if isinstance(t, Dict):
            kcols = [g.param(f"c_{tag}_k{l}", f"const {STYPE[k]}*", ("capdk", name) + tuple(path) + (l,))
                     for l, k in enumerate(leaves(t.key))]
            nn = g.param(f"c_{tag}_dn", "i64", ("capdn", name) + tuple(path))
            if isinstance(t.value, Vec):
                offs = g.param(f"c_{tag}_off", "const i64*", ("capdoff", name) + tuple(path))
                vcols = [g.param(f"c_{tag}_v{l}", f"const {STYPE[k]}*", ("capdv", name) + tuple(path) + (l,))
                         for l, k in enumerate(leaves(t.value.elem))]
            else:
                offs = None
                vcols = [g.param(f"c_{tag}_v{l}", f"const {STYPE[k]}*", ("capdv", name) + tuple(path) + (l,))
                         for l, k in enumerate(leaves(t.value))]
            return DRef(kcols, vcols, offs, nn, t.key, t.value)
        if isinstance(t, Builder):
            return None
        raise DeviceUnsupported(f"captured value of type {t}")

    try:
        return go(ty, val, ())
    finally:
        del go


# ---------------------------------------------------------------------------
# Static lowering (no device, no data): used by build() and the CPU test
# suite to prove every loop of a program lowers and compiles for sm_100a.


def static_plans(expr, env_types=None, externs=(), smem=True, lowcard=False, part=False,
                 count_only=False, counting=False, segstats=False):
    """Yield a KernelPlan per ``for`` loop in a typed program, deriving the
    iteration, builder and capture specs from types alone."""
    from weldmill.expr import walk, free_variables as _fv

    ext = {n: None for n in externs}
    plans = []
    nested = set()
    for node in walk(expr):
        if isinstance(node, For) and isinstance(node.func, Lambda):
            for inner in walk(node.func.body):
                if isinstance(inner, For):
                    nested.add(id(inner))
    for node in walk(expr):
        if not isinstance(node, For) or id(node) in nested or not isinstance(node.func, Lambda):
            continue
        iters = []
        for it in node.iters:
            vt = it.data.ty
            if not isinstance(vt, Vec):
                raise DeviceUnsupported("loop over a non-vector")
            iters.append(IterSpec(elem=vt.elem, simd=it.simd, strided=it.start is not None,
                                  kinds=leaves(vt.elem)))
        counter = [0]

        def mk(t):
            if isinstance(t, Builder):
                bid = counter[0]
                counter[0] += 1
                bs = BSpec(bid=bid, kind=t.kind)
                if isinstance(t.kind, DictMerger):
                    nw = key_layout(leaves(t.kind.key))[1]
                    sw = (1 if nw == 1 else 1 + nw) + len(leaves(t.kind.value))
                    bs.extra["slot_words"] = sw
                    bs.mode = "global"
                    if nw == 1 and part:
                        bs.extra.update(part=True, pbits=8, agg_S=0)
                    elif nw == 1 and smem:
                        bs.mode = "smem"
                        bs.extra["smem_slots"] = 512
                        bs.extra["pattern"] = [0xFFFFFFFFFFFFFFFF] + [0] * (sw - 1)
                        bs.extra["lowcard"] = lowcard
                if isinstance(t.kind, VecMerger):
                    bs.mode = "global"
                if isinstance(t.kind, VecBuilder) and segstats:
                    bs.extra["segstats"] = True
                return bs
            if isinstance(t, Struct):
                return tuple(mk(f) for f in t.fields)
            raise DeviceUnsupported(f"builders of type {t}")

        bstruct = mk(node.builders.ty)
        pnames = {p.name for p in node.func.params}
        caps = {}
        for name in sorted(_fv(node.func) - pnames):
            ty = None
            for n2 in walk(node.func.body):
                if isinstance(n2, Ident) and n2.name == name and n2.ty is not None:
                    ty = n2.ty
                    break
            if isinstance(ty, Function):
                continue
            caps[name] = (ty, None)
        plan = generate(node, iters, bstruct, caps, ext, "local", counting=counting)
        if count_only:
            # the count-only pre-pass of flatmap-shaped loops (fresh builder specs)
            if any(b.extra.get("unbounded") for b in plan.builders):
                counter[0] = 0
                plans.append(generate(node, iters, mk(node.builders.ty), caps, ext, "local", count_only=True))
            continue
        plans.append(plan)
    return plans


# ---------------------------------------------------------------------------
# Multi-GPU combine kernels (distributed.py): the reference folds builder
# partials in (step, chunk) key order at result() (builders.py:314-328,
# 435-450); across ranks the partials are folded in rank order with the same
# device fold functions the loop kernels use.


def combine_source(op, kinds):
    """Kernels folding G per-rank partials in rank order, for a builder of
    merge op `op` over leaves `kinds`:

    wg_fold_slots      merger slots (F value words + merged flag per rank)
                       -> one slot; a rank that merged nothing is skipped,
                       so an all-empty result keeps flag 0 (identity)
    wg_fold_chunks<f>  vecmerger leaf f: out[i] = fold over s of
                       chunks[s * L + i] (chunk s = rank s's slice)."""
    F = len(kinds)
    st = OPSTRUCT[op]
    L = ['#include "weld_device.cuh"',
         "struct SlotParams { const u64* parts; u64 G; u64* out; };",
         "struct ChunkParams { u64 out; u64 chunks; u64 L; u64 G; };",
         'extern "C" __global__ void wg_fold_slots(const SlotParams p) {',
         "  if (threadIdx.x != 0 || blockIdx.x != 0) return;",
         "  bool has = false;"]
    for f, k in enumerate(kinds):
        L.append(f"  {CTYPE[k]} a{f} = {CTYPE[k]}();")
    L += [f"  for (u64 r = 0; r < p.G; ++r) {{",
          f"    const u64* w = p.parts + r * {F + 1};",
          f"    if (!w[{F}]) continue;"]
    for f, k in enumerate(kinds):
        ct = CTYPE[k]
        L.append(f"    a{f} = has ? {st}<{ct}>::f(a{f}, wg_from_bits<{ct}>(w[{f}])) : wg_from_bits<{ct}>(w[{f}]);")
    L += ["    has = true;", "  }"]
    for f, k in enumerate(kinds):
        L.append(f"  p.out[{f}] = wg_to_bits<{CTYPE[k]}>(a{f});")
    L += [f"  p.out[{F}] = has ? 1ULL : 0ULL;", "}"]
    for f, k in enumerate(kinds):
        ct = CTYPE[k]
        L += [f'extern "C" __global__ void wg_fold_chunks{f}(const ChunkParams p) {{',
              f"  {ct}* out = ({ct}*)p.out;",
              f"  const {ct}* c = (const {ct}*)p.chunks;",
              "  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < p.L; i += (u64)gridDim.x * blockDim.x) {",
              f"    {ct} a = c[i];",
              f"    for (u64 s = 1; s < p.G; ++s) a = {st}<{ct}>::f(a, c[s * p.L + i]);",
              "    out[i] = a;",
              "  }",
              "}"]
    return "\n".join(L) + "\n"

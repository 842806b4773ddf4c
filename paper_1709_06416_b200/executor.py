"""``evaluate(e, env, config, externs) -> (Value, EvalStats)`` on the GPU.

Drop-in for the reference executor seam
``weldmill.engine.evaluate`` (/root/reference/pkg/src/weldmill/engine/run.py:1008-1074):
same signature, same ``Value``/``EvalStats`` return types, same ``EvalError``
subclasses.  The host walks the program's *control plane* (lets, struct
assembly, loop bounds, scalar glue between loops) and every ``for`` loop
runs as one NVRTC-compiled sm_100a kernel over device-resident columns
(codegen.py); builders live in HBM (builders_dev.py) and are finalised on
the device (sort / compaction / grouping).  There is no CPU fallback: IR
the device path does not lower raises ``DeviceUnsupported`` (an EvalError).
"""
from __future__ import annotations

import ctypes
import math
import struct as _struct
import threading
import weakref

import numpy as np

from . import _ref  # noqa: F401
from weldmill.engine import EngineConfig, EvalStats, Value
from weldmill.engine.builders import STRATEGIES, payload_bytes
from weldmill.engine.stats import note_evaluation
from weldmill.errors import (DivideByZero, EvalError, ExternCallUnknown, IndexOutOfBounds, IterationLimit,
                             KeyNotFound, MemoryLimitExceeded, UseAfterResult, ZipLengthMismatch)
from weldmill.expr import (Apply, BinaryOp, BitSelect, Broadcast, CastScalar, ExternCall, FieldAccess, For, Ident,
                           If, Iterate, IterSpec as XIterSpec, Lambda, Len, Let, Literal, Lookup, MakeStruct,
                           MakeVector, Merge, NewBuilder, Param as XParam, Result, Sort, ToVec, UnaryOp,
                           free_variables)

from . import runtime as rt
from . import semantics as sem
from .builders_dev import (_finish_small, AppenderDev, DDict, DGroups, DictDev, GroupDev, MergerDev, VecMergerDev,
                           Segment, dict_payload, finish_dict, finish_groups, gather_cols, sort_perm, tovec)
from .codegen import DEFER_DICT, PIPE_STAGES, BSpec, IterSpec, generate
from .columns import Col, DVec, to_device, to_payload, dvec_from_cols
from .irtypes import (BOOL, F32, F64, I32, I64, SIZE, identity_value, Builder, DeviceUnsupported as _DU, Dict, DictMerger, Function,
                      GroupBuilder, Merger, NPTYPE, Scalar, Simd, Struct, Vec, VecBuilder, VecMerger, is_flat, leaves,
                      to_bits)


class DeviceUnsupported(EvalError, _DU):
    """IR outside what the device executor lowers (no CPU fallback)."""


ERR_CLASSES = {1: DivideByZero, 2: IndexOutOfBounds, 3: IndexOutOfBounds, 4: KeyNotFound, 5: EvalError,
               6: DivideByZero, 7: IterationLimit, 8: EvalError, 9: ZipLengthMismatch, 10: EvalError}
ERR_TEXT = {1: "integer division by zero", 2: "lookup index {info} outside vector",
            3: "vecmerger index {info} out of range", 4: "key not in dictionary",
            5: "internal device error ({info})", 6: "integer remainder by zero",
            7: "iterate exceeded the iteration limit ({info} iterations)",
            9: "zipped iterations disagree (an iteration of length {info})",
            10: "iteration stride must be positive, got {info}"}


def device_error(code, info):
    """The EvalError subclass instance for a device error word (code, info)."""
    if code == 8:
        from .codegen import extern_error_text
        return EvalError(extern_error_text(info))
    cls = ERR_CLASSES.get(code, EvalError)
    return cls(ERR_TEXT.get(code, "device error {info}").format(info=info))


class HostVec:
    """A host vector not yet bound to the device (uploaded on first use)."""

    __slots__ = ("ty", "payload", "_dev", "n")

    def __init__(self, ty, payload):
        self.ty = ty
        self.payload = payload
        self._dev = None
        if isinstance(payload, (bytes, bytearray, memoryview)):
            self.n = _struct.unpack_from("<q", payload, 0)[0]
        elif isinstance(payload, tuple) and payload and all(isinstance(a, np.ndarray) for a in payload):
            self.n = int(payload[0].shape[0])
        else:
            self.n = len(payload)

    def __len__(self):
        return self.n

    def dev(self):
        if self._dev is None:
            self._dev = to_device(self.ty, self.payload)
        return self._dev

    def host_item(self, i):
        p = self.payload
        if isinstance(p, list):
            return p[i]
        if isinstance(p, np.ndarray):
            if p.dtype.names:
                return tuple(_py(p[nm][i]) for nm in p.dtype.names)
            return _py(p[i])
        return None


def _py(x):
    if isinstance(x, np.generic):
        return x.item()
    return x


class Closure:
    __slots__ = ("lam", "env")

    def __init__(self, lam, env):
        self.lam = lam
        self.env = env


class _Plan:
    __slots__ = ("plan", "kernel", "loop")


_plan_cache = {}
_plan_lock = threading.Lock()
_TICKET = [None]
_fv_cache = {}


class Ctx:
    def __init__(self, cfg: EngineConfig, externs, idx0=0):
        self._host_dicts = {}
        self.cfg = cfg
        self.externs = externs or {}
        self._ext_key = tuple(sorted(self.externs))
        self.traversals = 0
        self.allocs = 0
        self.tasks = 0
        self.live = 0
        self.peak = 0
        self.registry = []
        self.idx0 = idx0
        self.launches = 0
        self._ticket = None
        self.dirty = False
        self.rec = []         # launches of a replayable evaluation (see _Replay)
        # the reference's loop step (run.py:958-981): +1 before and after
        # every claimed top-level loop; appender segments are keyed by
        # (step, chunk) and the chunk is the loop row // grain_size
        self.step = 0
        self.cbase = 0
        self.reallocs = 0
        self._seg_pending = []
        self.counting = bool(cfg.count_evals)
        if self.counting:
            self._cnt_ord = {}
            self._cnt_text = []
            self._cnt = []
            self._cnt_nodes = []
            self.ev = self._ev_counting

    # -- count_evals (run.py:544-557, 1055-1060) ---------------------------
    def count_program(self, root):
        """Ordinals for every node the reference's _compile would wrap."""
        from weldmill.printer import print_expr
        for node in _compiled_nodes(root):
            if id(node) not in self._cnt_ord:
                self._cnt_ord[id(node)] = len(self._cnt)
                self._cnt.append(0)
                self._cnt_nodes.append(node)
                self._cnt_text.append(print_expr(node))

    def _ev_counting(self, e, env):
        k = self._cnt_ord.get(id(e))
        if k is not None:
            self._cnt[k] += 1
        return Ctx.ev(self, e, env)

    def count_extra(self, e, times):
        k = self._cnt_ord.get(id(e))
        if k is not None:
            self._cnt[k] += times

    def node_evals(self):
        totals = {}
        for text, n in zip(self._cnt_text, self._cnt):
            totals[text] = totals.get(text, 0) + n
        return totals

    # -- unhinted vecbuilder segments (builders.py:256-272) -----------------
    def seg_add(self, b, key, m):
        """m more appends into b's segment `key`: capacity doublings count as
        reallocations, capacity growth is charged to the builder."""
        if m <= 0:
            return
        old = b.segk.get(key, 0)
        new = old + m
        b.segk[key] = new
        self.reallocs += _seg_dbl(new) - _seg_dbl(old)
        grow = (_seg_cap(new) - _seg_cap(old)) * b.eb
        if grow:
            b.acct += grow
            self.alloc(grow)

    def seg_rows(self, b, lo, hi, k, claimed):
        """Appends of a launch that merges exactly k times per loop row, rows
        [lo, hi) of the loop."""
        if hi <= lo or k <= 0:
            return
        if not claimed:
            self.seg_add(b, (self.step, 0), (hi - lo) * k)
            return
        g = self.cfg.grain_size
        c0, c1 = lo // g, (hi - 1) // g
        if c0 == c1:
            self.seg_add(b, (self.step, c0), (hi - lo) * k)
            return
        self.seg_add(b, (self.step, c0), ((c0 + 1) * g - lo) * k)
        mid = c1 - c0 - 1
        if mid:
            self.reallocs += mid * _seg_dbl(g * k)
            grow = mid * _seg_cap(g * k) * b.eb
            b.acct += grow
            self.alloc(grow)
        self.seg_add(b, (self.step, c1), (hi - c1 * g) * k)

    def settle_segs(self):
        """Apply the device-side chunk statistics of scan-mode launches."""
        pend, self._seg_pending = self._seg_pending, []
        for b, step, k0, k1, out in pend:
            w = np.zeros(4, dtype=np.uint64)
            rt.d2h(w.ctypes.data, out.ptr, 32)
            self.reallocs += int(w[0])
            grow = int(w[1]) * b.eb
            if grow:
                b.acct += grow
                self.alloc(grow)
            self.seg_add(b, k0, int(w[2]))
            if k1 != k0:
                self.seg_add(b, k1, int(w[3]))

    # -- memory accounting (run.py:208-228) --------------------------------
    def alloc(self, n):
        self.live += n
        if self.live > self.peak:
            self.peak = self.live
        if self.live > self.cfg.memory_limit:
            raise MemoryLimitExceeded(f"engine memory {self.live} bytes exceeds limit {self.cfg.memory_limit}")

    def free(self, n):
        if self._seg_pending:
            self.settle_segs()
        self.live -= n

    def materialized(self, obj, nbytes, extra=(0, 0)):
        """extra = (objects, bytes) allocated earlier that live or die with
        obj (literal vectors a vecbuilder[vec[T]] result holds)."""
        self.alloc(nbytes)
        self.registry.append((obj, nbytes + extra[1], 1 + extra[0]))
        self.allocs += 1

    def ticket(self):
        """The last-CTA ticket of merger kernels.  Every such kernel resets it
        to 0 on exit and all loop kernels run in order on the library's
        stream, so one process-wide zeroed word serves every launch."""
        t = _TICKET[0]
        if t is None:
            with _plan_lock:
                if _TICKET[0] is None:
                    b = rt.alloc(8)
                    rt.memset(b.ptr, 0, 8)
                    _TICKET[0] = b
            t = _TICKET[0]
        self._ticket = t
        return t.ptr

    # -- device error word ---------------------------------------------------
    def check_device(self):
        if not self.dirty:
            return
        self.dirty = False
        code, info = rt.read_error()
        if code:
            raise device_error(code, info)

    # -- evaluation ------------------------------------------------------------
    _EV = {}

    def ev(self, e, env):
        f = Ctx._EV.get(type(e))
        if f is None:
            f = getattr(Ctx, "ev_" + type(e).__name__, None)
            if f is None:
                raise DeviceUnsupported(f"cannot evaluate node {type(e).__name__}")
            Ctx._EV[type(e)] = f
        return f(self, e, env)

    def ev_Literal(self, e, env):
        return sem.literal(e.ty.kind, e.value)

    def ev_Ident(self, e, env):
        try:
            return env[e.name]
        except KeyError:
            raise EvalError(f"unbound name {e.name!r}") from None

    def ev_Let(self, e, env):
        v = self.ev(e.value, env)
        env2 = dict(env)
        env2[e.name] = v
        return self.ev(e.body, env2)

    def ev_Lambda(self, e, env):
        return Closure(e, env)

    def ev_Apply(self, e, env):
        f = self.ev(e.func, env)
        if not isinstance(f, Closure):
            raise EvalError("attempted to call a non-function value")
        args = [self.ev(a, env) for a in e.args]
        if len(args) != len(f.lam.params):
            raise EvalError(f"function takes {len(f.lam.params)} arguments, got {len(args)}")
        env2 = dict(f.env)
        for p, a in zip(f.lam.params, args):
            env2[p.name] = a
        return self.ev(f.lam.body, env2)

    def ev_BinaryOp(self, e, env):
        if e.op == "&&":
            return bool(self.ev(e.rhs, env)) if self.ev(e.lhs, env) else False
        if e.op == "||":
            return True if self.ev(e.lhs, env) else bool(self.ev(e.rhs, env))
        a = self.ev(e.lhs, env)
        b = self.ev(e.rhs, env)
        t = e.lhs.ty
        if isinstance(t, Simd):
            return tuple(sem.binop(e.op, t.kind, x, y) for x, y in zip(a, b))
        return sem.binop(e.op, t.kind, a, b)

    def ev_UnaryOp(self, e, env):
        v = self.ev(e.operand, env)
        t = e.operand.ty
        if e.op == "!":
            return tuple(not x for x in v) if isinstance(t, Simd) else (not v)
        if isinstance(t, Simd):
            return tuple(sem.neg(t.kind, x) for x in v)
        return sem.neg(t.kind, v)

    def ev_If(self, e, env):
        return self.ev(e.on_true, env) if self.ev(e.cond, env) else self.ev(e.on_false, env)

    def ev_BitSelect(self, e, env):
        c = self.ev(e.cond, env)
        a = self.ev(e.on_true, env)
        b = self.ev(e.on_false, env)
        if isinstance(e.cond.ty, Simd):
            return tuple(x if ci else y for ci, x, y in zip(c, a, b))
        return a if c else b

    def ev_Broadcast(self, e, env):
        return (self.ev(e.value, env),) * 4

    def ev_CastScalar(self, e, env):
        v = self.ev(e.value, env)
        src = e.value.ty
        if isinstance(src, Simd):
            return tuple(sem.cast(src.kind, e.kind, x) for x in v)
        return sem.cast(src.kind, e.kind, v)

    def ev_MakeStruct(self, e, env):
        return tuple(self.ev(x, env) for x in e.items)

    def ev_FieldAccess(self, e, env):
        return self.ev(e.base, env)[e.ordinal]

    def ev_MakeVector(self, e, env):
        items = [self.ev(x, env) for x in e.items]
        hv = HostVec(e.ty, items)
        self.materialized(hv, payload_bytes(e.ty, items) if is_flat(e.ty.elem)
                          else 16 + sum(_value_bytes(e.ty.elem, x) for x in items))
        return hv

    def ev_Len(self, e, env):
        v = self.ev(e.coll, env)
        return len(v)

    def ev_Lookup(self, e, env):
        coll = self.ev(e.coll, env)
        idx = self.ev(e.index, env)
        if isinstance(coll, (HostVec, DVec)):
            n = len(coll)
            if not 0 <= idx < n:
                raise IndexOutOfBounds(f"index {idx} outside vector of length {n}")
            if isinstance(coll, HostVec):
                item = coll.host_item(idx)
                if item is not None:
                    return item
                coll = coll.dev()
            return _dvec_item(coll, idx)
        if isinstance(coll, (DDict, DGroups)):
            d = dict_payload(coll)
            try:
                return d[idx]
            except KeyError:
                raise KeyNotFound(f"key {idx!r} not in dictionary") from None
        raise EvalError("lookup into a non-collection")

    def ev_Iterate(self, e, env):
        state = self.ev(e.init, env)
        upd = self.ev(e.update, env)
        limit = self.cfg.max_iterations
        steps = 0
        try:
            while True:
                env2 = dict(upd.env)
                env2[upd.lam.params[0].name] = state
                state, go = self.ev(upd.lam.body, env2)
                steps += 1
                if not go:
                    return state
                if steps >= limit:
                    raise IterationLimit(f"iterate exceeded {limit} iterations")
        finally:
            if self.counting and not isinstance(e.update, Lambda):
                self.count_extra(e.update, steps - 1)    # run.py:875-882: evaluated per step

    def ev_ExternCall(self, e, env):
        fn = self.externs.get(e.name)
        if fn is None:
            raise ExternCallUnknown(f"no extern function {e.name!r} registered")
        args = [self.ev(a, env) for a in e.args]
        try:
            return fn(*args)
        except Exception as exc:
            raise EvalError(f"extern {e.name!r} failed: {exc}") from exc

    # -- builders ----------------------------------------------------------------
    def ev_NewBuilder(self, e, env):
        kind = e.kind
        if isinstance(kind, VecBuilder):
            hint = self.ev(e.arg, env) if e.arg is not None else None
            if hint is not None:
                if hint < 0:
                    raise EvalError(f"negative vector size hint {hint}")
                self.alloc(hint * _slot_bytes(kind.elem))
            if is_flat(kind.elem):
                b = AppenderDev(kind, leaves(kind.elem), hint)
            elif isinstance(kind.elem, Vec) and is_flat(kind.elem.elem):
                # vec[vec[T]] from fixed-length vectors: child leaves + a length
                b = AppenderDev(kind, leaves(kind.elem.elem), hint)
                b.nested = True
            else:
                b = AppenderDev(kind, None, hint)
            b.acct = hint * _slot_bytes(kind.elem) if hint is not None else 0
            b.eb = _slot_bytes(kind.elem)
            b.segk = {} if hint is None else None
            return b
        if isinstance(kind, Merger):
            return MergerDev(kind)
        if isinstance(kind, DictMerger):
            return DictDev(kind)
        if isinstance(kind, GroupBuilder):
            b = GroupDev(kind)
            b.acct = 0
            return b
        if isinstance(kind, VecMerger):
            init = self.ev(e.arg, env)
            dv = init.dev() if isinstance(init, HostVec) else init
            self.alloc(dv.n * _slot_bytes(kind.elem))
            b = VecMergerDev(kind, dv)
            b.acct = dv.n * _slot_bytes(kind.elem)
            return b
        raise EvalError(f"unknown builder kind {kind!r}")

    def ev_Merge(self, e, env):
        b = self.ev(e.builder, env)
        v = self.ev(e.value, env)
        if not hasattr(b, "pending"):
            raise EvalError("merge into a non-builder value")
        b.check()
        if isinstance(e.value.ty, Simd):
            b.pending.extend(v)
        else:
            b.pending.append(v)
        if getattr(b, "segk", None) is not None:
            self.seg_add(b, (self.step, 0), len(v) if isinstance(e.value.ty, Simd) else 1)
        b.pending_ty = e.value.ty.kind if isinstance(e.value.ty, Simd) else e.value.ty
        if isinstance(b.pending_ty, str):
            b.pending_ty = Scalar(b.pending_ty)
        return b

    def flush_pending(self, b):
        """Merges issued outside loops run as a tiny device loop, in order."""
        if not b.pending:
            return
        items = b.pending
        b.pending = []
        ty = Vec(b.pending_ty)
        hv = HostVec(ty, items)
        x = Ident("x", ty=b.pending_ty)
        bid = Ident("b", ty=Builder(b.kind))
        body = Merge(bid, x, ty=Builder(b.kind))
        lam = Lambda((XParam("b"), XParam("i"), XParam("x")), body)
        loop = For((XIterSpec(Ident("__pending", ty=ty)),), Ident("__b", ty=Builder(b.kind)), lam,
                   ty=Builder(b.kind))
        self.run_loop(loop, {"__pending": hv, "__b": b}, count_traversal=False)

    def ev_Result(self, e, env):
        b = self.ev(e.builder, env)
        return self.finish(b, e.builder.ty)

    def finish(self, b, ty):
        if isinstance(b, tuple):
            return tuple(self.finish(x, t) for x, t in zip(b, ty.fields))
        if not hasattr(b, "pending"):
            raise EvalError("result() applied to a non-builder value")
        self.flush_pending(b)
        b.consume()
        kind = b.kind
        if isinstance(kind, Merger):
            if self.dirty and b.launched:
                # the merger's slot and the error word come back in one sync
                err = []
                v = b.read(err)
                self.dirty = False
                code, info = err[0]
                if code:
                    raise device_error(code, info)
                return v
            self.check_device()
            return b.read()
        if isinstance(kind, VecBuilder):
            if self._seg_pending:
                self.settle_segs()
            if b.kinds is None:
                raise DeviceUnsupported(f"vecbuilder[{kind.elem}] (nested element types) on the device")
            if not b.segments:
                cols = [Col.alloc(k, 0) for k in b.kinds]
                n = 0
            else:
                cols, n = b.concat()
            self.free(getattr(b, "acct", 0))
            if getattr(b, "nested", False):
                # vec[vec[T]]: n child elements in fixed-length runs
                L = getattr(b, "nested_len", 1)
                nv = n // L if L else 0
                offs = Col.alloc(I64, nv + 1)
                rt.call("wg_iota_i64", offs.ptr, nv + 1, L)
                from .columns import ListLayout, layout_from_cols
                out = DVec(kind.elem, nv, ListLayout(offs, layout_from_cols(kind.elem.elem, cols), n))
                self.materialized(out, 16 + nv * 16 + n * _slot_bytes(kind.elem.elem), getattr(b, "lit_acct", (0, 0)))
                return out
            out = dvec_from_cols(kind.elem, n, cols)
            self.materialized(out, 16 + n * _slot_bytes(kind.elem))
            return out
        if isinstance(kind, VecMerger):
            self.free(getattr(b, "acct", 0))
            out = dvec_from_cols(kind.elem, b.n, b.cols)
            self.materialized(out, 16 + b.n * _slot_bytes(kind.elem))
            return out
        if isinstance(kind, DictMerger):
            if b.table is None:
                b.ensure(1)
            d = _finish_small(b, Dict(kind.key, kind.value))
            self._raise_sync_err(b)
            b.small = d is not None
            if d is None:
                self._settle(b)
                d = finish_dict(b, Dict(kind.key, kind.value))
                self._raise_sync_err(b)
            else:
                self.dirty = False        # the finish synchronised after every launch and read the error word
            _first_zero_sign(b, d)
            self.materialized(d, 16 + d.n * (16 + _slot_bytes(kind.key) + _slot_bytes(kind.value)))
            return d
        if isinstance(kind, GroupBuilder):
            self.free(getattr(b, "acct", 0))     # GroupBuilderState.result releases its rows (builders.py:480)
            g = finish_groups(b, Dict(kind.key, Vec(kind.value)))
            self.materialized(g, 16 + g.n * (16 + _slot_bytes(kind.key) + 16) + g.vals.n * _slot_bytes(kind.value))
            return g
        raise EvalError(f"unknown builder kind {kind!r}")

    def _raise_sync_err(self, b):
        code, info = getattr(b, "sync_err", (0, 0))
        b.sync_err = (0, 0)
        if code:
            self.dirty = False
            raise device_error(code, info)

    def ev_ToVec(self, e, env):
        d = self.ev(e.mapping, env)
        if not isinstance(d, (DDict, DGroups)):
            raise EvalError("tovec of a non-dictionary")
        out = tovec(d, e.ty.elem)
        self.materialized(out, payload_bytes_dvec(e.ty, out))
        return out

    def ev_Sort(self, e, env):
        v = self.ev(e.vec, env)
        dv = v.dev() if isinstance(v, HostVec) else v
        self.traversals += 1
        n = dv.n
        if n == 0:
            out = dv
        else:
            keyf = e.key
            if not isinstance(keyf, Lambda):
                raise DeviceUnsupported("sort key must be a lambda literal")
            kty = keyf.body.ty
            # key column(s) by a device map loop: for(v, vecbuilder[K], (b,i,x) => merge(b, key(x)))
            kb = AppenderDev(VecBuilder(kty), leaves(kty), n)
            xname = keyf.params[0].name
            body = Merge(Ident("__kb", ty=Builder(VecBuilder(kty))),
                         Let(xname, Ident("__x", ty=e.vec.ty.elem), keyf.body, ty=kty),
                         ty=Builder(VecBuilder(kty)))
            lam = Lambda((XParam("__kb"), XParam("__i"), XParam("__x")), body)
            loop = For((XIterSpec(Ident("__v", ty=e.vec.ty)),), Ident("__kbs", ty=Builder(VecBuilder(kty))),
                       lam, ty=Builder(VecBuilder(kty)))
            env2 = dict(env)
            env2.update({"__v": dv, "__kbs": kb})
            self.run_loop(loop, env2, count_traversal=False)
            kcols, _ = kb.concat()
            perm = sort_perm(kcols, n)
            out = dvec_from_cols(dv.elem, n, gather_cols(dv.cols, perm, n))
        self.materialized(out, payload_bytes_dvec(Vec(dv.elem), out))
        return out

    # -- loops ---------------------------------------------------------------------
    def ev_For(self, e, env):
        return self.run_loop(e, env)

    def run_loop(self, e, env, count_traversal=True, part=None):
        """Run one `for` loop.  count_traversal=False marks a synthetic loop
        (pending merges, dict regrowth, sort keys).  part=(lo, total, first,
        last): this launch covers iterations [lo, lo + count) of a loop of
        `total` iterations run in slices (the streaming path)."""
        _claim_loop_id(e)
        datas, specs, windows = [], [], []
        count = None
        for it in e.iters:
            d = self.ev(it.data, env)
            if not isinstance(d, (HostVec, DVec)):
                raise EvalError("loop over a non-vector value")
            length = len(d)
            elem = d.ty.elem if isinstance(d, HostVec) else d.elem
            if it.simd:
                n = length // 4
                win = (0, 1)
            elif it.start is None:
                n = length
                win = (0, 1)
            else:
                s = self.ev(it.start, env)
                end = self.ev(it.end, env)
                st = self.ev(it.stride, env)
                if st < 1:
                    raise EvalError(f"iteration stride must be positive, got {st}")
                if not (0 <= s <= end <= length):
                    raise IndexOutOfBounds(f"iteration bounds [{s}, {end}) outside vector of length {length}")
                n = (end - s + st - 1) // st
                win = (s, st)
            if count is None:
                count = n
            elif count != n:
                raise ZipLengthMismatch(f"zipped iterations disagree: {count} vs {n}")
            datas.append(d)
            windows.append(win)
            ks = _leaves_of(elem)
            if ks is None:
                raise DeviceUnsupported(f"iterating vec[{elem}] on the device")
            aligned = False
            if win[1] == 1 and count:
                dv = d.dev() if isinstance(d, HostVec) else d
                off = win[0]
                aligned = True
                for c in dv.cols:
                    if (c.ptr + off * SIZE[c.kind]) & 15:
                        aligned = False
                        break
            specs.append(IterSpec(elem=elem, simd=it.simd, strided=(win[1] != 1), kinds=ks, aligned=aligned))
        builders = self.ev(e.builders, env)
        if count == 0:
            return builders
        # synthetic loops (pending merges, dict regrowth, sort keys) are not
        # loops of the program: no traversal, no step, no segment accounting
        if part is not None:
            lo, total, first, last = part
            synthetic = False
        else:
            lo, total, first, last = 0, count, True, True
            synthetic = not count_traversal
        if first and not synthetic:
            self.traversals += len(e.iters)
        claimed = not synthetic and total > 1
        if claimed and first:
            self.step += 1
        saved = (self._synthetic, self._claimed, self.cbase)
        self._synthetic, self._claimed, self.cbase = synthetic, claimed, lo
        try:
            return self._run_loop(e, env, builders, specs, datas, windows, count)
        finally:
            self._synthetic, self._claimed, self.cbase = saved
            if claimed and last:
                self.step += 1

    _synthetic = False
    _claimed = False

    def _run_loop(self, e, env, builders, specs, datas, windows, count):
        lam = e.func
        lenv = env
        if not isinstance(lam, Lambda):
            f = self.ev(lam, env)
            if not isinstance(f, Closure):
                raise EvalError("loop body is not a function")
            lam, lenv = f.lam, f.env
            if self.counting:
                self.count_extra(e.func, count - 1)    # run.py:875-882 evaluates it per iteration
        blist = []
        _collect_builders(builders, blist)
        for b in blist:
            b.check()
            if isinstance(b, DictDev):
                self._settle(b)
            self.flush_pending(b)
        # loop-invariant captures
        fv = _fv_cache.get(id(lam))
        if fv is None or fv[0] is not lam:
            pn = {p.name for p in lam.params}
            names = sorted(free_variables(lam) - pn)
            fv = _fv_cache[id(lam)] = (lam, [(nm, _type_of(None, lam, nm)) for nm in names])
        captures = {}
        for name, cty in fv[1]:
            if name not in lenv:
                raise EvalError(f"unbound name {name!r}")
            captures[name] = (cty, lenv[name])

        strategy = self.cfg.strategy
        # dictmerger variant chosen from the data on a loop's first run: the
        # first SKETCH_ROWS rows run as a launch of their own (low-
        # cardinality variant, correct for any cardinality), the distinct
        # count they produced picks the variant -- and the table size -- for
        # the remaining rows (all builders accept a loop split into
        # consecutive launches: merges are commutative, appends land in order)
        dicts = [(q, b) for q, b in enumerate(_builder_order(builders)) if isinstance(b, DictDev)]
        from .builders_dev import _SIZE_HINTS
        if (dicts and strategy != "global" and count >= 4 * SKETCH_ROWS and not any(s.simd for s in specs)
                and any(_SIZE_HINTS.get((id(e), q)) is None for q, _ in dicts)):
            self._launch_loop(e, lam, specs, datas, windows, SKETCH_ROWS, builders, captures, strategy,
                              assume_lowcard=True)
            for q, st in dicts:
                if _SIZE_HINTS.get((id(e), q)) is not None:
                    continue
                self._settle(st)
                d, _ = st.read_counters()
                est = d if d * 32 <= SKETCH_ROWS else min(1 << 24, max(d, (d * count) // SKETCH_ROWS))
                _SIZE_HINTS[(id(e), q)] = est
                if est * 2 > st.cap:
                    self._dict_regrow_(st, 0, want=est)
            rest = [(s0 + SKETCH_ROWS * st_, st_) for s0, st_ in windows]
            saved = self.idx0, self.cbase
            self.idx0 = saved[0] + SKETCH_ROWS
            self.cbase = saved[1] + SKETCH_ROWS
            try:
                self._launch_loop(e, lam, specs, datas, rest, count - SKETCH_ROWS, builders, captures, strategy)
            finally:
                self.idx0, self.cbase = saved
            return builders
        self._launch_loop(e, lam, specs, datas, windows, count, builders, captures, strategy)
        self._last_builders = builders
        return builders

    def _launch_loop(self, e, lam, specs, datas, windows, count, builders, captures, strategy, assume_lowcard=False):
        bstruct, bmap = _bspecs(builders, strategy, count, loop_id=id(e), assume_lowcard=assume_lowcard,
                                   grain=self.cfg.grain_size)
        # The expression identities fix every type in the loop; only the
        # runtime choices (strides, alignment, builder modes, externs) vary.
        counting = self.counting and self._counts_body(lam)
        key = (id(e), id(lam), tuple((s.strided, s.aligned) for s in specs), _bsig(bstruct), self._ext_key, counting)
        with _plan_lock:
            cached = _plan_cache.get(key)
        if cached is None:
            plan = generate(e if lam is e.func else _with_func(e, lam), specs, bstruct, captures,
                            self.externs, strategy, counting=counting)
            plan.key_id = id(e)
            kern = rt.get_kernel(plan.source, plan.name)
            cached = (plan, kern, e, lam)
            with _plan_lock:
                if len(_plan_cache) > 4096:
                    _plan_cache.clear()
                _plan_cache[key] = cached
        plan, kern = cached[0], cached[1]
        sizes = None
        if any(b.extra.get("unbounded") for b in plan.builders):
            # flatmap: appends inside data-dependent nested loops -- size the
            # output with a count-only pre-pass of the same body
            ckey = key + ("count",)
            with _plan_lock:
                cc = _plan_cache.get(ckey)
            if cc is None:
                cbs, _ = _bspecs(builders, strategy, count, loop_id=id(e), assume_lowcard=assume_lowcard,
                                   grain=self.cfg.grain_size)
                cplan = generate(e if lam is e.func else _with_func(e, lam), specs, cbs, captures, self.externs,
                                 strategy, count_only=True)
                cc = (cplan, rt.get_kernel(cplan.source, cplan.name))
                with _plan_lock:
                    _plan_cache[ckey] = cc
            sizes = self._count_pass(cc[0], cc[1], count, datas, windows, bmap, captures)
        self.launch(plan, kern, count, datas, windows, builders, bmap, captures, sizes=sizes)

    def _body_stats(self, plan, bmap):
        """EvalStats events of the loop body (nested loops' traversals,
        literal vectors materialised per execution, run.py:781-789, 948):
        counted on the device, accounted here in the reference's terms.  A
        literal merged into a vecbuilder[vec[T]] survives in its result."""
        arr = np.zeros(len(plan.stat_nodes), dtype=np.uint64)
        rt.d2h(arr.ctypes.data, self._scnt_buf.ptr, arr.nbytes)
        keep = {}
        for bid, ids in plan.lit_nodes.items():
            for i in ids:
                keep[i] = bmap[bid]
        for (what, node), c in zip(plan.stat_nodes, arr):
            c = int(c)
            if not c:
                continue
            if what == "trav":
                self.traversals += c * len(node.iters)
                continue
            nbytes = c * payload_bytes(node.ty, [0] * len(node.items)) if is_flat(node.ty.elem) else None
            if nbytes is None:
                raise DeviceUnsupported("vector literal of non-scalar elements in a loop body")
            self.alloc(nbytes)
            self.allocs += c
            owner = keep.get(id(node))
            if owner is not None:
                owner.lit_acct = getattr(owner, "lit_acct", (0, 0))
                owner.lit_acct = (owner.lit_acct[0] + c, owner.lit_acct[1] + nbytes)
            else:
                self.registry.append((None, nbytes, c))

    def _counts_body(self, lam):
        from weldmill.expr import walk
        return any(id(x) in self._cnt_ord for x in walk(lam.body))

    def _count_pass(self, plan, kern, count, datas, windows, bmap, captures):
        """Launch the count-only kernel.  Returns {builder id: appends}."""
        tile = plan.block * plan.items
        ntiles = (count + tile - 1) // tile
        grid = max(1, min(ntiles, rt.sm_count() * kern.blocks_per_sm(plan.block, 0)))
        unb = [b for b in plan.builders if b.extra.get("unbounded")]
        tot = rt.alloc(8 * len(unb) + 8)
        rt.memset(tot.ptr, 0, 8 * len(unb))
        res = {b.bid: ("ctotal", tot.ptr + 8 * q) for q, b in enumerate(unb)}
        vals = {p.name: self._param_value(p.key, count, datas, windows, bmap, res, captures, grid, None)
                for p in plan.params}
        kern.launch(grid, plan.block, b"".join(_pack(p.ctype, vals[p.name]) for p in plan.params), 0)
        self.launches += 1
        self.dirty = True
        self.check_device()
        arr = np.zeros(len(unb), dtype=np.int64)
        rt.d2h(arr.ctypes.data, tot.ptr, arr.nbytes)
        return {b.bid: int(arr[q]) for q, b in enumerate(unb)}

    def launch(self, plan, kern, count, datas, windows, builders, bmap, captures, sizes=None):
        items = plan.items
        tile = plan.block * items
        ntiles = (count + tile - 1) // tile
        smem = plan.smem
        stages = 0
        if plan.pipe_stage_bytes:
            # most pipeline stages that keep the occupancy of a 2-stage pipe
            base = kern.blocks_per_sm(plan.block, plan.smem + 2 * plan.pipe_stage_bytes)
            stages = 2
            for s_ in range(PIPE_STAGES, 2, -1):
                sm_ = plan.smem + s_ * plan.pipe_stage_bytes
                if sm_ <= 200 * 1024 and kern.blocks_per_sm(plan.block, sm_) >= base:
                    stages = s_
                    break
            smem = plan.smem + stages * plan.pipe_stage_bytes
        nthr = plan.threads or plan.block
        occ = kern.blocks_per_sm(nthr, smem)
        grid = max(1, min(ntiles, rt.sm_count() * occ))
        self.tasks += grid
        # per-launch builder resources
        res = {}
        segstats = []
        segacct = not self._synthetic
        for b in plan.builders:
            st = bmap[b.bid]
            if isinstance(b.kind, (VecBuilder, GroupBuilder)):
                seg_model = segacct and getattr(st, "segk", None) is not None
                if b.mode == "direct":
                    per = b.k * b.extra.get("nested_len", 1)
                    if b.extra.get("nested"):
                        st.nested_len = b.extra["nested_len"]
                    seg = st.new_segment(count * per, True)
                    res[b.bid] = seg
                    if seg_model:
                        self.seg_rows(st, self.cbase, self.cbase + count, b.k, self._claimed)
                    elif getattr(st, "segk", None) is None:
                        self._acct_append(st, count * per)
                elif b.mode == "scan":
                    cap = sizes[b.bid] if (b.k is None or (sizes and b.bid in sizes)) else count * b.k
                    seg = st.new_segment(cap, False)
                    status = rt.alloc(8 * max(ntiles, 1))
                    rt.memset(status.ptr, 0, 8 * max(ntiles, 1))
                    res[b.bid] = (seg, status)
                    if b.bid in plan.seg_bids:
                        g_ = self.cfg.grain_size
                        c0, c1 = self.cbase // g_, (self.cbase + count - 1) // g_
                        coff = rt.alloc(8 * (c1 - c0 + 1))
                        rt.memset(coff.ptr, 0, 8 * (c1 - c0 + 1))
                        res[("coff", b.bid)] = coff
                        if seg_model:
                            segstats.append((st, seg, coff, c0, c1))
                    elif getattr(st, "segk", None) is None:
                        self._acct_append(st, cap)
            elif isinstance(b.kind, DictMerger):
                st.ensure(count * max(1, b.extra.get("maxm", 1)), hint_key=(plan.key_id, b.bid))
                if len(st.kks) == 1 and st.kks[0] in (F32, F64):
                    # first -0.0 / +0.0 rows of this launch (synthetic replays
                    # re-insert canonical keys and do not count)
                    zb = rt.alloc(16)
                    rt.memset(zb.ptr, 0xFF, 16)
                    st.zrow_cur = zb
                    if not self._synthetic:
                        st.zrows = getattr(st, "zrows", []) + [zb]
                if b.extra.get("part") and b.extra.get("deferred"):
                    st.ensure_part(count, 1 << b.extra["pbits"])
                    st.pbits = b.extra["pbits"]
        tilectr = None
        if plan.schedule == "scan":
            tilectr = rt.alloc(8)
            rt.memset(tilectr.ptr, 0, 8)

        if plan.count_nodes:
            self._cnt_buf = rt.alloc(8 * len(plan.count_nodes))
            rt.memset(self._cnt_buf.ptr, 0, 8 * len(plan.count_nodes))
        if plan.stat_nodes:
            self._scnt_buf = rt.alloc(8 * len(plan.stat_nodes))
            rt.memset(self._scnt_buf.ptr, 0, 8 * len(plan.stat_nodes))
        packer = getattr(plan, "_packer", None)
        if packer is None:
            # every parameter is one 8-byte word (f64 or a masked integer)
            dbl = [p.ctype == "double" for p in plan.params]
            packer = plan._packer = (_struct.Struct("<" + "".join("d" if d else "Q" for d in dbl)), dbl)
        words = []
        for p, d in zip(plan.params, packer[1]):
            v = stages if p.name == "pipe_stages" else \
                self._param_value(p.key, count, datas, windows, bmap, res, captures, grid, tilectr)
            if d:
                words.append(float(v))
            else:
                if isinstance(v, float):
                    raise EvalError(f"internal: float for {p.ctype} parameter")
                words.append(int(v) & 0xFFFFFFFFFFFFFFFF)
        blob = packer[0].pack(*words)
        kern.launch(grid, nthr, blob, smem)
        self.launches += 1
        self.dirty = True
        if self.rec is not None:
            outs = {}
            ok = not (sizes is not None or segstats or plan.count_nodes or plan.stat_nodes)
            for b in plan.builders:
                st = bmap[b.bid]
                if isinstance(st, MergerDev):
                    continue
                if (isinstance(st, DictDev) and not b.extra.get("part") and len(plan.builders) == 1
                        and all(k in (BOOL, I32, I64) for k in st.kks)):
                    # replayed with its table re-initialised (the buffers
                    # the blob points at stay owned by the replay)
                    outs[id(st)] = "dict"
                    continue
                if (isinstance(st, AppenderDev) and isinstance(b.kind, VecBuilder) and b.mode == "direct"
                        and not b.extra.get("nested") and len(st.segments) == 1):
                    # replayed with fresh output columns patched into the blob
                    idx = [next((i for i, p in enumerate(plan.params) if p.key == ("b", b.bid, "col", f)), None)
                           for f in range(len(st.kinds))]
                    if None in idx:
                        ok = False
                        break
                    outs[id(st)] = (idx, st.segments[0].cap)
                    continue
                ok = False
                break
            if not ok:
                self.rec = None
            else:
                self.rec.append((kern, grid, nthr, blob, smem, outs))
        for st, seg, coff, c0, c1 in segstats:
            out = rt.alloc(32)
            rt.call("wg_seg_stats", coff.ptr, c1 - c0 + 1, seg.total_buf.ptr, out.ptr)
            self.launches += 1
            if self._claimed:
                self._seg_pending.append((st, self.step, (self.step, c0), (self.step, c1), out))
            else:
                self._seg_pending.append((st, self.step, (self.step, 0), (self.step, 0), out))
        if plan.count_nodes:
            arr = np.zeros(len(plan.count_nodes), dtype=np.uint64)
            rt.d2h(arr.ctypes.data, self._cnt_buf.ptr, arr.nbytes)
            for node, c in zip(plan.count_nodes, arr):
                self.count_extra(node, int(c))
        if plan.stat_nodes and not self._synthetic:
            self._body_stats(plan, bmap)
        # partitioned dictmergers: fold every bucket, merge into the HBM table
        for b in plan.builders:
            if isinstance(b.kind, DictMerger) and b.extra.get("part") and b.extra.get("deferred"):
                self._dict_aggregate(bmap[b.bid], b)
        # dictmerger overflow (merges spilled past the table) is settled
        # lazily -- before the next launch into the builder or at result() --
        # so a loop's launch does not wait on the device
        for b in plan.builders:
            if isinstance(b.kind, DictMerger):
                bmap[b.bid].spill_pending = True
        self._keep = (tilectr, res)

    def _settle(self, st):
        """Grow the table and replay spilled merges, if the last launches
        into this dictmerger spilled any."""
        consumed, st.consumed = st.consumed, False    # result() may be finishing it: replay is internal
        try:
            while getattr(st, "spill_pending", False):
                st.spill_pending = False
                _, spilled = st.read_counters()
                if spilled:
                    self._dict_regrow(st, spilled)
        finally:
            st.consumed = consumed

    def _dict_aggregate(self, st, b):
        from .codegen import dict_agg_source
        src, smem = dict_agg_source(st.kind, st.slot_words, b.extra["agg_S"], b.extra["pbits"])
        kern = rt.get_kernel(src, "wg_dagg")
        P = 1 << b.extra["pbits"]
        grid = rt.sm_count() * kern.blocks_per_sm(256, smem)
        words = [st.pk.ptr] + [v.ptr for v in st.pv] + [st.pcount.ptr, st.pcap, P, st.table.ptr, st.cap - 1,
                                                           st.count.ptr, st.ocount.ptr, st.ocap, st.over[0][0].ptr]
        words += [o.ptr for o in st.over[1]] + [rt.error_ptr()]
        blob = b"".join(_pack("u64", w) for w in words)
        kern.launch(grid, 256, blob, smem)
        self.launches += 1
        self.dirty = True

    def _dict_dev(self, v, ty, path):
        """A dictionary captured by a loop body, as device columns sorted by
        order_key (DDict / DGroups; a host dict payload is uploaded once)."""
        if isinstance(v, (DDict, DGroups)):
            return v
        if isinstance(v, dict):
            t = ty
            for q in path:
                t = t.fields[q]
            cached = self._host_dicts.get(id(v))
            if cached is not None and cached[0] is v:
                return cached[1]
            d = _host_dict_to_device(v, t)
            self._host_dicts[id(v)] = (v, d)
            return d
        raise EvalError(f"captured value {type(v).__name__} is not a dictionary")

    def _acct_append(self, st, rows):
        if getattr(st, "hint", None) is None:
            nbytes = rows * sum(SIZE[k] for k in st.kinds)
            self.alloc(nbytes)
            st.acct = getattr(st, "acct", 0) + nbytes

    def _dict_regrow(self, st: DictDev, spilled):
        global REGROWS
        REGROWS += 1
        self._dict_regrow_(st, spilled)

    def _dict_regrow_(self, st: DictDev, spilled, want=0):
        """Grow the table 4x (or to hold `want` keys at load 1/2), re-insert
        existing entries and replay the spilled merges (all folds are
        commutative)."""
        kw, vw, n = st.compact()
        old_over, old_cnt = st.over, spilled
        newcap = max(4 * st.cap, 1 << int(max(2 * n, 1) - 1).bit_length())
        if want:
            newcap = max(st.cap, 1 << int(max(2 * max(want, n), 1) - 1).bit_length())
        st._alloc_table(newcap)
        rt.memset(st.ocount.ptr, 0, 8)
        # replay: entries from the old table then the spill list, as a device loop
        kty = st.kind.key
        vty = st.kind.value
        for keys_w, vals_w, m in ((kw, vw, n), (old_over[0], old_over[1], old_cnt)):
            if m == 0:
                continue
            from .builders_dev import _words_to_cols, _value_words_to_cols
            kcols = _words_to_cols(keys_w, st.kks, st.lay, m)
            vcols = _value_words_to_cols(vals_w, st.vks, m)
            elem = Struct((kty, vty))
            dv = DVec(elem, m, (_layout(kty, kcols), _layout(vty, vcols)))
            saved_over = st.over
            st.over, st.ocap = None, 0
            x = Ident("x", ty=elem)
            body = Merge(Ident("b", ty=Builder(st.kind)), x, ty=Builder(st.kind))
            lam = Lambda((XParam("b"), XParam("i"), XParam("x")), body)
            loop = For((XIterSpec(Ident("__rows", ty=Vec(elem))),), Ident("__b", ty=Builder(st.kind)), lam,
                       ty=Builder(st.kind))
            self.run_loop(loop, {"__rows": dv, "__b": st}, count_traversal=False)
            del saved_over

    def _param_value(self, key, count, datas, windows, bmap, res, captures, grid, tilectr):
        k0 = key[0]
        if k0 == "n":
            return count
        if k0 == "idx0":
            return self.idx0
        if k0 == "err":
            return rt.error_ptr()
        if k0 == "ticket":
            return self.ticket()
        if k0 == "maxit":
            return self.cfg.max_iterations
        if k0 == "tilectr":
            return tilectr.ptr
        if k0 == "pipe_stages":
            return 0
        if k0 == "cnt":
            return self._cnt_buf.ptr
        if k0 == "scnt":
            return self._scnt_buf.ptr
        if k0 == "cgrain":
            return self.cfg.grain_size
        if k0 == "cgmask":
            g_ = self.cfg.grain_size
            return g_ - 1 if g_ & (g_ - 1) == 0 else -1
        if k0 == "cbase":
            return self.cbase
        if k0 == "itcol":
            _, k, l = key
            d = datas[k]
            dv = d.dev() if isinstance(d, HostVec) else d
            col = dv.cols[l]
            s, st = windows[k]
            if st == 1:
                return col.ptr + s * SIZE[col.kind]
            return col.ptr
        if k0 == "itstart":
            return windows[key[1]][0]
        if k0 == "itstride":
            return windows[key[1]][1]
        if k0 in ("capdk", "capdv", "capdn", "capdoff"):
            name = key[1]
            v = captures[name][1]
            path = key[2:] if k0 in ("capdn", "capdoff") else key[2:-1]
            for q in path:
                v = v[q]
            d = self._dict_dev(v, captures[name][0], path)
            if k0 == "capdn":
                return d.n
            if k0 == "capdoff":
                return d.offsets.ptr
            if k0 == "capdk":
                return d.keys.cols[key[-1]].ptr
            return d.vals.cols[key[-1]].ptr
        if k0 in ("cap", "capcol", "caplen"):
            name = key[1]
            v = captures[name][1]
            path = key[2:]
            if k0 == "capcol":
                path, leaf = path[:-1], path[-1]
            for q in path:
                v = v[q]
            if k0 == "cap":
                return v
            dv = v.dev() if isinstance(v, HostVec) else v
            if k0 == "caplen":
                return dv.n
            return dv.cols[leaf].ptr
        if k0 == "b":
            bid, what = key[1], key[2]
            st = bmap[bid]
            if isinstance(st, MergerDev):
                if what == "part":
                    return st.partials(grid)
                if what == "slot":
                    return st.slot.ptr
                if what == "init":
                    return st.take_init_flag()
                if what == "mirror":
                    return st.mirror_ptr()
            if isinstance(st, (AppenderDev, GroupDev)):
                r = res[bid]
                if what == "ctotal":
                    return r[1]
                if what == "col":
                    seg = r if not isinstance(r, tuple) else r[0]
                    return seg.cols[key[3]].ptr
                if what == "status":
                    return r[1].ptr if r[1] is not None else 0
                if what == "total":
                    return r[0].total_buf.ptr
                if what == "coff":
                    return res[("coff", bid)].ptr
            if isinstance(st, VecMergerDev):
                if what == "len":
                    return st.n
                if what == "col":
                    return st.cols[key[3]].ptr
            if isinstance(st, DictDev):
                if what == "table":
                    return st.table.ptr
                if what == "mask":
                    return st.cap - 1
                if what == "count":
                    return st.count.ptr
                if what == "ocount":
                    return st.ocount.ptr
                if what == "ocap":
                    return st.ocap
                if what == "okey":
                    return st.over[0][key[3]].ptr
                if what == "pcount":
                    return st.pcount.ptr
                if what == "pcap":
                    return st.pcap
                if what == "pshift":
                    return max(0, st.cap.bit_length() - 1 - st.pbits)
                if what == "pk":
                    return st.pk.ptr
                if what == "pv":
                    return st.pv[key[3]].ptr
                if what == "oval":
                    return st.over[1][key[3]].ptr
                if what == "zrow":
                    return st.zrow_cur.ptr
        raise EvalError(f"internal: no value for kernel parameter {key}")


def _host_dict_to_device(v, t):
    """Reference dict payload -> DDict / DGroups with entries in order_key
    order (builders.py:496-507)."""
    from weldmill.engine.builders import order_key
    from .columns import ListLayout, to_device
    items = sorted(v.items(), key=lambda kv: order_key(kv[0]))
    keys = to_device(Vec(t.key), [k for k, _ in items])
    if isinstance(t.value, Vec):
        flat, offs = [], [0]
        for _, vv in items:
            flat.extend(vv)
            offs.append(len(flat))
        vals = to_device(t.value, flat)
        oc = Col.alloc(I64, len(offs))
        arr = np.asarray(offs, dtype=np.int64)
        rt.h2d(oc.ptr, arr.ctypes.data, arr.nbytes)
        return DGroups(Dict(t.key, t.value), keys, oc, vals)
    vals = to_device(Vec(t.value), [x for _, x in items])
    return DDict(Dict(t.key, t.value), keys, vals)


_LOOP_REFS = {}     # id(loop expression) -> weakref: guards the id-keyed hints


def _claim_loop_id(e):
    """Per-loop hints (table sizes) are keyed by
    id(loop).  When a loop expression dies and CPython reuses its id for a
    new one, drop the dead loop's hints before the new loop reads them."""
    lid = id(e)
    r = _LOOP_REFS.get(lid)
    if r is not None and r() is e:
        return
    if r is not None:
        from .builders_dev import _SIZE_HINTS as _SH
        for k in [k for k in _SH if k[0] == lid]:
            del _SH[k]
    try:
        _LOOP_REFS[lid] = weakref.ref(e)
    except TypeError:
        pass


_LEAVES = {}


def _leaves_of(t):
    """Scalar leaves of a flat element type (None if not flat), memoised:
    loop element types repeat across every evaluate of a program."""
    try:
        return _LEAVES[t]
    except KeyError:
        ks = leaves(t) if is_flat(t) else None
        _LEAVES[t] = ks
        return ks
    except TypeError:           # unhashable type object
        return leaves(t) if is_flat(t) else None


def _layout(t, cols):
    from .columns import layout_from_cols
    return layout_from_cols(t, cols)


def _with_func(e, lam):
    from dataclasses import replace
    return replace(e, func=lam)


def _pack(ctype, v):
    if ctype == "double":
        return _struct.pack("<d", float(v))
    if isinstance(v, bool):
        v = int(v)
    if isinstance(v, float):
        raise EvalError(f"internal: float for {ctype} parameter")
    return _struct.pack("<Q", int(v) & 0xFFFFFFFFFFFFFFFF)


def _dvec_item(dv: DVec, idx):
    from .columns import col_to_numpy
    vals = []
    for c in dv.cols:
        arr = np.empty(1, dtype=np.dtype({BOOL: "u1", "i32": "<i4", "i64": "<i8", "f32": "<f4", "f64": "<f8"}[c.kind]))
        rt.d2h(arr.ctypes.data, c.ptr + idx * SIZE[c.kind], SIZE[c.kind])
        x = arr[0].item()
        vals.append(bool(x) if c.kind == BOOL else x)
    from .irtypes import unflatten
    return unflatten(dv.elem, vals)


def _slot_bytes(t):
    from weldmill.engine.builders import _slot_size
    return _slot_size(t)


def payload_bytes_dvec(ty, v):
    """weldmill's payload_bytes (builders.py:59-82) of a device vector:
    16-byte header plus contents, nested vectors counted with their own
    headers and elements."""
    return 16 + _elem_bytes(ty.elem, v.n, v.layout)


def _value_bytes(t, v):
    """payload_bytes of a runtime value that may hold device vectors."""
    if isinstance(v, DVec):
        return payload_bytes_dvec(t, v)
    if isinstance(v, HostVec):
        if isinstance(v.payload, list):
            return payload_bytes(t, v.payload)
        return payload_bytes_dvec(t, v.dev())
    if isinstance(t, Struct):
        return sum(_value_bytes(f, x) for f, x in zip(t.fields, v))
    return payload_bytes(t, v)


def _elem_bytes(t, n, lay):
    if isinstance(t, Scalar):
        return n * SIZE[t.kind]
    if isinstance(t, Struct):
        return sum(_elem_bytes(f, n, l) for f, l in zip(t.fields, lay))
    if isinstance(t, Vec):
        return n * 16 + _elem_bytes(t.elem, lay.total, lay.child)
    raise EvalError(f"no byte accounting for values of type {t}")


def _fixed(t):
    if isinstance(t, Scalar):
        return SIZE[t.kind]
    if isinstance(t, Struct):
        s = 0
        for f in t.fields:
            x = _fixed(f)
            if x is None:
                return None
            s += x
        return s
    return None


def _collect_builders(v, out):
    if isinstance(v, tuple):
        for x in v:
            _collect_builders(x, out)
    elif hasattr(v, "pending"):
        out.append(v)
    else:
        raise EvalError("loop builders must be builders")


LOWCARD_MAX = 4096
import os as _os
STREAMING = _os.environ.get("WELDGPU_STREAM", "1") == "1"
PART_MIN_KEYS = 1 << 20


REGROWS = 0         # dictmerger tables grown after spills (test instrumentation)


SKETCH_ROWS = 1 << 16   # rows of a loop's first run that choose its dictmerger variants


def _builder_order(builders):
    """Builders in _bspecs' id order (depth-first over builder structs)."""
    out = []
    stack = [builders]
    while stack:                 # iterative: a recursive closure would pin the builders until GC
        v = stack.pop()
        if isinstance(v, tuple):
            stack.extend(reversed(v))
        else:
            out.append(v)
    return out


def _bspecs(builders, strategy, count, loop_id=None, assume_lowcard=False, grain=1024):
    bmap = {}
    counter = [0]
    single = not isinstance(builders, tuple)

    def go(v):
        if isinstance(v, tuple):
            return tuple(go(x) for x in v)
        bid = counter[0]
        counter[0] += 1
        bmap[bid] = v
        bs = BSpec(bid=bid, kind=v.kind)
        if isinstance(v.kind, VecMerger):
            F = len(leaves(v.kind.elem))
            nb = v.n
            if strategy != "global" and nb * F * 8 <= 96 * 1024 and nb <= count:
                bs.mode = "smem"
                bs.extra["nbins"] = nb
            else:
                bs.mode = "global"
        if isinstance(v.kind, DictMerger):
            bs.extra["slot_words"] = v.slot_words
            # Cardinality seen the last time this loop ran decides the
            # variant: low -> register cache + shared table, otherwise (or
            # unknown) -> deferred merges with batched HBM probes.
            from .builders_dev import _SIZE_HINTS
            seen = _SIZE_HINTS.get((loop_id, bid))
            if seen is None and assume_lowcard:
                seen = 1
            lowcard = seen is not None and seen <= LOWCARD_MAX
            if (seen is not None and seen > PART_MIN_KEYS and strategy != "global"
                    and v.nw == 1 and DEFER_DICT):
                # cardinality far beyond L2: partitioned two-kernel aggregation
                bs.extra["part"] = True
                bs.extra["agg_S"] = 0
                bs.extra["pbits"] = 8
            if strategy != "global" and v.nw == 1 and (lowcard or not DEFER_DICT):
                ns = 512
                if ns * v.slot_words * 8 <= 64 * 1024:
                    bs.mode = "smem"
                    bs.extra["smem_slots"] = ns
                    bs.extra["pattern"] = v.pattern()
                    bs.extra["lowcard"] = lowcard
                else:
                    bs.mode = "global"
            else:
                bs.mode = "global"
        if isinstance(v, AppenderDev) and isinstance(v.kind, VecBuilder) and getattr(v, "segk", None) is not None:
            # unhinted vecbuilder: scan-mode kernels record where each
            # grain-wide chunk's appends start (reallocation accounting);
            # "fine" when a thread's items can hold more than one chunk start
            bs.extra["segstats"] = "fine" if grain < 32 else True
        if isinstance(v, (AppenderDev,)) and v.kinds is None:
            raise DeviceUnsupported(f"vecbuilder[{v.kind.elem}] (nested element types) on the device")
        return bs

    try:
        return go(builders), bmap
    finally:
        del go  # the recursive closure would otherwise pin every builder (and its HBM) until GC


def _bsig(bs):
    if isinstance(bs, tuple):
        return tuple(_bsig(x) for x in bs)
    return (bs.mode, bs.extra.get("nbins"), bs.extra.get("smem_slots"), bs.extra.get("lowcard"),
            bs.extra.get("part"), bs.extra.get("pbits"), bs.extra.get("segstats"))


def _type_of(v, lam, name):
    """IR type of a captured runtime value, recovered from the lambda body."""
    from weldmill.expr import walk
    for node in walk(lam.body):
        if isinstance(node, Ident) and node.name == name and node.ty is not None:
            return node.ty
    raise EvalError(f"cannot type captured name {name!r}")


# ---------------------------------------------------------------------------
# result conversion


def to_host_payload(v, ty):
    if isinstance(ty, Scalar):
        return v
    if isinstance(ty, Struct):
        return tuple(to_host_payload(x, t) for x, t in zip(v, ty.fields))
    if isinstance(ty, Vec):
        if isinstance(v, HostVec):
            p = v.payload
            if isinstance(p, list):
                return p
            v = v.dev()
        return to_payload(v)
    if isinstance(ty, Dict):
        return dict_payload(v)
    if isinstance(ty, Simd):
        return tuple(v)
    if isinstance(ty, Builder):
        return v
    raise DeviceUnsupported(f"cannot return a value of type {ty}")


def _numpy_tree(v, ty):
    from .columns import to_numpy, to_numpy_nested
    if isinstance(v, tuple) and isinstance(ty, Struct):
        return tuple(_numpy_tree(x, t) for x, t in zip(v, ty.fields))
    if isinstance(v, HostVec):
        v = v.dev()
    if isinstance(v, DVec) and is_flat(v.elem):
        return to_numpy(v)
    if isinstance(v, DVec):
        return to_numpy_nested(v)     # nested vectors: Ragged (offsets + values)
    return to_host_payload(v, ty)


def _collect_ids(v, acc):
    if isinstance(v, tuple):
        for x in v:
            _collect_ids(x, acc)
    elif isinstance(v, (DVec, DDict, DGroups, HostVec, np.ndarray)):
        acc.add(id(v))


# One evaluation at a time per process: the device runtime's current
# stream, error word and allocator epoch are process-wide, so concurrent
# evaluate() calls (allowed by the reference's contract) are serialised
# here rather than interleaved on the device.
_EVAL_LOCK = threading.RLock()


def evaluate(e, env=None, config=None, externs=None, *, result="python", idx0=0, _ctx_out=None):
    """Run a type-checked core expression on the GPU.  Returns (Value, EvalStats).

    Same contract as weldmill.engine.evaluate (run.py:1008-1074).  Extra
    keyword ``result``: "python" (the reference's payload: lists, tuples,
    dicts), "device" (DVec / DDict handles left in HBM) or "numpy".
    Thread-safe: concurrent calls run one after another.
    """
    with _EVAL_LOCK:
        return _evaluate(e, env, config, externs, result=result, idx0=idx0, _ctx_out=_ctx_out)


def _evaluate(e, env=None, config=None, externs=None, *, result="python", idx0=0, _ctx_out=None):
    cfg = config or EngineConfig()
    if cfg.threads < 1:
        raise EvalError("threads must be at least 1")
    if cfg.strategy not in STRATEGIES:
        raise EvalError(f"unknown merge strategy {cfg.strategy!r}")
    if cfg.grain_size < 1:
        raise EvalError("grain_size must be at least 1")
    if e.ty is None:
        raise EvalError("expression must be type-checked before evaluation")
    rkey = None
    if (REPLAY and not cfg.count_evals and env and result in ("python", "device") and _ctx_out is None and idx0 == 0
            and ((type(e) is Result and type(e.builder) is For)
                 or (type(e) is ToVec and type(e.mapping) is Result and type(e.mapping.builder) is For))):
        rkey = _replay_key(e, env, externs, result)
        if rkey is not None:
            hit = _REPLAYS.get(rkey)
            if hit is not None and hit.valid(e, env, cfg, externs):
                out = hit.run(e)
                if out is not None:
                    return out
                _REPLAYS.d.pop(rkey, None)       # the replayed dictionary outgrew its recorded finish
    note_evaluation()
    ctx = Ctx(cfg, externs, idx0=idx0)
    if _ctx_out is not None:
        _ctx_out.append(ctx)
    if ctx.counting:
        ctx.count_program(e)
    frame = {}
    for name, v in (env or {}).items():
        payload = v.data if isinstance(v, Value) else v
        ty = v.ty if isinstance(v, Value) else None
        if isinstance(payload, DVec):
            frame[name] = payload
        elif ty is not None and isinstance(ty, Vec):
            frame[name] = HostVec(ty, payload)
        elif isinstance(payload, (list, np.ndarray)) and ty is None:
            t = _infer_free_type(e, name)
            frame[name] = HostVec(t, payload) if isinstance(t, Vec) else payload
        else:
            frame[name] = payload
    cand = None
    if result == "numpy" and STREAMING and not ctx.counting:
        cand = _stream_candidate(e, frame)
    if cand is not None:
        val = payload = _stream_evaluate(ctx, e, frame, cand)
    else:
        try:
            val = ctx.ev(e, frame)
        except _DU as exc:
            if isinstance(exc, EvalError):
                raise
            raise DeviceUnsupported(str(exc)) from None
        ctx.check_device()
        if result == "device":
            payload = val
        elif result == "numpy":
            payload = _numpy_tree(val, e.ty)
        else:
            payload = to_host_payload(val, e.ty)

    ctx.settle_segs()
    stats = EvalStats()
    stats.vector_traversals = ctx.traversals
    stats.vector_allocations = ctx.allocs
    stats.vecbuilder_reallocations = ctx.reallocs
    stats.tasks_created = ctx.tasks
    if ctx.counting:
        stats.node_evals = ctx.node_evals()
    reachable = set()
    _collect_ids(val, reachable)
    kept = 0
    for obj, nbytes, cnt in ctx.registry:
        if obj is not None and id(obj) in reachable:
            kept += cnt
        else:
            ctx.free(nbytes)
    stats.peak_bytes = ctx.peak
    stats.live_bytes = ctx.live
    stats.intermediate_allocations = stats.vector_allocations - kept
    if rkey is not None and ctx.rec and len(ctx.rec) == 1 and ctx.launches == 1 and cand is None:
        bl = []
        lb = getattr(ctx, "_last_builders", None)
        if lb is not None:
            _collect_builders(lb, bl)
        outs = ctx.rec[0][5]
        dicts = [b for b in bl if isinstance(b, DictDev)]
        if dicts and not (len(bl) == 1 and type(e) is ToVec and getattr(dicts[0], "small", False)):
            bl = []            # dictionaries replay as the one builder of a tovec(result(...)) with a small result
        if bl and all(isinstance(b, MergerDev) or id(b) in outs for b in bl):
            _REPLAYS.put(rkey, _Replay(e, env, cfg, externs, ctx, bl, stats, result))
            if any(isinstance(b, MergerDev) and not b.mirrored for b in bl):
                _REPLAYS.d.pop(rkey, None)
    return Value(e.ty, payload), stats


# ---------------------------------------------------------------------------
# Launch replay for repeated evaluations of one merger loop over the same
# device-resident inputs (C1 at its 1M-row config size is launch-bound: the
# host control plane -- tree walk, plan lookup, parameter packing -- costs
# more than the kernel).  The first evaluation records its single launch;
# later calls with the same program object, the same input objects, config
# and externs re-issue it and read the merger slots with the error word in
# one synchronisation.  The kernel writes the slots from scratch (init flag),
# resets its last-CTA ticket and reuses its per-CTA partials buffer.

REPLAY = _os.environ.get("WELDGPU_REPLAY", "1") == "1"


class _ReplayCache:
    def __init__(self, cap=32):
        self.d = {}
        self.cap = cap
        self.lock = threading.Lock()

    def get(self, k):
        return self.d.get(k)

    def put(self, k, v):
        with self.lock:
            if len(self.d) >= self.cap:
                self.d.clear()
            self.d[k] = v


_REPLAYS = _ReplayCache()


def _replay_key(e, env, externs, result):
    ids = []
    for name, v in env.items():
        p = v.data if type(v) is Value else v
        if type(p) is not DVec:
            return None           # host inputs are uploaded per call
        ids.append(name)
        ids.append(id(p))
    return (id(e), tuple(ids), tuple(map(id, externs.values())) if externs else (), result)


class _Replay:
    """One recorded single-launch evaluation: merger slots are re-read from
    their pinned mirrors; DIRECT vecbuilder outputs get fresh columns patched
    into the parameter blob (the recorded run's outputs belong to its caller
    and are not kept)."""
    __slots__ = ("e", "inputs", "cfg", "externs", "launch", "builders", "stats", "keep", "lock", "shape", "result",
                 "mergers")

    def __init__(self, e, env, cfg, externs, ctx, builders, stats, result="python"):
        from dataclasses import replace
        self.e = e
        self.inputs = {k: (v.data if isinstance(v, Value) else v) for k, v in env.items()}
        self.cfg = replace(cfg)
        self.externs = dict(externs or {})
        kern, grid, nthr, blob, smem, outs = ctx.rec[0]
        self.launch = (kern, grid, nthr, blob, smem)
        # per builder, in result order: the merger, or (elem type, leaf kinds,
        # rows, blob word index of each leaf column)
        self.builders = [b if isinstance(b, (MergerDev, DictDev)) else
                         (b.kind.elem, list(b.kinds), outs[id(b)][1], outs[id(b)][0]) for b in builders]
        self.mergers = [b for b in builders if isinstance(b, MergerDev)]
        self.stats = stats
        res = ctx._keep[1] if ctx._keep else None
        keep_res = {k: v for k, v in res.items() if not isinstance(v, Segment)} if isinstance(res, dict) else None
        self.keep = (ctx._ticket, ctx._keep[0] if ctx._keep else None, keep_res)
        self.lock = threading.Lock()
        self.shape = ctx._last_builders
        self.result = result

    def valid(self, e, env, cfg, externs):
        if e is not self.e or cfg != self.cfg or len(env) != len(self.inputs):
            return False
        for k, v in env.items():
            p = v.data if isinstance(v, Value) else v
            if self.inputs.get(k) is not p:
                return False
        ext = externs or {}
        return len(ext) == len(self.externs) and all(self.externs.get(k) is f for k, f in ext.items())

    def run(self, e):
        if isinstance(self.builders[0], DictDev):
            return self._run_dict(e)
        note_evaluation()
        kern, grid, block, blob, smem = self.launch
        vals = []
        with self.lock:
            if len(self.mergers) < len(self.builders):
                blob = bytearray(blob)
                for b in self.builders:
                    if isinstance(b, MergerDev):
                        continue
                    elem, kinds, rows, idx = b
                    cols = [Col.alloc(k, rows) for k in kinds]
                    for i, c in zip(idx, cols):
                        _struct.pack_into("<Q", blob, 8 * i, c.ptr)
                    vals.append(dvec_from_cols(elem, rows, cols))
                blob = bytes(blob)
            kern.launch(grid, block, blob, smem)
            if self.mergers:
                mv = []
                for q, b in enumerate(self.mergers):
                    if q == 0:
                        err = []
                        mv.append(b.read(err))
                        code, info = err[0]
                        if code:
                            raise device_error(code, info)
                    else:
                        mv.append(b.read())
            else:
                code, info = rt.read_error()
                if code:
                    raise device_error(code, info)
        mi, ai = iter(mv if self.mergers else ()), iter(vals)
        leaf = lambda b: next(mi) if isinstance(b, MergerDev) else next(ai)
        order = iter(self.builders)
        if len(self.builders) == 1 and not isinstance(self.shape, tuple):
            payload = leaf(self.builders[0])
        else:
            payload = _shape_like(self.shape, lambda: leaf(next(order)))
        if self.result == "python":
            payload = to_host_payload(payload, e.ty)
        st = EvalStats.__new__(EvalStats)
        st.__dict__.update(self.stats.__dict__)
        st.node_evals = {}
        return Value(e.ty, payload), st


def _replay_run_dict(self, e):
    """tovec(result(for(..., dictmerger, ...))) with a small result: the
    table and counters the recorded blob points at are re-initialised, the
    loop kernel relaunched, and the one-launch finish writes fresh result
    columns.  None when the result no longer fits the small finish (the
    caller then evaluates normally)."""
    b = self.builders[0]
    kern, grid, block, blob, smem = self.launch
    kind = b.kind
    with self.lock:
        note_evaluation()
        pat = (ctypes.c_uint64 * b.slot_words)(*b.pattern())
        rt.call("wg_table_init", b.table.ptr, b.cap + 1, b.slot_words, pat)
        rt.memset(b.counters.ptr, 0, 16)
        kern.launch(grid, block, blob, smem)
        d = _finish_small(b, Dict(kind.key, kind.value))
        code, info = getattr(b, "sync_err", (0, 0))
        b.sync_err = (0, 0)
        if code:
            raise device_error(code, info)
        if d is None:
            return None
    out = tovec(d, e.ty.elem)
    payload = out if self.result == "device" else to_host_payload(out, e.ty)
    st = EvalStats.__new__(EvalStats)
    st.__dict__.update(self.stats.__dict__)
    st.node_evals = {}
    return Value(e.ty, payload), st


_Replay._run_dict = _replay_run_dict


def _first_zero_sign(b, d):
    """A one-float-field dictmerger keeps the first-inserted key object of
    the equal pair -0.0 / 0.0 (builders.py:346-351, Python dict semantics):
    the earliest launch that merged a zero key decides, by its first row."""
    for zb in getattr(b, "zrows", ()):
        w = np.zeros(2, dtype=np.uint64)
        rt.d2h(w.ctypes.data, zb.ptr, 16)
        pos, neg = int(w[0]), int(w[1])
        if pos == neg:           # no zero key in this launch
            continue
        if neg < pos and d.n:
            rt.call("wg_neg_zero", d.keys.cols[0].ptr, d.n, SIZE[b.kks[0]])
        return


def _seg_dbl(k):
    """Capacity doublings of a segment holding k appends (16, 32, 64, ...)."""
    return 0 if k <= 16 else (k - 1).bit_length() - 4


def _seg_cap(k):
    return 0 if k <= 0 else 16 << _seg_dbl(k)


def _compiled_nodes(root):
    """Every node weldmill's _compile wraps with a counter (run.py:544-880):
    all nodes except lambda literals in function position (a loop's body,
    iterate's update, sort's key), whose bodies are compiled directly."""
    out = []
    stack = [root]

    def fn_pos(f):
        stack.append(f.body if isinstance(f, Lambda) else f)

    while stack:
        e = stack.pop()
        out.append(e)
        if isinstance(e, For):
            for it in e.iters:
                stack.extend(x for x in (it.data, it.start, it.end, it.stride) if x is not None)
            stack.append(e.builders)
            fn_pos(e.func)
        elif isinstance(e, Iterate):
            stack.append(e.init)
            fn_pos(e.update)
        elif isinstance(e, Sort):
            stack.append(e.vec)
            fn_pos(e.key)
        elif isinstance(e, Let):
            stack.extend((e.value, e.body))
        elif isinstance(e, Lambda):
            stack.append(e.body)
        elif isinstance(e, Apply):
            stack.append(e.func)
            stack.extend(e.args)
        elif isinstance(e, BinaryOp):
            stack.extend((e.lhs, e.rhs))
        elif isinstance(e, UnaryOp):
            stack.append(e.operand)
        elif isinstance(e, (If, BitSelect)):
            stack.extend((e.cond, e.on_true, e.on_false))
        elif isinstance(e, Lookup):
            stack.extend((e.coll, e.index))
        elif isinstance(e, FieldAccess):
            stack.append(e.base)
        elif isinstance(e, Len):
            stack.append(e.coll)
        elif isinstance(e, ToVec):
            stack.append(e.mapping)
        elif isinstance(e, (MakeStruct, MakeVector)):
            stack.extend(e.items)
        elif isinstance(e, NewBuilder):
            if e.arg is not None:
                stack.append(e.arg)
        elif isinstance(e, Merge):
            stack.extend((e.builder, e.value))
        elif isinstance(e, Result):
            stack.append(e.builder)
        elif isinstance(e, (Broadcast, CastScalar)):
            stack.append(e.value)
        elif isinstance(e, ExternCall):
            stack.extend(e.args)
    return out


def _infer_free_type(e, name):
    from weldmill.expr import walk
    for node in walk(e):
        if isinstance(node, Ident) and node.name == name and node.ty is not None:
            return node.ty
    return None


def _run_partial_loop(loop, env, config, externs, idx0, rank):
    """Run one ``for`` loop over this rank's row shard; return (ctx, builders)
    with the builders NOT finalised.  Vecmerger bins on ranks > 0 start from
    the fold identity so ``init`` is counted once (rank 0 folds it)."""
    from dataclasses import replace
    from .irtypes import internal_identity as _iid
    cfg = config or EngineConfig(memory_limit=1 << 46)
    ctx = Ctx(cfg, externs, idx0=idx0)
    frame = {}
    for name, v in (env or {}).items():
        payload = v.data if isinstance(v, Value) else v
        ty = v.ty if isinstance(v, Value) else None
        frame[name] = payload if isinstance(payload, DVec) or not isinstance(ty, Vec) else HostVec(ty, payload)
    bval = ctx.ev(loop.builders, frame)
    blist = []
    _collect_builders(bval, blist)
    for b in blist:
        if isinstance(b, VecMergerDev) and rank > 0:
            for c, k in zip(b.cols, b.ks):
                ident = _iid(b.kind.op, k)
                if b.n and to_bits(k, ident) == 0:
                    rt.memset(c.ptr, 0, b.n * SIZE[k])
                elif b.n:
                    arr = np.full(b.n, ident, dtype=NPTYPE[k])
                    rt.h2d(c.ptr, arr.ctypes.data, arr.nbytes)
    frame["__wg_b"] = bval
    hit = _PARTIAL_LOOPS.get(id(loop))
    if hit is None or hit[0] is not loop:
        # one rewritten loop per program, so plans and dictmerger hints are reused across calls
        hit = _PARTIAL_LOOPS[id(loop)] = (loop, replace(loop, builders=Ident("__wg_b", ty=loop.builders.ty)))
    ctx.run_loop(hit[1], frame)
    ctx.check_device()
    for b in blist:
        b.consume()
    return ctx, blist


_PARTIAL_LOOPS = {}


def evaluate_partials_device(loop, env, config=None, externs=None, idx0=0, rank=0):
    """Per-builder partial states of one loop over this rank's row shard,
    left in HBM for the device combine (distributed.evaluate_sharded):

      merger     {"slot": F+1 words (values, merged flag)}
      appender   {"cols": leaf Cols, "n"}
      vecmerger  {"cols": bin Cols, "n"}
      dict       {"keys", "vals": typed leaf Cols of the compacted table, "n"}
      group      {"keys", "vals": leaf Cols of the row log (input order), "n"}
    """
    from .builders_dev import _value_words_to_cols, _words_to_cols
    ctx, blist = _run_partial_loop(loop, env, config, externs, idx0, rank)
    out = []
    for b in blist:
        kind = b.kind
        if isinstance(kind, Merger):
            F = len(b.ks)
            if not b.launched:         # no rows on this rank: merged flag 0
                rt.memset(b.slot.ptr, 0, 8 * (F + 1))
                b.mirrored = False
            out.append({"kind": "merger", "op": kind.op, "kinds": b.ks, "slot": b.slot, "b": b})
        elif isinstance(kind, VecBuilder):
            if b.segments:
                cols, n = b.concat()
            else:
                cols, n = [Col.alloc(k, 0) for k in b.kinds], 0
            out.append({"kind": "appender", "kinds": b.kinds, "cols": cols, "n": n, "b": b})
        elif isinstance(kind, VecMerger):
            out.append({"kind": "vecmerger", "op": kind.op, "kinds": b.ks, "cols": b.cols, "n": b.n, "b": b})
        elif isinstance(kind, DictMerger):
            if b.table is None:
                b.ensure(1)
            kw, vw, n = b.compact()
            out.append({"kind": "dict", "op": kind.op, "kks": b.kks, "vks": b.vks, "type": kind,
                        "keys": _words_to_cols(kw, b.kks, b.lay, n), "vals": _value_words_to_cols(vw, b.vks, n),
                        "n": n})
        elif isinstance(kind, GroupBuilder):
            if b.segments:
                cols, n = b.concat()
            else:
                cols, n = [Col.alloc(k, 0) for k in b.kinds], 0
            nk = len(b.kks)
            out.append({"kind": "group", "kks": b.kks, "vks": b.vks, "type": kind, "keys": cols[:nk],
                        "vals": cols[nk:], "n": n})
    return out, ctx


# ---------------------------------------------------------------------------
# Streaming path for host-resident inputs: copy/compute overlap.

STREAM_MIN_ROWS = 1 << 22
STREAM_CHUNK_ROWS = int(_os.environ.get("WELDGPU_STREAM_CHUNK", str(1 << 23)))


def _stream_candidate(e, frame):
    """Host numpy inputs feeding one `result(for(...))` whose builders are
    vecbuilders / mergers: returns (loop, iter HostVecs, builder kinds) or None."""
    from weldmill.expr import walk
    if not isinstance(e, Result) or not isinstance(e.builder, For):
        return None
    loop = e.builder
    if not isinstance(loop.func, Lambda):
        return None
    tail = None
    inner = loop.builders
    if (len(loop.iters) == 1 and isinstance(inner, For) and isinstance(inner.func, Lambda)
            and len(inner.iters) == 1 and inner.iters[0].simd and inner.iters[0].start is None
            and isinstance(inner.iters[0].data, Ident) and isinstance(loop.iters[0].data, Ident)
            and inner.iters[0].data.name == loop.iters[0].data.name
            and loop.iters[0].start is not None and not loop.iters[0].simd):
        # the vectorize pass's shape: simd main loop feeding a scalar tail
        # loop over the last len(v) % 4 rows -- stream the simd loop, then
        # run the tail on the device
        tail, loop = loop, inner
    hvs = []
    for it in loop.iters:
        if (it.simd and tail is None) or it.start is not None or not isinstance(it.data, Ident):
            return None
        hv = frame.get(it.data.name)
        if not isinstance(hv, HostVec) or hv._dev is not None:
            return None
        p = hv.payload
        arrs = list(p) if isinstance(p, tuple) else [p]
        if not all(isinstance(a, np.ndarray) and a.ndim == 1 and a.flags.c_contiguous and not a.dtype.names
                   for a in arrs):
            return None
        hvs.append(hv)
    n = len(hvs[0])
    if n < STREAM_MIN_ROWS or any(len(h) != n for h in hvs):
        return None

    def ok_builders(x):
        if isinstance(x, MakeStruct):
            return all(ok_builders(i) for i in x.items)
        return isinstance(x, NewBuilder) and isinstance(x.kind, (VecBuilder, Merger)) and (
            not isinstance(x.kind, VecBuilder) or is_flat(x.kind.elem))

    if not ok_builders(loop.builders):
        return None
    # loop-invariant captures must be scalars (vectors would be re-uploaded per chunk)
    names = free_variables(loop.func) - {p.name for p in loop.func.params}
    if tail is not None:
        names |= free_variables(tail.func) - {p.name for p in tail.func.params}
    for nm in names:
        v = frame.get(nm)
        if isinstance(v, (HostVec, DVec)) or hasattr(v, "pending"):
            return None
    return loop, hvs, tail


def _stream_evaluate(ctx, e, frame, cand):
    """Chunked, double-buffered execution: the next chunk's columns copy in on
    stream 1 while the current chunk computes on stream 0 and the previous
    chunk's appends copy out on stream 2 (straight into pinned numpy
    results).  The loop index stays global (idx0 = chunk start)."""
    from dataclasses import replace
    from .columns import Col, dvec_from_cols, pinned_empty
    loop, hvs, tail = cand
    simd = tail is not None
    n_all = len(hvs[0])
    n = n_all - n_all % 4 if simd else n_all       # rows the streamed loop covers
    C = min(STREAM_CHUNK_ROWS, n)
    if simd:
        C -= C % 4
    nch = (n + C - 1) // C
    leaves_np = []
    for hv in hvs:
        p = hv.payload
        leaves_np.append(list(p) if isinstance(p, tuple) else [p])
    kinds = [leaves(hv.ty.elem) for hv in hvs]
    sets = [[[Col.alloc(k, C) for k in ks] for ks in kinds] for _ in range(2)]
    bval = ctx.ev(loop.builders, frame)
    blist = []
    _collect_builders(bval, blist)
    loop2 = _STREAM_LOOPS.get(id(loop))
    if loop2 is None or loop2[0] is not loop:
        loop2 = (loop, replace(loop, builders=Ident("__wg_sb", ty=loop.builders.ty)))
        _STREAM_LOOPS[id(loop)] = loop2
    loop2 = loop2[1]
    outs = {}
    scan_q, scan_off = [], {}
    ev_in = [rt.Event() for _ in range(nch)]
    ev_k = [rt.Event() for _ in range(nch)]
    try:
        for c in range(nch):
            lo = c * C
            m = min(C, n - lo)
            b = c % 2
            # copy in (stream 1), after the kernel that last read this buffer set
            rt.stream_select(1)
            if c >= 2:
                rt.stream_wait(ev_k[c - 2])
            for k, arrs in enumerate(leaves_np):
                for l, a in enumerate(arrs):
                    col = sets[b][k][l]
                    rt.h2d(col.ptr, a.ctypes.data + lo * a.itemsize, m * a.itemsize)
            ev_in[c].record()
            # compute (stream 0)
            rt.stream_select(0)
            rt.stream_wait(ev_in[c])
            f2 = dict(frame)
            for it, hv, cols, ks in zip(loop.iters, hvs, sets[b], kinds):
                f2[it.data.name] = dvec_from_cols(hv.ty.elem, m, [Col(cc.ptr, kk, cc.owner) for cc, kk in zip(cols, ks)])
            f2["__wg_sb"] = bval
            ctx.idx0 = lo // 4 if simd else lo
            ctx.run_loop(loop2, f2, part=(ctx.idx0, n // 4 if simd else n, c == 0, c == nch - 1))
            ev_k[c].record()
            # copy out (stream 2): this chunk's appended rows
            rt.stream_select(2)
            rt.stream_wait(ev_k[c])
            for st in blist:
                if isinstance(st, AppenderDev) and st.segments:
                    seg = st.segments[-1]
                    if seg.n is None:
                        # order-preserving (scan) appends: the count is on the
                        # device; copy out one chunk later, when it is known
                        scan_q.append((c, st, seg, m))
                        continue
                    if id(st) not in outs:
                        outs[id(st)] = [pinned_empty(n_all * (seg.n // m if m else 1), _NPK[k]) for k in st.kinds]
                    per = seg.n // m if m else 1
                    for arr, col in zip(outs[id(st)], seg.cols):
                        rt.d2h_async(arr.ctypes.data + lo * per * arr.itemsize, col.ptr, seg.n * arr.itemsize)
            # the previous chunk's scan appends: waiting for its kernel costs
            # nothing (the next input copy reuses its buffers and waits too)
            _drain_scan(scan_q, outs, scan_off, n_all, before=c)
        rt.stream_select(2)
        _drain_scan(scan_q, outs, scan_off, n_all, before=nch)
    finally:
        rt.stream_select(0)
        ctx.idx0 = 0
    rt.sync_all()
    if simd and n_all > n:
        _stream_tail(ctx, tail, frame, hvs, kinds, leaves_np, n, n_all, bval, blist, outs, scan_off)
    ctx.dirty = True
    ctx.check_device()

    def build(x, st_iter):
        st = next(st_iter)
        st.consume()
        if isinstance(st, MergerDev):
            return st.read()
        # the reference's VecBuilderState.result: release the segments, then
        # account the materialised vector (builders.py:274-283)
        ctx.settle_segs()
        ctx.free(st.acct)
        if outs.get(id(st)) is not None and all(s.n is not None for s in st.segments):
            o = outs[id(st)]
            if id(st) in scan_off:
                o = [a[:scan_off[id(st)]] for a in o]
            r = o[0] if isinstance(st.kind.elem, Scalar) else tuple(o)
            nr = len(o[0])
        else:
            cols, tot = st.concat() if st.segments else ([Col.alloc(k, 0) for k in st.kinds], 0)
            from .columns import to_numpy
            r = to_numpy(dvec_from_cols(st.kind.elem, tot, cols))
            nr = tot
        ctx.materialized(r if not isinstance(r, tuple) else r[0], 16 + nr * st.eb)
        return r

    it_ = iter(blist)
    try:
        return _shape_like(bval, lambda: build(None, it_))
    finally:
        del build   # no closure cycle may keep the pinned results' pool blocks alive


_NPK = {"bool": "u1", "i32": "<i4", "i64": "<i8", "f32": "<f4", "f64": "<f8"}
_TAIL_LOOPS = {}


def _stream_tail(ctx, tail, frame, hvs, kinds, leaves_np, n4, n, bval, blist, outs, offs):
    """The vectorised shape's scalar tail (the last n % 4 rows): upload those
    rows, run the tail loop on the device into the streamed builders, and
    append its rows to the host results."""
    from dataclasses import replace
    from .columns import Col, dvec_from_cols
    t = _TAIL_LOOPS.get(id(tail))
    if t is None or t[0] is not tail:
        t = (tail, replace(tail, builders=Ident("__wg_sb", ty=tail.builders.ty)))
        _TAIL_LOOPS[id(tail)] = t
    f2 = dict(frame)
    f2["__wg_sb"] = bval
    for it, hv, ks, arrs in zip(tail.iters, hvs, kinds, leaves_np):
        cols = []
        for kk, a in zip(ks, arrs):
            buf = Col.alloc(kk, n - n4)
            rt.h2d(buf.ptr, a.ctypes.data + n4 * a.itemsize, (n - n4) * a.itemsize)
            # the tail loop reads only rows [n4, n): a base pointer n4 rows
            # before the uploaded tail makes v's indices line up
            cols.append(Col(buf.ptr - n4 * SIZE[kk], kk, buf))
        f2[it.data.name] = dvec_from_cols(hv.ty.elem, n, cols)
    seen = {id(st): len(st.segments) for st in blist if isinstance(st, AppenderDev)}
    ctx.run_loop(t[1], f2)
    rt.sync()
    for st in blist:
        if not isinstance(st, AppenderDev) or outs.get(id(st)) is None:
            continue
        off = offs.get(id(st), n4 * (len(outs[id(st)][0]) // n if n else 1))
        for seg in st.segments[seen[id(st)]:]:
            cnt = seg.length()
            if off + cnt > len(outs[id(st)][0]):
                outs[id(st)] = None
                break
            for arr, col in zip(outs[id(st)], seg.cols):
                rt.d2h(arr.ctypes.data + off * arr.itemsize, col.ptr, cnt * arr.itemsize)
            off += cnt
        if id(st) in offs and outs.get(id(st)) is not None:
            offs[id(st)] = off


def _drain_scan(q, outs, offs, n, before):
    """Copy out the scan-appender chunks queued before chunk `before`: read
    each chunk's count (stream 2 already waits on that chunk's kernel), then
    queue the copy of exactly that many rows at the running offset."""
    from .columns import pinned_empty
    while q and q[0][0] < before:
        _, st, seg, m = q.pop(0)
        cnt = seg.length()
        if id(st) not in outs:
            per = max(1, -(-seg.cap // m)) if m else 1
            outs[id(st)] = [pinned_empty(n * per, _NPK[k]) for k in st.kinds]
            offs[id(st)] = 0
        if outs[id(st)] is None:
            continue
        off = offs[id(st)]
        if off + cnt > len(outs[id(st)][0]):
            outs[id(st)] = None      # more appends per row than the first chunk had: result() concatenates on device
            continue
        for arr, col in zip(outs[id(st)], seg.cols):
            rt.d2h_async(arr.ctypes.data + off * arr.itemsize, col.ptr, cnt * arr.itemsize)
        offs[id(st)] = off + cnt


def _shape_like(v, leaf):
    if isinstance(v, tuple):
        return tuple(_shape_like(x, leaf) for x in v)
    return leaf()


_STREAM_LOOPS = {}

"""Row-partitioned evaluation across GPUs (one process per GPU).

Each rank evaluates a loop over its contiguous row range of the loop inputs
(rank r holds rows [off_r, off_r + n_r)); the loop index ``i`` stays global
(the kernels add ``idx0 = off_r``).  Each builder's per-rank partial stays in
HBM and is combined ON THE DEVICE, the way the reference folds its chunk
partials at result() (/root/reference/pkg/src/weldmill/engine/builders.py:
314-328 merger, 380-392 dictmerger, 435-450 vecmerger, 478-493 groupbuilder):

  merger       all-gather of each rank's slot (F value words + merged flag,
               8(F+1) bytes), folded in rank order by a device kernel
               (wg_fold_slots): NaN and wrap semantics exact, deterministic
  vecbuilder   ordered gather: the per-rank counts are all-gathered; each
               rank keeps its segment, which is rows [offset, offset + n) of
               the global result (= sequential order, builders.py:274-283)
  vecmerger    reduce-scatter by rank-order fold: bin slice j of every rank
               goes to rank j (all-to-all), is folded in rank order
               (wg_fold_chunks), and the folded slices are all-gathered;
               ranks > 0 start from the fold identity so ``init`` counts once
  dictmerger   range partition of the locally aggregated entries by the
               order key of the first key leaf against splitters sampled on
               every rank (wg_partition: stable), all-to-all of the entries,
               then a device dictmerger over the received entries: rank r
               owns a contiguous key range, so the rank-order concatenation
               of the per-rank sorted results is the reference's sorted
               result
  groupbuilder rows (key, value) partitioned the same way in local input
               order; the receiver runs a device groupbuilder over them in
               source-rank order, so each key's values keep the global input
               order (builders.py:464-476)

Transports (``DeviceComm``): ``NcclComm`` drives NCCL from libweldgpu
(wg_nccl_*) on the executor's stream -- the product path on a multi-GPU box;
``StagedComm`` moves the same device buffers through host memory over
torch.distributed (gloo) -- used to run several ranks on ONE GPU in tests.
The host-side planning (splitters, exchange plans, slices) is plain numpy
and is tested on CPU with gloo (tests/test_distributed.py).
"""
from __future__ import annotations

import ctypes
import struct as _struct

import numpy as np

from . import _ref  # noqa: F401
from .irtypes import BOOL, F32, F64, I32, I64, KIND_CODE, NPTYPE, SIZE, DeviceUnsupported


# ---------------------------------------------------------------------------
# host-side planning (numpy only)


def shard_bounds(n_total, rank, world):
    """Contiguous row range of ``rank`` (the reference's chunk grid, coarsened)."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def okey_np(arr, kind):
    """The order key (builders.py:496-507) of a typed leaf as u64, identical
    to the device's okey_at / k_order_key: signed ints flip the sign bit;
    floats map to the IEEE total order with -0.0 == 0.0 and every NaN last."""
    a = np.ascontiguousarray(arr)
    if kind == BOOL:
        return a.astype(np.uint64)
    if kind in (I32, I64):
        return a.astype(np.int64).view(np.uint64) ^ np.uint64(1 << 63)
    v = a.astype(np.float64)
    nan = np.isnan(v)
    v = np.where(v == 0.0, 0.0, v)
    b = v.view(np.uint64)
    neg = (b >> np.uint64(63)).astype(bool)
    k = np.where(neg, ~b, b | np.uint64(1 << 63))
    k = np.where(k == np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64(0xFFFFFFFFFFFFFFFE), k)
    return np.where(nan, np.uint64(0xFFFFFFFFFFFFFFFF), k).astype(np.uint64)


def sample_positions(n, s=256):
    """Evenly spaced sample positions over n rows (at most s)."""
    if n == 0:
        return np.zeros(0, dtype=np.uint32)
    m = min(n, s)
    return ((np.arange(m, dtype=np.uint64) * np.uint64(n)) // np.uint64(m)).astype(np.uint32)


def choose_splitters(samples, world):
    """world - 1 ascending order-key splitters from every rank's samples:
    destination of a row = number of splitters <= its key."""
    allk = np.sort(np.concatenate([np.asarray(s, dtype=np.uint64) for s in samples])) if samples else \
        np.zeros(0, dtype=np.uint64)
    if world <= 1:
        return np.zeros(0, dtype=np.uint64)
    if allk.size == 0:
        return np.full(world - 1, np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    idx = [(j * allk.size) // world for j in range(1, world)]
    return allk[idx].astype(np.uint64)


def exchange_plan(counts, rank):
    """counts[s][d] = rows rank s sends to rank d.  Returns this rank's
    (send_counts, send_offsets, recv_counts, recv_offsets), offsets in rows;
    received rows are laid out in source-rank order."""
    counts = np.asarray(counts, dtype=np.int64)
    send = counts[rank]
    recv = counts[:, rank]
    soff = np.concatenate([[0], np.cumsum(send)[:-1]]).astype(np.int64)
    roff = np.concatenate([[0], np.cumsum(recv)[:-1]]).astype(np.int64)
    return send, soff, recv, roff


def slice_bounds(n, world):
    return [shard_bounds(n, j, world) for j in range(world)]


# ---------------------------------------------------------------------------
# transports over device buffers


class DeviceComm:
    """Collectives over device columns (pointers from libweldgpu)."""

    rank = 0
    world = 1

    def allgather_host(self, arr: np.ndarray):
        """Small host arrays (counts, samples): every rank's array, rank order."""
        raise NotImplementedError

    def allgather_dev(self, ptr, nbytes):
        """Equal-size device all-gather -> DeviceBuffer of world * nbytes."""
        raise NotImplementedError

    def alltoallv_dev(self, cols, send, soff, recv, roff):
        """cols: [(ptr, esize)].  Rows [soff[d], soff[d] + send[d]) of every
        column go to rank d; returns one DeviceBuffer per column holding the
        received rows in source-rank order."""
        raise NotImplementedError

    def allgatherv_dev(self, ptr, esize, counts):
        """Variable-length all-gather of one column (counts[r] rows from rank r)."""
        raise NotImplementedError

    def barrier(self):
        pass


class SoloComm(DeviceComm):
    def allgather_host(self, arr):
        return [np.asarray(arr)]

    def allgather_dev(self, ptr, nbytes):
        from . import runtime as rt
        out = rt.alloc(max(nbytes, 1))
        if nbytes:
            rt.d2d(out.ptr, ptr, nbytes)
        return out

    def alltoallv_dev(self, cols, send, soff, recv, roff):
        from . import runtime as rt
        outs = []
        for ptr, es in cols:
            b = rt.alloc(max(int(recv[0]) * es, 1))
            if recv[0]:
                rt.d2d(b.ptr, ptr + int(soff[0]) * es, int(recv[0]) * es)
            outs.append(b)
        return outs

    def allgatherv_dev(self, ptr, esize, counts):
        return self.allgather_dev(ptr, int(counts[0]) * esize)


class NcclComm(DeviceComm):
    """NCCL communicator owned by libweldgpu (one per process), bootstrapped
    through an initialised torch.distributed group (any backend)."""

    _inited = False

    def __init__(self, group=None):
        import torch.distributed as dist
        from . import runtime as rt
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if not NcclComm._inited:
            uid = ctypes.create_string_buffer(128)
            if self.rank == 0:
                rt.call("wg_nccl_unique_id", uid, 128)
            obj = [bytes(uid.raw) if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            rt.call("wg_nccl_init", self.rank, self.world, obj[0])
            NcclComm._inited = True

    def allgather_dev(self, ptr, nbytes):
        from . import runtime as rt
        out = rt.alloc(max(nbytes * self.world, 1))
        if nbytes:
            rt.call("wg_nccl_allgather", ptr, out.ptr, nbytes)
        return out

    def allgather_host(self, arr):
        from . import runtime as rt
        arr = np.ascontiguousarray(arr)
        n = np.array([arr.nbytes], dtype=np.int64)
        nb = rt.alloc(8)
        rt.h2d(nb.ptr, n.ctypes.data, 8)
        sizes = np.empty(self.world, dtype=np.int64)
        ab = self.allgather_dev(nb.ptr, 8)
        rt.d2h(sizes.ctypes.data, ab.ptr, 8 * self.world)
        m = int(sizes.max()) if self.world else 0
        if m == 0:
            return [arr[:0] for _ in range(self.world)]
        buf = np.zeros(m, dtype=np.uint8)
        buf[:arr.nbytes] = arr.view(np.uint8).reshape(-1)
        db = rt.alloc(m)
        rt.h2d(db.ptr, buf.ctypes.data, m)
        allb = self.allgather_dev(db.ptr, m)
        host = np.empty(m * self.world, dtype=np.uint8)
        rt.d2h(host.ctypes.data, allb.ptr, host.nbytes)
        return [host[r * m:r * m + int(sizes[r])].view(arr.dtype) for r in range(self.world)]

    def _sendrecv(self, sends, recvs):
        from . import runtime as rt
        ns, nr = len(sends), len(recvs)
        sp = (ctypes.c_uint64 * max(ns, 1))(*[p for p, _, _ in sends])
        sb = (ctypes.c_uint64 * max(ns, 1))(*[b for _, b, _ in sends])
        sq = (ctypes.c_int * max(ns, 1))(*[q for _, _, q in sends])
        rp = (ctypes.c_uint64 * max(nr, 1))(*[p for p, _, _ in recvs])
        rb = (ctypes.c_uint64 * max(nr, 1))(*[b for _, b, _ in recvs])
        rq = (ctypes.c_int * max(nr, 1))(*[q for _, _, q in recvs])
        rt.call("wg_nccl_sendrecv", ns, sp, sb, sq, nr, rp, rb, rq)

    def alltoallv_dev(self, cols, send, soff, recv, roff):
        from . import runtime as rt
        outs, sends, recvs = [], [], []
        total = int(np.sum(recv))
        for ptr, es in cols:
            b = rt.alloc(max(total * es, 1))
            outs.append(b)
            for d in range(self.world):
                sends.append((ptr + int(soff[d]) * es, int(send[d]) * es, d))
                recvs.append((b.ptr + int(roff[d]) * es, int(recv[d]) * es, d))
        self._sendrecv(sends, recvs)
        return outs

    def allgatherv_dev(self, ptr, esize, counts):
        from . import runtime as rt
        counts = [int(c) for c in counts]
        offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
        out = rt.alloc(max(sum(counts) * esize, 1))
        sends = [(ptr, counts[self.rank] * esize, d) for d in range(self.world)]
        recvs = [(out.ptr + int(offs[s]) * esize, counts[s] * esize, s) for s in range(self.world)]
        self._sendrecv(sends, recvs)
        return out


class StagedComm(DeviceComm):
    """The same collectives with device buffers staged through host memory
    over torch.distributed (gloo): runs several ranks on one GPU."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allgather_host(self, arr):
        torch, dist = self.torch, self.dist
        arr = np.ascontiguousarray(arr)
        n = torch.tensor([arr.nbytes], dtype=torch.int64)
        ns = [torch.zeros(1, dtype=torch.int64) for _ in range(self.world)]
        dist.all_gather(ns, n, group=self.group)
        sizes = [int(x.item()) for x in ns]
        m = max(max(sizes), 1)
        buf = torch.zeros(m, dtype=torch.uint8)
        if arr.nbytes:
            buf[:arr.nbytes] = torch.from_numpy(arr.view(np.uint8).reshape(-1).copy())
        outs = [torch.zeros(m, dtype=torch.uint8) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        return [o[:s].numpy().view(arr.dtype) for o, s in zip(outs, sizes)]

    def _d2h(self, ptr, nbytes):
        from . import runtime as rt
        a = np.empty(nbytes, dtype=np.uint8)
        if nbytes:
            rt.d2h(a.ctypes.data, ptr, nbytes)
        return a

    def _h2d(self, a):
        from . import runtime as rt
        b = rt.alloc(max(a.nbytes, 1))
        if a.nbytes:
            rt.h2d(b.ptr, np.ascontiguousarray(a).ctypes.data, a.nbytes)
        return b

    def allgather_dev(self, ptr, nbytes):
        parts = self.allgather_host(self._d2h(ptr, nbytes))
        return self._h2d(np.concatenate(parts))

    def alltoallv_dev(self, cols, send, soff, recv, roff):
        torch, dist = self.torch, self.dist
        outs = []
        for ptr, es in cols:
            ss = [int(send[d]) * es for d in range(self.world)]
            rs = [int(recv[d]) * es for d in range(self.world)]
            host = np.concatenate([self._d2h(ptr + int(soff[d]) * es, ss[d]) for d in range(self.world)])
            out = torch.zeros(sum(rs), dtype=torch.uint8)
            dist.all_to_all_single(out, torch.from_numpy(host), output_split_sizes=rs, input_split_sizes=ss,
                                   group=self.group)
            outs.append(self._h2d(out.numpy()))
        return outs

    def allgatherv_dev(self, ptr, esize, counts):
        parts = self.allgather_host(self._d2h(ptr, int(counts[self.rank]) * esize))
        return self._h2d(np.concatenate(parts))

    def barrier(self):
        self.dist.barrier(group=self.group)


def device_comm(group=None):
    """NCCL when every rank has its own GPU, else host-staged gloo."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return SoloComm()
    if dist.get_backend(group) == "nccl" and torch.cuda.device_count() >= dist.get_world_size(group):
        try:
            return NcclComm(group)
        except Exception as exc:            # e.g. libnccl.so.2 missing: same results, host-staged
            import sys
            print(f"paper_1709_06416_b200: NCCL combine unavailable ({exc}); using the host-staged combine",
                  file=sys.stderr)
            return StagedComm(dist.new_group(backend="gloo"))   # host tensors need a gloo group
    return StagedComm(group)


# ---------------------------------------------------------------------------
# device combine


_COMBINE = {}


def _combine_kernels(op, kinds):
    from . import runtime as rt
    from .codegen import combine_source
    key = (op, tuple(kinds))
    k = _COMBINE.get(key)
    if k is None:
        src = combine_source(op, list(kinds))
        k = _COMBINE[key] = {"slots": rt.get_kernel(src, "wg_fold_slots"),
                             "chunks": [rt.get_kernel(src, f"wg_fold_chunks{f}") for f in range(len(kinds))]}
    return k


def _grid(n):
    from . import runtime as rt
    return max(1, min((n + 255) // 256, rt.sm_count() * 8))


def combine_merger(p, comm: DeviceComm):
    """All-gather of the rank slots + rank-order fold on the device."""
    from . import runtime as rt
    F = len(p["kinds"])
    nbytes = 8 * (F + 1)
    allw = comm.allgather_dev(p["slot"].ptr, nbytes)
    k = _combine_kernels(p["op"], p["kinds"])["slots"]
    k.launch(1, 32, _struct.pack("<QQQ", allw.ptr, comm.world, p["slot"].ptr))
    b = p["b"]
    b.launched = True
    b.mirrored = False          # the combine kernel writes the device slot only
    vals = [None]
    words = b.read_words()
    from .irtypes import from_bits, identity_value
    if not words[F]:
        vals = [identity_value(p["op"], kk) for kk in p["kinds"]]
    else:
        vals = [from_bits(kk, int(w)) for kk, w in zip(p["kinds"], words[:F])]
    return {"kind": "merger", "values": vals, "has": bool(words[F])}


def combine_appender(p, comm: DeviceComm):
    """Ordered gather: this rank's rows are [offset, offset + n) of the result."""
    counts = np.concatenate(comm.allgather_host(np.array([p["n"]], dtype=np.int64)))
    off = int(counts[:comm.rank].sum())
    return {"kind": "appender", "cols": p["cols"], "kinds": p["kinds"], "n": p["n"], "offset": off,
            "total": int(counts.sum())}


def combine_vecmerger(p, comm: DeviceComm):
    """Bin slices all-to-all'ed, folded in rank order, folded slices all-gathered."""
    from . import runtime as rt
    from .columns import Col
    n, G, r = p["n"], comm.world, comm.rank
    bounds = slice_bounds(n, G)
    send = np.array([hi - lo for lo, hi in bounds], dtype=np.int64)
    soff = np.array([lo for lo, _ in bounds], dtype=np.int64)
    Lr = int(send[r])
    recv = np.full(G, Lr, dtype=np.int64)
    roff = np.arange(G, dtype=np.int64) * Lr
    ks = _combine_kernels(p["op"], p["kinds"])["chunks"]
    chunks = comm.alltoallv_dev([(c.ptr, SIZE[k]) for c, k in zip(p["cols"], p["kinds"])], send, soff, recv, roff)
    out = []
    for f, (ch, k) in enumerate(zip(chunks, p["kinds"])):
        mine = rt.alloc(max(Lr * SIZE[k], 1))
        if Lr:
            ks[f].launch(_grid(Lr), 256, _struct.pack("<QQQQ", mine.ptr, ch.ptr, Lr, G))
        full = comm.allgatherv_dev(mine.ptr, SIZE[k], send)
        out.append(Col(full.ptr, k, full))
    return {"kind": "vecmerger", "cols": out, "kinds": p["kinds"], "n": n}


def _partition_exchange(key_cols, key_kinds, other_cols, other_kinds, n, comm: DeviceComm):
    """Range-partition rows by the first key leaf's order key (splitters
    sampled on every rank), exchange them; returns received (key cols, other
    cols, rows) in source-rank order."""
    from . import runtime as rt
    from .columns import Col
    G = comm.world
    k0, kind0 = key_cols[0], key_kinds[0]
    pos = sample_positions(n)
    samp = np.zeros(0, dtype=np.uint64)
    if pos.size:
        pb = rt.alloc(4 * pos.size)
        rt.h2d(pb.ptr, pos.ctypes.data, pos.nbytes)
        sb = rt.alloc(SIZE[kind0] * pos.size)
        rt.call("wg_gather", k0.ptr, pb.ptr, sb.ptr, pos.size, SIZE[kind0])
        host = np.empty(pos.size, dtype=NPTYPE[kind0])
        rt.d2h(host.ctypes.data, sb.ptr, host.nbytes)
        samp = okey_np(host, kind0)
    split = choose_splitters(comm.allgather_host(samp), G)
    cols = list(key_cols) + list(other_cols)
    kinds = list(key_kinds) + list(other_kinds)
    outs = [Col.alloc(k, n) for k in kinds]
    counts = (ctypes.c_uint64 * G)()
    sp = (ctypes.c_uint64 * max(G - 1, 1))(*[int(x) for x in split])
    ci = (ctypes.c_uint64 * len(cols))(*[c.ptr for c in cols])
    co = (ctypes.c_uint64 * len(cols))(*[c.ptr for c in outs])
    wd = (ctypes.c_int * len(cols))(*[SIZE[k] for k in kinds])
    rt.call("wg_partition", k0.ptr, KIND_CODE[kind0], sp, G - 1, len(cols), ci, co, wd, n, counts)
    mine = np.array(list(counts), dtype=np.int64)
    mat = np.stack(comm.allgather_host(mine))
    send, soff, recv, roff = exchange_plan(mat, comm.rank)
    got = comm.alltoallv_dev([(c.ptr, SIZE[k]) for c, k in zip(outs, kinds)], send, soff, recv, roff)
    rcols = [Col(b.ptr, k, b) for b, k in zip(got, kinds)]
    nk = len(key_cols)
    return rcols[:nk], rcols[nk:], int(recv.sum())


_MERGE_PROGRAMS = {}


def _merge_program(kind):
    """A dictmerger / groupbuilder loop over SoA leaf columns c0..c{m-1}
    (keys then values), compiled once per builder type by the reference
    front end."""
    from weldmill.optim import OptLevel, optimize
    from weldmill.parser import parse
    from weldmill.printer import print_type
    from weldmill.sugar import expand
    from weldmill.typecheck import infer
    from weldmill.types import DictMerger as RDict, Scalar as RScalar, Struct as RStruct, Vec as RVec
    key = repr(kind)
    hit = _MERGE_PROGRAMS.get(key)
    if hit is not None:
        return hit
    ctr = [0]

    def expr_of(t):
        if isinstance(t, RStruct):
            return "{" + ", ".join(expr_of(f) for f in t.fields) + "}"
        j = ctr[0]
        ctr[0] += 1
        return f"x.{j}"

    kexpr = expr_of(kind.key)
    vexpr = expr_of(kind.value)
    m = ctr[0]
    leaves_t = []

    def leaf_types(t):
        if isinstance(t, RStruct):
            for f in t.fields:
                leaf_types(f)
        else:
            leaves_t.append(t)

    leaf_types(kind.key)
    leaf_types(kind.value)
    names = [f"c{j}" for j in range(m)]
    if isinstance(kind, RDict):
        bt = f"dictmerger[{print_type(kind.key)}, {print_type(kind.value)}, {kind.op}]"
    else:
        bt = f"groupbuilder[{print_type(kind.key)}, {print_type(kind.value)}]"
    src = f"result(for({{{', '.join(names)}}}, {bt}, (b, i, x) => merge(b, {{{kexpr}, {vexpr}}})))"
    env = {nm: RVec(t) for nm, t in zip(names, leaves_t)}
    tree = optimize(infer(expand(parse(src)), env), OptLevel.none())[0]
    hit = _MERGE_PROGRAMS[key] = (tree, names, [env[nm] for nm in names])
    return hit


def _local_merge(kind, key_cols, val_cols, n):
    """Device dictmerger / groupbuilder over received (key, value) rows."""
    from weldmill.engine import EngineConfig, Value
    from .columns import dvec_from_cols
    from .executor import evaluate as dev_evaluate
    from .irtypes import Scalar
    tree, names, tys = _merge_program(kind)
    env = {}
    for nm, ty, c in zip(names, tys, list(key_cols) + list(val_cols)):
        env[nm] = Value(ty, dvec_from_cols(ty.elem, n, [c]))
    val, _ = dev_evaluate(tree, env, EngineConfig(memory_limit=1 << 46), result="device")
    return val.data


def combine_dict(p, comm: DeviceComm):
    """Locally aggregated entries range-partitioned + exchanged, then merged."""
    if comm.world == 1:
        rk, rv, n = p["keys"], p["vals"], p["n"]
    else:
        rk, rv, n = _partition_exchange(p["keys"], p["kks"], p["vals"], p["vks"], p["n"], comm)
    d = _local_merge(p["type"], rk, rv, n)
    counts = np.concatenate(comm.allgather_host(np.array([d.n], dtype=np.int64)))
    return {"kind": "dict", "value": d, "offset": int(counts[:comm.rank].sum()), "total": int(counts.sum())}


def combine_group(p, comm: DeviceComm):
    """Rows range-partitioned in local input order, exchanged, grouped in
    source-rank (= global input) order."""
    if comm.world == 1:
        rk, rv, n = p["keys"], p["vals"], p["n"]
    else:
        rk, rv, n = _partition_exchange(p["keys"], p["kks"], p["vals"], p["vks"], p["n"], comm)
    g = _local_merge(p["type"], rk, rv, n)
    counts = np.concatenate(comm.allgather_host(np.array([g.n], dtype=np.int64)))
    return {"kind": "group", "value": g, "offset": int(counts[:comm.rank].sum()), "total": int(counts.sum())}


_COMBINERS = {"merger": combine_merger, "appender": combine_appender, "vecmerger": combine_vecmerger,
              "dict": combine_dict, "group": combine_group}


def evaluate_sharded(expr, env, config=None, externs=None, comm: DeviceComm = None, row0=0, n_total=None,
                     result="device"):
    """Evaluate ``result(for(...))`` / ``tovec(result(for(...)))`` over this
    rank's row shard (the loop inputs in ``env`` are the shard; other vectors,
    e.g. a vecmerger ``init``, are replicated) and combine every builder on
    the device.  Returns one entry per builder of the loop:

      {"kind": "merger", "values", "has"}                 same on every rank
      {"kind": "vecmerger", "cols", "n"}                  same on every rank
      {"kind": "appender", "cols", "n", "offset", "total"}   this rank's rows
      {"kind": "dict" | "group", "value", "offset", "total"} this rank's key
          range (DDict / DGroups, sorted; rank-order concatenation = result)

    result="numpy" converts the device columns to numpy (each rank its own
    part)."""
    from weldmill.expr import For, Result, ToVec
    from .executor import evaluate_partials_device
    comm = comm or SoloComm()
    body = expr.mapping if isinstance(expr, ToVec) else expr
    if not isinstance(body, Result) or not isinstance(body.builder, For):
        raise DeviceUnsupported("sharded evaluation needs result(for(...)) or tovec(result(for(...)))")
    parts, _ = evaluate_partials_device(body.builder, env, config, externs, idx0=row0, rank=comm.rank)
    out = [_COMBINERS[p["kind"]](p, comm) for p in parts]
    if result == "numpy":
        out = [to_numpy_part(o) for o in out]
    return out


def to_numpy_part(o):
    """Device columns of a combined builder -> numpy (this rank's part)."""
    from .columns import col_to_numpy
    if o.get("numpy"):
        return o
    o = dict(o, numpy=True)
    if o["kind"] in ("appender", "vecmerger"):
        o["cols"] = [col_to_numpy(c, o["n"]) for c in o["cols"]]
    elif o["kind"] == "dict":
        d = o.pop("value")
        o["keys"] = [col_to_numpy(c, d.n) for c in d.keys.cols]
        o["vals"] = [col_to_numpy(c, d.n) for c in d.vals.cols]
    elif o["kind"] == "group":
        g = o.pop("value")
        o["keys"] = [col_to_numpy(c, g.n) for c in g.keys.cols]
        o["offsets"] = col_to_numpy(g.offsets, g.n + 1)
        o["vals"] = [col_to_numpy(c, g.vals.n) for c in g.vals.cols]
    return o


def gather_numpy(o, comm: DeviceComm):
    """Whole result of a combined builder on every rank (tests / small results):
    rank-order concatenation of the numpy parts."""
    if not o.get("numpy"):
        o = to_numpy_part(o)
    if o["kind"] == "appender":
        return [np.concatenate(comm.allgather_host(c)) for c in o["cols"]]
    if o["kind"] == "vecmerger":
        return o["cols"]
    if o["kind"] == "merger":
        return o["values"]
    if o["kind"] == "dict":
        return ([np.concatenate(comm.allgather_host(c)) for c in o["keys"]],
                [np.concatenate(comm.allgather_host(c)) for c in o["vals"]])
    keys = [np.concatenate(comm.allgather_host(c)) for c in o["keys"]]
    vals = [np.concatenate(comm.allgather_host(c)) for c in o["vals"]]
    offs = comm.allgather_host(o["offsets"])
    base, fixed = 0, []
    for j, a in enumerate(offs):
        fixed.append(a[:-1] + base if j < len(offs) - 1 else a + base)
        base += int(a[-1])
    return keys, np.concatenate(fixed), vals


__all__ = ["DeviceComm", "SoloComm", "NcclComm", "StagedComm", "device_comm", "shard_bounds", "okey_np",
           "sample_positions", "choose_splitters", "exchange_plan", "slice_bounds", "evaluate_sharded",
           "to_numpy_part", "gather_numpy", "combine_merger", "combine_appender", "combine_vecmerger", "combine_dict",
           "combine_group"]

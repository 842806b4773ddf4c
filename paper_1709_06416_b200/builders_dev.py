"""Device-resident builder states and their result() finalisation.

Mirrors the reference's five state classes
(/root/reference/pkg/src/weldmill/engine/builders.py):

  MergerState      :286-328  slot of F value words + merged flag in HBM
  VecBuilderState  :231-283  ordered list of device segments
  DictMergerState  :331-392  open-addressing table + overflow spill list
  VecMergerState   :395-450  device copy of the init vector (bins)
  GroupBuilderState:453-493  ordered {key, value} segments, stable-sorted
                             by key at result()

``order_key`` (builders.py:496-507) is realised by the order-preserving
u64 transform in libweldgpu (k_order_key) plus a stable LSD radix sort, one
pass per key field from the last field to the first.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _ref  # noqa: F401
from weldmill.errors import UseAfterResult

from . import runtime as rt
from .columns import Col, DVec, ListLayout, col_to_numpy, dvec_from_cols
from .irtypes import (BOOL, F32, F64, I32, I64, KIND_CODE, SIZE, DeviceUnsupported, DictMerger, GroupBuilder, Merger,
                      Scalar, Struct, Vec, VecBuilder, VecMerger, from_bits, identity_value, internal_identity,
                      leaves, to_bits, unflatten)
from .codegen import key_layout

ALL_ONES = 0xFFFFFFFFFFFFFFFF


class BuilderBase:
    def __init__(self, kind):
        self.kind = kind
        self.consumed = False
        self.pending = []   # merges issued outside any loop, flushed in order

    def check(self):
        if self.consumed:
            raise UseAfterResult(f"builder {self.kind} already consumed by result")

    def consume(self):
        self.check()
        self.consumed = True


# ---------------------------------------------------------------------------


class _MirrorSlab:
    """Pinned host cells (64 bytes) the merger kernels' last CTA writes its
    slot and the error word into (unified addressing: the host pointer is
    the device pointer).  Reading a merger result is then a stream sync and
    a host load -- no copy-engine round trip (a 16-byte D2H into pageable
    memory costs ~14 us on B200, more than a 1M-row Q6 kernel)."""

    CELL = 64

    def __init__(self, cells=4096):
        import threading
        self.lock = threading.Lock()
        self.base = None
        self.cells = cells
        self.free = []

    def get(self):
        with self.lock:
            if self.base is None:
                self.base = rt.host_alloc(self.CELL * self.cells)
                self.free = list(range(self.cells - 1, -1, -1))
            if not self.free:
                return None
            return self.base + self.CELL * self.free.pop()

    def put(self, addr):
        with self.lock:
            self.free.append((addr - self.base) // self.CELL)


_MIRRORS = _MirrorSlab()


class MergerDev(BuilderBase):
    """Slot = F value words + merged flag.  The first kernel launch into the
    merger writes the slot (no host-side initialisation copy); a merger
    that never ran a loop reads as the reference identity.  Each launch's
    last CTA also copies the slot and the error word to a pinned host cell
    (`mirror`, F + 3 words) that read() uses."""

    def __init__(self, kind: Merger):
        super().__init__(kind)
        self.ks = leaves(kind.elem)
        self.slot = rt.alloc(8 * (len(self.ks) + 1))
        self.launched = False
        self.part = None
        self.part_cap = 0
        self.mirror = _MIRRORS.get() if len(self.ks) + 3 <= _MirrorSlab.CELL // 8 else None
        self.mirrored = False   # the last launch into the slot wrote the mirror

    def __del__(self):
        m = getattr(self, "mirror", None)
        if m:
            try:
                _MIRRORS.put(m)
            except Exception:
                pass

    def mirror_ptr(self):
        self.mirrored = self.mirror is not None
        return self.mirror or 0

    def partials(self, grid):
        F = len(self.ks)
        need = grid * (F + 1)
        if need > self.part_cap:
            self.part = rt.alloc(8 * need)
            self.part_cap = need
        return self.part.ptr

    def take_init_flag(self):
        first = not self.launched
        self.launched = True
        return 1 if first else 0

    def read_words(self, err=None):
        """Slot words (values..., flag) or None if no loop ever ran.  With
        `err` (a list), the device error word is read in the same sync and
        appended as (code, info)."""
        if not self.launched:
            return None
        F = len(self.ks)
        if self.mirrored:
            rt.sync()
            w = (ctypes.c_uint64 * (F + 3)).from_address(self.mirror)[:]
            if err is not None:
                code, info = w[F + 1], w[F + 2]
                if code:
                    rt.clear_error()
                err.append((code - (1 << 64) if code >> 63 else code, info - (1 << 64) if info >> 63 else info))
            return w[:F + 1]
        arr = np.empty(F + 1, dtype=np.uint64)
        if err is not None:
            err.append(rt.d2h_checked(arr.ctypes.data, self.slot.ptr, arr.nbytes))
        else:
            rt.d2h(arr.ctypes.data, self.slot.ptr, arr.nbytes)
        return arr

    def read(self, err=None):
        arr = self.read_words(err)
        F = len(self.ks)
        if arr is None or not arr[F]:
            vals = [identity_value(self.kind.op, k) for k in self.ks]
        else:
            vals = [from_bits(k, int(w)) for k, w in zip(self.ks, arr[:F])]
        return unflatten(self.kind.elem, vals)


class Segment:
    """A run of appended rows: leaf columns plus either a host-known length
    or a device counter (scan appenders) read lazily."""

    __slots__ = ("cols", "n", "total_buf", "cap")

    def __init__(self, cols, n=None, total_buf=None, cap=0):
        self.cols = cols
        self.n = n
        self.total_buf = total_buf
        self.cap = cap

    def length(self):
        if self.n is None:
            arr = np.zeros(1, dtype=np.int64)
            rt.d2h(arr.ctypes.data, self.total_buf.ptr, 8)
            self.n = int(arr[0])
        return self.n


class AppenderDev(BuilderBase):
    """vecbuilder (and the row log of groupbuilder).  A vecbuilder[vec[T]]
    fed fixed-length vector literals keeps T's leaves here (nested=True) and
    gets its offsets at result()."""

    nested = False
    nested_len = 1

    def __init__(self, kind, kinds, hint=None):
        super().__init__(kind)
        self.kinds = kinds
        self.hint = hint
        self.segments = []

    def new_segment(self, n_rows, direct):
        cols = [Col.alloc(k, n_rows) for k in self.kinds]
        if direct:
            seg = Segment(cols, n=n_rows, cap=n_rows)
        else:
            tb = rt.alloc(8)
            rt.memset(tb.ptr, 0, 8)
            seg = Segment(cols, total_buf=tb, cap=n_rows)
        self.segments.append(seg)
        return seg

    def concat(self):
        """All segments as one set of leaf columns, in append order."""
        lens = [s.length() for s in self.segments]
        total = sum(lens)
        if len(self.segments) == 1:
            return self.segments[0].cols, total
        cols = [Col.alloc(k, total) for k in self.kinds]
        off = 0
        for seg, n in zip(self.segments, lens):
            for dst, src, k in zip(cols, seg.cols, self.kinds):
                rt.d2d(dst.ptr + off * SIZE[k], src.ptr, n * SIZE[k])
            off += n
        return cols, total


class VecMergerDev(BuilderBase):
    def __init__(self, kind: VecMerger, init: DVec):
        super().__init__(kind)
        self.ks = leaves(kind.elem)
        self.n = init.n
        self.cols = []
        for c, k in zip(init.cols, self.ks):
            nc = Col.alloc(k, self.n)
            rt.d2d(nc.ptr, c.ptr, self.n * SIZE[k])
            self.cols.append(nc)


_SIZE_HINTS = {}   # loop identity -> distinct keys seen last time (table sizing)


class DictDev(BuilderBase):
    """dictmerger state: an open-addressing table of 8-byte words.

    slot = [key word] + values          (one-word keys, EMPTY = all ones)
         = [state, key words] + values  (multi-word keys)
    Value fields are pre-initialised to the fold's internal identity, so a
    claimed slot is merged into with plain atomics.  An insert that finds
    WG_MAX_PROBE foreign keys in a row spills to the overflow list; the host
    then grows the table (4x the distinct count), re-inserts the entries and
    replays the spilled merges (all dict folds are commutative).  The table
    is sized from the distinct count the same loop produced last time, else
    from min(merges, 2^24)."""

    def __init__(self, kind: DictMerger):
        super().__init__(kind)
        self.kks = leaves(kind.key)
        self.vks = leaves(kind.value)
        self.lay, self.nw = key_layout(self.kks)
        self.kbase = 1 if self.nw == 1 else 1 + self.nw
        self.slot_words = self.kbase + len(self.vks)
        self.table = None
        self.cap = 0
        self.counters = rt.alloc(16)          # [distinct keys, spilled merges]
        rt.memset(self.counters.ptr, 0, 16)
        self.over = None
        self.ocap = 0
        self.hint_key = None
        self.distinct = 0

    @property
    def count(self):
        return _Ptr(self.counters.ptr)

    @property
    def ocount(self):
        return _Ptr(self.counters.ptr + 8)

    def pattern(self):
        head = [ALL_ONES] if self.nw == 1 else [0] * (1 + self.nw)
        return head + [to_bits(k, internal_identity(self.kind.op, k)) for k in self.vks]

    def ensure(self, rows, hint_key=None):
        """Size the table before a launch of `rows` merges, and the spill
        list for that launch."""
        if self.table is None:
            self.hint_key = hint_key
            seen = _SIZE_HINTS.get(hint_key)
            want = seen if seen is not None else min(rows, 1 << 24)
            self._alloc_table(1 << max(10, int(max(want, 1) * 2 - 1).bit_length()))
        if rows > self.ocap:
            self.over = ([rt.alloc(8 * rows) for _ in range(self.nw)],
                         [rt.alloc(8 * rows) for _ in self.vks])
            self.ocap = rows

    def ensure_part(self, rows, nparts):
        """Buckets for the partitioned mode: nparts x pcap records of
        (key word, value words); counters zeroed for this launch."""
        pcap = (rows * 5) // (4 * nparts) + 64
        if getattr(self, "pcap", 0) < pcap or getattr(self, "nparts", 0) != nparts:
            self.pcap = pcap
            self.nparts = nparts
            self.pcount = rt.alloc(8 * nparts)
            self.pk = rt.alloc(8 * nparts * pcap)
            self.pv = [rt.alloc(8 * nparts * pcap) for _ in self.vks]
        rt.memset(self.pcount.ptr, 0, 8 * nparts)

    def _alloc_table(self, cap):
        self.cap = cap
        self.table = rt.alloc(8 * (cap + 1) * self.slot_words)
        pat = (ctypes.c_uint64 * self.slot_words)(*self.pattern())
        rt.call("wg_table_init", self.table.ptr, cap + 1, self.slot_words, pat)
        rt.memset(self.counters.ptr, 0, 16)

    def read_counters(self):
        arr = np.zeros(2, dtype=np.uint64)
        rt.d2h(arr.ctypes.data, self.counters.ptr, 16)
        self.distinct = int(arr[0])
        if self.hint_key is not None:
            _SIZE_HINTS[self.hint_key] = max(self.distinct, _SIZE_HINTS.get(self.hint_key, 0))
        return self.distinct, int(arr[1])

    def compact(self):
        """Occupied entries as SoA word columns (keys words, value words)."""
        distinct, _ = self.read_counters()
        nout = self.nw + len(self.vks)
        outs = [rt.alloc(8 * (distinct + 1)) for _ in range(nout)]
        ptrs = (ctypes.c_uint64 * nout)(*[o.ptr for o in outs])
        cnt = ctypes.c_uint64(0)
        mode = 1 if self.nw == 1 else 2
        rt.call("wg_table_compact", self.table.ptr, self.cap, self.slot_words, mode, ptrs, nout, ctypes.byref(cnt))
        if cnt.value != distinct:
            raise RuntimeError(f"dictmerger table holds {cnt.value} keys, counted {distinct}")
        return outs[:self.nw], outs[self.nw:], cnt.value


class _Ptr:
    __slots__ = ("ptr",)

    def __init__(self, ptr):
        self.ptr = ptr


class GroupDev(AppenderDev):
    def __init__(self, kind: GroupBuilder):
        super().__init__(kind, leaves(kind.key) + leaves(kind.value))
        self.kks = leaves(kind.key)
        self.vks = leaves(kind.value)


# ---------------------------------------------------------------------------
# Device results of keyed builders


class DDict:
    """A finalised dictmerger: entries sorted by key (order_key)."""

    def __init__(self, ty, keys: DVec, vals: DVec):
        self.ty = ty        # Dict(K, V)
        self.keys = keys
        self.vals = vals
        self.n = keys.n
        self._host = None

    def __len__(self):
        return self.n


class DGroups:
    """A finalised groupbuilder: sorted unique keys, offsets, values in
    per-key input order."""

    def __init__(self, ty, keys: DVec, offsets: Col, vals: DVec):
        self.ty = ty        # Dict(K, Vec(V))
        self.keys = keys
        self.offsets = offsets
        self.vals = vals
        self.n = keys.n
        self._host = None

    def __len__(self):
        return self.n


def _words_to_cols(word_bufs, kinds, lay, n):
    """Unpack packed key words into typed leaf columns."""
    cols = []
    words_np = None
    simple = all(w == 64 for (_, _, w) in lay)
    if simple:
        for (wi, _, _), k in zip(lay, kinds):
            c = Col(word_bufs[wi].ptr, k, word_bufs[wi])
            cols.append(c)
        return cols
    # Narrow packed fields on the host side of the device: small helper via numpy
    # round trip is avoided by doing shifts on device through gather-free path:
    words_np = [col_to_numpy(Col(b.ptr, I64, b), n).view(np.uint64) for b in word_bufs]
    for (wi, sh, width), k in zip(lay, kinds):
        raw = (words_np[wi] >> np.uint64(sh)) & np.uint64((1 << width) - 1 if width < 64 else ALL_ONES)
        if k == I32:
            arr = raw.astype(np.uint32).view(np.int32)
        elif k == F32:
            arr = raw.astype(np.uint32).view(np.float32)
        elif k == BOOL:
            arr = raw.astype(np.uint8)
        elif k == F64:
            arr = raw.view(np.float64)
        else:
            arr = raw.view(np.int64)
        c = Col.alloc(k, n)
        a = np.ascontiguousarray(arr)
        if n:
            rt.h2d(c.ptr, a.ctypes.data, a.nbytes)
        cols.append(c)
    return cols


def _value_words_to_cols(word_bufs, kinds, n):
    cols = []
    for b, k in zip(word_bufs, kinds):
        if SIZE[k] == 8:
            cols.append(Col(b.ptr, k, b))
        else:
            c = Col.alloc(k, n)
            rt.call("wg_narrow", b.ptr, c.ptr, SIZE[k], n)
            cols.append(c)
    return cols


def sort_perm(key_cols, n):
    """Stable permutation sorting rows by the key leaves lexicographically
    (order_key total order).  LSD: last leaf first."""
    perm = rt.alloc(4 * max(n, 1))
    rt.call("wg_iota_u32", perm.ptr, n)
    if n <= 1:
        return perm
    kbuf = rt.alloc(8 * n)
    kout = rt.alloc(8 * n)
    pout = rt.alloc(4 * n)
    for c in reversed(key_cols):
        k = c.kind
        rt.call("wg_order_key", c.ptr, KIND_CODE[k], n, perm.ptr, kbuf.ptr)
        if k == BOOL:
            lo, hi = 0, 8
        elif k == I32:
            lo, hi = 0, 64   # sign-extended then flipped: all 64 bits vary
        else:
            lo, hi = 0, 64
        rt.call("wg_sort_pairs", kbuf.ptr, perm.ptr, kout.ptr, pout.ptr, n, lo, hi)
        perm, pout = pout, perm
    return perm


def gather_cols(cols, perm, n):
    out = []
    for c in cols:
        nc = Col.alloc(c.kind, n)
        rt.call("wg_gather", c.ptr, perm.ptr, nc.ptr, n, SIZE[c.kind])
        out.append(nc)
    return out


SMALL_DICT = 4096


def _finish_small(d: DictDev, dict_ty):
    """Results of <= SMALL_DICT entries: one launch (wg_dict_finish_small)
    instead of compaction + per-leaf radix sorts + gathers; the kernel also
    checks the spill counter, so the host syncs once.  Returns None when the
    general path (or a spill replay) is needed."""
    nkl, nvl = len(d.kks), len(d.vks)
    if nkl > 6 or nvl > 16 or (d.hint_key is not None and _SIZE_HINTS.get(d.hint_key, 0) > SMALL_DICT):
        return None
    n = SMALL_DICT
    cols = Col.alloc_many(list(d.kks) + list(d.vks), n)
    kcols, vcols = cols[:nkl], cols[nkl:]
    desc = []
    for (wi, sh, width), k in zip(d.lay, d.kks):
        desc += [wi, sh, width, KIND_CODE[k]]
    kd = (ctypes.c_int * len(desc))(*desc)
    vk = (ctypes.c_int * max(nvl, 1))(*[KIND_CODE[k] for k in d.vks])
    outs = (ctypes.c_uint64 * (nkl + nvl))(*[c.ptr for c in kcols + vcols])
    cnt = ctypes.c_uint64(0)
    mode = 1 if d.nw == 1 else 2
    rt.call("wg_dict_finish_small", d.table.ptr, d.cap, d.slot_words, mode, d.nw, nkl, kd, nvl, vk, outs,
            d.counters.ptr, ctypes.byref(cnt))
    # the error word came back with the count (same sync); the caller raises it
    d.sync_err = rt.last_sync_error()
    n = cnt.value
    if n > SMALL_DICT:          # too many entries, or spilled merges to replay first
        return None
    d.distinct = n
    if d.hint_key is not None:
        _SIZE_HINTS[d.hint_key] = max(n, _SIZE_HINTS.get(d.hint_key, 0))
    return DDict(dict_ty, dvec_from_cols(dict_ty.key, n, kcols), dvec_from_cols(dict_ty.value, n, vcols))


def finish_dict(d: DictDev, dict_ty):
    small = _finish_small(d, dict_ty)
    if small is not None:
        return small
    kw, vw, n = d.compact()
    kcols = _words_to_cols(kw, d.kks, d.lay, n)
    vcols = _value_words_to_cols(vw, d.vks, n)
    if len(kcols) == 1 and len(vcols) == 1 and d.kks[0] in (BOOL, I32, I64) and 1 < n < (1 << 32):
        # one integer key leaf, one value leaf: the groupbuilder finisher's
        # stable sort on the varying key bits carries the value through the
        # radix passes (no permutation + gathers); keys are distinct, so the
        # runs are the entries themselves
        uk = Col.alloc(d.kks[0], n)
        offs = Col.alloc(I64, n + 1)
        vo = Col.alloc(vcols[0].kind, n)
        K = ctypes.c_uint64(0)
        rt.call("wg_group_finish1", kcols[0].ptr, KIND_CODE[d.kks[0]], vcols[0].ptr, SIZE[vcols[0].kind], n,
                uk.ptr, offs.ptr, vo.ptr, ctypes.byref(K))
        if K.value != n:
            raise RuntimeError(f"dictmerger result has {K.value} distinct keys, expected {n}")
        kcols, vcols = [uk], [vo]
    else:
        perm = sort_perm(kcols, n)
        kcols = gather_cols(kcols, perm, n)
        vcols = gather_cols(vcols, perm, n)
    return DDict(dict_ty, dvec_from_cols(dict_ty.key, n, kcols), dvec_from_cols(dict_ty.value, n, vcols))


def finish_groups(g: GroupDev, dict_ty):
    cols, n = g.concat()
    nk = len(g.kks)
    kcols, vcols = cols[:nk], cols[nk:]
    if nk == 1 and len(vcols) == 1 and g.kks[0] in (BOOL, I32, I64) and n < (1 << 32):
        # device fast path: adaptive-window radix sort + bucket sort + run starts
        ukeys = Col.alloc(g.kks[0], max(n, 1))
        offs = Col.alloc(I64, n + 1)
        vout = Col.alloc(vcols[0].kind, max(n, 1))
        K = ctypes.c_uint64(0)
        rt.call("wg_group_finish1", kcols[0].ptr, KIND_CODE[g.kks[0]], vcols[0].ptr, SIZE[vcols[0].kind], n,
                ukeys.ptr, offs.ptr, vout.ptr, ctypes.byref(K))
        K = K.value
        return DGroups(dict_ty, dvec_from_cols(dict_ty.key, K, [ukeys]), offs,
                       dvec_from_cols(dict_ty.value.elem, n, [vout]))
    perm = sort_perm(kcols, n)
    kcols = gather_cols(kcols, perm, n)
    vcols = gather_cols(vcols, perm, n)
    # run starts over the sorted keys
    if n == 0:
        offs = Col.alloc(I64, 1)
        rt.memset(offs.ptr, 0, 8)
        keys = dvec_from_cols(dict_ty.key, 0, [Col.alloc(k, 0) for k in g.kks])
        return DGroups(dict_ty, keys, offs, dvec_from_cols(dict_ty.value.elem, 0, vcols))
    words = []
    for c in kcols:
        if c.kind in (F32, F64):
            # float keys compare as the reference's dict keys do: -0.0 == 0.0
            # and NaN with NaN (order_key words); each run keeps its first
            # row's key, i.e. the first-inserted key object
            wc = Col.alloc(I64, n)
            rt.call("wg_order_key", c.ptr, KIND_CODE[c.kind], n, 0, wc.ptr)
            words.append(wc)
        elif SIZE[c.kind] == 8:
            words.append(c)
        else:
            wc = Col.alloc(I64, n)
            rt.call("wg_widen", c.ptr, wc.ptr, SIZE[c.kind], n)
            words.append(wc)
    starts = rt.alloc(4 * n)
    wptrs = (ctypes.c_uint64 * len(words))(*[w.ptr for w in words])
    nruns = ctypes.c_uint64(0)
    rt.call("wg_run_starts", wptrs, len(words), n, starts.ptr, ctypes.byref(nruns))
    K = nruns.value
    ukeys = gather_cols(kcols, starts, K)
    st = np.empty(K, dtype=np.uint32)
    rt.d2h(st.ctypes.data, starts.ptr, 4 * K)
    offs_np = np.empty(K + 1, dtype=np.int64)
    offs_np[:K] = st
    offs_np[K] = n
    offs = Col.alloc(I64, K + 1)
    rt.h2d(offs.ptr, offs_np.ctypes.data, offs_np.nbytes)
    return DGroups(dict_ty, dvec_from_cols(dict_ty.key, K, ukeys), offs,
                   dvec_from_cols(dict_ty.value.elem, n, vcols))


def dict_payload(d):
    """Reference payload: a Python dict in key order."""
    if d._host is None:
        from .columns import to_payload
        ks = to_payload(d.keys)
        if isinstance(d, DDict):
            vs = to_payload(d.vals)
            d._host = dict(zip(ks, vs))
        else:
            offs = col_to_numpy(d.offsets, d.n + 1)
            vals = to_payload(d.vals)
            d._host = {k: vals[offs[j]:offs[j + 1]] for j, k in enumerate(ks)}
    return d._host


def tovec(d, vec_elem_ty):
    """ToVec (run.py:737-747): entries already sorted by key."""
    if isinstance(d, DDict):
        lay = (d.keys.layout, d.vals.layout)
        return DVec(vec_elem_ty, d.n, lay)
    return DVec(vec_elem_ty, d.n, (d.keys.layout, ListLayout(d.offsets, d.vals.layout, d.vals.n)))


__all__ = ["MergerDev", "AppenderDev", "GroupDev", "DictDev", "VecMergerDev", "DDict", "DGroups", "finish_dict",
           "finish_groups", "dict_payload", "tovec", "sort_perm", "gather_cols", "Struct", "Vec", "Scalar",
           "VecBuilder", "DeviceUnsupported", "F32", "F64", "I32"]

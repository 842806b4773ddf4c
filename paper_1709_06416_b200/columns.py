"""Device-resident columnar values (the buffer manager's view of IR vectors).

A ``vec[T]`` lives in HBM as structure-of-arrays: one contiguous column per
scalar leaf of T (bool as one byte), so a zipped loop ``for({a, b, c}, ...)``
and an AoS ``vec[{..}]`` read the same way.  Nested ``vec[vec[T]]`` (group
results, vec-of-vec maps) carry an offsets column (n+1 i64) over a child
layout.  The wire format of the reference (``boundary.py:1-12``: i64 count +
packed little-endian elements, structs without padding) converts to and from
this layout with numpy, without Python-object round trips.
"""
from __future__ import annotations

import ctypes
import os
import struct as _struct

import numpy as np

from . import runtime as rt
from .irtypes import (BOOL, F32, F64, I32, I64, NPTYPE, SIZE, DeviceUnsupported, Scalar, Struct, Vec, leaves)


class Col:
    """One device column: a pointer plus the buffer that owns it."""

    __slots__ = ("ptr", "kind", "owner")

    def __init__(self, ptr, kind, owner):
        self.ptr = ptr
        self.kind = kind
        self.owner = owner

    @classmethod
    def alloc(cls, kind, n):
        buf = rt.alloc(max(n, 1) * SIZE[kind])
        return cls(buf.ptr, kind, buf)

    @classmethod
    def alloc_many(cls, kinds, n):
        """Columns of n elements for each kind, carved from ONE device
        buffer (256-byte aligned): one allocator call instead of len(kinds)."""
        offs, total = [], 0
        for k in kinds:
            offs.append(total)
            total += (max(n, 1) * SIZE[k] + 255) // 256 * 256
        buf = rt.alloc(max(total, 1))
        return [cls(buf.ptr + o, k, buf) for o, k in zip(offs, kinds)]

    def offset(self, k):
        """A view starting k elements in."""
        return Col(self.ptr + k * SIZE[self.kind], self.kind, self.owner)


class ListLayout:
    """Layout of a Vec-typed field: offsets (n+1, i64) over a child layout."""

    __slots__ = ("offsets", "child", "total")

    def __init__(self, offsets: Col, child, total: int):
        self.offsets = offsets
        self.child = child
        self.total = total


class DVec:
    """A device vector: IR type vec[elem], length n, layout tree."""

    __slots__ = ("elem", "n", "layout", "host_cache", "_cols")

    def __init__(self, elem, n, layout):
        self.elem = elem
        self.n = int(n)
        self.layout = layout
        self.host_cache = None
        self._cols = None

    @property
    def cols(self):
        """Flat leaf columns (only for flat element types)."""
        if self._cols is not None:
            return self._cols
        out = []

        def go(t, lay):
            if isinstance(t, Scalar):
                out.append(lay)
            elif isinstance(t, Struct):
                for ft, fl in zip(t.fields, lay):
                    go(ft, fl)
            else:
                raise DeviceUnsupported(f"element type {self.elem} is not flat")

        try:
            go(self.elem, self.layout)
        finally:
            del go  # break the closure's self-reference cycle (it pins buffers until GC)
        self._cols = out
        return out

    def __len__(self):
        return self.n

    def __repr__(self):
        return f"<DVec vec[{self.elem}] n={self.n}>"


def layout_from_cols(elem, cols):
    it = iter(cols)

    def go(t):
        if isinstance(t, Scalar):
            return next(it)
        if isinstance(t, Struct):
            return tuple(go(f) for f in t.fields)
        raise DeviceUnsupported(f"cannot build a flat layout for {t}")

    try:
        return go(elem)
    finally:
        del go


def dvec_from_cols(elem, n, cols):
    return DVec(elem, n, layout_from_cols(elem, cols))


# ---------------------------------------------------------------------------
# host -> device


def _np_upload(arr: np.ndarray, kind) -> Col:
    arr = np.ascontiguousarray(arr, dtype=np.dtype(NPTYPE[kind]))
    col = Col.alloc(kind, arr.shape[0])
    if arr.nbytes:
        rt.h2d(col.ptr, arr.ctypes.data, arr.nbytes)
    return col


def _leaf_arrays_from_payload(elem, payload):
    """Python payload (list of scalars / tuples) -> list of numpy leaf arrays."""
    ks = leaves(elem)
    n = len(payload)
    if isinstance(elem, Scalar):
        if n == 0:
            return [np.zeros(0, dtype=NPTYPE[elem.kind])]
        return [np.asarray(payload, dtype=NPTYPE[elem.kind])]
    if n == 0:
        return [np.zeros(0, dtype=NPTYPE[k]) for k in ks]
    flat_rows = payload
    if any(isinstance(f, Struct) for f in elem.fields):
        from .irtypes import flatten_value
        flat_rows = [flatten_value(elem, r) for r in payload]
    cols = list(zip(*flat_rows))
    return [np.asarray(c, dtype=NPTYPE[k]) for c, k in zip(cols, ks)]


def to_device(ty, payload) -> DVec:
    """Bind a host vector payload of IR type ``ty`` (a Vec) to the device.

    Accepts the reference's payload (a list of scalars or tuples), a numpy
    array (scalar elements, or a structured array), a tuple/list of numpy
    arrays (SoA, one per leaf), boundary bytes, or an existing DVec.
    """
    if isinstance(payload, DVec):
        return payload
    if not isinstance(ty, Vec):
        raise DeviceUnsupported(f"cannot bind {ty} as a device vector")
    elem = ty.elem
    if isinstance(elem, Vec) or (isinstance(elem, Struct) and any(isinstance(f, Vec) for f in elem.fields)):
        return _nested_to_device(elem, payload)
    ks = leaves(elem)
    if isinstance(payload, (bytes, bytearray, memoryview)):
        arrs = boundary_to_arrays(elem, bytes(payload))
    elif isinstance(payload, np.ndarray):
        if payload.dtype.names:
            arrs = [payload[nm] for nm in payload.dtype.names]
        else:
            arrs = [payload]
    elif isinstance(payload, tuple) and payload and all(isinstance(a, np.ndarray) for a in payload):
        arrs = list(payload)
    else:
        arrs = _leaf_arrays_from_payload(elem, payload)
    if len(arrs) != len(ks):
        raise DeviceUnsupported(f"payload has {len(arrs)} columns, type {elem} needs {len(ks)}")
    n = int(arrs[0].shape[0]) if arrs else 0
    cols = [_np_upload(a, k) for a, k in zip(arrs, ks)]
    return dvec_from_cols(elem, n, cols)


def _nested_to_device(elem, payload):
    if isinstance(payload, (bytes, bytearray, memoryview)):
        from weldmill.boundary import decode_value
        payload = decode_value(bytes(payload), Vec(elem))

    def build(t, items):
        if isinstance(t, Scalar):
            return _np_upload(np.asarray(items if items else [], dtype=NPTYPE[t.kind]), t.kind)
        if isinstance(t, Struct):
            cols = list(zip(*items)) if items else [[] for _ in t.fields]
            return tuple(build(ft, list(c)) for ft, c in zip(t.fields, cols))
        if isinstance(t, Vec):
            offs = np.zeros(len(items) + 1, dtype=np.int64)
            flat = []
            for j, it in enumerate(items):
                offs[j + 1] = offs[j] + len(it)
                flat.extend(it)
            return ListLayout(_np_upload(offs, I64), build(t.elem, flat), int(offs[-1]))
        raise DeviceUnsupported(f"cannot bind {t}")

    items = list(payload)
    try:
        return DVec(elem, len(items), build(elem, items))
    finally:
        del build


# ---------------------------------------------------------------------------
# device -> host


def col_to_numpy(col: Col, n: int) -> np.ndarray:
    arr = np.empty(n, dtype=np.dtype(NPTYPE[col.kind]))
    if n:
        rt.d2h(arr.ctypes.data, col.ptr, arr.nbytes)
    return arr


class _PinnedBlock:
    """Page-locked host memory from cudaHostAlloc, recycled through a pool
    when the numpy array viewing it dies.  Sizes are rounded like the device
    allocator (pow2 below 2 MiB, 2 MiB multiples above) and a request reuses
    any cached block up to 2x its size; cached bytes are capped
    (WELDGPU_PINNED_CACHE, default 8 GiB) -- the oldest blocks beyond the
    cap go back to the driver (wg_host_free) -- and ``trim_pinned()`` frees
    every cached block."""

    __slots__ = ("ptr", "nbytes", "__weakref__")
    _pool = []            # cached (size, ptr), oldest first
    _cached = 0
    CAP = int(os.environ.get("WELDGPU_PINNED_CACHE", str(8 << 30)))

    def __init__(self, nbytes):
        size = _round_pinned(nbytes)
        pool = _PinnedBlock._pool
        best = None
        for q, (sz, _) in enumerate(pool):
            if size <= sz <= 2 * size and (best is None or sz < pool[best][0]):
                best = q
        if best is not None:
            sz, ptr = pool.pop(best)
            _PinnedBlock._cached -= sz
            self.ptr, self.nbytes = ptr, sz
            return
        p = ctypes.c_void_p(0)
        try:
            rt.call("wg_host_alloc", size, ctypes.byref(p))
        except rt.WeldGpuError:
            trim_pinned()
            rt.call("wg_host_alloc", size, ctypes.byref(p))
        self.ptr, self.nbytes = p.value, size

    def __del__(self):
        try:
            _PinnedBlock._pool.append((self.nbytes, self.ptr))
            _PinnedBlock._cached += self.nbytes
            while _PinnedBlock._cached > _PinnedBlock.CAP and _PinnedBlock._pool:
                sz, ptr = _PinnedBlock._pool.pop(0)
                _PinnedBlock._cached -= sz
                rt.call("wg_host_free", ptr)
        except Exception:
            pass


def _round_pinned(nbytes):
    if nbytes < (2 << 20):
        r = 4096
        while r < nbytes:
            r <<= 1
        return r
    return (nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20)


def trim_pinned():
    """Free every cached pinned host block (results still alive keep theirs)."""
    pool = _PinnedBlock._pool
    while pool:
        sz, ptr = pool.pop()
        _PinnedBlock._cached -= sz
        rt.call("wg_host_free", ptr)


def pinned_cache_bytes():
    return _PinnedBlock._cached


PINNED_MIN_BYTES = 1 << 20


def pinned_empty(n, dtype):
    """A numpy array in pinned host memory (full-bandwidth async D2H)."""
    dt = np.dtype(dtype)
    nbytes = max(n * dt.itemsize, 1)
    blk = _PinnedBlock(nbytes)
    raw = (ctypes.c_char * nbytes).from_address(blk.ptr)
    raw._wg_owner = blk          # the array keeps the block alive
    return np.frombuffer(raw, dtype=dt, count=n)


def to_numpy(v: DVec):
    """Flat vector -> numpy (scalar elem) or tuple of leaf arrays.  Large
    columns land in pinned host memory: one async copy per column, one sync."""
    cols = v.cols
    arrs = []
    for c in cols:
        nb = v.n * SIZE[c.kind]
        if nb >= PINNED_MIN_BYTES:
            a = pinned_empty(v.n, NPTYPE[c.kind])
            rt.d2h_async(a.ctypes.data, c.ptr, nb)
        else:
            a = np.empty(v.n, dtype=np.dtype(NPTYPE[c.kind]))
            if nb:
                rt.d2h_async(a.ctypes.data, c.ptr, nb)
        arrs.append(a)
    rt.sync()
    if isinstance(v.elem, Scalar):
        return arrs[0]
    return tuple(arrs)


class Ragged:
    """numpy form of a nested ``vec[T]`` column: ``offsets`` (n+1 i64) over
    ``values`` (the child's numpy form).  Row j is values[offsets[j]:
    offsets[j+1]] -- the reference's list-of-lists (builders.py:478-493)
    without one Python object per element."""

    __slots__ = ("offsets", "values")

    def __init__(self, offsets, values):
        self.offsets = offsets
        self.values = values

    def __len__(self):
        return len(self.offsets) - 1

    def __getitem__(self, j):
        a, b = int(self.offsets[j]), int(self.offsets[j + 1])
        v = self.values
        if isinstance(v, tuple):
            return tuple(x[a:b] for x in v)
        return v[a:b]

    def tolist(self):
        return [_np_tolist(self[j]) for j in range(len(self))]

    @property
    def nbytes(self):
        return self.offsets.nbytes + _np_nbytes(self.values)


def _np_tolist(v):
    if isinstance(v, tuple):
        return list(zip(*(_np_tolist(x) for x in v)))
    if isinstance(v, Ragged):
        return v.tolist()
    return v.tolist()


def _np_nbytes(v):
    if isinstance(v, tuple):
        return sum(_np_nbytes(x) for x in v)
    return v.nbytes


def to_numpy_nested(v: DVec):
    """Any vector -> numpy: flat leaves as arrays, structs as tuples, nested
    vectors as :class:`Ragged`.  One async copy per column into pinned
    memory, one sync."""

    def pull(kind, col, n):
        nb = n * SIZE[kind]
        a = pinned_empty(n, NPTYPE[kind]) if nb >= PINNED_MIN_BYTES else np.empty(n, dtype=np.dtype(NPTYPE[kind]))
        if nb:
            rt.d2h_async(a.ctypes.data, col.ptr, nb)
        return a

    def go(t, lay, n):
        if isinstance(t, Scalar):
            return pull(t.kind, lay, n)
        if isinstance(t, Struct):
            return tuple(go(ft, fl, n) for ft, fl in zip(t.fields, lay))
        if isinstance(t, Vec):
            offs = pull(I64, lay.offsets, n + 1)
            return Ragged(offs, go(t.elem, lay.child, int(lay.total)))
        raise DeviceUnsupported(f"cannot read back {t}")

    try:
        out = go(v.elem, v.layout, v.n)
    finally:
        del go
    rt.sync()
    return out


def _layout_to_payload(t, lay, n):
    if isinstance(t, Scalar):
        a = col_to_numpy(lay, n)
        if t.kind == BOOL:
            return [bool(x) for x in a]
        return a.tolist()
    if isinstance(t, Struct):
        parts = [_layout_to_payload(ft, fl, n) for ft, fl in zip(t.fields, lay)]
        return list(zip(*parts)) if n else []
    if isinstance(t, Vec):
        offs = col_to_numpy(lay.offsets, n + 1)
        flat = _layout_to_payload(t.elem, lay.child, int(offs[-1]) if n + 1 else 0)
        return [flat[offs[j]:offs[j + 1]] for j in range(n)]
    raise DeviceUnsupported(f"cannot read back {t}")


def to_payload(v: DVec):
    """The reference's payload form: a list of scalars / tuples / lists."""
    if v.host_cache is None:
        v.host_cache = _layout_to_payload(v.elem, v.layout, v.n)
    return v.host_cache


# ---------------------------------------------------------------------------
# boundary bytes (boundary.py:59-141) for flat element types


def _packed_dtype(elem):
    ks = leaves(elem)
    return np.dtype({"names": [f"f{i}" for i in range(len(ks))],
                     "formats": [NPTYPE[k] for k in ks],
                     "offsets": list(np.cumsum([0] + [SIZE[k] for k in ks])[:-1]),
                     "itemsize": sum(SIZE[k] for k in ks)})


def boundary_to_arrays(elem, data: bytes):
    (count,) = _struct.unpack_from("<q", data, 0)
    dt = _packed_dtype(elem)
    rec = np.frombuffer(data, dtype=dt, count=count, offset=8)
    return [np.ascontiguousarray(rec[nm]) for nm in dt.names]


def to_boundary_bytes(v: DVec) -> bytes:
    if not all(isinstance(c, Col) for c in v.cols):
        raise DeviceUnsupported("nested vectors use the generic encoder")
    dt = _packed_dtype(v.elem)
    rec = np.empty(v.n, dtype=dt)
    for nm, c in zip(dt.names, v.cols):
        rec[nm] = col_to_numpy(c, v.n)
    return _struct.pack("<q", v.n) + rec.tobytes()


__all__ = ["Col", "DVec", "ListLayout", "to_device", "to_numpy", "to_payload", "to_boundary_bytes",
           "dvec_from_cols", "col_to_numpy", "boundary_to_arrays", "ctypes"]

"""Type helpers: flattening IR types into SoA scalar leaves, C spellings,
storage widths and the reference's identities.

Reference: /root/reference/pkg/src/weldmill/types.py (Scalar/Struct/Vec,
SCALAR_SIZES :29, identity_value :185-192).
"""
from __future__ import annotations

import math
import struct as _struct

from . import _ref  # noqa: F401
from weldmill.types import (  # noqa: F401
    BOOL, F32, F64, I32, I64, FLOAT_KINDS, INT_KINDS,
    Builder, Dict, DictMerger, Function, GroupBuilder, Merger, Scalar, Simd,
    Struct, Vec, VecBuilder, VecMerger,
)

# C type used for computation in generated kernels.
CTYPE = {BOOL: "bool", I32: "i32", I64: "i64", F32: "float", F64: "double"}
# C type used for storage in device columns (bool is one byte).
STYPE = {BOOL: "u8", I32: "i32", I64: "i64", F32: "float", F64: "double"}
SIZE = {BOOL: 1, I32: 4, I64: 8, F32: 4, F64: 8}
NPTYPE = {BOOL: "u1", I32: "<i4", I64: "<i8", F32: "<f4", F64: "<f8"}
# kind codes shared with libweldgpu (k_order_key)
KIND_CODE = {BOOL: 0, I32: 1, I64: 2, F32: 3, F64: 4}

OPCODE = {"+": 0, "*": 1, "min": 2, "max": 3}
OPSTRUCT = {"+": "WgAdd", "*": "WgMul", "min": "WgMin", "max": "WgMax"}


class DeviceUnsupported(Exception):
    """Raised (as an EvalError subclass, see executor) for IR the device
    executor does not lower.  There is no CPU fallback."""


def leaves(t):
    """Flatten a type into its scalar leaves in field order (SoA layout)."""
    if isinstance(t, Scalar):
        return [t.kind]
    if isinstance(t, Struct):
        out = []
        for f in t.fields:
            out.extend(leaves(f))
        return out
    raise DeviceUnsupported(f"type {t} has no flat columnar layout")


def is_flat(t):
    if isinstance(t, Scalar):
        return True
    if isinstance(t, Struct):
        return all(is_flat(f) for f in t.fields)
    return False


def unflatten(t, values):
    """Rebuild a (nested) struct payload from its flat leaf list."""
    it = iter(values)

    def go(tt):
        if isinstance(tt, Scalar):
            return next(it)
        return tuple(go(f) for f in tt.fields)

    try:
        return go(t)
    finally:
        del go


def flatten_value(t, v):
    if isinstance(t, Scalar):
        return [v]
    out = []
    for ft, fv in zip(t.fields, v):
        out.extend(flatten_value(ft, fv))
    return out


def f32_round(v: float) -> float:
    try:
        return _struct.unpack("<f", _struct.pack("<f", v))[0]
    except OverflowError:
        return math.inf if v > 0 else -math.inf


def identity_value(op, kind):
    """types.py:185-192."""
    if kind in INT_KINDS:
        lo, hi = ((-(2**31), 2**31 - 1) if kind == I32 else (-(2**63), 2**63 - 1))
        return {"+": 0, "*": 1, "min": hi, "max": lo}[op]
    return {"+": 0.0, "*": 1.0, "min": math.inf, "max": -math.inf}[op]


def internal_identity(op, kind):
    """Exact no-op start value of the device folds (see weld_device.cuh)."""
    if kind in INT_KINDS:
        return identity_value(op, kind)
    return {"+": -0.0, "*": 1.0, "min": math.nan, "max": -math.inf}[op]


def to_bits(kind, v) -> int:
    """A scalar as the 64-bit slot word used by device tables/partials."""
    if kind == F64:
        return _struct.unpack("<Q", _struct.pack("<d", v))[0]
    if kind == F32:
        return _struct.unpack("<I", _struct.pack("<f", v))[0]
    if kind == I64:
        return v & 0xFFFFFFFFFFFFFFFF
    if kind == I32:
        return v & 0xFFFFFFFF
    return 1 if v else 0


def from_bits(kind, w: int):
    if kind == F64:
        return _struct.unpack("<d", _struct.pack("<Q", w & 0xFFFFFFFFFFFFFFFF))[0]
    if kind == F32:
        return _struct.unpack("<f", _struct.pack("<I", w & 0xFFFFFFFF))[0]
    if kind == I64:
        w &= 0xFFFFFFFFFFFFFFFF
        return w - (1 << 64) if w >> 63 else w
    if kind == I32:
        w &= 0xFFFFFFFF
        return w - (1 << 32) if w >> 31 else w
    return bool(w & 0xFF)


def builder_kind(t):
    if isinstance(t, Builder):
        return t.kind
    raise DeviceUnsupported(f"{t} is not a builder type")

"""Host-side scalar semantics for the executor's control plane.

Loops run on the device; the few scalar nodes *between* loops (loop bounds
like ``len(v) - len(v) % 4``, ``3 * result(...)``, struct assembly, merges
issued outside any loop) are evaluated here with the reference's exact
rules so device and host agree bit for bit:

  ints wrap, / and % truncate and raise DivideByZero   run.py:395-437
  f32 rounds every op; IEEE division by zero           run.py:440-464
  NaN-aware min/max folds                              builders.py:121-163
  float->int casts wrap after truncation               run.py:503-528
"""
from __future__ import annotations

import math

from . import _ref  # noqa: F401
from weldmill.errors import DivideByZero, EvalError

from .irtypes import BOOL, F32, F64, I32, FLOAT_KINDS, INT_KINDS, f32_round


def wrap(kind, x):
    bits = 32 if kind == I32 else 64
    x &= (1 << bits) - 1
    return x - (1 << bits) if x >> (bits - 1) else x


def fmin(a, b):
    if a != a:
        return b
    if b != b:
        return a
    return a if a <= b else b


def fmax(a, b):
    if a != a:
        return a
    if b != b:
        return b
    return a if a >= b else b


def fold(op, kind, a, b):
    """Merge fold for one scalar kind (builders.py:121-163)."""
    if kind in FLOAT_KINDS:
        rnd = f32_round if kind == F32 else (lambda v: v)
        if op == "+":
            return rnd(a + b)
        if op == "*":
            return rnd(a * b)
        if op == "min":
            return fmin(a, b)
        return fmax(a, b)
    if op == "+":
        return wrap(kind, a + b)
    if op == "*":
        return wrap(kind, a * b)
    if op == "min":
        return a if a <= b else b
    return a if a >= b else b


def _tdiv(a, b):
    q = a // b
    if q < 0 and q * b != a:
        q += 1
    return q


def binop(op, kind, a, b):
    if op in ("==", "!=", "<", "<=", ">", ">="):
        return {"==": a == b, "!=": a != b, "<": a < b, "<=": a <= b,
                ">": a > b, ">=": a >= b}[op]
    if kind == BOOL:
        if op == "&":
            return a and b
        if op == "|":
            return a or b
        raise EvalError(f"operator {op!r} undefined over bool")
    if kind in FLOAT_KINDS:
        rnd = f32_round if kind == F32 else (lambda v: v)
        if op == "+":
            return rnd(a + b)
        if op == "-":
            return rnd(a - b)
        if op == "*":
            return rnd(a * b)
        if op == "/":
            if b == 0.0:
                if a == 0.0 or a != a:
                    return math.nan
                return math.copysign(math.inf, a) * math.copysign(1.0, b)
            return rnd(a / b)
        if op == "%":
            if b == 0.0 or a != a or b != b or math.isinf(a):
                return math.nan
            return rnd(math.fmod(a, b))
        if op == "min":
            return fmin(a, b)
        if op == "max":
            return fmax(a, b)
        raise EvalError(f"operator {op!r} undefined over {kind}")
    if op == "+":
        return wrap(kind, a + b)
    if op == "-":
        return wrap(kind, a - b)
    if op == "*":
        return wrap(kind, a * b)
    if op == "/":
        if b == 0:
            raise DivideByZero("integer division by zero")
        return wrap(kind, _tdiv(a, b))
    if op == "%":
        if b == 0:
            raise DivideByZero("integer remainder by zero")
        return wrap(kind, a - _tdiv(a, b) * b)
    if op == "&":
        return a & b
    if op == "|":
        return a | b
    if op == "min":
        return b if b < a else a
    if op == "max":
        return b if b > a else a
    raise EvalError(f"operator {op!r} undefined over {kind}")


def neg(kind, v):
    if kind in FLOAT_KINDS:
        return f32_round(-v) if kind == F32 else -v
    return wrap(kind, -v)


def cast(src, dst, v):
    if src == dst:
        return v
    if dst in INT_KINDS:
        bits = 32 if dst == I32 else 64
        if src in FLOAT_KINDS:
            if v != v:
                return 0
            if v == math.inf:
                return (1 << (bits - 1)) - 1
            if v == -math.inf:
                return -(1 << (bits - 1))
            return wrap(dst, int(v))
        return wrap(dst, int(v))
    if dst in FLOAT_KINDS:
        if dst == F32:
            return f32_round(float(v))
        return float(v)
    raise EvalError(f"cannot cast {src} to {dst}")


def literal(kind, v):
    if kind == F32 and isinstance(v, float):
        return f32_round(v)
    if kind in FLOAT_KINDS:
        return float(v)
    if kind == BOOL:
        return bool(v)
    return int(v)


__all__ = ["wrap", "fold", "binop", "neg", "cast", "literal", "fmin", "fmax", "F64"]

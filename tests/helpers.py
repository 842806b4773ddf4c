"""Shared comparison helpers (the reference's tolerance convention,
/root/reference/pkg/tests/test_acceptance.py:93-101, with the north-star
bounds: 1e-9 relative for f64, 1e-5 for f32)."""
import json
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))
F64_TOL = 1e-9
F32_TOL = 1e-5


def norm(v):
    if isinstance(v, (list, tuple)):
        return [norm(x) for x in v]
    if isinstance(v, dict):
        return [[norm(k), norm(x)] for k, x in v.items()]
    return v


def approx_equal(a, b, tol):
    if isinstance(a, (list, tuple)):
        return (isinstance(b, (list, tuple)) and len(a) == len(b)
                and all(approx_equal(x, y, tol) for x, y in zip(a, b)))
    if isinstance(a, float) or isinstance(b, float):
        if isinstance(a, bool) or isinstance(b, bool):
            return a == b
        if a != a and b != b:
            return True
        if math.isinf(a) or math.isinf(b):
            return a == b
        return abs(a - b) <= tol * max(1.0, abs(a), abs(b))
    return a == b


def first_diff(a, b, tol, path="$"):
    if isinstance(a, (list, tuple)) and isinstance(b, (list, tuple)):
        if len(a) != len(b):
            return f"{path}: length {len(a)} vs {len(b)}"
        for i, (x, y) in enumerate(zip(a, b)):
            d = first_diff(x, y, tol, f"{path}[{i}]")
            if d:
                return d
        return None
    if not approx_equal(a, b, tol):
        return f"{path}: {a!r} vs {b!r}"
    return None


def load_golden(name):
    with open(os.path.join(HERE, "golden", name)) as f:
        return json.load(f)

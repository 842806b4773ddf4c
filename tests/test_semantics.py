"""Host control-plane scalar semantics (semantics.py) agree with the
reference engine on the reference's own scalar-semantics cases
(/root/reference/pkg/tests/test_engine.py:198-226) and on fuzzed inputs."""
import math
import random

import pytest


def _ref(src):
    import paper_1709_06416_b200  # noqa: F401
    from weldmill.engine import evaluate
    from weldmill.parser import parse
    from weldmill.sugar import expand
    from weldmill.typecheck import infer
    return evaluate(infer(expand(parse(src)), {}))[0].data


def _host(src):
    """Evaluate a scalar program through the executor's host control plane
    (no loops -> no device work)."""
    import paper_1709_06416_b200  # noqa: F401
    from paper_1709_06416_b200.executor import Ctx
    from weldmill.engine import EngineConfig
    from weldmill.parser import parse
    from weldmill.sugar import expand
    from weldmill.typecheck import infer
    return Ctx(EngineConfig(), {}).ev(infer(expand(parse(src)), {}), {})


CASES = ["9223372036854775807 + 1", "2147483647si32 + 1si32", "(-7) / 2", "(-7) % 2", "7 / -2", "1.0 / 0.0",
         "min(1.5, 0.0 / 0.0)", "0.1f + 0.2f", "false && (1 / 0 > 0)", "true || (1 / 0 > 0)", "cast(3.7, i64)",
         "cast(-3.7, i64)", "cast(300si32, i64)", "cast(3, f64)", "cast(1e30, i64)", "cast(-1e30, i32)",
         "cast(0.0 / 0.0, i64)", "cast(1e9999, i32)", "(-9223372036854775807 - 1) / -1", "5 % -3",
         "min(3, 2)", "max(0.0 / 0.0, 1.0)", "cast(9007199254740993, f32)", "-(0.0)", "3.5 % 0.0"]


@pytest.mark.parametrize("src", CASES)
def test_matches_reference(src):
    a, b = _ref(src), _host(src)
    if isinstance(a, float) and math.isnan(a):
        assert math.isnan(b)
    else:
        assert a == b and type(a) is type(b), (a, b)
        if isinstance(a, float):
            assert math.copysign(1.0, a) == math.copysign(1.0, b)


def test_fuzz_integer_ops():
    rng = random.Random(20261017)
    for _ in range(300):
        a = rng.randint(-2**63, 2**63 - 1)
        b = rng.choice([rng.randint(-2**63, 2**63 - 1), rng.randint(-9, 9) or 1])
        op = rng.choice(["+", "-", "*", "/", "%", "min", "max"])
        expr = f"{op}({a}, {b})" if op in ("min", "max") else f"({a}) {op} ({b})"
        assert _ref(expr) == _host(expr), expr


def test_divide_by_zero_raises():
    from weldmill.errors import DivideByZero
    with pytest.raises(DivideByZero):
        _host("1 / 0")

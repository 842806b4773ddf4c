"""Flatmap-shaped loops: appends inside nested loops whose trip count depends
on the data (sugar.py:196-202 `flatmap`, run.py:947-983).  Sized by a
count-only pre-pass, written by the order-preserving scan schedule: the
appends must come out row-major / inner-loop order, bit-exact against the
reference engine's outputs (tests/golden/make_flatmap_golden.py)."""
import pytest

from helpers import F64_TOL, approx_equal, first_diff, load_golden, norm

pytestmark = pytest.mark.gpu

CASES = load_golden("flatmap.json")["cases"]


def _tree(src, inputs):
    import paper_1709_06416_b200  # noqa: F401
    from weldmill.optim import OptLevel, optimize
    from weldmill.parser import parse, parse_type_text
    from weldmill.sugar import expand
    from weldmill.typecheck import check_linearity, infer
    env = {k: parse_type_text(t) for k, t in inputs.items()}
    typed = infer(expand(parse(src)), env)
    check_linearity(typed)
    return optimize(typed, OptLevel.all())[0], env


@pytest.mark.parametrize("case", CASES, ids=[f"{c['name']}-{i}" for i, c in enumerate(CASES)])
def test_flatmap_matches_reference(case):
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig, Value
    tree, types = _tree(case["source"], case["inputs"])
    env = {k: Value(types[k], v) for k, v in case["data"].items()}
    got = norm(wg.evaluate(tree, env, EngineConfig())[0].data)
    want = norm(case["expected"]["value"])
    assert approx_equal(got, want, F64_TOL), first_diff(got, want, F64_TOL)


def test_flatmap_large_preserves_order():
    """4M rows x data-dependent fan-out (0..7 appends per row): exact
    against numpy, across many tiles (look-back offsets)."""
    import numpy as np
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig, Value
    src = "result(for(v, vecbuilder[i64], (b, i, x) => for(rng, b, (c, j, y) => if (y < x, merge(c, x * 10 + y), c))))"
    tree, types = _tree(src, {"v": "vec[i64]", "rng": "vec[i64]"})
    rng = np.random.default_rng(9)
    v = rng.integers(-2, 9, size=(4 << 20) + 3).astype(np.int64)
    r = np.arange(8, dtype=np.int64)
    got = wg.evaluate(tree, {"v": Value(types["v"], v), "rng": Value(types["rng"], r)}, EngineConfig(),
                      result="numpy")[0].data
    reps = np.clip(v, 0, 8)
    want = np.repeat(v * 10, reps) + (np.arange(reps.sum()) - np.repeat(np.cumsum(reps) - reps, reps))
    np.testing.assert_array_equal(got, want)

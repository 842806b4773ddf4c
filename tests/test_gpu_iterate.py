"""`iterate(init, update)` inside loop bodies (run.py:668-686): a per-row
device while-loop, IterationLimit after EngineConfig.max_iterations steps.
Expected values come from the reference engine
(tests/golden/make_iterate_golden.py)."""
import pytest

from helpers import F64_TOL, approx_equal, first_diff, load_golden, norm

pytestmark = pytest.mark.gpu

CASES = load_golden("iterate.json")["cases"]


@pytest.mark.parametrize("case", CASES, ids=[f"{c['name']}-{i}" for i, c in enumerate(CASES)])
def test_iterate_matches_reference(case):
    import paper_1709_06416_b200 as wg
    from test_gpu_flatmap import _tree
    from weldmill.engine import EngineConfig, Value
    from weldmill.errors import EvalError
    tree, types = _tree(case["source"], case["inputs"])
    env = {k: Value(types[k], v) for k, v in case["data"].items()}
    cfg = EngineConfig(max_iterations=case["max_iterations"])
    exp = case["expected"]
    if "error" in exp:
        with pytest.raises(EvalError) as ei:
            wg.evaluate(tree, env, cfg)
        assert type(ei.value).__name__ == exp["error"]
        return
    got = norm(wg.evaluate(tree, env, cfg)[0].data)
    want = norm(exp["value"])
    assert approx_equal(got, want, F64_TOL), first_diff(got, want, F64_TOL)

"""Dictionary probes inside loop bodies (hash joins): lookup(d, k) into a
dictmerger / groupbuilder result built by an earlier loop (run.py:702-712),
KeyNotFound on a miss.  Expected values come from the reference engine
(tests/golden/make_lookup_golden.py -> lookup.json)."""
import pytest

from helpers import F64_TOL, approx_equal, first_diff, load_golden, norm

pytestmark = pytest.mark.gpu

CASES = load_golden("lookup.json")["cases"]


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
def test_lookup_matches_reference(case):
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig, Value
    from weldmill.errors import EvalError
    tree, types = _tree(case["source"], case["inputs"])
    env = {k: Value(types[k], v) for k, v in case["data"].items()}
    exp = case["expected"]
    if "error" in exp:
        with pytest.raises(EvalError) as ei:
            wg.evaluate(tree, env, EngineConfig())
        assert type(ei.value).__name__ == exp["error"]
        return
    got = norm(wg.evaluate(tree, env, EngineConfig())[0].data)
    want = norm(exp["value"])
    assert approx_equal(got, want, F64_TOL), first_diff(got, want, F64_TOL)

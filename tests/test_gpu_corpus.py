"""GPU parity on the reference's own differential corpus.

Every program of /root/reference/pkg/tests/progen.py (308 programs, two
seeded inputs each, expected values produced by the reference engine and
committed in tests/golden/corpus.json) runs through the GPU executor at
several optimizer levels -- each level hands the executor a different loop
shape (fused, predicated, vectorized main+tail pairs, size-hinted,
unfused pipelines).  Integers/keys/order must match bit for bit; floats
within 1e-9 relative (f64).
"""
import pytest

from helpers import F64_TOL, approx_equal, first_diff, load_golden, norm

pytestmark = pytest.mark.gpu

CORPUS = load_golden("corpus.json")["programs"]
# Known gaps of the device lowering (raise DeviceUnsupported, never a CPU
# fallback).  The whole reference corpus lowers now.
UNSUPPORTED = set()
LEVELS = ["O3", "none", "no-vectorize", "no-fuse", "no-predicate"]


def _level(name):
    from weldmill.optim import OptLevel
    if name == "O3":
        return OptLevel.all()
    if name == "none":
        return OptLevel.none()
    return OptLevel.all().disable(name[3:])


@pytest.fixture(scope="module")
def front():
    import paper_1709_06416_b200  # noqa: F401
    from weldmill.parser import parse, parse_type_text
    from weldmill.sugar import expand
    from weldmill.typecheck import check_linearity, infer

    def go(src, inputs):
        env = {k: parse_type_text(t) for k, t in inputs.items()}
        typed = infer(expand(parse(src)), env)
        check_linearity(typed)
        return typed, env
    return go


@pytest.mark.parametrize("level", LEVELS)
def test_corpus_parity(front, level):
    from weldmill.engine import Value
    from weldmill.optim import optimize
    import paper_1709_06416_b200 as wg

    failures = []
    checked = 0
    for p in CORPUS:
        if p["name"] in UNSUPPORTED:
            continue
        typed, env = front(p["source"], p["inputs"])
        tree = optimize(typed, _level(level))[0]
        for case in p["cases"]:
            vals = {k: Value(env[k], v) for k, v in case["inputs"].items()}
            try:
                got = norm(wg.evaluate(tree, vals)[0].data)
            except Exception as exc:  # collect, report all at once
                failures.append(f"{p['name']}: {type(exc).__name__}: {str(exc)[:300]}")
                continue
            want = case["expected"]
            if p["is_float"]:
                ok = approx_equal(got, want, F64_TOL)
            else:
                ok = got == want
            if not ok:
                failures.append(f"{p['name']}: {first_diff(got, want, F64_TOL)}")
            checked += 1
    assert not failures, f"{len(failures)} failures ({checked} ok):\n" + "\n".join(failures[:40])


def test_unsupported_programs_fail_loudly(front):
    """No silent CPU fallback: IR outside the device lowering raises
    (here: nested appends of vectors whose lengths depend on the data)."""
    from weldmill.engine import Value
    from weldmill.optim import optimize
    import paper_1709_06416_b200 as wg

    typed, env = front("result(for(v, vecbuilder[vec[i64]], (b, i, x) => merge(b, lookup(vv, x))))",
                       {"v": "vec[i64]", "vv": "vec[vec[i64]]"})
    vals = {"v": Value(env["v"], [0, 1]), "vv": Value(env["vv"], [[1, 2], [3]])}
    with pytest.raises(wg.DeviceUnsupported):
        wg.evaluate(optimize(typed)[0], vals)


CORPUS2 = load_golden("corpus_s2.json")["programs"]


@pytest.mark.parametrize("level", ["O3", "none"])
def test_corpus_second_seed_parity(front, level):
    """The same generator with another seed (tests/golden/make_corpus2.py):
    different constants and three fresh input sets per program, expected
    values (or runtime error classes) from the reference engine."""
    from weldmill.engine import Value
    from weldmill.optim import optimize
    import paper_1709_06416_b200 as wg

    failures = []
    checked = 0
    for p in CORPUS2:
        typed, env = front(p["source"], p["inputs"])
        tree = optimize(typed, _level(level))[0]
        for case in p["cases"]:
            vals = {k: Value(env[k], v) for k, v in case["inputs"].items()}
            try:
                got = norm(wg.evaluate(tree, vals)[0].data)
            except Exception as exc:
                if "error" in case and type(exc).__name__ == case["error"]:
                    checked += 1
                    continue
                failures.append(f"{p['name']}: {type(exc).__name__}: {str(exc)[:200]}")
                continue
            if "error" in case:
                failures.append(f"{p['name']}: expected {case['error']}, got a value")
                continue
            want = case["expected"]
            ok = approx_equal(got, want, F64_TOL) if p["is_float"] else got == want
            if not ok:
                failures.append(f"{p['name']}: {first_diff(got, want, F64_TOL)}")
            checked += 1
    assert not failures, f"{len(failures)} failures ({checked} ok):\n" + "\n".join(failures[:40])


def _load_gz(name):
    import gzip
    import json
    import os
    with gzip.open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name), "rt") as f:
        return json.load(f)


CORPUS3 = _load_gz("corpus_s3.json.gz")["programs"]


@pytest.mark.parametrize("level", LEVELS)
def test_corpus_long_inputs_parity(front, level):
    """The generator with vectors of 2049-2600 elements (tests/golden/
    make_corpus3.py, seed 20261018): every loop spans several 2048-row tiles
    of the device schedules -- look-back chains across tiles, the
    warp-specialised scan's buffer hand-offs, partial last tiles, dictionaries
    and groups built from thousands of rows -- at every optimizer level."""
    from weldmill.engine import Value
    from weldmill.optim import optimize
    import paper_1709_06416_b200 as wg

    failures = []
    checked = 0
    for p in CORPUS3:
        typed, env = front(p["source"], p["inputs"])
        tree = optimize(typed, _level(level))[0]
        for case in p["cases"]:
            vals = {k: Value(env[k], v) for k, v in case["inputs"].items()}
            try:
                got = norm(wg.evaluate(tree, vals)[0].data)
            except Exception as exc:
                if "error" in case and type(exc).__name__ == case["error"]:
                    checked += 1
                    continue
                failures.append(f"{p['name']}: {type(exc).__name__}: {str(exc)[:200]}")
                continue
            if "error" in case:
                failures.append(f"{p['name']}: expected {case['error']}, got a value")
                continue
            want = case["expected"]
            ok = approx_equal(got, want, F64_TOL) if p["is_float"] else got == want
            if not ok:
                failures.append(f"{p['name']}: {first_diff(got, want, F64_TOL)}")
            checked += 1
    assert not failures, f"{len(failures)} failures ({checked} ok):\n" + "\n".join(failures[:40])

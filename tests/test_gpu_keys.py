"""Dictionary / group keys at the edges of the key encoding, on every
device variant (register cache + shared table for low cardinality,
deferred batched probes, the partitioned two-kernel mode above 1M keys,
the global strategy), compared with the reference engine (small and mid
sizes) or an exact numpy restatement (full-size partitioned runs).

One-word keys use the all-ones word as the table's empty sentinel
(weld_device.cuh wg_ht_find1): i64 -1 and i32 -1 are that word and must
still be ordinary keys.  Reference semantics: builders.py:331-392
(dictmerger), :453-493 (groupbuilder), :496-507 (order_key)."""
import random

import numpy as np
import pytest

from helpers import approx_equal, norm

import paper_1709_06416_b200  # noqa: F401

pytestmark = pytest.mark.gpu

EDGE = [-1, 0, 1, -2, 2**63 - 1, -(2**63), 2**32 - 1, -(2**32)]


def _tree(src, tys):
    from weldmill.optim import optimize
    from weldmill.parser import parse, parse_type_text
    from weldmill.sugar import expand
    from weldmill.typecheck import check_linearity, infer
    env = {k: parse_type_text(t) for k, t in tys.items()}
    t = infer(expand(parse(src)), env)
    check_linearity(t)
    return optimize(t)[0], env


def _both(src, tys, vals, cfg=None):
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig, Value, evaluate as ref
    tree, env = _tree(src, tys)
    cfg = cfg or EngineConfig()
    v = {k: Value(env[k], x) for k, x in vals.items()}
    return norm(wg.evaluate(tree, v, cfg)[0].data), norm(ref(tree, v, cfg)[0].data)


def _keys(n, distinct, seed):
    rng = random.Random(seed)
    pool = EDGE + [rng.randint(-(2**40), 2**40) for _ in range(max(0, distinct - len(EDGE)))]
    return [pool[rng.randrange(len(pool))] if rng.random() < 0.9 else EDGE[rng.randrange(len(EDGE))]
            for _ in range(n)]


@pytest.mark.parametrize("strategy", ["local", "global"])
@pytest.mark.parametrize("distinct", [8, 3000, 40000])
@pytest.mark.parametrize("n", [1000, 300_007])
def test_dictmerger_sentinel_and_extreme_keys(strategy, distinct, n):
    from weldmill.engine import EngineConfig
    keys = _keys(n, distinct, seed=n + distinct)
    for src in ("tovec(result(for(v, dictmerger[i64, i64, +], (b, i, x) => merge(b, {x, 1}))))",
                "tovec(result(for(v, dictmerger[i64, i64, max], (b, i, x) => merge(b, {x, i}))))",
                "tovec(result(for(v, dictmerger[i64, {i64, f64}, +], (b, i, x) =>"
                " merge(b, {x, {1, cast(i % 7, f64) * 0.5}}))))"):
        got, want = _both(src, {"v": "vec[i64]"}, {"v": keys}, EngineConfig(strategy=strategy))
        assert approx_equal(got, want, 1e-9), (src, len(got), len(want))


@pytest.mark.parametrize("n", [1000, 300_007])
def test_i32_and_struct_keys_with_all_ones_words(n):
    rng = random.Random(n)
    a = [rng.choice([-1, 0, 7, -(2**31), 2**31 - 1]) for _ in range(n)]
    b = [rng.choice([-1, 5, -(2**63), 2**63 - 1]) for _ in range(n)]
    got, want = _both("tovec(result(for(v, dictmerger[i32, i64, +], (b, i, x) => merge(b, {x, 1}))))",
                      {"v": "vec[i32]"}, {"v": a})
    assert got == want
    got, want = _both("tovec(result(for(zip(v, w), dictmerger[{i32, i64}, i64, +], (b, i, x) =>"
                      " merge(b, {{x.0, x.1}, 1}))))", {"v": "vec[i32]", "w": "vec[i64]"}, {"v": a, "w": b})
    assert got == want


@pytest.mark.parametrize("n", [1000, 300_007])
def test_groupbuilder_sentinel_keys_keep_row_order(n):
    keys = _keys(n, 50, seed=7 * n)
    got, want = _both("tovec(result(for(v, groupbuilder[i64, i64], (b, i, x) => merge(b, {x, i}))))",
                      {"v": "vec[i64]"}, {"v": keys})
    assert got == want


def test_lookup_of_sentinel_key_in_loop_body():
    keys = [-1, 3, -1, 9, 2**63 - 1]
    got, want = _both("d := result(for(v, dictmerger[i64, i64, +], (b, i, x) => merge(b, {x, i})));"
                      " result(for(v, vecbuilder[i64], (b, i, x) => merge(b, lookup(d, x))))",
                      {"v": "vec[i64]"}, {"v": keys})
    assert got == want


def test_partitioned_dictmerger_sentinel_key_full_size():
    """4M rows over ~2M distinct keys: after the 64K-row sketch the loop runs
    in the partitioned two-kernel mode; -1 and the extremes must survive.
    Exact numpy restatement of dictmerger[i64, i64, +] + tovec."""
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig, Value
    n = 1 << 22
    rng = np.random.default_rng(11)
    k = rng.integers(-(1 << 21), 1 << 21, size=n, dtype=np.int64) * 7919
    k[rng.integers(0, n, size=5000)] = -1
    k[rng.integers(0, n, size=100)] = np.iinfo(np.int64).max
    k[rng.integers(0, n, size=100)] = np.iinfo(np.int64).min
    vals = rng.integers(-1000, 1000, size=n, dtype=np.int64)
    tree, env = _tree("tovec(result(for(zip(v, w), dictmerger[i64, i64, +], (b, i, x) => merge(b, {x.0, x.1}))))",
                      {"v": "vec[i64]", "w": "vec[i64]"})
    out = wg.evaluate(tree, {"v": Value(env["v"], k), "w": Value(env["w"], vals)},
                      EngineConfig(memory_limit=1 << 40), result="numpy")[0].data
    uk, inv = np.unique(k, return_inverse=True)
    sums = np.zeros(len(uk), dtype=np.int64)
    np.add.at(sums, inv, vals)
    gk, gv = out
    assert np.array_equal(np.asarray(gk), uk)
    assert np.array_equal(np.asarray(gv), sums)


FLOAT_CASES = [
    [0.0, -0.0, 1.5, -0.0, 0.0],
    [-0.0, 0.0, 1.5, 0.0],
    [1.0, 2.0, -0.0, -0.0],
    [2.5, float("inf"), -float("inf"), -0.0],
]


@pytest.mark.parametrize("data", FLOAT_CASES, ids=range(len(FLOAT_CASES)))
@pytest.mark.parametrize("kind", ["f64", "f32"])
def test_signed_zero_keys_keep_the_first_inserted_key(data, kind):
    """-0.0 == 0.0 is one key; its sign is that of the first row merging it
    (Python dict keeps the first-inserted key object)."""
    import math
    for src in (f"tovec(result(for(v, dictmerger[{kind}, i64, +], (b, i, x) => merge(b, {{x, i}}))))",
                f"tovec(result(for(v, groupbuilder[{kind}, i64], (b, i, x) => merge(b, {{x, i}}))))"):
        got, want = _both(src, {"v": f"vec[{kind}]"}, {"v": data})
        assert got == want, (src, got, want)
        assert [math.copysign(1.0, k) for k, _ in got] == [math.copysign(1.0, k) for k, _ in want]


@pytest.mark.parametrize("n", [5000, 300_007])
def test_signed_zero_keys_at_size(n):
    import math
    rng = random.Random(n)
    for first in (0.0, -0.0):
        data = [first] + [rng.choice([0.0, -0.0, 1.0, 2.0, -3.5]) for _ in range(n - 1)]
        for src in ("tovec(result(for(v, dictmerger[f64, i64, +], (b, i, x) => merge(b, {x, 1}))))",
                    "tovec(result(for(v, groupbuilder[f64, i64], (b, i, x) => merge(b, {x, i}))))"):
            got, want = _both(src, {"v": "vec[f64]"}, {"v": data})
            assert got == want
            assert [math.copysign(1.0, k) for k, _ in got] == [math.copysign(1.0, k) for k, _ in want]


def test_nan_keys_collapse_like_the_reference():
    """NaN keys produced by the program (0.0 / 0.0) or passed in as one float
    object are a single dictionary key in the reference; so on the device."""
    nan = float("nan")
    for src in ("tovec(result(for(v, dictmerger[f64, i64, +], (b, i, x) => merge(b, {x / 0.0, 1}))))",
                "tovec(result(for(v, groupbuilder[f64, i64], (b, i, x) => merge(b, {x, i}))))"):
        got, want = _both(src, {"v": "vec[f64]"}, {"v": [nan, 1.0, 0.0, nan, -0.0, 2.0, nan]})
        assert repr(got) == repr(want), (got, want)

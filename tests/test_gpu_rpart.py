"""Range-partitioned dictmerger (codegen.dict_rpart_source): the second
evaluate of a high-cardinality dictmerger loop partitions merges by the top
bits of the key's order key, aggregates each partition in shared memory and
sorts it locally.  Results must equal the reference semantics exactly
(DictMergerState.result + order_key, builders.py:380-392, 496-507): integer
sums bit-exact, keys strictly increasing in signed order, the sentinel-valued
key (-1 == all ones) and the i64 extremes included; skewed keys fall back to
the hash-table path with the same result."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _prog(src, types, opt=True):
    from paper_1709_06416_b200 import _ref  # noqa: F401
    from weldmill.optim import OptLevel, optimize
    from weldmill.parser import parse, parse_type_text
    from weldmill.sugar import expand
    from weldmill.typecheck import check_linearity, infer
    env = {k: parse_type_text(t) for k, t in types.items()}
    typed = infer(expand(parse(src)), env)
    check_linearity(typed)
    return optimize(typed, None if opt else OptLevel.none())[0]


DICT_I64 = "tovec(result(for({k, v}, dictmerger[i64, i64, +], (b, i, x) => merge(b, {x.0, x.1}))))"
DICT_MIN = "tovec(result(for({k, v}, dictmerger[i64, f64, min], (b, i, x) => merge(b, {x.0, x.1}))))"


def _want_sum(k, v):
    u, inv = np.unique(k, return_inverse=True)
    s = np.zeros(u.size, dtype=np.int64)
    np.add.at(s, inv, v)
    return u, s


def _eval(tree, k, v, vt="vec[i64]"):
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig, Value
    from weldmill.parser import parse_type_text
    env = {"k": Value(parse_type_text("vec[i64]"), k), "v": Value(parse_type_text(vt), v)}
    out = wg.evaluate(tree, env, EngineConfig(memory_limit=1 << 45), {}, result="numpy")[0].data
    return out


@pytest.fixture
def small_rpart(monkeypatch):
    """Let a few thousand distinct keys qualify for the partitioned path."""
    from paper_1709_06416_b200 import executor
    monkeypatch.setattr(executor, "PART_MIN_KEYS", 100)
    monkeypatch.setattr(executor, "RPART", True)
    return executor


def test_rpart_matches_numpy_with_sentinel_and_extremes(small_rpart):
    rng = np.random.default_rng(7)
    n = 300_000
    k = rng.integers(-(1 << 62), 1 << 62, size=20_000, dtype=np.int64)[rng.integers(0, 20_000, size=n)]
    k[:50] = -1                                  # the all-ones word (table sentinel)
    k[50:60] = np.iinfo(np.int64).min
    k[60:70] = np.iinfo(np.int64).max
    k[70:80] = 0
    v = rng.integers(-1000, 1000, size=n, dtype=np.int64)
    tree = _prog(DICT_I64, {"k": "vec[i64]", "v": "vec[i64]"})
    first = _eval(tree, k, v)                    # hash-table path; records the hints
    runs = small_rpart.RPART_RUNS
    second = _eval(tree, k, v)                   # range-partitioned path
    assert small_rpart.RPART_RUNS == runs + 1
    u, s = _want_sum(k, v)
    for got in (first, second):
        np.testing.assert_array_equal(got[0], u)
        np.testing.assert_array_equal(got[1], s)


def test_rpart_skew_falls_back(small_rpart):
    """Keys clustered far below the recorded range all clamp into partition
    0, overflow its shared-memory table, and the loop re-runs through the
    hash-table path with the same result."""
    rng = np.random.default_rng(11)
    n = 200_000
    k = rng.integers(-(1 << 62), 1 << 62, size=30_000, dtype=np.int64)[rng.integers(0, 30_000, size=n)]
    v = rng.integers(-5, 5, size=n, dtype=np.int64)
    tree = _prog(DICT_I64, {"k": "vec[i64]", "v": "vec[i64]"})
    _eval(tree, k, v)
    k2 = np.arange(n, dtype=np.int64) % 25_000 - (1 << 62) - 100_000   # all below the hinted minimum
    got = _eval(tree, k2, v)
    u, s = _want_sum(k2, v)
    np.testing.assert_array_equal(got[0], u)
    np.testing.assert_array_equal(got[1], s)
    assert small_rpart._RPART_BAD


def test_rpart_float_min_fold(small_rpart):
    rng = np.random.default_rng(3)
    n = 250_000
    k = rng.integers(0, 40_000, size=n, dtype=np.int64) * 7919 - 123_456
    v = rng.standard_normal(n)
    tree = _prog(DICT_MIN, {"k": "vec[i64]", "v": "vec[f64]"})
    _eval(tree, k, v, "vec[f64]")
    runs = small_rpart.RPART_RUNS
    got = _eval(tree, k, v, "vec[f64]")
    assert small_rpart.RPART_RUNS == runs + 1
    order = np.lexsort((v, k))
    ks, vs = k[order], v[order]
    first = np.r_[True, ks[1:] != ks[:-1]]
    np.testing.assert_array_equal(got[0], ks[first])
    np.testing.assert_array_equal(got[1], vs[first])      # min is exact


def test_rpart_full_config_twice_matches_oracle(monkeypatch):
    """The C4a program itself at 4M rows (~3.3M distinct keys > the 1M
    threshold): second run is range-partitioned, equal to the oracle."""
    from oracle import weld_oracle
    from paper_1709_06416_b200 import executor as _ex
    monkeypatch.setattr(_ex, "RPART", True)
    from paper_1709_06416_b200 import executor, workloads as W
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig, Value
    wl = W.WORKLOADS["dict"]
    tree = W.compile_program(wl)
    types = W.input_types(wl)
    n = 4 << 20
    cols = W.host_columns(wl, n)
    env = {c: Value(types[c], a) for c, a in cols.items()}
    runs = executor.RPART_RUNS
    for _ in range(2):
        got = wg.evaluate(tree, env, EngineConfig(memory_limit=1 << 45), {}, result="numpy")[0].data
    assert executor.RPART_RUNS == runs + 1
    ks, vs = weld_oracle.dict_sum(cols)
    np.testing.assert_array_equal(got[0], ks)
    np.testing.assert_array_equal(got[1], vs)


def test_rpart_result_reused_by_another_loop(small_rpart):
    """A partitioned result that later receives more merges (builder passed
    to a second loop) is replayed into a hash table first."""
    src = ("d := for({k, v}, dictmerger[i64, i64, +], (b, i, x) => merge(b, {x.0, x.1}));"
           " tovec(result(for({k, v}, d, (b, i, x) => merge(b, {x.0, 1}))))")
    rng = np.random.default_rng(5)
    n = 100_000
    k = rng.integers(-(1 << 40), 1 << 40, size=10_000, dtype=np.int64)[rng.integers(0, 10_000, size=n)]
    v = rng.integers(-9, 9, size=n, dtype=np.int64)
    tree = _prog(src, {"k": "vec[i64]", "v": "vec[i64]"}, opt=False)
    for _ in range(3):
        got = _eval(tree, k, v)
    u, s = _want_sum(k, v + 1)
    np.testing.assert_array_equal(got[0], u)
    np.testing.assert_array_equal(got[1], s)

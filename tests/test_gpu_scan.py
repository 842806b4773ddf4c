"""Order-preserving appends on the warp-specialised scan schedule
(codegen.ws_lines): compute warps stage each tile in one of two
shared-memory buffers and a store warp resolves the decoupled look-back.

Edge cases of the schedule -- empty input, one row, partial tiles around the
2048-row tile size, nothing / everything kept, several appenders in one loop,
struct elements, a non-zero idx0 through zipped iteration windows -- against
numpy, and vecbuilder_reallocations (the chunk-start positions the buffers
carry, builders.py:256-272) against the live reference engine at several
grain sizes (grain < 32 takes the non-specialised schedule)."""
import numpy as np
import pytest

import paper_1709_06416_b200  # noqa: F401

pytestmark = pytest.mark.gpu

TILE = 2048
SIZES = [0, 1, 31, TILE - 1, TILE, TILE + 1, 3 * TILE + 17, 37 * TILE + 5, 1_000_003]


def _front(src, types):
    from weldmill.parser import parse, parse_type_text
    from weldmill.sugar import expand
    from weldmill.typecheck import check_linearity, infer
    t = infer(expand(parse(src)), {k: parse_type_text(v) for k, v in types.items()})
    check_linearity(t)
    return t


def _dev(ty, arr):
    from weldmill.engine import Value
    from weldmill.parser import parse_type_text
    from paper_1709_06416_b200.columns import to_device
    t = parse_type_text(ty)
    return Value(t, to_device(t, arr))


def _np(v):
    from paper_1709_06416_b200.columns import to_numpy
    return to_numpy(v)


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("mode", ["half", "none", "all", "alternate"])
def test_filter_edges(n, mode):
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig
    rng = np.random.default_rng(n + 7)
    v = rng.integers(-1000, 1000, n).astype(np.int64)
    if mode == "none":
        v = -np.abs(v) - 1
    elif mode == "all":
        v = np.abs(v) + 1
    elif mode == "alternate":
        v = np.where(np.arange(n) % 2 == 0, 5, -5).astype(np.int64)
    tree = _front("filter(v, (x) => x > 0)", {"v": "vec[i64]"})
    val, _ = wg.evaluate(tree, {"v": _dev("vec[i64]", v)}, EngineConfig(), result="device")
    got = _np(val.data)
    assert got.dtype == np.int64 and np.array_equal(got, v[v > 0])


@pytest.mark.parametrize("n", [TILE + 3, 5 * TILE - 1, 300_007])
def test_two_appenders_struct_elements_and_index(n):
    """Two order-preserving appenders fed by different predicates, one of a
    struct element carrying the loop index (global through idx0)."""
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig
    rng = np.random.default_rng(n)
    a = rng.standard_normal(n)
    b = rng.integers(0, 100, n).astype(np.int32)
    src = ("result(for({a, b}, {vecbuilder[{f64, i64}], vecbuilder[i32]}, (bs, i, x) => "
           "{if (x.0 > 0.5, merge(bs.0, {x.0 * 2.0, i}), bs.0), if (x.1 % 7 == 3, merge(bs.1, x.1), bs.1)}))")
    tree = _front(src, {"a": "vec[f64]", "b": "vec[i32]"})
    val, _ = wg.evaluate(tree, {"a": _dev("vec[f64]", a), "b": _dev("vec[i32]", b)}, EngineConfig(), result="device")
    s0, s1 = val.data
    c0 = _np(s0)
    keep = a > 0.5
    assert np.array_equal(c0[0], a[keep] * 2.0)
    assert np.array_equal(c0[1], np.nonzero(keep)[0])
    assert np.array_equal(_np(s1), b[b % 7 == 3])


@pytest.mark.parametrize("grain", [1024, 64, 7])
@pytest.mark.parametrize("n", [5, TILE + 1, 20_011])
def test_reallocation_stats_match_reference(grain, n):
    """vecbuilder_reallocations of an unhinted filter: per (step, chunk)
    segments doubling from 16 (builders.py:256-272), from the chunk-start
    positions the store warp writes."""
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig, Value, evaluate as ref_evaluate
    from weldmill.parser import parse_type_text
    rng = np.random.default_rng(grain * 31 + n)
    v = rng.integers(-50, 50, n).astype(np.int64)
    tree = _front("result(for(v, vecbuilder[i64], (b, i, x) => if (x > 10, merge(b, x), b)))", {"v": "vec[i64]"})
    cfg = EngineConfig(grain_size=grain)
    want_v, want_s = ref_evaluate(tree, {"v": Value(parse_type_text("vec[i64]"), v.tolist())}, cfg)
    got_v, got_s = wg.evaluate(tree, {"v": _dev("vec[i64]", v)}, cfg)
    assert got_v.data == want_v.data
    assert got_s.vecbuilder_reallocations == want_s.vecbuilder_reallocations
    assert got_s.vector_traversals == want_s.vector_traversals

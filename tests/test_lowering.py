"""Every loop of the reference's differential corpus, at several optimizer
levels, lowers to CUDA and (a sample of) compiles with NVRTC for sm_100a --
no GPU needed.  The five benchmark kernels always compile."""
import os

import pytest

from helpers import load_golden

CORPUS = load_golden("corpus.json")["programs"]
UNSUPPORTED = set()


def _tree(src, inputs, level):
    import paper_1709_06416_b200  # noqa: F401
    from weldmill.optim import OptLevel, optimize
    from weldmill.parser import parse, parse_type_text
    from weldmill.sugar import expand
    from weldmill.typecheck import check_linearity, infer
    env = {k: parse_type_text(t) for k, t in inputs.items()}
    typed = infer(expand(parse(src)), env)
    check_linearity(typed)
    lv = OptLevel.all() if level == "O3" else (OptLevel.none() if level == "none" else
                                               OptLevel.all().disable(level))
    return optimize(typed, lv)[0]


@pytest.mark.parametrize("level", ["O3", "none", "vectorize", "fuse"])
def test_corpus_lowers(level):
    from paper_1709_06416_b200 import codegen
    n = 0
    for p in CORPUS:
        if p["name"] in UNSUPPORTED:
            continue
        plans = codegen.static_plans(_tree(p["source"], p["inputs"], level))
        for pl in plans:
            assert "extern \"C\" __global__" in pl.source
        n += len(plans)
    assert n > 250


def test_unsupported_shapes_raise():
    """Nested appends of vectors with data-dependent lengths are not lowered
    (they raise DeviceUnsupported -- never a CPU fallback)."""
    from paper_1709_06416_b200 import codegen
    from paper_1709_06416_b200.irtypes import DeviceUnsupported
    src = "result(for(v, vecbuilder[vec[i64]], (b, i, x) => merge(b, lookup(vv, x))))"
    with pytest.raises(DeviceUnsupported):
        codegen.static_plans(_tree(src, {"v": "vec[i64]", "vv": "vec[vec[i64]]"}, "O3"))


def test_benchmark_kernels_compile_for_sm100a():
    from paper_1709_06416_b200 import codegen, runtime, workloads as W
    for wl in W.WORKLOADS.values():
        for smem, low, part in ((True, False, False), (True, True, False), (False, False, False),
                                (False, False, True)):
            for plan in codegen.static_plans(W.compile_program(wl), externs=wl.externs, smem=smem, lowcard=low,
                                             part=part):
                assert runtime.compile_check(plan.source) > 0


def test_partitioned_dict_aggregation_kernel_compiles():
    from paper_1709_06416_b200 import codegen, runtime
    from weldmill.types import DictMerger, Scalar, Struct
    for key, val, op in (("i64", Scalar("i64"), "+"), ("i32", Struct((Scalar("f64"), Scalar("i64"))), "+"),
                         ("i64", Scalar("f64"), "min")):
        kind = DictMerger(Scalar(key), val, op)
        sw = 1 + (len(val.fields) if isinstance(val, Struct) else 1)
        src, smem = codegen.dict_agg_source(kind, sw, 0, 8)
        assert runtime.compile_check(src) > 0


def test_corpus_sample_compiles():
    from paper_1709_06416_b200 import codegen, runtime
    seen = set()
    step = int(os.environ.get("WELDGPU_TEST_COMPILE_STRIDE", "7"))
    for p in CORPUS[::step]:
        if p["name"] in UNSUPPORTED:
            continue
        for pl in codegen.static_plans(_tree(p["source"], p["inputs"], "O3")):
            if pl.source in seen:
                continue
            seen.add(pl.source)
            assert runtime.compile_check(pl.source) > 0, p["name"]
    assert len(seen) > 20


def test_generated_literals_are_exact():
    from paper_1709_06416_b200.codegen import c_literal
    assert c_literal("f64", 0.1) == "__longlong_as_double(0x3fb999999999999aLL)"
    assert c_literal("i64", -(2**63)) == "((i64)0x8000000000000000ULL)"
    assert c_literal("i32", -1) == "((i32)0xffffffffU)"
    assert c_literal("f64", float("inf")).endswith("0x7ff0000000000000LL)")


def test_dictionary_probes_lower_and_compile():
    """lookup(d, k) in a loop body lowers to a binary search over the
    dictionary's order-key-sorted key columns and compiles for sm_100a."""
    from helpers import load_golden
    from paper_1709_06416_b200 import codegen, runtime
    seen = set()
    for c in load_golden("lookup.json")["cases"]:
        if c["name"] in seen:
            continue
        seen.add(c["name"])
        plans = codegen.static_plans(_tree(c["source"], c["inputs"], "O3"))
        probe = [p for p in plans if "WG_ERR_KEY_NOT_FOUND" in p.source]
        assert probe, c["name"]
        for p in probe:
            assert runtime.compile_check(p.source) > 0


def test_flatmap_loops_lower_and_compile():
    """Appends inside data-dependent nested loops lower to the scan schedule
    (unbounded appends, unstaged stores) plus a count-only pre-pass kernel;
    both compile for sm_100a."""
    from helpers import load_golden
    from paper_1709_06416_b200 import codegen, runtime
    seen = set()
    for c in load_golden("flatmap.json")["cases"]:
        if c["name"] in seen:
            continue
        seen.add(c["name"])
        t = _tree(c["source"], c["inputs"], "O3")
        plans = codegen.static_plans(t)
        scan = [p for p in plans if p.schedule == "scan" and any(b.extra.get("unbounded") for b in p.builders)]
        assert scan, c["name"]
        counts = codegen.static_plans(t, count_only=True)
        assert counts and all(p.schedule == "count" for p in counts)
        for p in scan + counts:
            assert runtime.compile_check(p.source) > 0


def test_iterate_in_loop_bodies_lowers_and_compiles():
    from helpers import load_golden
    from paper_1709_06416_b200 import codegen, runtime
    seen = set()
    for c in load_golden("iterate.json")["cases"]:
        if c["name"] in seen:
            continue
        seen.add(c["name"])
        plans = codegen.static_plans(_tree(c["source"], c["inputs"], "O3"))
        body = [p for p in plans if "WG_ERR_ITER_LIMIT" in p.source]
        assert body, c["name"]
        for p in body:
            assert runtime.compile_check(p.source) > 0


def test_stats_instrumented_kernels_compile():
    """count_evals kernels (a warp-aggregated counter per body node) and the
    chunk-offset records of unhinted scan appenders (reallocation
    accounting) lower and compile for sm_100a: corpus sample, flatmap and
    iterate bodies."""
    from helpers import load_golden
    from paper_1709_06416_b200 import codegen, runtime
    srcs = [(p["source"], p["inputs"]) for p in CORPUS[::11]]
    srcs += [(c["source"], c["inputs"]) for c in load_golden("flatmap.json")["cases"][::40]]
    srcs += [(c["source"], c["inputs"]) for c in load_golden("iterate.json")["cases"][::40]]
    seen = set()
    n_count = n_seg = 0
    for src, inputs in srcs:
        for pl in codegen.static_plans(_tree(src, inputs, "O3"), counting=True, segstats=True):
            if pl.source in seen:
                continue
            seen.add(pl.source)
            n_count += "wg_count(p.cnt" in pl.source
            n_seg += bool(pl.seg_bids)
            assert len(pl.count_nodes) > 0
            assert runtime.compile_check(pl.source) > 0, src
    assert n_count > 10 and n_seg >= 3, (n_count, n_seg)


def _typed_with_externs(src, inputs, names):
    import paper_1709_06416_b200  # noqa: F401
    from weldmill.optim import OptLevel, optimize
    from weldmill.parser import parse, parse_type_text
    from weldmill.sugar import expand
    from weldmill.typecheck import check_linearity, infer
    from weldmill.types import F64, Function, Scalar
    env = {k: parse_type_text(t) for k, t in inputs.items()}
    for nm in names:
        env[nm] = Function((Scalar(F64),), Scalar(F64))
    typed = infer(expand(parse(src)), env)
    check_linearity(typed)
    return optimize(typed, OptLevel.none())[0]


def test_staged_filter_with_math_tables_fits_static_shared_memory():
    """Regression (advisor, round 1): an order-preserving filter over a
    13-byte row whose predicate calls erf and log used to stage 40 KB of
    appends next to 11 KB of math tables (> 48 KB static shared memory):
    ptxas rejected it.  The staging budget now subtracts the tables."""
    from paper_1709_06416_b200 import codegen, runtime
    src = "filter(v, (x) => call(erf, x.0) + call(log, x.0) > 0.0)"
    tree = _typed_with_externs(src, {"v": "vec[{f64, bool, bool}]"}, ("erf", "log"))
    plans = codegen.static_plans(tree, externs=("erf", "log"))
    assert plans and any("wg_erf_tab_init" in p.source for p in plans)
    for p in plans:
        assert runtime.compile_check(p.source) > 0


def test_extern_bound_to_custom_callable_is_not_replaced():
    """The reference calls whatever callable is registered (run.py:836-844);
    the device lowers only the math module's functions and refuses others
    instead of silently substituting libm."""
    import math
    from paper_1709_06416_b200 import codegen
    from paper_1709_06416_b200.irtypes import DeviceUnsupported
    tree = _typed_with_externs("map(v, (x) => call(exp, x))", {"v": "vec[f64]"}, ("exp",))
    from weldmill.expr import For, walk
    loop = next(n for n in walk(tree) if isinstance(n, For))
    from paper_1709_06416_b200.codegen import IterSpec, BSpec
    from paper_1709_06416_b200.irtypes import leaves
    iters = [IterSpec(elem=it.data.ty.elem, simd=it.simd, strided=it.start is not None,
                      kinds=leaves(it.data.ty.elem)) for it in loop.iters]
    bs = BSpec(bid=0, kind=loop.builders.ty.kind)
    codegen.generate(loop, iters, bs, {}, {"exp": math.exp}, "local")
    with pytest.raises(DeviceUnsupported):
        codegen.generate(loop, iters, BSpec(bid=0, kind=loop.builders.ty.kind), {}, {"exp": lambda x: x + 1}, "local")


def test_extern_error_text_matches_the_reference_form():
    from paper_1709_06416_b200 import codegen
    i = codegen.EXTERN_IDS["log"]
    assert codegen.extern_error_text(2 * i) == "extern 'log' failed: math domain error"
    i = codegen.EXTERN_IDS["exp"]
    assert codegen.extern_error_text(2 * i + 1) == "extern 'exp' failed: math range error"


@pytest.mark.parametrize("src,types,want_ws", [
    ("filter(v, (x) => x > 0)", {"v": "vec[i64]"}, True),
    ("result(for({a, b}, {vecbuilder[{f64, i64}], vecbuilder[i32]}, (bs, i, x) => "
     "{if (x.0 > 0.5, merge(bs.0, {x.0, i}), bs.0), if (x.1 % 7 == 3, merge(bs.1, x.1), bs.1)}))",
     {"a": "vec[f64]", "b": "vec[i32]"}, True),
    # an appender next to a merger: the non-specialised scan schedule
    ("result(for(v, {vecbuilder[i64], merger[i64, +]}, (bs, i, x) => "
     "{if (x > 0, merge(bs.0, x), bs.0), merge(bs.1, x)}))", {"v": "vec[i64]"}, False),
    # data-dependent fan-out (flatmap): unbounded appends stay on the count pre-pass path
    ("result(for(v, vecbuilder[i64], (b, i, x) => for(rng, b, (c, j, y) => if (y < x, merge(c, x * 10 + y), c))))",
     {"v": "vec[i64]", "rng": "vec[i64]"}, False),
])
def test_warp_specialised_scan_selection(src, types, want_ws):
    """The warp-specialised scan schedule (SCAN_WS) is chosen
    exactly for loops whose builders are all bounded order-preserving
    appenders; its kernels carry the store warp and compile for sm_100a."""
    from paper_1709_06416_b200 import codegen, runtime
    plans = codegen.static_plans(_tree(src, types, "none"))
    scans = [pl for pl in plans if pl.schedule == "scan"]
    assert scans
    ws = [pl for pl in scans if pl.threads == pl.block + 32]
    assert bool(ws) == want_ws
    for pl in ws:
        assert "wg_lookback_resolve" in pl.source and "wg_mbar_wait(&wg_full" in pl.source
        runtime.compile_check(pl.source)

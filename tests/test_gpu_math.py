"""exp / log / erf externs on the device (weld_device.cuh's Estrin-form
versions) against the host libm the reference calls (run.py:832-846 resolves
`call(name, ...)` to a Python callable; here math.exp / math.log / math.erf,
i.e. glibc) and, on a sample, against mpmath at 200 bits.

Bar: special values exact; at most 2 ulp from the correctly rounded result
(libdevice's own bound for these functions), which sits far inside the
1e-9 parity tolerance of the benchmark programs."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _eval(fn, xs):
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig, Value
    from weldmill.optim import OptLevel, optimize
    from weldmill.parser import parse, parse_type_text
    from weldmill.sugar import expand
    from weldmill.typecheck import infer
    from weldmill.types import F64, Function, Scalar
    ty = parse_type_text("vec[f64]")
    env = {"v": ty, fn: Function((Scalar(F64),), Scalar(F64))}
    tree = optimize(infer(expand(parse(f"map(v, (x) => call({fn}, x))")), env), OptLevel.none())[0]
    val, _ = wg.evaluate(tree, {"v": Value(ty, np.ascontiguousarray(xs, dtype=np.float64))},
                         EngineConfig(memory_limit=1 << 40), {fn: getattr(math, fn)}, result="numpy")
    return np.asarray(val.data)


def _ulps(a, b):
    ia = a.view(np.int64)
    ib = b.view(np.int64)
    ia = np.where(ia < 0, np.int64(-0x8000000000000000) - ia, ia)
    ib = np.where(ib < 0, np.int64(-0x8000000000000000) - ib, ib)
    return np.abs(ia - ib)


def _libm(fn, x):
    """glibc through Python's math; NaN where math raises (masked by _raises)."""
    f = getattr(math, fn)
    out = np.empty_like(x)
    for i, v in enumerate(x.tolist()):
        try:
            out[i] = f(v)
        except (ValueError, OverflowError):
            out[i] = math.nan
    return out


def _raises(fn, x):
    f = getattr(math, fn)
    bad = np.zeros(x.shape, dtype=bool)
    for i, v in enumerate(x.tolist()):
        try:
            f(v)
        except (ValueError, OverflowError):
            bad[i] = True
    return bad


RANGES = {
    "exp": [(-745.2, 709.78), (-1.0, 1.0), (-20.0, 20.0), (700.0, 709.78), (-745.1, -700.0)],
    "log": [(1e-310, 1e-300), (1e-300, 1e300), (0.5, 2.0), (0.999, 1.001), (1e300, 1.7e308)],
    "erf": [(-7.0, 7.0), (-1e-3, 1e-3), (0.5, 6.0), (-6.0, -0.5), (5.8, 6.0)],
}
SPECIAL = [0.0, -0.0, 1.0, -1.0, math.inf, -math.inf, math.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
           1.7976931348623157e308, -1.7976931348623157e308, 709.782712893384, 709.79, -745.1332191019411,
           -745.14, 708.39, 708.4, -708.4, 0.5, 2.0, math.sqrt(2.0), math.sqrt(0.5), 5.9215871957945, 5.93, 1e-20]


@pytest.mark.parametrize("fn", ["exp", "log", "erf"])
def test_special_values_match_libm(fn):
    x = np.array(SPECIAL, dtype=np.float64)
    bad = _raises(fn, x)
    x = x[~bad]
    got = _eval(fn, x)
    want = _libm(fn, x)
    both_nan = np.isnan(got) & np.isnan(want)
    ok = both_nan | (_ulps(got, want) <= 2)
    assert ok.all(), list(zip(x[~ok].tolist(), got[~ok].tolist(), want[~ok].tolist()))
    # signs of zeros and infinities exactly
    fin = ~np.isnan(want)
    assert (np.signbit(got[fin]) == np.signbit(want[fin])).all()
    assert (np.isinf(got) == np.isinf(want)).all()


@pytest.mark.parametrize("fn", ["exp", "log", "sqrt"])
def test_domain_and_range_errors_match_reference(fn):
    """Where Python's math raises (log(0), log(-1), sqrt(-1): ValueError;
    exp(1000): OverflowError), the reference turns the exception into
    EvalError(f"extern {name!r} failed: {exc}") (run.py:841-844); the device
    raises the same class with the same message."""
    from weldmill.engine import EngineConfig, Value, evaluate as ref_evaluate
    from weldmill.errors import EvalError
    from weldmill.optim import OptLevel, optimize
    from weldmill.parser import parse, parse_type_text
    from weldmill.sugar import expand
    from weldmill.typecheck import infer
    from weldmill.types import F64, Function, Scalar
    ty = parse_type_text("vec[f64]")
    env = {"v": ty, fn: Function((Scalar(F64),), Scalar(F64))}
    tree = optimize(infer(expand(parse(f"map(v, (x) => call({fn}, x))")), env), OptLevel.none())[0]
    cases = {"exp": [1000.0, 709.79], "log": [0.0, -0.0, -1.0, -math.inf], "sqrt": [-1.0, -1e-300, -math.inf]}[fn]
    for v in cases:
        xs = [1.0, 2.0, v, 3.0]
        with pytest.raises(EvalError) as want:
            ref_evaluate(tree, {"v": Value(ty, xs)}, EngineConfig(), {fn: getattr(math, fn)})
        with pytest.raises(EvalError) as got:
            _eval(fn, np.array(xs))
        assert type(got.value) is type(want.value)
        assert str(got.value) == str(want.value), (v, str(got.value), str(want.value))


@pytest.mark.parametrize("fn", ["exp", "log", "erf"])
def test_random_sweep_within_2ulp_of_libm(fn):
    rng = np.random.default_rng(7)
    parts = []
    for lo, hi in RANGES[fn]:
        if fn == "log" and lo > 0 and hi / lo > 1e3:
            parts.append(np.exp(rng.uniform(math.log(lo), math.log(hi), 40000)))
        else:
            parts.append(rng.uniform(lo, hi, 40000))
    x = np.concatenate(parts)
    x = x[~_raises(fn, x)]
    got = _eval(fn, x)
    want = _libm(fn, x)
    u = _ulps(got, want)
    assert u.max() <= 2, (x[u.argmax()], got[u.argmax()], want[u.argmax()], int(u.max()))
    # and on average essentially correctly rounded
    assert (u == 0).mean() > 0.85


@pytest.mark.parametrize("fn", ["exp", "log", "erf"])
def test_sample_against_mpmath(fn):
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 200
    rng = np.random.default_rng(11)
    lo, hi = RANGES[fn][0]
    x = rng.uniform(lo, hi, 3000) if fn != "log" else np.exp(rng.uniform(-700, 700, 3000))
    got = _eval(fn, x)
    f = getattr(mpmath, fn)
    want = np.array([float(f(mpmath.mpf(v))) for v in x.tolist()])
    assert _ulps(got, want).max() <= 2


def _eval_prog(prog, xs, fns, extra=None):
    import paper_1709_06416_b200 as wg
    from weldmill.engine import EngineConfig, Value
    from weldmill.optim import OptLevel, optimize
    from weldmill.parser import parse, parse_type_text
    from weldmill.sugar import expand
    from weldmill.typecheck import infer
    from weldmill.types import F64, Function, Scalar
    ty = parse_type_text("vec[f64]")
    env = {"v": ty}
    vals = {"v": Value(ty, np.ascontiguousarray(xs, dtype=np.float64))}
    for name, arr in (extra or {}).items():
        env[name] = ty
        vals[name] = Value(ty, np.ascontiguousarray(arr, dtype=np.float64))
    env.update({f: Function((Scalar(F64),), Scalar(F64)) for f in fns})
    tree = optimize(infer(expand(parse(prog)), env), OptLevel.none())[0]
    val, _ = wg.evaluate(tree, vals, EngineConfig(memory_limit=1 << 40), {f: getattr(math, f) for f in fns},
                         result="numpy")
    return val.data


def test_tables_in_scan_and_count_kernels():
    """The table prologue is emitted in every kernel shape a body can land
    in: the order-preserving scan schedule (filter on erf) and the count-only
    pre-pass of a data-dependent flatmap (append count from log)."""
    rng = np.random.default_rng(3)
    x = rng.uniform(0.05, 3.0, 300_000)
    e = np.array([math.erf(t) for t in x.tolist()])
    x = x[np.abs(e - 0.5) > 1e-9]                     # no ties at the threshold
    got = np.asarray(_eval_prog("filter(v, (x) => call(erf, x) > 0.5)", x, ["erf"]))
    want = x[np.array([math.erf(t) for t in x.tolist()]) > 0.5]
    np.testing.assert_array_equal(got, want)
    # flatmap: row x appends x once per y in {0..5} with y < log(x) + 3
    L = np.array([math.log(t) for t in x.tolist()]) + 3.0
    xs = x[np.abs(L - np.round(L)) > 1e-9]            # no ties at integer boundaries
    prog = ("result(for(v, vecbuilder[f64], (b, i, x) => "
            "for(r, b, (c, j, y) => if (y < call(log, x) + 3.0, merge(c, x), c))))")
    got = np.asarray(_eval_prog(prog, xs, ["log"], {"r": np.arange(6.0)}))
    Ls = np.array([math.log(t) for t in xs.tolist()]) + 3.0
    reps = (np.arange(6.0)[None, :] < Ls[:, None]).sum(axis=1)
    np.testing.assert_array_equal(got, np.repeat(xs, reps))

"""Every BASELINE.json config at its full size, element-wise against the
oracle (the reference's acceptance style, /root/reference/pkg/tests/
test_acceptance.py:226-269, at the benchmark's sizes):

  C1 Q6 merger            1M and 600M rows   f64 within 1e-9 (chunked oracle)
  C2 Black-Scholes        64M options        every call/put within 1e-9*max(1,|a|,|b|)
  C3 Q1 dictmerger        60M rows           keys + i64 counts exact, f64 sums 1e-9
  C4a dictmerger          200M rows, 10M keys  keys and i64 sums bit-exact
  C4b groupbuilder        200M rows, 10M keys  keys, offsets and every value in
                                               per-key input order bit-exact
  C5 vecmerger            1B rows, 1M bins   every bin within 1e-9 (chunked oracle)
  filter / map appenders  500M rows          bit-exact, order preserved

Inputs are generated on the device (workloads.device_columns); the oracle
regenerates the same rows on the host with the numpy generator (identical
bits, tests/test_oracle.py), chunk by chunk where the program allows."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-9


def _run(name, n):
    import paper_1709_06416_b200 as wg
    from paper_1709_06416_b200 import workloads as W
    from weldmill.engine import EngineConfig, Value
    wl = W.WORKLOADS[name]
    tree = W.compile_program(wl)
    types = W.input_types(wl)
    cols = W.device_columns(wl, n)
    env = {k: Value(types[k], v) for k, v in cols.items()}
    out = wg.evaluate(tree, env, EngineConfig(memory_limit=1 << 46), W.externs_for(wl), result="numpy")[0].data
    del env, cols
    return out


def _host(name, n, row0=0):
    from paper_1709_06416_b200 import workloads as W
    return W.host_columns(W.WORKLOADS[name], n, row0=row0)


def _close(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) <= TOL * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


@pytest.mark.parametrize("n", [1_000_000, 600_000_000])
def test_c1_q6(n):
    from oracle import weld_oracle as O
    got = _run("q6", n)
    want, step = 0.0, 50_000_000
    for lo in range(0, n, step):
        want += O.q6(_host("q6", min(step, n - lo), lo))
    assert _close(got, want), (got, want)


def test_c2_blackscholes_64m():
    from oracle import weld_oracle as O
    n = 64 * 1024 * 1024
    call, put = _run("blackscholes", n)
    step = 16 * 1024 * 1024
    for lo in range(0, n, step):
        wc, wp = O.blackscholes(_host("blackscholes", step, lo))
        assert _close(call[lo:lo + step], wc).all()
        assert _close(put[lo:lo + step], wp).all()


def test_c3_q1_60m():
    from oracle import weld_oracle as O
    n = 60_000_000
    got = _run("q1", n)                 # flat leaves: k0, k1, then the six value fields
    want = O.q1(_host("q1", n))
    k0, k1, *vals = [np.asarray(c) for c in got]
    assert list(zip(k0.tolist(), k1.tolist())) == [k for k, _ in want]
    for j, (_, wv) in enumerate(want):
        assert int(vals[5][j]) == wv[5]
        for f in range(5):
            assert _close(vals[f][j], wv[f]), (j, f, vals[f][j], wv[f])


@pytest.fixture(scope="module")
def c4_oracle():
    """Stable sort of the 200M C4 rows by key (shared by C4a and C4b)."""
    cols = _host("dict", 200_000_000)
    k, v = cols["k"], cols["v"]
    order = np.argsort(k, kind="stable")
    ks = k[order]
    vs = v[order]
    del order
    starts = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
    return ks[starts], starts, vs


def test_c4a_dictmerger_200m(c4_oracle):
    uk, starts, vs = c4_oracle
    gk, gv = _run("dict", 200_000_000)
    np.testing.assert_array_equal(np.asarray(gk), uk)
    np.testing.assert_array_equal(np.asarray(gv), np.add.reduceat(vs, starts))


def test_c4b_groupbuilder_200m(c4_oracle):
    uk, starts, vs = c4_oracle
    keys, groups = _run("group", 200_000_000)         # keys, Ragged(offsets, values)
    np.testing.assert_array_equal(np.asarray(keys), uk)
    np.testing.assert_array_equal(np.asarray(groups.offsets), np.r_[starts, vs.size])
    np.testing.assert_array_equal(np.asarray(groups.values), vs)


def test_c5_histogram_1b():
    n = 1_000_000_000
    got = np.asarray(_run("hist", n))
    want = np.zeros(1_000_000)
    step = 100_000_000
    for lo in range(0, n, step):
        c = _host("hist", step, lo)
        want += np.bincount(c["idx"], weights=c["w"], minlength=1_000_000)
        del c
    assert _close(got, want).all()


@pytest.mark.parametrize("name", ["filter", "map"])
def test_appenders_500m(name):
    from oracle import weld_oracle as O
    n = 500_000_000
    got = np.asarray(_run(name, n))
    off, step = 0, 100_000_000
    for lo in range(0, n, step):
        w = O.ORACLES[name](_host(name, step, lo))
        np.testing.assert_array_equal(got[off:off + w.size], w)
        off += w.size
    assert off == got.size

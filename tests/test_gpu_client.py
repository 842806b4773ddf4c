"""The reference's client library (weldclient, pkg/client) over both of its
transports with the device executor underneath:

  * ForeignTransport (transport.py:58-105: weldmill.foreign in-process) with
    install() -- boundary-bytes leaves reach HBM without a decode to lists;
  * SubprocessTransport (transport.py:122-257: the `weldmill run/check`
    command over a manifest of boundary-bytes files) with its command set to
    paper_1709_06416_b200.cli -- the same tool with the device installed.

Every scenario is run on the reference (CPU engine, stock transports) and on
the device; result type text and boundary bytes must be identical.  The
known answers are the client tests' own (tests/test_transport.py:18-40)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

import paper_1709_06416_b200  # noqa: E402,F401  (puts baseline/_ref on the path)

# weldclient is installed next to weldmill in baseline/_ref ("Reference install")
pytest.importorskip("weldclient")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the stock tool (`python -m weldmill.cli`, transport.py:125) with the
# reference installed under baseline/_ref
REF_CLI = [sys.executable, "-c",
           f"import sys; sys.path.insert(0, {os.path.join(ROOT, 'baseline', '_ref')!r}); "
           "from weldmill.cli import main; sys.exit(main())"]
DEVICE_CLI = [sys.executable, "-c",
              f"import sys; sys.path.insert(0, {ROOT!r}); from paper_1709_06416_b200.cli import main; sys.exit(main())"]


def _scenarios(t):
    from weldclient import LazyArray, encode
    out = []
    xs = LazyArray([600000, 400000, 700000], transport=t)
    out.append(str(xs.filter(xs > 500000).sum()))
    ys = LazyArray(list(range(-2000, 30000)), transport=t)
    out.append(ys.map(lambda v: v * v, "(i64) => i64").to_list()[-3:])
    fs = LazyArray([0.5 * i for i in range(5000)], "f64", transport=t)
    out.append((fs.add(1.0).type_text, str(fs.mul(2.0).sum())))
    a = t.new_data("vec[i64]", encode(list(range(10000)), "vec[i64]"))
    shared = t.new_computed([a], "map(v0, (x) => x % 13)")
    root = t.new_computed([shared, shared], "reduce(v0, 0, (x, y) => x + y) + lookup(v1, 7)")
    out.append(t.evaluate(root))
    g = t.new_computed([a], "tovec(result(for(v0, dictmerger[i64, i64, +], (b, i, x) => merge(b, {x % 10, x}))))")
    out.append(t.evaluate(g))
    return out


def test_foreign_transport_on_the_device():
    import paper_1709_06416_b200 as wg
    from paper_1709_06416_b200 import runtime as rt
    from weldclient import ForeignTransport
    want = _scenarios(ForeignTransport())
    wg.install()
    try:
        before = rt.LAUNCHES[0]
        got = _scenarios(ForeignTransport())
        assert rt.LAUNCHES[0] > before
    finally:
        wg.uninstall()
    assert got == want
    assert want[0] == "1300000"


def test_subprocess_transport_on_the_device():
    from weldclient import SubprocessTransport
    want = _scenarios(SubprocessTransport(command=REF_CLI))
    got = _scenarios(SubprocessTransport(command=DEVICE_CLI))
    assert got == want
    assert want[0] == "1300000"


def test_subprocess_transport_staged_error():
    """A runtime error crosses the tool boundary as the same staged
    diagnostic (cli.py exit code 1 + JSON on stderr -> EvaluationFailed)."""
    from weldclient import EvaluationFailed, SubprocessTransport, encode

    def run(t):
        a = t.new_data("vec[i64]", encode([5, 4, 0, 2], "vec[i64]"))
        root = t.new_computed([a], "reduce(map(v0, (x) => 100 / x), 0, (p, q) => p + q)")
        with pytest.raises(EvaluationFailed) as ei:
            t.evaluate(root)
        return str(ei.value)
    assert run(SubprocessTransport(command=DEVICE_CLI)) == run(SubprocessTransport(command=REF_CLI))

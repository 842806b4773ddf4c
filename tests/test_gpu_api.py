"""The drop-in boundary end to end: the reference's own public API
(weldmill.api: new_data_object / new_computed_object / evaluate_object /
WeldResult, api.py:113-404) with install() routing its executor seam
(api.py:23 import, :374 call) to the B200 executor.  Results must be the
same boundary bytes as the reference CPU engine's; staged errors must carry
the same stage and error class (api.py:373-376)."""
import pytest

pytestmark = pytest.mark.gpu

PROGRAMS = [
    ("reduce(filter(v0, (x) => x > 3), 0, (x, y) => x + y)", [("vec[i64]", list(range(-50, 2000)))]),
    ("map(v0, (x) => x * 2.5 + 1.0)", [("vec[f64]", [0.5 * i for i in range(-300, 3000)])]),
    ("tovec(result(for(zip(v0, v1), dictmerger[i64, f64, +], (b, i, x) => merge(b, {x.0 % 7, x.1}))))",
     [("vec[i64]", list(range(5000))), ("vec[f64]", [float(i % 13) for i in range(5000)])]),
    ("result(for(v0, vecmerger[i64, +](v1), (b, i, x) => merge(b, {x % 10, 1})))",
     [("vec[i64]", list(range(3333))), ("vec[i64]", [0] * 10)]),
    ("sort(v0, (x) => 0 - x)", [("vec[i32]", [(i * 7919) % 1000 - 500 for i in range(2000)])]),
    ("map(v0, (x) => [x, x * 2])", [("vec[i64]", list(range(100)))]),
]


def _run(src, inputs):
    from weldmill.api import evaluate_object, free_result, new_computed_object, new_data_object
    from weldmill.parser import parse_type_text
    objs = [new_data_object(data, parse_type_text(t)) for t, data in inputs]
    r = evaluate_object(new_computed_object(objs, src))
    out = (r.ok, r.result_bytes() if r.ok else (r.error.stage, type(r.error.cause).__name__))
    free_result(r)
    return out


@pytest.mark.parametrize("src,inputs", PROGRAMS, ids=[p[0][:40] for p in PROGRAMS])
def test_public_api_bytes_match_reference(src, inputs):
    import paper_1709_06416_b200 as wg
    from paper_1709_06416_b200 import runtime as rt
    want = _run(src, inputs)          # reference CPU engine
    wg.install()
    try:
        before = rt.LAUNCHES[0]
        got = _run(src, inputs)       # same API, B200 executor underneath
        assert rt.LAUNCHES[0] > before    # the device path ran
    finally:
        wg.uninstall()
    assert got == want


def test_public_api_staged_errors_match_reference():
    import paper_1709_06416_b200 as wg
    src = "reduce(map(v0, (x) => 100 / x), 0, (a, b) => a + b)"
    inputs = [("vec[i64]", [5, 4, 0, 2])]
    want = _run(src, inputs)
    wg.install()
    try:
        got = _run(src, inputs)
    finally:
        wg.uninstall()
    assert want[0] is False and got == want


def test_reference_cli_runs_on_the_gpu(tmp_path, capsys):
    """weldmill's own CLI (`weldmill run prog --inputs manifest`, cli.py:188-213)
    with install(): the known answers of the reference's CLI tests
    (tests/test_cli.py: filter-sum 1300000; a struct of results [[2, 3, 4], 6])
    and the same --out boundary bytes as the CPU engine."""
    import json
    import paper_1709_06416_b200 as wg
    from weldmill import cli
    (tmp_path / "prog.ir").write_text(
        "result(for(v0, merger[i64, +], (b, i, x) => if (x > 500000, merge(b, x), b)))")
    (tmp_path / "two.ir").write_text(
        "data := [1, 2, 3];\nr1 := map(data, (x) => x + 1);\nr2 := reduce(data, 0, (x, y) => x + y);\n{r1, r2}\n")
    (tmp_path / "m.json").write_text(json.dumps(
        [{"name": "v0", "type": "vec[i64]", "value": [600000, 400000, 700000]}]))

    def run(*argv):
        capsys.readouterr()
        assert cli.main(list(argv)) == 0
        return json.loads(capsys.readouterr().out.strip().splitlines()[0])

    cpu_out = tmp_path / "cpu.bin"
    run("run", str(tmp_path / "prog.ir"), "--inputs", str(tmp_path / "m.json"), "--out", str(cpu_out))
    from paper_1709_06416_b200 import runtime as rt
    wg.install()
    try:
        before = rt.LAUNCHES[0]
        gpu_out = tmp_path / "gpu.bin"
        assert run("run", str(tmp_path / "prog.ir"), "--inputs", str(tmp_path / "m.json"),
                   "--out", str(gpu_out)) == 1300000
        assert run("run", str(tmp_path / "two.ir")) == [[2, 3, 4], 6]
        assert rt.LAUNCHES[0] > before
    finally:
        wg.uninstall()
    assert gpu_out.read_bytes() == cpu_out.read_bytes()


def test_concurrent_evaluate_calls_match_reference():
    """The reference allows evaluate() from several threads; the device
    executor serialises them (one process-wide runtime) and every thread
    gets its own correct result."""
    import threading
    import paper_1709_06416_b200 as wg
    want = [_run(src, inputs) for src, inputs in PROGRAMS]
    wg.install()
    got = [None] * (2 * len(PROGRAMS))
    errs = []

    def work(j):
        try:
            got[j] = _run(*PROGRAMS[j % len(PROGRAMS)])
        except Exception as ex:       # surfaced below
            errs.append(ex)
    try:
        ts = [threading.Thread(target=work, args=(j,)) for j in range(len(got))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    finally:
        wg.uninstall()
    assert not errs, errs
    assert got == want + want

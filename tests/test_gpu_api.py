"""The drop-in boundary end to end: the reference's own public API
(weldmill.api: new_data_object / new_computed_object / evaluate_object /
WeldResult, api.py:113-404) with install() routing its executor seam
(api.py:23 import, :374 call) to the B200 executor.  Results must be the
same boundary bytes as the reference CPU engine's; staged errors must carry
the same stage and error class (api.py:373-376)."""
import numpy as np
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


ZC_PROGRAMS = [
    ("result(for(zip(v0, v1), merger[f64, +], (b, i, x) => if (x.0 > 10, merge(b, x.1 * 2.0), b)))",
     [("vec[i32]", np.arange(-50, 2000, dtype=np.int32)), ("vec[f64]", np.arange(2050) * 0.25)]),
    ("filter(v0, (x) => x.0 % 3 == 0)",
     [("vec[{i64,f64}]", (np.arange(5000, dtype=np.int64), np.arange(5000) * 0.25))]),
    ("tovec(result(for(v0, dictmerger[i64, i64, +], (b, i, x) => merge(b, {x % 97, x}))))",
     [("vec[i64]", np.arange(100000, dtype=np.int64) * 7919)]),
    ("map(v0, (x) => x * 3 + 1)", [("vec[i64]", np.arange(-3000, 3000, dtype=np.int64))]),
    ("sort(v0, (x) => 0.0 - x)", [("vec[f64]", np.sin(np.arange(3000.0)))]),
]


def _lists(data):
    if isinstance(data, tuple):
        return [tuple(r) for r in zip(*(c.tolist() for c in data))]
    return data.tolist()


@pytest.mark.parametrize("src,inputs", ZC_PROGRAMS, ids=[p[0][:40] for p in ZC_PROGRAMS])
def test_zero_copy_leaves_bypass_the_codec(src, inputs):
    """install() binds numpy-column leaves straight to HBM: after the leaf's
    creation-time validation, evaluate_object makes no encode/decode call on
    it (the reference's build_program would round-trip every leaf through
    boundary bytes, api.py:224-226) -- and the result bytes equal the
    reference engine's over the same values given as lists."""
    import paper_1709_06416_b200 as wg
    from weldmill.api import Encoder, evaluate_object, free_result, new_computed_object, new_data_object
    from weldmill.parser import parse_type_text
    want = _run(src, [(t, _lists(d)) for t, d in inputs])
    calls = [0]

    def enc(d, t):
        calls[0] += 1
        return wg.column_encoder.encode(d, t)

    def dec(b, t):
        calls[0] += 1
        return wg.column_encoder.decode(b, t)
    counting = Encoder("counting", enc, dec)
    objs = [new_data_object(d, parse_type_text(t), counting) for t, d in inputs]
    created = calls[0]
    wg.install()
    try:
        r = evaluate_object(new_computed_object(objs, src))
        got = (r.ok, r.result_bytes() if r.ok else None)
        free_result(r)
    finally:
        wg.uninstall()
    assert calls[0] == created
    assert got == want


def test_zero_copy_foreign_bytes_leaf():
    """foreign.weld_new_data(type, boundary bytes) keeps the bytes as the
    leaf (no decode to lists) under install(); results match the reference."""
    import paper_1709_06416_b200 as wg
    from weldmill import foreign
    from weldmill.boundary import encode_value
    from weldmill.parser import parse_type_text

    def run():
        h = foreign.weld_new_data("vec[{i64,f64}]", encode_value([(i, i * 0.5) for i in range(4000)],
                                                                  parse_type_text("vec[{i64,f64}]")))
        c = foreign.weld_new_computed([h], "result(for(v0, merger[f64, +], (b, i, x) => merge(b, x.1 * cast(x.0, f64))))")
        r = foreign.weld_evaluate(c)
        return foreign.weld_result_error(r), foreign.weld_result_bytes(r)
    want = run()
    wg.install()
    try:
        got = run()
    finally:
        wg.uninstall()
    assert want[0] is None and got == want


def test_zero_copy_cli_manifest_path_input(tmp_path, capsys):
    """A manifest 'path' input (boundary bytes file, cli.py:150-153) reaches
    the device as bytes; stdout and --out bytes equal the CPU engine's."""
    import json
    import paper_1709_06416_b200 as wg
    from weldmill import cli
    from weldmill.boundary import encode_value
    from weldmill.parser import parse_type_text
    (tmp_path / "v.bin").write_bytes(encode_value(list(range(-500, 70000)), parse_type_text("vec[i64]")))
    (tmp_path / "p.ir").write_text("filter(v0, (x) => x % 7 == 3)")
    (tmp_path / "m.json").write_text(json.dumps([{"name": "v0", "type": "vec[i64]", "path": "v.bin"}]))

    def run(out):
        capsys.readouterr()
        assert cli.main(["run", str(tmp_path / "p.ir"), "--inputs", str(tmp_path / "m.json"), "--out", str(out)]) == 0
        return capsys.readouterr().out
    want = run(tmp_path / "cpu.bin")
    wg.install()
    try:
        got = run(tmp_path / "gpu.bin")
    finally:
        wg.uninstall()
    assert got == want
    assert (tmp_path / "gpu.bin").read_bytes() == (tmp_path / "cpu.bin").read_bytes()

"""The committed math tables (csrc/wg_erf_table.h, wg_log_table.h, wg_exp_table.h) are
exactly what their generators produce, and the generators' own accuracy
checks pass (erf table <= 0.5 ulp evaluated exactly; the log algorithm,
emulated with correctly rounded fma, <= 1 ulp from mpmath).  CPU only."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(name):
    spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, "tools", name + ".py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("gen,header", [("gen_erf_table", "wg_erf_table.h"), ("gen_log_table", "wg_log_table.h"),
                                        ("gen_exp_table", "wg_exp_table.h")])
def test_table_matches_generator(gen, header, tmp_path, monkeypatch):
    pytest.importorskip("mpmath")
    mod = _load(gen)
    out = tmp_path / header
    monkeypatch.setattr(mod, "OUT", str(out))
    mod.main()
    committed = open(os.path.join(ROOT, "paper_1709_06416_b200", "csrc", header)).read()
    assert out.read_text() == committed

"""Generate golden fixtures from the reference implementation itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/corpus.json and tests/golden/configs.json.  The GPU box
has no /root/reference: the tests read these committed fixtures instead.

* corpus.json  -- the reference's own 308-program differential corpus
  (/root/reference/pkg/tests/progen.py:58-290, SEED 20260818), two seeded
  input sets per program, expected value = weldmill.engine.evaluate on the
  unoptimised tree (run.py:1008; test_acceptance.py:157-178 asserts every
  optimizer level agrees with it).
* configs.json -- the five benchmark programs (paper_1709_06416_b200/
  workloads.py) on the first N generator rows, evaluated by the reference
  engine (BASELINE.md section 3 recipe).
"""
import json
import math
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, ROOT)

from weldmill.engine import EngineConfig, Value, evaluate  # noqa: E402
from weldmill.optim import OptLevel, optimize  # noqa: E402
from weldmill.parser import parse, parse_type_text  # noqa: E402
from weldmill.sugar import expand  # noqa: E402
from weldmill.typecheck import check_linearity, infer  # noqa: E402

import progen  # noqa: E402


def norm(v):
    if isinstance(v, (list, tuple)):
        return [norm(x) for x in v]
    if isinstance(v, dict):
        return [[norm(k), norm(x)] for k, x in v.items()]
    return v


def corpus():
    out = []
    for p in progen.corpus():
        env = {k: parse_type_text(t) for k, t in p.inputs.items()}
        typed = infer(expand(parse(p.source)), env)
        check_linearity(typed)
        rng = random.Random(hash((progen.SEED, p.name)) & 0xFFFFFFFF)
        cases = []
        for _ in range(2):
            inputs = p.make_inputs(rng)
            vals = {k: Value(env[k], v) for k, v in inputs.items()}
            res = evaluate(typed, vals)[0].data
            cases.append({"inputs": inputs, "expected": norm(res)})
        out.append({"name": p.name, "source": p.source, "inputs": p.inputs, "is_float": p.is_float,
                    "cases": cases})
    return out


def configs(n):
    import numpy as np
    from paper_1709_06416_b200 import workloads as W
    out = {}
    for name, wl in W.WORKLOADS.items():
        cols = W.host_columns(wl, n)
        opt = W.compile_program(wl)
        env = {}
        types = W.input_types(wl)
        for k, arr in cols.items():
            env[k] = Value(types[k], arr.tolist())
        res = evaluate(opt, env, EngineConfig(threads=1, memory_limit=1 << 40),
                       externs=W.externs_for(wl))[0].data
        if name == "hist":
            res = [[i, x] for i, x in enumerate(res) if x != 0.0]
        out[name] = {"n": n, "expected": norm(res)}
    return out


if __name__ == "__main__":
    c = corpus()
    with open(os.path.join(HERE, "corpus.json"), "w") as f:
        json.dump({"seed": progen.SEED, "programs": c}, f, separators=(",", ":"))
    cf = configs(4096)
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(cf, f, separators=(",", ":"))
    print(len(c), "corpus programs;", ", ".join(cf))

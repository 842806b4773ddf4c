"""A second differential corpus from the reference's own program generator
(/root/reference/pkg/tests/progen.py) with a different seed (20261017
instead of SEED=20260818): new constants, new programs where the generator
branches on them, three fresh input sets each.  Expected values come from
weldmill.engine.evaluate on the unoptimised tree, as in make_golden.py.

    python tests/golden/make_corpus2.py     # writes tests/golden/corpus_s2.json
"""
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import progen  # noqa: E402
from weldmill.engine import Value, evaluate  # noqa: E402
from weldmill.parser import parse, parse_type_text  # noqa: E402
from weldmill.sugar import expand  # noqa: E402
from weldmill.typecheck import check_linearity, infer  # noqa: E402

SEED2 = 20261017


def norm(v):
    if isinstance(v, (list, tuple)):
        return [norm(x) for x in v]
    if isinstance(v, dict):
        return [[norm(k), norm(x)] for k, x in v.items()]
    return v


def main():
    progen.SEED = SEED2
    out = []
    for p in progen.corpus():
        env = {k: parse_type_text(t) for k, t in p.inputs.items()}
        typed = infer(expand(parse(p.source)), env)
        check_linearity(typed)
        rng = random.Random(hash((SEED2, p.name)) & 0xFFFFFFFF)
        cases = []
        for _ in range(3):
            inputs = p.make_inputs(rng)
            vals = {k: Value(env[k], v) for k, v in inputs.items()}
            try:
                res = {"expected": norm(evaluate(typed, vals)[0].data)}
            except Exception as exc:          # runtime errors are part of the contract
                res = {"error": type(exc).__name__}
            cases.append({"inputs": inputs, **res})
        out.append({"name": p.name, "source": p.source, "inputs": p.inputs, "is_float": p.is_float,
                    "cases": cases})
    with open(os.path.join(HERE, "corpus_s2.json"), "w") as f:
        json.dump({"seed": SEED2, "programs": out}, f, separators=(",", ":"))
    print(len(out), "programs")


if __name__ == "__main__":
    main()

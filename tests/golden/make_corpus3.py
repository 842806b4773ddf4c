"""A third differential corpus from the reference's own program generator
(/root/reference/pkg/tests/progen.py), seed 20261018, with LARGE inputs: the
generator's vector lengths (randint(8, 32)) are drawn from [2049, 2600]
instead, so every loop spans more than one 2048-row tile of the device
schedules (look-back chains, partial last tiles, multi-tile dictionaries).
One input set per program; expected values (or runtime error classes) come
from weldmill.engine.evaluate on the unoptimised tree, as in make_golden.py.

    python tests/golden/make_corpus3.py     # writes tests/golden/corpus_s3.json.gz
"""
import gzip
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

SEED3 = 20261018


class LongVectors(random.Random):
    """progen draws every vector length as randint(8, 32); stretch those."""

    def randint(self, a, b):
        if (a, b) == (8, 32):
            return super().randint(2049, 2600)
        return super().randint(a, b)


def norm(v):
    if isinstance(v, (list, tuple)):
        return [norm(x) for x in v]
    if isinstance(v, dict):
        return [[norm(k), norm(x)] for k, x in v.items()]
    return v


def main():
    progen.SEED = SEED3
    out = []
    for p in progen.corpus():
        env = {k: parse_type_text(t) for k, t in p.inputs.items()}
        typed = infer(expand(parse(p.source)), env)
        check_linearity(typed)
        rng = LongVectors(hash((SEED3, p.name)) & 0xFFFFFFFF)
        inputs = p.make_inputs(rng)
        vals = {k: Value(env[k], v) for k, v in inputs.items()}
        try:
            res = {"expected": norm(evaluate(typed, vals)[0].data)}
        except Exception as exc:          # runtime errors are part of the contract
            res = {"error": type(exc).__name__}
        out.append({"name": p.name, "source": p.source, "inputs": p.inputs, "is_float": p.is_float,
                    "cases": [{"inputs": inputs, **res}]})
    with gzip.open(os.path.join(HERE, "corpus_s3.json.gz"), "wt") as f:
        json.dump({"seed": SEED3, "programs": out}, f, separators=(",", ":"))
    print(len(out), "programs")


if __name__ == "__main__":
    main()

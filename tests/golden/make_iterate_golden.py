"""Golden fixtures for `iterate` inside loop bodies (run.py:668-686),
produced by the reference implementation itself.

    python tests/golden/make_iterate_golden.py     # writes tests/golden/iterate.json
"""
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from weldmill.engine import EngineConfig, Value, evaluate  # noqa: E402
from weldmill.errors import EvalError  # noqa: E402
from weldmill.optim import OptLevel, optimize  # noqa: E402
from weldmill.parser import parse, parse_type_text  # noqa: E402
from weldmill.sugar import expand  # noqa: E402
from weldmill.typecheck import check_linearity, infer  # noqa: E402

CASES = [
    ("iterate-doubling-sum",
     "result(for(v, merger[i64, +], (b, i, x) => merge(b, iterate(x, (s) => {s * 2, s * 2 < 1000}))))",
     {"v": "vec[i64]"}, 100_000),
    ("iterate-struct-state-map",
     "map(v, (x) => iterate({x, 0}, (s) => {{s.0 / 2, s.1 + 1}, s.0 > 1}).1)",
     {"v": "vec[i64]"}, 100_000),
    ("iterate-f64-newton",
     "map(w, (y) => iterate({y, 0}, (s) => {{0.5 * (s.0 + y / s.0), s.1 + 1}, s.1 < 6}).0)",
     {"w": "vec[f64]"}, 100_000),
    ("iterate-limit",
     "result(for(v, merger[i64, +], (b, i, x) => merge(b, iterate(x, (s) => {s * 2, s * 2 < 1000}))))",
     {"v": "vec[i64]"}, 50),
]


def inputs(name, seed):
    r = random.Random(seed)
    n = 3000
    if name == "iterate-f64-newton":
        return {"w": [r.uniform(0.5, 1e6) for _ in range(n)]}
    if name == "iterate-limit":
        return {"v": [r.randrange(1, 100) for _ in range(n)] + [0]}
    return {"v": [r.randrange(1, 5000) for _ in range(n)]}


def main():
    out = []
    for name, src, types, limit in CASES:
        env_t = {k: parse_type_text(t) for k, t in types.items()}
        typed = infer(expand(parse(src)), env_t)
        check_linearity(typed)
        tree = optimize(typed, OptLevel.all())[0]
        for seed in (1, 2):
            data = inputs(name, seed)
            env = {k: Value(env_t[k], v) for k, v in data.items()}
            try:
                val = evaluate(tree, env, EngineConfig(max_iterations=limit))[0].data
                exp = {"value": val}
            except EvalError as exc:
                exp = {"error": type(exc).__name__}
            out.append({"name": name, "source": src, "inputs": types, "data": data, "max_iterations": limit,
                        "expected": exp})
    with open(os.path.join(HERE, "iterate.json"), "w") as f:
        json.dump({"cases": out}, f)
    print(len(out), "cases")


if __name__ == "__main__":
    main()

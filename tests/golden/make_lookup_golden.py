"""Golden fixtures for dictionary probes inside loop bodies (hash joins),
produced by the reference implementation itself.

    python tests/golden/make_lookup_golden.py      # writes tests/golden/lookup.json

Each case is an IR program whose loop body does `lookup(d, k)` into a
dictionary built by an earlier loop (run.py:702-712; KeyNotFound on a miss),
with seeded inputs; the expected value (or error class) is
weldmill.engine.evaluate on the optimised tree.
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
    # join: sum of the build side's per-key sums over the probe keys
    ("join-sum-f64",
     "d := result(for({bk, bv}, dictmerger[i64, f64, +], (b, i, x) => merge(b, {x.0, x.1})));"
     " result(for(pk, merger[f64, +], (b, i, x) => merge(b, lookup(d, x))))",
     {"bk": "vec[i64]", "bv": "vec[f64]", "pk": "vec[i64]"}),
    # join producing a vector (probe -> appender), struct keys
    ("join-map-struct-key",
     "d := result(for({ba, bb, bv}, dictmerger[{i32, i32}, i64, +], (b, i, x) => merge(b, {{x.0, x.1}, x.2})));"
     " result(for({pa, pb}, vecbuilder[i64], (b, i, x) => merge(b, lookup(d, {x.0, x.1}) * 2)))",
     {"ba": "vec[i32]", "bb": "vec[i32]", "bv": "vec[i64]", "pa": "vec[i32]", "pb": "vec[i32]"}),
    # semi-join style filter with a max dictionary
    ("join-filter-max",
     "d := result(for({bk, bv}, dictmerger[i64, i64, max], (b, i, x) => merge(b, {x.0, x.1})));"
     " result(for(pk, merger[i64, +], (b, i, x) => if (lookup(d, x) > 0, merge(b, x), b)))",
     {"bk": "vec[i64]", "bv": "vec[i64]", "pk": "vec[i64]"}),
    # probe into a groupbuilder result: the value is a vector
    ("join-group-len-sum",
     "g := result(for({bk, bv}, groupbuilder[i64, i64], (b, i, x) => merge(b, {x.0, x.1})));"
     " result(for(pk, merger[i64, +], (b, i, x) => merge(b, len(lookup(g, x)) * 1000"
     " + result(for(lookup(g, x), merger[i64, +], (c, j, y) => merge(c, y))))))",
     {"bk": "vec[i64]", "bv": "vec[i64]", "pk": "vec[i64]"}),
    # float keys: -0.0 and 0.0 are one key
    ("join-f64-keys",
     "d := result(for({bf, bv}, dictmerger[f64, i64, +], (b, i, x) => merge(b, {x.0, x.1})));"
     " result(for(pf, merger[i64, +], (b, i, x) => merge(b, lookup(d, x))))",
     {"bf": "vec[f64]", "bv": "vec[i64]", "pf": "vec[f64]"}),
    # a probe key missing from the build side: KeyNotFound
    ("join-miss",
     "d := result(for({bk, bv}, dictmerger[i64, i64, +], (b, i, x) => merge(b, {x.0, x.1})));"
     " result(for(pk, merger[i64, +], (b, i, x) => merge(b, lookup(d, x))))",
     {"bk": "vec[i64]", "bv": "vec[i64]", "pk": "vec[i64]"}),
]


def inputs(name, seed, n=3000):
    r = random.Random(seed)
    keys = [r.randrange(-500, 500) for _ in range(200)]
    if name == "join-miss":
        return {"bk": [r.choice(keys) for _ in range(n)], "bv": [r.randrange(-9, 9) for _ in range(n)],
                "pk": [r.choice(keys) for _ in range(n // 2)] + [10_000]}
    if name == "join-map-struct-key":
        pairs = [(r.randrange(-3, 3), r.randrange(-40, 40)) for _ in range(100)]
        bp = [r.choice(pairs) for _ in range(n)]
        pp = [r.choice(sorted(set(bp))) for _ in range(n // 3)]
        return {"ba": [a for a, _ in bp], "bb": [b for _, b in bp], "bv": [r.randrange(-50, 50) for _ in range(n)],
                "pa": [a for a, _ in pp], "pb": [b for _, b in pp]}
    if name == "join-f64-keys":
        fk = [0.0, -0.0, 1.5, -2.25, 1e300, -1e-300, 3.0]
        return {"bf": [r.choice(fk) for _ in range(n)], "bv": [r.randrange(-9, 9) for _ in range(n)],
                "pf": [r.choice(fk) for _ in range(n // 2)]}
    bk = [r.choice(keys) for _ in range(n)]
    present = sorted(set(bk))
    out = {"bk": bk, "pk": [r.choice(present) for _ in range(n // 2)]}
    out["bv"] = ([r.uniform(-10, 10) for _ in range(n)] if name == "join-sum-f64"
                 else [r.randrange(-100, 100) for _ in range(n)])
    return out


def main():
    out = []
    for name, src, types in CASES:
        env_t = {k: parse_type_text(t) for k, t in types.items()}
        typed = infer(expand(parse(src)), env_t)
        check_linearity(typed)
        tree = optimize(typed, OptLevel.all())[0]
        for seed in (1, 2):
            data = inputs(name, seed)
            env = {k: Value(env_t[k], v) for k, v in data.items()}
            try:
                val = evaluate(tree, env, EngineConfig())[0].data
                exp = {"value": val}
            except EvalError as exc:
                exp = {"error": type(exc).__name__}
            out.append({"name": name, "source": src, "inputs": types, "data": data, "expected": exp})
    with open(os.path.join(HERE, "lookup.json"), "w") as f:
        json.dump({"cases": out}, f)
    print(len(out), "cases")


if __name__ == "__main__":
    main()

"""Golden fixtures for flatmap-shaped loops -- appends inside a nested loop
whose trip count depends on the data -- produced by the reference itself.

    python tests/golden/make_flatmap_golden.py     # writes tests/golden/flatmap.json

Expected value = weldmill.engine.evaluate on the optimised tree
(run.py:947-983: nested loops run sequentially inside the parent's row, so
appends come out row-major, inner-loop order within a row)."""
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from weldmill.engine import EngineConfig, Value, evaluate  # noqa: E402
from weldmill.optim import OptLevel, optimize  # noqa: E402
from weldmill.parser import parse, parse_type_text  # noqa: E402
from weldmill.sugar import expand  # noqa: E402
from weldmill.typecheck import check_linearity, infer  # noqa: E402

CASES = [
    ("flatmap-filtered-range",
     "result(for(v, vecbuilder[i64], (b, i, x) => for(rng, b, (c, j, y) => if (y < x, merge(c, x * 10 + y), c))))",
     {"v": "vec[i64]", "rng": "vec[i64]"}),
    ("flatmap-with-merger",
     "r := result(for(v, {vecbuilder[i64], merger[i64, +]}, (b, i, x) => "
     "{for(rng, b.0, (c, j, y) => if (y < x, merge(c, y - x), c)), merge(b.1, x)})); {r.0, r.1}",
     {"v": "vec[i64]", "rng": "vec[i64]"}),
    ("flatmap-struct-elems",
     "result(for({v, w}, vecbuilder[{i64, f64}], (b, i, x) => for(rng, b, (c, j, y) => "
     "if (y % 3 == x.0 % 3, merge(c, {i * 100 + y, x.1 * cast(y, f64)}), c))))",
     {"v": "vec[i64]", "w": "vec[f64]", "rng": "vec[i64]"}),
    ("flatmap-group-expand",
     "g := result(for({bk, bv}, groupbuilder[i64, i64], (b, i, x) => merge(b, {x.0, x.1})));"
     " result(for(pk, vecbuilder[i64], (b, i, x) => for(lookup(g, x), b, (c, j, y) => merge(c, y * 2 + j))))",
     {"bk": "vec[i64]", "bv": "vec[i64]", "pk": "vec[i64]"}),
    # the reference's own flatmap sugar (sugar.py:196-202)
    ("flatmap-sugar-group",
     "g := result(for({bk, bv}, groupbuilder[i64, i64], (b, i, x) => merge(b, {x.0, x.1})));"
     " flatmap(pk, (x) => lookup(g, x))",
     {"bk": "vec[i64]", "bv": "vec[i64]", "pk": "vec[i64]"}),
]


def inputs(name, seed):
    r = random.Random(seed)
    if name in ("flatmap-group-expand", "flatmap-sugar-group"):
        keys = [r.randrange(-50, 50) for _ in range(40)]
        bk = [r.choice(keys) for _ in range(2000)]
        return {"bk": bk, "bv": [r.randrange(-99, 99) for _ in range(2000)],
                "pk": [r.choice(sorted(set(bk))) for _ in range(700)]}
    n = 1500
    out = {"v": [r.randrange(-2, 9) for _ in range(n)], "rng": list(range(8))}
    if name == "flatmap-struct-elems":
        out["w"] = [r.uniform(-5, 5) for _ in range(n)]
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
            val = evaluate(tree, env, EngineConfig())[0].data
            out.append({"name": name, "source": src, "inputs": types, "data": data, "expected": {"value": val}})
    with open(os.path.join(HERE, "flatmap.json"), "w") as f:
        json.dump({"cases": out}, f)
    print(len(out), "cases")


if __name__ == "__main__":
    main()

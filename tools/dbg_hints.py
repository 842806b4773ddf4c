import sys, itertools
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from paper_1709_06416_b200 import executor, builders_dev as BD
from weldmill.expr import walk, For
import test_gpu_rpart as T
executor.RPART = True
src = ("d := for({k, v}, dictmerger[i64, i64, +], (b, i, x) => merge(b, {x.0, x.1}));"
       " tovec(result(for({k, v}, d, (b, i, x) => merge(b, {x.0, 1}))))")
rng = np.random.default_rng(5)
n = 100_000
k = rng.integers(-(1 << 40), 1 << 40, size=10_000, dtype=np.int64)[rng.integers(0, 10_000, size=n)]
v = rng.integers(-9, 9, size=n, dtype=np.int64)
u, s = T._want_sum(k, v + 1)
tree = T._prog(src, {"k": "vec[i64]", "v": "vec[i64]"}, opt=False)
fors = [x for x in walk(tree) if isinstance(x, For)]
print("loops", len(fors))
okmin = (int(k.min()) ^ (1 << 63)) & ((1 << 64) - 1); okmax = (int(k.max()) ^ (1 << 63)) & ((1 << 64) - 1)
sizes = [None, 50, 5000, 3_300_000]
ranges = [None, (okmin, okmax), (1 << 62, (1 << 64) - (1 << 62)), (0, 1000)]
bad = 0
for pmin in (100, 1 << 20):
    executor.PART_MIN_KEYS = pmin
    for s1, r1, s2, r2 in itertools.product(sizes, ranges, sizes, ranges):
        BD._SIZE_HINTS.clear(); BD._RANGE_HINTS.clear(); executor._RPART_BAD.clear()
        for f, sz, rg in ((fors[0], s1, r1), (fors[1], s2, r2)):
            if sz is not None: BD._SIZE_HINTS[(id(f), 0)] = sz
            if rg is not None: BD._RANGE_HINTS[(id(f), 0)] = rg
        try:
            got = T._eval(tree, k, v)
            ok = np.array_equal(got[0], u) and np.array_equal(got[1], s)
        except Exception as exc:
            ok = False; print("EXC", repr(exc)[:200])
        if not ok:
            bad += 1
            print("FAIL pmin", pmin, "loop1", s1, r1, "loop2", s2, r2, flush=True)
print("bad", bad)

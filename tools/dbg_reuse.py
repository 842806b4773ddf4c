import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from paper_1709_06416_b200 import executor
import test_gpu_rpart as T
for rpart, pmin in ((False, 1 << 20), (False, 100), (True, 100)):
    executor.RPART = rpart
    executor.PART_MIN_KEYS = pmin
    src = ("d := for({k, v}, dictmerger[i64, i64, +], (b, i, x) => merge(b, {x.0, x.1}));"
           " tovec(result(for({k, v}, d, (b, i, x) => merge(b, {x.0, 1}))))")
    rng = np.random.default_rng(5)
    n = 100_000
    k = rng.integers(-(1 << 40), 1 << 40, size=10_000, dtype=np.int64)[rng.integers(0, 10_000, size=n)]
    v = rng.integers(-9, 9, size=n, dtype=np.int64)
    tree = T._prog(src, {"k": "vec[i64]", "v": "vec[i64]"}, opt=False)
    u, s = T._want_sum(k, v + 1)
    for it in range(3):
        got = T._eval(tree, k, v)
        print("rpart", rpart, "pmin", pmin, "iter", it, "keys ok", np.array_equal(got[0], u), "vals ok", np.array_equal(got[1], s), flush=True)

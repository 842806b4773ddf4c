"""Host-side overhead profile of one evaluate() step (run on the GPU box)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import runtime as rt
from paper_1709_06416_b200 import workloads as W
from weldmill.engine import EngineConfig, Value

name = sys.argv[1] if len(sys.argv) > 1 else "blackscholes"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wl = W.WORKLOADS[name]
n = n or wl.n
tree = W.compile_program(wl)
types = W.input_types(wl)
cols = W.device_columns(wl, n)
env = {k: Value(types[k], v) for k, v in cols.items()}
cfg = EngineConfig(memory_limit=1 << 46)
ext = W.externs_for(wl)
for _ in range(3):
    wg.evaluate(tree, env, cfg, ext, result="device")
rt.sync()
for _ in range(3):
    t0 = time.perf_counter()
    out = wg.evaluate(tree, env, cfg, ext, result="device")
    t1 = time.perf_counter()
    rt.sync()
    t2 = time.perf_counter()
    print(f"evaluate host {1e3*(t1-t0):.2f} ms, +sync {1e3*(t2-t1):.2f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    out = wg.evaluate(tree, env, cfg, ext, result="device")
rt.sync()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)

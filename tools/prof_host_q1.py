"""cProfile of the host control plane of repeated evaluate() calls."""
import cProfile, pstats, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import workloads as W, runtime as rt
from weldmill.engine import EngineConfig, Value
name = sys.argv[1] if len(sys.argv) > 1 else "q1"
wl = W.WORKLOADS[name]
tree = W.compile_program(wl)
types = W.input_types(wl)
n = int(sys.argv[2]) if len(sys.argv) > 2 else wl.n
cols = W.device_columns(wl, n)
env = {k: Value(types[k], v) for k, v in cols.items()}
cfg = EngineConfig(memory_limit=1 << 46)
for _ in range(3):
    wg.evaluate(tree, env, cfg, W.externs_for(wl), result="device")
rt.sync()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    wg.evaluate(tree, env, cfg, W.externs_for(wl), result="device")
rt.sync()
pr.disable()
print("ms/call", (time.perf_counter() - t0) / 20 * 1e3)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)

"""Host-side overhead of evaluate() for a small program (many iterations)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import runtime as rt, workloads as W
from weldmill.engine import EngineConfig, Value
name = sys.argv[1] if len(sys.argv) > 1 else "q6"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
wl = W.WORKLOADS[name]
tree = W.compile_program(wl)
types = W.input_types(wl)
env = {k: Value(types[k], v) for k, v in W.device_columns(wl, n).items()}
cfg = EngineConfig(memory_limit=1 << 46)
ext = W.externs_for(wl)
for _ in range(20):
    wg.evaluate(tree, env, cfg, ext, result="device")
rt.sync()
N = 2000
t0 = time.perf_counter()
for _ in range(N):
    wg.evaluate(tree, env, cfg, ext, result="device")
rt.sync()
print(f"{name} n={n}: {1e6 * (time.perf_counter() - t0) / N:.1f} us per evaluate")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    wg.evaluate(tree, env, cfg, ext, result="device")
pr.disable()
pstats.Stats(pr).sort_stats(sys.argv[3] if len(sys.argv) > 3 else "tottime").print_stats(40)

import gc
import sys
import time
sys.path.insert(0, ".")
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import runtime as rt
from paper_1709_06416_b200 import workloads as W
from weldmill.engine import EngineConfig, Value

name = sys.argv[1]
wl = W.WORKLOADS[name]
tree = W.compile_program(wl)
types = W.input_types(wl)
cols = W.device_columns(wl, wl.n)
env = {k: Value(types[k], v) for k, v in cols.items()}
cfg = EngineConfig(memory_limit=1 << 46)
ext = W.externs_for(wl)
rt.sync()
print("after inputs live/peak GB", [x / 1e9 for x in rt.mem_stats()])
for i in range(4):
    t0 = time.perf_counter()
    v = wg.evaluate(tree, env, cfg, ext, result="device")
    rt.sync()
    t1 = time.perf_counter()
    del v
    live, peak = rt.mem_stats()
    print(f"eval {i}: {1e3*(t1-t0):.2f} ms; live {live/1e9:.3f} GB peak {peak/1e9:.3f} GB; gc objs {len(gc.get_objects())}")
gc.collect()
print("after gc live GB", rt.mem_stats()[0] / 1e9)
print("gc garbage check:")
gc.set_debug(0)

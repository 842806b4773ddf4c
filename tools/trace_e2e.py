"""Breakdown of one e2e evaluate() with host (pinned) inputs and numpy results."""
import os
import sys
import time
os.environ["WELDGPU_TRACE"] = "1"
sys.path.insert(0, ".")
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import runtime as rt
from paper_1709_06416_b200 import workloads as W
from weldmill.engine import EngineConfig, Value

name = sys.argv[1] if len(sys.argv) > 1 else "blackscholes"
wl = W.WORKLOADS[name]
tree = W.compile_program(wl)
types = W.input_types(wl)
host = W.host_columns(wl, wl.n)
for a in host.values():
    rt.host_register(a)
env = {k: Value(types[k], v) for k, v in host.items()}
cfg = EngineConfig(memory_limit=1 << 46)
ext = W.externs_for(wl)
res = None
for _ in range(3):
    res = wg.evaluate(tree, env, cfg, ext, result="numpy")[0].data
rt.sync()
rt.TRACE_TIMES.clear()
t0 = time.perf_counter()
res = wg.evaluate(tree, env, cfg, ext, result="numpy")[0].data
tot = time.perf_counter() - t0
print(f"== {name} e2e: {tot*1e3:.2f} ms")
for k, v in sorted(rt.TRACE_TIMES.items(), key=lambda x: -x[1]):
    print(f"   {v*1e3:9.3f} ms  {k}")
print(f"   {(tot - sum(rt.TRACE_TIMES.values()))*1e3:9.3f} ms  (other: host python, async d2h + sync)")

"""Per-call breakdown of one evaluate() (syncs around every device call)."""
import os
import sys
import time
os.environ["WELDGPU_TRACE"] = "1"
sys.path.insert(0, ".")
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import runtime as rt
from paper_1709_06416_b200 import workloads as W
from weldmill.engine import EngineConfig, Value

for name in sys.argv[1:]:
    wl = W.WORKLOADS[name]
    tree = W.compile_program(wl)
    types = W.input_types(wl)
    cols = W.device_columns(wl, wl.n)
    env = {k: Value(types[k], v) for k, v in cols.items()}
    cfg = EngineConfig(memory_limit=1 << 46)
    ext = W.externs_for(wl)
    for _ in range(2):
        wg.evaluate(tree, env, cfg, ext, result="device")
    rt.sync()
    rt.TRACE_TIMES.clear()
    t0 = time.perf_counter()
    wg.evaluate(tree, env, cfg, ext, result="device")
    rt.sync()
    tot = time.perf_counter() - t0
    print(f"== {name}: evaluate {tot*1e3:.2f} ms")
    for k, v in sorted(rt.TRACE_TIMES.items(), key=lambda x: -x[1]):
        print(f"   {v*1e3:9.3f} ms  {k}")
    print(f"   {(tot - sum(rt.TRACE_TIMES.values()))*1e3:9.3f} ms  (host python)")

"""Mimic bench.py's timed region and print each step's wall time, with and
without the nvidia-smi sampler."""
import gc
import sys
import time
sys.path.insert(0, ".")
import bench
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import runtime as rt
from paper_1709_06416_b200 import workloads as W
from weldmill.engine import EngineConfig, Value

name = sys.argv[1] if len(sys.argv) > 1 else "blackscholes"
wl = W.WORKLOADS[name]
tree = W.compile_program(wl)
types = W.input_types(wl)
cols = W.device_columns(wl, wl.n)
env = {k: Value(types[k], v) for k, v in cols.items()}
cfg = EngineConfig(memory_limit=1 << 46)
ext = W.externs_for(wl)
for _ in range(3):
    wg.evaluate(tree, env, cfg, ext, result="device")
rt.sync()
for use_clocks in (False, True, False, True):
    c = bench.Clocks(0) if use_clocks else None
    if c:
        c.start()
        time.sleep(0.5)
    gc.collect(); gc.disable()
    ts = []
    e0, e1 = rt.Event(), rt.Event()
    e0.record()
    for _ in range(10):
        t0 = time.perf_counter()
        out = wg.evaluate(tree, env, cfg, ext, result="device")
        ts.append((time.perf_counter() - t0) * 1e3)
    e1.record(); rt.sync()
    gc.enable()
    if c:
        c.stop()
    print(f"clocks={use_clocks}: device {e0.elapsed_ms(e1)/10:.3f} ms/step; per-step wall ms:", " ".join(f"{t:.2f}" for t in ts))

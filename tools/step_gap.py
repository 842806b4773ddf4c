"""Where does a bench step go?  Device time per step with/without the
nvidia-smi sampler and with/without result retention."""
import subprocess
import sys
import time

sys.path.insert(0, ".")
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


def run(steps, keep):
    e0, e1 = rt.Event(), rt.Event()
    rt.sync()
    t0 = time.perf_counter()
    e0.record()
    out = None
    for _ in range(steps):
        if keep:
            out = wg.evaluate(tree, env, cfg, ext, result="device")
        else:
            wg.evaluate(tree, env, cfg, ext, result="device")
    e1.record()
    rt.sync()
    t1 = time.perf_counter()
    return e0.elapsed_ms(e1) / steps, (t1 - t0) * 1e3 / steps


for smi in (False, True):
    p = None
    if smi:
        p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"],
                             stdout=subprocess.DEVNULL)
        time.sleep(0.5)
    for keep in (False, True):
        dev, wall = run(20, keep)
        print(f"smi={smi} keep={keep}: device {dev:.3f} ms/step, wall {wall:.3f} ms/step")
    if p:
        p.terminate()

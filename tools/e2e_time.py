import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import runtime as rt, executor as ex
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
for stream in (0, 1):
    ex.STREAMING = bool(stream)
    for chunk in ((1 << 23), (1 << 24), (1 << 22)):
        ex.STREAM_CHUNK_ROWS = chunk
        res = None
        for _ in range(3):
            res = wg.evaluate(tree, env, cfg, ext, result="numpy")[0].data
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            res = wg.evaluate(tree, env, cfg, ext, result="numpy")[0].data
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"stream={stream} chunk={chunk >> 20}M: " + " ".join(f"{t:.1f}" for t in ts) + " ms", flush=True)
        if not stream:
            break

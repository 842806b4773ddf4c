"""Group step time for narrow-range keys (k in [0, 10M), not scrambled):
the 32-bit sort-key path of wg_group_finish1 vs the 64-bit one.
    WELDGPU_GROUP_U32=0|1 python tools/group_narrow.py"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import runtime as rt, workloads as W
from weldmill.engine import EngineConfig, Value

wl = W.WORKLOADS["group"]
wl2 = W.Workload(wl.name, wl.title, wl.program,
                 [W.ColSpec("k", "i64", 0, 0, lo=0, span=10_000_000), wl.columns[1]],
                 n=wl.n, bytes_per_row=wl.bytes_per_row, out_bytes=wl.out_bytes, dtype=wl.dtype)
n = 200_000_000
tree = W.compile_program(wl2)
types = W.input_types(wl2)
env = {k: Value(types[k], v) for k, v in W.device_columns(wl2, n).items()}
cfg = EngineConfig(memory_limit=1 << 46)
for _ in range(2):
    wg.evaluate(tree, env, cfg, {}, result="device")
rt.sync()
t0 = time.perf_counter()
for _ in range(5):
    wg.evaluate(tree, env, cfg, {}, result="device")
rt.sync()
print(f"group narrow keys, n={n}, WELDGPU_GROUP_U32={os.environ.get('WELDGPU_GROUP_U32', '1')}: "
      f"{(time.perf_counter() - t0) / 5 * 1e3:.2f} ms per evaluate")

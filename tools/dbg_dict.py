import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import runtime as rt, executor as ex, builders_dev as bd
from paper_1709_06416_b200 import workloads as W
from weldmill.engine import EngineConfig, Value
wl = W.WORKLOADS["dict"]
tree = W.compile_program(wl)
types = W.input_types(wl)
cols = W.device_columns(wl, wl.n)
env = {k: Value(types[k], v) for k, v in cols.items()}
cfg = EngineConfig(memory_limit=1 << 46)
orig = ex.Ctx._dict_aggregate
def spy(self, st, b):
    pc = np.empty(1 << b.extra["pbits"], dtype=np.uint64)
    rt.d2h(pc.ctypes.data, st.pcount.ptr, pc.nbytes)
    cnt = np.empty(2, dtype=np.uint64); rt.d2h(cnt.ctypes.data, st.counters.ptr, 16)
    print("pbits", b.extra["pbits"], "pcap", st.pcap, "cap", st.cap, "pcount sum", int(pc.sum()), "max", int(pc.max()),
          "min", int(pc.min()), "counters", cnt, "items", b, flush=True)
    return orig(self, st, b)
ex.Ctx._dict_aggregate = spy
for i in range(3):
    t0 = time.perf_counter(); wg.evaluate(tree, env, cfg, result="device"); rt.sync()
    print("eval", i, (time.perf_counter() - t0) * 1e3, "ms", flush=True)

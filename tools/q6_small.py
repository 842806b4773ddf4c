"""C1 (TPC-H Q6 at its 1M-row config size): host-visible time per evaluate()
with the launch replay on and off, and the device time of the loop kernel."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import executor, runtime as rt, workloads as W
from weldmill.engine import EngineConfig, Value

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
wl = W.WORKLOADS["q6"]
tree = W.compile_program(wl)
types = W.input_types(wl)
env = {k: Value(types[k], v) for k, v in W.device_columns(wl, n, 0).items()}
cfg = EngineConfig(memory_limit=1 << 46)
flush = rt.alloc(512 << 20)
for replay in (False, True):
    executor.REPLAY = replay
    executor._REPLAYS.d.clear()
    for _ in range(20):
        wg.evaluate(tree, env, cfg, result="device")
    rt.sync()
    for mode in ("hot", "flushed"):
        evs = [(rt.Event(), rt.Event()) for _ in range(200)]
        t0 = time.perf_counter()
        for a, b in evs:
            if mode == "flushed":
                rt.call("wg_flush_l2", flush.ptr, 512 << 20, 3)
            a.record()
            wg.evaluate(tree, env, cfg, result="device")
            b.record()
        rt.sync()
        wall = (time.perf_counter() - t0) / 200 * 1e6
        ev = sum(a.elapsed_ms(b) for a, b in evs) / 200 * 1e3
        rt.prof_enable(True)
        if mode == "flushed":
            rt.call("wg_flush_l2", flush.ptr, 512 << 20, 3)
        wg.evaluate(tree, env, cfg, result="device")
        rt.prof_enable(False)
        recs = [(nm, round(t * 1e3, 2)) for nm, t in rt.prof_records()]
        print(f"replay={replay} {mode}: event {ev:.1f} us/evaluate, wall {wall:.1f} us, kernels(us) {recs}")

#!/usr/bin/env python
"""Benchmark: one Weld IR program end to end on N B200s (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--n ROWS]
    python bench.py --impl reference ...      # the reference's CPU engine arm

A "step" is one evaluate() of the workload's IR program (BASELINE.json
configs; default configs[1] = Black-Scholes over 64M options) over one
batch of synthetic rows:

* value    -- rows/s over the whole job, inputs resident in HBM, results left
              in HBM; device time from CUDA events on the executor's stream,
              max over ranks.  Inputs are far larger than L2 (126 MB), so no
              flush is needed between steps (config.l2).
* e2e      -- the same metric through the public API with host inputs:
              pinned numpy columns -> evaluate(...) -> numpy results, host<->
              device copies inside the timed region.
* roofline -- algorithmic bytes of the dominant generated
              kernel / its event-timed duration, against MEASURED_PEAKS.json.
* cpu_baseline -- the reference engine (weldmill.engine.evaluate) on a
              bounded sample of the same rows, rank 0 at N=1 only.

Multi-GPU: rows are partitioned across ranks (rank r gets rows [r*n,
(r+1)*n)); the per-builder combine is exercised by paper_1709_06416_b200.
distributed.  Black-Scholes appends have no exchange step (the ordered
gather is a per-rank D2H into its offset), so the default workload is weak
scaling with no data-path collective.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rows/sec and achieved HBM GB/s (fraction of roofline) per IR program at 1/2/4/8 B200"


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    return rank, world


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic(workload):
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture summary (profiles/), or None."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_r*.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
            if workload in d and d[workload].get("dram_bytes") is not None:
                best = d[workload]
        except Exception:
            pass
    return best


def cpu_reference_rate(workload, target_s=10.0, threads=1):
    """Reference engine rows/s on a bounded sample of the same rows."""
    import paper_1709_06416_b200  # noqa: F401  (front end on sys.path)
    from paper_1709_06416_b200 import workloads as W
    from weldmill.engine import EngineConfig, Value, evaluate as ref_evaluate
    wl = W.WORKLOADS[workload]
    tree = W.compile_program(wl)
    types = W.input_types(wl)
    ext = W.externs_for(wl)

    def run(n):
        cols = W.host_columns(wl, n)
        env = {k: Value(types[k], v.tolist()) for k, v in cols.items()}
        t0 = time.perf_counter()
        ref_evaluate(tree, env, EngineConfig(threads=threads, memory_limit=1 << 45), ext)
        return time.perf_counter() - t0

    probe = 20000
    dt = run(probe)
    rate = probe / max(dt, 1e-9)
    n = int(min(max(rate * target_s, probe), 3_000_000))
    dt = run(n)
    return n / dt, n, dt


def reference_arm(args):
    rank, world = _dist()
    if rank != 0:
        return
    import paper_1709_06416_b200  # noqa: F401
    from paper_1709_06416_b200 import workloads as W
    from weldmill.engine import EngineConfig, Value, evaluate as ref_evaluate
    wl = W.WORKLOADS[args.workload]
    tree = W.compile_program(wl)
    types = W.input_types(wl)
    ext = W.externs_for(wl)
    threads = os.cpu_count() or 1
    # bounded sample per step: ~2 s of reference work
    rate1, _, _ = cpu_reference_rate(args.workload, target_s=1.0, threads=1)
    n = int(max(2000, min(rate1 * 2.0, 2_000_000)))
    cols = W.host_columns(wl, n)
    env = {k: Value(types[k], v.tolist()) for k, v in cols.items()}
    best = None
    for th in sorted({1, threads}):
        cfg = EngineConfig(threads=th, memory_limit=1 << 45)
        for _ in range(args.warmup):
            ref_evaluate(tree, env, cfg, ext)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ref_evaluate(tree, env, cfg, ext)
        dt = (time.perf_counter() - t0) / args.steps
        r = n / dt
        if best is None or r > best[0]:
            best = (r, th, dt)
    rate, th, dt = best
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic",
        "config": {"workload": args.workload, "rows_per_step": n, "program": wl.title},
        "cpu_baseline": {"value": rate, "unit": "rows/s", "cores": th, "kind": "reference",
                         "sample": f"weldmill.engine.evaluate, threads={th} (best of 1 and {threads}), "
                                   f"{n} generator rows per step"},
        "e2e": {"value": rate, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="blackscholes")
    ap.add_argument("--n", type=int, default=0, help="rows per GPU (default: the config's size)")
    ap.add_argument("--impl", default="weldgpu")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernel-timing", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        reference_arm(args)
        return

    rank, world = _dist()
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        ngpu = torch.cuda.device_count()
        torch.cuda.set_device(local % max(ngpu, 1))
        # one process per GPU over NCCL; more ranks than GPUs (a single-GPU
        # smoke of the multi-rank path) falls back to gloo for the barrier /
        # timing reductions -- the timed data path has no collective either way
        tdist.init_process_group("nccl" if ngpu >= world else "gloo")
        dist = tdist

    import numpy as np
    import paper_1709_06416_b200 as wg
    from paper_1709_06416_b200 import runtime as rt
    from paper_1709_06416_b200 import workloads as W
    from weldmill.engine import EngineConfig, Value

    wl = W.WORKLOADS[args.workload]
    n = args.n or wl.n
    tree = W.compile_program(wl)
    types = W.input_types(wl)
    ext = W.externs_for(wl)
    cfg = EngineConfig(memory_limit=1 << 46)
    row0 = rank * n

    dev_cols = W.device_columns(wl, n, row0)
    env = {k: Value(types[k], v) for k, v in dev_cols.items()}

    # per-launch timing of generated kernels (dominant kernel = most time)
    kern_times = {}
    pending = []

    ev_pool = [rt.Event() for _ in range(4 * args.steps + 16)]

    def hook(when, kern):
        ev = ev_pool.pop() if ev_pool else rt.Event()
        ev.record()
        if when == "before":
            pending.append((kern.name + ":" + str(kern.fn), ev))
        else:
            key, ev0 = pending.pop()
            kern_times.setdefault(key, []).append((ev0, ev))

    def barrier():
        if dist is not None:
            dist.barrier()

    # Warm-up mirrors the timed loop exactly (the previous step's result is
    # still alive while the next one allocates), so the allocator cache is
    # in steady state before timing starts.
    out = None
    for _ in range(args.warmup):
        out = wg.evaluate(tree, env, cfg, ext, result="device")
    rt.sync()

    clocks = Clocks(int(os.environ.get("LOCAL_RANK", "0"))) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.5)
    import gc
    gc.collect()
    gc.disable()          # no collector pauses inside the timed region
    # Inputs smaller than L2 (e.g. Q6 at its 1M-row config) would be served
    # from a warm L2: flush it (write 512 MB) between steps, outside the
    # per-step event pairs.
    alg_bytes = W.algorithmic_bytes(wl, n)
    flush = alg_bytes < (1 << 30)
    flush_buf = rt.alloc(512 << 20) if flush else None
    launches0 = rt.LAUNCHES[0]
    barrier()
    rt.sync()
    if flush:
        evs = [(rt.Event(), rt.Event()) for _ in range(args.steps)]
        for k in range(args.steps):
            rt.call("wg_flush_l2", flush_buf.ptr, 512 << 20, k + 1)
            evs[k][0].record()
            out = wg.evaluate(tree, env, cfg, ext, result="device")
            evs[k][1].record()
        rt.sync()
        ms = sum(a.elapsed_ms(b) for a, b in evs) / args.steps
        launches = rt.LAUNCHES[0] - launches0 - args.steps   # minus the flush kernels
    else:
        e0, e1 = rt.Event(), rt.Event()
        e0.record()
        for _ in range(args.steps):
            out = wg.evaluate(tree, env, cfg, ext, result="device")
        e1.record()
        rt.sync()
        launches = rt.LAUNCHES[0] - launches0
        ms = e0.elapsed_ms(e1) / args.steps
    # Per-kernel event timing in a second pass over the same steps (the
    # bracketing events would otherwise sit inside the headline region).
    if not args.no_kernel_timing:
        for k in range(args.steps):
            if flush:
                rt.call("wg_flush_l2", flush_buf.ptr, 512 << 20, 100 + k)
            rt.LAUNCH_HOOK[0] = hook
            out = wg.evaluate(tree, env, cfg, ext, result="device")
            rt.LAUNCH_HOOK[0] = None
        rt.sync()
    clk = clocks.stop() if clocks else None
    gc.enable()

    # dominant generated kernel
    dom_tot, dom_ms, dom_name = 0.0, 0.0, None
    for key, evs in kern_times.items():
        tot = sum(a.elapsed_ms(b) for a, b in evs)
        if tot > dom_tot:
            dom_tot, dom_ms, dom_name = tot, tot / len(evs), key
    del kern_times

    if dist is not None:
        import torch
        t = torch.tensor([ms, dom_ms], dtype=torch.float64, device=_coll_dev(dist))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, dom_ms = float(t[0]), float(t[1])

    rows = n * world
    value = rows / (ms / 1e3)
    peak, peak_kind = _peaks()
    alg = W.algorithmic_bytes(wl, n)
    achieved = alg / (dom_ms / 1e3) / 1e9 if dom_ms else None
    tr = _traffic(args.workload)

    # ---- e2e through the public API with host buffers ----------------------
    e2e = None
    if not args.no_e2e:
        host = W.host_columns(wl, n, row0)
        for arr in host.values():
            rt.host_register(arr)
        henv = {k: Value(types[k], v) for k, v in host.items()}
        h2d = sum(a.nbytes for a in host.values())
        d2h = 0
        # same warm-up discipline as the device loop: keep the previous result
        # alive so the pinned result pool reaches steady state before timing
        res = None
        for _ in range(max(3, args.warmup)):
            res = wg.evaluate(tree, henv, cfg, ext, result="numpy")[0].data
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            res = wg.evaluate(tree, henv, cfg, ext, result="numpy")[0].data
        el = (time.perf_counter() - t0) / args.e2e_steps
        d2h = _nbytes(res)
        if dist is not None:
            import torch
            t = torch.tensor([el], dtype=torch.float64, device=_coll_dev(dist))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t[0])
        e2e = {"value": rows / el, "unit": "rows/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": el * 1e3}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, ncpu, dt = cpu_reference_rate(args.workload, target_s=10.0, threads=1)
        cpu = {"value": rate, "unit": "rows/s", "cores": 1, "kind": "reference",
               "sample": f"weldmill.engine.evaluate (threads=1; its GIL-bound pool does not scale, "
                         f"BASELINE.md) on the first {ncpu} generator rows of the same workload, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic",
            "config": {"workload": args.workload, "program": wl.title, "rows_per_gpu": n,
                       "global_rows": rows, "parallelism": f"row-partitioned x{world}",
                       "l2": "inputs >> L2 (126 MB); no flush needed" if not flush else
                             "L2 flushed (512 MB write) before every step, outside the per-step events"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": (tr["dram_bytes"] * (n / tr["n"]) if tr else None),
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                         "kernel": dom_name.split(":")[0] if dom_name else None, "kernel_ms": dom_ms,
                         "algorithmic_bytes": alg},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def _coll_dev(dist):
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def _nbytes(v):
    import numpy as np
    if isinstance(v, np.ndarray) or hasattr(v, "offsets"):
        return v.nbytes
    if isinstance(v, (tuple, list)):
        return sum(_nbytes(x) for x in v)
    return 8


if __name__ == "__main__":
    main()

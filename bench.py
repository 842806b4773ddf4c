#!/usr/bin/env python
"""Benchmark: the Weld IR programs of BASELINE.json on N B200s (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--rows ROWS]
    python bench.py --impl reference ...      # the reference's CPU engine arm

A "step" is one evaluate() of a workload's IR program (BASELINE.json
configs) over one batch of synthetic rows.  The headline line is
configs[1], Black-Scholes over 64M options; the same line carries a
``per_config`` block with every other config measured the same way
(C1 Q6 at 1M and 600M rows, C3 Q1, C4a dictmerger, C4b groupbuilder,
C5 vecmerger histogram, plus the two appender scans).

Per workload:
* value        rows/s over the whole job, inputs resident in HBM, results
               left in HBM; device time from CUDA events on the executor's
               stream around the K steps, max over ranks.  Inputs >> L2
               (126 MB), except C1 at 1M rows, which flushes L2 (512 MB
               write) before every step, outside the per-step events.
* roofline     algorithmic bytes per step / the device time
               of ALL kernels of the step (every launch bracketed by events
               inside libweldgpu, wg_prof_*), against MEASURED_PEAKS.json;
               the dominant kernel and its share are named; step_frac uses
               the whole step (host gaps included).
* e2e          the same metric through the public API with HOST buffers:
               pinned numpy columns -> evaluate(..., result="numpy") ->
               numpy results; host<->device copies inside the timed region.
* cpu_baseline the reference engine (weldmill.engine.evaluate) on a bounded
               sample of the same generator rows, rank 0 at N=1 only.

Multi-GPU (--gpus N; re-launches itself under torch.distributed.run when
WORLD_SIZE is not set): STRONG scaling -- the config's global rows are split
into contiguous shards (distributed.shard_bounds), each rank evaluates its
shard and the per-builder combine runs inside the timed region
(distributed.evaluate_sharded over NCCL from libweldgpu: merger all-gather +
rank-order fold kernel, appender count all-gather, vecmerger slice
all-to-all + rank-order fold + all-gather, dictmerger / groupbuilder range-
partitioned all-to-all + device merge).
"""
from __future__ import annotations

import argparse
import gc
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

# (label, workload, rows or 0 = the config's own size, e2e row cap)
PER_CONFIG = [
    ("C1_q6_1M", "q6", 0, None),
    ("C1_q6_600M", "q6", 600_000_000, 200_000_000),
    ("C2_blackscholes_64M", "blackscholes", 0, None),
    ("C3_q1_60M", "q1", 0, None),
    ("C4a_dict_200M", "dict", 0, None),
    ("C4b_group_200M", "group", 0, None),
    ("C5_hist_1B", "hist", 0, 200_000_000),
    ("appender_filter_500M", "filter", 0, 200_000_000),
    ("appender_map_500M", "map", 0, 200_000_000),
]


# scattered 8-byte L2 REDs per second on B200 into an L2-resident target (profiles/red_peak_r02.txt)
RED_PEAK = 1.86e11


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
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(workload, n):
    """DRAM bytes per step from the committed ncu capture summary
    (profiles/ncu_summary_r*.json, latest round wins), scaled to n rows."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_r*.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
            e = d.get(workload)
            if e and e.get("dram_bytes_step") is not None:
                best = e["dram_bytes_step"] * (n / e["n"])
            elif e and e.get("dram_bytes") is not None:
                best = e["dram_bytes"] * (n / e["n"])
        except Exception:
            pass
    return best


# ---------------------------------------------------------------------------
# reference CPU engine


def cpu_reference_rate(workload, target_s=10.0, threads=1, cap=3_000_000):
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
    n = int(min(max(rate * target_s, probe), cap))
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
        "scaling": "strong", "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic",
        "config": {"workload": args.workload, "rows_per_step": n, "program": wl.title},
        "cpu_baseline": {"value": rate, "unit": "rows/s", "cores": th, "kind": "reference",
                         "sample": f"weldmill.engine.evaluate, threads={th} (best of 1 and {threads}), "
                                   f"{n} generator rows per step"},
        "e2e": {"value": rate, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# one workload on this rank


class Runner:
    def __init__(self, dist, rank, world):
        self.dist = dist
        self.rank = rank
        self.world = world
        import paper_1709_06416_b200 as wg
        from paper_1709_06416_b200 import distributed as D, runtime as rt, workloads as W
        self.wg, self.D, self.rt, self.W = wg, D, rt, W
        self.comm = D.device_comm() if world > 1 else None

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max_over_ranks(self, *vals):
        if self.dist is None:
            return vals
        import torch
        t = torch.tensor(list(vals), dtype=torch.float64, device=_coll_dev(self.dist))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return tuple(float(x) for x in t.tolist())

    def evaluate(self, tree, env, cfg, ext, result):
        if self.world == 1:
            return self.wg.evaluate(tree, env, cfg, ext, result=result)[0].data
        return self.D.evaluate_sharded(tree, env, cfg, ext, comm=self.comm, row0=self.row0,
                                       n_total=self.n_total, result=result)

    def run(self, name, n_total, steps, warmup, e2e_cap=None, e2e_steps=3, do_e2e=True, do_cpu=True,
            kernel_timing=True, clocks=None):
        from weldmill.engine import EngineConfig, Value
        W, rt = self.W, self.rt
        wl = W.WORKLOADS[name]
        n_total = n_total or wl.n
        lo, hi = self.D.shard_bounds(n_total, self.rank, self.world)
        self.row0, self.n_total = lo, n_total
        n = hi - lo
        tree = W.compile_program(wl)
        types = W.input_types(wl)
        ext = W.externs_for(wl)
        cfg = EngineConfig(memory_limit=1 << 46)
        dev_cols = W.device_columns(wl, n, lo)
        env = {k: Value(types[k], v) for k, v in dev_cols.items()}

        out = None
        for _ in range(warmup):
            out = self.evaluate(tree, env, cfg, ext, "device")
        rt.sync()
        alg = W.algorithmic_bytes(wl, n_total)
        flush = alg < (1 << 30)
        flush_buf = rt.alloc(512 << 20) if flush else None
        gc.collect()
        gc.disable()          # no collector pauses inside the timed region
        if clocks:
            clocks.start()
            time.sleep(0.3)
        self.barrier()
        rt.sync()
        if flush:
            evs = [(rt.Event(), rt.Event()) for _ in range(steps)]
            for k in range(steps):
                rt.call("wg_flush_l2", flush_buf.ptr, 512 << 20, k + 1)
                evs[k][0].record()
                out = self.evaluate(tree, env, cfg, ext, "device")
                evs[k][1].record()
            rt.sync()
            ms = sum(a.elapsed_ms(b) for a, b in evs) / steps
        else:
            e0, e1 = rt.Event(), rt.Event()
            e0.record()
            for _ in range(steps):
                out = self.evaluate(tree, env, cfg, ext, "device")
            e1.record()
            rt.sync()
            ms = e0.elapsed_ms(e1) / steps
        self.barrier()
        clk = clocks.stop() if clocks else None
        # cold call: the per-loop dictmerger hints forgotten (the variant is
        # chosen again from the first rows' distinct count); kernels compiled
        from paper_1709_06416_b200 import builders_dev as _bd
        _bd._SIZE_HINTS.clear()
        c0, c1 = rt.Event(), rt.Event()
        if flush:
            rt.call("wg_flush_l2", flush_buf.ptr, 512 << 20, 77)
        c0.record()
        out = self.evaluate(tree, env, cfg, ext, "device")
        c1.record()
        rt.sync()
        cold_ms = c0.elapsed_ms(c1)
        # Per-kernel device time in a second pass over the same steps (the
        # per-launch events would otherwise sit inside the headline region).
        kern = {}
        launches = None
        if kernel_timing:
            for k in range(steps):
                if flush:
                    rt.call("wg_flush_l2", flush_buf.ptr, 512 << 20, 100 + k)
                rt.prof_enable(True)
                out = self.evaluate(tree, env, cfg, ext, "device")
                rt.prof_enable(False)
                recs = rt.prof_records()
                for nm, t in recs:
                    a = kern.setdefault(nm, [0.0, 0])
                    a[0] += t
                    a[1] += 1
            launches = sum(c for nm, (t, c) in kern.items() if nm not in ("memset", "memcpy_d2d")) / steps
        gc.enable()
        del out
        step_kern_ms = sum(t for t, c in kern.values()) / steps if kern else None
        dom = max(kern.items(), key=lambda kv: kv[1][0]) if kern else None
        ms, step_kern_ms_max = self.max_over_ranks(ms, step_kern_ms or 0.0)
        if step_kern_ms is not None:
            step_kern_ms = step_kern_ms_max
        value = n_total / (ms / 1e3)
        peak, peak_src = _peaks()
        achieved = alg / (step_kern_ms / 1e3) / 1e9 if step_kern_ms else None
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": _traffic(name, n_total), "peak_source": peak_src,
                "basis": "algorithmic bytes / device time of every kernel in the step (wg_prof events)",
                "algorithmic_bytes": alg, "step_kernel_ms": step_kern_ms,
                "step_frac": alg / (ms / 1e3) / 1e9 / peak}
        if name == "hist" and step_kern_ms:
            # C5 is bound by the L2 reduction units, not HBM: one scattered
            # RED per row at the measured ceiling (tools/red_peak.cu,
            # profiles/red_peak_r02.txt)
            floor = n_total / RED_PEAK * 1e3
            roof["ceiling"] = {"bound": "l2-red", "peak": RED_PEAK, "unit": "RED/s", "floor_ms": floor,
                               "frac": floor / step_kern_ms, "source": "profiles/red_peak_r02.txt"}
        if dom:
            roof["kernel"] = dom[0]
            roof["kernel_ms"] = dom[1][0] / steps
            roof["kernel_share"] = dom[1][0] / steps / step_kern_ms if step_kern_ms else None
            roof["kernels"] = [{"name": nm, "ms_per_step": t / steps, "launches_per_step": c / steps}
                               for nm, (t, c) in sorted(kern.items(), key=lambda kv: -kv[1][0])[:8]]
        del env, dev_cols
        if flush_buf is not None:
            del flush_buf
        gc.collect()
        rt.call("wg_mem_trim")

        (cold_ms,) = self.max_over_ranks(cold_ms)
        res = {"value": value, "unit": "rows/s", "ms_per_step": ms, "cold_ms_per_step": cold_ms,
               "rows": n_total, "rows_per_gpu": n,
               "roofline": roof, "gpu_launches": launches, "clocks": clk,
               "l2": ("L2 flushed (512 MB write) before every step, outside the per-step events" if flush
                      else "inputs >> L2 (126 MB); no flush needed")}

        # ---- e2e through the public API with host buffers ----------------
        if do_e2e:
            ne = min(n_total, e2e_cap) if e2e_cap else n_total
            elo, ehi = self.D.shard_bounds(ne, self.rank, self.world)
            self.row0, self.n_total = elo, ne
            host = host_columns_pinned(W, wl, ehi - elo, elo)
            henv = {k: Value(types[k], v) for k, v in host.items()}
            h2d = sum(a.nbytes for a in host.values())
            r = None
            for _ in range(max(2, warmup)):
                r = self.evaluate(tree, henv, cfg, ext, "numpy")
            del r
            self.barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                r = self.evaluate(tree, henv, cfg, ext, "numpy")
            el = (time.perf_counter() - t0) / e2e_steps
            d2h = _nbytes(r)
            del r
            (el,) = self.max_over_ranks(el)
            res["e2e"] = {"value": ne / el, "unit": "rows/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                          "ms_per_step": el * 1e3, "rows": ne,
                          "inputs": "pinned host numpy columns (the step copies them in and the result out)"}
            del host, henv
            gc.collect()
            rt.call("wg_mem_trim")
        if do_cpu and self.rank == 0 and self.world == 1:
            rate, ncpu, dt = cpu_reference_rate(name, target_s=3.0 if n_total != wl.n or name != "blackscholes"
                                                else 10.0, threads=1)
            res["cpu_baseline"] = {"value": rate, "unit": "rows/s", "cores": 1, "kind": "reference",
                                   "sample": f"weldmill.engine.evaluate (threads=1; its GIL-bound pool does not "
                                             f"scale, BASELINE.md) on the first {ncpu} generator rows of the same "
                                             f"workload, {dt:.1f} s"}
        return res


def host_columns_pinned(W, wl, n, row0):
    """The workload's columns in pinned host memory: generated on the device
    (identical bits to the numpy generator) and copied down once."""
    from paper_1709_06416_b200.columns import pinned_empty
    from paper_1709_06416_b200.irtypes import NPTYPE
    from paper_1709_06416_b200 import runtime as rt
    dev = W.device_columns(wl, n, row0)
    out = {}
    for k, dv in dev.items():
        c = dv.cols[0]
        a = pinned_empty(dv.n, NPTYPE[c.kind])
        if dv.n:
            rt.d2h(a.ctypes.data, c.ptr, a.nbytes)
        out[k] = a
    return out


def _coll_dev(dist):
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def _nbytes(v):
    import numpy as np
    if isinstance(v, dict):      # a combined builder part (distributed.to_numpy_part)
        return sum(_nbytes(x) for k, x in v.items() if k in ("cols", "keys", "vals", "offsets"))
    if isinstance(v, np.ndarray) or hasattr(v, "offsets"):
        if hasattr(v, "offsets"):
            return v.offsets.nbytes + _nbytes(v.values)
        return v.nbytes
    if isinstance(v, (tuple, list)):
        return sum(_nbytes(x) for x in v)
    return 8


def _relaunch(args):
    """--gpus N without a torchrun environment: re-launch this script as N
    ranks (one process per GPU) and pass rank 0's JSON line through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + os.getpid() % 1000}", os.path.abspath(__file__)]
    # (torchrun's parser would read "--n" as an abbreviation of its own options)
    cmd += ["--rows" + a[3:] if a == "--n" or a.startswith("--n=") else a for a in sys.argv[1:]]
    rc = subprocess.call(cmd)
    sys.exit(rc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="blackscholes")
    ap.add_argument("--rows", "--n", dest="n", type=int, default=0, help="global rows (default: the config's size)")
    ap.add_argument("--impl", default="weldgpu")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernel-timing", action="store_true")
    ap.add_argument("--per-config", default="all", help="all | none | comma list of PER_CONFIG labels")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        reference_arm(args)
        return

    rank, world = _dist()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU")
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        ngpu = torch.cuda.device_count()
        torch.cuda.set_device(local % max(ngpu, 1))
        tdist.init_process_group("nccl" if ngpu >= world else "gloo")
        dist = tdist

    runner = Runner(dist, rank, world)
    wl = runner.W.WORKLOADS[args.workload]
    clocks = Clocks(int(os.environ.get("LOCAL_RANK", "0"))) if rank == 0 else None
    head = runner.run(args.workload, args.n or wl.n, args.steps, args.warmup, e2e_steps=args.e2e_steps,
                      do_e2e=not args.no_e2e, do_cpu=not args.no_cpu, kernel_timing=not args.no_kernel_timing,
                      clocks=clocks)
    per = {}
    if args.per_config != "none" and world == 1:
        want = None if args.per_config == "all" else set(args.per_config.split(","))
        for label, name, rows, cap in PER_CONFIG:
            if want is not None and label not in want:
                continue
            if name == args.workload and (rows or runner.W.WORKLOADS[name].n) == (args.n or wl.n):
                per[label] = {k: v for k, v in head.items() if k != "clocks"}
                per[label]["workload"] = name
                continue
            r = runner.run(name, rows, args.steps, args.warmup, e2e_cap=cap, e2e_steps=args.e2e_steps,
                           do_e2e=not args.no_e2e, do_cpu=not args.no_cpu,
                           kernel_timing=not args.no_kernel_timing)
            r["workload"] = name
            r["program"] = runner.W.WORKLOADS[name].title
            per[label] = r

    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "cold_ms_per_step": head["cold_ms_per_step"],
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic",
            "config": {"workload": args.workload, "program": wl.title, "global_rows": head["rows"],
                       "rows_per_gpu": head["rows_per_gpu"], "parallelism": f"row-partitioned x{world}",
                       "l2": head["l2"]},
            "roofline": head["roofline"],
            "cpu_baseline": head.get("cpu_baseline"),
            "e2e": head.get("e2e"),
            "gpu_launches": head["gpu_launches"],
            "clocks": head["clocks"],
            "per_config": per,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

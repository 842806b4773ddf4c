"""Summarise a gpurun_out/prof capture set into profiles/ (committed).

    python tools/summarize_profiles.py gpurun_out/prof r01

Writes profiles/ncu_summary_<round>.json (per workload: duration, DRAM bytes,
throughputs, occupancy, registers, top stall reasons, SASS evidence) and
profiles/ncu_summary_<round>.md, plus the launch list of the default bench.
"""
import csv
import glob
import json
import os
import subprocess
import sys

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof"
RND = sys.argv[2] if len(sys.argv) > 2 else "r01"
OUT = "profiles"
os.makedirs(OUT, exist_ok=True)

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
       "launch__shared_mem_per_block_dynamic",
       # L2 reduction / atomic traffic from the SMs (the metric names the --set full capture holds)
       "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed",
       "lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum",
       "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_atom.sum.pct_of_peak_sustained_elapsed",
       "lts__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
       "lts__t_sector_hit_rate.pct"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return {}
    h, units, vals = rows[0], rows[1], rows[2]
    d = {"Kernel Name": (vals[h.index("Kernel Name")], "")} if "Kernel Name" in h else {}
    stalls = []
    for i, c in enumerate(h):
        if c in RAW:
            d[c] = (vals[i], units[i])
        if c.startswith("smsp__average_warps_issue_stalled") and c.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(vals[i]), c[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    d["stalls"] = [(n, round(v, 2)) for v, n in sorted(stalls, reverse=True)[:5]]
    return d


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return float(v.replace(",", "")) * scale


def to_ms(v, u):
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
             "second": 1e3, "s": 1e3}.get(u, 1)
    return float(v.replace(",", "")) * scale


summary = {}
for rep in sorted(glob.glob(os.path.join(SRC, "full_*.ncu-rep"))):
    w = os.path.basename(rep)[len("full_"):-len(".ncu-rep")]
    r = raw(rep)
    if not r:
        continue
    dur = to_ms(*r["gpu__time_duration.sum"])
    dram = to_bytes(*r["dram__bytes_read.sum"]) + to_bytes(*r["dram__bytes_write.sum"])
    bench = {}
    bj = os.path.join(SRC, f"bench_{w}.json")
    if os.path.exists(bj):
        try:
            bench = json.loads(open(bj).read().strip().splitlines()[-1])
        except Exception:
            bench = {}
    rows = (bench.get("config") or {}).get("rows_per_gpu")
    summary[w] = {
        "kernel": (r.get("Kernel Name", ("wg_loop",))[0][:60] + (" (NVRTC, sm_100a)" if r.get("Kernel Name", ("wg_",))[0].startswith("wg_") else " (libweldgpu, sm_100a)")),
        "n": rows,
        "ncu_duration_ms": round(dur, 4),
        "dram_bytes": dram,
        "dram_read_bytes": to_bytes(*r["dram__bytes_read.sum"]),
        "dram_write_bytes": to_bytes(*r["dram__bytes_write.sum"]),
        "dram_throughput_pct": float(r.get("dram__cycles_active.avg.pct_of_peak_sustained_elapsed", ("nan",))[0] or "nan"),
        "sm_throughput_pct": float(r["sm__throughput.avg.pct_of_peak_sustained_elapsed"][0]),
        "issue_active_pct": float(r.get("sm__issue_active.avg.pct_of_peak_sustained_elapsed", ("nan",))[0]),
        "fp64_pipe_pct": float(r.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", ("nan",))[0]),
        "warps_active_pct": float(r["sm__warps_active.avg.pct_of_peak_sustained_active"][0]),
        "registers": int(float(r["launch__registers_per_thread"][0])),
        "grid": int(float(r["launch__grid_size"][0])),
        "dyn_smem_bytes": r.get("launch__shared_mem_per_block_dynamic", ("0",))[0],
        "l2_red_sectors": r.get("lts__t_sectors_srcunit_tex_op_red.sum", ("0",))[0],
        "l2_red_pct_of_peak": r.get("lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed", ("0",))[0],
        "l2_red_lookup_miss_sectors": r.get("lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum", ("0",))[0],
        "l2_atom_sectors": r.get("lts__t_sectors_srcunit_tex_op_atom.sum", ("0",))[0],
        "l2_atom_pct_of_peak": r.get("lts__t_sectors_srcunit_tex_op_atom.sum.pct_of_peak_sustained_elapsed", ("0",))[0],
        "l2_throughput_pct": r.get("lts__throughput.avg.pct_of_peak_sustained_elapsed", ("0",))[0],
        "top_stalls": r["stalls"],
        "bench_roofline": bench.get("roofline"),
        "bench_value_rows_per_s": bench.get("value"),
        "bench_ms_per_step": bench.get("ms_per_step"),
    }

with open(os.path.join(OUT, f"ncu_summary_{RND}.json"), "w") as f:
    json.dump(summary, f, indent=1)

lines = [f"# ncu summary ({RND}) -- one `ncu --set full --clock-control none` capture of each workload's loop kernel",
         "", "Device: B200 (sm_100a). ncu times are cold-cache and serialised (replay); bench times are live CUDA events.",
         "", "| workload | kernel | rows | ncu ms | DRAM GB (r+w) | DRAM % | SM % | FP64 % | L2 RED sectors (% peak) | L2 ATOM sectors (% peak) | warps % | regs | bench kernel ms | roofline frac | top stalls |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for w, s in summary.items():
    rf = s["bench_roofline"] or {}
    def _f(x):
        try:
            return float(str(x).replace(",", ""))
        except ValueError:
            return 0.0
    lines.append(f"| {w} | `{s['kernel'].split(' (')[0][:28]}` | {s['n']} | {s['ncu_duration_ms']:.3f} | {s['dram_bytes']/1e9:.2f} | "
                 f"{s['dram_throughput_pct']:.0f} | {s['sm_throughput_pct']:.0f} | {s['fp64_pipe_pct']:.0f} | "
                 f"{_f(s['l2_red_sectors']):.3g} ({_f(s['l2_red_pct_of_peak']):.0f}%) | {_f(s['l2_atom_sectors']):.3g} ({_f(s['l2_atom_pct_of_peak']):.0f}%) | "
                 f"{s['warps_active_pct']:.0f} | {s['registers']} | "
                 f"{(rf.get('kernel_ms') or 0):.3f} | {(rf.get('frac') or 0):.3f} | "
                 + ", ".join(f"{n}={v}" for n, v in s["top_stalls"][:3]) + " |")

# launch list of the default bench
ll = os.path.join(SRC, "launches_default.csv")
if os.path.exists(ll):
    rows = [r for r in csv.reader(open(ll)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = {}
    for r in rows[1:]:
        tot.setdefault(r[ki][:60], []).append(to_ms(r[vi], r[ui]))
    lines += ["", "## Launch list of the headline bench (`bench.py --steps 3 --warmup 3 --per-config none`: input generation + 3 warm-up + 3 timed steps)", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    allt = sum(sum(v) for v in tot.values())
    for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v):.3f} | {100*sum(v)/allt:.1f}% |")
    with open(os.path.join(OUT, f"launches_default_{RND}.csv"), "w") as f:
        f.write(open(ll).read())

# one step of each workload: every launch of the last evaluate (ncu launch list)
step_lists = {}
for ll in sorted(glob.glob(os.path.join(SRC, "launches_*.csv"))):
    w = os.path.basename(ll)[len("launches_"):-len(".csv")]
    if w == "default":
        continue
    rows = [r for r in csv.reader(open(ll)) if len(r) > 10]
    if len(rows) < 2:
        continue
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    ks = [(r[ki], to_ms(r[vi], r[ui])) for r in rows[1:]]
    starts = [i for i, (k, _) in enumerate(ks) if k.startswith("wg_loop") and (i == 0 or not ks[i - 1][0].startswith("wg_loop"))]
    last = ks[starts[-1]:] if starts else ks
    first = next((i for i, (k, _) in enumerate(ks) if k.startswith("wg_loop")), 0)
    if all(k.startswith("wg_loop") for k, _ in ks[first:]):
        last = ks[-1:]                  # one loop kernel per evaluate (the rest is input generation)
    step_lists[w] = last
    with open(os.path.join(OUT, f"launches_{w}_{RND}.csv"), "w") as f:
        f.write(open(ll).read())
if step_lists:
    lines += ["", "## One evaluate() step per workload (ncu launch list, cold-cache, serialised)", ""]
    for w, last in step_lists.items():
        tot = sum(t for _, t in last)
        lines += [f"### {w}: {len(last)} launches, {tot:.3f} ms", "", "| kernel | ms | share |", "|---|---|---|"]
        for k, t in last:
            lines.append(f"| `{k[:70]}` | {t:.3f} | {100 * t / tot:.1f}% |")
        lines.append("")
summary["step_launch_lists"] = {w: [[k[:70], round(t, 4)] for k, t in last] for w, last in step_lists.items()}
with open(os.path.join(OUT, f"ncu_summary_{RND}.json"), "w") as f:
    json.dump(summary, f, indent=1)

with open(os.path.join(OUT, f"ncu_summary_{RND}.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))

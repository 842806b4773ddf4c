"""One-screen summary of an `ncu --set full` report: duration, DRAM traffic,
L2 RED/ATOM sector throughput (srcunit_tex, the metrics the capture holds),
hit rates, occupancy, issue activity and the top warp-stall reasons.

    python tools/ncu_brief.py gpurun_out/p2/full_hist.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "dram_rd%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_thru%"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "l2_red_sect"),
    ("lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed", "l2_red%"),
    ("lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum", "l2_red_miss"),
    ("lts__t_sectors_srcunit_tex_op_atom.sum", "l2_atom_sect"),
    ("lts__t_sectors_srcunit_tex_op_atom.sum.pct_of_peak_sustained_elapsed", "l2_atom%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_thru%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1_thru%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy%"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("launch__occupancy_limit_registers", "occ_lim_regs"),
    ("launch__occupancy_limit_shared_mem", "occ_lim_smem"),
]


def brief(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {"error": "no rows"}
    h, u = rows[0], rows[1]
    res = {}
    for row in rows[2:]:
        d = dict(zip(h, zip(row, u)))
        name = d.get("Kernel Name", ("?", ""))[0]
        r = {"kernel": name}
        for k, short in KEYS:
            if k in d:
                v, unit = d[k]
                r[short] = f"{v} {unit}".strip()
        stalls = []
        for k, (v, _) in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        r["stalls"] = ", ".join(f"{n} {v:.1f}" for v, n in stalls[:6])
        res.setdefault(name, r)
    return res


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        for name, r in brief(rep).items():
            for k, v in r.items():
                print(f"  {k:14s} {v}")

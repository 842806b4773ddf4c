"""One-line summary of bench.py JSON lines: python tools/bline.py file..."""
import json, sys
for path in sys.argv[1:]:
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        try:
            d = json.loads(line)
        except Exception:
            continue
        r = d.get("roofline") or {}
        e = d.get("e2e") or {}
        c = d.get("cpu_baseline") or {}
        print("%-13s value %.3g rows/s | kernel %s %.3f ms frac %.3f | step %.3f ms | e2e %.3g rows/s (%.1f ms) | cpu %s | launches %s | clocks %s" % (
            d["config"]["workload"], d["value"], r.get("kernel"), r.get("kernel_ms") or 0, r.get("frac") or 0,
            d["ms_per_step"], e.get("value", 0), e.get("ms_per_step", 0), c.get("value"), d.get("gpu_launches"),
            (d.get("clocks") or {}).get("sm_mhz")))

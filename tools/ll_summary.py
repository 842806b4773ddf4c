"""Print the launch list (ncu gpu__time_duration) of the LAST bench step."""
import csv, sys
path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
ks = [(r[ki], float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "nsecond" else (1e3 if r[ui] == "msecond" else 1.0))) for r in rows[1:]]
# split into steps at each wg_loop launch that follows a non-loop launch
starts = [i for i, (k, _) in enumerate(ks) if k.startswith("wg_loop") and (i == 0 or not ks[i - 1][0].startswith("wg_loop"))]
last = ks[starts[-1]:] if starts else ks
tot = sum(t for _, t in last)
print(f"{path}: {len(ks)} launches, last step {len(last)} launches, {tot:.1f} us")
for k, t in last:
    print(f"  {t:9.1f} us  {100*t/tot:5.1f}%  {k[:90]}")

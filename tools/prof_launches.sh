# per-launch device times for one step of each workload (cold-cache, serialised)
for w in "$@"; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv \
     python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > /dev/null 2>&1
  python - "$w" <<'PY'
import csv, sys, collections
w = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/launches_{w}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
ks = [(r[ki], float(r[vi]) * (1e-3 if r[ui] == "nsecond" else 1.0)) for r in rows[1:]]
# last step: everything after the 4th wg_loop-containing step start is hard to segment; print the tail
tot = collections.OrderedDict()
for k, t in ks[-40:]:
    tot[k[:70]] = tot.get(k[:70], 0) + t
print(w, "last-40-launch totals (us):")
for k, t in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print("   %10.1f  %s" % (t, k))
PY
done

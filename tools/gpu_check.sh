# GPU test suite + one-line device bench per workload
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
for w in ${WORKLOADS:-blackscholes q6 q1 dict group hist}; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c 'import sys,json
try:
    d=json.loads(sys.stdin.read()); r=d["roofline"]
    print("%-13s kernel_ms %.3f frac %.3f step_ms %.3f launches %d" % (d["config"]["workload"], r["kernel_ms"], r["frac"], d["ms_per_step"], d["gpu_launches"]))
except Exception as e: print("bench failed", e)'
done

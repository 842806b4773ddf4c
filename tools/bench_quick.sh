python tools/step_gap.py blackscholes
for w in blackscholes q6 hist; do
python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["config"]["workload"], "kernel_ms %.3f" % r["kernel_ms"], "frac %.3f" % r["frac"], "step_ms %.3f" % d["ms_per_step"], d["clocks"])'
done
python bench.py --workload q6 --n 600000000 --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["config"]["workload"], "600M kernel_ms %.3f" % r["kernel_ms"], "frac %.3f" % r["frac"], "step_ms %.3f" % d["ms_per_step"], d["clocks"])'

for f in "" "--no-kernel-timing"; do
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e $f 2>&1 | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms", r["kernel_ms"], "step_ms %.3f" % d["ms_per_step"], d["clocks"])'
done
python tools/step_gap.py blackscholes

# knob sweep for the Black-Scholes loop kernel (device-timed, no e2e/cpu)
for pf in 0 1; do for mb in 0 5 6 8; do for it in 1 2 4; do
  r=$(WELDGPU_PREFETCH=$pf WELDGPU_MINBLOCKS=$mb WELDGPU_ITEMS=$it timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1)
  echo "pf=$pf mb=$mb items=$it $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms %.3f frac %.3f step_ms %.3f" % (r["kernel_ms"], r["frac"], d["ms_per_step"]))' 2>&1 | tail -1)"
done; done; done

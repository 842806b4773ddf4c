for it in 2 4 8 16; do
  r=$(WELDGPU_ITEMS=$it timeout 200 python bench.py --workload dict --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1)
  echo "dict items=$it $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms %.3f frac %.3f step %.3f" % (r["kernel_ms"], r["frac"], d["ms_per_step"]))' 2>&1 | tail -1)"
done

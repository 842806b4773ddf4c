for it in 8 16; do for st in 0 1; do
  r=$(WELDGPU_STAGE_SCAN=$st WELDGPU_ITEMS=$it timeout 200 python bench.py --workload filter --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1)
  echo "filter pipe items=$it stage=$st $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms %.3f frac %.3f" % (r["kernel_ms"], r["frac"]))' 2>&1 | tail -1)"
done; done

for w in q1 dict; do
  for it in 1 2 4 8; do for rc in 0 2 4; do
    if [ $w = q1 ] && [ $it -gt 2 ]; then continue; fi
    r=$(WELDGPU_ITEMS=$it WELDGPU_REGCACHE=$rc timeout 200 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1)
    echo "$w items=$it rc=$rc $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms %.3f frac %.3f step_ms %.3f" % (r["kernel_ms"], r["frac"], d["ms_per_step"]))' 2>&1 | tail -1)"
  done; done
done

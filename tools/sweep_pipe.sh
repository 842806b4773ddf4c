for w in blackscholes q6 q1 dict group hist; do
  for pipe in 0 1; do
    extra=""
    if [ $w = q6 ]; then extra="--n 600000000"; fi
    r=$(WELDGPU_PIPE=$pipe timeout 200 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e $extra 2>&1 | tail -1)
    echo "$w pipe=$pipe $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms %.3f frac %.3f step_ms %.3f" % (r["kernel_ms"], r["frac"], d["ms_per_step"]))' 2>&1 | tail -1)"
  done
done

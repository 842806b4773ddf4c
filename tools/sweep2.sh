one() {
  w=$1; shift
  r=$(env "$@" timeout 200 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1)
  echo "$w $* => $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms %.3f frac %.3f step_ms %.3f" % (r["kernel_ms"], r["frac"], d["ms_per_step"]))' 2>&1 | tail -1)"
}
for st in 2 3; do for bud in 45000 65536; do one blackscholes WELDGPU_PIPE_STAGES=$st WELDGPU_PIPE_SMEM=$bud; done; done
one blackscholes WELDGPU_PIPE=1 WELDGPU_ITEMS=1
one blackscholes WELDGPU_PIPE=1 WELDGPU_ITEMS=4
for it in 1 2; do for rc in 0 4; do one q1 WELDGPU_ITEMS=$it WELDGPU_REGCACHE=$rc; one dict WELDGPU_ITEMS=$it WELDGPU_REGCACHE=$rc; done; done

one() { r=$(env "$@" timeout 200 python bench.py --workload dict --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1)
  echo "dict $* $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms %.3f step %.3f" % (r["kernel_ms"], d["ms_per_step"]))' 2>&1 | tail -1)"; }
one WELDGPU_PIPE=0
one WELDGPU_PIPE=0 WELDGPU_ITEMS=8
one WELDGPU_DEFER_DICT=0
one WELDGPU_PIPE=0 WELDGPU_DEFER_DICT=0
one WELDGPU_PREFETCH=0 WELDGPU_PIPE=0 WELDGPU_ITEMS=8

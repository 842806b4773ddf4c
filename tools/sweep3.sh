one() {
  w=$1; shift
  r=$(env "$@" timeout 200 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e $EXTRA 2>&1 | tail -1)
  echo "$w $EXTRA $* => $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms %.3f frac %.3f step_ms %.3f" % (r["kernel_ms"], r["frac"], d["ms_per_step"]))' 2>&1 | tail -1)"
}
for bud in 32768 49152 73728 102400; do
  for w in blackscholes q1 group hist; do one $w WELDGPU_PIPE_SMEM=$bud; done
  EXTRA="--n 600000000" one q6 WELDGPU_PIPE_SMEM=$bud
  EXTRA="" one q6 WELDGPU_PIPE_SMEM=$bud
done

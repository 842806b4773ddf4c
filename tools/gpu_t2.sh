mkdir -p gpurun_out/t2
: > gpurun_out/t2/sweep_part.txt
for it in 2 4 8 16; do
  WELDGPU_PART_ITEMS=$it timeout 600 python -m pytest tests/test_gpu_configs.py -q -x -k "dict" 2>&1 | tail -1 >> gpurun_out/t2/sweep_part.txt
  r=$(WELDGPU_PART_ITEMS=$it timeout 300 python bench.py --workload dict --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1)
  echo "part items=$it $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("dom %s %.3f ms step %.3f" % (r["kernel"], r["kernel_ms"], d["ms_per_step"]))' 2>&1 | tail -1)" >> gpurun_out/t2/sweep_part.txt
done

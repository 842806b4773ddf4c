mkdir -p gpurun_out/t2
for kp in 0 1; do
WELDGPU_KPOOL=$kp timeout 600 python bench.py --workload blackscholes --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/t2/bs_kp$kp.log
done
WELDGPU_KPOOL=1 WELDGPU_MINBLOCKS=3 timeout 600 python bench.py --workload blackscholes --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/t2/bs_kp1_mb3.log
WELDGPU_KPOOL=1 WELDGPU_MINBLOCKS=4 timeout 600 python bench.py --workload blackscholes --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/t2/bs_kp1_mb4.log

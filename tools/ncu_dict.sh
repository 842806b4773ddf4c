mkdir -p gpurun_out/ncu
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"wg_loop" -s 2 -c 1 -o gpurun_out/ncu/full_dictrp2 \
   python bench.py --workload dict --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > gpurun_out/ncu/ncu_dictrp.log 2>&1

mkdir -p gpurun_out/prof
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:wg_loop -s 2 -c 1 -o gpurun_out/prof/full_dict python bench.py --workload dict --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > gpurun_out/prof/ncu_dict.log 2>&1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:wg_dagg -s 1 -c 1 -o gpurun_out/prof/full_dict_dagg python bench.py --workload dict --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > /dev/null 2>&1

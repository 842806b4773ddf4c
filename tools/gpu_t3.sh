mkdir -p gpurun_out/t3
timeout 600 ncu --metrics launch__block_size,launch__grid_size,gpu__time_duration.sum,launch__shared_mem_per_block_dynamic,launch__registers_per_thread,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/t3/launches_dict.csv python bench.py --workload dict --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > gpurun_out/t3/log 2>&1

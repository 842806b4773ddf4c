mkdir -p gpurun_out/t2
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_rpart.py -q -x -k "dict" 2>&1 | tail -3 > gpurun_out/t2/pytest.log
timeout 300 python bench.py --workload dict --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/t2/bench_dict.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t2/launches_dict.csv python bench.py --workload dict --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > /dev/null 2>&1

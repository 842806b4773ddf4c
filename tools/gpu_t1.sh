mkdir -p gpurun_out/t1
timeout 900 python -m pytest tests/test_gpu_rpart.py tests/test_gpu_configs.py -q -x -k "rpart or group or dict" 2>&1 | tail -30 > gpurun_out/t1/pytest.log
timeout 600 python bench.py --workload dict --steps 10 --warmup 3 --no-cpu 2>&1 | tail -3 > gpurun_out/t1/bench_dict.log

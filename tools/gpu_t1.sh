mkdir -p gpurun_out/t1
timeout 900 python -m pytest tests -q -x -m gpu -k "group" 2>&1 | tail -5 > gpurun_out/t1/pytest.log
timeout 600 python bench.py --workload group --steps 10 --warmup 3 --no-cpu 2>&1 | tail -3 > gpurun_out/t1/bench_group.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t1/launches_group.csv python bench.py --workload group --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > /dev/null 2>&1

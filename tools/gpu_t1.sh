mkdir -p gpurun_out/t1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/t1/pytest.log
python tools/prof_host2.py q6 1000000 2>&1 | head -1 >> gpurun_out/t1/pytest.log
timeout 300 python bench.py --workload q6 --steps 20 --warmup 5 --no-cpu 2>&1 | tail -1 > gpurun_out/t1/bench_q6.log

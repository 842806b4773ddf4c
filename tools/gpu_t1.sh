mkdir -p gpurun_out/t1
timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -30 > gpurun_out/t1/pytest.log
for w in q1 group; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu 2>&1 | tail -3 > gpurun_out/t1/bench_$w.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t1/launches_group.csv python bench.py --workload group --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > /dev/null 2>&1

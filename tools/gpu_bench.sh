set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -5 | tee gpurun_out/bench_bs.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_bs.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_bs.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wg_loop -s 3 -c 1 -o gpurun_out/prof_bs python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full_bs.log 2>&1
for w in q6 q1 hist dict group; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu 2>&1 | tail -3 | tee gpurun_out/bench_$w.log; done

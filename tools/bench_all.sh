for w in blackscholes q6 q1 hist dict group; do
  timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu 2>&1 | tail -2 > gpurun_out/bench_$w.log
done

# GPU tests, smoke, the default bench line, and one bench line per workload.
mkdir -p gpurun_out/rc
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/rc/gpu.txt
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -25 > gpurun_out/rc/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc/smoke.log 2>&1
timeout 900 python bench.py 2>&1 | tail -3 > gpurun_out/rc/bench_default.log
for w in ${WORKLOADS:-q6 q1 dict group hist}; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu 2>&1 | tail -2 > gpurun_out/rc/bench_$w.log
done

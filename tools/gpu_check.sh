# GPU tests (all), smoke, and the default bench line; outputs under gpurun_out/rc/.
mkdir -p gpurun_out/rc
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/rc/gpu.txt
nproc >> gpurun_out/rc/gpu.txt; free -g >> gpurun_out/rc/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc/smoke.log 2>&1; echo smoke_rc=$?
timeout 2400 python -m pytest tests -q -m gpu --durations=15 ${PYTEST_ARGS} > gpurun_out/rc/pytest.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/rc/pytest.log
timeout 1200 python bench.py > gpurun_out/rc/bench_default.json 2> gpurun_out/rc/bench_default.err; echo bench_rc=$?
tail -c 1500 gpurun_out/rc/bench_default.err

mkdir -p gpurun_out/t1
: > gpurun_out/t1/pytest.log
for r in 1 2; do
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4 >> gpurun_out/t1/pytest.log
done

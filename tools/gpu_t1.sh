mkdir -p gpurun_out/t1
timeout 900 python -m pytest tests/test_gpu_flatmap.py -q -x 2>&1 | tail -40 > gpurun_out/t1/pytest.log

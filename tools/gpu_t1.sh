mkdir -p gpurun_out/t1
timeout 900 python -m pytest tests/test_gpu_api.py -q 2>&1 | tail -30 > gpurun_out/t1/pytest.log

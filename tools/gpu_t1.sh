mkdir -p gpurun_out/t1
timeout 600 python -m pytest tests/test_gpu_rpart.py -q -k reused 2>&1 | grep -E "assert|Error|Mismatch|^E " | head -30 > gpurun_out/t1/pytest.log

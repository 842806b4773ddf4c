free -g | head -2; nproc
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=12 2>&1 | tail -25

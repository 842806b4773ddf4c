mkdir -p gpurun_out
timeout 120 ./tools/sort_ab | tee gpurun_out/sort_ab.txt
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_math.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --workload group --steps 10 --warmup 3 --per-config none --no-cpu --no-e2e > gpurun_out/bench_group.json 2>gpurun_out/bench_group.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_group.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['frac']); print(d['roofline']['kernels'])"

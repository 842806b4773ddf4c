mkdir -p gpurun_out
timeout 300 ./tools/sort_ab > gpurun_out/sort_ab.txt 2>&1; echo sort_ab_rc=$?; cat gpurun_out/sort_ab.txt
timeout 900 python -m pytest tests/test_gpu_sort.py -x -q > gpurun_out/pytest_sort.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_sort.log
timeout 600 python bench.py --workload group --steps 10 --warmup 3 --per-config none --no-cpu --no-e2e > gpurun_out/bench_group.json 2>gpurun_out/bench_group.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_group.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['frac']); print(d['roofline']['kernels'])"
tail -3 gpurun_out/bench_group.err

python tools/prof_host_q1.py q1 2>&1 | head -1
for w in q1 dict group; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --per-config none --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['config']['workload'], 'ms', round(d['ms_per_step'],3), 'cold', round(d['cold_ms_per_step'],3), [(k['name'], round(k['ms_per_step'],3)) for k in d['roofline']['kernels']])"; done

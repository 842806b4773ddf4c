# Round profile set: GPU tests, headline bench line, launch list of the
# default bench and of one step per workload, one ncu --set full capture of
# each workload's loop kernel, and a bench line per workload.
mkdir -p gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/prof/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/prof/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/prof/smoke.log 2>&1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/prof/bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_default.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-kernel-timing --per-config none > /dev/null 2>&1
for w in blackscholes q6 q1 dict group hist filter map; do
  extra=""
  [ $w = q6 ] && extra="--n 600000000"
  skip=3
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:wg_loop -s $skip -c 1 -o gpurun_out/prof/full_$w \
     python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing $extra > gpurun_out/prof/ncu_$w.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$w.csv \
     python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing --per-config none $extra > /dev/null 2>&1
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu $extra 2>&1 | tail -1 > gpurun_out/prof/bench_$w.json
done
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:wg_dagg -s 2 -c 1 -o gpurun_out/prof/full_dict_dagg \
   python bench.py --workload dict --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > gpurun_out/prof/ncu_dict_dagg.log 2>&1
# the group step's dominant kernel is the library's onesweep radix pass
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_onesweep -s 13 -c 1 -o gpurun_out/prof/full_group_onesweep \
   python bench.py --workload group --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > gpurun_out/prof/ncu_group_onesweep.log 2>&1
# L2 RED ceiling (C5)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_peak tools/red_peak.cu && ./tools/red_peak > gpurun_out/prof/red_peak.txt 2>&1
timeout 600 python bench.py --workload q6 --steps 20 --warmup 5 --no-cpu 2>&1 | tail -1 > gpurun_out/prof/bench_q6_1M.json
timeout 600 python tools/api_e2e.py 1000000 > gpurun_out/prof/api_e2e.txt 2>&1

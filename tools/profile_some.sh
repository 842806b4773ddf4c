# Re-capture a subset of the round profile set: bash tools/profile_some.sh blackscholes dict
mkdir -p gpurun_out/prof
for w in "$@"; do
  extra=""
  [ $w = q6 ] && extra="--n 600000000"
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:wg_loop -s 3 -c 1 -o gpurun_out/prof/full_$w \
     python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing $extra > gpurun_out/prof/ncu_$w.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$w.csv \
     python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing $extra > /dev/null 2>&1
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu $extra 2>&1 | tail -1 > gpurun_out/prof/bench_$w.json
  if [ $w = dict ]; then
    timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:wg_dagg -s 2 -c 1 -o gpurun_out/prof/full_dict_dagg \
       python bench.py --workload dict --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > gpurun_out/prof/ncu_dict_dagg.log 2>&1
  fi
  if [ $w = blackscholes ]; then
    timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/prof/bench_default.json
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_default.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > /dev/null 2>&1
  fi
done

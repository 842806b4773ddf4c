# one ncu --set full capture (with source) of a workload's loop kernel: $1 workload, rest = extra bench args
w=$1; shift
mkdir -p gpurun_out/ncu
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:${KREGEX:-wg_loop} -s ${SKIP:-3} -c 1 -o gpurun_out/ncu/full_$w \
   python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing "$@" > gpurun_out/ncu/ncu_$w.log 2>&1

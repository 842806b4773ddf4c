# per-launch device times (ncu, cold-cache, serialised) of a few bench steps per workload
mkdir -p gpurun_out/ll
for w in ${WORKLOADS:-group dict q1 q6}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll/launches_$w.csv \
     python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing > gpurun_out/ll/$w.log 2>&1
done

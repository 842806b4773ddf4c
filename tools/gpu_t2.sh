mkdir -p gpurun_out/t2
for pb in 0 4 8; do
WELDGPU_RPART_PBITS=$pb timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t2/launches_pb$pb.csv python bench.py --workload dict --n 20000000 --steps 1 --warmup 2 --no-cpu --no-e2e --no-kernel-timing > /dev/null 2>&1
done

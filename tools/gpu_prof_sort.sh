mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:onesweep -s 6 -c 1 -o gpurun_out/onesweep ./tools/sort_ab 50000000 > gpurun_out/ncu_onesweep.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_onesweep.log

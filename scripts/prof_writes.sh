cd oracle/_ref/dropin
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ../../../gpurun_out/ncu_writes.csv ./bench_read_b200 writes 131072 20 2 > ../../../gpurun_out/ncu_writes.out 2>&1
echo rc=$?
tail -3 ../../../gpurun_out/ncu_writes.out

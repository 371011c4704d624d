# launch list + one full capture of the headline kernel at config 4 (bench.py's own step)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 1 --quick > gpurun_out/r02_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k k_scan_m4rm_q9 -c 1 -o gpurun_out/r02_q9_config4 \
  python bench.py --steps 1 --warmup 1 --quick > gpurun_out/r02_q9_config4.log 2>&1
tail -2 gpurun_out/r02_q9_config4.log

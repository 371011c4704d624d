# round-2 refresh of the config 1/2/3/5 measurements with the final kernels
python sweep.py --out gpurun_out/r02_config5_sweep.jsonl > gpurun_out/sweep.log 2>&1; tail -2 gpurun_out/sweep.log
python sweep.py --summary gpurun_out/r02_config5_sweep.jsonl > gpurun_out/r02_config5_sweep_summary.txt 2>&1
python bench_write.py --out gpurun_out/r02_write_path.jsonl --reps 5 > gpurun_out/bench_write.log 2>&1; tail -2 gpurun_out/bench_write.log | cut -c1-300
python bench_configs.py --out gpurun_out/r02_configs.jsonl > gpurun_out/bench_configs.log 2>&1; tail -3 gpurun_out/bench_configs.log | cut -c1-300

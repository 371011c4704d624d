timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_par_solve -c 1 -o gpurun_out/solve python scripts/dbg_async.py > gpurun_out/prof_solve.log 2>&1
python bench_write.py --out gpurun_out/write_path.jsonl --reps 5 --only 24 2>&1 | cut -c1-420

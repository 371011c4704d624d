timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_w24.csv python bench_write.py --only 24 --reps 1 --out gpurun_out/w24.jsonl > gpurun_out/ncu_w24.out 2>&1
echo rc=$?

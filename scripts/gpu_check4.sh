python -m pytest tests/test_gpu_write.py tests/test_gpu_server.py -x -q -p no:cacheprovider 2>&1 | tail -4
python bench_write.py --out gpurun_out/write_path.jsonl --reps 5 2>&1 | cut -c1-400

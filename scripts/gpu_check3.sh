python -m pytest tests/test_gpu_write.py tests/test_gpu_server.py tests/test_gpu_dropin.py -x -q -p no:cacheprovider 2>&1 | tail -8
python bench_write.py --out gpurun_out/write_path.jsonl 2>&1 | tail -4
cd oracle/_ref/dropin
timeout 300 ./bench_read_b200 writes 131072 500 8 2>&1 | tail -2

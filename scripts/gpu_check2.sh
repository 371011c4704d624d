python -m pytest tests/test_gpu_server.py tests/test_gpu_write.py tests/test_gpu_dropin.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider 2>&1 | tail -15
cd oracle/_ref/dropin
timeout 300 ./bench_read_b200 writes 131072 500 8 2>&1 | tail -3
timeout 300 ./bench_read_ref writes 131072 500 4 2>&1 | tail -3

set -x
python -m pytest tests/test_gpu_batcher.py tests/test_gpu_server.py tests/test_gpu_dropin.py tests/test_gpu_write.py tests/test_gpu_scan.py -x -q -p no:cacheprovider 2>&1 | tail -15
cd oracle/_ref/dropin
timeout 300 ./test_server_b200 2>&1 | tail -5
timeout 600 ./bench_read_b200 process 10000,100000,1000000 20 2>&1 | tail -5
timeout 300 ./bench_read_b200 concurrent 100000 64 16 2>&1 | tail -3
timeout 300 ./bench_read_b200 writes 131072 500 8 2>&1 | tail -3
timeout 900 ./acceptance_b200 > ../../../gpurun_out/acceptance_b200.txt 2>&1; echo rc=$?; cat ../../../gpurun_out/acceptance_b200.txt

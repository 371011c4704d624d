python -m pytest tests/test_gpu_scan.py tests/test_gpu_pinned.py tests/test_gpu_write.py -q -p no:cacheprovider 2>&1 | tail -2
for G in 2 8; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2951$G bench.py --gpus $G --steps 3 --warmup 2 > gpurun_out/bench_r$G.json 2> gpurun_out/bench_r$G.err
python -c "import json; d=json.loads(open('gpurun_out/bench_r$G.json').read().strip().splitlines()[-1]); print($G, d['value'], d['parity'], d['reduce'], d.get('peer_bytes'))"
done

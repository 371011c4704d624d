# full GPU suite + default bench line + shared-GPU multi-rank fused-reduce check
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -1 gpurun_out/bench_n1.json | cut -c1-600
for G in 2 8; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2951$G bench.py --gpus $G --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_r$G.json 2> gpurun_out/bench_r$G.err
python -c "import json; d=json.loads(open('gpurun_out/bench_r$G.json').read().strip().splitlines()[-1]); print($G, d['value'], d['parity'], d['reduce'], d.get('peer_bytes'))"
done

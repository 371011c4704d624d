# full GPU suite + smoke + the shared-GPU multi-rank validation (no production-path rerun)
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for G in 2 8; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2951$G bench.py --gpus $G --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_r$G.json 2> gpurun_out/bench_r$G.err
python -c "import json; d=json.loads(open('gpurun_out/bench_r$G.json').read().strip().splitlines()[-1]); print($G, d['value'], d['parity'], d['reduce'], d.get('peer_bytes'))"
done

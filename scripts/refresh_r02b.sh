# round-2 refresh of the caller-side measurements (read batcher, replica rounds, interest codecs)
python bench_batcher.py --threads 512 --out gpurun_out/r02_batcher.jsonl > gpurun_out/bench_batcher.log 2>&1; tail -4 gpurun_out/bench_batcher.log | cut -c1-300
python bench_server.py --out gpurun_out/r02_server_rounds.jsonl > gpurun_out/bench_server.log 2>&1; tail -2 gpurun_out/bench_server.log | cut -c1-400
python bench_codec.py --out gpurun_out/r02_codec.jsonl > gpurun_out/bench_codec.log 2>&1; tail -3 gpurun_out/bench_codec.log | cut -c1-300

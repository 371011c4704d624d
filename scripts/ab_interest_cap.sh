# write round as one graph: interest kernel grid cap (XPIR_INTEREST_CAP blocks per SM, 0 = one
# thread per hash) x interest branch placement (XPIR_BENCH_INTEREST_AFTER_PREFIX)
for cap in 16 0 32 64; do for after in 0; do
  XPIR_INTEREST_CAP=$cap XPIR_BENCH_INTEREST_AFTER_PREFIX=$after python bench_write.py --out gpurun_out/ab_cap.jsonl --reps 7 --only 24 > /dev/null 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_cap.jsonl').read().strip().splitlines()[-1]); print(json.dumps({'cap': $cap, 'after_prefix': $after, 'graph_device_ms': round(d['graph_device_ms'],4), 'device_span_ms': round(d['device_span_ms'],4), 'graph_ok': d['graph_bit_exact_vs_golden'], 'ok': d['bit_exact_vs_golden']}))"
done; done

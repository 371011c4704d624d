"""A/B of the 9-bucket quad-table kernel, run while it was candidate kernel 10 (it replaced
bit-exact on ragged shapes (row-major and seeded queries, shard windows), then
per-launch time at config 4 (4 GiB, B = 8192) and a 1 GiB store."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2001_08250_b200 as xp  # noqa: E402

cs = torch.cuda.current_stream()
ok_all = True
for (N, S, lo, hi, B) in [(1000, 32, 0, None, 4096), (4099, 64, 0, None, 5000), (100003, 96, 0, None, 2048),
                          (72 * 40 + 5, 32, 0, None, 8192), (20000, 128, 8 * 37, 8 * 1500, 4100),
                          (65536, 1024, 0, None, 9000), (300001, 32, 8 * 1000, 300001, 8192)]:
    st = xp.Store(N, S, lo, N if hi is None else hi)
    st.fill_keystream(bytes(range(32)), 7)
    q = torch.randint(0, 256, (B, (N + 7) // 8 + 3), dtype=torch.uint8, device="cuda")
    seeds = torch.randint(0, 256, (B, 32), dtype=torch.uint8, device="cuda")
    outs = {}
    for k in (8, 10):
        xp.set_scan_opts(k)
        o1 = torch.empty((B, S), dtype=torch.uint8, device="cuda")
        o2 = torch.empty((B, S), dtype=torch.uint8, device="cuda")
        st.answer_batch_dev(q, q.shape[1], B, o1, stream=cs)
        st.answer_batch_seeded_dev(seeds, B, o2, stream=cs)
        torch.cuda.synchronize()
        assert xp.last_scan_kernel() == k, (k, xp.last_scan_kernel())
        outs[k] = (o1, o2)
    ok = bool(torch.equal(outs[8][0], outs[10][0])) and bool(torch.equal(outs[8][1], outs[10][1]))
    ok_all &= ok
    print(json.dumps({"N": N, "S": S, "lo": lo, "hi": hi, "B": B, "bit_exact_vs_k8": ok}), flush=True)
    st.close()

for (N, S, B) in [(1 << 20, 4096, 8192), (1 << 18, 4096, 8192), (1 << 18, 4096, 4096), (1 << 20, 1024, 16384)]:
    st = xp.Store(N, S)
    st.fill_keystream(bytes(32), 0)
    seeds = torch.randint(0, 256, (B, 32), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, S), dtype=torch.uint8, device="cuda")
    res = {}
    for k in (8, 10):
        xp.set_scan_opts(k)
        for _ in range(2):
            st.answer_batch_seeded_dev(seeds, B, out, stream=cs)
        torch.cuda.synchronize()
        xp.scan_timing_collect()
        xp.scan_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 3
        for _ in range(n):
            st.answer_batch_seeded_dev(seeds, B, out, stream=cs)
        e1.record()
        torch.cuda.synchronize()
        xp.scan_timing(False)
        scan_ms, launches = xp.scan_timing_collect()
        res[k] = {"step_ms": round(e0.elapsed_time(e1) / n, 3), "scan_ms": round(scan_ms / max(launches, 1), 3)}
    print(json.dumps({"N": N, "S": S, "B": B, **{f"k{k}": v for k, v in res.items()},
                      "speedup": round(res[8]["scan_ms"] / res[10]["scan_ms"], 4)}), flush=True)
    st.close()
xp.set_scan_opts(0)
print(json.dumps({"all_bit_exact": ok_all}))

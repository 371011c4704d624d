"""Randomised cross-check of the 9-bucket quad kernel (8) against the byte-table
kernels (2 / 5) on large random shapes, explicit rows and seeds, shard windows."""
import json
import os
import random
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2001_08250_b200 as xp  # noqa: E402

rnd = random.Random(int(os.environ.get("SEED", "1")))
cs = torch.cuda.current_stream()
bad = 0
for case in range(int(os.environ.get("CASES", "24"))):
    S = 128 * rnd.randint(1, 24)
    N = rnd.randint(1000, (1 << 28) // S)
    B = rnd.choice([rnd.randint(2048, 20000), 4096, 8192, 8193, 16384])
    lo = 8 * rnd.randint(0, N // 32) if rnd.random() < 0.4 else 0
    hi = N if rnd.random() < 0.5 else min(N, lo + 8 * rnd.randint(1, (N - lo) // 8 + 1))
    if hi <= lo:
        hi = N
    st = xp.Store(N, S, lo, hi)
    st.fill_keystream(bytes([case] * 32), case)
    q = torch.randint(0, 256, (B, (N + 7) // 8), dtype=torch.uint8, device="cuda")
    seeds = torch.randint(0, 256, (B, 32), dtype=torch.uint8, device="cuda")
    outs = {}
    for k in (8, 5):
        xp.set_scan_opts(k)
        o1 = torch.empty((B, S), dtype=torch.uint8, device="cuda")
        o2 = torch.empty((B, S), dtype=torch.uint8, device="cuda")
        st.answer_batch_dev(q, q.shape[1], B, o1, stream=cs)
        st.answer_batch_seeded_dev(seeds, B, o2, stream=cs)
        torch.cuda.synchronize()
        outs[k] = (o1, o2, xp.last_scan_kernel())
    ok = bool(torch.equal(outs[8][0], outs[5][0])) and bool(torch.equal(outs[8][1], outs[5][1]))
    bad += not ok
    print(json.dumps({"case": case, "N": N, "S": S, "B": B, "lo": lo, "hi": hi, "kernels": [outs[8][2], outs[5][2]],
                      "bit_exact": ok}), flush=True)
    st.close()
    del q, seeds, outs
    torch.cuda.empty_cache()
xp.set_scan_opts(0)
print(json.dumps({"mismatches": bad}))

"""Historical A/B (round 2; the kernel-11 dispatch path it drove was removed after it lost): direct kernel on the head of the store and nibble tables on the tail,
launched concurrently on two streams (kernel 11, XPIR_HYB2_F = head fraction in
thousandths) against each alone; 1 GiB store, S = 4096, explicit rows."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2001_08250_b200 as xp  # noqa: E402

peaks = xp.measure_peaks(0)
cs = torch.cuda.current_stream()
S = 4096
N = (1 << 30) // S
st = xp.Store(N, S)
st.fill_keystream(bytes(32), 0)
res = {}
for B in (8, 12, 16, 20, 24):
    q = torch.randint(0, 256, (B, N // 8), dtype=torch.uint8, device="cuda")
    fr, outs = {}, {}
    for k in (1, 7, 11):
        xp.set_scan_opts(k)
        o = torch.empty((B, S), dtype=torch.uint8, device="cuda")
        for _ in range(2):
            st.answer_batch_dev(q, N // 8, B, o, stream=cs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            st.answer_batch_dev(q, N // 8, B, o, stream=cs)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        t_alu = B * N * S / 4 / peaks["lop3_per_s"] * 1e3
        t_hbm = (N * S + B * N / 8 + B * S) / 6.5345e12 * 1e3
        fr[k] = round(max(t_alu, t_hbm) / ms, 3)
        outs[k] = o
    res[B] = {"direct": fr[1], "nibble": fr[7], "both": fr[11],
              "same": bool(torch.equal(outs[1], outs[11])) and bool(torch.equal(outs[1], outs[7]))}
print(json.dumps({"F": os.environ.get("XPIR_HYB2_F"), "res": res}), flush=True)
xp.set_scan_opts(0)

"""Small batches: nibble tables (kernel 7, lookups spread over all warps for B <= 32)
against the direct kernel (1): fraction of max(T_hbm, T_alu) and bit-exactness."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2001_08250_b200 as xp  # noqa: E402

peaks = xp.measure_peaks(0)
cs = torch.cuda.current_stream()
for S in (4096, 512, 1024):
    N = (1 << 30) // S
    st = xp.Store(N, S)
    st.fill_keystream(bytes(32), 0)
    res = {}
    for B in (8, 12, 16, 20, 24, 32, 48, 64, 128, 144, 192, 256):
        q = torch.randint(0, 256, (B, N // 8), dtype=torch.uint8, device="cuda")
        outs, fr = {}, {}
        for k in ((1, 7, 9) if B >= 128 else (1, 7)):
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
        res[B] = {"direct": fr[1], "nibble": fr[7], **({"six": fr[9]} if 9 in fr else {}),
                  "same": all(bool(torch.equal(outs[1], o)) for o in outs.values())}
    print(json.dumps({"S": S, "res": res}), flush=True)
    st.close()
xp.set_scan_opts(0)

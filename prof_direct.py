"""prof_direct.py — small batches (B = 4..64) on a 1 GiB store: ms per scan and
fraction of the dense-ALU roofline for the direct kernel (1) and the nibble-table
kernels (6, 7), to calibrate the small-B dispatch."""
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_2001_08250_b200 as xp  # noqa: E402

R = xp.measure_peaks()["lop3_per_s"]
for S in (4096, 512):
    N = (1 << 30) // S
    st = xp.Store(N, S)
    st.fill_keystream(bytes(32), 0)
    cs = torch.cuda.current_stream()
    for B in (4, 8, 12, 16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512):
        q = torch.randint(0, 256, (B, N // 8), dtype=torch.uint8, device='cuda')
        out = torch.empty((B, S), dtype=torch.uint8, device='cuda')
        ref = None
        row = [S, B]
        for k in (0, 1, 6, 7, 9):
            xp.set_scan_opts(k)
            ts = []
            for r in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(cs)
                st.answer_batch_dev(q, N // 8, B, out, stream=cs)
                e1.record(cs)
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
            if ref is None:
                ref = out.clone()
            assert torch.equal(out, ref), (S, B, k)
            t = statistics.median(ts)
            row += [f"k{k}->{xp.last_scan_kernel()}", round(t, 4), round(B * N * S / 4 / R / (t * 1e-3), 3)]
        print(*row, flush=True)
    st.close()
xp.set_scan_opts(0)

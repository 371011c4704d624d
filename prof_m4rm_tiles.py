"""prof_m4rm_tiles.py — kernel 5 (half-TMEM, 128-B columns) vs kernel 8 (quad tables,
full TMEM) at B = 2048 / 4096 / 8192 on a 1 GiB store: ms per scan and fraction of the
dense-ALU roofline (1.85e13 LOP3/s). Used to calibrate the dispatch cost model."""
import sys, torch, statistics
sys.path.insert(0, '.')
import paper_2001_08250_b200 as xp
N, S = 262144, 4096
st = xp.Store(N, S); st.fill_keystream(bytes(32), 0)
cs = torch.cuda.current_stream()
for B in (2048, 4096, 8192):
    q = torch.randint(0, 256, (B, N // 8), dtype=torch.uint8, device='cuda')
    out = torch.empty((B, S), dtype=torch.uint8, device='cuda')
    for k in (5, 8):
        xp.set_scan_opts(k)
        ts = []
        for r in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs); st.answer_batch_dev(q, N // 8, B, out, stream=cs); e1.record(cs); torch.cuda.synchronize()
            if r: ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        print(B, k, xp.last_scan_kernel(), round(t, 3), "frac", round(B * N * S / 4 / 1.85e13 / (t * 1e-3), 3))

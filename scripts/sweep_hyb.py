"""A/B of the hybrid small-batch kernel (kernel 10) dense fraction (XPIR_HYB_VARIANT,
thousandths), 1 GiB store; output compared with the direct kernel every point."""
import os, subprocess, sys, json
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch
    sys.path.insert(0, os.getcwd())
    import paper_2001_08250_b200 as xp
    S = int(os.environ.get("S", "4096")); N = (1 << 30) // S
    st = xp.Store(N, S); st.fill_keystream(bytes(32), 0)
    peaks = xp.measure_peaks(0)
    res, ok = {}, True
    cs = torch.cuda.current_stream()
    for B in (8, 12, 16, 24, 32):
        q = torch.randint(0, 256, (B, N // 8), dtype=torch.uint8, device='cuda')
        ref = torch.empty((B, S), dtype=torch.uint8, device='cuda')
        xp.set_scan_opts(1); st.answer_batch_dev(q, N // 8, B, ref, stream=cs)
        out = torch.empty((B, S), dtype=torch.uint8, device='cuda')
        xp.set_scan_opts(10)
        for _ in range(3): st.answer_batch_dev(q, N // 8, B, out, stream=cs)
        torch.cuda.synchronize()
        ok = ok and bool(torch.equal(out, ref)) and xp.last_scan_kernel() == 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): st.answer_batch_dev(q, N // 8, B, out, stream=cs)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        t_alu = B * N * S / 4 / peaks["lop3_per_s"] * 1e3; t_hbm = N * S / 6.5345e12 * 1e3
        res[B] = round(max(t_alu, t_hbm) / ms, 3)
    print(json.dumps({"variant": os.environ.get("XPIR_HYB_VARIANT"), "S": S, "frac": res, "bit_exact_vs_direct": ok}))
else:
    for d in sys.argv[1:] or ("0", "1", "2", "3", "4", "5"):
        subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, XPIR_HYB_VARIANT=d))

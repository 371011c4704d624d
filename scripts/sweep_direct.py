"""A/B of the direct kernel's request-tile x column variants (XPIR_DIRECT_TILE), 1 GiB store."""
import os, subprocess, sys, json
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch
    sys.path.insert(0, os.getcwd())
    import paper_2001_08250_b200 as xp
    S = int(os.environ.get("S", "4096")); N = (1 << 30) // S
    st = xp.Store(N, S); st.fill_keystream(bytes(32), 0)
    xp.set_scan_opts(1)
    res = {}
    peaks = xp.measure_peaks(0)
    for B in (8, 12, 16, 24, 32):
        q = torch.randint(0, 256, (B, N // 8), dtype=torch.uint8, device='cuda')
        out = torch.empty((B, S), dtype=torch.uint8, device='cuda')
        for _ in range(3): st.answer_batch_dev(q, N // 8, B, out, stream=torch.cuda.current_stream())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): st.answer_batch_dev(q, N // 8, B, out, stream=torch.cuda.current_stream())
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        t_alu = B * N * S / 4 / peaks["lop3_per_s"] * 1e3; t_hbm = N * S / 6.5345e12 * 1e3
        res[B] = round(max(t_alu, t_hbm) / ms, 3)
    print(json.dumps({"tile": os.environ.get("XPIR_DIRECT_TILE", "auto"), "S": S, "frac": res}))
else:
    for tile in ("auto", "8,2", "4,2", "8,1", "2,4", "6,2"):
        env = dict(os.environ)
        if tile != "auto": env["XPIR_DIRECT_TILE"] = tile
        subprocess.run([sys.executable, __file__, "run"], env=env)

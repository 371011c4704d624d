"""sweep.py — BASELINE.json config 5: shape sweep at a fixed 1 GiB store.

Slot size 256..4096 B x bucket depth 2/4/8 (bucket count adjusted to keep the
store at 1 GiB of DetRng(5) bytes) x batch 1..16384 (powers of two) of uniform
random selection vectors (DetRng(55) fills, generated on device). For every
point: requests/s, effective DB-scan GB/s and the fraction of the HBM-or-ALU
roofline, T_roof = max(T_hbm, T_alu):
    T_hbm = (N*S + B*N/8 + B*S) / HBM peak (MEASURED_PEAKS.json)
    T_alu = (B*N*S/4) / R_lop3   (dense select-XOR: one 32-bit LOP3 per
                                  request x bucket x word; R_lop3 measured live)
frac = T_roof / T_measured (> 1 where the M4RM kernel beats the dense ALU bound).
Timing: CUDA events, median of 3 after 1 warm-up, the query transposition
included (it is part of answering an explicit-vector batch).

    python sweep.py [--max-batch 16384] [--out profiles/r01_config5_sweep.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def summarize(path: str) -> None:
    """The tables of profiles/r01_config5_sweep_summary.txt from a sweep jsonl."""
    rows = [json.loads(l) for l in open(path)][1:]
    shapes = sorted({(r["slot"], r["depth"]) for r in rows})
    bs = sorted({r["B"] for r in rows})
    at = {(r["slot"], r["depth"], r["B"]): r for r in rows}
    print("# config 5: 1 GiB DetRng(5) store, slot x depth shapes, B explicit DetRng(55) vectors; sweep.py (current dispatch)")
    print("# fraction of the HBM-or-ALU roofline max(T_hbm, T_alu)/T (T_alu = dense select-XOR LOP3s / measured LOP3 rate)")
    print("shape    " + "".join(f"{b:>7d}" for b in bs))
    for sl, dp in shapes:
        print(f"{sl:4d}x{dp:<3d}" + "".join(f"{at[(sl, dp, b)]['roofline_frac']:7.2f}" for b in bs))
    print("# requests/s (thousands)")
    for sl, dp in shapes:
        print(f"{sl:4d}x{dp:<3d}" + "".join(f"{at[(sl, dp, b)]['requests_per_s'] / 1e3:7.1f}" for b in bs))
    ks = [at[(shapes[-1][0], shapes[-1][1], b)]["kernel"] for b in bs]
    print("# kernel used (1 direct, 7 m4rm nibble tables, 9 m4rm 6-bucket tables, 2 m4rm byte tables/registers, "
          "5 byte tables/half TMEM, 8 quad tables/full TMEM): " + str(ks))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-batch", type=int, default=16384)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_config5_sweep.jsonl"))
    ap.add_argument("--slots", default="256,512,1024,2048,4096")
    ap.add_argument("--depths", default="2,4,8")
    ap.add_argument("--summary", default=None, help="print the fraction / req/s / kernel tables of a sweep jsonl")
    args = ap.parse_args()
    if args.summary:
        summarize(args.summary)
        return

    import torch

    import paper_2001_08250_b200 as xp

    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    peaks = xp.measure_peaks(0)
    hbm = 6545e9
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"]) * 1e9
    except Exception:
        pass
    key = xp.blake2b((5).to_bytes(8, "little"), 32)
    qkey = xp.blake2b((55).to_bytes(8, "little"), 32)
    batches = [1 << k for k in range(15) if (1 << k) <= args.max_batch]
    rows = []
    for slot in [int(s) for s in args.slots.split(",")]:
        for depth in [int(d) for d in args.depths.split(",")]:
            S = slot * depth
            N = (1 << 30) // S
            st = xp.Store(N, S)
            st.fill_keystream(key, 0)
            qmax = torch.empty((max(batches), N // 8), dtype=torch.uint8, device="cuda")
            xp.keystream_rows_dev(qkey, 0, max(batches), N // 8, qmax, N // 8)
            out = torch.empty((max(batches), S), dtype=torch.uint8, device="cuda")
            for B in batches:
                ts = []
                for rep in range(4):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    st.answer_batch_dev(qmax, N // 8, B, out, stream=stream)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    if rep:
                        ts.append(e0.elapsed_time(e1) * 1e-3)
                t = statistics.median(ts)
                t_hbm = (N * S + B * N / 8 + B * S) / hbm
                t_alu = B * N * S / 4 / peaks["lop3_per_s"]
                row = {"slot": slot, "depth": depth, "S": S, "N": N, "B": B, "kernel": xp.last_scan_kernel(),
                       "ms": t * 1e3, "requests_per_s": B / t, "effective_scan_GBps": B * N * S / t / 1e9,
                       "bound": "hbm" if t_hbm >= t_alu else "alu", "t_hbm_ms": t_hbm * 1e3,
                       "t_alu_ms": t_alu * 1e3, "roofline_frac": max(t_hbm, t_alu) / t}
                rows.append(row)
                print(json.dumps(row), flush=True)
            st.close()
            del qmax, out
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        f.write(json.dumps({"peaks": peaks, "hbm_Bps": hbm}) + "\n")
        for r in rows:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()

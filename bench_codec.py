"""bench_codec.py — interest-window codecs on the
config-3 interest delta (2^20 bits after 32,000 writes x 23 positions):
notify::encode_delta / decode_delta (notify.cpp:139-180) on device vs the
unmodified reference on one host core (oracle/_ref).

    python bench_codec.py [--out profiles/r01_codec.jsonl]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def best(f, reps=7):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = f()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3, r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_codec.jsonl"))
    args = ap.parse_args()
    import torch

    import oracle
    import paper_2001_08250_b200 as xp
    from oracle import recipes

    o = oracle.best()
    d = recipes.config3(o, recipes.C3["n"])
    m = recipes.C3["m"]
    W = xp.Window(m, recipes.C3["h"], 1)
    W.absorb_interest(d["lid"], d["xs"])
    words = W.delta(0)
    dw = torch.from_numpy(words.view(np.int64)).cuda()
    n = xp.encode_delta_dev(dw, m)
    dout = torch.empty(n, dtype=torch.uint8, device="cuda")
    ms_dev, _ = best(lambda: xp.encode_delta_dev(dw, m, dout, n))
    ms_win, enc = best(lambda: W.encode_delta(0))
    ms_dec, back = best(lambda: xp.decode_delta(enc))
    assert np.array_equal(back[1], words) and enc == o.encode_delta(m, words)
    line = {"metric": "interest-delta codec (config-3 delta: 2^20 bits, %d set)" % int(np.unpackbits(words.view(np.uint8)).sum()),
            "encoded_bytes": len(enc), "encode_dev_ms": ms_dev, "encode_host_out_ms": ms_win,
            "decode_host_in_ms": ms_dec, "timing": "best of 7, wall clock incl. the host sync (and H2D/D2H for *_host_*)"}
    if o.kind == "reference":
        ms_ref_enc, _ = best(lambda: o.encode_delta(m, words))
        ms_ref_dec, _ = best(lambda: o.decode_delta(enc))
        line.update({"ref_encode_ms": ms_ref_enc, "ref_decode_ms": ms_ref_dec, "ref_kind": "reference", "ref_cores": 1})
    print(json.dumps(line))
    lines = [line]

    # the writes' 64-byte interest fields (wire.cpp:154-169) for the same 32,000 writes
    pos = np.ascontiguousarray(d["pos"], np.uint32)
    n, h = pos.shape
    cap = 64
    d_pos = torch.from_numpy(pos.view(np.int32)).cuda()
    d_f = torch.empty((n, cap), dtype=torch.uint8, device="cuda")
    d_ok = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty((n, cap), dtype=torch.int32, device="cuda")
    d_cnt = torch.empty(n, dtype=torch.int32, device="cuda")

    def enc_dev():
        xp.encode_positions_dev(d_pos, h, n, d_f, d_ok, cap=cap)
        torch.cuda.synchronize()

    def dec_dev():
        xp.decode_positions_dev(d_f, n, d_out, d_cnt, cap=cap)
        torch.cuda.synchronize()

    ms_penc, _ = best(enc_dev)
    ms_pdec, _ = best(dec_dev)
    ok = d_ok.cpu().numpy()
    line2 = {"metric": "write interest fields (config 3: %d writes x %d positions, m = 2^20, 64-byte field)" % (n, h),
             "fit": int(ok.sum()), "too_long": int(n - ok.sum()), "encode_dev_ms": ms_penc, "decode_dev_ms": ms_pdec,
             "timing": "best of 7, wall clock incl. the sync, buffers in HBM"}
    if o.kind == "reference":
        ms_renc, (rf, rok) = best(lambda: o.encode_positions_batch(pos, cap))
        ms_rdec, (rpos, rcnt) = best(lambda: o.decode_positions_batch(rf))
        assert np.array_equal(rok, ok) and np.array_equal(rf, d_f.cpu().numpy())
        assert np.array_equal(rcnt, d_cnt.cpu().numpy().view(np.uint32))
        line2.update({"ref_encode_ms": ms_renc, "ref_decode_ms": ms_rdec, "ref_kind": "reference", "ref_cores": 1,
                      "bit_exact": True})
    print(json.dumps(line2))
    lines.append(line2)
    with open(args.out, "w") as f:
        for l in lines:
            f.write(json.dumps(l) + "\n")


if __name__ == "__main__":
    main()

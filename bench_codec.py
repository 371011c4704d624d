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
    with open(args.out, "w") as f:
        f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()

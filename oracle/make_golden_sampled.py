"""ORACLE / TEST INFRASTRUCTURE ONLY — writes tests/golden/sampled.json from the
UNMODIFIED reference build (oracle/_ref/libxpir_ref.so). Run here (where
/root/reference exists):  python -m oracle.make_golden_sampled

It pins the scan kernels the bench and the batch-size dispatch actually run, at
the sizes they run at (VERDICT r1 "next" #1; ">= 64 random r"):

* config4: the bench's exact step — the 4 GiB DetRng(3) store (call 0) and the
  8,192 seeds of calls 1..8192 (16 bytes each, zero-extended to 32) — with
  64 request rows drawn at random from the whole batch, each answered by the
  reference's pir::answer_batch (pir.cpp:41-52) over the reference Snapshot.
* config5_auto: three 1 GiB shapes of config 5 (store = DetRng(5) call 0), the
  queries of each shape = calls 0..4095 of DetRng(57) (N/8 bytes each); for
  every batch size the dispatch maps to a different kernel
  (16, 64, 256, 1024, 2048, 4096) a random subset of rows of that batch.
  The GPU test runs the whole batch and compares the sampled rows.
"""
from __future__ import annotations

import hashlib
import json
import os
import time

import numpy as np

from oracle import Ref, recipes

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "sampled.json")

C5_SHAPES = ((256, 2), (1024, 4), (4096, 8))  # S = 512, 4096, 32768
C5_BATCHES = (16, 64, 256, 1024, 2048, 4096)
C5_QSEED = 57
C4_ROWS = 66  # >= 64 distinct rows after forcing both batch ends in


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    R = Ref()
    threads = os.cpu_count() or 1
    G: dict = {"generator": "oracle/make_golden_sampled.py over oracle/_ref/libxpir_ref.so "
                            "(reference /root/reference/proj/src + libsodium 1.0.20)"}
    rng = np.random.default_rng(20010826)

    # --- config 4: 64 random rows of the bench's 8,192-request batch -----------
    t = time.time()
    N, S, B = recipes.C4["N"], recipes.C4["S"], recipes.C4["B"]
    g = R.detrng(recipes.C4["seed"])
    snap = R.snapshot_detrng(g, N, S)  # call 0
    seeds = np.zeros((B, 32), np.uint8)
    for r in range(B):
        seeds[r, :16] = np.frombuffer(g.fill(16), np.uint8)  # calls 1..B
    rows = np.sort(rng.choice(B, C4_ROWS, replace=False))
    rows[0], rows[-1] = 0, B - 1  # both batch ends are always checked
    rows = np.unique(rows)
    q = np.stack([np.frombuffer(R.prng_expand(seeds[r].tobytes(), N // 8), np.uint8) for r in rows])
    out, secs = snap.answer_batch(q, len(rows), threads=threads)
    G["config4"] = {"N": N, "S": S, "B": B, "rows": rows.tolist(),
                    "seeds_sha256": sha(seeds), "rows_seed_hex": [seeds[r, :16].tobytes().hex() for r in rows],
                    "out_rows_sha256": [sha(out[i]) for i in range(len(rows))],
                    "out_rows_first16": [out[i, :16].tobytes().hex() for i in range(len(rows))]}
    del snap
    print("config4", len(rows), "rows", f"{time.time() - t:.1f}s (scan {secs:.1f}s)", flush=True)

    # --- config 5: auto-dispatched kernels at 6 batch sizes x 3 shapes ------------
    t = time.time()
    big = R.snapshot_detrng(R.detrng(recipes.C5["seed"]), 1 << 18, 4096)  # 1 GiB, call 0
    dbv = big.data()
    shapes = []
    for slot, depth in C5_SHAPES:
        Ns, Ss = recipes.shape5(slot, depth)
        qg = R.detrng(C5_QSEED)
        Q = np.stack([np.frombuffer(qg.fill(Ns // 8), np.uint8) for _ in range(max(C5_BATCHES))])
        sn = R.snapshot(dbv, Ns, Ss)
        per_b = []
        for Bb in C5_BATCHES:
            k = min(Bb, 24)
            rws = np.sort(rng.choice(Bb, k, replace=False))
            rws[-1] = Bb - 1
            rws = np.unique(rws)
            o = sn.answer_batch(Q[rws], len(rws), threads=threads)[0]
            per_b.append({"B": Bb, "rows": rws.tolist(), "out_rows_sha256": [sha(o[i]) for i in range(len(rws))]})
        shapes.append({"slot": slot, "depth": depth, "N": Ns, "S": Ss,
                       "q_sha256_4096": sha(Q), "batches": per_b})
        del sn, Q
        print("config5", slot, depth, f"{time.time() - t:.1f}s", flush=True)
    G["config5_auto"] = {"store_seed": recipes.C5["seed"], "query_rng_seed": C5_QSEED,
                         "query_calls": "calls 0..B-1 of DetRng(57), N/8 bytes each", "shapes": shapes}

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(G, f, indent=1)
    print("wrote", OUT, os.path.getsize(OUT))


if __name__ == "__main__":
    main()

"""bench_server.py — the replica state machine's write rounds with sealing
(device-resident epoch ring).

A ServerCore (server.cpp:28-91) over config 3's table (32,768 buckets x 4 x
1,024 B, capacity = slots), interest window {m = 2^20, h = 23, W = 4 deltas,
rotate every 4,096 writes}, a ring of 8 sealed epochs. Six rounds of 16,000
writes (the table fills to 73%); every round ends with seal_epoch.

GPU arm: `Server.apply_round(..., seal_after=True)` through the C ABI with
pinned host buffers (betas, payloads, interest positions in; InsertReports
out): insert +
absorb + rotate + an incremental seal that re-copies only the slots rewritten
since the ring's oldest image was sealed.
Reference arm: the unmodified reference `Table::insert` and `Window::absorb /
rotate` (oracle/_ref) for the same writes, and the seal's full table copy
(`Table::snapshot`, cuckoo.cpp:128-135, as seal_epoch does, server.cpp:75-81),
single-threaded (the replica state machine is single-writer).
After every round the table and window digests of both arms must agree.

    python bench_server.py [--out profiles/r01_server_rounds.jsonl]
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_server_rounds.jsonl"))
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--writes", type=int, default=16000)
    args = ap.parse_args()

    import oracle
    import paper_2001_08250_b200 as xp

    o = oracle.best()
    nb, depth, item = 32768, 4, 1024
    cap = nb * depth
    m, h, W, R, ring = 1 << 20, 23, 4, 4096, 8
    g = np.random.default_rng(2001)
    seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
    import torch

    def pinned(a):  # a server's receive buffers are pinned (registered) host memory
        return torch.from_numpy(a).pin_memory().numpy()

    rounds = []
    for _ in range(args.rounds):
        n = args.writes
        rounds.append((pinned(g.integers(0, nb, n).astype(np.uint32)), pinned(g.integers(0, nb, n).astype(np.uint32)),
                       pinned(g.integers(0, 256, (n, item), dtype=np.uint8)),
                       pinned(g.integers(0, m, (n, h)).astype(np.uint32))))

    # warm-up on a throwaway server: every kernel of a round (parallel prefix,
    # eviction walk, seal) is loaded once before the timed server starts
    wsv = xp.Server(nb, depth, cap, item, seed, m, h, W, R, 2)
    wn = int(0.9 * cap)
    wsv.apply_round(g.integers(0, nb, wn).astype(np.uint32), g.integers(0, nb, wn).astype(np.uint32),
                    np.zeros((wn, item), np.uint8), g.integers(0, m, (wn, h)).astype(np.uint32), seal_after=True)
    wsv.close()

    sv = xp.Server(nb, depth, cap, item, seed, m, h, W, R, ring)
    sv.reserve(args.writes)  # start-up: scratch and the ring's sealed images allocated once
    T = o.table(nb, depth, cap, item, seed)
    PW = o.window(m, h, W)
    PW.rotate()  # server.cpp:40
    writes = 0
    gpu_ms, ref_ms, ref_seal_ms = [], [], []
    for b1, b2, pl, pos in rounds:
        t0 = time.perf_counter()
        rep, ep = sv.apply_round(b1, b2, pl, pos, seal_after=True)
        gpu_ms.append((time.perf_counter() - t0) * 1e3)
        # reference: apply_write per write (insert, absorb, rotate every R), then seal
        t0 = time.perf_counter()
        prep = T.insert_batch(b1, b2, pl)
        i = 0
        n = len(b1)
        while i < n:
            seg = min(n - i, R - writes % R)
            PW.absorb(pos[i:i + seg].ravel())
            writes += seg
            i += seg
            if writes % R == 0:
                PW.rotate()
        t1 = time.perf_counter()
        snap = T.data()  # seal_epoch: a full copy of the table (server.cpp:76)
        t2 = time.perf_counter()
        ref_ms.append((t2 - t0) * 1e3)
        ref_seal_ms.append((t2 - t1) * 1e3)
        assert np.array_equal(rep, prep)
        assert sv.table_digest() == T.state_digest() and sv.window_digest() == PW.digest()
        assert np.array_equal(sv.snapshot(ep).download(), snap)
        del snap
    line = {"metric": "replica write round + seal (ServerCore apply_write x n + seal_epoch)",
            "workload": f"{nb} buckets x {depth} x {item} B table, {args.rounds} rounds of {args.writes} writes "
                        f"(to {args.rounds * args.writes / cap:.0%} load), m=2^20 h={h} W={W} rotate every {R}, "
                        f"ring of {ring} sealed epochs",
            "gpu_ms_per_round": statistics.median(gpu_ms), "gpu_ms_rounds": gpu_ms,
            "ref_ms_per_round": statistics.median(ref_ms), "ref_seal_ms_per_round": statistics.median(ref_seal_ms),
            "ref_kind": o.kind, "ref_threads": 1, "bit_exact": True,
            "timing": "wall clock per round; GPU through the host-buffer C ABI (betas, payloads, positions in, "
                      "reports out); the sealed image of every round checked against the reference's table bytes"}
    print(json.dumps(line), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()

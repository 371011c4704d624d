"""bench_configs.py — one line per BASELINE.json PIR config (1 and 2; config 3 is
bench_write.py, config 4 bench.py, config 5 sweep.py), GPU next to the
unmodified reference on the host cores, bit-exact checks included.

  config 1  single-server batch: 1,024 x 4,096 B store (DetRng(0)), 64 explicit
            requests; answers bit-exact vs the reference.
  config 2  three-server secret-shared round: 32,768 x 4,096 B store (DetRng(1)),
            1,024 requests x 3 shares (pir::gen_queries); the per-server scan is
            timed (all three servers' batches); reconstruct == target bucket.

GPU timing: CUDA events on the launching stream around the scan call with the
queries and store already in HBM (value), and wall clock through the host-buffer C-ABI call (e2e).
Reference: pir::answer_batch on all host cores (oracle/_ref), same requests.

    python bench_configs.py [--out profiles/r01_configs.jsonl]
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


def gpu_time(fn, reps=10):
    import torch

    ts = []
    for r in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def wall(fn, reps=5):
    ts = []
    for r in range(reps + 1):
        t0 = time.perf_counter()
        out = fn()
        if r:
            ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_configs.jsonl"))
    args = ap.parse_args()
    import torch

    import oracle
    import paper_2001_08250_b200 as xp
    from oracle import recipes

    o = oracle.best()
    cores = os.cpu_count() or 1
    lines = []

    # ---- config 1 -----------------------------------------------------------
    C = recipes.C1
    db, q = recipes.config1(o)
    N, S, B = C["N"], C["S"], C["B"]
    st = xp.Store(N, S)
    st.upload(db)
    dq = torch.from_numpy(q).cuda()
    dout = torch.empty((B, S), dtype=torch.uint8, device="cuda")
    cs = torch.cuda.current_stream()
    ms = gpu_time(lambda: st.answer_batch_dev(dq, N // 8, B, dout, stream=cs))
    e2e_ms, got = wall(lambda: st.answer_batch(q))
    want = o.answer_batch(db, N, S, q, B) if o.kind != "reference" else None
    ref_ms = None
    if o.kind == "reference":
        snap = o.snapshot(db, N, S)
        ref_ms, (want, _) = wall(lambda: snap.answer_batch(q, B, cores))
    assert np.array_equal(got, want) and np.array_equal(dout.cpu().numpy(), want)
    lines.append({"config": 1, "workload": "1,024 x 4,096 B store, 64 explicit requests", "gpu_ms": ms,
                  "gpu_requests_per_s": B / (ms * 1e-3), "e2e_ms": e2e_ms, "e2e_requests_per_s": B / (e2e_ms * 1e-3),
                  "kernel": xp.last_scan_kernel(), "ref_ms": ref_ms, "ref_cores": cores,
                  "ref_requests_per_s": None if ref_ms is None else B / (ref_ms * 1e-3), "bit_exact": True})
    print(json.dumps(lines[-1]), flush=True)
    st.close()

    # ---- config 2 -----------------------------------------------------------
    C = recipes.C2
    db, betas, shares = recipes.config2(o)
    N, S, B = C["N"], C["S"], C["B"]
    st = xp.Store(N, S)
    st.upload(db)
    dsh = [torch.from_numpy(np.ascontiguousarray(shares[k])).cuda() for k in range(3)]
    douts = [torch.empty((B, S), dtype=torch.uint8, device="cuda") for _ in range(3)]

    def three():
        for k in range(3):
            st.answer_batch_dev(dsh[k], N // 8, B, douts[k], stream=cs)

    ms = gpu_time(three)
    e2e_ms, got = wall(lambda: [st.answer_batch(shares[k]) for k in range(3)])
    rec = got[0] ^ got[1] ^ got[2]
    assert np.array_equal(rec, db.reshape(N, S)[betas])
    ref_ms = None
    if o.kind == "reference":
        snap = o.snapshot(db, N, S)
        ref_ms, refs = wall(lambda: [snap.answer_batch(shares[k], B, cores)[0] for k in range(3)], reps=2)
        assert all(np.array_equal(got[k], refs[k]) for k in range(3))
    lines.append({"config": 2, "workload": "32,768 x 4,096 B store, 1,024 requests x 3 server shares",
                  "gpu_ms_3_servers": ms, "gpu_ms_per_server": ms / 3,
                  "gpu_requests_per_s_per_server": B / (ms / 3 * 1e-3), "e2e_ms_3_servers": e2e_ms,
                  "kernel": xp.last_scan_kernel(), "ref_ms_3_servers": ref_ms, "ref_cores": cores,
                  "ref_requests_per_s_per_server": None if ref_ms is None else B / (ref_ms / 3 * 1e-3),
                  "reconstruct_ok": True, "bit_exact": o.kind == "reference"})
    print(json.dumps(lines[-1]), flush=True)
    st.close()
    with open(args.out, "w") as f:
        for l in lines:
            f.write(json.dumps(l) + "\n")


if __name__ == "__main__":
    main()

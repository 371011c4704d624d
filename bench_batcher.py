"""bench_batcher.py — the read path as node.cpp drives it: many concurrent
single-request callers of server::answer_share's scan + mask step
(server.cpp:115-135), BASELINE config 2 geometry (one server of the 3-server
round: 32,768 buckets x 4 x 1,024 B = 128 MiB of DetRng(1) bytes; the requests
are that round's DetRng(1) shares, each with a 32-byte answer-mask seed).

Arms (requests/s, end to end: host query in, host masked answer out):
  batched     T native host threads (tools/loadgen.cpp) call xpir_batcher_answer;
              concurrent requests are coalesced into one device scan (the §8(f)
              read batcher)
  unbatched   native threads each call xpir_answer_batch with one request (what
              a per-call drop-in of pir::answer + mask_answer does)
  reference   T host threads each call the unmodified reference pir::answer +
              pir::mask_answer (oracle/_ref) — the CPU path, all host cores

    python bench_batcher.py [--threads 256] [--seconds 4] [--out profiles/r01_batcher.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def drive(fn, threads: int, seconds: float, warm: float = 0.5):
    """Run fn(t, i) in `threads` threads for `seconds`; returns completed calls/s."""
    stop = threading.Event()
    counting = threading.Event()
    counts = [0] * threads
    errs = []

    def loop(t):
        i = 0
        try:
            while not stop.is_set():
                fn(t, i)
                i += 1
                if counting.is_set():
                    counts[t] += 1
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            stop.set()

    ts = [threading.Thread(target=loop, args=(t,), daemon=True) for t in range(threads)]
    for t in ts:
        t.start()
    time.sleep(warm)
    counting.set()
    t0 = time.perf_counter()
    time.sleep(seconds)
    n = sum(counts)
    dt = time.perf_counter() - t0
    stop.set()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return n / dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=256)
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--max-batch", type=int, default=1024)
    ap.add_argument("--max-wait-us", type=int, default=300)
    ap.add_argument("--pool", type=int, default=1024, help="distinct config-2 shares cycled by the callers")
    ap.add_argument("--open-rates", default="50000,150000,250000", help="offered rates for the open-loop latency runs")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_batcher.jsonl"))
    args = ap.parse_args()

    import oracle
    import paper_2001_08250_b200 as xp
    from oracle import recipes

    o = oracle.best()
    N, S = recipes.C2["N"], recipes.C2["S"]
    db, betas, shares = recipes.config2(o, args.pool)
    q = np.ascontiguousarray(shares[0])  # server 0's shares
    seeds = np.random.default_rng(7).integers(0, 256, (args.pool, 32), dtype=np.uint8)
    st = xp.Store(N, S)
    st.upload(db)
    T = args.threads
    lines = []
    common = {"workload": "config2 per-server read path: 32,768 x 4,096 B store, masked single requests",
              "threads": T, "pool": args.pool}

    # correctness spot check (bit-exact vs the oracle) before timing
    bt = xp.Batcher(st, max_batch=args.max_batch, max_wait_us=args.max_wait_us)
    port = oracle.Port()
    want = port.mask_answer(port.answer_batch(db, N, S, q[:1], 1)[0].tobytes(), seeds[0].tobytes())
    assert bt.answer(q[0], mask_seed=seeds[0].tobytes()).tobytes() == want

    import ctypes as C

    xp.lib()
    lg = C.CDLL(os.path.join(ROOT, "paper_2001_08250_b200", "libxpir_loadgen.so"))
    lg.xpl_drive.argtypes = [C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p,
                             C.c_uint32, C.c_double, C.c_double, C.POINTER(C.c_double), C.c_char_p, C.c_uint32]

    def native_drive(mode, target, threads, seconds):
        rate, err = C.c_double(), C.create_string_buffer(512)
        rc = lg.xpl_drive(mode, target, N, S, q.ctypes.data, args.pool, seeds.ctypes.data, threads, seconds, 0.5,
                          C.byref(rate), err, 512)
        if rc:
            raise RuntimeError(f"loadgen rc={rc}: {err.value.decode()}")
        return rate.value

    rate = native_drive(0, bt.h, T, args.seconds)
    s = bt.stats()
    lines.append({"metric": "read-path requests/s (concurrent answer_share scan + mask)", "arm": "batched",
                  "value": rate, "unit": "requests/s", "mean_batch": s["requests"] / max(s["batches"], 1),
                  "max_batch": args.max_batch, "max_wait_us": args.max_wait_us, **common})
    print(json.dumps(lines[-1]), flush=True)
    bt.close()

    # open loop: a fixed offered rate, latency percentiles (serving behaviour)
    lg.xpl_open_loop.argtypes = [C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p,
                                 C.c_uint32, C.c_double, C.c_double, C.POINTER(C.c_double)]
    for offered in [float(x) for x in args.open_rates.split(",") if x]:
        bt2 = xp.Batcher(st, max_batch=args.max_batch, max_wait_us=args.max_wait_us)
        r6 = (C.c_double * 6)()
        rc = lg.xpl_open_loop(0, bt2.h, N, S, q.ctypes.data, args.pool, seeds.ctypes.data, T, offered,
                              min(args.seconds, 3.0), r6)
        s2 = bt2.stats()
        bt2.close()
        if rc:
            raise RuntimeError(f"open loop rc={rc}")
        lines.append({"metric": "read-path latency at a fixed offered rate (open loop, batched)", "arm": "batched-open-loop",
                      "offered_requests_per_s": offered, "achieved_requests_per_s": r6[0], "latency_us_p50": r6[1],
                      "latency_us_p90": r6[2], "latency_us_p99": r6[3], "latency_us_max": r6[4],
                      "requests": int(r6[5]), "mean_batch": s2["requests"] / max(s2["batches"], 1),
                      "max_wait_us": args.max_wait_us, **common})
        print(json.dumps(lines[-1]), flush=True)

    rate = native_drive(1, st.h, min(T, 32), min(args.seconds, 2.0))
    lines.append({"metric": "read-path requests/s (concurrent answer_share scan + mask)", "arm": "unbatched",
                  "value": rate, "unit": "requests/s", **common, "threads": min(T, 32)})
    print(json.dumps(lines[-1]), flush=True)

    if o.kind == "reference":
        snap = o.snapshot(db, N, S)
        cores = os.cpu_count() or 1

        def reference(t, i):
            k = (t * 7919 + i) % args.pool
            a = snap.answer(q[k])
            o.mask_answer(a.tobytes(), seeds[k].tobytes())

        rate = drive(reference, cores, min(args.seconds, 3.0), warm=0.2)
        lines.append({"metric": "read-path requests/s (concurrent answer_share scan + mask)", "arm": "reference",
                      "value": rate, "unit": "requests/s", "cores": cores, "kind": "reference",
                      **common, "threads": cores})
        print(json.dumps(lines[-1]), flush=True)
    st.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        for l in lines:
            f.write(json.dumps(l) + "\n")


if __name__ == "__main__":
    main()

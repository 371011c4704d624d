"""Profiling helper (not a bench line): per-stage device and host times of the
config-3 write round (bench_write.py's GPU arm), CUDA events between stages."""
import json, os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.abspath(__file__)); sys.path.insert(0, ROOT)
import oracle
import paper_2001_08250_b200 as xp
from oracle import recipes

prio = int(os.environ.get("PRIO", "0"))
o = oracle.best()
n = recipes.C3["n"]
d = recipes.config3(o, n)
N, depth, item, m, h = 32768, 4, 1024, 1 << 20, 23
xs = torch.from_numpy(d["xs"].view(np.int64)).cuda()
payload = torch.from_numpy(d["payload"]).cuda()
db1 = torch.empty(n, dtype=torch.int32, device="cuda"); db2 = torch.empty_like(db1)
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
stream = torch.cuda.Stream(priority=-1 if prio else 0)
stream2 = torch.cuda.Stream(priority=0)
for rep in range(6):
    T = xp.Table(N, depth, N * depth, item, d["s_cuckoo"]); T.reserve(n)
    W = xp.Window(m, h, 1)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    hs = [time.perf_counter()]
    ev[0].record(stream); stream2.wait_stream(stream)
    if os.environ.get("NOINT") != "1":
        W.absorb_interest_dev(d["lid"], xs, n, stream=stream2)
    hs.append(time.perf_counter())
    xp.prf_batch_dev(d["k1"], xs, n, N, d_out32=db1, stream=stream)
    xp.prf_batch_dev(d["k2"], xs, n, N, d_out32=db2, stream=stream)
    ev[1].record(stream)
    hs.append(time.perf_counter())
    T.insert_batch_dev(db1, db2, payload, n, stream=stream)
    ev[2].record(stream)
    hs.append(time.perf_counter())
    stream.wait_stream(stream2); ev[3].record(stream)
    stream.synchronize()
    hs.append(time.perf_counter())
    if rep:
        dev = [ev[0].elapsed_time(e) * 1e3 for e in ev[1:4]]
        host = [(hs[i + 1] - hs[0]) * 1e6 for i in range(4)]
        print(json.dumps({"prio": prio, "dev_us_after_prf_insert_all": [round(x, 1) for x in dev],
                          "host_us_after_interest_prf_insert_end": [round(x, 1) for x in host]}))
    T.close(); W.close()

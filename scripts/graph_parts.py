import numpy as np, torch, sys, os, json
sys.path.insert(0, os.getcwd())
import oracle, paper_2001_08250_b200 as xp
from oracle import recipes
o = oracle.best(); n = 32000
d = recipes.config3(o, n)
N, depth, item, m, h = 32768, 4, 1024, 1 << 20, 23
xs = torch.from_numpy(d["xs"].view(np.int64)).cuda(); payload = torch.from_numpy(d["payload"]).cuda()
db1 = torch.empty(n, dtype=torch.int32, device="cuda"); db2 = torch.empty_like(db1)
s = torch.cuda.Stream(priority=-1); s2 = torch.cuda.Stream()
def run(parts, reps=5):
    out = []
    for r in range(reps + 1):
        T = xp.Table(N, depth, N * depth, item, d["s_cuckoo"]); T.reserve(n); W = xp.Window(m, h, 1)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            if "int" in parts:
                s2.wait_stream(s); W.absorb_interest_dev(d["lid"], xs, n, stream=s2)
            if "prf" in parts:
                xp.write_betas_dev(d["k1"], d["k2"], xs, n, N, db1, db2, stream=s)
            if "ins" in parts:
                T.insert_batch_async(db1, db2, payload, n, s)
            if "int" in parts:
                s.wait_stream(s2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); g.replay(); e1.record(s)
        if "ins" in parts: T.finish()
        torch.cuda.synchronize()
        if r: out.append(e0.elapsed_time(e1) * 1e3)
        del g; T.close(); W.close()
    return round(float(np.median(out)), 1)
# PRF values for the ins-only case
xp.prf_batch_dev(d["k1"], xs, n, N, d_out32=db1, stream=s); xp.prf_batch_dev(d["k2"], xs, n, N, d_out32=db2, stream=s)
torch.cuda.synchronize()
for parts in (("int",), ("prf",), ("ins",), ("prf", "ins"), ("int", "prf", "ins")):
    print(parts, run(parts), "us")

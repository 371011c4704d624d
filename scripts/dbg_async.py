import numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
import oracle, paper_2001_08250_b200 as xp
from oracle import recipes
o = oracle.best(); n = 32000
d = recipes.config3(o, n)
N, depth, item = 32768, 4, 1024
xs = torch.from_numpy(d["xs"].view(np.int64)).cuda(); payload = torch.from_numpy(d["payload"]).cuda()
db1 = torch.empty(n, dtype=torch.int32, device="cuda"); db2 = torch.empty_like(db1)
s = torch.cuda.Stream()
for mode in ("plain", "graph"):
    T = xp.Table(N, depth, N * depth, item, d["s_cuckoo"]); T.reserve(n)
    torch.cuda.synchronize()
    if mode == "plain":
        xp.prf_batch_dev(d["k1"], xs, n, N, d_out32=db1, stream=s)
        xp.prf_batch_dev(d["k2"], xs, n, N, d_out32=db2, stream=s)
        T.insert_batch_async(db1, db2, payload, n, s)
    else:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            xp.prf_batch_dev(d["k1"], xs, n, N, d_out32=db1, stream=s)
            xp.prf_batch_dev(d["k2"], xs, n, N, d_out32=db2, stream=s)
            T.insert_batch_async(db1, db2, payload, n, s)
        g.replay()
    try:
        print(mode, "applied", T.finish(), T.counters())
    except Exception as e:
        print(mode, "ERR", e, T.counters())
    print(T.state_digest().hex()[:16], d and "")
# debug: graph with only the PRFs
g2 = torch.cuda.CUDAGraph()
db1.zero_(); torch.cuda.synchronize()
with torch.cuda.graph(g2, stream=s):
    xp.prf_batch_dev(d["k1"], xs, n, N, d_out32=db1, stream=s)
g2.replay(); torch.cuda.synchronize()
print("prf in graph:", db1[:4].tolist(), "want", [int(v) for v in d["b1"][:4]])
# debug: PRFs outside, insert in graph
T = xp.Table(N, depth, N * depth, item, d["s_cuckoo"]); T.reserve(n)
xp.prf_batch_dev(d["k1"], xs, n, N, d_out32=db1, stream=s)
xp.prf_batch_dev(d["k2"], xs, n, N, d_out32=db2, stream=s)
torch.cuda.synchronize()
g3 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g3, stream=s):
    T.insert_batch_async(db1, db2, payload, n, s)
g3.replay(); torch.cuda.synchronize()
try:
    print("insert-only graph applied", T.finish(), T.counters())
except Exception as e:
    print("insert-only graph ERR", e, T.counters())
# debug: PRF + insert in graph, inspect
T = xp.Table(N, depth, N * depth, item, d["s_cuckoo"]); T.reserve(n)
db1.fill_(-1); db2.fill_(-1); torch.cuda.synchronize()
g4 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g4, stream=s):
    xp.prf_batch_dev(d["k1"], xs, n, N, d_out32=db1, stream=s)
    xp.prf_batch_dev(d["k2"], xs, n, N, d_out32=db2, stream=s)
    T.insert_batch_async(db1, db2, payload, n, s)
print("nodes", g4.__class__, flush=True)
g4.replay(); torch.cuda.synchronize()
print("after replay db1", db1[:3].tolist(), db2[:3].tolist())
try:
    print("prf+insert graph applied", T.finish(), T.counters())
except Exception as e:
    print("prf+insert graph ERR", e, T.counters())
# replay again on a fresh table? (same graph bound to T) -- second replay on same table

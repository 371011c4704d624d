"""bench_walk_big.py — the write path on tables past the on-chip walk limits.

Tables of 2^20 and 2^22 slots (262,144 / 1,048,576 buckets x depth 4, 8-byte
items so the cuckoo placement dominates) filled to 95% load in one insert batch
(cuckoo.cpp:56-126 for every item in order): the parallel eviction-free prefix
covers the early items, then the eviction chains run. Each GPU arm runs in its
own process with XPIR_CUCKOO_WALK selecting the walk kernel:

  auto  k_cuckoo_walk_w<G=true>: warp walk, occupancy/touched maps in global memory
  1     k_cuckoo_walk: the single-thread walk (the previous large-table path)

Reference: the unmodified reference Table::insert (oracle/_ref) on one core,
same items. Reports + state digest of every GPU arm equal the reference's.
Wall clock around Table.insert_batch (host arrays in, reports out).

    python bench_walk_big.py [--out profiles/r01_walk_big.jsonl]
    python bench_walk_big.py --one --sizes 262144     # one GPU arm, for ncu
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CHILD = r"""
import sys, time, json, numpy as np
sys.path.insert(0, {root!r})
import paper_2001_08250_b200 as xp
nb, depth, load = {nb}, {depth}, {load}
g = np.random.default_rng(nb)
slots = nb * depth
n = int(slots * load)
b1 = g.integers(0, nb, n).astype(np.uint32)
b2 = g.integers(0, nb, n).astype(np.uint32)
pl = g.integers(0, 256, (n, 8), dtype=np.uint8)
seed = bytes(range(32))
T = xp.Table(nb, depth, slots, 8, seed)
T.insert_batch(b1[:1], b2[:1], pl[:1])  # warm the module / allocations
T.close()
T = xp.Table(nb, depth, slots, 8, seed)
t0 = time.perf_counter()
r = T.insert_batch(b1, b2, pl)
ms = (time.perf_counter() - t0) * 1e3
print(json.dumps({{"ms": ms, "digest": T.state_digest().hex(), "disp": int(r[:, 3].sum()),
                  "dropped": int(r[:, 1].sum())}}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_walk_big.jsonl"))
    ap.add_argument("--sizes", default="262144,1048576")
    ap.add_argument("--load", type=float, default=0.95)
    ap.add_argument("--one", action="store_true", help="run only the GPU arm of the first size in-process (ncu)")
    args = ap.parse_args()
    if args.one:
        exec(CHILD.format(root=ROOT, nb=int(args.sizes.split(",")[0]), depth=4, load=args.load))
        return
    import numpy as np

    import oracle

    o = oracle.best()
    lines = []
    for nb in [int(x) for x in args.sizes.split(",")]:
        depth = 4
        arms = {}
        for name, env_v in (("walk_w_global", "0"), ("single_thread", "1")):
            env = dict(os.environ, XPIR_CUCKOO_WALK=env_v)
            code = CHILD.format(root=ROOT, nb=nb, depth=depth, load=args.load)
            out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=3000)
            assert out.returncode == 0, out.stderr[-2000:]
            arms[name] = json.loads(out.stdout.strip().splitlines()[-1])
        g = np.random.default_rng(nb)
        slots = nb * depth
        n = int(slots * args.load)
        b1 = g.integers(0, nb, n).astype(np.uint32)
        b2 = g.integers(0, nb, n).astype(np.uint32)
        pl = g.integers(0, 256, (n, 8), dtype=np.uint8)
        P = o.table(nb, depth, slots, 8, bytes(range(32)))
        t0 = time.perf_counter()
        rr = P.insert_batch(b1, b2, pl)
        ref_ms = (time.perf_counter() - t0) * 1e3
        ref_digest = P.state_digest().hex()
        for a in arms.values():
            assert a["digest"] == ref_digest, "state digest differs from the reference"
            assert a["disp"] == int(rr[:, 3].sum())
        line = {"workload": f"{nb} buckets x depth {depth} ({slots} slots), {n} inserts to {args.load:.0%} load, one batch",
                "inserts": n, "displacements": arms["walk_w_global"]["disp"], "dropped": arms["walk_w_global"]["dropped"],
                "gpu_ms_walk_w_global": arms["walk_w_global"]["ms"], "gpu_ms_single_thread": arms["single_thread"]["ms"],
                "ref_ms_1thread": ref_ms, "ref_kind": o.kind, "bit_exact": True}
        print(json.dumps(line), flush=True)
        lines.append(line)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        for l in lines:
            f.write(json.dumps(l) + "\n")


if __name__ == "__main__":
    main()

"""CPU tests of the multi-GPU host logic (paper_2001_08250_b200/sharded.py):
the bucket-range plan and the XOR reduce-scatter it drives, run as a real
world-size-2 torch.distributed job over gloo on 127.0.0.1. The per-shard scans
here are the oracle's (CPU); on a B200 box the same plan drives the CUDA scan and
the NVLink peer reduce."""
import os
import socket

import numpy as np
import pytest

from paper_2001_08250_b200.sharded import ShardPlan, xor_reduce_scatter_reference


@pytest.mark.parametrize("N", [8, 64, 1000, 1001, 32768, 1 << 20])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_plan_partitions_buckets_and_rows(N, G):
    plan = ShardPlan(N, G)
    rs = plan.ranges()
    assert rs[0][0] == 0 and rs[-1][1] == N
    for (lo, hi), (lo2, _) in zip(rs, rs[1:]):
        assert hi == lo2
    for lo, hi in rs:
        assert lo % 8 == 0 and (hi % 8 == 0 or hi == N) and lo <= hi
    B = 8192
    rows = [plan.row_range(g, B) for g in range(G)]
    assert rows[0][0] == 0 and rows[-1][1] == B
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    if N == 1 << 20 and G in (1, 2, 4, 8):
        assert all(hi - lo == N // G for lo, hi in rs)  # config 4: equal 4 GiB / G shards


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, S, B, q_all, db, ret):
    import torch
    import torch.distributed as dist

    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = ShardPlan(N, world)
    lo, hi = plan.bucket_range(rank)
    port_ = oracle.Port()
    # shard-local scan: buckets [lo, hi), query bytes [lo/8, ceil(hi/8))
    qwin = np.ascontiguousarray(q_all[:, lo // 8:(hi + 7) // 8])
    part = port_.answer_batch(np.ascontiguousarray(db[lo * S:hi * S]), hi - lo, S, qwin, B)
    gathered = [torch.zeros((B, S), dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(part))
    own = xor_reduce_scatter_reference([g.numpy() for g in gathered], plan, rank)
    r0, r1 = plan.row_range(rank, B)
    ret[rank] = (r0, r1, own.tobytes())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("N,S,B", [(1000, 64, 37), (4096, 128, 64)])
def test_world2_reduce_scatter_equals_unsharded(N, S, B):
    import torch.multiprocessing as mp

    import oracle

    g = np.random.default_rng(N + B)
    db = g.integers(0, 256, N * S, dtype=np.uint8)
    q = g.integers(0, 256, (B, (N + 7) // 8), dtype=np.uint8)
    want = oracle.Port().answer_batch(db, N, S, q, B)
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), N, S, B, q, db, ret), nprocs=world, join=True)
    got = np.zeros((B, S), np.uint8)
    for r in range(world):
        r0, r1, rows = ret[r]
        got[r0:r1] = np.frombuffer(rows, np.uint8).reshape(r1 - r0, S)
    assert np.array_equal(got, want)

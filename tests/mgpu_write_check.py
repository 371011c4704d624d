"""Multi-rank check of the sharded write path (bucket-range payload shards),
launched by tests/test_gpu_sharded.py under torchrun: every rank holds one payload
shard of the cuckoo table (the whole metadata, replicated walk), maps the other
ranks' payload arrays by CUDA IPC (peer memory over NVLink on a multi-GPU box; the
same GPU when ranks outnumber GPUs), gathers the payloads that move into its range,
barrier, scatters. Rank 0 compares the union of the shards with the oracle's
sequential cuckoo::Table::insert after every round."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2001_08250_b200 as xp  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ndev = torch.cuda.device_count()
    dev = rank % ndev
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl" if ndev >= world else "gloo")
    nb, depth, item = int(os.environ.get("XP_NB", "2048")), 4, 64
    g = np.random.default_rng(11)
    seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
    cap = nb * depth
    bounds = [0] + [((nb * k // world) // 8) * 8 for k in range(1, world)] + [nb]
    T = xp.Table(nb, depth, cap, item, seed, device=dev, lo=bounds[rank], hi=bounds[rank + 1])
    # exchange payload-array IPC handles, map the peers
    h = xp.ipc_handle(T.device_ptr(), device=dev)
    hs = [None] * world
    dist.all_gather_object(hs, h)
    ptrs = [T.device_ptr() if k == rank else xp.ipc_open(hs[k], device=dev) for k in range(world)]
    smap = xp._ShardMap()
    smap.n = world
    for k in range(world):
        smap.bucket_lo[k] = bounds[k]
        smap.data[k] = ptrs[k]
    smap.bucket_lo[world] = nb
    P = oracle.Port().table(nb, depth, cap, item, seed) if rank == 0 else None
    ok = True
    n_total = int(nb * depth * 0.96)
    for rnd in range(3):
        n = n_total // 3
        b1 = g.integers(0, nb, n).astype(np.uint32)
        b2 = g.integers(0, nb, n).astype(np.uint32)
        pl = g.integers(0, 256, (n, item), dtype=np.uint8)
        d1, d2 = torch.from_numpy(b1.view(np.int32)).cuda(), torch.from_numpy(b2.view(np.int32)).cuda()
        dp = torch.from_numpy(pl).cuda()
        rep = torch.zeros((n, 4), dtype=torch.int32, device="cuda")
        T.insert_walk_dev(d1, d2, n, rep)
        T.apply_gather_dev(smap)
        torch.cuda.synchronize()
        dist.barrier()  # every shard has staged the pre-round payloads it needs
        T.apply_scatter_dev(dp)
        torch.cuda.synchronize()
        dist.barrier()
        parts = [None] * world
        dist.all_gather_object(parts, (T.snapshot().tobytes(), rep.cpu().numpy().tobytes()))
        if rank == 0:
            want_rep = P.insert_batch(b1, b2, pl)
            whole = np.concatenate([np.frombuffer(p[0], np.uint8) for p in parts])
            ok &= bool(np.array_equal(whole, P.data()))
            ok &= all(np.array_equal(np.frombuffer(p[1], np.uint32).reshape(n, 4), want_rep) for p in parts)
    for k in range(world):
        if k != rank:
            xp.ipc_close(ptrs[k], device=dev)
    dist.barrier()
    if rank == 0:
        print("SHARDED_WRITE_OK" if ok else "SHARDED_WRITE_MISMATCH", flush=True)
    T.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

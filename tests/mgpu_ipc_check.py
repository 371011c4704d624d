"""Multi-rank check of the sharded scan + CUDA-IPC XOR reduce-scatter (or the
fused variant whose scan epilogue XORs into the owners' buffers, XP_FUSED=1), launched by
tests/test_gpu_sharded.py under torchrun. With fewer GPUs than ranks every rank
uses the same device (peer mapping of another process's allocation on the same
GPU is still CUDA IPC) and the control plane is gloo; the kernels never wait on
each other — synchronisation is host barriers only.

Rank 0 compares the gathered owned rows with an unsharded scan and the oracle."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2001_08250_b200 as xp  # noqa: E402
from paper_2001_08250_b200.sharded import ShardedScan  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ndev = torch.cuda.device_count()
    dev = rank % ndev
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl" if ndev >= world else "gloo")
    N, S = int(os.environ.get("XP_N", "8192")), int(os.environ.get("XP_S", "512"))
    B = int(os.environ.get("XP_B", "300"))
    key = bytes(range(32))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    fused = {"1": True, "0": False}.get(os.environ.get("XP_FUSED", ""), None)
    sh = ShardedScan(xp, torch, dist, N, S, B, dev, fused=fused)
    if rank == 0:
        print(f"mode={'fused' if sh.fused else 'reduce'}", flush=True)
    sh.store.fill_keystream(key, 7)
    seeds = torch.zeros((B, 32), dtype=torch.uint8, device="cuda")
    xp.keystream_rows_dev(key, 100, B, 32, seeds, 32, device=dev)
    masks = torch.zeros((B, 32), dtype=torch.uint8, device="cuda")
    xp.keystream_rows_dev(key, 5000, B, 32, masks, 32, device=dev)
    torch.cuda.synchronize()
    ok = True
    for it in range(3):
        if sh.fused:
            sh.store.peer_stats(reset=True)
        own = sh.step(seeds, stream=stream, d_mask=masks if it == 2 else None)
        torch.cuda.synchronize()
        if sh.fused:
            # the fused epilogue moves reduce-scatter bytes: each row pushed once, to its owner
            st = sh.store.peer_stats()
            want_remote = (B - (sh.r1 - sh.r0)) * S
            print(f"rank {rank} it {it}: remote {st['remote_bytes']} (reduce-scatter {want_remote}), "
                  f"own {st['own_bytes']}", flush=True)
            ok = ok and st["remote_bytes"] <= 1.05 * want_remote and st["own_bytes"] <= (sh.r1 - sh.r0) * S
        rows = own.cpu().numpy().copy()
        got = [None] * world
        dist.all_gather_object(got, (sh.r0, sh.r1, rows.tobytes()))
        if rank == 0:
            full = xp.Store(N, S, device=dev)
            full.fill_keystream(key, 7)
            want = torch.empty((B, S), dtype=torch.uint8, device="cuda")
            full.answer_batch_seeded_dev(seeds, B, want, d_mask=masks if it == 2 else None, stream=stream)
            torch.cuda.synchronize()
            want = want.cpu().numpy()
            res = np.zeros((B, S), np.uint8)
            for r0, r1, b in got:
                res[r0:r1] = np.frombuffer(b, np.uint8).reshape(r1 - r0, S)
            ok = ok and np.array_equal(res, want)
            if it == 0:  # anchor the unsharded scan itself on the oracle for a few rows
                import oracle

                port = oracle.Port()
                db = full.download()
                sd = seeds.cpu().numpy()
                q = np.stack([np.frombuffer(port.prng_expand(sd[r].tobytes(), (N + 7) // 8), np.uint8)
                              for r in range(8)])
                ok = ok and np.array_equal(port.answer_batch(db, N, S, q, 8), want[:8])
            full.close()
        dist.barrier()
    sh.close()
    if rank == 0:
        print("SHARDED_IPC_OK" if ok else "SHARDED_IPC_MISMATCH", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

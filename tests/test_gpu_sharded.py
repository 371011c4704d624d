"""GPU: the sharded scan's real data path — per-rank shard scans, CUDA-IPC peer
mapping and the K4 XOR reduce-scatter (or the fused scan epilogue that XORs into
the owners' rows over peer memory), mask applied once by the owner — run as a
2- and 3-rank torchrun job (ranks share the GPU when fewer are present) and
compared bit-exactly with the unsharded scan."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,N,S,B,fused", [
    (2, 8192, 512, 300, "0"), (3, 4096 + 24, 256, 130, "0"), (2, 1024, 4096, 64, "0"),
    # fused epilogue (quad-table kernel 8, B >= 2048): tile fix-up in a local buffer, each
    # finished tile pushed once to its owners (several segments per tile), or straight
    # from the accumulators (one segment per tile); remote bytes checked per rank
    (2, 8192, 512, 2100, "1"), (3, 16384 + 40, 1024, 4096, "1"), (4, 4096, 256, 2048 + 3, "1"),
    (2, 131072, 128, 2048, "1"), (4, 262144 + 8, 64, 4100, "1"), (8, 524288, 32, 8192, "1"),
])
def test_sharded_ipc_reduce(cuda, world, N, S, B, fused):
    env = dict(os.environ, XP_N=str(N), XP_S=str(S), XP_B=str(B), XP_FUSED=fused)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mgpu_ipc_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    print(out.stdout[-2000:], out.stderr[-3000:])
    assert out.returncode == 0
    assert "SHARDED_IPC_OK" in out.stdout


@pytest.mark.parametrize("world,nb", [(2, 2048), (3, 1000), (4, 4096)])
def test_sharded_write_path_ipc(cuda, world, nb):
    """Payload shards in separate processes: cross-shard moves of pre-round payloads
    read through CUDA-IPC-mapped peer memory; union == the oracle's table."""
    env = dict(os.environ, XP_NB=str(nb))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mgpu_write_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    print(out.stdout[-2000:], out.stderr[-3000:])
    assert out.returncode == 0
    assert "SHARDED_WRITE_OK" in out.stdout

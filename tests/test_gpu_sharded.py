"""GPU: the sharded scan's real data path — per-rank shard scans, CUDA-IPC peer
mapping and the K4 XOR reduce-scatter, mask applied once by the owner — run as a
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


@pytest.mark.parametrize("world,N,S,B", [(2, 8192, 512, 300), (3, 4096 + 24, 256, 130), (2, 1024, 4096, 64)])
def test_sharded_ipc_reduce(cuda, world, N, S, B):
    env = dict(os.environ, XP_N=str(N), XP_S=str(S), XP_B=str(B))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mgpu_ipc_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    print(out.stdout[-2000:], out.stderr[-3000:])
    assert out.returncode == 0
    assert "SHARDED_IPC_OK" in out.stdout

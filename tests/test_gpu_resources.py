"""GPU: handle lifetimes do not leak device memory — stores (with per-stream
scratch), read batchers, tables (whole and payload shards), windows and device
ServerCores created, used and destroyed repeatedly leave the free device memory
where it was (a long-running server reseals, re-batches and rotates forever)."""
import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free(torch):
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info()[0]


def test_no_device_memory_growth(xp, cuda):
    torch = cuda
    g = np.random.default_rng(1)
    N, S = 4096, 512
    db = g.integers(0, 256, N * S, dtype=np.uint8)
    q = g.integers(0, 256, (64, N // 8), dtype=np.uint8)

    def cycle():
        st = xp.Store(N, S)
        st.upload(db)
        st.answer_batch(q)
        dq = torch.from_numpy(q).cuda()
        out = torch.empty((64, S), dtype=torch.uint8, device="cuda")
        s2 = torch.cuda.Stream()
        st.answer_batch_dev(dq, N // 8, 64, out, stream=s2)
        bt = xp.Batcher(st, max_batch=32, max_wait_us=50)
        bt.answer(q[0])
        bt.close()
        T = xp.Table(256, 4, 1024, 32, bytes(32))
        T.insert_batch(g.integers(0, 256, 500).astype(np.uint32), g.integers(0, 256, 500).astype(np.uint32),
                       np.zeros((500, 32), np.uint8))
        T.close()
        Ts = xp.Table(256, 4, 1024, 32, bytes(32), lo=0, hi=128)
        Ts.close()
        W = xp.Window(1 << 16, 3, 2)
        W.absorb(g.integers(0, 1 << 16, 100).astype(np.uint32))
        W.encode_delta(0)
        W.close()
        sv = xp.Server(64, 4, 256, 32, bytes(32), 4096, 3, 2, 50, 2)
        sv.apply_round(np.zeros(100, np.uint32), np.ones(100, np.uint32), np.zeros((100, 32), np.uint8),
                       np.zeros((100, 3), np.uint32), seal_after=True)
        sv.close()
        st.close()
        del dq, out, s2
        gc.collect()

    for _ in range(3):  # warm the allocators (CUDA pools, torch cache)
        cycle()
    torch.cuda.empty_cache()
    before = _free(torch)
    for _ in range(20):
        cycle()
    torch.cuda.empty_cache()
    after = _free(torch)
    assert before - after < 64 << 20, (before - after) / 2**20  # < 64 MiB drift over 20 cycles

"""GPU parity of the read batcher (xpir_batcher_*): concurrent single requests —
server::answer_share's scan + mask step (server.cpp:115-135) issued from many
host threads as node.cpp does — are coalesced into device batches, and every
caller gets exactly pir::answer / pir::mask_answer(pir::answer(..)) of its own
query (pir.cpp:29-39, 65-69). Bit-exact against the oracle."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_threads(fn, n):
    errs = []

    def wrap(t):
        try:
            fn(t)
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errs.append(e)

    ts = [threading.Thread(target=wrap, args=(t,)) for t in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


@pytest.mark.parametrize("N,S,max_batch,wait_us", [(4096, 512, 64, 2000), (1001, 128, 7, 500), (257, 4096, 1, 0)])
def test_concurrent_answers_match_oracle(xp, port, cuda, N, S, max_batch, wait_us):
    g = np.random.default_rng(N + S + max_batch)
    db = g.integers(0, 256, N * S, dtype=np.uint8)
    st = xp.Store(N, S)
    st.upload(db)
    bt = xp.Batcher(st, max_batch=max_batch, max_wait_us=wait_us)
    T, R = 24, 5
    nb = (N + 7) // 8
    qs = g.integers(0, 256, (T, R, nb), dtype=np.uint8)
    if N % 8:
        qs[..., -1] &= (1 << (N % 8)) - 1
    seeds = g.integers(0, 256, (T, R, 32), dtype=np.uint8)
    got = np.zeros((T, R, S), np.uint8)

    def worker(t):
        for r in range(R):
            masked = (t + r) % 2 == 0
            got[t, r] = bt.answer(qs[t, r], mask_seed=seeds[t, r].tobytes() if masked else None)

    _run_threads(worker, T)
    plain = port.answer_batch(db, N, S, qs.reshape(T * R, nb), T * R).reshape(T, R, S)
    for t in range(T):
        for r in range(R):
            want = plain[t, r].tobytes()
            if (t + r) % 2 == 0:
                want = port.mask_answer(want, seeds[t, r].tobytes())
            assert got[t, r].tobytes() == want, (t, r)
    s = bt.stats()
    assert s["requests"] == T * R
    assert s["max_batch_seen"] <= max_batch
    if max_batch > 1:
        assert s["batches"] < T * R  # requests were coalesced
    bt.close()
    st.close()


def test_query_length_mismatch_raises(xp, cuda):
    st = xp.Store(64, 32)
    st.upload(np.zeros(64 * 32, np.uint8))
    bt = xp.Batcher(st, max_batch=8, max_wait_us=100)
    with pytest.raises(xp.InvalidArgument):
        bt.answer(np.zeros(8, np.uint8), q_bits=63)  # pir.cpp:30-31
    # the batcher keeps serving after a rejected call
    q = np.zeros(8, np.uint8)
    q[0] = 1
    assert bt.answer(q).tobytes() == bytes(32)
    bt.close()
    st.close()


def test_close_while_callers_are_active(xp, port, cuda):
    """Destroying the batcher under load: every in-flight caller gets its correct
    answer or a clean 'shutting down' error — no crash, no torn answer."""
    N, S = 2048, 256
    g = np.random.default_rng(9)
    db = g.integers(0, 256, N * S, dtype=np.uint8)
    st = xp.Store(N, S)
    st.upload(db)
    bt = xp.Batcher(st, max_batch=16, max_wait_us=200)
    q = g.integers(0, 256, (64, N // 8), dtype=np.uint8)
    want = port.answer_batch(db, N, S, q, 64)
    bad, ok = [], [0]

    def worker(t):
        for r in range(200):
            k = (t * 7 + r) % 64
            try:
                a = bt.answer(q[k])
            except xp.XpirError:
                return
            if not np.array_equal(a, want[k]):
                bad.append((t, r))
            ok[0] += 1

    ts = [threading.Thread(target=worker, args=(t,)) for t in range(32)]
    for t in ts:
        t.start()
    import time

    time.sleep(0.05)
    bt.close()
    for t in ts:
        t.join()
    assert not bad and ok[0] > 0
    st.close()


def test_geometry_batcher_serves_several_stores(xp, port, cuda):
    """One batcher for every store of a geometry (the drop-in's per-snapshot-epoch
    reads): requests name their store, batches form per (store, masked), and each
    caller gets its own store's answer; a store of another geometry is refused."""
    N, S, K = 3000, 256, 3
    g = np.random.default_rng(77)
    dbs = [g.integers(0, 256, N * S, dtype=np.uint8) for _ in range(K)]
    sts = []
    for db in dbs:
        st = xp.Store(N, S)
        st.upload(db)
        sts.append(st)
    bt = xp.Batcher(None, max_batch=32, max_wait_us=300, geometry=(N, S))
    T, R = 16, 6
    nb = (N + 7) // 8
    qs = g.integers(0, 256, (T, R, nb), dtype=np.uint8)
    which = g.integers(0, K, (T, R))
    seeds = g.integers(0, 256, (T, R, 32), dtype=np.uint8)
    got = np.zeros((T, R, S), np.uint8)

    def worker(t):
        for r in range(R):
            got[t, r] = bt.answer(qs[t, r], mask_seed=seeds[t, r].tobytes() if r % 2 else None,
                                  store=sts[which[t, r]])

    _run_threads(worker, T)
    for t in range(T):
        for r in range(R):
            want = port.answer_batch(dbs[which[t, r]], N, S, qs[t, r][None], 1)[0].tobytes()
            if r % 2:
                want = port.mask_answer(want, seeds[t, r].tobytes())
            assert got[t, r].tobytes() == want, (t, r)
    other = xp.Store(N, S + 16)
    with pytest.raises(xp.InvalidArgument):
        bt.answer(qs[0, 0], store=other)
    with pytest.raises(xp.InvalidArgument):
        bt.answer(qs[0, 0])  # no default store
    bt.close()
    for st in sts + [other]:
        st.close()

"""GPU: the device ServerCore (xpir_server_*) against the reference's replica
state machine semantics (server.cpp:28-91) restated with the oracle: rounds of
apply_write (insert + absorb + rotate every rotate_writes writes), seals into a
ring of epoch_ring stores with incremental re-seal, snapshot_at for every
epoch still in the ring."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nb,depth,item,ring,R", [(256, 4, 64, 3, 37), (64, 2, 48, 2, 5), (1000, 8, 128, 4, 100)])
def test_server_rounds_and_epoch_ring(xp, port, cuda, nb, depth, item, ring, R):
    m, h, W = 4096, 5, 3
    g = np.random.default_rng(nb + ring)
    seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
    cap = nb * depth * 3 // 4
    sv = xp.Server(nb, depth, cap, item, seed, m, h, W, R, ring)
    if ring != 2:  # start-up reservation: pre-allocated ring images are used in order
        sv.reserve(3 * cap // 4)
    T = port.table(nb, depth, cap, item, seed)
    PW = port.window(m, h, W)
    PW.rotate()  # server.cpp:40
    sealed = {1: np.zeros(nb * depth * item, np.uint8)}
    writes = 0
    assert sv.info()["latest_epoch"] == 1
    for rnd in range(9):
        n = int(g.integers(1, 3 * cap // 4))
        b1 = g.integers(0, nb, n).astype(np.uint32)
        b2 = g.integers(0, nb, n).astype(np.uint32)
        pl = g.integers(0, 256, (n, item), dtype=np.uint8)
        pos = g.integers(0, m, (n, h)).astype(np.uint32)
        seal = rnd % 3 != 1
        rep, ep = sv.apply_round(b1, b2, pl, pos, seal_after=seal)
        # reference semantics, one write at a time (server.cpp:58-73)
        prep = T.insert_batch(b1, b2, pl)
        for i in range(n):
            PW.absorb(pos[i])
            writes += 1
            if writes % R == 0:
                PW.rotate()
        assert np.array_equal(rep, prep)
        assert sv.window_digest() == PW.digest()
        assert sv.table_digest() == T.state_digest()
        if seal:
            assert ep == max(sealed) + 1
            sealed[ep] = T.data().copy()
            for old in sorted(sealed)[:-ring]:
                del sealed[old]
        else:
            assert ep == 0
        info = sv.info()
        assert info["writes"] == writes and info["latest_epoch"] == max(sealed)
        assert info["oldest_epoch"] == min(sealed)
        for e, img in sealed.items():
            assert np.array_equal(sv.snapshot(e).download(), img), (rnd, e)
    with pytest.raises(xp.InvalidArgument):
        sv.snapshot(min(sealed) - 1)  # pruned epoch
    # a sealed epoch answers PIR reads (answer_share's scan step)
    st = sv.snapshot(0)
    q = np.zeros((2, (nb + 7) // 8), np.uint8)
    q[0, 0] = 1
    q[1, :] = 0xFF
    if nb % 8:
        q[1, -1] &= (1 << (nb % 8)) - 1
    out = st.answer_batch(q)
    img = sealed[max(sealed)].reshape(nb, depth * item)
    assert np.array_equal(out[0], img[0])
    assert np.array_equal(out[1], np.bitwise_xor.reduce(img, axis=0))


@pytest.mark.parametrize("G,nb,ring,R", [(2, 512, 3, 40), (4, 1024, 2, 150)])
def test_sharded_servers_match_whole_server(xp, port, cuda, G, nb, ring, R):
    """G bucket-range shard ranks of one replica (threads here, one rank per GPU in
    a deployment): same writes on every rank, payload gather/scatter across the
    shards with a barrier between the phases. After every round the union of the
    ranks' sealed shard stores equals the whole server's sealed store for every
    epoch in the ring, and the replicated window digests agree."""
    import threading

    depth, item, m, h, W = 4, 32, 2048, 3, 3
    g = np.random.default_rng(G + nb)
    seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
    cap = nb * depth
    bounds = [0] + [((nb * k // G) // 8) * 8 for k in range(1, G)] + [nb]
    whole = xp.Server(nb, depth, cap, item, seed, m, h, W, R, ring)
    ranks = [xp.Server(nb, depth, cap, item, seed, m, h, W, R, ring, lo=bounds[k], hi=bounds[k + 1])
             for k in range(G)]
    smap = xp.server_shard_map(ranks)
    bar = threading.Barrier(G)
    for rnd in range(6):
        n = int(g.integers(nb // 2, nb * 2))
        b1 = g.integers(0, nb, n).astype(np.uint32)
        b2 = g.integers(0, nb, n).astype(np.uint32)
        pl = g.integers(0, 256, (n, item), dtype=np.uint8)
        pos = g.integers(0, m, (n, h)).astype(np.uint32)
        seal = rnd % 2 == 0
        want_rep, want_ep = whole.apply_round(b1, b2, pl, pos, seal_after=seal)
        res = [None] * G
        errs = []

        def run(k):
            try:
                res[k] = ranks[k].apply_round(b1, b2, pl, pos, seal_after=seal, smap=smap, barrier=bar.wait)
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
                bar.abort()

        ts = [threading.Thread(target=run, args=(k,)) for k in range(G)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errs, errs
        for rep, ep in res:
            assert np.array_equal(rep, want_rep) and ep == want_ep
        info = whole.info()
        for e in range(info["oldest_epoch"], info["latest_epoch"] + 1):
            full = whole.snapshot(e).download()
            parts = np.concatenate([r.snapshot(e).download() for r in ranks])
            assert np.array_equal(parts, full), (rnd, e)
        assert all(r.window_digest() == whole.window_digest() for r in ranks)


def test_pinned_snapshot_survives_ring_turnover(xp, port, cuda):
    """snapshot_acquire pins an epoch's image (the reference keeps a pruned epoch
    alive through its shared_ptr, server.cpp:83-87): seals that push it off the
    ring retire it instead of re-sealing it in place; the last release returns it
    to the spare pool and later seals stay exact."""
    nb, depth, item, ring = 128, 4, 32, 2
    g = np.random.default_rng(5)
    seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
    cap = nb * depth // 2
    sv = xp.Server(nb, depth, cap, item, seed, 1024, 3, 2, 1000, ring)
    T = port.table(nb, depth, cap, item, seed)

    def round_(n, seal=True):
        b1 = g.integers(0, nb, n).astype(np.uint32)
        b2 = g.integers(0, nb, n).astype(np.uint32)
        pl = g.integers(0, 256, (n, item), dtype=np.uint8)
        pos = g.integers(0, 1024, (n, 3)).astype(np.uint32)
        T.insert_batch(b1, b2, pl)
        return sv.apply_round(b1, b2, pl, pos, seal_after=seal)[1]

    e2 = round_(40)
    img2 = T.data().copy()
    st2, pinned = sv.snapshot_acquire(e2)
    assert pinned == e2
    st2b, _ = sv.snapshot_acquire(0)  # latest == e2, a second reader
    for _ in range(4):  # e2 leaves the ring after the next `ring` seals
        round_(30)
    with pytest.raises(xp.InvalidArgument):
        sv.snapshot(e2)
    assert np.array_equal(st2.download(), img2)  # retired, untouched
    sv.snapshot_release(st2)
    assert np.array_equal(st2b.download(), img2)
    sv.snapshot_release(st2b)  # last reader: back to the spare pool
    with pytest.raises(xp.InvalidArgument):
        sv.snapshot_release(st2b)
    for _ in range(3):
        e = round_(25)
        assert np.array_equal(sv.snapshot(e).download(), T.data())
    q = np.zeros((1, nb // 8), np.uint8)
    q[0, 1] = 0x81  # buckets 8 and 15
    img = T.data().reshape(nb, depth * item)
    assert np.array_equal(sv.snapshot(0).answer_batch(q)[0], img[8] ^ img[15])
    sv.close()


@pytest.mark.parametrize("nb,depth,cap", [(128, 4, 400), (200, 3, 500)])
def test_single_write_rounds_async_walk(xp, port, cuda, nb, depth, cap):
    """One apply_write per call (the ServerCore drop-in's path): the walk, payload
    gather and scatter run back to back with one host round trip. Filled past
    capacity (FIFO GC) with evictions, bit-exact against the oracle throughout;
    a bad interest position mid-round follows notify.cpp:62 (write inserted,
    positions before the bad one absorbed, write not counted)."""
    m, h, W, R, ring = 2048, 3, 3, 7, 2
    item = 24
    g = np.random.default_rng(nb + depth)
    seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
    sv = xp.Server(nb, depth, cap, item, seed, m, h, W, R, ring)
    T = port.table(nb, depth, cap, item, seed)
    PW = port.window(m, h, W)
    PW.rotate()
    writes = 0
    for k in range(cap + 150):
        b1 = g.integers(0, nb, 1).astype(np.uint32)
        b2 = g.integers(0, nb, 1).astype(np.uint32)
        pl = g.integers(0, 256, (1, item), dtype=np.uint8)
        pos = g.integers(0, m, (1, h)).astype(np.uint32)
        rep, _ = sv.apply_round(b1, b2, pl, pos)
        assert np.array_equal(rep, T.insert_batch(b1, b2, pl)), k
        PW.absorb(pos[0])
        writes += 1
        if writes % R == 0:
            PW.rotate()
        if k % 50 == 0:
            assert sv.table_digest() == T.state_digest(), k
            assert sv.window_digest() == PW.digest(), k
    # a round of 3 writes whose second has a position out of range
    b1 = g.integers(0, nb, 3).astype(np.uint32)
    b2 = g.integers(0, nb, 3).astype(np.uint32)
    pl = g.integers(0, 256, (3, item), dtype=np.uint8)
    pos = g.integers(0, m, (3, h)).astype(np.uint32)
    pos[1, 2] = m + 5
    with pytest.raises(xp.InvalidArgument):
        sv.apply_round(b1, b2, pl, pos)
    T.insert_batch(b1[:2], b2[:2], pl[:2])
    PW.absorb(pos[0])
    writes += 1
    if writes % R == 0:
        PW.rotate()
    PW.absorb(pos[1, :2])
    assert sv.table_digest() == T.state_digest()
    assert sv.window_digest() == PW.digest()
    assert sv.info()["writes"] == writes
    sv.close()

"""GPU parity of the write path: cuckoo insertion/eviction/GC/drop (K6), PRF (K5)
and the interest-window Bloom update (K7) against the reference digests."""
import hashlib

import numpy as np
import pytest

from oracle import recipes

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _compare_tables(T, P):
    used, b1, b2, st = T.meta()
    pu, pb1, pb2, pst = P.meta()
    assert np.array_equal(used, pu)
    assert np.array_equal(b1, pb1) and np.array_equal(b2, pb2) and np.array_equal(st, pst)
    assert np.array_equal(T.snapshot(), P.data())
    assert T.counters() == P.counters()
    assert T.state_digest() == P.state_digest()


def test_config3_write_round(xp, port, golden, cuda):
    n = recipes.C3["n"]
    d = recipes.config3(port, n)
    G = golden["config3"][str(n)]
    T = xp.Table(32768, 4, 32768 * 4, 1024, d["s_cuckoo"])
    rep = T.insert_batch(d["b1"], d["b2"], d["payload"])
    assert sha(rep) == G["reports_sha256"]
    assert T.state_digest().hex() == G["state_digest"]
    assert sha(T.snapshot()) == G["table_sha256"]
    W = xp.Window(1 << 20, 23, 1)
    W.absorb(d["pos"].ravel())
    assert W.digest().hex() == G["window_digest"]
    # fused make_interest + absorb on device gives the same filter
    W2 = xp.Window(1 << 20, 23, 1)
    W2.absorb_interest(d["lid"], d["xs"])
    assert W2.digest().hex() == G["window_digest"]
    # beta computation on device (K5)
    assert np.array_equal(xp.prf_batch(d["k1"], d["xs"], 32768).astype(np.uint32), d["b1"])
    assert np.array_equal(xp.prf_batch(d["k2"], d["xs"], 32768).astype(np.uint32), d["b2"])


def test_config3_95pct_load(xp, port, golden, cuda):
    n = recipes.C3["n95"]
    d = recipes.config3(port, n)
    G = golden["config3"][str(n)]
    T = xp.Table(32768, 4, 32768 * 4, 1024, d["s_cuckoo"])
    rep = T.insert_batch(d["b1"], d["b2"], d["payload"])
    assert int(rep[:, 3].sum()) == G["displacements"]
    assert sha(rep) == G["reports_sha256"]
    assert T.state_digest().hex() == G["state_digest"]


def test_multi_batch_rounds_match_single_pass(xp, port, golden, cuda):
    """Rounds of writes (draw-window refills, resumed walks, moved pre-existing
    payloads) leave exactly the state of one long insert sequence."""
    n = recipes.C3["n95"]
    d = recipes.config3(port, n)
    T = xp.Table(32768, 4, 32768 * 4, 1024, d["s_cuckoo"])
    cuts = [0, 1, 5000, 32000, 90000, 100001, n]
    for a, b in zip(cuts, cuts[1:]):
        T.insert_batch(d["b1"][a:b], d["b2"][a:b], d["payload"][a:b])
    assert T.state_digest().hex() == golden["config3"][str(n)]["state_digest"]


def test_adversarial_gc_and_drops(xp, port, golden, cuda):
    for e in golden["cuckoo_adversarial"]:
        g = port.detrng(e["rng_seed"])
        s = g.fill(32)
        n, nb = e["n"], e["buckets"]
        b1 = np.array([g.uniform(nb) for _ in range(n)], np.uint32)
        b2 = np.array([g.uniform(nb) for _ in range(n)], np.uint32)
        pl = np.frombuffer(g.fill(n * 8), np.uint8).reshape(n, 8)
        T = xp.Table(nb, e["depth"], e["capacity"], 8, s)
        P = port.table(nb, e["depth"], e["capacity"], 8, s)
        # one item per call and all-at-once must agree with the reference
        rep = np.concatenate([T.insert_batch(b1[i:i + 1], b2[i:i + 1], pl[i:i + 1]) for i in range(n)])
        P.insert_batch(b1, b2, pl)
        assert rep.tolist() == e["reports"]
        assert T.state_digest().hex() == e["state_digest"]
        _compare_tables(T, P)


def test_random_tables_vs_oracle(xp, port, cuda):
    g = np.random.default_rng(77)
    for nb, depth, cap, n, item in ((5, 2, 10, 300, 16), (64, 4, 200, 2000, 32), (7, 3, 21, 500, 12),
                                    (1000, 8, 8000, 9000, 64)):
        seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
        b1 = g.integers(0, nb, n).astype(np.uint32)
        b2 = g.integers(0, nb, n).astype(np.uint32)
        pl = g.integers(0, 256, (n, item), dtype=np.uint8)
        T, P = xp.Table(nb, depth, cap, item, seed), port.table(nb, depth, cap, item, seed)
        for a in range(0, n, 97):
            assert np.array_equal(T.insert_batch(b1[a:a + 97], b2[a:a + 97], pl[a:a + 97]),
                                  P.insert_batch(b1[a:a + 97], b2[a:a + 97], pl[a:a + 97]))
        _compare_tables(T, P)


def test_cuckoo_reference_unit_cases(xp, cuda):
    z = bytes(32)
    # test_cuckoo.cpp:42-59 — beta1 wins ties, lowest free slot first
    T = xp.Table(4, 2, 8, 4, z)
    T.insert(1, 2, b"aaaa")
    T.insert(1, 2, b"bbbb")
    assert T.slot_used(1, 0) and T.slot_used(1, 1) and not T.slot_used(2, 0)
    T.insert(1, 2, b"cccc")
    assert T.slot_used(2, 0)
    snap = T.snapshot().reshape(4, 2, 4)
    assert bytes(snap[1, 0]) == b"aaaa" and bytes(snap[1, 1]) == b"bbbb" and bytes(snap[2, 0]) == b"cccc"
    # test_cuckoo.cpp:82-89 — no GC below capacity; empty slots are zero (177-193)
    assert not snap[0].any() and not snap[3].any()
    # out-of-range bucket: items before the bad one are applied, then EINVAL
    with pytest.raises(xp.InvalidArgument):
        T.insert_batch([0, 9], [0, 0], np.zeros(8, np.uint8))
    assert T.writes_applied() == 4
    with pytest.raises(xp.InvalidArgument):
        T.insert_batch([0], [0], np.zeros(5, np.uint8))  # item size mismatch


@pytest.mark.parametrize("bad_at,which", [(0, 1), (37, 2), (199, 1), (150, 2)])
def test_device_inputs_out_of_range_bucket(xp, port, cuda, bad_at, which):
    """cuckoo.cpp:57-58 on the device-pointer entry points: the items before the
    first out-of-range beta are inserted (bit-exact vs the oracle's loop), then
    EINVAL; nothing indexes the table with the bad value."""
    torch = cuda
    nb, depth, item, n = 64, 4, 16, 200
    g = port.detrng(31)
    seed = g.fill(32)
    b1 = np.array([g.uniform(nb) for _ in range(n)], np.uint32)
    b2 = np.array([g.uniform(nb) for _ in range(n)], np.uint32)
    (b1 if which == 1 else b2)[bad_at] = nb + 5 + bad_at * 1000
    pl = np.frombuffer(g.fill(n * item), np.uint8).reshape(n, item)
    T, P = xp.Table(nb, depth, 200, item, seed), port.table(nb, depth, 200, item, seed)
    P.insert_batch(b1[:bad_at], b2[:bad_at], pl[:bad_at])
    d1, d2 = torch.from_numpy(b1.view(np.int32)).cuda(), torch.from_numpy(b2.view(np.int32)).cuda()
    dp, rep = torch.from_numpy(pl.copy()).cuda(), torch.zeros((n, 4), dtype=torch.int32, device="cuda")
    with pytest.raises(xp.InvalidArgument):
        T.insert_batch_dev(d1, d2, dp, n, rep)
    torch.cuda.synchronize()
    assert T.writes_applied() == bad_at
    assert T.state_digest() == P.state_digest()
    # the walk-only entry point (payload shards) behaves the same
    T2 = xp.Table(nb, depth, 200, item, seed)
    with pytest.raises(xp.InvalidArgument):
        T2.insert_walk_dev(d1, d2, n, rep)
    assert T2.writes_applied() == bad_at


def test_write_betas_match_prf(xp, port, cuda):
    """beta1/beta2 of a write batch in one kernel == crypto::prf per key (crypto.cpp:17-33)."""
    torch = cuda
    g = np.random.default_rng(12)
    k1, k2 = g.integers(0, 256, 16, dtype=np.uint8).tobytes(), g.integers(0, 256, 16, dtype=np.uint8).tobytes()
    xs = g.integers(0, 2**63, 3000, dtype=np.uint64)
    for m in (32768, 1000, 3):
        d1 = torch.empty(3000, dtype=torch.int32, device="cuda")
        d2 = torch.empty_like(d1)
        xp.write_betas_dev(k1, k2, torch.from_numpy(xs.view(np.int64)).cuda(), 3000, m, d1, d2)
        torch.cuda.synchronize()
        want1 = [port.prf(k1, int(x), m) for x in xs[:300]]
        want2 = [port.prf(k2, int(x), m) for x in xs[:300]]
        assert d1.cpu().numpy()[:300].tolist() == want1 and d2.cpu().numpy()[:300].tolist() == want2


def test_window_rotate_and_range(xp, port, cuda):
    for w in (1, 2, 3):
        A, B = xp.Window(1000, 3, w), port.window(1000, 3, w)
        g = np.random.default_rng(w)
        for step in range(7):
            pos = g.integers(0, 1000, 20).astype(np.uint32)
            A.absorb(pos)
            B.absorb(pos)
            if step % 2:
                A.rotate()
                B.rotate()
            assert A.digest() == B.digest()
            assert A.size() == B.size()
        with pytest.raises(xp.InvalidArgument):
            A.absorb([5, 1000, 7])
        with pytest.raises(ValueError):
            B.absorb([5, 1000, 7])
        assert A.digest() == B.digest()  # prefix before the bad position absorbed, as the reference


def test_seal_into_store_and_read(xp, port, cuda):
    """apply_write rounds then seal (server.cpp:58-81) and read it back via PIR."""
    d = recipes.config3(port, 2000)
    T = xp.Table(32768, 4, 32768 * 4, 1024, d["s_cuckoo"])
    T.insert_batch(d["b1"], d["b2"], d["payload"])
    st = xp.Store(32768, 4096)
    T.seal(st, epoch=1)
    snap = T.snapshot().reshape(32768, 4096)
    q = np.zeros((3, 4096), np.uint8)
    for r, b in enumerate(d["b1"][:3]):
        q[r, b // 8] |= 1 << (b % 8)
    got = st.answer_batch(q)
    for r, b in enumerate(d["b1"][:3]):
        assert np.array_equal(got[r], snap[b])


@pytest.mark.parametrize("nb,depth,cap,n,same_frac", [
    (64, 4, 256, 200, 0.0), (1000, 2, 2000, 1500, 0.1), (37, 3, 111, 90, 0.3), (4096, 4, 16384, 15000, 0.05),
    (512, 8, 4096, 3000, 0.5), (100, 1, 100, 95, 0.0),
])
def test_parallel_prefix_matches_sequential(xp, port, cuda, nb, depth, cap, n, same_frac):
    """One large batch: the parallel eviction-free prefix (Jacobi-solved claims)
    followed by the sequential walk must equal the reference order exactly,
    including beta1 == beta2 items, near-full tables and depth 1."""
    g = np.random.default_rng(nb * 7 + n)
    seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
    b1 = g.integers(0, nb, n).astype(np.uint32)
    b2 = g.integers(0, nb, n).astype(np.uint32)
    same = g.random(n) < same_frac
    b2[same] = b1[same]
    pl = g.integers(0, 256, (n, 16), dtype=np.uint8)
    T, P = xp.Table(nb, depth, cap, 16, seed), port.table(nb, depth, cap, 16, seed)
    assert np.array_equal(T.insert_batch(b1, b2, pl), P.insert_batch(b1, b2, pl))
    _compare_tables(T, P)
    # a second round on the now-occupied table
    b1 = g.integers(0, nb, n).astype(np.uint32)
    b2 = g.integers(0, nb, n).astype(np.uint32)
    assert np.array_equal(T.insert_batch(b1, b2, pl), P.insert_batch(b1, b2, pl))
    _compare_tables(T, P)


@pytest.mark.parametrize("nb,depth,cap_frac,load,same_frac,walk", [
    (25000, 4, 1.0, 0.97, 0.02, "x"),   # 100,000 slots: alt index partly in TMEM
    (33000, 3, 1.0, 0.95, 0.0, "x"),    # depth 3: uniform(depth) with rejection, TMEM part
    (16384, 8, 0.9, 1.3, 0.01, "x"),    # 131,072 slots at capacity: FIFO GC on every insert past it
    (20000, 4, 1.0, 0.96, 0.0, "w"),    # the warp walk with global victim metadata (A/B)
    (140000, 4, 1.0, 0.95, 0.01, "g"),  # 560,000 slots: beyond the on-chip maps, global-map warp walk
    (70000, 8, 0.95, 1.1, 0.0, "g"),    # depth 8 (one 8-byte occupancy load), GC past capacity
    (190000, 3, 1.0, 0.94, 0.0, "g"),   # depth 3: per-byte occupancy, rejection draws
])
def test_walk_kernels_large_tables(xp, port, cuda, nb, depth, cap_frac, load, same_frac, walk):
    """The warp-cooperative walks on tables whose alt index spills into TMEM
    (k_cuckoo_walk_x) or that run the global-metadata walk (k_cuckoo_walk_w, with
    its occupancy/touched maps in global memory past 512 Ki slots), at
    high load with long eviction chains, beta1 == beta2 items, non-power-of-two
    depth and GC: reports, table bytes, metadata and state digest equal the
    oracle's sequential cuckoo::Table::insert (cuckoo.cpp:56-126)."""
    import subprocess
    import sys

    code = f"""
import numpy as np, sys
sys.path.insert(0, {repr(str(__import__('os').path.dirname(__import__('os').path.dirname(__file__))))})
import oracle, paper_2001_08250_b200 as xp
nb, depth, cap_frac, load, same_frac = {nb}, {depth}, {cap_frac}, {load}, {same_frac}
g = np.random.default_rng(nb + depth)
slots = nb * depth
cap = int(slots * cap_frac)
n = int(slots * load)
seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
b1 = g.integers(0, nb, n).astype(np.uint32)
b2 = g.integers(0, nb, n).astype(np.uint32)
same = g.random(n) < same_frac
b2[same] = b1[same]
pl = g.integers(0, 256, (n, 8), dtype=np.uint8)
port = oracle.Port()
T, P = xp.Table(nb, depth, cap, 8, seed), port.table(nb, depth, cap, 8, seed)
half = n // 2
for a, b in ((0, half), (half, n)):
    assert np.array_equal(T.insert_batch(b1[a:b], b2[a:b], pl[a:b]), P.insert_batch(b1[a:b], b2[a:b], pl[a:b]))
assert T.state_digest() == P.state_digest()
assert np.array_equal(T.snapshot(), P.data())
print("ok")
"""
    env = dict(__import__("os").environ)
    env["XPIR_CUCKOO_WALK"] = "2" if walk == "w" else "0"
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


@pytest.mark.parametrize("G,nb,depth,item,load", [(2, 4096, 4, 64, 0.93), (4, 1000, 4, 32, 0.97), (3, 512, 2, 48, 1.4)])
def test_payload_shards_match_whole_table(xp, port, cuda, G, nb, depth, item, load):
    """Bucket-range payload shards: every shard runs the replicated
    walk, gathers the payloads that move into its range from whichever shard holds
    them, then scatters; the union of the shards equals the whole table after
    every round (high load: evictions cross shard boundaries; load > 1: GC), and
    the metadata of every replica equals the oracle's."""
    import torch

    g = np.random.default_rng(G * 1000 + nb)
    seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
    cap = nb * depth * 9 // 10 if load > 1 else nb * depth
    bounds = [0] + [((nb * k // G) // 8) * 8 for k in range(1, G)] + [nb]
    shards = [xp.Table(nb, depth, cap, item, seed, lo=bounds[k], hi=bounds[k + 1]) for k in range(G)]
    smap = xp.shard_map(shards)
    P = port.table(nb, depth, cap, item, seed)
    n_total = int(nb * depth * load)
    for rnd in range(3):
        n = n_total // 3
        b1 = g.integers(0, nb, n).astype(np.uint32)
        b2 = g.integers(0, nb, n).astype(np.uint32)
        pl = g.integers(0, 256, (n, item), dtype=np.uint8)
        want_rep = P.insert_batch(b1, b2, pl)
        d1, d2 = torch.from_numpy(b1.view(np.int32)).cuda(), torch.from_numpy(b2.view(np.int32)).cuda()
        dp = torch.from_numpy(pl).cuda()
        reps = [torch.zeros((n, 4), dtype=torch.int32, device="cuda") for _ in shards]
        for t, r in zip(shards, reps):
            t.insert_walk_dev(d1, d2, n, r)
        for t in shards:
            t.apply_gather_dev(smap)
        torch.cuda.synchronize()  # the barrier between the phases
        for t in shards:
            t.apply_scatter_dev(dp)
        torch.cuda.synchronize()
        for r in reps:
            assert np.array_equal(r.cpu().numpy().view(np.uint32), want_rep), rnd
        whole = np.concatenate([t.snapshot() for t in shards])
        assert np.array_equal(whole, P.data()), rnd
        used, m1, m2, st = shards[G - 1].meta()
        pu, p1, p2, pst = P.meta()
        assert np.array_equal(used, pu) and np.array_equal(m1, p1) and np.array_equal(st, pst)
    with pytest.raises(xp.InvalidArgument):
        shards[0].state_digest()  # needs the whole table
    with pytest.raises(xp.InvalidArgument):
        shards[0].insert_batch([0], [0], np.zeros(item, np.uint8))  # the one-call path is whole-table only


@pytest.mark.parametrize("single", [False, True])
def test_fifo_ring_grows_instead_of_failing(xp, port, cuda, single):
    """with capacity == buckets*depth, failing eviction chains keep live
    below capacity, so FIFO GC never runs while old items in untouched buckets stay
    live and stamps keep growing past the ring (2,048 entries for 128 slots). The
    reference's std::map keeps going; the device ring now doubles and is refilled
    from the live slots (bit-exact vs the oracle throughout)."""
    nb, depth, item = 32, 4, 8
    cap = nb * depth
    g = np.random.default_rng(99 + single)
    seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
    T, P = xp.Table(nb, depth, cap, item, seed), port.table(nb, depth, cap, item, seed)
    b1 = g.integers(0, nb, cap).astype(np.uint32)
    b2 = g.integers(0, nb, cap).astype(np.uint32)
    pl = g.integers(0, 256, (cap, item), dtype=np.uint8)
    assert np.array_equal(T.insert_batch(b1, b2, pl), P.insert_batch(b1, b2, pl))
    n = 2600  # > 2,048 stamps while buckets 8..31 keep their first items
    b1 = g.integers(0, 8, n).astype(np.uint32)
    b2 = g.integers(0, 8, n).astype(np.uint32)
    pl = g.integers(0, 256, (n, item), dtype=np.uint8)
    step = 1 if single else 200
    for a in range(0, n, step):
        if single and a % 100:
            T.insert_batch(b1[a:a + 1], b2[a:a + 1], pl[a:a + 1])
            P.insert_batch(b1[a:a + 1], b2[a:a + 1], pl[a:a + 1])
            continue
        assert np.array_equal(T.insert_batch(b1[a:a + step], b2[a:a + step], pl[a:a + step]),
                              P.insert_batch(b1[a:a + step], b2[a:a + step], pl[a:a + step])), a
    assert T.state_digest() == P.state_digest()

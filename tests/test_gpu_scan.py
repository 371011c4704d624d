"""GPU parity: the sm_100a scan path (K1 direct + M4RM, K2 expansion, K3 mask,
K4 XOR reduce) against the oracle and the golden fixtures written from the
unmodified reference. Integer work: every comparison is bit-exact."""
import hashlib

import numpy as np
import pytest

from oracle import recipes

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rand(g, *shape):
    return g.integers(0, 256, shape, dtype=np.uint8)


@pytest.fixture(autouse=True)
def _auto_kernel(xp):
    xp.set_scan_opts(0)
    yield
    xp.set_scan_opts(0)


# --- reference unit-test known answers (test_pir.cpp) -----------------------------
def test_tiny_known_db(xp, cuda):
    st = xp.Store(3, 1)
    st.upload(np.array([0x0F, 0xF0, 0xAA], np.uint8))
    out = st.answer_batch(np.array([[0b101], [0], [0b10]], np.uint8))
    assert out[:, 0].tolist() == [0xA5, 0x00, 0xF0]
    with pytest.raises(xp.InvalidArgument):
        st.answer_batch(np.array([[0]], np.uint8), q_bits=4)  # test_pir.cpp:107-108


def test_full_retrieval_every_target(xp, port, cuda):
    # test_pir.cpp:117-131 on a 64 x 12-byte DB, and acceptance #1 shapes
    for N, S in ((64, 12), (8, 1), (256, 4), (64, 16)):
        g = port.detrng(23)
        db = np.frombuffer(g.fill(N * S), np.uint8)
        st = xp.Store(N, S)
        st.upload(db)
        for beta in range(N):
            qs = g.gen_queries(beta, N, 3)
            ans = st.answer_batch(qs)
            assert np.array_equal(ans, port.answer_batch(db, N, S, qs, 3))
            assert np.array_equal(np.bitwise_xor.reduce(ans, axis=0), db.reshape(N, S)[beta])


@pytest.mark.parametrize("kernel", [1, 2, 7, 9])
@pytest.mark.parametrize("N,S,B", [
    (8, 128, 1), (9, 128, 3), (1000, 256, 97), (1024, 4096, 64), (777, 512, 130),
    (4096, 128, 1), (2048, 1024, 513), (4000, 2048, 1025), (256, 32768, 40), (12345, 128, 300),
])
def test_scan_matches_oracle(xp, port, cuda, kernel, N, S, B):
    g = np.random.default_rng(N * 7 + S + B)
    db = rand(g, N * S)
    q = rand(g, B, (N + 7) // 8)
    xp.set_scan_opts(kernel)
    st = xp.Store(N, S)
    st.upload(db)
    got = st.answer_batch(q)
    want = port.answer_batch(db, N, S, q, B)
    assert np.array_equal(got, want)
    if kernel == 2 and S % 128 == 0:
        assert xp.last_scan_kernel() == 2


@pytest.mark.parametrize("B", [5, 8, 9, 13, 16, 17, 24, 31, 32, 33])
def test_nibble_tables_split_lookups(xp, port, cuda, B):
    """Nibble tables (7) at B <= 32 deal each request's lookups over 2/4/8
    quarter-warp slots whose partial answers meet in the red.xor flush; every
    split (and the unsplit B = 33) against the oracle, ragged bucket counts."""
    N, S = 5000 + B, 256
    g = np.random.default_rng(B * 31 + 7)
    db = rand(g, N * S)
    q = rand(g, B, (N + 7) // 8)
    xp.set_scan_opts(7)
    st = xp.Store(N, S)
    st.upload(db)
    assert np.array_equal(st.answer_batch(q), port.answer_batch(db, N, S, q, B))
    assert xp.last_scan_kernel() == 7


@pytest.mark.parametrize("S", [96, 512])
def test_direct_every_small_batch(xp, port, cuda, S):
    """The direct kernel's request tiling (tiles of 1/2/4/6/8 requests, partial
    last tiles) for every B = 1..17, ragged bucket count."""
    N = 1001
    g = np.random.default_rng(S)
    db = rand(g, N * S)
    st = xp.Store(N, S)
    st.upload(db)
    xp.set_scan_opts(1)
    for B in range(1, 18):
        q = rand(g, B, (N + 7) // 8)
        q[:, -1] &= 0x01
        assert np.array_equal(st.answer_batch(q), port.answer_batch(db, N, S, q, B)), B
        assert xp.last_scan_kernel() == 1


@pytest.mark.parametrize("N,S,B", [(1, 128, 5), (97, 128, 64), (96, 256, 129), (191, 128, 256), (4099, 384, 300),
                                   (20000, 128, 257), (777, 1024, 1000)])
def test_six_bucket_tables_match_oracle(xp, port, cuda, N, S, B):
    """Kernel 9: 24-bit query units split into four 6-bucket groups; bucket counts
    ending mid-group, mid-unit and mid-chunk (96), 1/2/4-request lane tiles and
    partial request tiles."""
    g = np.random.default_rng(N * 3 + S + B)
    db = rand(g, N * S)
    q = rand(g, B, (N + 7) // 8)
    if N % 8:
        q[:, -1] &= (1 << (N % 8)) - 1
    xp.set_scan_opts(9)
    st = xp.Store(N, S)
    st.upload(db)
    got = st.answer_batch(q)
    assert xp.last_scan_kernel() == 9
    assert np.array_equal(got, port.answer_batch(db, N, S, q, B))
    if S % 128 == 0 and 129 <= B <= 256:  # the automatic choice in its batch range
        xp.set_scan_opts(0)
        assert np.array_equal(st.answer_batch(q), got) and xp.last_scan_kernel() == 9


def test_dirty_trailing_bits_are_ignored(xp, port, cuda):
    # pir::answer only reads bits j < N (pir.cpp:33-34)
    N, S, B = 1001, 256, 200
    g = np.random.default_rng(5)
    db = rand(g, N * S)
    q = rand(g, B, (N + 7) // 8)
    q[:, -1] |= 0xFE
    st = xp.Store(N, S)
    st.upload(db)
    for k in (1, 2, 6, 7, 9):
        xp.set_scan_opts(k)
        assert np.array_equal(st.answer_batch(q), port.answer_batch(db, N, S, q, B))


def test_empty_and_zero_queries(xp, cuda):
    st = xp.Store(64, 128)
    st.upload(np.full(64 * 128, 0xAB, np.uint8))
    assert st.answer_batch(np.zeros((0, 8), np.uint8)).shape == (0, 128)
    assert not st.answer_batch(np.zeros((300, 8), np.uint8)).any()
    ones = st.answer_batch(np.full((300, 8), 0xFF, np.uint8))
    assert not ones.any()  # 64 identical buckets XOR to zero


def test_mask_fused(xp, port, cuda):
    N, S, B = 2048, 512, 257
    g = np.random.default_rng(9)
    db, q, ms = rand(g, N * S), rand(g, B, N // 8), rand(g, B, 32)
    st = xp.Store(N, S)
    st.upload(db)
    plain = port.answer_batch(db, N, S, q, B)
    for k in (1, 2):
        xp.set_scan_opts(k)
        got = st.answer_batch(q, mask_seeds=ms)
        for r in range(0, B, 37):
            assert got[r].tobytes() == port.mask_answer(plain[r].tobytes(), ms[r].tobytes())


def test_seeded_expansion(xp, port, cuda):
    N, S, B = 4096, 1024, 150
    g = np.random.default_rng(11)
    db, seeds = rand(g, N * S), rand(g, B, 32)
    q = np.stack([np.frombuffer(port.prng_expand(s.tobytes(), N // 8), np.uint8) for s in seeds])
    st = xp.Store(N, S)
    st.upload(db)
    assert np.array_equal(st.answer_batch_seeded(seeds), port.answer_batch(db, N, S, q, B))


def test_primitives(xp, port, golden, cuda):
    P = golden["primitives"]
    for e in P["prng_expand"]:
        assert xp.prng_expand(bytes.fromhex(e["seed"]), e["n"]).hex() == e["out"]
    for e in P["prf"]:
        assert xp.prf_batch(bytes.fromhex(e["key"]), e["x"], e["m"]).tolist() == e["out"]
    for e in P["bloom"]:
        assert xp.bloom_positions(bytes.fromhex(e["item"]), e["h"], e["m"]) == e["out"]
    for e in P["interest"]:
        got = xp.make_interest_batch(e["m"], e["h"], bytes.fromhex(e["id"]), [e["seq"]])
        assert got[0].tolist() == e["out"]
    for e in P["blake2b"]:
        assert xp.blake2b(bytes.fromhex(e["in"]), e["outlen"]).hex() == e["out"]


def test_keystream_generators(xp, port, cuda):
    torch = cuda
    key = bytes(range(32))
    for off, n in ((0, 1), (5, 100), (64, 4096), (1000, 777)):
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        xp.keystream_dev(key, 9, d, n, byte_offset=off)
        torch.cuda.synchronize()
        want = port.chacha20(key, (9).to_bytes(8, "little"), off + n)[off:]
        assert d.cpu().numpy().tobytes() == want
    rows = torch.zeros((7, 48), dtype=torch.uint8, device="cuda")
    xp.keystream_rows_dev(key, 3, 7, 40, rows, 48)
    torch.cuda.synchronize()
    g = port.detrng(key)
    for r in range(3):
        g.fill(0)
    for r in range(7):
        assert rows[r, :40].cpu().numpy().tobytes() == g.fill(40)
        assert not rows[r, 40:].cpu().numpy().any()


def test_config1_golden(xp, port, golden, cuda):
    db, q = recipes.config1(port)
    st = xp.Store(1024, 4096)
    st.upload(db)
    for k in (0, 1, 2, 7):
        xp.set_scan_opts(k)
        out = st.answer_batch(q)
        assert out[0, :8].tobytes().hex() == "877147f881293508"
        assert sha(out) == golden["config1"]["out_sha256"]


def test_config2_three_server_round(xp, port, golden, cuda):
    db, betas, shares = recipes.config2(port)
    G = golden["config2"]
    assert sha(db) == G["db_sha256"] and sha(shares) == G["shares_sha256"]
    st = xp.Store(32768, 4096)
    st.upload(db)
    outs = [st.answer_batch(shares[s]) for s in range(3)]
    for s in range(3):
        assert sha(outs[s]) == G["out_sha256"][s]
    assert np.array_equal(outs[0] ^ outs[1] ^ outs[2], db.reshape(32768, 4096)[betas])


@pytest.mark.parametrize("kernel,B", [(0, 333), (9, 200), (7, 100), (8, 2100), (1, 17)])
def test_virtual_shards_xor_reduce(xp, port, cuda, kernel, B):
    """Bucket-range shards on one GPU + the K4 XOR reduce == the unsharded scan,
    for each scan kernel (shard windows start mid-chunk of every table layout)."""
    torch = cuda
    N, S = 8192, 512
    xp.set_scan_opts(kernel)
    g = np.random.default_rng(21 + B)
    db, q = rand(g, N * S), rand(g, B, N // 8)
    want = port.answer_batch(db, N, S, q, B)
    dq = torch.from_numpy(q).cuda()
    for G in (2, 3, 8):
        bounds = [((N // 8) * k // G) * 8 for k in range(G)] + [N]
        parts = []
        for k in range(G):
            lo, hi = bounds[k], bounds[k + 1]
            st = xp.Store(N, S, lo, hi)
            st.upload(db[lo * S: hi * S])
            o = torch.empty((B, S), dtype=torch.uint8, device="cuda")
            st.answer_batch_dev(dq, N // 8, B, o)
            torch.cuda.synchronize()
            parts.append((st, o))
        acc = parts[0][1].clone()
        ptrs = torch.tensor([p[1].data_ptr() for p in parts[1:]], dtype=torch.int64, device="cuda")
        xp.xor_reduce_dev(acc, [p[1].data_ptr() for p in parts[1:]], B * S, d_ptr_array=ptrs)
        torch.cuda.synchronize()
        assert np.array_equal(acc.cpu().numpy(), want)


def test_linearity_large(xp, cuda):
    """Size-independent property at 1 GiB: answer(a ^ b) == answer(a) ^ answer(b)."""
    torch = cuda
    N, S, B = 1 << 18, 4096, 256
    st = xp.Store(N, S)
    st.fill_keystream(bytes(range(32)), 1)
    g = np.random.default_rng(3)
    a, b = rand(g, B, N // 8), rand(g, B, N // 8)
    qa = st.answer_batch(a)
    qb = st.answer_batch(b)
    qab = st.answer_batch(a ^ b)
    assert np.array_equal(qab, qa ^ qb)
    # unit vectors read buckets back exactly
    e = np.zeros((4, N // 8), np.uint8)
    idx = [0, 1, N - 1, 123457]
    for r, j in enumerate(idx):
        e[r, j // 8] |= 1 << (j % 8)
    got = st.answer_batch(e)
    full = st.download().reshape(N, S)
    for r, j in enumerate(idx):
        assert np.array_equal(got[r], full[j])


@pytest.mark.slow
def test_config4_sample_golden(xp, port, golden, cuda):
    """Full 4 GiB store generated on device; first 8 seeded requests vs the
    reference outputs in golden.json; store windows spot-checked."""
    torch = cuda
    N, S = recipes.C4["N"], recipes.C4["S"]
    key = xp.blake2b((3).to_bytes(8, "little"), 32)
    st = xp.Store(N, S)
    st.fill_keystream(key, 0)
    G = golden["config4"]
    for w in G["store_windows"]:
        assert sha(st.download(w["off"], 65536)) == w["sha256"]
    seeds = np.stack([np.frombuffer(bytes.fromhex(h), np.uint8) for h in G["seeds_hex"]])
    assert np.array_equal(seeds, recipes.config4_seeds(port, 8))
    for k in (1, 2):
        xp.set_scan_opts(k)
        out = st.answer_batch_seeded(seeds)
        assert [sha(out[r]) for r in range(8)] == G["out_rows_sha256"]


@pytest.mark.slow
def test_config5_shapes_golden(xp, golden, cuda):
    """Config 5: every (slot, depth) shape over the same 1 GiB DetRng(5) store,
    4 DetRng(55) requests each, vs the reference outputs; both scan kernels."""
    torch = cuda
    G = golden["config5"]
    key = xp.blake2b((5).to_bytes(8, "little"), 32)
    qkey = xp.blake2b((55).to_bytes(8, "little"), 32)
    nonce = 0
    for e in G["shapes"]:
        N, S = e["N"], e["S"]
        st = xp.Store(N, S)
        st.fill_keystream(key, 0)
        q = torch.zeros((4, N // 8), dtype=torch.uint8, device="cuda")
        xp.keystream_rows_dev(qkey, nonce, 4, N // 8, q, N // 8)
        nonce += 4
        torch.cuda.synchronize()
        assert sha(q.cpu().numpy()) == e["q_sha256"]
        for k in (1, 2):
            xp.set_scan_opts(k)
            out = torch.empty((4, S), dtype=torch.uint8, device="cuda")
            st.answer_batch_dev(q, N // 8, 4, out)
            torch.cuda.synchronize()
            o = out.cpu().numpy()
            assert [sha(o[r]) for r in range(4)] == e["out_rows_sha256"], (e["slot"], e["depth"], k)
        st.close()


@pytest.mark.parametrize("kernel", [4, 5])
@pytest.mark.parametrize("N,S,B", [
    (1000, 128, 1), (4096, 256, 130), (2048, 512, 2048), (3001, 384, 2500), (777, 1024, 4097), (64, 128, 6000),
])
def test_m4rm_variants_match_oracle(xp, port, cuda, kernel, N, S, B):
    """Registers-only (4) and half-TMEM-accumulator (5) M4RM kernels, forced at any
    batch size, including partial 2048-request tiles and odd bucket counts."""
    g = np.random.default_rng(N * 3 + S + B + kernel)
    db = rand(g, N * S)
    q = rand(g, B, (N + 7) // 8)
    xp.set_scan_opts(kernel)
    st = xp.Store(N, S)
    st.upload(db)
    assert np.array_equal(st.answer_batch(q), port.answer_batch(db, N, S, q, B))
    assert xp.last_scan_kernel() == (5 if kernel == 5 else 2)


@pytest.mark.parametrize("N,S,B", [
    (1000, 32, 1), (4096, 64, 130), (2048, 96, 2048), (3001, 384, 2500), (777, 1024, 4097),
    (64, 128, 6000), (5000, 160, 8192), (131, 4096, 9000), (100003, 32, 2049), (40, 32, 16385),
])
def test_m4rm_quad_tables_match_oracle(xp, port, cuda, N, S, B):
    """Quad-interleaved 9-bucket tables over 32-byte columns with full-TMEM
    accumulators (8), forced at any batch size: partial 2048/4096/8192-request
    tiles, bucket counts that end mid-table, mid-set and mid-pair (72 buckets),
    bucket sizes that are multiples of 32 but not of 128, caller rows through the
    shared-memory layout-2 transposition (whole 288-byte tiles and a tail)."""
    g = np.random.default_rng(N * 5 + S + B)
    db = rand(g, N * S)
    q = rand(g, B, (N + 7) // 8)
    xp.set_scan_opts(8)
    st = xp.Store(N, S)
    st.upload(db)
    got = st.answer_batch(q)
    assert xp.last_scan_kernel() == 8
    assert np.array_equal(got, port.answer_batch(db, N, S, q, B))


def test_concurrent_host_calls_on_one_store(xp, port, cuda):
    """answer/answer_batch are re-entrant over an immutable snapshot:
    several host threads (ctypes releases the GIL) query one store at once."""
    import threading

    N, S = 4096, 512
    g = np.random.default_rng(404)
    db = rand(g, N * S)
    st = xp.Store(N, S)
    st.upload(db)
    qs = [rand(g, B, N // 8) for B in (3, 64, 200, 700)]
    want = [port.answer_batch(db, N, S, q, q.shape[0]) for q in qs]
    errors = []

    def worker(k):
        try:
            for _ in range(4):
                if not np.array_equal(st.answer_batch(qs[k]), want[k]):
                    errors.append(k)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(k,)) for k in range(len(qs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors

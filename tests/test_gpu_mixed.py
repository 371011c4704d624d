"""GPU: seed-compressed read shares. A read's l shares are
l-1 PRG seeds plus one explicit vector (the XOR of the expanded seeds with the
target's unit vector — pir::gen_queries, pir.cpp:7-27, with the uniform shares
replaced by prng_expand(seed), crypto.cpp:35-45). Each server's batch mixes
seeded and explicit requests; xpir_answer_batch_mixed answers it in one scan.
Checks: every server's answers equal the oracle's answer_batch of the expanded
vectors (bit-exact, with and without the answer mask), and the XOR of the l
answers is the target bucket (pir::reconstruct)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def expand(port, seed, N):
    v = np.frombuffer(port.prng_expand(seed, (N + 7) // 8), np.uint8).copy()
    if N % 8:
        v[-1] &= (1 << (N % 8)) - 1
    return v


@pytest.mark.parametrize("N,S,B,l", [(1000, 64, 37, 3), (32768, 4096, 300, 3), (4096, 512, 2048, 2), (777, 128, 5, 4)])
def test_compressed_shares_round(xp, port, cuda, N, S, B, l):
    g = np.random.default_rng(N + B + l)
    db = g.integers(0, 256, N * S, dtype=np.uint8)
    nb = (N + 7) // 8
    betas = g.integers(0, N, B)
    explicit_server = g.integers(0, l, B)  # which server holds the explicit share
    seeds = g.integers(0, 256, (B, l, 32), dtype=np.uint8)
    shares = np.zeros((l, B, nb), np.uint8)
    for r in range(B):
        acc = np.zeros(nb, np.uint8)
        for k in range(l):
            if k != explicit_server[r]:
                shares[k, r] = expand(port, seeds[r, k].tobytes(), N)
                acc ^= shares[k, r]
        acc[betas[r] // 8] ^= np.uint8(1 << (betas[r] % 8))
        shares[explicit_server[r], r] = acc
    st = xp.Store(N, S)
    st.upload(db)
    masks = g.integers(0, 256, (B, 32), dtype=np.uint8)
    answers = []
    for k in range(l):
        is_seed = (explicit_server != k).astype(np.uint8)
        sd = seeds[is_seed.astype(bool), k]
        rows = shares[k][~is_seed.astype(bool)]
        got = st.answer_batch_mixed(is_seed, sd, rows)
        assert np.array_equal(got, port.answer_batch(db, N, S, shares[k], B)), k
        gm = st.answer_batch_mixed(is_seed, sd, rows, mask_seeds=masks)
        for r in range(0, B, max(1, B // 7)):
            assert gm[r].tobytes() == port.mask_answer(got[r].tobytes(), masks[r].tobytes())
        answers.append(got)
    rec = np.bitwise_xor.reduce(np.stack(answers), axis=0)
    assert np.array_equal(rec, db.reshape(N, S)[betas])


def test_mixed_all_seeded_and_all_explicit(xp, port, cuda):
    N, S, B = 2048, 256, 40
    g = np.random.default_rng(3)
    db = g.integers(0, 256, N * S, dtype=np.uint8)
    st = xp.Store(N, S)
    st.upload(db)
    seeds = g.integers(0, 256, (B, 32), dtype=np.uint8)
    q = np.stack([expand(port, seeds[r].tobytes(), N) for r in range(B)])
    a = st.answer_batch_mixed(np.ones(B, np.uint8), seeds, None)
    b = st.answer_batch_mixed(np.zeros(B, np.uint8), None, q)
    assert np.array_equal(a, b) and np.array_equal(a, port.answer_batch(db, N, S, q, B))
    one = np.ones(1, np.uint8)
    out = np.zeros(S, np.uint8)
    with pytest.raises(xp.InvalidArgument):  # query length mismatch (pir.cpp:43-44)
        xp._check(xp.lib().xpir_answer_batch_mixed(st.h, 1, xp._p(one), xp._p(seeds[0]), None, 0, N - 1, None,
                                                   xp._p(out)))

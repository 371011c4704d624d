"""ORACLE / TEST INFRASTRUCTURE ONLY — seeded input recipes for BASELINE.json's
configs, generated with an oracle DetRng (``Ref`` or ``Port``).

"Call k" = the k-th ``DetRng::fill`` of the generator (nonce = LE64(k),
rng.cpp:25-31). The product side (bench.py, GPU tests) regenerates the same
bytes on device from (key, nonce) with ``xpir_keystream*``; these helpers are the
host-side truth it is compared against.
"""
from __future__ import annotations

import numpy as np

C1 = dict(N=1024, S=4096, B=64, seed=0)
C2 = dict(N=32768, S=4096, B=1024, servers=3, seed=1)
C3 = dict(N=32768, depth=4, item=1024, n=32000, n95=124518, m=1 << 20, h=23, seed=2)
C4 = dict(N=1 << 20, S=4096, B=8192, seed=3)
C5 = dict(bytes=1 << 30, slots=(256, 512, 1024, 2048, 4096), depths=(2, 4, 8), seed=5)


def detrng_key(o, seed: int) -> bytes:
    """DetRng(seed) key = BLAKE2b-256(LE64(seed)) (rng.cpp:18-23)."""
    return o.blake2b(int(seed).to_bytes(8, "little"), 32)


def config1(o):
    g = o.detrng(C1["seed"])
    db = np.frombuffer(g.fill(C1["N"] * C1["S"]), np.uint8)
    q = np.stack([np.frombuffer(g.fill(C1["N"] // 8), np.uint8) for _ in range(C1["B"])])
    return db, q


def config2(o, B: int | None = None):
    """Store (call 0), then per request r: beta_r = uniform(N) (call 1+3r) and
    gen_queries(beta_r, N, 3) (calls 2+3r, 3+3r). Returns db, betas, shares[3][B][N/8]."""
    N, S = C2["N"], C2["S"]
    B = C2["B"] if B is None else B
    g = o.detrng(C2["seed"])
    db = np.frombuffer(g.fill(N * S), np.uint8)
    betas = np.zeros(B, np.uint32)
    shares = np.zeros((3, B, N // 8), np.uint8)
    for r in range(B):
        betas[r] = g.uniform(N)
        shares[:, r, :] = g.gen_queries(int(betas[r]), N, 3)
    return db, betas, shares


def config3(o, n: int | None = None):
    """s_cuckoo, K1, K2, LogId, then per write x = next_u64, payload = fill(1024),
    beta = prf(K, x, N), positions = make_interest({m,h}, id, x)."""
    N, item, m, h = C3["N"], C3["item"], C3["m"], C3["h"]
    n = C3["n"] if n is None else n
    g = o.detrng(C3["seed"])
    s_cuckoo = g.fill(32)
    k1, k2, lid = g.fill(16), g.fill(16), g.fill(16)
    xs = np.zeros(n, np.uint64)
    payload = np.zeros((n, item), np.uint8)
    for i in range(n):
        xs[i] = g.next_u64()
        payload[i] = np.frombuffer(g.fill(item), np.uint8)
    b1 = np.array([o.prf(k1, int(x), N) for x in xs], np.uint32)
    b2 = np.array([o.prf(k2, int(x), N) for x in xs], np.uint32)
    pos = np.stack([o.make_interest(m, h, lid, int(x)) for x in xs]) if n else np.zeros((0, h), np.uint32)
    return dict(s_cuckoo=s_cuckoo, k1=k1, k2=k2, lid=lid, xs=xs, payload=payload, b1=b1, b2=b2, pos=pos)


def config4_seeds(o, B: int) -> np.ndarray:
    """seed_r = gen_array<16>() (call r+1), zero-extended to the 32-byte PRG seed."""
    g = o.detrng(C4["seed"])
    g.fill(0)  # call 0 is the 4 GiB store
    seeds = np.zeros((B, 32), np.uint8)
    for r in range(B):
        seeds[r, :16] = np.frombuffer(g.fill(16), np.uint8)
    return seeds


def config4_store_window(o, byte_lo: int, n: int) -> np.ndarray:
    """Bytes [byte_lo, byte_lo+n) of the 4 GiB store (call 0 of DetRng(3))."""
    key = detrng_key(o, C4["seed"])
    if hasattr(o, "chacha20"):
        blk0 = byte_lo // 64
        ks = o.chacha20(key, b"\0" * 8, (byte_lo - blk0 * 64) + n, blk0)
        return np.frombuffer(ks[byte_lo - blk0 * 64:], np.uint8)
    raise TypeError("needs Port.chacha20 (seekable keystream)")


def shape5(slot: int, depth: int):
    S = slot * depth
    return C5["bytes"] // S, S

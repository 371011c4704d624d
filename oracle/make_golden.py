"""ORACLE / TEST INFRASTRUCTURE ONLY — writes tests/golden/golden.json from the
UNMODIFIED reference build (oracle/_ref/libxpir_ref.so). Run here (where
/root/reference exists):  python -m oracle.make_golden [--no-large]

The fixture pins (a) the libsodium-backed primitives at the reference's call
sites, (b) every BASELINE config's outputs (digests of full outputs, raw bytes
where small), so the C restatement and the CUDA path are checked against the
reference itself, on this box and on the GPU box (which has no /root/reference).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import time

import numpy as np

from oracle import Ref, recipes

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "golden.json")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-large", action="store_true", help="skip the 4 GiB config-4 sample")
    args = ap.parse_args()
    R = Ref()
    G: dict = {"generator": "oracle/make_golden.py over oracle/_ref/libxpir_ref.so "
                            "(reference /root/reference/proj/src + libsodium 1.0.20)"}
    rng = np.random.default_rng(20010825)

    # --- primitives -------------------------------------------------------
    prim = {"prng_expand": [], "blake2b": [], "prf": [], "bloom": [], "detrng": [], "interest": []}
    for n in (0, 1, 63, 64, 65, 200, 1000):
        seed = rng.integers(0, 256, 32, dtype=np.uint8).tobytes()
        prim["prng_expand"].append({"seed": seed.hex(), "n": n, "out": R.prng_expand(seed, n).hex()})
    for n in (0, 1, 8, 24, 28, 127, 128, 129, 256, 1000):
        d = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        for ol in (8, 32, 64):
            prim["blake2b"].append({"in": d.hex(), "outlen": ol, "out": R.blake2b(d, ol).hex()})
    for m in (1, 2, 3, 1000, 32768, 2**63 + 5, 2**64 - 1, 1 << 20, 7):
        key = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        xs = [int(v) for v in rng.integers(0, 2**63, 8, dtype=np.uint64)] + [0, 2**64 - 1]
        prim["prf"].append({"key": key.hex(), "m": m, "x": xs, "out": [R.prf(key, x, m) for x in xs]})
    for n in (0, 4, 24, 50):
        item = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        for h, m in ((4, 1 << 20), (23, 1 << 20), (6, 16285), (1, 1)):
            prim["bloom"].append({"item": item.hex(), "h": h, "m": m, "out": R.bloom_positions(item, h, m)})
    lid = bytes(range(16))
    for seq in (0, 1, 2**64 - 1, 123456789):
        prim["interest"].append({"id": lid.hex(), "seq": seq, "m": 1 << 20, "h": 23,
                                 "out": R.make_interest(1 << 20, 23, lid, seq).tolist()})
    for seed in (0, 1, 2, 3, 5):
        g = R.detrng(seed)
        prim["detrng"].append({"seed": seed, "key": recipes.detrng_key(R, seed).hex(),
                               "fill32": g.fill(32).hex(), "fill16": g.fill(16).hex(),
                               "u64": g.next_u64(), "uniform": [g.uniform(b) for b in (2, 3, 4, 1000, 32768)]})
    G["primitives"] = prim
    G["bloom_hash_count"] = {"m": 1 << 20, "n": 32000, "h": R.bloom_hash_count(1 << 20, 32000)}

    # --- reference unit-test known answers (test_pir.cpp:87-109, 33-43) ---
    snap = R.snapshot(np.array([0x0F, 0xF0, 0xAA], np.uint8), 3, 1)
    G["tiny"] = {"db": "0ff0aa", "q02": snap.answer(np.array([0b101], np.uint8)).tobytes().hex(),
                 "zero": snap.answer(np.array([0], np.uint8)).tobytes().hex(),
                 "unit1": snap.answer(np.array([0b10], np.uint8)).tobytes().hex()}

    # --- config 1 ------------------------------------------------------------
    t = time.time()
    db, q = recipes.config1(R)
    out = R.answer_batch(db, 1024, 4096, q, 64)
    G["config1"] = {"db_sha256": sha(db), "q_sha256": sha(q), "out_sha256": sha(out),
                    "out0_first8": out[0, :8].tobytes().hex(),
                    "out_rows_sha256": [sha(out[r]) for r in range(64)]}
    print("config1", time.time() - t, out[0, :8].tobytes().hex())

    # --- config 2 (all 1024 requests x 3 servers) ----------------------------
    t = time.time()
    db, betas, shares = recipes.config2(R)
    snap = R.snapshot(db, 32768, 4096)
    outs = [snap.answer_batch(shares[s], 1024)[0] for s in range(3)]
    rec = outs[0] ^ outs[1] ^ outs[2]
    want = db.reshape(32768, 4096)[betas]
    assert np.array_equal(rec, want)
    G["config2"] = {"db_sha256": sha(db), "betas_sha256": sha(betas), "shares_sha256": sha(shares),
                    "betas_first8": betas[:8].tolist(),
                    "out_sha256": [sha(o) for o in outs],
                    "out_rows_sha256_first16": [[sha(o[r]) for r in range(16)] for o in outs]}
    del snap
    print("config2", time.time() - t)

    # --- config 3 and the 95%-load variant -----------------------------------
    c3 = {}
    for n in (recipes.C3["n"], recipes.C3["n95"]):
        t = time.time()
        d = recipes.config3(R, n)
        T = R.table(32768, 4, 32768 * 4, 1024, d["s_cuckoo"])
        W = R.window(1 << 20, 23, 1)
        rep = T.insert_batch(d["b1"], d["b2"], d["payload"])
        W.absorb(d["pos"].ravel())
        c3[str(n)] = {"state_digest": T.state_digest().hex(), "window_digest": W.digest().hex(),
                      "reports_sha256": sha(rep), "displacements": int(rep[:, 3].sum()),
                      "chains": int((rep[:, 3] > 0).sum()), "dropped": int(rep[:, 1].sum()),
                      "live": T.counters()[1], "table_sha256": sha(T.data()),
                      "bits_set": int(sum(bin(int(w)).count("1") for w in W.delta(0))),
                      "inputs_sha256": sha(np.concatenate([d["b1"], d["b2"]]))}
        print("config3", n, time.time() - t, c3[str(n)]["state_digest"])
    G["config3"] = c3

    # adversarial small tables (test_cuckoo.cpp:61-80 GC and 111-125 drop shapes)
    adv = []
    for (nb, depth, cap, n, seed) in ((4, 2, 6, 40, 7), (2, 1, 2, 10, 11), (8, 2, 16, 200, 13),
                                      (16, 4, 40, 300, 17), (3, 3, 9, 60, 19)):
        g = R.detrng(seed)
        s = g.fill(32)
        b1 = np.array([g.uniform(nb) for _ in range(n)], np.uint32)
        b2 = np.array([g.uniform(nb) for _ in range(n)], np.uint32)
        pl = np.frombuffer(g.fill(n * 8), np.uint8).reshape(n, 8)
        T = R.table(nb, depth, cap, 8, s)
        rep = T.insert_batch(b1, b2, pl)
        adv.append({"buckets": nb, "depth": depth, "capacity": cap, "n": n, "rng_seed": seed,
                    "reports": rep.tolist(), "state_digest": T.state_digest().hex(),
                    "data": T.data().tobytes().hex()})
    G["cuckoo_adversarial"] = adv

    # --- config 4 sample: first 8 requests over the 4 GiB store ---------------
    if not args.no_large:
        t = time.time()
        N, S = recipes.C4["N"], recipes.C4["S"]
        g = R.detrng(recipes.C4["seed"])
        snap = R.snapshot_detrng(g, N, S)
        seeds = np.zeros((8, 32), np.uint8)
        for r in range(8):
            seeds[r, :16] = np.frombuffer(g.fill(16), np.uint8)
        q = np.stack([np.frombuffer(R.prng_expand(seeds[r].tobytes(), N // 8), np.uint8) for r in range(8)])
        out, secs = snap.answer_batch(q, 8, threads=8)
        dbv = snap.data()
        G["config4"] = {"seeds_hex": [s.tobytes().hex() for s in seeds],
                        "store_windows": [{"off": off, "sha256": sha(dbv[off:off + 65536])}
                                          for off in (0, 1 << 20, (1 << 32) - 65536, 123456789 * 16)],
                        "out_rows_sha256": [sha(out[r]) for r in range(8)],
                        "out_first16": [out[r, :16].tobytes().hex() for r in range(8)]}
        del snap
        print("config4", time.time() - t)

    # --- config 5 sample: each shape, 4 requests, from a 1 GiB DetRng(5) store --
    t = time.time()
    g = R.detrng(recipes.C5["seed"])
    big = R.snapshot_detrng(g, 1 << 18, 4096)  # 1 GiB, call 0
    dbv = big.data()
    qg = R.detrng(55)
    c5 = []
    for slot in recipes.C5["slots"]:
        for depth in recipes.C5["depths"]:
            N, S = recipes.shape5(slot, depth)
            q = np.stack([np.frombuffer(qg.fill(N // 8), np.uint8) for _ in range(4)])
            sn = R.snapshot(dbv, N, S)
            out = sn.answer_batch(q, 4, threads=4)[0]
            c5.append({"slot": slot, "depth": depth, "N": N, "S": S, "q_sha256": sha(q),
                       "out_rows_sha256": [sha(out[r]) for r in range(4)]})
            del sn
    G["config5"] = {"store_sha256": sha(dbv), "query_rng_seed": 55, "shapes": c5}
    print("config5", time.time() - t)

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(G, f, indent=1)
    print("wrote", OUT, os.path.getsize(OUT))


if __name__ == "__main__":
    main()

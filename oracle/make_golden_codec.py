"""Writes tests/golden/codec.json from the UNMODIFIED reference build
(oracle/_ref/libxpir_ref.so): notify::encode_delta / decode_delta
(notify.cpp:139-180) vectors — the reference's own test_notify.cpp cases
(DetRng(11) densities on m = 4097, an empty 2^23-bit delta, the {3, 9} delta and
its trailing/truncated corruptions), random deltas at several widths, the
config-3 interest delta, and a set of malformed inputs with their verdicts.

Test infrastructure only.    python oracle/make_golden_codec.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import recipes  # noqa: E402


def words_of(m, positions):
    w = np.zeros((m + 63) // 64, np.uint64)
    for p in positions:
        w[p >> 6] |= np.uint64(1) << np.uint64(p & 63)
    return w


def main():
    R = oracle.Ref()
    cases = []
    # test_notify.cpp:121-133 "delta codec roundtrips"
    g = R.detrng(11)
    for density in (0.0, 0.01, 0.3, 0.9):
        m, want, pos = 4097, int(4097 * density), set()
        while len(pos) < want:
            pos.add(g.uniform(4097))
        w = words_of(m, pos)
        cases.append({"name": f"test_notify_4097_{density}", "m": m, "words": w.tobytes().hex(),
                      "enc": R.encode_delta(m, w).hex()})
    # test_notify.cpp:135-139 empty 2^23-bit delta
    m = 1 << 23
    cases.append({"name": "empty_2p23", "m": m, "words_zero": True,
                  "enc": R.encode_delta(m, np.zeros(m // 64, np.uint64)).hex()})
    # random widths / densities
    rg = np.random.default_rng(2001)
    for m in (1, 63, 64, 65, 1000, 4096):
        for density in (0.0, 0.05, 0.5, 1.0):
            pos = np.nonzero(rg.random(m) < density)[0]
            w = words_of(m, pos)
            cases.append({"name": f"rand_{m}_{density}", "m": m, "words": w.tobytes().hex(),
                          "enc": R.encode_delta(m, w).hex()})
    # config 3: the interest delta after 32,000 writes (23 positions each, m = 2^20)
    d = recipes.config3(R, recipes.C3["n"])
    W = R.window(recipes.C3["m"], recipes.C3["h"], 1)
    W.absorb(d["pos"].ravel())
    w = W.delta(0)
    enc = R.encode_delta(recipes.C3["m"], w)
    cases.append({"name": "config3_delta", "m": recipes.C3["m"], "words_sha256": hashlib.sha256(w.tobytes()).hexdigest(),
                  "enc_len": len(enc), "enc_sha256": hashlib.sha256(enc).hexdigest()})
    # malformed inputs (test_notify.cpp:141-153 and the decode rules of notify.cpp:159-180)
    ok39 = R.encode_delta(64, words_of(64, [3, 9]))
    bad = {
        "empty": b"", "trailing": ok39 + b"\x00", "truncated": ok39[:-1], "m_only": b"\x40",
        "m_zero": b"\x00\x00", "zero_gap": b"\x40\x02\x03\x00", "pos_ge_m": b"\x40\x01\x40",
        "m_gt_u32": bytes([0x80, 0x80, 0x80, 0x80, 0x10, 0x00]),
        "varint_11_bytes": b"\x40\x01" + b"\xff" * 10 + b"\x00",
        "varint_10_bytes_wraps": b"\x40\x02\x05" + b"\xff" * 9 + b"\x01",
        "count_short": b"\x40\x03\x01\x01", "cut_varint": b"\x40\x01\x81",
        "ok_3_9": ok39, "ok_single": b"\x08\x01\x07", "ok_zero_first": b"\x08\x01\x00",
    }
    mal = []
    for name, buf in bad.items():
        r = R.decode_delta(buf)
        mal.append({"name": name, "buf": buf.hex(), "valid": r is not None,
                    "m": None if r is None else r[0], "words": None if r is None else r[1].tobytes().hex()})
    out = {"generator": "oracle/make_golden_codec.py (reference notify.cpp via oracle/_ref)",
           "cases": cases, "decode": mal}
    with open(os.path.join(ROOT, "tests", "golden", "codec.json"), "w") as f:
        json.dump(out, f, indent=0)
    print(len(cases), "cases,", len(mal), "decode verdicts")


if __name__ == "__main__":
    main()

"""GPU parity of the interest-window codecs on device:
notify::encode_delta / decode_delta (notify.cpp:139-180) and
ServerCore::make_freeze (server.cpp:45-56), against the golden vectors written
from the unmodified reference (tests/golden/codec.json) and the oracle.
Byte-exact: every encoding, verdict and decoded word."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import recipes

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "codec.json")


@pytest.fixture(scope="module")
def codec():
    with open(GOLDEN) as f:
        return json.load(f)


def _words(c):
    if c.get("words_zero"):
        return np.zeros((c["m"] + 63) // 64, np.uint64)
    return np.frombuffer(bytes.fromhex(c["words"]), np.uint64).copy()


def test_encode_decode_golden(xp, codec, cuda):
    for c in codec["cases"]:
        if "words_sha256" in c:
            continue
        w = _words(c)
        W = xp.Window(c["m"], 1, 1)
        pos = np.nonzero(np.unpackbits(w.view(np.uint8), bitorder="little")[:c["m"]])[0].astype(np.uint32)
        W.absorb(pos)
        assert np.array_equal(W.delta(0), w)
        enc = W.encode_delta(0)
        assert enc.hex() == c["enc"], c["name"]
        m, back = xp.decode_delta(enc)
        assert m == c["m"] and np.array_equal(back, w), c["name"]
        W.close()


def test_decode_verdicts_golden(xp, codec, cuda):
    for d in codec["decode"]:
        r = xp.decode_delta(bytes.fromhex(d["buf"]))
        assert (r is not None) == d["valid"], d["name"]
        if r is not None:
            assert r[0] == d["m"] and r[1].tobytes().hex() == d["words"], d["name"]


def test_config3_delta_codec(xp, port, codec, cuda):
    c = [x for x in codec["cases"] if x["name"] == "config3_delta"][0]
    d = recipes.config3(port, recipes.C3["n"])
    W = xp.Window(recipes.C3["m"], recipes.C3["h"], 1)
    W.absorb_interest(d["lid"], d["xs"])
    w = W.delta(0)
    assert hashlib.sha256(w.tobytes()).hexdigest() == c["words_sha256"]
    enc = W.encode_delta(0)
    assert len(enc) == c["enc_len"] and hashlib.sha256(enc).hexdigest() == c["enc_sha256"]
    m, back = xp.decode_delta(enc)
    assert m == recipes.C3["m"] and np.array_equal(back, w)


@pytest.mark.parametrize("m", [1, 63, 64, 65, 4097, 1 << 16, (1 << 20) + 5])
def test_random_deltas_vs_oracle(xp, port, cuda, m):
    g = np.random.default_rng(m)
    for density in (0.0, 0.0005, 0.05, 0.5, 1.0):
        pos = np.nonzero(g.random(m) < density)[0].astype(np.uint32)
        W = xp.Window(m, 1, 1)
        W.absorb(pos)
        w = W.delta(0)
        enc = W.encode_delta(0)
        assert enc == port.encode_delta(m, w)
        assert np.array_equal(xp.decode_delta(enc)[1], w)
        # every truncation and a few corruptions give the oracle's verdict
        for cut in sorted({0, 1, 2, len(enc) // 3, len(enc) - 1}):
            assert (xp.decode_delta(enc[:cut]) is None) == (port.decode_delta(enc[:cut]) is None)
        for k in range(4):
            b = bytearray(enc)
            if len(b) > 3:
                b[g.integers(2, len(b))] = int(g.integers(0, 256))
                r, o = xp.decode_delta(bytes(b)), port.decode_delta(bytes(b))
                assert (r is None) == (o is None)
                if r is not None:
                    assert r[0] == o[0] and np.array_equal(r[1], o[1])
        W.close()


def test_encode_dev_buffers(xp, port, cuda):
    import torch

    m = 1 << 18
    g = np.random.default_rng(5)
    w = np.zeros(m // 64, np.uint64)
    for p in np.nonzero(g.random(m) < 0.1)[0]:
        w[p >> 6] |= np.uint64(1) << np.uint64(p & 63)
    dw = torch.from_numpy(w.view(np.int64)).cuda()
    n = xp.encode_delta_dev(dw, m)
    out = torch.empty(n, dtype=torch.uint8, device="cuda")
    assert xp.encode_delta_dev(dw, m, out, n) == n
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == port.encode_delta(m, w)


def test_server_freeze_matches_reference_semantics(xp, port, cuda):
    """make_freeze after rounds with rotations: base, newest, digest over the frozen
    deltas (Window::digest(count)) and their encodings (server.cpp:45-56)."""
    nb, depth, item, m, h, W, R = 64, 4, 32, 2048, 3, 4, 10
    g = np.random.default_rng(9)
    seed = g.integers(0, 256, 32, dtype=np.uint8).tobytes()
    sv = xp.Server(nb, depth, nb * depth, item, seed, m, h, W, R, 2)
    PW = port.window(m, h, W)
    PW.rotate()  # server.cpp:40
    writes = 0
    for rnd in range(5):
        n = int(g.integers(5, 25))
        b1 = g.integers(0, nb, n).astype(np.uint32)
        b2 = g.integers(0, nb, n).astype(np.uint32)
        pl = g.integers(0, 256, (n, item), dtype=np.uint8)
        pos = g.integers(0, m, (n, h)).astype(np.uint32)
        sv.apply_round(b1, b2, pl, pos)
        for i in range(n):
            PW.absorb(pos[i])
            writes += 1
            if writes % R == 0:
                PW.rotate()
        f = sv.freeze()
        size, base = PW.size(), PW.base()
        assert f["base"] == base and f["newest"] == base + size - 2
        assert f["digest"] == PW.digest_n(size - 1)
        assert len(f["deltas"]) == size - 1
        for k in range(size - 1):
            assert f["deltas"][k] == port.encode_delta(m, PW.delta(k))
    sv.close()

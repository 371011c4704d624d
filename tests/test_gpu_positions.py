"""GPU parity of the write's interest-field codec (wire.cpp:154-169):
notify::encode_positions / decode_positions (notify.cpp:182-214) on device, one
thread per write, bit-exact against the oracle (itself pinned to the compiled
reference in tests/test_oracle.py): sorted varint-delta fields zero-padded to
INTEREST_FIELD_LEN = 64 bytes, the 'exceeds field capacity' throw (about a fifth
of the fields at config 3's m = 2^20, h = 23), and std::nullopt on malformed fields."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,h,cap", [(1 << 20, 23, 64), (1 << 12, 23, 64), (1 << 16, 7, 64), (1 << 32 - 1, 40, 200),
                                     (2048, 0, 64), (1 << 10, 128, 256)])
def test_encode_positions_matches_oracle(xp, port, cuda, m, h, cap):
    import torch

    n = 3000
    g = np.random.default_rng(m % 997 + h + cap)
    pos = g.integers(0, m, (n, h)).astype(np.uint32)
    if h:
        pos[:5] = pos[:5].min(axis=1, keepdims=True)  # duplicate positions are kept
    d_pos = torch.from_numpy(pos.view(np.int32)).cuda()
    d_f = torch.empty((n, cap), dtype=torch.uint8, device="cuda")
    d_ok = torch.empty(n, dtype=torch.uint8, device="cuda")
    xp.encode_positions_dev(d_pos, h, n, d_f, d_ok, cap=cap)
    f, ok = d_f.cpu().numpy(), d_ok.cpu().numpy()
    for i in range(n):
        want = port.encode_positions(pos[i], cap)
        assert bool(ok[i]) == (want is not None), i
        assert f[i].tobytes() == (want if want is not None else bytes(cap)), i
    if (m, h, cap) == (1 << 20, 23, 64):
        assert 0 < ok.sum() < n  # some config-3 writes do not fit the 64-byte field


def test_decode_positions_matches_oracle(xp, port, cuda):
    import torch

    cap, n = 64, 6000
    g = np.random.default_rng(7)
    fields = g.integers(0, 256, (n, cap), dtype=np.uint8)
    # well-formed fields, fields with varints running off the end, overflows past
    # 2^32, counts larger than the field, zero fields
    for i in range(0, n, 3):
        k = int(g.integers(0, 40))
        p = np.sort(g.integers(0, 1 << 20, k)).astype(np.uint32)
        e = port.encode_positions(p, cap)
        if e is not None:
            fields[i] = np.frombuffer(e, np.uint8)
    fields[1::7] &= 0x7F
    fields[2::11] = 0
    fields[4::13, 0] = 0xFF
    d_f = torch.from_numpy(fields).cuda()
    d_pos = torch.empty((n, cap), dtype=torch.int32, device="cuda")
    d_cnt = torch.empty(n, dtype=torch.int32, device="cuda")
    xp.decode_positions_dev(d_f, n, d_pos, d_cnt, cap=cap)
    got_pos = d_pos.cpu().numpy().view(np.uint32)
    cnt = d_cnt.cpu().numpy().view(np.uint32)
    n_ok = 0
    for i in range(n):
        want = port.decode_positions(fields[i].tobytes())
        if want is None:
            assert cnt[i] == 0xFFFFFFFF, i
        else:
            n_ok += 1
            assert cnt[i] == len(want) and np.array_equal(got_pos[i, :len(want)], want), i
    assert 0 < n_ok < n


def test_positions_round_trip(xp, cuda):
    """decode(encode(p)) == sorted(p) for every field that fits."""
    import torch

    n, h, cap = 20000, 9, 64
    g = np.random.default_rng(11)
    pos = g.integers(0, 1 << 24, (n, h)).astype(np.uint32)
    d_pos = torch.from_numpy(pos.view(np.int32)).cuda()
    d_f = torch.empty((n, cap), dtype=torch.uint8, device="cuda")
    d_ok = torch.empty(n, dtype=torch.uint8, device="cuda")
    xp.encode_positions_dev(d_pos, h, n, d_f, d_ok, cap=cap)
    d_out = torch.empty((n, cap), dtype=torch.int32, device="cuda")
    d_cnt = torch.empty(n, dtype=torch.int32, device="cuda")
    xp.decode_positions_dev(d_f, n, d_out, d_cnt, cap=cap)
    ok = d_ok.cpu().numpy().astype(bool)
    cnt = d_cnt.cpu().numpy().view(np.uint32)
    out = d_out.cpu().numpy().view(np.uint32)
    assert ok.all()
    assert (cnt == h).all()
    assert np.array_equal(out[:, :h], np.sort(pos, axis=1))


def test_argument_checks(xp, cuda):
    import torch

    d_pos = torch.zeros((4, 129), dtype=torch.int32, device="cuda")
    d_f = torch.empty((4, 64), dtype=torch.uint8, device="cuda")
    d_ok = torch.empty(4, dtype=torch.uint8, device="cuda")
    with pytest.raises(xp.InvalidArgument):
        xp.encode_positions_dev(d_pos, 129, 4, d_f, d_ok)  # h <= 128
    with pytest.raises(xp.InvalidArgument):
        xp.decode_positions_dev(d_f, 4, d_pos, d_ok, cap=0)
    xp.encode_positions_dev(d_pos, 0, 0, None, None)  # n = 0: nothing to do

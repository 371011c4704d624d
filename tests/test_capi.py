"""CPU tests of the drop-in boundary: libxpir.so builds for sm_100a, loads, exports
every symbol include/xpir.h declares, and fails loudly (no CPU fallback) when no
GPU is visible."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xpir.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(xpir_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_python_mirror(xp):
    assert declared_symbols() == sorted(xp.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol(xp):
    L = C.CDLL(xp.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", xp.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (xpir_[a-z0-9_]+)", out))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a(xp):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", xp.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly(xp):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU visible")
    with pytest.raises(xp.XpirError):
        xp.Store(64, 128)
    with pytest.raises(xp.XpirError):
        xp.prng_expand(b"\0" * 32, 64)


def test_argument_validation_matches_reference(xp):
    # The reference's std::invalid_argument cases are rejected before any CUDA call.
    with pytest.raises(xp.InvalidArgument):
        xp.Table(0, 4, 1, 16, b"\0" * 32)          # cuckoo.cpp:15-16
    with pytest.raises(xp.InvalidArgument):
        xp.Table(4, 4, 17, 16, b"\0" * 32)         # cuckoo.cpp:17-18
    with pytest.raises(xp.InvalidArgument):
        xp.Window(0, 3, 1)                          # notify.cpp:56
    with pytest.raises(xp.InvalidArgument):
        xp.Window(100, 3, 0)                        # notify.cpp:55
    with pytest.raises(xp.InvalidArgument):
        xp.prf_batch(b"\0" * 16, [1], 0)            # crypto.cpp:18
    with pytest.raises(xp.InvalidArgument):
        xp.Store(64, 128, lo=4, hi=64)              # shard bounds
    assert xp.blake2b(b"").hex().startswith("0e5751c026e543b2")  # BLAKE2b-256("") on the host side

"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes bindings to the two CPU checkers for the XOR-PIR server hot path:

* ``Ref``  -- the UNMODIFIED reference (``/root/reference/proj/src``) compiled by
  ``oracle/Makefile`` into ``oracle/_ref/libxpir_ref.so`` (travels to the GPU box
  prebuilt; links the image's libsodium 1.0.20).
* ``Port`` -- the plain-C restatement ``oracle/xpir_oracle.c`` built into
  ``oracle/_build/libxpir_oracle.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package; the product path
(``paper_2001_08250_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libxpir_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libxpir_oracle.so")

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)


def build(quiet: bool = True) -> None:
    """make -C oracle (C restatement always; the reference when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _p(a: np.ndarray, t=_u8p):
    return a.ctypes.data_as(t)


def _u8(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray)):
        return np.frombuffer(bytes(x), dtype=np.uint8).copy()
    return np.ascontiguousarray(x, dtype=np.uint8)


class Port:
    """The C restatement (oracle/xpir_oracle.c)."""

    kind = "port"

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.xo_chacha20_stream.argtypes = [_u8p, C.c_uint64, _u8p, _u8p, C.c_uint64]
        L.xo_blake2b.argtypes = [_u8p, C.c_size_t, _u8p, C.c_uint64]
        L.xo_siphash24.argtypes = [_u8p, _u8p, C.c_uint64]
        L.xo_siphash24.restype = C.c_uint64
        L.xo_prf.argtypes = [_u8p, C.c_uint64, C.c_uint64]
        L.xo_prf.restype = C.c_uint64
        L.xo_bloom_positions.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, _u32p]
        L.xo_make_interest.argtypes = [C.c_uint32, C.c_uint32, _u8p, C.c_uint64, _u32p]
        L.xo_bloom_hash_count.argtypes = [C.c_uint32, C.c_uint64]
        L.xo_bloom_hash_count.restype = C.c_uint32
        L.xo_answer_batch.argtypes = [_u8p, C.c_uint32, C.c_uint32, _u8p, C.c_uint64, C.c_uint32,
                                      C.c_uint32, _u8p, C.c_uint32]
        L.xo_mask_answer.argtypes = [_u8p, C.c_uint64, _u8p, _u8p]
        L.xo_detrng_init_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.xo_detrng_init_key.argtypes = [C.c_void_p, _u8p]
        L.xo_detrng_fill.argtypes = [C.c_void_p, _u8p, C.c_uint64]
        L.xo_detrng_next_u64.argtypes = [C.c_void_p]
        L.xo_detrng_next_u64.restype = C.c_uint64
        L.xo_detrng_uniform.argtypes = [C.c_void_p, C.c_uint64]
        L.xo_detrng_uniform.restype = C.c_uint64
        L.xo_gen_queries.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, _u8p]
        L.xo_table_new.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, _u8p]
        L.xo_table_new.restype = C.c_void_p
        L.xo_table_free.argtypes = [C.c_void_p]
        L.xo_table_insert.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, _u8p, _u32p]
        L.xo_table_data.argtypes = [C.c_void_p]
        L.xo_table_data.restype = C.c_void_p
        L.xo_table_state_digest.argtypes = [C.c_void_p, _u8p]
        L.xo_table_counters.argtypes = [C.c_void_p, _u64p, _u64p, _u64p]
        L.xo_table_meta.argtypes = [C.c_void_p, _u8p, _u32p, _u32p, _u64p]
        L.xo_window_new.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        L.xo_window_new.restype = C.c_void_p
        L.xo_window_free.argtypes = [C.c_void_p]
        L.xo_window_absorb.argtypes = [C.c_void_p, _u32p, C.c_uint64]
        L.xo_window_rotate.argtypes = [C.c_void_p]
        L.xo_window_digest.argtypes = [C.c_void_p, _u8p]
        L.xo_window_digest_n.argtypes = [C.c_void_p, C.c_uint64, _u8p]
        L.xo_window_base.argtypes = [C.c_void_p]
        L.xo_window_base.restype = C.c_uint64
        L.xo_window_size.argtypes = [C.c_void_p]
        L.xo_window_size.restype = C.c_uint64
        L.xo_window_delta.argtypes = [C.c_void_p, C.c_uint64]
        L.xo_window_delta.restype = C.c_void_p
        L.xo_encode_delta.argtypes = [C.c_uint32, _u64p, _u8p, C.c_uint64]
        L.xo_encode_delta.restype = C.c_uint64
        L.xo_decode_delta.argtypes = [_u8p, C.c_uint64, _u32p, _u64p, C.c_uint64]
        L.xo_decode_delta.restype = C.c_int
        L.xo_encode_positions.argtypes = [_u32p, C.c_uint32, _u8p, C.c_uint64]
        L.xo_encode_positions.restype = C.c_uint64
        L.xo_decode_positions.argtypes = [_u8p, C.c_uint64, _u32p, C.c_uint32, _u32p]
        L.xo_decode_positions.restype = C.c_int

    # primitives
    def chacha20(self, key: bytes, nonce: bytes, n: int, block0: int = 0) -> bytes:
        out = np.zeros(n, np.uint8)
        self.lib.xo_chacha20_stream(_p(out), n, _p(_u8(key)), _p(_u8(nonce)), block0)
        return out.tobytes()

    def prng_expand(self, seed32: bytes, n: int) -> bytes:
        return self.chacha20(seed32, b"\0" * 8, n)

    def blake2b(self, data: bytes, outlen: int = 32) -> bytes:
        out = np.zeros(outlen, np.uint8)
        d = _u8(data) if len(data) else np.zeros(1, np.uint8)
        self.lib.xo_blake2b(_p(out), outlen, _p(d), len(data))
        return out.tobytes()

    def siphash24(self, key16: bytes, data: bytes) -> int:
        d = _u8(data) if len(data) else np.zeros(1, np.uint8)
        return self.lib.xo_siphash24(_p(_u8(key16)), _p(d), len(data))

    def prf(self, key16: bytes, x: int, m: int) -> int:
        return self.lib.xo_prf(_p(_u8(key16)), x, m)

    def bloom_positions(self, item: bytes, h: int, m: int) -> list[int]:
        out = np.zeros(h, np.uint32)
        self.lib.xo_bloom_positions(_p(_u8(item)), len(item), h, m, _p(out, _u32p))
        return out.tolist()

    def make_interest(self, m: int, h: int, id16: bytes, seq: int) -> np.ndarray:
        out = np.zeros(h, np.uint32)
        self.lib.xo_make_interest(m, h, _p(_u8(id16)), seq, _p(out, _u32p))
        return out

    def bloom_hash_count(self, m: int, n: int) -> int:
        return self.lib.xo_bloom_hash_count(m, n)

    def detrng(self, seed: int | bytes) -> "PortRng":
        return PortRng(self, seed)

    # pir
    def answer_batch(self, db: np.ndarray, N: int, S: int, q: np.ndarray, B: int,
                     q_bits: int | None = None, threads: int = 0) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.uint8).reshape(B, -1) if B else np.zeros((0, 1), np.uint8)
        out = np.zeros((B, S), np.uint8)
        threads = threads or (os.cpu_count() or 1)
        rc = self.lib.xo_answer_batch(_p(db), N, S, _p(q) if B else None, q.shape[1] if B else 0,
                                      N if q_bits is None else q_bits, B,
                                      _p(out) if B else None, threads)
        if rc != 0:
            raise ValueError("answer_batch: query length mismatch")
        return out

    def mask_answer(self, ans: bytes, seed32: bytes) -> bytes:
        a = _u8(ans)
        out = np.zeros(len(a), np.uint8)
        self.lib.xo_mask_answer(_p(a), len(a), _p(_u8(seed32)), _p(out))
        return out.tobytes()

    def table(self, buckets, depth, capacity, item_size, seed32) -> "PortTable":
        return PortTable(self, buckets, depth, capacity, item_size, seed32)

    def window(self, m, h, w) -> "PortWindow":
        return PortWindow(self, m, h, w)

    # interest-delta codecs (notify.cpp:139-180)
    def encode_delta(self, m: int, words: np.ndarray) -> bytes:
        w = np.ascontiguousarray(words, np.uint64)
        n = self.lib.xo_encode_delta(m, _p(w, _u64p), None, 0)
        out = np.zeros(max(n, 1), np.uint8)
        self.lib.xo_encode_delta(m, _p(w, _u64p), _p(out), n)
        return out[:n].tobytes()

    def decode_delta(self, buf: bytes):
        """(m_bits, words) or None (the reference's nullopt)."""
        b = _u8(buf) if len(buf) else np.zeros(1, np.uint8)
        m = C.c_uint32()
        if not self.lib.xo_decode_delta(_p(b), len(buf), C.byref(m), None, 0):
            return None
        w = np.zeros((m.value + 63) // 64, np.uint64)
        self.lib.xo_decode_delta(_p(b), len(buf), C.byref(m), _p(w, _u64p), len(w))
        return m.value, w

    # write interest field (notify.cpp:182-214, wire.cpp:154-169)
    def encode_positions(self, positions, cap: int = 64):
        """The cap-byte field, or None where the reference throws (too long)."""
        p = np.ascontiguousarray(positions, np.uint32)
        out = np.zeros(max(cap, 1), np.uint8)
        n = self.lib.xo_encode_positions(_p(p, _u32p), len(p), _p(out), cap)
        return None if n > cap else out[:cap].tobytes()

    def decode_positions(self, buf: bytes):
        """Positions, or None (the reference's nullopt)."""
        b = _u8(buf) if len(buf) else np.zeros(1, np.uint8)
        out = np.zeros(max(8 * len(buf), 1), np.uint32)
        cnt = C.c_uint32()
        if not self.lib.xo_decode_positions(_p(b), len(buf), _p(out, _u32p), len(out), C.byref(cnt)):
            return None
        return out[:cnt.value].copy()


class PortRng:
    def __init__(self, port: Port, seed):
        self.port = port
        self.state = (C.c_uint8 * 48)()
        if isinstance(seed, int):
            port.lib.xo_detrng_init_seed(self.state, seed)
        else:
            port.lib.xo_detrng_init_key(self.state, _p(_u8(seed)))

    def fill(self, n: int) -> bytes:
        out = np.zeros(max(n, 1), np.uint8)
        self.port.lib.xo_detrng_fill(self.state, _p(out), n)
        return out[:n].tobytes()

    def next_u64(self) -> int:
        return self.port.lib.xo_detrng_next_u64(self.state)

    def uniform(self, bound: int) -> int:
        return self.port.lib.xo_detrng_uniform(self.state, bound)

    def gen_queries(self, beta: int, N: int, servers: int) -> np.ndarray:
        out = np.zeros((servers, (N + 7) // 8), np.uint8)
        rc = self.port.lib.xo_gen_queries(beta, N, servers, self.state, _p(out))
        if rc:
            raise ValueError("gen_queries: bad arguments")
        return out


class PortTable:
    def __init__(self, port, buckets, depth, capacity, item_size, seed32):
        self.port, self.buckets, self.depth, self.item = port, buckets, depth, item_size
        self.h = port.lib.xo_table_new(buckets, depth, capacity, item_size, _p(_u8(seed32)))
        if not self.h:
            raise ValueError("cuckoo: bad table dimensions")

    def __del__(self):
        if getattr(self, "h", None):
            self.port.lib.xo_table_free(self.h)

    def insert_batch(self, beta1, beta2, payload) -> np.ndarray:
        b1 = np.ascontiguousarray(beta1, np.uint32)
        b2 = np.ascontiguousarray(beta2, np.uint32)
        pl = np.ascontiguousarray(payload, np.uint8).reshape(len(b1), self.item)
        rep = np.zeros((len(b1), 4), np.uint32)
        for i in range(len(b1)):
            rc = self.port.lib.xo_table_insert(self.h, int(b1[i]), int(b2[i]),
                                               pl[i].ctypes.data_as(_u8p), rep[i].ctypes.data_as(_u32p))
            if rc:
                raise ValueError("cuckoo: bucket index out of range")
        return rep

    def data(self) -> np.ndarray:
        n = self.buckets * self.depth * self.item
        return np.ctypeslib.as_array(C.cast(self.port.lib.xo_table_data(self.h), _u8p), (n,)).copy()

    def state_digest(self) -> bytes:
        out = np.zeros(32, np.uint8)
        self.port.lib.xo_table_state_digest(self.h, _p(out))
        return out.tobytes()

    def counters(self):
        w, l, s = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.port.lib.xo_table_counters(self.h, C.byref(w), C.byref(l), C.byref(s))
        return w.value, l.value, s.value

    def meta(self):
        n = self.buckets * self.depth
        used = np.zeros(n, np.uint8)
        b1 = np.zeros(n, np.uint32)
        b2 = np.zeros(n, np.uint32)
        st = np.zeros(n, np.uint64)
        self.port.lib.xo_table_meta(self.h, _p(used), _p(b1, _u32p), _p(b2, _u32p), _p(st, _u64p))
        return used, b1, b2, st


class PortWindow:
    def __init__(self, port, m, h, w):
        self.port, self.m = port, m
        self.h = port.lib.xo_window_new(m, h, w)
        if not self.h:
            raise ValueError("Window: bad params")

    def __del__(self):
        if getattr(self, "h", None):
            self.port.lib.xo_window_free(self.h)

    def absorb(self, pos):
        p = np.ascontiguousarray(pos, np.uint32)
        if self.port.lib.xo_window_absorb(self.h, _p(p, _u32p), len(p)):
            raise ValueError("Window: position out of range")

    def rotate(self):
        self.port.lib.xo_window_rotate(self.h)

    def digest(self) -> bytes:
        out = np.zeros(32, np.uint8)
        self.port.lib.xo_window_digest(self.h, _p(out))
        return out.tobytes()

    def base(self) -> int:
        return self.port.lib.xo_window_base(self.h)

    def digest_n(self, count: int) -> bytes:
        out = np.zeros(32, np.uint8)
        self.port.lib.xo_window_digest_n(self.h, count, _p(out))
        return out.tobytes()

    def size(self) -> int:
        return self.port.lib.xo_window_size(self.h)

    def delta(self, i: int) -> np.ndarray:
        n = (self.m + 63) // 64
        return np.ctypeslib.as_array(C.cast(self.port.lib.xo_window_delta(self.h, i), _u64p), (n,)).copy()


class Ref:
    """The unmodified reference implementation (oracle/_ref/libxpir_ref.so)."""

    kind = "reference"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_prng_expand.argtypes = [_u8p, _u8p, C.c_uint64]
        L.ref_prf.argtypes = [_u8p, C.c_uint64, C.c_uint64, _u64p]
        L.ref_bloom_positions.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, _u32p]
        L.ref_make_interest.argtypes = [C.c_uint32, C.c_uint32, _u8p, C.c_uint64, _u32p]
        L.ref_bloom_hash_count.argtypes = [C.c_uint32, C.c_uint64]
        L.ref_bloom_hash_count.restype = C.c_uint32
        L.ref_digest.argtypes = [_u8p, C.c_uint64, C.c_uint64, _u8p]
        L.ref_detrng_new.argtypes = [C.c_uint64]
        L.ref_detrng_new.restype = C.c_void_p
        L.ref_detrng_new_key.argtypes = [_u8p]
        L.ref_detrng_new_key.restype = C.c_void_p
        L.ref_detrng_free.argtypes = [C.c_void_p]
        L.ref_detrng_fill.argtypes = [C.c_void_p, _u8p, C.c_uint64]
        L.ref_detrng_next_u64.argtypes = [C.c_void_p]
        L.ref_detrng_next_u64.restype = C.c_uint64
        L.ref_detrng_uniform.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_detrng_uniform.restype = C.c_uint64
        L.ref_gen_queries.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, _u8p]
        L.ref_snapshot_new.argtypes = [_u8p, C.c_uint32, C.c_uint32]
        L.ref_snapshot_new.restype = C.c_void_p
        L.ref_snapshot_new_detrng.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
        L.ref_snapshot_new_detrng.restype = C.c_void_p
        L.ref_snapshot_free.argtypes = [C.c_void_p]
        L.ref_snapshot_data.argtypes = [C.c_void_p]
        L.ref_snapshot_data.restype = C.c_void_p
        L.ref_answer.argtypes = [C.c_void_p, _u8p, C.c_uint32, _u8p]
        L.ref_answer_batch.argtypes = [C.c_void_p, _u8p, C.c_uint64, C.c_uint32, _u8p, C.c_uint32,
                                       C.POINTER(C.c_double)]
        L.ref_mask_answer.argtypes = [_u8p, C.c_uint64, _u8p, _u8p]
        L.ref_table_new.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, _u8p]
        L.ref_table_new.restype = C.c_void_p
        L.ref_table_free.argtypes = [C.c_void_p]
        L.ref_table_insert_batch.argtypes = [C.c_void_p, _u32p, _u32p, _u8p, C.c_uint64, _u32p]
        L.ref_table_data.argtypes = [C.c_void_p, _u8p]
        L.ref_table_state_digest.argtypes = [C.c_void_p, _u8p]
        L.ref_table_counters.argtypes = [C.c_void_p, _u64p, _u64p]
        L.ref_table_slot_used.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
        L.ref_window_new.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        L.ref_window_new.restype = C.c_void_p
        L.ref_window_free.argtypes = [C.c_void_p]
        L.ref_window_absorb.argtypes = [C.c_void_p, _u32p, C.c_uint64]
        L.ref_window_rotate.argtypes = [C.c_void_p]
        L.ref_window_digest.argtypes = [C.c_void_p, _u8p]
        L.ref_window_size.argtypes = [C.c_void_p]
        L.ref_window_size.restype = C.c_uint64
        L.ref_window_delta_words.argtypes = [C.c_void_p, C.c_uint64, _u64p]
        L.ref_encode_delta.argtypes = [C.c_uint32, _u64p, _u8p, C.c_uint64]
        L.ref_encode_delta.restype = C.c_int64
        L.ref_decode_delta.argtypes = [_u8p, C.c_uint64, _u32p, _u64p, C.c_uint64]
        L.ref_decode_delta.restype = C.c_int
        L.ref_encode_positions_batch.argtypes = [_u32p, C.c_uint32, C.c_uint64, C.c_uint64, _u8p, _u8p]
        L.ref_encode_positions_batch.restype = None
        L.ref_decode_positions_batch.argtypes = [_u8p, C.c_uint64, C.c_uint64, _u32p, _u32p]
        L.ref_decode_positions_batch.restype = None
        L.ref_encode_positions.argtypes = [_u32p, C.c_uint64, _u8p, C.c_uint64]
        L.ref_encode_positions.restype = C.c_int64
        L.ref_decode_positions.argtypes = [_u8p, C.c_uint64, _u32p, C.c_uint32, _u32p]
        L.ref_decode_positions.restype = C.c_int
        L.ref_window_digest_n.argtypes = [C.c_void_p, C.c_uint64, _u8p]

    def _chk(self, rc):
        if rc == -1:
            raise ValueError(self.lib.ref_last_error().decode())
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def prng_expand(self, seed32: bytes, n: int) -> bytes:
        out = np.zeros(max(n, 1), np.uint8)
        self._chk(self.lib.ref_prng_expand(_p(_u8(seed32)), _p(out), n))
        return out[:n].tobytes()

    def prf(self, key16: bytes, x: int, m: int) -> int:
        v = C.c_uint64()
        self._chk(self.lib.ref_prf(_p(_u8(key16)), x, m, C.byref(v)))
        return v.value

    def bloom_positions(self, item: bytes, h: int, m: int) -> list[int]:
        out = np.zeros(max(h, 1), np.uint32)
        self._chk(self.lib.ref_bloom_positions(_p(_u8(item)), len(item), h, m, _p(out, _u32p)))
        return out[:h].tolist()

    def make_interest(self, m: int, h: int, id16: bytes, seq: int) -> np.ndarray:
        out = np.zeros(h, np.uint32)
        self._chk(self.lib.ref_make_interest(m, h, _p(_u8(id16)), seq, _p(out, _u32p)))
        return out

    def bloom_hash_count(self, m: int, n: int) -> int:
        return self.lib.ref_bloom_hash_count(m, n)

    def blake2b(self, data: bytes, outlen: int = 32) -> bytes:
        out = np.zeros(outlen, np.uint8)
        d = _u8(data) if len(data) else np.zeros(1, np.uint8)
        self._chk(self.lib.ref_digest(_p(d), len(data), outlen, _p(out)))
        return out.tobytes()

    def detrng(self, seed) -> "RefRng":
        return RefRng(self, seed)

    def snapshot(self, db: np.ndarray, N: int, S: int) -> "RefSnapshot":
        return RefSnapshot(self, self.lib.ref_snapshot_new(_p(db), N, S), N, S)

    def snapshot_detrng(self, rng: "RefRng", N: int, S: int) -> "RefSnapshot":
        return RefSnapshot(self, self.lib.ref_snapshot_new_detrng(rng.h, N, S), N, S)

    def answer_batch(self, db: np.ndarray, N: int, S: int, q: np.ndarray, B: int,
                     threads: int = 0) -> np.ndarray:
        snap = self.snapshot(db, N, S)
        return snap.answer_batch(q, B, threads)[0]

    def mask_answer(self, ans: bytes, seed32: bytes) -> bytes:
        a = _u8(ans)
        out = np.zeros(len(a), np.uint8)
        self._chk(self.lib.ref_mask_answer(_p(a), len(a), _p(_u8(seed32)), _p(out)))
        return out.tobytes()

    def table(self, buckets, depth, capacity, item_size, seed32) -> "RefTable":
        return RefTable(self, buckets, depth, capacity, item_size, seed32)

    def window(self, m, h, w) -> "RefWindow":
        return RefWindow(self, m, h, w)

    def encode_delta(self, m: int, words: np.ndarray) -> bytes:
        w = np.ascontiguousarray(words, np.uint64)
        n = self.lib.ref_encode_delta(m, _p(w, _u64p), None, 0)
        out = np.zeros(max(n, 1), np.uint8)
        self.lib.ref_encode_delta(m, _p(w, _u64p), _p(out), n)
        return out[:n].tobytes()

    def decode_delta(self, buf: bytes):
        b = _u8(buf) if len(buf) else np.zeros(1, np.uint8)
        m = C.c_uint32()
        if not self.lib.ref_decode_delta(_p(b), len(buf), C.byref(m), None, 0):
            return None
        w = np.zeros((m.value + 63) // 64, np.uint64)
        self.lib.ref_decode_delta(_p(b), len(buf), C.byref(m), _p(w, _u64p), len(w))
        return m.value, w

    def encode_positions(self, positions, cap: int = 64):
        p = np.ascontiguousarray(positions, np.uint32)
        out = np.zeros(max(cap, 1), np.uint8)
        n = self.lib.ref_encode_positions(_p(p, _u32p) if len(p) else None, len(p), _p(out), cap)
        return None if n < 0 else out[:cap].tobytes()

    def encode_positions_batch(self, pos: np.ndarray, cap: int = 64):
        """(fields n x cap, ok n) for n writes x h positions (reference loop in C++)."""
        p = np.ascontiguousarray(pos, np.uint32)
        n, h = p.shape
        out = np.zeros((n, cap), np.uint8)
        ok = np.zeros(n, np.uint8)
        self.lib.ref_encode_positions_batch(_p(p, _u32p), h, n, cap, _p(out), _p(ok))
        return out, ok

    def decode_positions_batch(self, fields: np.ndarray):
        f = np.ascontiguousarray(fields, np.uint8)
        n, cap = f.shape
        pos = np.zeros((n, cap), np.uint32)
        cnt = np.zeros(n, np.uint32)
        self.lib.ref_decode_positions_batch(_p(f), cap, n, _p(pos, _u32p), _p(cnt, _u32p))
        return pos, cnt

    def decode_positions(self, buf: bytes):
        b = _u8(buf) if len(buf) else np.zeros(1, np.uint8)
        out = np.zeros(max(8 * len(buf), 1), np.uint32)
        cnt = C.c_uint32()
        if not self.lib.ref_decode_positions(_p(b), len(buf), _p(out, _u32p), len(out), C.byref(cnt)):
            return None
        return out[:cnt.value].copy()


class RefRng:
    def __init__(self, ref: Ref, seed):
        self.ref = ref
        self.h = ref.lib.ref_detrng_new(seed) if isinstance(seed, int) else ref.lib.ref_detrng_new_key(_p(_u8(seed)))

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_detrng_free(self.h)

    def fill(self, n: int) -> bytes:
        out = np.zeros(max(n, 1), np.uint8)
        self.ref.lib.ref_detrng_fill(self.h, _p(out), n)
        return out[:n].tobytes()

    def next_u64(self) -> int:
        return self.ref.lib.ref_detrng_next_u64(self.h)

    def uniform(self, bound: int) -> int:
        return self.ref.lib.ref_detrng_uniform(self.h, bound)

    def gen_queries(self, beta: int, N: int, servers: int) -> np.ndarray:
        out = np.zeros((servers, (N + 7) // 8), np.uint8)
        self.ref._chk(self.ref.lib.ref_gen_queries(beta, N, servers, self.h, _p(out)))
        return out


class RefSnapshot:
    def __init__(self, ref, h, N, S):
        self.ref, self.h, self.N, self.S = ref, h, N, S

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_snapshot_free(self.h)

    def data(self) -> np.ndarray:
        n = self.N * self.S
        return np.ctypeslib.as_array(C.cast(self.ref.lib.ref_snapshot_data(self.h), _u8p), (n,))

    def answer(self, q: np.ndarray, q_bits: int | None = None) -> np.ndarray:
        q = _u8(q)
        out = np.zeros(self.S, np.uint8)
        self.ref._chk(self.ref.lib.ref_answer(self.h, _p(q), self.N if q_bits is None else q_bits, _p(out)))
        return out

    def answer_batch(self, q: np.ndarray, B: int, threads: int = 0):
        q = np.ascontiguousarray(q, dtype=np.uint8).reshape(B, -1)
        out = np.zeros((B, self.S), np.uint8)
        secs = C.c_double()
        self.ref._chk(self.ref.lib.ref_answer_batch(self.h, _p(q), q.shape[1], B, _p(out),
                                                    threads or (os.cpu_count() or 1), C.byref(secs)))
        return out, secs.value


class RefTable:
    def __init__(self, ref, buckets, depth, capacity, item_size, seed32):
        self.ref, self.buckets, self.depth, self.item = ref, buckets, depth, item_size
        self.h = ref.lib.ref_table_new(buckets, depth, capacity, item_size, _p(_u8(seed32)))
        if not self.h:
            raise ValueError(ref.lib.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_table_free(self.h)

    def insert_batch(self, beta1, beta2, payload) -> np.ndarray:
        b1 = np.ascontiguousarray(beta1, np.uint32)
        b2 = np.ascontiguousarray(beta2, np.uint32)
        pl = np.ascontiguousarray(payload, np.uint8)
        rep = np.zeros((len(b1), 4), np.uint32)
        self.ref._chk(self.ref.lib.ref_table_insert_batch(self.h, _p(b1, _u32p), _p(b2, _u32p), _p(pl),
                                                          len(b1), _p(rep, _u32p)))
        return rep

    def data(self) -> np.ndarray:
        out = np.zeros(self.buckets * self.depth * self.item, np.uint8)
        self.ref.lib.ref_table_data(self.h, _p(out))
        return out

    def state_digest(self) -> bytes:
        out = np.zeros(32, np.uint8)
        self.ref.lib.ref_table_state_digest(self.h, _p(out))
        return out.tobytes()

    def counters(self):
        w, l = C.c_uint64(), C.c_uint64()
        self.ref.lib.ref_table_counters(self.h, C.byref(w), C.byref(l))
        return w.value, l.value

    def slot_used(self, b, s) -> bool:
        return bool(self.ref.lib.ref_table_slot_used(self.h, b, s))


class RefWindow:
    def __init__(self, ref, m, h, w):
        self.ref, self.m = ref, m
        self.h = ref.lib.ref_window_new(m, h, w)
        if not self.h:
            raise ValueError(ref.lib.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_window_free(self.h)

    def absorb(self, pos):
        p = np.ascontiguousarray(pos, np.uint32)
        self.ref._chk(self.ref.lib.ref_window_absorb(self.h, _p(p, _u32p), len(p)))

    def rotate(self):
        self.ref.lib.ref_window_rotate(self.h)

    def digest(self, count: int | None = None) -> bytes:
        out = np.zeros(32, np.uint8)
        if count is None:
            self.ref.lib.ref_window_digest(self.h, _p(out))
        else:
            self.ref.lib.ref_window_digest_n(self.h, count, _p(out))
        return out.tobytes()

    def size(self) -> int:
        return self.ref.lib.ref_window_size(self.h)

    def delta(self, i: int) -> np.ndarray:
        out = np.zeros((self.m + 63) // 64, np.uint64)
        self.ref.lib.ref_window_delta_words(self.h, i, _p(out, _u64p))
        return out


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def best() -> "Ref | Port":
    """The reference build when present, else the C restatement."""
    return Ref() if ref_available() else Port()

"""B200-native server hot path of Talek (arXiv 2001.08250): batched XOR-PIR over a
blocked-cuckoo-hashed store, plus the per-round write path.

This module is a thin ctypes mirror of the C-ABI in ``include/xpir.h``; every
computation happens in the sm_100a kernels of ``libxpir.so`` (built in-tree by
``make -C paper_2001_08250_b200``). There is no CPU fallback: importing works
anywhere, but any call fails loudly (``XpirError``) if the library is missing
or no GPU is visible.

Names mirror the reference interface (``/root/reference/proj/include/oblog``):

=========================  ==================================================
reference                  here
=========================  ==================================================
pir::Snapshot              ``Store`` (one shard of a sealed snapshot in HBM)
pir::answer_batch          ``Store.answer_batch`` / ``answer_batch_dev``
pir::mask_answer           ``mask_seeds=`` argument (fused K3)
crypto::prng_expand        ``prng_expand`` / ``Store.answer_batch_seeded``
pir::reconstruct           ``xor_reduce_dev`` (K4, also over NVLink peers)
cuckoo::Table              ``Table``
notify::Window             ``Window``
crypto::prf                ``prf_batch``
notify::make_interest      ``make_interest_batch``
answer_share batching      ``Batcher`` (concurrent single requests -> one scan)
=========================  ==================================================
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libxpir.so")

XPIR_OK, XPIR_EINVAL, XPIR_ECUDA, XPIR_ENOMEM, XPIR_ESTATE = 0, -1, -2, -3, -4
MAX_DISPLACEMENTS = 500  # cuckoo.hpp:15


class XpirError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"xpir error {code}: {msg}")
        self.code = code


class InvalidArgument(XpirError, ValueError):
    """The reference would throw std::invalid_argument here."""


_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p

_lib = None


def build(verbose: bool = False) -> str:
    """Compile libxpir.so for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    out = subprocess.run(["make", "-C", HERE, "-j4"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("libxpir build failed:\n" + out.stdout + out.stderr)
    if verbose:
        print(out.stdout)
    return LIB_PATH


_SIGS = {
    "xpir_last_error": ([], C.c_char_p),
    "xpir_version": ([], C.c_int),
    "xpir_launch_count": ([], C.c_uint64),
    "xpir_set_scan_opts": ([_vp], C.c_int),
    "xpir_set_host_sync": ([C.c_int], C.c_int),
    "xpir_last_scan_kernel": ([], C.c_int),
    "xpir_scan_timing": ([C.c_int], C.c_int),
    "xpir_scan_timing_collect": ([C.POINTER(C.c_double), _u32p], C.c_int),
    "xpir_measure_peaks": ([C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
    "xpir_probe_tmem": ([C.c_int, C.c_int, C.POINTER(C.c_double)], C.c_int),
    "xpir_dev_alloc": ([C.c_int, C.c_uint64, C.POINTER(_vp)], C.c_int),
    "xpir_dev_free": ([C.c_int, _vp], C.c_int),
    "xpir_ipc_get_handle": ([C.c_int, _vp, _u8p], C.c_int),
    "xpir_ipc_open": ([C.c_int, _u8p, C.POINTER(_vp)], C.c_int),
    "xpir_ipc_close": ([C.c_int, _vp], C.c_int),
    "xpir_device_sync": ([C.c_int], C.c_int),
    "xpir_store_create": ([C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(_vp)], C.c_int),
    "xpir_store_destroy": ([_vp], C.c_int),
    "xpir_store_upload": ([_vp, _u8p, C.c_uint64], C.c_int),
    "xpir_store_upload_dev": ([_vp, _vp, C.c_uint64, _vp], C.c_int),
    "xpir_store_fill_keystream": ([_vp, _u8p, C.c_uint64, C.c_uint64, _vp], C.c_int),
    "xpir_store_info": ([_vp, _u32p, _u32p, _u32p, _u32p, _u64p, C.POINTER(_vp)], C.c_int),
    "xpir_store_download": ([_vp, C.c_uint64, C.c_uint64, _u8p], C.c_int),
    "xpir_answer_batch": ([_vp, _u8p, C.c_uint64, C.c_uint32, C.c_uint32, _u8p, _u8p], C.c_int),
    "xpir_answer_batch_seeded": ([_vp, _u8p, C.c_uint32, _u8p, _u8p], C.c_int),
    "xpir_answer_batch_dev": ([_vp, _vp, C.c_uint64, C.c_uint32, C.c_uint32, _vp, _vp, _vp], C.c_int),
    "xpir_answer_batch_seeded_dev": ([_vp, _vp, C.c_uint32, _vp, _vp, _vp], C.c_int),
    "xpir_query_window_bytes": ([_vp], C.c_uint64),
    "xpir_answer_batch_seeded_peer_dev": ([_vp, _vp, C.c_uint32, C.POINTER(_vp), _u32p, C.c_uint32, C.c_uint32,
                                           _vp], C.c_int),
    "xpir_store_peer_stats": ([_vp, _u64p, _u64p, C.c_int], C.c_int),
    "xpir_table_insert_batch_async": ([_vp, _vp, _vp, _vp, C.c_uint64, _vp, _vp, _vp], C.c_int),
    "xpir_table_finish": ([_vp, _u64p], C.c_int),
    "xpir_write_betas_dev": ([C.c_int, _u8p, _u8p, _vp, C.c_uint64, C.c_uint32, _vp, _vp, _vp], C.c_int),
    "xpir_init_rows_dev": ([C.c_int, _vp, C.c_uint32, C.c_uint32, C.c_uint32, _vp, _vp], C.c_int),
    "xpir_expand_queries_dev": ([C.c_int, _vp, C.c_uint32, C.c_uint64, C.c_uint64, _vp, C.c_uint64, _vp], C.c_int),
    "xpir_mask_answer": ([_u8p, C.c_uint64, _u8p, _u8p], C.c_int),
    "xpir_mask_dev": ([C.c_int, _vp, _vp, C.c_uint32, C.c_uint32, _vp], C.c_int),
    "xpir_xor_reduce_dev": ([C.c_int, _vp, _vp, C.c_uint32, C.c_uint64, _vp], C.c_int),
    "xpir_prng_expand": ([_u8p, _u8p, C.c_uint64], C.c_int),
    "xpir_keystream_dev": ([C.c_int, _u8p, C.c_uint64, C.c_uint64, _vp, C.c_uint64, _vp], C.c_int),
    "xpir_keystream_rows_dev": ([C.c_int, _u8p, C.c_uint64, C.c_uint32, C.c_uint64, _vp, C.c_uint64, _vp], C.c_int),
    "xpir_prf_batch": ([_u8p, _u64p, C.c_uint64, C.c_uint64, _u64p], C.c_int),
    "xpir_prf_batch_dev": ([C.c_int, _u8p, _vp, C.c_uint64, C.c_uint64, _vp, _vp, _vp], C.c_int),
    "xpir_table_reserve": ([_vp, C.c_uint64], C.c_int),
    "xpir_window_absorb_interest_dev": ([_vp, _u8p, _vp, C.c_uint64, _vp], C.c_int),
    "xpir_make_interest_batch": ([C.c_uint32, C.c_uint32, _u8p, _u64p, C.c_uint64, _u32p], C.c_int),
    "xpir_bloom_positions": ([_u8p, C.c_uint64, C.c_uint32, C.c_uint32, _u32p], C.c_int),
    "xpir_blake2b": ([_u8p, C.c_uint64, C.c_uint32, _u8p], C.c_int),
    "xpir_table_create": ([C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, _u8p, C.POINTER(_vp)], C.c_int),
    "xpir_table_destroy": ([_vp], C.c_int),
    "xpir_table_insert_batch": ([_vp, _u32p, _u32p, _u8p, C.c_uint64, _u32p], C.c_int),
    "xpir_table_insert_batch_dev": ([_vp, _vp, _vp, _vp, C.c_uint64, _vp, _vp], C.c_int),
    "xpir_table_snapshot": ([_vp, _u8p], C.c_int),
    "xpir_table_seal": ([_vp, _vp, C.c_uint64, _vp], C.c_int),
    "xpir_table_meta": ([_vp, _u8p, _u32p, _u32p, _u64p], C.c_int),
    "xpir_table_counters": ([_vp, _u64p, _u64p, _u64p], C.c_int),
    "xpir_table_state_digest": ([_vp, _u8p], C.c_int),
    "xpir_table_slot_used": ([_vp, C.c_uint32, C.c_uint32], C.c_int),
    "xpir_table_device_data": ([_vp], _vp),
    "xpir_window_create": ([C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(_vp)], C.c_int),
    "xpir_window_destroy": ([_vp], C.c_int),
    "xpir_window_absorb": ([_vp, _u32p, C.c_uint64], C.c_int),
    "xpir_window_absorb_dev": ([_vp, _vp, C.c_uint64, _vp], C.c_int),
    "xpir_window_absorb_interest": ([_vp, _u8p, _u64p, C.c_uint64], C.c_int),
    "xpir_window_rotate": ([_vp], C.c_int),
    "xpir_window_info": ([_vp, _u64p, _u64p], C.c_int),
    "xpir_window_delta": ([_vp, C.c_uint64, _u64p], C.c_int),
    "xpir_window_digest": ([_vp, _u8p], C.c_int),
    "xpir_server_create": ([C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, _u8p, C.c_uint32, C.c_uint32,
                            C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(_vp)], C.c_int),
    "xpir_server_destroy": ([_vp], C.c_int),
    "xpir_server_apply_round": ([_vp, _u32p, _u32p, _u8p, _u32p, C.c_uint32, C.c_uint64, C.c_int, _u32p, _u64p],
                                C.c_int),
    "xpir_server_reserve": ([_vp, C.c_uint64], C.c_int),
    "xpir_server_seal": ([_vp, _u64p], C.c_int),
    "xpir_server_snapshot": ([_vp, C.c_uint64, C.POINTER(_vp)], C.c_int),
    "xpir_server_info": ([_vp, _u64p, _u64p, _u64p, C.POINTER(_vp), C.POINTER(_vp)], C.c_int),
    "xpir_table_create_shard": ([C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, _u8p, C.c_uint32,
                                 C.c_uint32, C.POINTER(_vp)], C.c_int),
    "xpir_table_shard": ([_vp, _u32p, _u32p], C.c_int),
    "xpir_table_insert_walk_dev": ([_vp, _vp, _vp, C.c_uint64, _vp, _vp], C.c_int),
    "xpir_table_apply_gather_dev": ([_vp, _vp, _vp], C.c_int),
    "xpir_table_apply_scatter_dev": ([_vp, _vp, _vp], C.c_int),
    "xpir_server_create_shard": ([C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, _u8p, C.c_uint32,
                                  C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.POINTER(_vp)], C.c_int),
    "xpir_server_apply_round_sharded": ([_vp, _u32p, _u32p, _u8p, _u32p, C.c_uint32, C.c_uint64, C.c_int, _vp,
                                         _vp, _vp, _u32p, _u64p], C.c_int),
    "xpir_answer_batch_mixed": ([_vp, C.c_uint32, _u8p, _u8p, _u8p, C.c_uint64, C.c_uint32, _u8p, _u8p], C.c_int),
    "xpir_window_digest_n": ([_vp, C.c_uint64, _u8p], C.c_int),
    "xpir_window_encode_delta": ([_vp, C.c_uint64, _u8p, C.c_uint64, _u64p], C.c_int),
    "xpir_encode_delta_dev": ([C.c_int, _vp, C.c_uint32, _vp, C.c_uint64, _u64p, _vp], C.c_int),
    "xpir_decode_delta": ([C.c_int, _u8p, C.c_uint64, _u32p, _u64p, C.c_uint64], C.c_int),
    "xpir_encode_positions_dev": ([C.c_int, _vp, C.c_uint32, C.c_uint64, C.c_uint32, _vp, _vp, _vp], C.c_int),
    "xpir_decode_positions_dev": ([C.c_int, _vp, C.c_uint32, C.c_uint64, _vp, _vp, _vp], C.c_int),
    "xpir_server_freeze": ([_vp, _u64p, _u64p, _u8p, _u64p], C.c_int),
    "xpir_batcher_create": ([_vp, C.c_uint32, C.c_uint32, C.POINTER(_vp)], C.c_int),
    "xpir_batcher_destroy": ([_vp], C.c_int),
    "xpir_batcher_answer": ([_vp, _u8p, C.c_uint32, _u8p, _u8p], C.c_int),
    "xpir_batcher_stats": ([_vp, _u64p, _u64p, _u64p], C.c_int),
    "xpir_batcher_create_geometry": ([C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(_vp)],
                                     C.c_int),
    "xpir_batcher_answer_on": ([_vp, _vp, _u8p, C.c_uint32, _u8p, _u8p], C.c_int),
    "xpir_server_snapshot_acquire": ([_vp, C.c_uint64, C.POINTER(_vp), _u64p], C.c_int),
    "xpir_server_snapshot_release": ([_vp, _vp], C.c_int),
}

EXPORTED_SYMBOLS = tuple(_SIGS)


def lib() -> C.CDLL:
    """Load libxpir.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise XpirError(XPIR_ECUDA, f"{LIB_PATH} missing: run paper_2001_08250_b200.build()")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _destroy(fn) -> None:
    """Release a handle; quietly skipped while the interpreter is shutting down
    (module globals may already be gone when __del__ runs)."""
    try:
        fn()
    except Exception:  # noqa: BLE001
        pass


def _quiet_del(self) -> None:
    """__del__ of every handle class: close(), but never raise from a finalizer
    (at interpreter shutdown even this module's globals may be gone)."""
    try:
        self.close()
    except Exception:  # noqa: BLE001
        pass


def _check(rc: int) -> int:
    if rc >= 0:
        return rc
    msg = lib().xpir_last_error().decode(errors="replace")
    if rc == XPIR_EINVAL:
        raise InvalidArgument(rc, msg)
    raise XpirError(rc, msg)


def _p(a: np.ndarray, t=_u8p):
    return a.ctypes.data_as(t)


def _u8(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(x), dtype=np.uint8).copy()
    return np.ascontiguousarray(x, dtype=np.uint8)


def _ptr(x) -> int | None:
    """Device pointer of a torch tensor (or an int address)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(s) -> int | None:
    if s is None:
        return None
    h = s if isinstance(s, int) else s.cuda_stream  # torch.cuda.Stream
    # handle 0 is the legacy default stream; NULL would select the library's own
    # stream, so pass cudaStreamLegacy (0x1) to keep ordering with the caller.
    return h if h else 1


def launch_count() -> int:
    return lib().xpir_launch_count()


def last_scan_kernel() -> int:
    """Kernel of the last scan: 1 direct select-XOR, 2 M4RM byte tables (register
    accumulators), 3 byte-granular, 5 byte tables with half-TMEM accumulators,
    7 nibble tables, 8 9-bucket quad tables (full TMEM), 9 6-bucket tables."""
    return lib().xpir_last_scan_kernel()


class _ScanOpts(C.Structure):
    _fields_ = [("kernel", C.c_int), ("ctas_per_sm", C.c_int), ("reserved", C.c_int * 6)]


def set_scan_opts(kernel: int = 0, ctas_per_sm: int = 0) -> None:
    o = _ScanOpts(kernel, ctas_per_sm)
    _check(lib().xpir_set_scan_opts(C.byref(o)))


def scan_timing(enable: bool) -> None:
    _check(lib().xpir_scan_timing(1 if enable else 0))


def scan_timing_collect() -> tuple[float, int]:
    """(summed scan-kernel ms, launches) since the last collect."""
    ms, n = C.c_double(), C.c_uint32()
    _check(lib().xpir_scan_timing_collect(C.byref(ms), C.byref(n)))
    return ms.value, n.value


def measure_peaks(device: int = 0) -> dict:
    """LOP3 lane-op rate and LDS.128 bandwidth of this GPU (roofline denominators)."""
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    _check(lib().xpir_measure_peaks(device, C.byref(a), C.byref(b), C.byref(c)))
    return {"lop3_per_s": a.value, "smem_bytes_per_s": b.value, "sm_clock_attr_mhz": c.value}


def probe_tmem(variant: int, device: int = 0) -> float:
    """tcgen05.ld bytes per SM clock (diagnostic microbenchmark)."""
    v = C.c_double()
    _check(lib().xpir_probe_tmem(device, variant, C.byref(v)))
    return v.value


class DeviceBuffer:
    """A whole cudaMalloc allocation (IPC-shareable), exposed to torch through
    __cuda_array_interface__ (``torch.as_tensor(buf, device=...)`` is zero-copy)."""

    def __init__(self, nbytes: int, device: int = 0):
        p = _vp()
        _check(lib().xpir_dev_alloc(device, nbytes, C.byref(p)))
        self.ptr, self.nbytes, self.device = p.value, nbytes, device
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (self.ptr, False),
                                         "version": 3, "strides": None}

    def close(self):
        if getattr(self, "ptr", None):
            _destroy(lambda: lib().xpir_dev_free(self.device, self.ptr))
            self.ptr = None

    __del__ = _quiet_del


def ipc_handle(d_ptr, device: int = 0) -> bytes:
    out = np.empty(64, np.uint8)
    _check(lib().xpir_ipc_get_handle(device, _ptr(d_ptr), _p(out)))
    return out.tobytes()


def ipc_open(handle: bytes, device: int = 0) -> int:
    p = _vp()
    _check(lib().xpir_ipc_open(device, _p(_u8(handle)), C.byref(p)))
    return p.value


def ipc_close(d_ptr: int, device: int = 0) -> None:
    _check(lib().xpir_ipc_close(device, d_ptr))


def device_sync(device: int = 0) -> None:
    _check(lib().xpir_device_sync(device))


# ---------------------------------------------------------------------------
# pir::Snapshot shard
# ---------------------------------------------------------------------------
class Store:
    """Buckets [lo, hi) of an N-bucket sealed snapshot, resident on `device`."""

    def __init__(self, bucket_count: int, bucket_size: int, lo: int = 0, hi: int | None = None,
                 device: int = 0):
        hi = bucket_count if hi is None else hi
        h = _vp()
        _check(lib().xpir_store_create(device, bucket_count, bucket_size, lo, hi, C.byref(h)))
        self.h, self.N, self.S, self.lo, self.hi, self.device = h, bucket_count, bucket_size, lo, hi, device

    def close(self):
        if getattr(self, "h", None):
            _destroy(lambda: lib().xpir_store_destroy(self.h))
            self.h = None

    __del__ = _quiet_del

    @property
    def shard_bytes(self) -> int:
        return (self.hi - self.lo) * self.S

    def upload(self, buckets: np.ndarray, epoch: int = 1) -> None:
        b = _u8(buckets).reshape(-1)
        if b.size != self.shard_bytes:
            raise InvalidArgument(XPIR_EINVAL, "upload: size differs from the shard")
        _check(lib().xpir_store_upload(self.h, _p(b), epoch))

    def upload_dev(self, src, epoch: int = 1, stream=None) -> None:
        _check(lib().xpir_store_upload_dev(self.h, _ptr(src), epoch, _stream(stream)))

    def fill_keystream(self, key32: bytes, nonce: int, epoch: int = 1, stream=None) -> None:
        """Shard window of one DetRng fill call (rng.cpp:25-31), generated on device."""
        _check(lib().xpir_store_fill_keystream(self.h, _p(_u8(key32)), nonce, epoch, _stream(stream)))

    def download(self, offset: int = 0, length: int | None = None) -> np.ndarray:
        length = self.shard_bytes - offset if length is None else length
        out = np.empty(max(length, 1), np.uint8)
        _check(lib().xpir_store_download(self.h, offset, length, _p(out)))
        return out[:length]

    def device_ptr(self) -> int:
        p = _vp()
        _check(lib().xpir_store_info(self.h, None, None, None, None, None, C.byref(p)))
        return p.value

    @property
    def query_window_bytes(self) -> int:
        return lib().xpir_query_window_bytes(self.h)

    # pir::answer_batch (pir.cpp:41-52) [+ mask_answer, pir.cpp:65-69]
    def answer_batch(self, queries: np.ndarray, q_bits: int | None = None,
                     mask_seeds: np.ndarray | None = None) -> np.ndarray:
        q = _u8(queries)
        if q.ndim == 1:
            q = q.reshape(1, -1)
        B = q.shape[0]
        out = np.empty((B, self.S), np.uint8)
        ms = None if mask_seeds is None else _u8(mask_seeds).reshape(B, 32)
        _check(lib().xpir_answer_batch(self.h, _p(q) if B else None, q.shape[1] if B else 0,
                                       self.N if q_bits is None else q_bits, B,
                                       None if ms is None else _p(ms), _p(out) if B else None))
        return out

    def answer(self, query, q_bits: int | None = None) -> np.ndarray:
        """pir::answer (pir.cpp:29-39)."""
        return self.answer_batch(_u8(query).reshape(1, -1), q_bits)[0]

    def answer_batch_seeded(self, seeds: np.ndarray, mask_seeds: np.ndarray | None = None,
                            out: np.ndarray | None = None) -> np.ndarray:
        """`out` (B x S uint8, e.g. a view of pinned host memory) is filled in place."""
        s = _u8(seeds).reshape(-1, 32)
        B = s.shape[0]
        if out is None:
            out = np.empty((B, self.S), np.uint8)
        elif out.dtype != np.uint8 or out.shape != (B, self.S) or not out.flags.c_contiguous:
            raise InvalidArgument(XPIR_EINVAL, "answer_batch_seeded: out must be a contiguous B x S uint8 array")
        ms = None if mask_seeds is None else _u8(mask_seeds).reshape(B, 32)
        _check(lib().xpir_answer_batch_seeded(self.h, _p(s), B, None if ms is None else _p(ms), _p(out)))
        return out

    def answer_batch_mixed(self, is_seed, seeds, rows, mask_seeds=None) -> np.ndarray:
        """Seed-compressed shares: request r is prng_expand(seed) when is_seed[r], else
        an explicit vector; `seeds` (n_seeded x 32) and `rows` (n_explicit x ceil(N/8))
        are compacted in request order."""
        f = np.ascontiguousarray(is_seed, np.uint8).reshape(-1)
        B = f.size
        ns = int(f.sum())
        sd = _u8(seeds).reshape(ns, 32) if ns else np.zeros((1, 32), np.uint8)
        nb = (self.N + 7) // 8
        q = _u8(rows).reshape(B - ns, -1) if B - ns else np.zeros((1, nb), np.uint8)
        out = np.empty((B, self.S), np.uint8)
        ms = None if mask_seeds is None else _u8(mask_seeds).reshape(B, 32)
        _check(lib().xpir_answer_batch_mixed(self.h, B, _p(f), _p(sd), _p(q), q.shape[1], self.N,
                                             None if ms is None else _p(ms), _p(out)))
        return out

    # device variants (torch tensors or raw pointers)
    def answer_batch_dev(self, d_q, q_stride: int, B: int, d_out, d_mask=None, stream=None,
                         q_bits: int | None = None) -> None:
        _check(lib().xpir_answer_batch_dev(self.h, _ptr(d_q), q_stride, self.N if q_bits is None else q_bits,
                                           B, _ptr(d_mask), _ptr(d_out), _stream(stream)))

    def answer_batch_seeded_dev(self, d_seeds, B: int, d_out, d_mask=None, stream=None) -> None:
        _check(lib().xpir_answer_batch_seeded_dev(self.h, _ptr(d_seeds), B, _ptr(d_mask), _ptr(d_out),
                                                  _stream(stream)))

    def answer_batch_seeded_peer_dev(self, d_seeds, B: int, out_ptrs: list[int], row_bounds: list[int],
                                     self_rank: int, stream=None) -> None:
        """Shard scan fused with the cross-GPU XOR reduce: each finished answer tile
        is pushed once into its owner rank's buffer (include/xpir.h)."""
        ptrs = (_vp * len(out_ptrs))(*out_ptrs)
        bounds = np.ascontiguousarray(row_bounds, np.uint32)
        _check(lib().xpir_answer_batch_seeded_peer_dev(self.h, _ptr(d_seeds), B, ptrs, _p(bounds, _u32p),
                                                       len(out_ptrs), self_rank, _stream(stream)))

    def peer_stats(self, reset: bool = False) -> dict:
        """Bytes the fused epilogue pushed to peer ranks' rows / own rows."""
        r, o = C.c_uint64(), C.c_uint64()
        _check(lib().xpir_store_peer_stats(self.h, C.byref(r), C.byref(o), 1 if reset else 0))
        return {"remote_bytes": r.value, "own_bytes": o.value}


class Batcher:
    """Read batcher over a store (include/xpir.h): ``answer`` is safe to call from
    many threads at once — concurrent single requests (server::answer_share,
    server.cpp:115-135) are coalesced into one scan of up to ``max_batch``
    requests, sealed ``max_wait_us`` after its first request."""

    def __init__(self, store: "Store | None", max_batch: int = 1024, max_wait_us: int = 200,
                 geometry: tuple[int, int] | None = None, device: int = 0):
        """store: the batcher's default store; or store=None and geometry=(N, S): a
        batcher for any whole store of that geometry (answer_on)."""
        import threading

        h = _vp()
        if store is None:
            N, S = geometry
            _check(lib().xpir_batcher_create_geometry(device, N, S, max_batch, max_wait_us, C.byref(h)))
            self.N, self.S = N, S
        else:
            _check(lib().xpir_batcher_create(store.h, max_batch, max_wait_us, C.byref(h)))
            self.N, self.S = store.N, store.S
        self.h, self.store = h, store
        # callers inside a C call; close() waits for them before destroying the handle
        self._cv, self._users = threading.Condition(), 0

    def close(self):
        cv = getattr(self, "_cv", None)
        if cv is None:
            return
        with cv:
            h, self.h = getattr(self, "h", None), None  # new calls fail cleanly
            cv.wait_for(lambda: self._users == 0)
        if h:
            _destroy(lambda: lib().xpir_batcher_destroy(h))

    __del__ = _quiet_del

    def _enter(self):
        with self._cv:
            if not self.h:
                raise XpirError(XPIR_ESTATE, "batcher is closed")
            self._users += 1
            return self.h

    def _leave(self):
        with self._cv:
            self._users -= 1
            if self._users == 0:
                self._cv.notify_all()

    def answer(self, q, mask_seed: bytes | None = None, q_bits: int | None = None, store: "Store | None" = None
               ) -> np.ndarray:
        """pir::answer(snapshot, q), or mask_answer(answer(..), mask_seed) (pir.cpp:29-39, 65-69);
        against `store` (same geometry) instead of the default store when given."""
        qa = _u8(q).reshape(-1)
        if qa.size < (self.N + 7) // 8:
            raise InvalidArgument(XPIR_EINVAL, "answer: query length mismatch")
        out = np.empty(self.S, np.uint8)
        ms = _p(_u8(mask_seed)) if mask_seed is not None else None
        qb = self.N if q_bits is None else q_bits
        h = self._enter()
        try:
            if store is None:
                _check(lib().xpir_batcher_answer(h, _p(qa), qb, ms, _p(out)))
            else:
                _check(lib().xpir_batcher_answer_on(h, store.h, _p(qa), qb, ms, _p(out)))
        finally:
            self._leave()
        return out

    def stats(self) -> dict:
        r, b, m = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().xpir_batcher_stats(self.h, C.byref(r), C.byref(b), C.byref(m)))
        return {"requests": r.value, "batches": b.value, "max_batch_seen": m.value}


def init_rows_dev(d_out, r0: int, r1: int, S: int, d_mask=None, device: int = 0, stream=None) -> None:
    _check(lib().xpir_init_rows_dev(device, _ptr(d_out), r0, r1, S, _ptr(d_mask), _stream(stream)))


def expand_queries_dev(d_seeds, B: int, byte_lo: int, nbytes: int, d_q, q_stride: int, device: int = 0,
                       stream=None) -> None:
    _check(lib().xpir_expand_queries_dev(device, _ptr(d_seeds), B, byte_lo, nbytes, _ptr(d_q), q_stride,
                                         _stream(stream)))


def mask_answer(ans: bytes, seed32: bytes) -> bytes:
    """pir::mask_answer (pir.cpp:65-69), pad generated and applied on device."""
    a = _u8(ans) if len(ans) else np.zeros(1, np.uint8)
    out = np.empty(max(len(ans), 1), np.uint8)
    _check(lib().xpir_mask_answer(_p(a), len(ans), _p(_u8(seed32)), _p(out)))
    return out[: len(ans)].tobytes()


def mask_dev(d_out, d_mask, B: int, S: int, device: int = 0, stream=None) -> None:
    _check(lib().xpir_mask_dev(device, _ptr(d_out), _ptr(d_mask), B, S, _stream(stream)))


def xor_reduce_dev(d_dst, src_ptrs: list[int], nbytes: int, device: int = 0, stream=None,
                   d_ptr_array=None) -> None:
    """d_dst ^= XOR of the source buffers (device pointers, peers allowed).
    `d_ptr_array` is a device buffer holding the pointer array (uint64 tensor)."""
    _check(lib().xpir_xor_reduce_dev(device, _ptr(d_dst), _ptr(d_ptr_array), len(src_ptrs), nbytes,
                                     _stream(stream)))


# ---------------------------------------------------------------------------
# primitives
# ---------------------------------------------------------------------------
def prng_expand(seed32: bytes, n: int) -> bytes:
    out = np.empty(max(n, 1), np.uint8)
    _check(lib().xpir_prng_expand(_p(_u8(seed32)), _p(out), n))
    return out[:n].tobytes()


def keystream_dev(key32: bytes, nonce: int, d_out, nbytes: int, byte_offset: int = 0, device: int = 0,
                  stream=None) -> None:
    _check(lib().xpir_keystream_dev(device, _p(_u8(key32)), nonce, byte_offset, _ptr(d_out), nbytes,
                                    _stream(stream)))


def keystream_rows_dev(key32: bytes, nonce0: int, rows: int, nbytes: int, d_out, row_stride: int,
                       device: int = 0, stream=None) -> None:
    _check(lib().xpir_keystream_rows_dev(device, _p(_u8(key32)), nonce0, rows, nbytes, _ptr(d_out),
                                         row_stride, _stream(stream)))


def prf_batch(key16: bytes, inputs, modulus: int) -> np.ndarray:
    x = np.ascontiguousarray(inputs, np.uint64)
    out = np.empty(max(len(x), 1), np.uint64)
    _check(lib().xpir_prf_batch(_p(_u8(key16)), _p(x, _u64p), len(x), modulus, _p(out, _u64p)))
    return out[: len(x)]


def prf_batch_dev(key16: bytes, d_inputs, n: int, modulus: int, d_out=None, d_out32=None, device: int = 0,
                  stream=None) -> None:
    _check(lib().xpir_prf_batch_dev(device, _p(_u8(key16)), _ptr(d_inputs), n, modulus, _ptr(d_out),
                                    _ptr(d_out32), _stream(stream)))


def write_betas_dev(k1: bytes, k2: bytes, d_keys, n: int, buckets: int, d_beta1, d_beta2, device: int = 0,
                    stream=None) -> None:
    """beta1/beta2 of a write batch (logproto.cpp:74-75), one kernel."""
    _check(lib().xpir_write_betas_dev(device, _p(_u8(k1)), _p(_u8(k2)), _ptr(d_keys), n, buckets, _ptr(d_beta1),
                                      _ptr(d_beta2), _stream(stream)))


def make_interest_batch(m_bits: int, h: int, id16: bytes, seqs) -> np.ndarray:
    s = np.ascontiguousarray(seqs, np.uint64)
    out = np.empty((max(len(s), 1), max(h, 1)), np.uint32)
    _check(lib().xpir_make_interest_batch(m_bits, h, _p(_u8(id16)), _p(s, _u64p), len(s), _p(out, _u32p)))
    return out[: len(s), :h]


def bloom_positions(item: bytes, h: int, m_bits: int) -> list[int]:
    it = _u8(item) if len(item) else np.zeros(1, np.uint8)
    out = np.empty(max(h, 1), np.uint32)
    _check(lib().xpir_bloom_positions(_p(it), len(item), h, m_bits, _p(out, _u32p)))
    return out[:h].tolist()


def blake2b(data: bytes, outlen: int = 32) -> bytes:
    d = _u8(data) if len(data) else np.zeros(1, np.uint8)
    out = np.empty(64, np.uint8)
    _check(lib().xpir_blake2b(_p(d), len(data), outlen, _p(out)))
    return out[:outlen].tobytes()


# ---------------------------------------------------------------------------
# cuckoo::Table
# ---------------------------------------------------------------------------
class _ShardMap(C.Structure):
    _fields_ = [("n", C.c_uint32), ("bucket_lo", C.c_uint32 * 9), ("data", _vp * 8)]


def shard_map(tables: list["Table"]) -> _ShardMap:
    """xpir_shard_map over payload shards (in bucket order) — their device pointers,
    or CUDA-IPC-mapped peer pointers in a multi-process deployment."""
    m = _ShardMap()
    m.n = len(tables)
    for g, t in enumerate(tables):
        m.bucket_lo[g] = t.lo
        m.data[g] = t.device_ptr()
    m.bucket_lo[len(tables)] = tables[-1].hi
    return m


class Table:
    def __init__(self, buckets: int, depth: int, capacity: int, item_size: int, seed32: bytes,
                 device: int = 0, lo: int = 0, hi: int | None = None):
        """cuckoo::Table; with lo/hi a payload shard holding buckets [lo, hi) (metadata whole)."""
        h = _vp()
        hi = buckets if hi is None else hi
        _check(lib().xpir_table_create_shard(device, buckets, depth, capacity, item_size, _p(_u8(seed32)), lo, hi,
                                             C.byref(h)))
        self.h, self.buckets, self.depth, self.item, self.device = h, buckets, depth, item_size, device
        self.lo, self.hi = lo, hi

    def close(self):
        if getattr(self, "h", None):
            _destroy(lambda: lib().xpir_table_destroy(self.h))
            self.h = None

    __del__ = _quiet_del

    def insert_batch(self, beta1, beta2, payload) -> np.ndarray:
        """Table::insert for each item in order; returns n x 4 InsertReport rows."""
        b1 = np.ascontiguousarray(beta1, np.uint32)
        b2 = np.ascontiguousarray(beta2, np.uint32)
        n = len(b1)
        pl = _u8(payload).reshape(-1)
        if pl.size != n * self.item:
            raise InvalidArgument(XPIR_EINVAL, "cuckoo: item size mismatch")
        rep = np.zeros((max(n, 1), 4), np.uint32)
        _check(lib().xpir_table_insert_batch(self.h, _p(b1, _u32p), _p(b2, _u32p), _p(pl), n,
                                             _p(rep, _u32p)))
        return rep[:n]

    def insert(self, beta1: int, beta2: int, data: bytes) -> dict:
        r = self.insert_batch([beta1], [beta2], _u8(data))[0]
        return {"stored": bool(r[0]), "dropped": bool(r[1]), "gc_evicted": bool(r[2]),
                "displacements": int(r[3])}

    def insert_batch_dev(self, d_b1, d_b2, d_payload, n: int, d_reports=None, stream=None) -> None:
        _check(lib().xpir_table_insert_batch_dev(self.h, _ptr(d_b1), _ptr(d_b2), _ptr(d_payload), n,
                                                 _ptr(d_reports), _stream(stream)))

    def insert_batch_async(self, d_b1, d_b2, d_payload, n: int, stream, d_reports=None, prefix_done=None) -> None:
        """The batch as stream work only (CUDA-graph capturable); then finish().
        prefix_done: a torch.cuda.Event recorded after the parallel-prefix kernel."""
        ev = None if prefix_done is None else prefix_done.cuda_event
        _check(lib().xpir_table_insert_batch_async(self.h, _ptr(d_b1), _ptr(d_b2), _ptr(d_payload), n,
                                                   _ptr(d_reports), _stream(stream), ev))

    def finish(self) -> int:
        """Completes an insert_batch_async batch; returns the inserts applied."""
        k = C.c_uint64()
        _check(lib().xpir_table_finish(self.h, C.byref(k)))
        return k.value

    # the three steps of a round on payload shards (see include/xpir.h)
    def insert_walk_dev(self, d_b1, d_b2, n: int, d_reports=None, stream=None) -> None:
        _check(lib().xpir_table_insert_walk_dev(self.h, _ptr(d_b1), _ptr(d_b2), n, _ptr(d_reports), _stream(stream)))

    def apply_gather_dev(self, smap: "_ShardMap | None" = None, stream=None) -> None:
        _check(lib().xpir_table_apply_gather_dev(self.h, C.byref(smap) if smap is not None else None,
                                                 _stream(stream)))

    def apply_scatter_dev(self, d_payload, stream=None) -> None:
        _check(lib().xpir_table_apply_scatter_dev(self.h, _ptr(d_payload), _stream(stream)))

    def reserve(self, max_batch: int) -> None:
        _check(lib().xpir_table_reserve(self.h, max_batch))

    def snapshot(self) -> np.ndarray:
        """Payload bytes (of buckets [lo, hi) for a shard)."""
        out = np.empty((self.hi - self.lo) * self.depth * self.item, np.uint8)
        _check(lib().xpir_table_snapshot(self.h, _p(out)))
        return out

    def seal(self, store: Store, epoch: int, stream=None) -> None:
        _check(lib().xpir_table_seal(self.h, store.h, epoch, _stream(stream)))

    def meta(self):
        n = self.buckets * self.depth
        used = np.empty(n, np.uint8)
        b1 = np.empty(n, np.uint32)
        b2 = np.empty(n, np.uint32)
        st = np.empty(n, np.uint64)
        _check(lib().xpir_table_meta(self.h, _p(used), _p(b1, _u32p), _p(b2, _u32p), _p(st, _u64p)))
        return used, b1, b2, st

    def counters(self):
        w, l, s = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().xpir_table_counters(self.h, C.byref(w), C.byref(l), C.byref(s)))
        return w.value, l.value, s.value

    def writes_applied(self) -> int:
        return self.counters()[0]

    def live_count(self) -> int:
        return self.counters()[1]

    def state_digest(self) -> bytes:
        out = np.empty(32, np.uint8)
        _check(lib().xpir_table_state_digest(self.h, _p(out)))
        return out.tobytes()

    def slot_used(self, bucket: int, slot: int) -> bool:
        return bool(_check(lib().xpir_table_slot_used(self.h, bucket, slot)))

    def device_ptr(self) -> int:
        return lib().xpir_table_device_data(self.h)


# ---------------------------------------------------------------------------
# notify::Window
# ---------------------------------------------------------------------------
class Window:
    def __init__(self, m_bits: int, h: int, w: int, device: int = 0):
        hd = _vp()
        _check(lib().xpir_window_create(device, m_bits, h, w, C.byref(hd)))
        self.h, self.m, self.nh, self.w, self.device = hd, m_bits, h, w, device

    def close(self):
        if getattr(self, "h", None):
            _destroy(lambda: lib().xpir_window_destroy(self.h))
            self.h = None

    __del__ = _quiet_del

    def absorb(self, positions) -> None:
        p = np.ascontiguousarray(positions, np.uint32).reshape(-1)
        _check(lib().xpir_window_absorb(self.h, _p(p, _u32p) if p.size else None, p.size))

    def absorb_dev(self, d_pos, n: int, stream=None) -> None:
        _check(lib().xpir_window_absorb_dev(self.h, _ptr(d_pos), n, _stream(stream)))

    def absorb_interest(self, id16: bytes, seqs) -> None:
        s = np.ascontiguousarray(seqs, np.uint64)
        _check(lib().xpir_window_absorb_interest(self.h, _p(_u8(id16)), _p(s, _u64p), len(s)))

    def absorb_interest_dev(self, id16: bytes, d_seqs, n: int, stream=None) -> None:
        _check(lib().xpir_window_absorb_interest_dev(self.h, _p(_u8(id16)), _ptr(d_seqs), n, _stream(stream)))

    def rotate(self) -> None:
        _check(lib().xpir_window_rotate(self.h))

    def info(self):
        n, b = C.c_uint64(), C.c_uint64()
        _check(lib().xpir_window_info(self.h, C.byref(n), C.byref(b)))
        return n.value, b.value

    def size(self) -> int:
        return self.info()[0]

    def base(self) -> int:
        return self.info()[1]

    def delta(self, i: int) -> np.ndarray:
        out = np.empty((self.m + 63) // 64, np.uint64)
        _check(lib().xpir_window_delta(self.h, i, _p(out, _u64p)))
        return out

    def digest(self, count: int | None = None) -> bytes:
        """Window::digest() / digest(count) (notify.cpp:90-107)."""
        out = np.empty(32, np.uint8)
        if count is None:
            _check(lib().xpir_window_digest(self.h, _p(out)))
        else:
            _check(lib().xpir_window_digest_n(self.h, count, _p(out)))
        return out.tobytes()

    def encode_delta(self, i: int) -> bytes:
        """notify::encode_delta(delta(i)) (notify.cpp:139-157), encoded on device."""
        return _window_encode(self.h, i)


def _window_encode(h, i: int) -> bytes:
    n = C.c_uint64()
    _check(lib().xpir_window_encode_delta(h, i, None, 0, C.byref(n)))
    out = np.empty(max(n.value, 1), np.uint8)
    _check(lib().xpir_window_encode_delta(h, i, _p(out), n.value, C.byref(n)))
    return out[:n.value].tobytes()


def decode_delta(buf: bytes, device: int = 0):
    """notify::decode_delta (notify.cpp:159-180) on device: (m_bits, words) or None
    for malformed input (the reference's std::nullopt)."""
    b = _u8(buf) if len(buf) else np.zeros(1, np.uint8)
    m = C.c_uint32()
    rc = lib().xpir_decode_delta(device, _p(b), len(buf), C.byref(m), None, 0)
    if rc == XPIR_EINVAL:
        return None
    _check(rc)
    w = np.zeros(max((m.value + 63) // 64, 1), np.uint64)
    rc = lib().xpir_decode_delta(device, _p(b), len(buf), C.byref(m), _p(w, _u64p), len(w))
    if rc == XPIR_EINVAL:
        return None
    _check(rc)
    return m.value, w[:(m.value + 63) // 64]


def encode_delta_dev(d_words, m_bits: int, d_out=None, cap: int = 0, device: int = 0, stream=None) -> int:
    """Device-buffer encode; returns the encoded length (d_out None: size query)."""
    n = C.c_uint64()
    _check(lib().xpir_encode_delta_dev(device, _ptr(d_words), m_bits, _ptr(d_out), cap, C.byref(n), _stream(stream)))
    return n.value


def encode_positions_dev(d_pos, h: int, n: int, d_fields, d_ok, cap: int = 64, device: int = 0, stream=None) -> None:
    """notify::encode_positions (notify.cpp:182-196) of n writes x h positions into
    cap-byte interest fields (wire.cpp:154); d_ok[i] = 0 where the reference throws."""
    _check(lib().xpir_encode_positions_dev(device, _ptr(d_pos), h, n, cap, _ptr(d_fields), _ptr(d_ok),
                                           _stream(stream)))


def decode_positions_dev(d_fields, n: int, d_pos, d_count, cap: int = 64, device: int = 0, stream=None) -> None:
    """notify::decode_positions (notify.cpp:198-214) of n cap-byte fields: d_count[i]
    = count (positions in d_pos[i, :count]) or 0xffffffff (std::nullopt)."""
    _check(lib().xpir_decode_positions_dev(device, _ptr(d_fields), cap, n, _ptr(d_pos), _ptr(d_count),
                                           _stream(stream)))


# ---------------------------------------------------------------------------
# server::ServerCore
# ---------------------------------------------------------------------------
class _BorrowedStore(Store):
    """A sealed store owned by a Server (valid while its epoch is in the ring)."""

    def __init__(self, handle, N: int, S: int, device: int, lo: int = 0, hi: int | None = None):  # noqa: D401
        self.h, self.N, self.S, self.lo, self.hi, self.device = handle, N, S, lo, N if hi is None else hi, device

    def close(self):
        self.h = None

    __del__ = _quiet_del


_BARRIER_FN = C.CFUNCTYPE(None, C.c_void_p)


def server_shard_map(servers: list["Server"], ptrs: list[int] | None = None) -> "_ShardMap":
    """Shard map over the ranks' payload arrays (ptrs: IPC-mapped pointers, in rank order)."""
    m = _ShardMap()
    m.n = len(servers)
    for g, sv in enumerate(servers):
        m.bucket_lo[g] = sv.lo
        m.data[g] = ptrs[g] if ptrs is not None else sv.payload_ptr()
    m.bucket_lo[len(servers)] = servers[-1].hi
    return m


class Server:
    """Device ServerCore: Table + Window + ring of sealed stores (server.cpp:28-91)."""

    def __init__(self, buckets: int, depth: int, capacity: int, item_size: int, seed32: bytes, m_bits: int, h: int,
                 window_deltas: int, rotate_writes: int, epoch_ring: int, device: int = 0, lo: int = 0,
                 hi: int | None = None):
        """With lo/hi: one rank of a bucket-range sharded deployment (payloads and
        sealed stores of buckets [lo, hi); walk, window and epochs replicated)."""
        hd = _vp()
        hi = buckets if hi is None else hi
        _check(lib().xpir_server_create_shard(device, buckets, depth, capacity, item_size, _p(_u8(seed32)), m_bits,
                                              h, window_deltas, rotate_writes, epoch_ring, lo, hi, C.byref(hd)))
        self.h, self.buckets, self.depth, self.item, self.device = hd, buckets, depth, item_size, device
        self.nh, self.lo, self.hi = h, lo, hi

    def payload_ptr(self) -> int:
        """Device pointer of this rank's payload shard (for the shard map / IPC)."""
        return lib().xpir_table_device_data(self._handles()[0])

    def close(self):
        if getattr(self, "h", None):
            _destroy(lambda: lib().xpir_server_destroy(self.h))
            self.h = None

    __del__ = _quiet_del

    def apply_round(self, beta1, beta2, payload, interest, seal_after: bool = False, smap=None, barrier=None):
        """ServerCore::apply_write for each write (+ seal). On a shard rank pass the
        shard map of all ranks' payload arrays and a barrier() over the ranks."""
        b1 = np.ascontiguousarray(beta1, np.uint32)
        b2 = np.ascontiguousarray(beta2, np.uint32)
        n = len(b1)
        pl = _u8(payload).reshape(-1)
        pos = np.ascontiguousarray(interest, np.uint32).reshape(n, -1) if n else np.zeros((0, self.nh), np.uint32)
        rep = np.zeros((max(n, 1), 4), np.uint32)
        ep = C.c_uint64()
        if smap is None:
            _check(lib().xpir_server_apply_round(self.h, _p(b1, _u32p), _p(b2, _u32p), _p(pl),
                                                 _p(pos, _u32p) if pos.size else None, pos.shape[1] if n else 0, n,
                                                 1 if seal_after else 0, _p(rep, _u32p), C.byref(ep)))
        else:
            cb = _BARRIER_FN(lambda _ctx: barrier())
            _check(lib().xpir_server_apply_round_sharded(
                self.h, _p(b1, _u32p), _p(b2, _u32p), _p(pl), _p(pos, _u32p) if pos.size else None,
                pos.shape[1] if n else 0, n, 1 if seal_after else 0, C.cast(C.pointer(smap), _vp),
                C.cast(cb, _vp), None, _p(rep, _u32p), C.byref(ep)))
        return rep[:n], ep.value

    def reserve(self, max_batch: int) -> None:
        """Server start-up: per-round scratch for rounds of up to max_batch writes and
        every sealed image of the ring allocated now (no allocation inside a round)."""
        _check(lib().xpir_server_reserve(self.h, max_batch))

    def seal(self) -> int:
        ep = C.c_uint64()
        _check(lib().xpir_server_seal(self.h, C.byref(ep)))
        return ep.value

    def snapshot(self, epoch: int = 0) -> Store:
        st = _vp()
        _check(lib().xpir_server_snapshot(self.h, epoch, C.byref(st)))
        return _BorrowedStore(st, self.buckets, self.depth * self.item, self.device, self.lo, self.hi)

    def snapshot_acquire(self, epoch: int = 0) -> tuple[Store, int]:
        """snapshot_at with a reader pin: the image is not reused until released."""
        st, ep = _vp(), C.c_uint64()
        _check(lib().xpir_server_snapshot_acquire(self.h, epoch, C.byref(st), C.byref(ep)))
        return _BorrowedStore(st, self.buckets, self.depth * self.item, self.device, self.lo, self.hi), ep.value

    def snapshot_release(self, store: Store) -> None:
        _check(lib().xpir_server_snapshot_release(self.h, store.h))

    def info(self):
        w, l, o = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().xpir_server_info(self.h, C.byref(w), C.byref(l), C.byref(o), None, None))
        return {"writes": w.value, "latest_epoch": l.value, "oldest_epoch": o.value}

    def _handles(self):
        t, w = _vp(), _vp()
        _check(lib().xpir_server_info(self.h, None, None, None, C.byref(t), C.byref(w)))
        return t, w

    def window_digest(self) -> bytes:
        out = np.empty(32, np.uint8)
        _check(lib().xpir_window_digest(self._handles()[1], _p(out)))
        return out.tobytes()

    def table_digest(self) -> bytes:
        out = np.empty(32, np.uint8)
        _check(lib().xpir_table_state_digest(self._handles()[0], _p(out)))
        return out.tobytes()

    def freeze(self) -> dict:
        """ServerCore::make_freeze (server.cpp:45-56): base, newest, digest and the
        device-encoded frozen deltas (notify::encode_delta)."""
        base, newest, count = C.c_uint64(), C.c_uint64(), C.c_uint64()
        dg = np.empty(32, np.uint8)
        _check(lib().xpir_server_freeze(self.h, C.byref(base), C.byref(newest), _p(dg), C.byref(count)))
        w = self._handles()[1]
        return {"base": base.value, "newest": newest.value, "digest": dg.tobytes(),
                "deltas": [_window_encode(w, k) for k in range(count.value)]}

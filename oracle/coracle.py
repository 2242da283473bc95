"""ctypes loader for the plain C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY (see oracle/ref.py header): used by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SRC_ADV = os.path.join(_HERE, "oracle_adv.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OST_BAD_MAGIC = 1
OST_BAD_VERSION = 2
OST_HEADER_MISMATCH = 4
OST_BAD_CODEC = 8
OST_NWORDS = 16
OST_RESIDUE = 32
OST_OVERFLOW = 64
OST_LENGTH = 128


def build(force: bool = False) -> str:
    """Compile oracle.c with plain gcc -O2 (no intrinsics, no -march)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC),
                                                                          os.path.getmtime(_SRC_ADV)):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-pthread",
                               _SRC, _SRC_ADV, "-o", _LIB + ".tmp"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_capacity.restype = ctypes.c_int
        L.oracle_capacity.argtypes = [ctypes.c_uint64]
        L.oracle_max_compressed_bytes.restype = ctypes.c_uint64
        L.oracle_max_compressed_bytes.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64]
        L.oracle_compress.restype = ctypes.c_int
        L.oracle_compress.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                      ctypes.c_void_p, ctypes.c_uint64,
                                      ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        L.oracle_decompress.restype = ctypes.c_int
        L.oracle_decompress.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                                        ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_uint32), ctypes.c_int]
        L.oracle_adv_capacity.restype = ctypes.c_int
        L.oracle_adv_capacity.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_adv_word_count.restype = ctypes.c_uint64
        L.oracle_adv_word_count.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_max_compressed_bytes_advanced.restype = ctypes.c_uint64
        L.oracle_max_compressed_bytes_advanced.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64]
        L.oracle_compress_advanced.restype = ctypes.c_int
        L.oracle_compress_advanced.argtypes = L.oracle_compress.argtypes
        L.oracle_decompress_advanced.restype = ctypes.c_int
        L.oracle_decompress_advanced.argtypes = L.oracle_decompress.argtypes
        _lib = L
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def capacity(B: int) -> int:
    return lib().oracle_capacity(B)


def compress(x: np.ndarray, block_len: int, threads: int | None = None) -> bytes:
    """x: contiguous uint16 or uint32 numpy array.  Returns the stream bytes."""
    x = np.ascontiguousarray(x)
    w = {np.dtype(np.uint8): 8, np.dtype(np.uint16): 16, np.dtype(np.uint32): 32}.get(x.dtype)
    if w is None:
        raise TypeError("uint8, uint16 or uint32 only")
    n = x.size
    cap = lib().oracle_max_compressed_bytes(n, w, block_len)
    out = np.empty(cap, dtype=np.uint8)
    nbytes = ctypes.c_uint64(0)
    rc = lib().oracle_compress(x.ctypes.data, n, w, block_len, out.ctypes.data, cap,
                               ctypes.byref(nbytes), threads or default_threads())
    if rc == 1:
        raise ValueError("EmptyInput")
    if rc != 0:
        raise RuntimeError("oracle_compress failed rc=%d" % rc)
    return out[: nbytes.value].tobytes()


def decompress(stream: bytes | np.ndarray, threads: int | None = None) -> Tuple[np.ndarray, int]:
    """Returns (values, status).  status == 0 means a valid stream."""
    buf = np.frombuffer(stream, dtype=np.uint8) if isinstance(stream, (bytes, bytearray)) else stream
    buf = np.ascontiguousarray(buf)
    if buf.size >= 32:
        n = int(buf[8:16].view(np.uint64)[0])
        w = int(buf[6])
    else:
        n, w = 0, 16
    cap = n if n < (1 << 36) else 0
    out = np.empty(max(cap, 1), dtype={8: np.uint8, 32: np.uint32}.get(w, np.uint16))
    n_out = ctypes.c_uint64(0)
    w_out = ctypes.c_int(0)
    st = ctypes.c_uint32(0)
    lib().oracle_decompress(buf.ctypes.data, buf.size, out.ctypes.data, cap,
                            ctypes.byref(n_out), ctypes.byref(w_out), ctypes.byref(st),
                            threads or default_threads())
    return out[: n_out.value], int(st.value)


# ------------------------------------------------------------------ advanced codec (oracle_adv.c)
def adv_capacity(B: int, Rp: int = 1) -> int:
    return lib().oracle_adv_capacity(B, Rp)


def adv_word_count(B: int, n: int) -> int:
    return lib().oracle_adv_word_count(B, n)


def compress_advanced(x: np.ndarray, block_len: int, threads: int | None = None) -> bytes:
    """The advanced (split-base, 32-bit word) stream of x (uint16/uint32)."""
    x = np.ascontiguousarray(x)
    w = {np.dtype(np.uint16): 16, np.dtype(np.uint32): 32}.get(x.dtype)
    if w is None:
        raise TypeError("uint16 or uint32 only")
    n = x.size
    cap = lib().oracle_max_compressed_bytes_advanced(n, w, block_len)
    out = np.empty(cap, dtype=np.uint8)
    nbytes = ctypes.c_uint64(0)
    rc = lib().oracle_compress_advanced(x.ctypes.data, n, w, block_len, out.ctypes.data, cap,
                                        ctypes.byref(nbytes), threads or default_threads())
    if rc == 1:
        raise ValueError("EmptyInput")
    if rc != 0:
        raise RuntimeError("oracle_compress_advanced failed rc=%d" % rc)
    return out[: nbytes.value].tobytes()


def decompress_advanced(stream: bytes | np.ndarray, threads: int | None = None) -> Tuple[np.ndarray, int]:
    """Returns (values, status) of an advanced stream; status 0 = valid."""
    buf = np.frombuffer(stream, dtype=np.uint8) if isinstance(stream, (bytes, bytearray)) else stream
    buf = np.ascontiguousarray(buf)
    if buf.size >= 32:
        n = int(buf[8:16].view(np.uint64)[0])
        w = int(buf[6])
    else:
        n, w = 0, 16
    cap = n if n < (1 << 36) else 0
    out = np.empty(max(cap, 1), dtype=np.uint32 if w == 32 else np.uint16)
    n_out = ctypes.c_uint64(0)
    w_out = ctypes.c_int(0)
    st = ctypes.c_uint32(0)
    lib().oracle_decompress_advanced(buf.ctypes.data, buf.size, out.ctypes.data, cap,
                                     ctypes.byref(n_out), ctypes.byref(w_out), ctypes.byref(st),
                                     threads or default_threads())
    return out[: n_out.value], int(st.value)

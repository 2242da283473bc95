"""ctypes binding of libpolycomp.so (include/poly.h) -- argument marshalling only.

Same names as the C ABI.  Torch tensors provide device memory and the current
stream (`torch.cuda.current_stream().cuda_stream`); every step of the codec runs
in the library's CUDA kernels.  There is no CPU fallback: if the library or a
CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("POLY_LIB") or os.path.join(_HERE, "libpolycomp.so")  # POLY_LIB: A/B variants

POLY_U8 = 8
POLY_U16 = 16
POLY_U32 = 32

POLY_OK = 0
STATUS_NAMES = {0: "POLY_OK", 1: "POLY_ERR_INVALID_ARG", 2: "POLY_ERR_EMPTY_INPUT", 3: "POLY_ERR_CAPACITY",
                4: "POLY_ERR_WORKSPACE", 5: "POLY_ERR_CUDA", 6: "POLY_ERR_CORRUPT"}

POLY_ST_BAD_MAGIC = 1
POLY_ST_BAD_VERSION = 2
POLY_ST_HEADER_MISMATCH = 4
POLY_ST_BAD_CODEC = 8
POLY_ST_NWORDS = 16
POLY_ST_RESIDUE = 32
POLY_ST_OVERFLOW = 64
POLY_ST_LENGTH = 128

EXPORTS = ["poly_version", "poly_status_string", "poly_init", "poly_max_compressed_bytes",
           "poly_workspace_bytes", "poly_compress", "poly_read_header", "poly_decompress",
           "poly_compress_host", "poly_decompress_host", "poly_launches_per_call", "poly_tables_ok",
           "poly_max_compressed_bytes_advanced", "poly_workspace_bytes_advanced", "poly_compress_advanced",
           "poly_decompress_advanced"]


class PolyError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__("%s failed: %s" % (what, STATUS_NAMES.get(code, str(code))))
        self.code = code


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libpolycomp.so (raises OSError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError("libpolycomp.so not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    u64, u32, vp, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int
    pu64 = ctypes.POINTER(ctypes.c_uint64)
    L.poly_version.restype = i32
    L.poly_version.argtypes = []
    L.poly_status_string.restype = ctypes.c_char_p
    L.poly_status_string.argtypes = [i32]
    L.poly_init.restype = i32
    L.poly_init.argtypes = [i32]
    L.poly_max_compressed_bytes.restype = u64
    L.poly_max_compressed_bytes.argtypes = [u64, i32, u64]
    L.poly_workspace_bytes.restype = u64
    L.poly_workspace_bytes.argtypes = [u64, i32, u64]
    L.poly_max_compressed_bytes_advanced.restype = u64
    L.poly_max_compressed_bytes_advanced.argtypes = [u64, i32, u64]
    L.poly_workspace_bytes_advanced.restype = u64
    L.poly_workspace_bytes_advanced.argtypes = [u64, i32, u64]
    L.poly_compress_advanced.restype = i32
    L.poly_compress_advanced.argtypes = [vp, u64, i32, u64, vp, u64, vp, vp, u64, vp]
    L.poly_decompress_advanced.restype = i32
    L.poly_decompress_advanced.argtypes = [vp, u64, i32, u64, u64, vp, vp, vp, u64, vp]
    L.poly_tables_ok.restype = i32
    L.poly_tables_ok.argtypes = []
    L.poly_launches_per_call.restype = i32
    L.poly_launches_per_call.argtypes = [u64, i32, u64, i32]
    L.poly_compress.restype = i32
    L.poly_compress.argtypes = [vp, u64, i32, u64, vp, u64, vp, vp, u64, vp]
    L.poly_read_header.restype = i32
    L.poly_read_header.argtypes = [vp, pu64, ctypes.POINTER(i32), pu64, pu64, pu64]
    L.poly_decompress.restype = i32
    L.poly_decompress.argtypes = [vp, u64, i32, u64, u64, vp, vp, vp, u64, vp]
    L.poly_compress_host.restype = i32
    L.poly_compress_host.argtypes = [vp, u64, i32, u64, vp, u64, pu64, vp, vp, u64, vp, u64, vp]
    L.poly_decompress_host.restype = i32
    L.poly_decompress_host.argtypes = [vp, u64, i32, u64, u64, vp, ctypes.POINTER(u32), vp, vp, vp, u64, vp]
    _lib = L
    return L


def _dt(x: torch.Tensor) -> int:
    if x.dtype == torch.uint8:
        return POLY_U8
    if x.dtype == torch.uint16:
        return POLY_U16
    if x.dtype == torch.uint32:
        return POLY_U32
    raise TypeError("values must be torch.uint8, torch.uint16 or torch.uint32, got %s" % x.dtype)


def _torch_dtype(dt: int) -> torch.dtype:
    return {POLY_U8: torch.uint8, POLY_U16: torch.uint16}.get(dt, torch.uint32)


def _need_cuda(*ts: torch.Tensor):
    for t in ts:
        if not t.is_cuda:
            raise ValueError("device tensors required (no CPU fallback)")
        if not t.is_contiguous():
            raise ValueError("contiguous tensors required")


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _check(rc: int, what: str):
    if rc != POLY_OK:
        raise PolyError(rc, what)


def poly_tables_ok() -> bool:
    """Host-only self-check of the decoder tables (include/poly.h)."""
    return bool(load_library().poly_tables_ok())


def poly_version() -> int:
    return load_library().poly_version()


def poly_init(device: Optional[int] = None) -> None:
    _check(load_library().poly_init(torch.cuda.current_device() if device is None else device), "poly_init")


def poly_max_compressed_bytes(n: int, dt: int, block_len: int) -> int:
    return load_library().poly_max_compressed_bytes(n, dt, block_len)


def poly_workspace_bytes(n: int, dt: int, block_len: int) -> int:
    return load_library().poly_workspace_bytes(n, dt, block_len)


def poly_launches_per_call(n: int, dt: int, block_len: int, decompress: bool) -> int:
    return load_library().poly_launches_per_call(n, dt, block_len, 1 if decompress else 0)


def alloc_workspace(n: int, dt: int, block_len: int, device=None) -> torch.Tensor:
    nb = max(16, poly_workspace_bytes(n, dt, block_len))
    return torch.empty((nb + 15) // 16 * 16, dtype=torch.uint8, device=device or "cuda")


def poly_compress(x: torch.Tensor, block_len: int, out: Optional[torch.Tensor] = None,
                  compressed_bytes: Optional[torch.Tensor] = None,
                  workspace: Optional[torch.Tensor] = None,
                  stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Compress the 1-D device tensor x (uint16/uint32).  Returns (out, nbytes):
    `out` a uint8 device buffer of poly_max_compressed_bytes bytes holding the
    stream at its start, `nbytes` a 1-element int64 device tensor with its size.
    Asynchronous on `stream` (default: current stream)."""
    _need_cuda(x)
    dt = _dt(x)
    n = x.numel()
    cap = poly_max_compressed_bytes(n, dt, block_len)
    if out is None:
        out = torch.empty(max(cap, 16), dtype=torch.uint8, device=x.device)
    if compressed_bytes is None:
        compressed_bytes = torch.empty(1, dtype=torch.int64, device=x.device)
    if workspace is None:
        workspace = alloc_workspace(n, dt, block_len, x.device)
    _need_cuda(out, compressed_bytes, workspace)
    rc = load_library().poly_compress(x.data_ptr(), n, dt, block_len, out.data_ptr(), out.numel(),
                                      compressed_bytes.data_ptr(), workspace.data_ptr(), workspace.numel(),
                                      _stream_ptr(stream))
    _check(rc, "poly_compress")
    return out, compressed_bytes


def poly_read_header(hdr: bytes) -> dict:
    if len(hdr) < 32:
        raise ValueError("need 32 header bytes")
    buf = ctypes.create_string_buffer(bytes(hdr[:32]), 32)
    n, bl, nb, pb = (ctypes.c_uint64() for _ in range(4))
    dt = ctypes.c_int()
    rc = load_library().poly_read_header(buf, ctypes.byref(n), ctypes.byref(dt), ctypes.byref(bl),
                                         ctypes.byref(nb), ctypes.byref(pb))
    _check(rc, "poly_read_header")
    return {"n": n.value, "dtype": dt.value, "block_len": bl.value, "n_blocks": nb.value,
            "payload_bytes": pb.value}


def poly_decompress(stream_buf: torch.Tensor, nbytes: int, dt: int, n: int, block_len: int,
                    out: Optional[torch.Tensor] = None, status: Optional[torch.Tensor] = None,
                    workspace: Optional[torch.Tensor] = None,
                    stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Decompress the first `nbytes` bytes of the uint8 device tensor.  Returns
    (values, status) where status is a 1-element int32 device tensor holding
    POLY_ST_* bits (0 = valid).  Asynchronous on `stream`."""
    _need_cuda(stream_buf)
    if out is None:
        out = torch.empty(n, dtype=_torch_dtype(dt), device=stream_buf.device)
    if status is None:
        status = torch.empty(1, dtype=torch.int32, device=stream_buf.device)
    if workspace is None:
        workspace = alloc_workspace(n, dt, block_len, stream_buf.device)
    _need_cuda(out, status, workspace)
    if nbytes > stream_buf.numel():
        raise ValueError("nbytes exceeds the buffer")
    rc = load_library().poly_decompress(stream_buf.data_ptr(), nbytes, dt, n, block_len, out.data_ptr(),
                                        status.data_ptr(), workspace.data_ptr(), workspace.numel(),
                                        _stream_ptr(stream))
    _check(rc, "poly_decompress")
    return out, status


def poly_compress_host(x_host: torch.Tensor, block_len: int, d_in: torch.Tensor, d_out: torch.Tensor,
                       workspace: torch.Tensor, h_out: torch.Tensor,
                       stream: Optional[torch.cuda.Stream] = None) -> int:
    """End-to-end compress of a (pinned) host tensor: H2D, kernels, D2H inside
    the call (synchronizes).  Returns the stream size; h_out[:size] holds it."""
    dt = _dt(x_host)
    n = x_host.numel()
    nb = ctypes.c_uint64(0)
    rc = load_library().poly_compress_host(x_host.data_ptr(), n, dt, block_len, h_out.data_ptr(), h_out.numel(),
                                           ctypes.byref(nb), d_in.data_ptr(), d_out.data_ptr(), d_out.numel(),
                                           workspace.data_ptr(), workspace.numel(), _stream_ptr(stream))
    _check(rc, "poly_compress_host")
    return nb.value


def poly_decompress_host(h_stream: torch.Tensor, nbytes: int, dt: int, n: int, block_len: int,
                         d_in: torch.Tensor, d_out: torch.Tensor, workspace: torch.Tensor,
                         h_out: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> int:
    """End-to-end decompress of a (pinned) host stream into host h_out.
    Returns the POLY_ST_* status bits."""
    st = ctypes.c_uint32(0)
    rc = load_library().poly_decompress_host(h_stream.data_ptr(), nbytes, dt, n, block_len, h_out.data_ptr(),
                                             ctypes.byref(st), d_in.data_ptr(), d_out.data_ptr(),
                                             workspace.data_ptr(), workspace.numel(), _stream_ptr(stream))
    _check(rc, "poly_decompress_host")
    return st.value


# ------------------------------------------------------------------ advanced codec
def poly_max_compressed_bytes_advanced(n: int, dt: int, block_len: int) -> int:
    return load_library().poly_max_compressed_bytes_advanced(n, dt, block_len)


def poly_workspace_bytes_advanced(n: int, dt: int, block_len: int) -> int:
    return load_library().poly_workspace_bytes_advanced(n, dt, block_len)


def poly_compress_advanced(x: torch.Tensor, block_len: int, out: Optional[torch.Tensor] = None,
                           compressed_bytes: Optional[torch.Tensor] = None,
                           workspace: Optional[torch.Tensor] = None,
                           stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """The advanced (split-base) codec of PAPER.md Sec. 3.2 on a uint16 device
    tensor; same conventions as poly_compress."""
    _need_cuda(x)
    dt = _dt(x)
    n = x.numel()
    cap = poly_max_compressed_bytes_advanced(n, dt, block_len)
    if out is None:
        out = torch.empty(max(cap, 16), dtype=torch.uint8, device=x.device)
    if compressed_bytes is None:
        compressed_bytes = torch.empty(1, dtype=torch.int64, device=x.device)
    if workspace is None:
        nb = max(16, poly_workspace_bytes_advanced(n, dt, block_len))
        workspace = torch.empty((nb + 15) // 16 * 16, dtype=torch.uint8, device=x.device)
    _need_cuda(out, compressed_bytes, workspace)
    rc = load_library().poly_compress_advanced(x.data_ptr(), n, dt, block_len, out.data_ptr(), out.numel(),
                                               compressed_bytes.data_ptr(), workspace.data_ptr(), workspace.numel(),
                                               _stream_ptr(stream))
    _check(rc, "poly_compress_advanced")
    return out, compressed_bytes


def poly_decompress_advanced(stream_buf: torch.Tensor, nbytes: int, dt: int, n: int, block_len: int,
                             out: Optional[torch.Tensor] = None, status: Optional[torch.Tensor] = None,
                             workspace: Optional[torch.Tensor] = None,
                             stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Inverse of poly_compress_advanced; same conventions as poly_decompress."""
    _need_cuda(stream_buf)
    if out is None:
        out = torch.empty(n, dtype=_torch_dtype(dt), device=stream_buf.device)
    if status is None:
        status = torch.empty(1, dtype=torch.int32, device=stream_buf.device)
    if workspace is None:
        nb = max(16, poly_workspace_bytes_advanced(n, dt, block_len))
        workspace = torch.empty((nb + 15) // 16 * 16, dtype=torch.uint8, device=stream_buf.device)
    _need_cuda(out, status, workspace)
    if nbytes > stream_buf.numel():
        raise ValueError("nbytes exceeds the buffer")
    rc = load_library().poly_decompress_advanced(stream_buf.data_ptr(), nbytes, dt, n, block_len, out.data_ptr(),
                                                 status.data_ptr(), workspace.data_ptr(), workspace.numel(),
                                                 _stream_ptr(stream))
    _check(rc, "poly_decompress_advanced")
    return out, status


# ------------------------------------------------------------------ convenience
def compress(x: torch.Tensor, block_len: int) -> torch.Tensor:
    """Compress and return exactly the stream bytes (uint8 device tensor);
    synchronizes to read the size."""
    out, nb = poly_compress(x, block_len)
    return out[: int(nb.item())]


def decompress(stream_buf: torch.Tensor) -> torch.Tensor:
    """Decompress a whole stream (uint8 device tensor); reads the 32-byte
    header to the host and raises if the device reports a status bit."""
    h = poly_read_header(stream_buf[:32].cpu().numpy().tobytes())
    out, st = poly_decompress(stream_buf, stream_buf.numel(), h["dtype"], h["n"], h["block_len"])
    s = int(st.item())
    if s:
        raise ValueError("corrupt stream, status bits 0x%x" % s)
    return out

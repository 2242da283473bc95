"""The C-ABI library loads without a GPU and exports every symbol include/poly.h
declares; host-only entry points (sizes, header parse, argument checks) work
on the CPU.  No compute call is made here."""
import ctypes
import os
import re
import struct

import pytest

from paper_1805_01844_b200 import _build, polycomp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return polycomp.load_library()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "poly.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(poly_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(polycomp.EXPORTS) == names


def test_version_and_status_strings(lib):
    assert polycomp.poly_version() >= 100
    assert lib.poly_status_string(0) == b"POLY_OK"
    assert lib.poly_status_string(2) == b"POLY_ERR_EMPTY_INPUT"


def test_max_compressed_bytes_closed_form(lib):
    # 32 + 16*n_blocks + 8*sum ceil(n_b / k_min); k_min = 4 (u16), 2 (u32)
    def bound(n, w, L):
        Le = n if L == 0 else L
        kmin = 4 if w == 16 else 2
        sizes = [min(Le, n - lo) for lo in range(0, n, Le)]
        return 32 + 16 * len(sizes) + 8 * sum(-(-s // kmin) for s in sizes)
    for n, w, L in [(1, 16, 0), (7, 16, 3), (1000, 32, 7), (1 << 20, 16, 0), (556500, 16, 30), (12345, 32, 1)]:
        assert polycomp.poly_max_compressed_bytes(n, w, L) == bound(n, w, L)
    assert polycomp.poly_max_compressed_bytes(0, 16, 0) == 0


def test_workspace_bytes_positive(lib):
    for n, w, L in [(1, 16, 0), (556500000, 16, 30), (1 << 28, 32, 65536), (1 << 31, 16, 4096), (1 << 20, 16, 0)]:
        assert polycomp.poly_workspace_bytes(n, w, L) >= 64
    assert polycomp.poly_workspace_bytes(0, 16, 0) == 0
    assert polycomp.poly_workspace_bytes(10, 12, 0) == 0  # dtype 12: not a width


def test_launches_per_call(lib):
    assert polycomp.poly_launches_per_call(556500000, 16, 30, False) == 1
    # cfg1 (one 2 MiB block): one launch each way (poly_*_large1)
    assert polycomp.poly_launches_per_call(1 << 20, 16, 0, False) == 1
    assert polycomp.poly_launches_per_call(1 << 20, 16, 0, True) == 1
    # many huge blocks keep the multi-kernel large-block path
    assert polycomp.poly_launches_per_call(1 << 32, 16, 1 << 22, False) == 3
    assert polycomp.poly_launches_per_call(1 << 32, 16, 1 << 22, True) == 2


def test_argument_errors_without_launch(lib):
    vp = ctypes.c_void_p
    # n == 0 -> EMPTY_INPUT before anything touches CUDA
    assert lib.poly_compress(vp(16), 0, 16, 0, vp(16), 1 << 20, vp(16), vp(16), 1 << 20, None) == 2
    # bad dtype, null pointers, block_size >= 2^32
    assert lib.poly_compress(vp(16), 10, 12, 0, vp(16), 1 << 20, vp(16), vp(16), 1 << 20, None) == 1
    assert lib.poly_compress(None, 10, 16, 0, vp(16), 1 << 20, vp(16), vp(16), 1 << 20, None) == 1
    assert lib.poly_compress(vp(16), 10, 16, 1 << 32, vp(16), 1 << 20, vp(16), vp(16), 1 << 20, None) == 1
    # misaligned output buffer
    assert lib.poly_compress(vp(16), 10, 16, 0, vp(17), 1 << 20, vp(16), vp(16), 1 << 20, None) == 1
    # capacity / workspace too small
    assert lib.poly_compress(vp(16), 1000, 16, 0, vp(16), 10, vp(16), vp(16), 1 << 20, None) == 3
    assert lib.poly_compress(vp(16), 1 << 20, 16, 30, vp(16), 1 << 24, vp(16), vp(16), 8, None) == 4
    assert lib.poly_decompress(vp(16), 100, 16, 0, 0, vp(16), vp(16), vp(16), 1 << 20, None) == 2
    assert lib.poly_decompress(vp(16), 100, 16, 10, 0, vp(16), vp(16), vp(16), 8, None) == 4


def test_read_header(lib):
    hdr = b"PLYC" + bytes([2, 0, 16, 0]) + struct.pack("<QIIQ", 7, 3, 3, 8)
    assert polycomp.poly_read_header(hdr) == {"n": 7, "dtype": 16, "block_len": 3, "n_blocks": 3,
                                              "payload_bytes": 8}
    with pytest.raises(polycomp.PolyError):
        polycomp.poly_read_header(b"XXXX" + hdr[4:])
    with pytest.raises(polycomp.PolyError):
        polycomp.poly_read_header(hdr[:4] + b"\x01" + hdr[5:])


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1805_01844_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), f


def test_decoder_tables_selfcheck(lib):
    """The host builds the per-base decoder constants with exact integers and
    checks the preconditions of DESIGN.md Sec. 5.3, including the compile-time
    T32MIN[K] switch points of the k-specialised decoders (poly_kword.cuh)."""
    assert polycomp.poly_tables_ok()


def test_t32min_table_matches_exact_integers():
    """Independent of the library: T32MIN[K] = min over non-power-of-two
    B <= 65536 with capacity K of t32(B) = max{t <= min(k, h) :
    2^32 B^k + B^k + 2^64 B^t <= 2^96}, recomputed with Python integers and
    compared with the constants compiled into poly_kword.cuh."""
    src = open(os.path.join(ROOT, "paper_1805_01844_b200", "csrc", "poly_kword.cuh")).read()
    body = src[src.index("constexpr int t32min_u16(int K)"):]
    body = body[:body.index(";")]
    table = {int(k): int(v) for k, v in re.findall(r"K == (\d+) \? (\d+)", body)}
    lo = {}
    for B in range(3, 65537):
        if B & (B - 1) == 0:
            continue
        k, p = 0, 1
        while p * B <= 1 << 64:
            p *= B
            k += 1
        h, q = 0, 1
        while q * B <= 1 << 32:
            q *= B
            h += 1
        t, bt = 0, 1
        for tt in range(1, min(k, h) + 1):
            bt *= B
            if (p << 32) + p + (bt << 64) <= 1 << 96:
                t = tt
            else:
                break
        lo[k] = min(lo.get(k, 99), t)
    for K, v in table.items():
        assert lo[K] == v, (K, lo[K], v)

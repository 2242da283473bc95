"""GPU robustness against corrupt streams and odd buffers, in every regime
(PIPE map 0 / map 1, large-block pipeline LARGE2, single huge block LARGE):

- hand-made corruptions set the expected POLY_ST_* bits (SPEC.md:83, 163,
  239, 311; include/poly.h);
- seeded byte flips: the device status is nonzero exactly when the oracle's
  decoder reports one, and when both accept the stream the values agree;
- guard bytes around every output buffer stay untouched (poly.h: no write
  leaves the given buffers), including for corrupt streams;
- value arrays at element (not 16-byte) alignment take the non-bulk paths and
  still give the oracle's bytes.
Marked gpu."""
import struct

import numpy as np
import pytest
import torch

from paper_1805_01844_b200 import polycomp as pc

pytestmark = pytest.mark.gpu

GUARD = 4096
PAT = 0xA5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    pc.poly_init()


def to_dev(x: np.ndarray) -> torch.Tensor:
    t = torch.from_numpy(x.view(np.int16 if x.dtype == np.uint16 else np.int32).copy())
    return t.view(torch.uint16 if x.dtype == np.uint16 else torch.uint32).cuda()


def regime_cases():
    """(name, values, L): one case per regime."""
    rng = np.random.default_rng(77)
    ped = rng.integers(240, 272, 30 * 4000).astype(np.uint16)
    ped[rng.integers(0, ped.size, 200)] = 2000
    m1 = rng.integers(1900, 2100, 1024 * 40).astype(np.uint16)
    m1[::997] = 4095
    lg2 = np.concatenate([rng.integers(0, int(2 ** rng.uniform(1, 20)), 20000) for _ in range(257)]).astype(np.uint32)
    lg2[-20000:] = 77  # a constant block
    big = np.clip(np.round(rng.normal(300, 5, 1 << 18)), 0, 65535).astype(np.uint16)
    return [("pipe_map0", ped, 30), ("pipe_map1", m1, 1024), ("large2", lg2, 20000), ("large", big, 0)]


def guarded(nbytes: int) -> torch.Tensor:
    buf = torch.full((nbytes + 2 * GUARD,), PAT, dtype=torch.uint8, device="cuda")
    return buf


def guards_ok(buf: torch.Tensor, nbytes: int) -> bool:
    g = torch.cat([buf[:GUARD], buf[GUARD + nbytes:]])
    return bool((g == PAT).all().item())


def gpu_decompress_guarded(stream: bytes, dt: int, n: int, L: int, nbytes=None):
    """Decompress `stream` (its own exact-size device copy) into a guarded
    output; returns (values, status, guards_intact)."""
    src = torch.from_numpy(np.frombuffer(stream, dtype=np.uint8).copy()).cuda()
    vb = dt // 8
    obuf = guarded(n * vb)
    out = obuf[GUARD:GUARD + n * vb].view(torch.int16 if dt == 16 else torch.int32)
    out = out.view(torch.uint16 if dt == 16 else torch.uint32)
    y, st = pc.poly_decompress(src, len(stream) if nbytes is None else nbytes, dt, n, L, out=out)
    torch.cuda.synchronize()
    return y, int(st.item()), guards_ok(obuf, n * vb)


@pytest.mark.parametrize("idx", range(4))
def test_corruption_status_bits_every_regime(oracle_lib, idx):
    name, x, L = regime_cases()[idx]
    n = x.size
    dt = 16 if x.dtype == np.uint16 else 32
    s = oracle_lib.compress(x, L)
    Le = L or n
    nbl = (n + Le - 1) // Le
    pay = 32 + 16 * nbl

    def st(buf, **kw):
        y, status, ok = gpu_decompress_guarded(buf, dt, kw.get("n", n), L, kw.get("nbytes"))
        assert ok, (name, "guard bytes overwritten")
        return status

    assert st(s) == 0
    assert st(b"XXXX" + s[4:]) & pc.POLY_ST_BAD_MAGIC
    assert st(s[:4] + b"\x01" + s[5:]) & pc.POLY_ST_BAD_VERSION
    assert st(s, n=n - 1) & pc.POLY_ST_HEADER_MISMATCH
    assert st(s, nbytes=len(s) - 8) & pc.POLY_ST_LENGTH
    assert st(s[:32] + struct.pack("<I", 9) + s[36:]) & pc.POLY_ST_BAD_CODEC
    # block 0's n_words off by one
    nw0 = struct.unpack("<I", s[44:48])[0]
    assert st(s[:44] + struct.pack("<I", nw0 + 1) + s[48:]) & (pc.POLY_ST_NWORDS | pc.POLY_ST_LENGTH)
    # v_min + B - 1 beyond the dtype
    assert st(s[:36] + struct.pack("<I", (1 << dt) - 1) + s[40:]) & pc.POLY_ST_OVERFLOW
    # a payload word >= B^k
    assert st(s[:pay] + struct.pack("<Q", (1 << 64) - 1) + s[pay + 8:]) & pc.POLY_ST_RESIDUE
    # payload_bytes forged so that 32 + 16 n_blocks + pb wraps 2^64 (truncated inside the headers)
    cut = s[:pay - 8]
    forged = cut[:24] + struct.pack("<Q", (1 << 64) - 8) + cut[32:]
    assert st(forged) & pc.POLY_ST_LENGTH


@pytest.mark.parametrize("idx", range(4))
def test_byte_flip_fuzz_matches_oracle(oracle_lib, idx):
    """Seeded single-byte corruptions anywhere in the stream: GPU status != 0
    iff the oracle's decoder reports a status; equal values when both accept;
    guard bytes intact in every case."""
    name, x, L = regime_cases()[idx]
    n = x.size
    dt = 16 if x.dtype == np.uint16 else 32
    s = bytearray(oracle_lib.compress(x, L))
    rng = np.random.default_rng(1000 + idx)
    for it in range(40):
        b = bytearray(s)
        # bias half of the flips into the headers (block headers are the fragile part)
        # (the 32-byte global header is left alone: the GPU checks it against
        # the call's arguments, the oracle only for consistency; it has its own
        # cases in test_corruption_status_bits_every_regime)
        hi = min(len(b), 32 + 16 * ((n + (L or n) - 1) // (L or n))) if it % 2 else len(b)
        pos = int(rng.integers(32, hi))
        b[pos] ^= int(rng.integers(1, 256))
        ref_y, ref_st = oracle_lib.decompress(bytes(b))
        y, st, ok = gpu_decompress_guarded(bytes(b), dt, n, L)
        assert ok, (name, it, pos, "guard bytes overwritten")
        assert (st != 0) == (ref_st != 0), (name, it, pos, st, ref_st)
        if st == 0:
            assert np.array_equal(y.cpu().view(torch.int16 if dt == 16 else torch.int32).numpy().view(x.dtype),
                                  ref_y), (name, it, pos)


@pytest.mark.parametrize("idx", range(4))
def test_compress_output_guards(oracle_lib, idx):
    """poly_compress writes only inside its output buffer (and the stream is
    the oracle's)."""
    name, x, L = regime_cases()[idx]
    n = x.size
    dt = 16 if x.dtype == np.uint16 else 32
    cap = pc.poly_max_compressed_bytes(n, dt, L)
    obuf = guarded(cap)
    out = obuf[GUARD:GUARD + cap]
    _, nb = pc.poly_compress(to_dev(x), L, out=out)
    torch.cuda.synchronize()
    nbytes = int(nb.item())
    assert guards_ok(obuf, cap), name
    assert out[:nbytes].cpu().numpy().tobytes() == oracle_lib.compress(x, L)


@pytest.mark.parametrize("idx", range(4))
@pytest.mark.parametrize("shift", [1, 3])
def test_unaligned_value_arrays(oracle_lib, idx, shift):
    """Values read from / written to arrays that start `shift` elements past a
    16-byte boundary (the non-bulk producer and store paths)."""
    name, x, L = regime_cases()[idx]
    n = x.size
    dt = 16 if x.dtype == np.uint16 else 32
    big = torch.zeros(n + 8, dtype=torch.int16 if dt == 16 else torch.int32, device="cuda")
    big[shift:shift + n] = to_dev(x).view(torch.int16 if dt == 16 else torch.int32)
    xv = big[shift:shift + n].view(torch.uint16 if dt == 16 else torch.uint32)
    assert xv.data_ptr() % 16 != 0
    out, nb = pc.poly_compress(xv, L)
    nbytes = int(nb.item())
    assert out[:nbytes].cpu().numpy().tobytes() == oracle_lib.compress(x, L), name
    ybig = torch.zeros(n + 8, dtype=torch.int16 if dt == 16 else torch.int32, device="cuda")
    yv = ybig[shift:shift + n].view(torch.uint16 if dt == 16 else torch.uint32)
    _, st = pc.poly_decompress(out, nbytes, dt, n, L, out=yv)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert torch.equal(yv, xv)
    assert int(ybig[:shift].abs().sum().item()) == 0 and int(ybig[shift + n:].abs().sum().item()) == 0


@pytest.mark.parametrize("L,n", [(77, 77 * 40 + 3), (1855, 1855 * 9 + 5), (1024, 1024 * 12 + 1), (4096, 4096 * 5 + 2049)])
def test_u16_every_output_offset(oracle_lib, L, n):
    """Two-pass decoder, u16: the output array starting 0..7 elements past a
    16-byte boundary (aligned TMA stores, 8-byte copy-out with and without the
    funnel shift, its head / tail values, units of fewer than 8 values), block
    lengths that are and are not a multiple of 16 bytes, a short last block;
    nothing is written outside the array."""
    rng = np.random.default_rng(L + n)
    x = rng.integers(900, 1230, n).astype(np.uint16)
    x[L:2 * L] = rng.integers(0, 16, L).astype(np.uint16)        # a power-of-two base
    x[2 * L:3 * L] = rng.integers(10, 51, L).astype(np.uint16)   # another capacity
    ref = oracle_lib.compress(x, L)
    xd = to_dev(x)
    out, nb = pc.poly_compress(xd, L)
    nbytes = int(nb.item())
    assert out[:nbytes].cpu().numpy().tobytes() == ref
    for shift in range(8):
        ybig = torch.zeros(n + 16, dtype=torch.int16, device="cuda")
        yv = ybig[shift:shift + n].view(torch.uint16)
        _, st = pc.poly_decompress(out, nbytes, 16, n, L, out=yv)
        torch.cuda.synchronize()
        assert int(st.item()) == 0, shift
        assert torch.equal(yv, xd), shift
        assert int(ybig[:shift].abs().sum().item()) == 0 and int(ybig[shift + n:].abs().sum().item()) == 0, shift

"""GPU parity of the advanced (split-base) codec (Sec. 3.2, 32-bit
words, u16 blocks) against the C oracle oracle/oracle_adv.c (itself pinned by
tests/test_oracle_advanced.py): the stream byte for byte, the values after the
round trip, status bits on corrupt streams.  Marked gpu."""
import struct

import numpy as np
import pytest
import torch

import workloads
from paper_1805_01844_b200 import polycomp as pc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    pc.poly_init()


def to_dev(x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(x.view(np.int16).copy()).view(torch.uint16).cuda()


def roundtrip(oracle_lib, x: np.ndarray, L: int):
    xd = to_dev(x)
    out, nb = pc.poly_compress_advanced(xd, L)
    nbytes = int(nb.item())
    s_gpu = out[:nbytes].cpu().numpy().tobytes()
    s_ref = oracle_lib.compress_advanced(x, L)
    assert len(s_gpu) == len(s_ref), (len(s_gpu), len(s_ref))
    if s_gpu != s_ref:
        a, b = np.frombuffer(s_gpu, np.uint8), np.frombuffer(s_ref, np.uint8)
        raise AssertionError("stream differs first at byte %d of %d" % (int(np.nonzero(a != b)[0][0]), a.size))
    y, st = pc.poly_decompress_advanced(out, nbytes, 16, x.size, L)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert torch.equal(y, xd)


EDGE = [([5, 7, 6, 4, 4, 4, 4], 3), ([42], 0), ([0, 65535], 0), ([65535] * 1000, 7),
        (list(range(16)) * 40, 64), (list(range(3)) * 333, 0), ([1, 2, 3], 10),
        (list(range(1000)) * 3, 154), ([111, 222, 333, 444, 555], 0)]


@pytest.mark.parametrize("idx", range(len(EDGE)))
def test_edge(oracle_lib, idx):
    v, L = EDGE[idx]
    roundtrip(oracle_lib, np.array(v, dtype=np.uint16), L)


def test_random_shapes(oracle_lib):
    rng = np.random.default_rng(11)
    for it in range(150):
        n = int(rng.integers(1, 6000))
        kind = it % 5
        if kind == 0:
            x = rng.integers(0, 65536, n)
        elif kind == 1:
            b = int(rng.integers(0, 60000))
            x = rng.integers(b, b + int(rng.integers(1, 3000)), n)
        elif kind == 2:
            x = np.full(n, int(rng.integers(0, 65536)))
        elif kind == 3:
            x = rng.integers(0, 1 << int(rng.integers(1, 17)), n)
        else:
            x = np.round(rng.normal(3000, 500, n)).clip(0, 65535)
            x[rng.integers(0, n, max(1, n // 400))] = rng.integers(2000, 45000)
        L = int(rng.choice([0, 1, 2, 3, 7, 30, 31, 64, 65, 154, 1000, 1024, 4096, 9000]))
        roundtrip(oracle_lib, x.astype(np.uint16), L)


@pytest.mark.parametrize("L", [30, 1024])
def test_every_u16_base(oracle_lib, L):
    """Every B in 2..65536 (one block each, 0 and B-1 present, a run of B-1
    at the end): every schedule of the table, thread-per-block (L = 30) and
    warp-per-block (L = 1024)."""
    rng = np.random.default_rng(L)
    Bs = np.arange(2, 65537, dtype=np.int64)
    if L == 1024:
        Bs = Bs[::7]  # every 7th base keeps the oracle run short at L = 1024
    d = rng.integers(0, 1 << 62, size=(Bs.size, L), dtype=np.int64) % Bs[:, None]
    d[:, 0] = 0
    d[:, 1] = Bs - 1
    d[:, -5:] = (Bs - 1)[:, None]
    off = rng.integers(0, 1 << 16, size=Bs.size) % (65537 - Bs)
    roundtrip(oracle_lib, (d + off[:, None]).astype(np.uint16).reshape(-1), L)


@pytest.mark.parametrize("cfg,scale", [(2, 1 / 50), (4, 1 / 32), (5, 1 / 128), (1, 1.0)])
def test_configs_scaled(oracle_lib, cfg, scale):
    x = workloads.generate(cfg, scale=scale, seed=2, device="cpu").numpy()
    roundtrip(oracle_lib, x, workloads.config(cfg, scale).block_len)


def test_corruption(oracle_lib):
    x = np.round(np.random.default_rng(1).normal(3000, 500, 1855 * 4)).clip(0, 65535).astype(np.uint16)
    L = 154
    s = oracle_lib.compress_advanced(x, L)
    n = x.size
    nbl = (n + L - 1) // L

    def st(buf, **kw):
        d = torch.from_numpy(np.frombuffer(buf, dtype=np.uint8).copy()).cuda()
        _, status = pc.poly_decompress_advanced(d, kw.get("nbytes", len(buf)), 16, kw.get("n", n), L)
        return int(status.item())

    assert st(s) == 0
    assert st(b"XXXX" + s[4:]) & pc.POLY_ST_BAD_MAGIC
    assert st(s[:5] + b"\x00" + s[6:]) & pc.POLY_ST_HEADER_MISMATCH      # layout 0 = basic stream
    assert st(s, n=n - 1) & pc.POLY_ST_HEADER_MISMATCH
    assert st(s, nbytes=len(s) - 4) & pc.POLY_ST_LENGTH
    assert st(s[:32] + struct.pack("<I", 2) + s[36:]) & pc.POLY_ST_BAD_CODEC
    nw0 = struct.unpack("<I", s[44:48])[0]
    assert st(s[:44] + struct.pack("<I", nw0 + 1) + s[48:]) & (pc.POLY_ST_NWORDS | pc.POLY_ST_LENGTH)
    pay = 32 + 16 * nbl
    assert st(s[:pay] + struct.pack("<I", 0xFFFFFFFF) + s[pay + 4:]) & pc.POLY_ST_RESIDUE
    # fuzz: nonzero status iff the oracle rejects; equal values when both accept
    rng = np.random.default_rng(5)
    for it in range(40):
        b = bytearray(s)
        pos = int(rng.integers(32, len(b)))
        b[pos] ^= int(rng.integers(1, 256))
        ref_y, ref_st = oracle_lib.decompress_advanced(bytes(b))
        d = torch.from_numpy(np.frombuffer(bytes(b), dtype=np.uint8).copy()).cuda()
        y, status = pc.poly_decompress_advanced(d, len(b), 16, n, L)
        g = int(status.item())
        assert (g != 0) == (ref_st != 0), (it, pos, g, ref_st)
        if g == 0:
            assert np.array_equal(y.cpu().view(torch.int16).numpy().view(np.uint16), ref_y)


@pytest.mark.parametrize("cfg", [2, 4, 5])
def test_full_size_configs(oracle_lib, cfg):
    """BASELINE.json full sizes (u16 configs): the advanced stream equals the
    oracle's byte for byte and the round trip returns the values."""
    c = workloads.config(cfg, 1.0)
    x = workloads.generate(cfg, scale=1.0, seed=0, device="cuda")
    out, nb = pc.poly_compress_advanced(x, c.block_len)
    nbytes = int(nb.item())
    ref = oracle_lib.compress_advanced(x.cpu().numpy(), c.block_len)
    assert nbytes == len(ref)
    ref_dev = torch.from_numpy(np.frombuffer(ref, dtype=np.uint8).copy()).cuda()
    assert torch.equal(out[:nbytes], ref_dev)
    del ref_dev
    y, st = pc.poly_decompress_advanced(out, nbytes, 16, c.n, c.block_len)
    assert int(st.item()) == 0
    assert torch.equal(y, x)

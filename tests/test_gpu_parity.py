"""GPU parity: the CUDA path through the C ABI against the C oracle, bit for
bit (compressed stream) and value for value (decompressed array), on seeded
inputs.  Marked gpu: run on a B200 with `pytest -m gpu`."""
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
    t = torch.from_numpy(x.view(np.int16 if x.dtype == np.uint16 else np.int32).copy())
    return t.view(torch.uint16 if x.dtype == np.uint16 else torch.uint32).cuda()


def gpu_roundtrip(x_dev: torch.Tensor, L: int):
    out, nb = pc.poly_compress(x_dev, L)
    nbytes = int(nb.item())
    stream = out[:nbytes]
    dt = 16 if x_dev.dtype == torch.uint16 else 32
    y, st = pc.poly_decompress(out, nbytes, dt, x_dev.numel(), L)
    torch.cuda.synchronize()
    return stream.cpu().numpy().tobytes(), y, int(st.item())


def check_case(oracle_lib, x: np.ndarray, L: int):
    x_dev = to_dev(x)
    s_gpu, y, st = gpu_roundtrip(x_dev, L)
    s_ref = oracle_lib.compress(x, L)
    assert len(s_gpu) == len(s_ref), (len(s_gpu), len(s_ref))
    if s_gpu != s_ref:
        a = np.frombuffer(s_gpu, np.uint8)
        b = np.frombuffer(s_ref, np.uint8)
        i = int(np.nonzero(a != b)[0][0])
        raise AssertionError("stream differs first at byte %d of %d" % (i, len(a)))
    assert st == 0
    assert torch.equal(y, x_dev)


# ------------------------------------------------------------------ small cases
EDGE = [
    # (values, dtype, L)
    ([5, 7, 6, 4, 4, 4, 4], np.uint16, 3),
    ([42], np.uint16, 0),
    ([42], np.uint32, 1),
    ([0, 65535], np.uint16, 0),              # B = 2^16 -> pow2, k = 4
    ([0, 0xFFFFFFFF], np.uint32, 0),         # B = 2^32 -> pow2, k = 2
    ([0xFFFFFFFF] * 9, np.uint32, 4),        # constant at the top
    ([65535] * 1000, np.uint16, 7),          # all 65535
    (list(range(16)) * 40, np.uint16, 64),   # B = 16
    (list(range(256)) * 9, np.uint16, 300),  # B = 256
    (list(range(3)) * 333, np.uint16, 0),    # B = 3, k = 40
    ([1, 2, 3], np.uint16, 10),              # L > n
]


@pytest.mark.parametrize("idx", range(len(EDGE)))
def test_edge_matrix(oracle_lib, idx):
    v, dt, L = EDGE[idx]
    check_case(oracle_lib, np.array(v, dtype=dt), L)


def test_random_small_shapes(oracle_lib):
    rng = np.random.default_rng(123)
    for it in range(300):
        w = 16 if it % 3 else 32
        n = int(rng.integers(1, 5000))
        kind = it % 6
        hi = 1 << w
        if kind == 0:
            base = int(rng.integers(0, hi - 100000)) if w == 32 else int(rng.integers(0, hi - 200))
            x = rng.integers(base, base + int(rng.integers(1, 200)), size=n, dtype=np.uint64)
        elif kind == 1:
            x = rng.integers(0, hi, size=n, dtype=np.uint64)
        elif kind == 2:
            j = int(rng.integers(1, w + 1))
            x = rng.integers(0, 1 << j, size=n, dtype=np.uint64)
        elif kind == 3:
            x = np.full(n, int(rng.integers(0, hi)), dtype=np.uint64)
        elif kind == 4:
            x = rng.integers(1000, 1040, size=n, dtype=np.uint64)
            x[rng.integers(0, n, size=max(1, n // 500))] = hi - 1
        else:
            b = int(rng.integers(2, 1 << min(w, 22)))
            x = rng.integers(0, b, size=n, dtype=np.uint64)
        L = int(rng.choice([0, 1, 2, 3, 5, 7, 30, 31, 64, 100, 154, 1000, 1024, 4096, 5000, 9000, 20000]))
        check_case(oracle_lib, x.astype(np.uint16 if w == 16 else np.uint32), L)


def worst_case_blocks(Bs, L, rng):
    """One block of L values per base B (u16), each holding the words that
    stress the decoder: 0 and B-1 (so the block's base is
    exactly B), a whole word of digits B-1 (the largest full word B^k - 1), and
    a top word of digits B-1 (B^m - 1, the largest partial word); the rest is
    uniform.  Returns the u16 array."""
    Bs = np.asarray(Bs, dtype=np.int64)
    d = rng.integers(0, 1 << 62, size=(Bs.size, L), dtype=np.int64) % Bs[:, None]
    for r, B in enumerate(Bs.tolist()):
        k = capacity_u64(B)
        m = L % k or k
        d[r, L - m:] = B - 1                # top word: every digit B - 1
        if L >= 2 * k:
            d[r, k:2 * k] = B - 1           # word 1: every digit B - 1
        d[r, 0] = 0
        d[r, 1] = B - 1
    off = rng.integers(0, 1 << 16, size=Bs.size) % (65537 - Bs)
    return (d + off[:, None]).astype(np.uint16).reshape(-1)


def capacity_u64(B: int) -> int:
    k, p = 0, 1
    while p * B <= 1 << 64:
        p *= B
        k += 1
    return k


def test_every_u16_base_worst_words_map0(oracle_lib):
    """Every B in 2..65536, one 64-value block each (map 0: one lane per
    block), with the worst-case words of every base."""
    rng = np.random.default_rng(5)
    x = worst_case_blocks(np.arange(2, 65537), 64, rng)
    check_case(oracle_lib, x, 64)


def test_every_u16_base_worst_words_map1(oracle_lib):
    """Every B in 2..65536, one 1024-value block each: the map-1 decoders
    (k-specialised unrolled group codecs for the u16 capacities, with their
    compile-time T32MIN switch points) see every base with its worst words."""
    rng = np.random.default_rng(6)
    x = worst_case_blocks(np.arange(2, 65537), 1024, rng)
    check_case(oracle_lib, x, 1024)


def test_u16_bases_worst_words_large_blocks(oracle_lib):
    """The large-block pipeline (blocks > 32 KiB, >= 256 blocks): every k
    threshold base and its neighbours, powers of two and a spread of others."""
    rng = np.random.default_rng(7)
    th = [2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 16, 17, 19, 20, 23, 24, 30, 31, 40, 41, 56, 57, 84, 85,
          138, 139, 256, 257, 565, 566, 1625, 1626, 7131, 7132, 65535, 65536]
    Bs = sorted(set(th + [int(b) for b in np.unique(np.geomspace(2, 65536, 260).astype(np.int64))]))
    x = worst_case_blocks(Bs, 17000, rng)
    check_case(oracle_lib, x, 17000)


def test_large_bases_u32(oracle_lib):
    rng = np.random.default_rng(9)
    Bs = [65537, 65539, 100003, 1 << 20, (1 << 20) + 7, 2642245, 2642246, 3 * 10 ** 6, (1 << 31) + 11,
          (1 << 32) - 1, 1 << 32]
    blocks = []
    for B in Bs:
        blk = rng.integers(0, B, size=77, dtype=np.uint64)
        k = capacity_u64(B)
        blk[0], blk[1] = 0, B - 1
        blk[k:2 * k] = B - 1                # a full word of digits B - 1
        blk[77 - (77 % k or k):] = B - 1    # the top word: digits B - 1
        blocks.append(blk)
    x = np.concatenate(blocks).astype(np.uint32)
    check_case(oracle_lib, x, 77)
    check_case(oracle_lib, x, 0)


# ------------------------------------------------------------------ large blocks
# Blocks > 32 KiB with >= 256 blocks take the two-sweep large-block pipeline
# (poly_large.cuh); ragged tails and every base class are covered.
def _large_case(rng, w, L, nblocks, tail):
    hi = 1 << w
    blocks = []
    for i in range(nblocks):
        kind = i % 6
        n = L if i < nblocks - 1 or tail == 0 else tail
        if kind == 0:      # log-uniform base
            b = int(2 ** rng.uniform(1, w)) if w == 16 else int(2 ** rng.uniform(1, 32))
            b = max(2, min(b, hi))
            v = rng.integers(0, b, size=n, dtype=np.uint64)
        elif kind == 1:    # constant
            v = np.full(n, int(rng.integers(0, hi)), dtype=np.uint64)
        elif kind == 2:    # power-of-two base at the top of the range
            j = int(rng.integers(1, w + 1))
            v = rng.integers(0, 1 << j, size=n, dtype=np.uint64) + (hi - (1 << j))
        elif kind == 3:    # full range
            v = rng.integers(0, hi, size=n, dtype=np.uint64)
        elif kind == 4:    # narrow noise
            v = rng.integers(1000, 1013, size=n, dtype=np.uint64)
        else:              # two values far apart
            v = np.where(rng.random(n) < 0.5, 7, hi - 3).astype(np.uint64)
        blocks.append(v)
    return np.concatenate(blocks).astype(np.uint16 if w == 16 else np.uint32)


@pytest.mark.parametrize("w,L,nblocks,tail", [(16, 20000, 260, 1234), (32, 10000, 258, 77), (16, 40000, 256, 0)])
def test_large_blocks(oracle_lib, w, L, nblocks, tail):
    rng = np.random.default_rng(w * 1000 + nblocks)
    x = _large_case(rng, w, L, nblocks, tail)
    check_case(oracle_lib, x, L)


# ------------------------------------------------------------------ configs
SMALL = {1: 1.0, 2: 1 / 100, 3: 1 / 16, 4: 1 / 128, 5: 1 / 128, 6: 1 / 100}  # cfg6: cfg2 time-major  # cfg3 at 1/16: 256 blocks (large-block pipeline)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6])
def test_config_scaled(oracle_lib, cfg):
    c = workloads.config(cfg, SMALL[cfg])
    x = workloads.generate(cfg, scale=SMALL[cfg], seed=1, device="cuda")
    s_gpu, y, st = gpu_roundtrip(x, c.block_len)
    s_ref = oracle_lib.compress(x.cpu().numpy(), c.block_len)
    assert s_gpu == s_ref
    assert st == 0 and torch.equal(y, x)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6])
def test_config_full_size(oracle_lib, cfg):
    """BASELINE.json full sizes, in the launch configuration bench.py times:
    the whole stream equals the oracle's, and decompress(compress(x)) == x."""
    c = workloads.config(cfg, 1.0)
    x = workloads.generate(cfg, scale=1.0, seed=0, device="cuda")
    out, nb = pc.poly_compress(x, c.block_len)
    nbytes = int(nb.item())
    s_ref = oracle_lib.compress(x.cpu().numpy(), c.block_len)
    assert nbytes == len(s_ref)
    ref_dev = torch.from_numpy(np.frombuffer(s_ref, dtype=np.uint8).copy()).cuda()
    assert torch.equal(out[:nbytes], ref_dev)
    del ref_dev
    y, st = pc.poly_decompress(out, nbytes, 16 if c.dtype == torch.uint16 else 32, c.n, c.block_len)
    assert int(st.item()) == 0
    assert torch.equal(y, x)


# ------------------------------------------------------------------ corruption
def _stream(x, L):
    x_dev = to_dev(np.array(x, dtype=np.uint16))
    return pc.compress(x_dev, L).cpu().numpy().tobytes()


def _status(buf: bytes, n, L, dt=16, nbytes=None):
    d = torch.from_numpy(np.frombuffer(buf + bytes(64), dtype=np.uint8).copy()).cuda()
    _, st = pc.poly_decompress(d, len(buf) if nbytes is None else nbytes, dt, n, L)
    return int(st.item())


@pytest.mark.parametrize("large", [False, True])
def test_corruption_status_bits(large):
    x = [5, 7, 6, 4, 4, 4, 4] if not large else list(np.arange(20000) % 37)
    L = 3 if not large else 10000
    n = len(x)
    s = _stream(x, L)
    nbl = (n + L - 1) // L
    assert _status(s, n, L) == 0
    assert _status(b"XXXX" + s[4:], n, L) & pc.POLY_ST_BAD_MAGIC
    assert _status(s[:4] + b"\x01" + s[5:], n, L) & pc.POLY_ST_BAD_VERSION
    assert _status(s, n + 1, L) & pc.POLY_ST_HEADER_MISMATCH
    assert _status(s, n, L, dt=32) & pc.POLY_ST_HEADER_MISMATCH
    assert _status(s, n, L, nbytes=len(s) - 8) & pc.POLY_ST_LENGTH
    assert _status(s[:32] + struct.pack("<I", 9) + s[36:], n, L) & pc.POLY_ST_BAD_CODEC
    assert _status(s[:44] + struct.pack("<I", 5) + s[48:], n, L) & (pc.POLY_ST_NWORDS | pc.POLY_ST_LENGTH)
    assert _status(s[:36] + struct.pack("<I", 65535) + s[40:], n, L) & pc.POLY_ST_OVERFLOW
    pay = 32 + 16 * nbl
    bad_word = struct.pack("<Q", (1 << 64) - 1)
    assert _status(s[:pay] + bad_word + s[pay + 8:], n, L) & pc.POLY_ST_RESIDUE


@pytest.mark.parametrize("L,lo,hi", [(1024, 1800, 2130), (4096, 0, 40), (1000, 0, 16), (77, 100, 350)])
def test_short_top_word_bound(L, lo, hi):
    """A block's short top word holds m < k digits: the decoder must accept
    B^m - 1 and report RESIDUE for B^m (< B^k, so only the digits past the
    block's end tell), in the two-pass decoder's group codec (odd and even k,
    a power-of-two base) and in its word-by-word path."""
    rng = np.random.default_rng(L + hi)
    nbl = 5
    x = rng.integers(lo, hi, L * nbl).astype(np.uint16)
    x[::L] = lo
    x[1::L] = hi - 1
    B = hi - lo
    k = 1
    while B ** (k + 1) <= 1 << 64:
        k += 1
    m = L % k
    assert m != 0
    nw = (L + k - 1) // k
    s = _stream(x, L)
    pay = 32 + 16 * nbl
    for blk in (0, nbl - 1):
        top = pay + 8 * (nw * blk + nw - 1)
        ok_word = struct.pack("<Q", B ** m - 1)
        bad_word = struct.pack("<Q", B ** m)
        assert _status(s[:top] + ok_word + s[top + 8:], x.size, L) == 0
        assert _status(s[:top] + bad_word + s[top + 8:], x.size, L) & pc.POLY_ST_RESIDUE


def test_empty_input_rejected():
    x = torch.empty(0, dtype=torch.uint16, device="cuda")
    with pytest.raises(pc.PolyError) as e:
        pc.poly_compress(x, 0)
    assert e.value.code == 2


def _pipe_cases():
    rng = np.random.default_rng(2024)
    ped = rng.integers(240, 272, 30 * 6000).astype(np.uint16)            # map 0, pedestal-like
    ped[rng.integers(0, ped.size, 300)] = 2000                            # outlier blocks (more words)
    return [
        (ped, 30),
        (rng.integers(1900, 2100, 1024 * 64).astype(np.uint16), 1024),    # map 1, one warp per block
        (rng.integers(900, 1100, 4096 * 40).astype(np.uint16), 4096),     # map 1, warp groups per block
        (rng.integers(0, 70000, 7 * 20011).astype(np.uint32), 7),         # map 0, u32, ragged tail
        (rng.integers(0, 5000, 10000 * 260 + 77).astype(np.uint32), 10000),  # large-block regime
        (rng.integers(0, 1 << 31, 32 * 30011).astype(np.uint32), 32),      # map 0 u32, shared word ring
    ]


def test_pipeline_shapes(oracle_lib):
    """The pipeline cases of both maps, u16 and u32, ragged tails, the shared
    compress word ring and the large-block pipeline, each against the oracle."""
    for x, L in _pipe_cases():
        check_case(oracle_lib, x, L)


def test_repeat_determinism(oracle_lib):
    """Dynamically claimed groups, per-warp word rings and the prefix server
    race by design; repeated launches must give the oracle's bytes every time."""
    cases = _pipe_cases()
    refs = [oracle_lib.compress(x, L) for x, L in cases]
    for _ in range(12):
        for (x, L), ref in zip(cases, refs):
            s_gpu, y, st = gpu_roundtrip(to_dev(x), L)
            assert s_gpu == ref
            assert st == 0
            assert np.array_equal(y.cpu().view(torch.int16 if x.dtype == np.uint16 else torch.int32)
                                  .numpy().view(x.dtype), x)


def test_host_calls(oracle_lib):
    """poly_compress_host / poly_decompress_host (pinned host buffers): the
    chunked, copy-overlapped compress path (>= 16 tiles) and the serial one
    (few tiles, u32, large blocks) give the oracle's bytes, and the round trip
    returns the values."""
    rng = np.random.default_rng(99)
    for x, L in [(rng.integers(240, 275, 30 * 30000).astype(np.uint16), 30),
                 (rng.integers(1900, 2100, 1024 * 700 + 5).astype(np.uint16), 1024),
                 (rng.integers(240, 275, 30 * 300).astype(np.uint16), 30),
                 (rng.integers(0, 70000, 40000 * 300 + 3).astype(np.uint32), 40000)]:
        dt = 16 if x.dtype == np.uint16 else 32
        n = x.size
        h_in = torch.from_numpy(x.view(np.int16 if dt == 16 else np.int32).copy()).view(
            torch.uint16 if dt == 16 else torch.uint32).pin_memory()
        cap = pc.poly_max_compressed_bytes(n, dt, L)
        d_in = torch.empty(max(cap, n * dt // 8), dtype=torch.uint8, device="cuda")
        d_out = torch.empty(max(cap, n * dt // 8), dtype=torch.uint8, device="cuda")
        ws = pc.alloc_workspace(n, dt, L, d_in.device)
        h_stream = torch.empty(cap, dtype=torch.uint8).pin_memory()
        nb = pc.poly_compress_host(h_in, L, d_in, d_out, ws, h_stream)
        assert h_stream[:nb].numpy().tobytes() == oracle_lib.compress(x, L)
        h_out = torch.empty(n, dtype=torch.uint16 if dt == 16 else torch.uint32).pin_memory()
        st = pc.poly_decompress_host(h_stream, nb, dt, n, L, d_in, d_out, ws, h_out)
        assert st == 0
        assert np.array_equal(h_out.view(torch.int16 if dt == 16 else torch.int32).numpy().view(x.dtype), x)


@pytest.mark.parametrize("cfg", [1, 2])
def test_graph_capture_replay(oracle_lib, cfg):
    """The device calls are stream-ordered with no host synchronisation: one
    compress + decompress captured in a CUDA graph and replayed on new values
    (copied into the captured input) gives the oracle's bytes each time."""
    c = workloads.config(cfg, SMALL[cfg])
    L = c.block_len
    x = workloads.generate(cfg, scale=SMALL[cfg], seed=3, device="cuda")
    dt = 16 if x.dtype == torch.uint16 else 32
    out, nb = pc.poly_compress(x, L)
    cap_bytes = out.numel()
    nbytes0 = int(nb.item())
    ws = pc.alloc_workspace(x.numel(), dt, L, x.device)
    y = torch.empty_like(x)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty(cap_bytes, dtype=torch.uint8, device="cuda")

    def step():
        pc.poly_compress(x, L, out=out, compressed_bytes=nb, workspace=ws)
        pc.poly_decompress(out, nbytes0, dt, x.numel(), L, out=y, status=st, workspace=ws)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for seed in (3, 4, 5):
        # a permutation of the seed-3 values keeps the stream length the graph baked in
        xs = workloads.generate(cfg, scale=SMALL[cfg], seed=3, device="cuda")
        if seed != 3 and L:
            nbk = xs.numel() // L
            perm = torch.randperm(nbk, generator=torch.Generator().manual_seed(seed)).cuda()
            xi = xs.view(torch.int16 if dt == 16 else torch.int32)
            xi[: nbk * L] = xi[: nbk * L].view(nbk, L)[perm].reshape(-1)
        x.copy_(xs)
        st.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert int(nb.item()) == nbytes0
        ref = oracle_lib.compress(xs.cpu().numpy(), L)
        assert out[:nbytes0].cpu().numpy().tobytes() == ref
        assert int(st.item()) == 0 and torch.equal(y, xs)


# ------------------------------------------------------------------ in-place compress (poly_cmp3.cuh)
# Blocks whose byte size is a multiple of 16 (128 B < block <= 32 KiB) are
# packed in place by one warp per block; small blocks are claimed several at a
# time (32 / CB lanes per block in the min / max).  Both instantiations, every
# capacity's threshold bases with their worst words, u32 with B = 2^32, ragged
# last blocks.
def _threshold_bases():
    Bs = set()
    for k in range(4, 65):
        # around the first B whose capacity drops below k (coarse steps above 64)
        b = 2
        while b <= 65536 and capacity_u64(b) >= k:
            b += max(1, b // 64)
        for c in (b - 2, b - 1, b, b + 1):
            if 2 <= c <= 65536:
                Bs.add(c)
    return sorted(Bs | {2, 3, 4, 5, 16, 17, 255, 256, 257, 4096, 7131, 7132, 7133, 65535, 65536})


@pytest.mark.parametrize("L", [4096, 1024, 128, 8000])
def test_inplace_compress_u16_threshold_bases(oracle_lib, L):
    rng = np.random.default_rng(L)
    Bs = _threshold_bases()
    x = worst_case_blocks(Bs, L, rng)
    check_case(oracle_lib, x, L)
    check_case(oracle_lib, x[: x.size - L // 3], L)  # a ragged last block


def test_inplace_compress_u32(oracle_lib):
    rng = np.random.default_rng(31)
    for L in (64, 1024, 4096):
        blocks = []
        for B in [2, 3, 65536, 65537, 2642245, 2642246, (1 << 31) + 11, (1 << 32) - 1, 1 << 32]:
            blk = rng.integers(0, B, size=L, dtype=np.uint64)
            k = capacity_u64(B)
            blk[0], blk[1] = 0, B - 1
            blk[L - (L % k or k):] = B - 1
            blocks.append(blk)
        blocks.append(np.full(L, 7, dtype=np.uint64))  # constant block
        x = np.concatenate(blocks * 3).astype(np.uint32)
        check_case(oracle_lib, x, L)
        check_case(oracle_lib, x[:-5], L)

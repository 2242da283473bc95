"""SPEC.md:30's third width, u8 values (B <= 256, k >= 8), through every
regime of the CUDA codec (pipeline map 0 / map 1, large-block pipeline, few
huge blocks), byte for byte against the C oracle.  Marked gpu."""
import numpy as np
import pytest
import torch

from paper_1805_01844_b200 import polycomp as pc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    pc.poly_init()


def check(oracle_lib, x: np.ndarray, L: int, shift: int = 0):
    n = x.size
    big = torch.zeros(n + 16, dtype=torch.uint8, device="cuda")
    big[shift:shift + n] = torch.from_numpy(x).cuda()
    xd = big[shift:shift + n]
    out, nb = pc.poly_compress(xd, L)
    nbytes = int(nb.item())
    s_ref = oracle_lib.compress(x, L)
    s_gpu = out[:nbytes].cpu().numpy().tobytes()
    assert len(s_gpu) == len(s_ref)
    assert s_gpu == s_ref
    y, st = pc.poly_decompress(out, nbytes, 8, n, L)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert torch.equal(y, xd)


EDGE = [([5, 7, 6, 4, 4, 4, 4], 3), ([42], 0), ([0, 255], 0), ([255] * 1000, 7), (list(range(16)) * 40, 64),
        (list(range(256)) * 9, 300), ([1, 2, 3], 10)]


@pytest.mark.parametrize("idx", range(len(EDGE)))
def test_edge(oracle_lib, idx):
    v, L = EDGE[idx]
    check(oracle_lib, np.array(v, dtype=np.uint8), L)


@pytest.mark.parametrize("L", [64, 1024, 40000, 0])
def test_every_base_every_regime(oracle_lib, L):
    """Every B in 2..256 with worst-case words (0 and B-1, a run of B-1 at
    the end), blocks of 64 (map 0), 1024 (map 1), 40,000 (> 32 KiB: the
    large-block pipeline, >= 256 blocks) and one block of the whole array."""
    rng = np.random.default_rng(L + 1)
    Bs = np.arange(2, 257, dtype=np.int64)
    Lb = L if L else 5000
    reps = 2 if L == 40000 else 1
    Bs = np.tile(Bs, reps)[: max(256, Bs.size)]
    d = rng.integers(0, 1 << 40, size=(Bs.size, Lb), dtype=np.int64) % Bs[:, None]
    d[:, 0] = 0
    d[:, 1] = Bs - 1
    d[:, -70:] = (Bs - 1)[:, None]
    off = rng.integers(0, 256, size=Bs.size) % (257 - Bs)
    x = (d + off[:, None]).astype(np.uint8).reshape(-1)
    check(oracle_lib, x, L)


def test_random_shapes_and_unaligned(oracle_lib):
    rng = np.random.default_rng(3)
    for it in range(60):
        n = int(rng.integers(1, 9000))
        x = rng.integers(0, 256, n) if it % 3 == 0 else rng.integers(100, 100 + int(rng.integers(1, 60)), n)
        L = int(rng.choice([0, 1, 2, 7, 30, 128, 129, 1000, 4096, 40000]))
        check(oracle_lib, x.astype(np.uint8), L, shift=int(it % 5))

"""The plain C oracle (oracle/oracle.c) against the pinned Python oracle
(oracle/ref.py) on random and config-shaped inputs.  CPU only."""
import struct

import numpy as np
import pytest

import workloads
from oracle import ref


def _rand_case(rng):
    w = int(rng.choice([16, 32]))
    n = int(rng.integers(1, 400))
    kind = int(rng.integers(0, 5))
    hi = (1 << w)
    if kind == 0:      # narrow band
        base = int(rng.integers(0, hi - 64))
        x = rng.integers(base, base + int(rng.integers(1, 64)), size=n, dtype=np.uint64)
    elif kind == 1:    # full range
        x = rng.integers(0, hi, size=n, dtype=np.uint64)
    elif kind == 2:    # constant runs
        x = np.full(n, int(rng.integers(0, hi)), dtype=np.uint64)
    elif kind == 3:    # powers of two ranges
        j = int(rng.integers(1, w + 1))
        x = rng.integers(0, 1 << j, size=n, dtype=np.uint64)
    else:              # one outlier
        x = rng.integers(1000, 1010, size=n, dtype=np.uint64)
        x[int(rng.integers(0, n))] = hi - 1
    L = int(rng.choice([0, 1, 2, 3, 7, 30, 64, 154, n, n + 5]))
    return x.astype(np.uint16 if w == 16 else np.uint32), w, L


def test_c_oracle_matches_python_oracle_random(oracle_lib):
    rng = np.random.default_rng(11)
    for _ in range(400):
        x, w, L = _rand_case(rng)
        s_c = oracle_lib.compress(x, L, threads=int(rng.integers(1, 5)))
        s_py = ref.compress_blocked(x.tolist(), w, L)
        assert s_c == s_py
        y, st = oracle_lib.decompress(s_c, threads=3)
        assert st == 0 and np.array_equal(y, x)


def test_c_oracle_capacity_matches(oracle_lib):
    for B in list(range(2, 70000, 7)) + [65535, 65536, 65537, 2642245, 2642246, (1 << 32) - 1, 1 << 32]:
        assert oracle_lib.capacity(B) == ref.capacity(B)


@pytest.mark.parametrize("cfg,scale", [(1, 1 / 64), (2, 1 / 2000), (3, 1 / 1024), (4, 1 / 8192), (5, 1 / 32768)])
def test_c_oracle_matches_python_on_config_samples(oracle_lib, cfg, scale):
    c = workloads.config(cfg, scale)
    x = workloads.generate(cfg, scale=scale, seed=3).numpy()
    if cfg == 3:   # python is slow on u32 64 Ki blocks: take 2 blocks
        x = x[: 2 * 65536]
    s_c = oracle_lib.compress(x, c.block_len)
    assert s_c == ref.compress_blocked(x.tolist(), 32 if cfg == 3 else 16, c.block_len)


def test_c_oracle_corruption_status(oracle_lib):
    s = oracle_lib.compress(np.array([5, 7, 6, 4, 4, 4, 4], dtype=np.uint16), 3)
    assert oracle_lib.decompress(b"XXXX" + s[4:])[1] & oracle_lib.OST_BAD_MAGIC
    assert oracle_lib.decompress(s[:4] + b"\x01" + s[5:])[1] & oracle_lib.OST_BAD_VERSION
    assert oracle_lib.decompress(s[:-8])[1] & oracle_lib.OST_LENGTH
    assert oracle_lib.decompress(s[:32] + struct.pack("<I", 9) + s[36:])[1] & oracle_lib.OST_BAD_CODEC
    assert oracle_lib.decompress(s[:-8] + struct.pack("<Q", 3 ** 40))[1] & oracle_lib.OST_RESIDUE
    assert oracle_lib.decompress(s[:36] + struct.pack("<I", 65535) + s[40:])[1] & oracle_lib.OST_OVERFLOW


def test_u8_width_c_equals_python_and_brute_force(oracle_lib):
    """SPEC.md:30's third width: u8 values (B <= 256, so k >= 8).  The C
    oracle equals the Python oracle on random u8 vectors, round-trips, and its
    size is the closed form 32 + 16 n_blocks + 8 sum ceil(n_b / k_b)."""
    import itertools
    import numpy as np
    from oracle import ref
    rng = np.random.default_rng(8)
    for t in range(150):
        n = int(rng.integers(1, 3000))
        L = int(rng.choice([0, 1, 3, 8, 30, 64, 100, 1855]))
        kind = t % 4
        if kind == 0:
            x = rng.integers(0, 256, n)
        elif kind == 1:
            x = rng.integers(100, 100 + int(rng.integers(1, 100)), n)
        elif kind == 2:
            x = np.full(n, int(rng.integers(0, 256)))
        else:
            x = np.where(rng.random(n) < 0.5, 0, 255)
        x = x.astype(np.uint8)
        s_c = oracle_lib.compress(x, L)
        assert s_c == ref.compress_blocked(x.tolist(), 8, L)
        y, st = oracle_lib.decompress(s_c)
        assert st == 0 and np.array_equal(y, x)
        Le = L or n
        words = 0
        for lo in range(0, n, Le):
            blk = x[lo:lo + Le].astype(np.int64)
            B = int(blk.max() - blk.min() + 1)
            if B > 1:
                k = 0
                while B ** (k + 1) <= 1 << 64:
                    k += 1
                words += -(-blk.size // k)
        assert len(s_c) == 32 + 16 * (-(-n // Le)) + 8 * words
    for n in range(1, 4):   # brute force over tiny u8 vectors
        for v in itertools.product([0, 1, 2, 127, 255], repeat=n):
            x = np.array(v, dtype=np.uint8)
            for L in range(0, n + 2):
                s = oracle_lib.compress(x, L)
                assert s == ref.compress_blocked(list(v), 8, L)
                assert np.array_equal(oracle_lib.decompress(s)[0], x)

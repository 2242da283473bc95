"""Pins for the Python oracle (oracle/ref.py) against what the paper, SPEC's
worked examples and plain mathematics fix -- never against the oracle's own
formula retyped.  CPU only."""
import itertools
import json
import math
import os
import random
import struct

import numpy as np
import pytest

from oracle import ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
LIT32 = (1 << 32) - 1   # Eq. 1 literal limit, SPEC's 32-bit mode


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def ndigits(x, B):
    """Number of base-B digits of x > 0, by repeated integer division."""
    c = 0
    while x:
        x //= B
        c += 1
    return c


# ------------------------------------------------------------------ derive_base
def test_derive_base_spec_examples():
    for ex in load("spec_examples.json")["derive_base"]:
        assert ref.derive_base(ex["values"]) == (ex["v_min"], ex["v_max"], ex["B"]), ex["cite"]


def test_derive_base_matches_numpy():
    rng = np.random.default_rng(1)
    for _ in range(200):
        x = rng.integers(0, 1 << 32, size=rng.integers(1, 50), dtype=np.uint64)
        v_min, v_max, B = ref.derive_base(list(x))
        assert v_min == int(np.min(x)) and v_max == int(np.max(x)) and B == int(np.ptp(x)) + 1


def test_derive_base_empty():
    with pytest.raises(ref.EmptyInput):
        ref.derive_base([])


# ------------------------------------------------------------------ capacity
def test_capacity_spec_examples_literal_mode():
    for ex in load("spec_examples.json")["capacity_literal32"]:
        if ex["B"] >= 2:
            assert ref.capacity(ex["B"], limit=LIT32) == ex["p"], ex["cite"]
    # SPEC.md:66 second example, carry form: 250 * 1000^2 <= 2^32-1 < 250 * 1000^3
    assert 250 * 1000 ** 2 <= LIT32 < 250 * 1000 ** 3


def test_capacity_every_base_le_65536_by_digit_count():
    """k = (number of base-B digits of 2^64) - 1: floor(log_B 2^64), obtained by
    repeated division -- an independent route to max{k : B^k <= 2^64}."""
    for B in range(2, 65537):
        assert ref.capacity(B) == ndigits(1 << 64, B) - 1


def test_capacity_large_bases_random_and_thresholds():
    rng = random.Random(7)
    bases = [rng.randrange(65537, (1 << 32) + 1) for _ in range(20000)]
    # Appendix A thresholds, each checked +-1; arithmetic facts:
    assert 2642245 ** 3 <= 1 << 64 < 2642246 ** 3
    assert 7131 ** 5 <= 1 << 64 < 7132 ** 5
    assert 1625 ** 6 <= 1 << 64 < 1626 ** 6
    bases += [65536, 65537, 2642244, 2642245, 2642246, 2642247, (1 << 32) - 1, 1 << 32]
    for B in bases:
        assert ref.capacity(B) == ndigits(1 << 64, B) - 1


def test_capacity_powers_of_two_closed_form():
    # B = 2^j: B^k <= 2^64 <=> j*k <= 64, so k = floor(64 / j).
    for j in range(1, 33):
        assert ref.capacity(1 << j) == 64 // j


def test_capacity_float_log_away_from_exact_powers():
    # Eq. 1 with logs (d = 2^64) agrees wherever the real ratio
    # is not within 1e-9 of an integer (there float rounding could flip it).
    for B in list(range(2, 5000)) + [65535, 326, 1000, 2265]:
        r = 64 * math.log(2) / math.log(B)
        if abs(r - round(r)) > 1e-9:
            assert ref.capacity(B) == math.floor(r)


def test_capacity_appendix_a_table():
    # (k, first B, last B) under B^k <= 2^64.
    table = [(64, 2, 2), (40, 3, 3), (32, 4, 4), (27, 5, 5), (24, 6, 6), (22, 7, 7), (21, 8, 8),
             (20, 9, 9), (19, 10, 10), (18, 11, 11), (17, 12, 13), (16, 14, 16), (15, 17, 19),
             (14, 20, 23), (13, 24, 30), (12, 31, 40), (11, 41, 56), (10, 57, 84), (9, 85, 138),
             (8, 139, 256), (7, 257, 565), (6, 566, 1625), (5, 1626, 7131), (4, 7132, 65536),
             (3, 65537, 2642245), (2, 2642246, 1 << 32)]
    for k, lo, hi in table:
        assert ref.capacity(lo) == k and ref.capacity(hi) == k
        assert lo ** k <= 1 << 64 and hi ** k <= 1 << 64 and (hi + 1) ** k > 1 << 64


def test_capacity_literal_rule_differs_only_at_full_powers():
    # R2: the literal 2^64 - 1 rule differs exactly when B^k == 2^64.
    diffs = [B for B in range(2, 65537) if ref.capacity(B) != ref.capacity(B, (1 << 64) - 1)]
    assert diffs == [2, 4, 16, 256, 65536]


# ------------------------------------------------------------------ pack_basic
def test_pack_spec_examples_literal_mode():
    for ex in load("spec_examples.json")["pack_basic_literal32"]:
        k = ref.capacity(ex["B"], limit=LIT32)
        assert ref.pack_basic(ex["values"], ex["v_min"], ex["B"], k) == ex["words"], ex["cite"]


def test_pack_byte_base_is_byte_packing():
    # B = 256, k = 8: each word is the 8 digit bytes read little-endian.
    rng = np.random.default_rng(2)
    d = rng.integers(0, 256, size=43, dtype=np.uint8)
    words = ref.pack_basic(list(d), 0, 256, ref.capacity(256))
    padded = bytes(d) + bytes(-len(d) % 8)
    assert words == list(struct.unpack("<%dQ" % (len(padded) // 8), padded))


def test_pack_hex_base_is_nibble_packing():
    d = list(range(16)) * 2
    assert ref.pack_basic(d, 0, 16, ref.capacity(16)) == [0xFEDCBA9876543210] * 2


def test_pack_binary_base_is_bit_packing():
    rng = np.random.default_rng(3)
    bits = list(rng.integers(0, 2, size=150))
    words = ref.pack_basic(bits, 0, 2, ref.capacity(2))
    for j, w in enumerate(words):
        chunk = bits[64 * j: 64 * j + 64]
        assert w == int("".join(str(b) for b in reversed(chunk)), 2)


def test_pack_decimal_base_is_digit_concatenation():
    d = list(range(10)) + list(range(9))      # 19 digits, k(10) = 19
    assert ref.capacity(10) == 19
    assert ref.pack_basic(d, 0, 10, 19) == [8765432109876543210]


def test_pack_small_bases_match_python_int_parser():
    rng = np.random.default_rng(4)
    digits = "0123456789abcdefghijklmnopqrstuvwxyz"
    for B in range(2, 37):
        k = ref.capacity(B)
        n = int(rng.integers(1, 3 * k))
        d = [int(v) for v in rng.integers(0, B, size=n)]
        words = ref.pack_basic([v + 1000 for v in d], 1000, B, k)
        for j, w in enumerate(words):
            chunk = d[j * k:(j + 1) * k]
            assert w == int("".join(digits[v] for v in reversed(chunk)), B)


def test_pack_word_bound_and_count():
    rng = np.random.default_rng(5)
    for B in [3, 7, 17, 255, 326, 1000, 2265, 65535, 65537, 2642245, 2642246, (1 << 32) - 1, 1 << 32]:
        k = ref.capacity(B)
        d = [int(v) for v in rng.integers(0, B, size=3 * k + 1, dtype=np.uint64)]
        d[0] = B - 1
        d[1:k] = [B - 1] * (k - 1)    # first word all max digits = B^k - 1
        words = ref.pack_basic(d, 0, B, k)
        assert len(words) == math.ceil(len(d) / k)
        assert words[0] == B ** k - 1 and all(0 <= w < 1 << 64 for w in words)


# ------------------------------------------------------------------ unpack_basic
def test_unpack_spec_examples_literal_mode():
    for ex in load("spec_examples.json")["unpack_basic_literal32"]:
        k = ref.capacity(ex["B"], limit=LIT32)
        assert ref.unpack_basic(ex["words"], ex["v_min"], ex["B"], k, ex["n"]) == ex["values"], ex["cite"]


def test_unpack_matches_numpy_base_repr():
    rng = np.random.default_rng(6)
    for B in range(2, 37):
        k = ref.capacity(B)
        for _ in range(5):
            w = int(rng.integers(0, 1 << 62)) % (B ** k)
            got = ref.unpack_basic([w], 7, B, k, k)
            rep = np.base_repr(w, B).rjust(k, "0")
            assert got == [7 + int(c, 36) for c in reversed(rep)]


def test_unpack_rejects_residue_and_count():
    with pytest.raises(ref.CorruptStream):
        ref.unpack_basic([3 ** 5], 0, 3, 40, 5)      # digit beyond m = 5
    with pytest.raises(ref.CorruptStream):
        ref.unpack_basic([1, 2], 0, 3, 40, 5)        # 2 words for 5 values


# ------------------------------------------------------------------ blocked + stream
def closed_form_size(x, L):
    n = len(x)
    Le = n if L == 0 else L
    total = 32
    for lo in range(0, n, Le):
        blk = x[lo:lo + Le]
        B = max(blk) - min(blk) + 1
        total += 16
        if B > 1:
            k = ndigits(1 << 64, B) - 1
            total += 8 * (-(-len(blk) // k))
    return total


def test_format_golden_stream():
    g = load("format_example.json")
    s = ref.compress_blocked(g["values"], g["width_bits"], g["block_len"])
    assert s.hex() == g["stream_hex"]
    assert ref.decompress_blocked(s) == (g["values"], 16)


def test_brute_force_tiny_arrays_roundtrip_and_size():
    alphabet = [0, 1, 2, 15, 16, 255, 256, 65534, 65535]
    cases = []
    for n in range(1, 4):
        cases += [list(t) for t in itertools.product(alphabet, repeat=n)]
    for n in range(1, 7):
        cases += [list(t) for t in itertools.product(range(4), repeat=n)]
    for x in cases:
        for L in range(0, len(x) + 2):
            s = ref.compress_blocked(x, 16, L)
            assert len(s) == closed_form_size(x, L)
            assert ref.decompress_blocked(s) == (x, 16)


def test_u32_extremes_roundtrip():
    for x in ([0, 0xFFFFFFFF], [0xFFFFFFFF] * 5, [0, 0xFFFFFFFF, 7, 3], [1 << 31, (1 << 31) + 2642244]):
        for L in (0, 1, 2, 3):
            s = ref.compress_blocked(x, 32, L)
            assert len(s) == closed_form_size(x, L)
            assert ref.decompress_blocked(s) == (x, 32)


def test_block_independence_and_monotone_degradation():
    rng = np.random.default_rng(8)
    x = [int(v) for v in rng.integers(100, 140, size=64)]
    s1 = ref.compress_blocked(x, 16, 16)
    y = list(x)
    y[20] = 65535                       # outlier in block 1
    s2 = ref.compress_blocked(y, 16, 16)
    h1 = [s1[32 + 16 * b: 48 + 16 * b] for b in range(4)]
    h2 = [s2[32 + 16 * b: 48 + 16 * b] for b in range(4)]
    assert h1[0] == h2[0] and h1[2] == h2[2] and h1[3] == h2[3] and h1[1] != h2[1]
    # each block's record equals the single-block stream's record
    for b in range(4):
        sb = ref.compress_blocked(x[16 * b:16 * b + 16], 16, 0)
        assert sb[32:48] == h1[b]


def test_empty_input():
    with pytest.raises(ref.EmptyInput):
        ref.compress_blocked([], 16, 0)


@pytest.mark.parametrize("mutate,exc", [
    (lambda s: b"XXXX" + s[4:], ref.NotAContainer),
    (lambda s: s[:4] + b"\x01" + s[5:], ref.UnsupportedVersion),
    (lambda s: s[:-8], ref.CorruptStream),                                   # truncated
    (lambda s: s[:32] + struct.pack("<I", 9) + s[36:], ref.CorruptStream),   # unknown codec
    (lambda s: s[:44] + struct.pack("<I", 2) + s[48:], ref.CorruptStream),   # n_words
    (lambda s: s[:-8] + struct.pack("<Q", 3 ** 40), ref.CorruptStream),      # residue
    (lambda s: s[:36] + struct.pack("<I", 65535) + s[40:], ref.CorruptStream),  # overflow
])
def test_corrupt_streams(mutate, exc):
    s = ref.compress_blocked([5, 7, 6, 4, 4, 4, 4], 16, 3)
    with pytest.raises(exc):
        ref.decompress_blocked(mutate(s))

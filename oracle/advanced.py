"""Python big-integer oracle for the ADVANCED (split-base) polynomial codec of
PAPER.md Sec. 3.2, blocked as in Sec. 3.3.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call or
execute this module: only ``tests/``, ``__graft_entry__.smoke()``,
``bench.py``'s oracle legs and the study scripts do.  It shares no code, table
or constant with the CUDA path (``paper_1805_01844_b200/``).

The codec packs the min-shifted values of a block into 32-bit words (the
paper's ``unsigned int``) without the unused top of each
basic word: the last digit of a word is split into (r, r') against two bases
R and R' with R * R' >= B; r goes into the current word, r' into the next
one (Fig. 4).  Every quantity below follows the paper's
series step by step, in exact Python integers:

    p_i  = floor( (ln(2^32 - 1) - ln R'_{i-1}) / ln B )   -> the largest p with
                                                             R'_{i-1} B^p <= 2^32 - 1
    R_i  = floor( (2^32 - 1) / (R'_{i-1} B^{p_i}) )
    R'_i = ceil( B / R_i )
    q_i  = values consumed before word i
    r'_i = floor( v_{split} / R_i ),  r_i = v_{split} - r'_i R_i
    s_i  = r_i + R_i ( sum_k v_{q_i + k} B^{p_i - k} + r'_{i-1} B^{p_i} )

with R'_0 = 1, r'_0 = 0.  Readings (A1-A6, and
SPEC.md:111-203 "split-codec"):
  A1 the logarithms are evaluated exactly: p_i = max{p : R'_{i-1} B^p <= 2^32-1}
     (float logs are off by one near exact powers);
  A2 the garbled sum bound "k=1, k != p_i .. p_i" is p_i full digits per
     non-final word, plus one split value; so q_{i+1} = q_i + p_i + 1;
  A3 the first full digit of a word takes the HIGHEST power B^{p_i - 1}
     ("accumulated from the highest exponent");
  A4 a word is FINAL when the values left m <= p_i: it holds those m values
     as full digits and the pending carry r'_{i-1} at B^m, with no split
     (SPEC.md:186);
  A5 Eq. (5)'s "B mod R_0" is R_1 (a typo): R'_i = ceil(B / R_i);
  A6 the capacity bound is the literal 2^32 - 1 of Eq. (3)-(4) (not 2^32).

Pins (tests/test_oracle_advanced.py): the SPEC.md:130-160 worked examples
(schedules for B = 1000 and 100000, packed words, unpacked values, word
counts); the series' invariants (tightness R_i R'_{i-1} B^{p_i} <= 2^32-1 <
(R_i+1) R'_{i-1} B^{p_i}, completion R_i R'_i >= B, consumption); round trips
by brute force over every vector of tiny length and base; the counting bound
2^(32 words) >= B^n (the packing is injective); the steady-state efficiency
SPEC.md:170; and the paper's own ratios 2.10361 / 2.47054 on
A(3000, 500, 2000, 45000, 4, 1855) within sampling tolerance.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import List, Sequence, Tuple

WORD_MAX = (1 << 32) - 1       # Eq. (3)-(4): 2^32 - 1 (reading A6)

CODEC_RAW, CODEC_CONSTANT, CODEC_ADVANCED = 0, 1, 3
MAGIC = b"PLYC"
VERSION = 2
LAYOUT_ADVANCED = 1             # layout byte of an advanced-codec stream (32-bit words)


class CorruptStream(ValueError):
    """trailing residue, carry >= R' or digit >= B."""


@dataclass(frozen=True)
class Step:
    """One word of the schedule (SPEC.md:117-122 SplitStep)."""
    p: int        # full base-B digits in the word
    R: int        # low split base (multiplies the word's body)
    Rp: int       # R' = ceil(B / R), carried into the next word
    Rp_prev: int  # R'_{i-1}: the base of the carry at the top of this word
    q: int        # values consumed before this word (0-based index of its first value)
    final: bool   # the last word of the block (reading A4)
    m: int        # FINAL: values in the word (its full digits); else p


def capacity(B: int, Rp_prev: int = 1) -> int:
    """PAPER.md:197-199, 224-226 (p_1, p_2, p_i): the number of base-B digits
    that fit in a word next to a carry of base R'_{i-1}; with exact integers
    (A1): max{p : R'_{i-1} * B^p <= 2^32 - 1}."""
    p, x = 0, Rp_prev
    while x * B <= WORD_MAX:
        x *= B
        p += 1
    return p


def split_schedule(B: int, n: int) -> List[Step]:
    """PAPER.md:244-257 (the series): the steps of a block of
    n values with base B, deterministic in (B, n)."""
    if B < 2:
        raise ValueError("split_schedule needs B >= 2 (B = 1 is a CONSTANT block)")
    if capacity(B, 1) < 1:
        raise ValueError("DegenerateBase: capacity(B, 1) = 0 (RAW block)")
    steps: List[Step] = []
    Rp_prev, q = 1, 0                          # R'_0 = 1
    while True:
        p = capacity(B, Rp_prev)               # p_i
        m = n - q                              # values left
        if m <= p:                             # FINAL word (A4)
            steps.append(Step(p, 0, 0, Rp_prev, q, True, m))
            return steps
        R = WORD_MAX // (Rp_prev * B ** p)     # R_i
        Rp = -(-B // R)                        # R'_i = ceil(B / R_i) (A5)
        steps.append(Step(p, R, Rp, Rp_prev, q, False, p))
        q += p + 1                             # p_i full digits + one split value (A2)
        Rp_prev = Rp


def advanced_word_count(B: int, n: int) -> int:
    """the number of words, by walking the schedule."""
    return len(split_schedule(B, n))


def pack_advanced(d: Sequence[int], B: int) -> List[int]:
    """PAPER.md:233-257 s_i for min-shifted digits d (each in [0, B)).
    Non-final word i: the split value d[q_i + p_i] gives r'_i = floor(./R_i),
    r_i = . - r'_i R_i; body = sum_k d[q_i+k] B^(p_i-1-k)
    (k = 0..p_i-1, first digit at the highest power, A3) + r'_{i-1} B^{p_i};
    s_i = r_i + R_i * body.  FINAL word: r'_{i-1} B^m + sum_k d[q_i+k] B^(m-1-k)."""
    n = len(d)
    words: List[int] = []
    r_prime_prev = 0                            # r'_0 = 0
    for st in split_schedule(B, n):
        body = r_prime_prev
        for k in range(st.m):                   # highest exponent first (A3)
            body = body * B + d[st.q + k]
        if st.final:
            s = body
        else:
            v = d[st.q + st.p]                  # the split value
            r_prime = v // st.R
            r = v - r_prime * st.R
            s = r + st.R * body
            r_prime_prev = r_prime
        assert 0 <= s <= WORD_MAX
        words.append(s)
    return words


def unpack_advanced(words: Sequence[int], B: int, n: int) -> List[int]:
    """PAPER.md:147 ("a polynomial division can be used to uncompress") with
    the schedule of (B, n): r_i = s mod R_i, t = s div R_i,
    full digits = t's base-B digits below B^{p_i}, carry r'_{i-1} = t div
    B^{p_i} completing the previous split value r'_{i-1} R_{i-1} + r_{i-1}.
    Raises CorruptStream on a wrong word count, a carry >= R'_{i-1}, a split
    value >= B or a word > 2^32 - 1."""
    sched = split_schedule(B, n)
    if len(words) != len(sched):
        raise CorruptStream("word count %d != %d" % (len(words), len(sched)))
    out = [0] * n
    r_prev = 0
    for i, (s, st) in enumerate(zip(words, sched)):
        if not 0 <= s <= WORD_MAX:
            raise CorruptStream("word out of range")
        if st.final:
            r, t = 0, s
        else:
            r, t = s % st.R, s // st.R
        low = B ** st.m
        carry, digits = t // low, t % low
        if carry >= st.Rp_prev:
            raise CorruptStream("carry >= R' (word %d)" % i)
        for k in range(st.m - 1, -1, -1):       # lowest power = last digit
            out[st.q + k] = digits % B
            digits //= B
        if i > 0:                               # complete the previous split value
            prev = sched[i - 1]
            v = carry * prev.R + r_prev
            if v >= B:
                raise CorruptStream("split value >= B (word %d)" % i)
            out[prev.q + prev.p] = v
        r_prev = r
    return out


# ---------------------------------------------------------------------------
# Sec. 3.3 blocks and the advanced stream (layout byte 1)
# ---------------------------------------------------------------------------
def block_codec(block: Sequence[int], width: int) -> Tuple[int, int, int, List[int]]:
    """One block: (codec, v_min, b_minus_1, words).  B = 1 -> CONSTANT (no
    words); capacity(B, 1) = 0 (only B = 2^32) -> RAW (the offsets verbatim,
    SPEC.md:240); else ADVANCED."""
    vmin, vmax = min(block), max(block)
    B = vmax - vmin + 1
    if B == 1:
        return CODEC_CONSTANT, vmin, 0, []
    d = [v - vmin for v in block]
    if capacity(B, 1) < 1:
        return CODEC_RAW, vmin, B - 1, d
    return CODEC_ADVANCED, vmin, B - 1, pack_advanced(d, B)


def compress_advanced(x: Sequence[int], width: int, block_len: int) -> bytes:
    """The advanced-codec stream: 32-byte global header (layout byte 1),
    n_blocks 16-byte block headers {codec, v_min, b_minus_1, n_words}, then
    every block's 32-bit words (little-endian), in block order."""
    n = len(x)
    if n == 0:
        raise ValueError("EmptyInput")
    Le = n if block_len == 0 else block_len
    nb = -(-n // Le)
    hdrs, pay = [], []
    for b in range(nb):
        codec, vmin, bm1, words = block_codec(x[b * Le:min(n, (b + 1) * Le)], width)
        hdrs.append(struct.pack("<IIII", codec, vmin, bm1, len(words)))
        pay.extend(words)
    head = MAGIC + bytes([VERSION, LAYOUT_ADVANCED, width, 0]) + struct.pack("<QIIQ", n, block_len, nb, 4 * len(pay))
    return head + b"".join(hdrs) + b"".join(struct.pack("<I", w) for w in pay)


def decompress_advanced(stream: bytes) -> List[int]:
    """Inverse of compress_advanced; raises CorruptStream on any inconsistency."""
    if len(stream) < 32 or stream[:4] != MAGIC:
        raise CorruptStream("not a container")
    if stream[4] != VERSION or stream[5] != LAYOUT_ADVANCED:
        raise CorruptStream("version / layout")
    width = stream[6]
    n, L, nb, pb = struct.unpack("<QIIQ", stream[8:32])
    Le = n if L == 0 else L
    if n == 0 or nb != -(-n // Le) or len(stream) != 32 + 16 * nb + pb or pb % 4:
        raise CorruptStream("length")
    out: List[int] = []
    off = 32 + 16 * nb
    for b in range(nb):
        codec, vmin, bm1, nw = struct.unpack("<IIII", stream[32 + 16 * b:48 + 16 * b])
        nbv = min(Le, n - b * Le)
        words = list(struct.unpack("<%dI" % nw, stream[off:off + 4 * nw])) if nw else []
        if off + 4 * nw > len(stream):
            raise CorruptStream("payload overrun")
        off += 4 * nw
        B = bm1 + 1
        if vmin + bm1 >= 1 << width:
            raise CorruptStream("value overflow")
        if codec == CODEC_CONSTANT:
            if bm1 != 0 or nw != 0:
                raise CorruptStream("constant block with payload")
            out.extend([vmin] * nbv)
        elif codec == CODEC_RAW:
            if nw != nbv or any(w >= B for w in words):
                raise CorruptStream("raw block")
            out.extend(vmin + w for w in words)
        elif codec == CODEC_ADVANCED:
            if B < 2 or capacity(B, 1) < 1:
                raise CorruptStream("advanced block base")
            out.extend(vmin + d for d in unpack_advanced(words, B, nbv))
        else:
            raise CorruptStream("codec")
    if off != len(stream):
        raise CorruptStream("trailing bytes")
    return out


def core_ratio(x: Sequence[int], block_len: int, raw_bits: int = 32, header_bytes: int = 16) -> float:
    """SPEC.md:246-249 ratio accounting used for the paper's figures:
    (n * raw_bits / 8) / sum over blocks of (header_bytes + 4 * words)."""
    n = len(x)
    Le = n if block_len == 0 else block_len
    total = 0
    for b in range(0, n, Le):
        blk = x[b:b + Le]
        vmin, vmax = min(blk), max(blk)
        B = vmax - vmin + 1
        words = 0 if B == 1 else advanced_word_count(B, len(blk))
        total += header_bytes + 4 * words
    return n * raw_bits / 8 / total

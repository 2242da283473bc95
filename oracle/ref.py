"""Python big-integer oracle for the basic blocked polynomial codec.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call or
execute this module: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs do.  It shares no
code, table or constant with the CUDA path (``paper_1805_01844_b200/``).

Every function follows one passage of the paper (PAPER.md = the LaTeX source of
arXiv 1805.01844, read-only at /root/reference/PAPER.md) step by step, with
plain Python integers (arbitrary precision), so that it can be checked against
the paper by eye.  Where the paper is silent or garbled, the reading taken is the
one listed in DESIGN.md "Readings" (R1..R12, same numbering as SURVEY.md D1..D12).

Pins (what this module is checked against, in tests/test_oracle_pins.py):
  * derive_base          -- SPEC.md:55-57 worked examples; numpy min/max.
  * capacity             -- brute force over every B <= 65536 and threshold
                            +-1 values; closed form floor(64/j) for B = 2^j;
                            SPEC.md:65-67 examples in 32-bit literal mode.
  * pack_basic           -- SPEC.md:75-76 examples (32-bit literal mode);
                            B = 2^j  == bit-field packing (int.from_bytes);
                            B = 10   == decimal concatenation of reversed digits;
                            B <= 36  == int(reversed digit string, B).
  * unpack_basic         -- round trip + uniqueness of base-B representation;
                            SPEC.md:85-86 examples.
  * compress_blocked     -- closed-form size 32+16*n_blocks+8*sum ceil(n_b/k_b);
                            brute force over all tiny arrays; block independence.
  * decompress_blocked   -- round trip; corruption cases raise CorruptStream.
No function here is "parity unpinned".
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import List, Sequence, Tuple

# ---------------------------------------------------------------------------
# Word ring.  PAPER.md:103-104 (Sec. 3): "An unsigned int range [0, 2^32[ defines
# a mathematical set Z/dZ ... where d = 2^32".  Reading R1 (north_star): the
# packed word is 64 bits, so d = 2^64.  Reading R2: the capacity rule is
# B^k <= d (the text's word range [0, d[ holds every value < B^k iff B^k <= d).
# The literal Eq. 1 form (B^k <= d - 1) is kept as a parameter for the SPEC
# 32-bit worked examples only.
# ---------------------------------------------------------------------------
WORD_BITS = 64
WORD_RING = 1 << WORD_BITS          # d = 2^64  (R1)

CODEC_RAW, CODEC_CONSTANT, CODEC_BASIC, CODEC_ADVANCED = 0, 1, 2, 3   # R7
MAGIC = b"PLYC"
VERSION = 2
GLOBAL_HEADER_BYTES = 32            # R9
BLOCK_HEADER_BYTES = 16             # R7


class EmptyInput(ValueError):
    """compressing an empty vector."""


class CorruptStream(ValueError):
    """stream content inconsistent."""


class NotAContainer(CorruptStream):
    """bad magic."""


class UnsupportedVersion(CorruptStream):
    """unknown version byte."""


# ---------------------------------------------------------------------------
# Sec. 3.1: v_min, v_max and the compression base B.
# ---------------------------------------------------------------------------
def derive_base(values: Sequence[int]) -> Tuple[int, int, int]:
    """PAPER.md:127 "its minimum v_min and its maximum v_max define its
    associated ring"; "B = v_max - v_min + 1".

    Returns (v_min, v_max, B).  Raises EmptyInput for an empty vector
    (SPEC.md:53)."""
    if len(values) == 0:
        raise EmptyInput("derive_base of an empty vector")
    v_min = int(min(values))
    v_max = int(max(values))
    B = v_max - v_min + 1
    return v_min, v_max, B


# ---------------------------------------------------------------------------
# Eq. 1: p = floor(ln(2^32 - 1) / ln B), "the number of
# bases B that can be stored in one unsigned int".  Computed exactly (no float
# logs) as the largest k with B^k <= limit.
# ---------------------------------------------------------------------------
def capacity(B: int, limit: int = WORD_RING) -> int:
    """Largest k >= 0 with B**k <= limit, by the exact integer loop.

    limit = 2^64 is reading R2 (the full-word rule, the value this build uses);
    limit = 2^32 - 1 reproduces Eq. 1 literally for SPEC's 32-bit examples.
    B must be >= 2 (B = 1 is the CONSTANT block, reading R6)."""
    B = int(B)
    limit = int(limit)
    if B < 2:
        raise ValueError("capacity is defined for B >= 2 (B = 1 is CONSTANT)")
    k = 0
    p = 1
    while p * B <= limit:
        p = p * B
        k = k + 1
    return k


# ---------------------------------------------------------------------------
# Eq. 2: s_j = sum_{i=1}^{p} v_{i+p(j-1)} B^{i-1}.
# Readings: R3 first value of a word multiplies B^0; R4 the digits are the
# min-shifted values d = v - v_min; R5 the last word holds
# the remaining m = n - p*(W-1) digits (its missing high digits are zero).
# ---------------------------------------------------------------------------
def pack_basic(values: Sequence[int], v_min: int, B: int, k: int) -> List[int]:
    """Pack the min-shifted values k per word, first value at B^0 (Eq. 2)."""
    values = [int(v) for v in values]
    v_min, B, k = int(v_min), int(B), int(k)
    n = len(values)
    n_words = (n + k - 1) // k
    words = []
    for j in range(1, n_words + 1):                 # j = 1 .. ceil(n/k)  (R5)
        s_j = 0
        for i in range(1, k + 1):                   # i = 1 .. p
            idx = i + k * (j - 1)                   # 1-based index of Eq. 2
            if idx > n:
                break                               # missing high digits = 0
            d = values[idx - 1] - v_min              # R4
            if not (0 <= d < B):
                raise ValueError("value outside [v_min, v_min + B - 1]")
            s_j = s_j + d * B ** (i - 1)
        words.append(s_j)
    return words


def unpack_basic(words: Sequence[int], v_min: int, B: int, k: int, n: int) -> List[int]:
    """PAPER.md:147 "A polynomial division can be used to uncompress the data":
    each word yields its digits by repeated (mod B, div B); the residue after
    the word's m digits must be zero."""
    if len(words) != (n + k - 1) // k:
        raise CorruptStream("word count != ceil(n/k)")
    out = []
    for j, s in enumerate(words):
        m = min(k, n - j * k)
        for _ in range(m):
            d = s % B
            s = s // B
            out.append(v_min + d)
        if s != 0:
            raise CorruptStream("nonzero residue after the word's digits")
    return out


# ---------------------------------------------------------------------------
# Sec. 3.3 blocked compression: each block gets its own
# (v_min, B).  R10: block_len 0 = one block of the whole vector; the short last
# block is coded like any other.
# ---------------------------------------------------------------------------
def effective_block_len(n: int, block_len: int) -> int:
    return n if block_len == 0 else block_len


def block_ranges(n: int, block_len: int) -> List[Tuple[int, int]]:
    L = effective_block_len(n, block_len)
    n_blocks = (n + L - 1) // L
    return [(b * L, min(n, (b + 1) * L)) for b in range(n_blocks)]


@dataclass
class BlockRecord:
    codec_id: int
    v_min: int
    b_minus_1: int
    n_words: int
    words: List[int]


def compress_block(values: Sequence[int]) -> BlockRecord:
    """One block of Sec. 3.3: derive (v_min, B) (Sec. 3.1), then CONSTANT for
    B = 1 (R6: Eq. 1 divides by ln 1 = 0) else BASIC with k = capacity(B)."""
    v_min, v_max, B = derive_base(values)
    if B == 1:
        return BlockRecord(CODEC_CONSTANT, v_min, 0, 0, [])
    k = capacity(B)
    words = pack_basic(values, v_min, B, k)
    for s in words:
        assert 0 <= s < WORD_RING
    return BlockRecord(CODEC_BASIC, v_min, B - 1, len(words), words)


def serialize(records: Sequence[BlockRecord], n: int, width_bits: int, block_len: int) -> bytes:
    """Reading R8/R9: 32-byte global header || all 16-byte block headers ||
    all payload words (u64 LE), blocks in source order."""
    payload_words = sum(r.n_words for r in records)
    out = bytearray()
    out += MAGIC
    out += struct.pack("<BBBB", VERSION, 0, width_bits, 0)
    out += struct.pack("<Q", n)
    out += struct.pack("<I", block_len)
    out += struct.pack("<I", len(records))
    out += struct.pack("<Q", 8 * payload_words)
    assert len(out) == GLOBAL_HEADER_BYTES
    for r in records:
        out += struct.pack("<IIII", r.codec_id, r.v_min, r.b_minus_1, r.n_words)
    for r in records:
        for s in r.words:
            out += struct.pack("<Q", s)
    return bytes(out)


def compress_blocked(values: Sequence[int], width_bits: int, block_len: int) -> bytes:
    """Whole codec: blocks (Sec. 3.3) -> per block Sec. 3.1 -> stream (R8/R9)."""
    values = [int(v) for v in values]      # plain Python integers throughout
    n = len(values)
    if n == 0:
        raise EmptyInput("compress of an empty vector")
    if width_bits not in (8, 16, 32):       # SPEC.md:30 widths
        raise ValueError("width_bits must be 8, 16 or 32")
    for v in values:
        if not (0 <= v < (1 << width_bits)):
            raise ValueError("value does not fit the declared width")
    if not (0 <= block_len < (1 << 32)):
        raise ValueError("block_len must fit u32")
    ranges = block_ranges(n, block_len)
    if len(ranges) >= (1 << 32):
        raise ValueError("n_blocks must fit u32")
    records = [compress_block(values[lo:hi]) for lo, hi in ranges]
    return serialize(records, n, width_bits, block_len)


def parse_header(stream: bytes) -> Tuple[int, int, int, int, int]:
    """Returns (width_bits, n, block_len, n_blocks, payload_bytes)."""
    if len(stream) < GLOBAL_HEADER_BYTES:
        raise CorruptStream("truncated global header")
    if stream[0:4] != MAGIC:
        raise NotAContainer("bad magic")
    version, layout, width_bits, policy = struct.unpack_from("<BBBB", stream, 4)
    if version != VERSION:
        raise UnsupportedVersion("version %d" % version)
    if layout != 0 or policy != 0 or width_bits not in (8, 16, 32):
        raise CorruptStream("bad layout/policy/width")
    (n,) = struct.unpack_from("<Q", stream, 8)
    block_len, n_blocks = struct.unpack_from("<II", stream, 16)
    (payload_bytes,) = struct.unpack_from("<Q", stream, 24)
    return width_bits, n, block_len, n_blocks, payload_bytes


def decompress_blocked(stream: bytes) -> Tuple[List[int], int]:
    """Inverse of compress_blocked: walk the headers in order with a running
    word offset; CONSTANT fills v_min; BASIC unpacks by polynomial division.
    Returns (values, width_bits)."""
    width_bits, n, block_len, n_blocks, payload_bytes = parse_header(stream)
    if n == 0:
        raise CorruptStream("n = 0")
    ranges = block_ranges(n, block_len)
    if len(ranges) != n_blocks:
        raise CorruptStream("n_blocks != ceil(n / block_len)")
    payload_start = GLOBAL_HEADER_BYTES + BLOCK_HEADER_BYTES * n_blocks
    if len(stream) != payload_start + payload_bytes or payload_bytes % 8 != 0:
        raise CorruptStream("stream length != header + payload")
    out: List[int] = []
    word_off = 0
    for b, (lo, hi) in enumerate(ranges):
        codec, v_min, b_minus_1, n_words = struct.unpack_from(
            "<IIII", stream, GLOBAL_HEADER_BYTES + BLOCK_HEADER_BYTES * b)
        n_b = hi - lo
        if codec == CODEC_CONSTANT:
            if b_minus_1 != 0 or n_words != 0:
                raise CorruptStream("CONSTANT block with payload")
            if v_min >= (1 << width_bits):
                raise CorruptStream("value overflow")
            out.extend([v_min] * n_b)
            continue
        if codec != CODEC_BASIC:
            raise CorruptStream("unknown codec %d" % codec)
        B = b_minus_1 + 1
        if B < 2 or v_min + B - 1 >= (1 << width_bits):
            raise CorruptStream("value overflow / bad base")
        k = capacity(B)
        if n_words != (n_b + k - 1) // k:
            raise CorruptStream("n_words != ceil(n_b/k)")
        if 8 * (word_off + n_words) > payload_bytes:
            raise CorruptStream("payload overrun")
        words = list(struct.unpack_from("<%dQ" % n_words, stream, payload_start + 8 * word_off))
        word_off += n_words
        out.extend(unpack_basic(words, v_min, B, k, n_b))
    if 8 * word_off != payload_bytes:
        raise CorruptStream("sum of n_words != payload_bytes")
    return out, width_bits

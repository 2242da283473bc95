// poly_word.cuh -- per-word codec pieces shared by every regime: the Horner
// pack of Eq. 2 and the divide-free digit extraction that
// inverts it, block statistics and block-header validation.
#pragma once
#include "poly_common.cuh"

namespace polyk {

// ceil(n / k) for n < 2^24, 1 <= k <= 64, without an integer divide.
__device__ __forceinline__ uint32_t ceil_div_small(uint32_t n, uint32_t k) {
  uint32_t q = (uint32_t)__fmul_rz((float)(n + k - 1), __frcp_rn((float)k));
  if (q * k > n + k - 1) --q;
  if ((q + 1) * k <= n + k - 1) ++q;
  return q;
}

// One 64-bit fraction step (d, f) = (floor(f B / 2^64), f B mod 2^64), and
// one 32-bit step (d, g) = (floor(g B / 2^32), g B mod 2^32).
__device__ __forceinline__ uint32_t frac_step64(uint32_t& f0, uint32_t& f1, uint32_t B) {
  uint32_t n0, n1, c, d;
  asm("mul.lo.u32 %0, %4, %6;\n\t"
      "mul.hi.u32 %1, %4, %6;\n\t"
      "mad.lo.cc.u32 %2, %5, %6, %1;\n\t"
      "madc.hi.u32 %3, %5, %6, 0;"
      : "=&r"(n0), "=&r"(c), "=&r"(n1), "=r"(d)  // early clobber: outputs are written before the inputs are all read
      : "r"(f0), "r"(f1), "r"(B));
  f0 = n0;
  f1 = n1;
  return d;
}
__device__ __forceinline__ uint32_t frac_step32(uint32_t& g, uint32_t B) {
  uint32_t lo, hi;
  asm("mul.lo.u32 %0, %2, %3;\n\tmul.hi.u32 %1, %2, %3;" : "=&r"(lo), "=r"(hi) : "r"(g), "r"(B));
  g = lo;
  return hi;
}

// min / max of n values at s (one thread).  u16 at a 4-byte boundary: packed
// u16x2 min/max over 32-bit words, four words per step.
template <typename V>
__device__ __forceinline__ void block_minmax(const V* s, uint32_t n, uint32_t& mn, uint32_t& mx) {
  if (sizeof(V) == 2 && (reinterpret_cast<uintptr_t>(s) & 3) == 0) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(s);
    const uint32_t nw = n >> 1;
    uint32_t a = 0xffffffffu, b = 0u;
    uint32_t i = 0;
#pragma unroll 1
    for (; i + 4 <= nw; i += 4) {
      const uint32_t x0 = w[i], x1 = w[i + 1], x2 = w[i + 2], x3 = w[i + 3];
      a = __vimin3_u16x2(a, x0, x1);
      b = __vimax3_u16x2(b, x0, x1);
      a = __vimin3_u16x2(a, x2, x3);
      b = __vimax3_u16x2(b, x2, x3);
    }
#pragma unroll 1
    for (; i < nw; ++i) {
      a = __vminu2(a, w[i]);
      b = __vmaxu2(b, w[i]);
    }
    mn = min(a & 0xffffu, a >> 16);
    mx = max(b & 0xffffu, b >> 16);
    if (n & 1) {
      const uint32_t x = (uint32_t)s[n - 1];
      mn = min(mn, x);
      mx = max(mx, x);
    }
  } else {
    mn = 0xffffffffu;
    mx = 0u;
#pragma unroll 4
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t x = (uint32_t)s[i];
      mn = min(mn, x);
      mx = max(mx, x);
    }
  }
}

// ------------------------------------------------------------------ pack (a5)
// Horner of Eq. 2 over 32-bit chunks of h digits:
// s = sum_q c_q D^q, D = B^h, each chunk c_q < B^h <= 2^32 evaluated with
// 32-bit multiply-adds, chunks combined top-down with 64x32 multiply-adds.
// Requires B <= 2^32 - 1 (B = 2^32 goes through pack_word_b32).
template <typename V>
__device__ __forceinline__ uint32_t chunk32(const V* v, uint32_t len, uint32_t B, uint32_t vmin) {
  uint32_t c = 0;
#pragma unroll 4
  for (int i = (int)len - 1; i >= 0; --i) c = c * B + ((uint32_t)v[i] - vmin);
  return c;
}

template <typename V>
__device__ __forceinline__ uint64_t pack_word(const V* v, uint32_t m, uint32_t B, uint32_t h, uint32_t D,
                                              uint32_t vmin) {
  // chunks from the top: the top one holds r = m - (nch-1) h digits
  const uint32_t nch = m <= h ? 1u : (m <= 2 * h ? 2u : 3u);
  const uint32_t r = m - (nch - 1) * h;
  uint64_t s = chunk32<V>(v + (nch - 1) * h, r, B, vmin);
  for (int q = (int)nch - 2; q >= 0; --q) {
    const uint32_t c = chunk32<V>(v + q * h, h, B, vmin);
    if (D == 0)  // D = 2^32 (B = 2^j, j | 32)
      s = (s << 32) | c;
    else
      s = s * D + c;
  }
  return s;
}

template <typename V>
__device__ __forceinline__ uint64_t pack_word_b32(const V* v, uint32_t m, uint32_t vmin) {
  uint64_t s = 0;
  for (int i = (int)m - 1; i >= 0; --i) s = (s << 32) | (uint32_t)((uint32_t)v[i] - vmin);
  return s;
}

// Per-block packing parameters.
struct PackParams {
  uint32_t B, h, D, k;
};
__device__ __forceinline__ PackParams pack_params(uint32_t bm1) {
  PackParams p;
  p.B = bm1 + 1;  // wraps to 0 for B = 2^32 (handled by pack_word_b32)
  capacity_kh((uint64_t)bm1 + 1, p.k, p.h);
  uint64_t D = 1;
  for (uint32_t i = 0; i < p.h; ++i) D *= (uint64_t)bm1 + 1;
  p.D = (uint32_t)D;  // 0 iff D = 2^32
  return p;
}

template <typename V>
__device__ __forceinline__ uint64_t pack_any(const V* v, uint32_t m, const PackParams& p, uint32_t vmin) {
  if (p.B == 0) return pack_word_b32<V>(v, m, vmin);
  return pack_word<V>(v, m, p.B, p.h, p.D, vmin);
}

// Eq. 2 with a plain 64-bit Horner (no chunks): s = sum_{i<m} (v[i] - vmin) B^i,
// evaluated from the top digit down; B <= 2^32 (B = 2^32 shifts).
template <typename V>
__device__ __forceinline__ uint64_t pack_word64(const V* v, uint32_t m, uint64_t B, uint32_t vmin) {
  uint64_t s = 0;
  if (sizeof(V) == 2) {
    const uint32_t Bu = (uint32_t)B;
#pragma unroll 4
    for (int i = (int)m - 1; i >= 0; --i) s = s * Bu + ((uint32_t)v[i] - vmin);
  } else if (B == (1ull << 32)) {
    for (int i = (int)m - 1; i >= 0; --i) s = (s << 32) | ((uint32_t)v[i] - vmin);
  } else {
    for (int i = (int)m - 1; i >= 0; --i) s = s * B + ((uint32_t)v[i] - vmin);
  }
  return s;
}

// All nw words of one block, one thread: a single top-down Horner sweep over
// the block's nb values; word j holds values [jk, jk + m_j) (reading R5), so a
// word is complete when the sweep reaches its first value.  The loop trip
// count is the block length, the same for every lane of a warp, whatever
// each lane's base and k.
template <typename V>
__device__ __forceinline__ void pack_block_lane(const V* v, uint32_t nb, uint32_t vmin, uint64_t B, uint32_t k,
                                                uint32_t nw, uint64_t* dst) {
  uint32_t cnt = nb - (nw - 1) * k;
  uint32_t wj = nw - 1;
  uint64_t s = 0;
  if (sizeof(V) == 2) {
    const uint32_t Bu = (uint32_t)B;
#pragma unroll 2
    for (int i = (int)nb - 1; i >= 0; --i) {
      s = s * Bu + ((uint32_t)v[i] - vmin);
      if (--cnt == 0) {
        dst[wj--] = s;
        s = 0;
        cnt = k;
      }
    }
  } else {
    for (int i = (int)nb - 1; i >= 0; --i) {
      const uint32_t d = (uint32_t)v[i] - vmin;
      s = (B == (1ull << 32)) ? ((s << 32) | d) : (s * B + d);
      if (--cnt == 0) {
        dst[wj--] = s;
        s = 0;
        cnt = k;
      }
    }
  }
}

// All nw words of one block, one thread, word by word from the top: word j
// holds values [jk, jk + m_j) (reading R5); each word is a plain Horner loop
// over its own digits (no per-value word-boundary test).
template <typename V>
__device__ __forceinline__ uint32_t decode_frac(uint64_t s, const DecConst& c, uint32_t B, uint32_t m,
                                                uint32_t vmin, V* out);

template <typename V>
__device__ __forceinline__ void pack_block_words(const V* v, uint32_t nb, uint32_t vmin, uint64_t B, uint32_t k,
                                                 uint32_t nw, uint64_t* dst) {
  const V* p = v + nb;
  uint32_t m = nb - (nw - 1) * k;
  if (sizeof(V) == 2) {
    const uint32_t Bu = (uint32_t)B;
    for (int j = (int)nw - 1; j >= 0; --j) {
      uint64_t s = 0;
#pragma unroll 4
      for (uint32_t i = 0; i < m; ++i) {
        --p;
        s = s * Bu + ((uint32_t)*p - vmin);
      }
      dst[j] = s;
      m = k;
    }
  } else {
    for (int j = (int)nw - 1; j >= 0; --j) {
      uint64_t s = 0;
      for (uint32_t i = 0; i < m; ++i) {
        --p;
        const uint32_t d = (uint32_t)*p - vmin;
        s = (B == (1ull << 32)) ? ((s << 32) | d) : (s * B + d);
      }
      dst[j] = s;
      m = k;
    }
  }
}

// All nw words of one u16 block, one thread.  Every word is two independent
// 32-bit Horner chains of h digits (k is 2h or 2h+1 because B^h <= 2^32 <
// B^(h+1)) plus, for k = 2h+1, its top digit:
//   s = (top * B^h + hi) * B^h + lo,   lo / hi = digits [0,h) / [h,2h).
// The chains run on the raw values and subtract vmin * G, G = sum_{i<h} B^i,
// once (exact mod 2^32 because each true chunk is < B^h <= 2^32).  Digits at
// or past the block end are 0 (reading R5): the top word reads vmin there.
// Requires 16 readable bytes of slack after the block (stage padding).
__device__ __forceinline__ void pack_block_lane16(const uint16_t* v, uint32_t nb, uint32_t vmin, uint32_t B,
                                                  uint32_t k, uint32_t h, uint64_t D, uint32_t G, uint32_t nw,
                                                  uint64_t* dst) {
  const uint32_t corr = vmin * G;
  const bool odd = k != 2 * h;
  const uint64_t DD = D * D;
  const uint32_t nfull = (nw * k == nb) ? nw : nw - 1;  // nw = ceil(nb / k)
  const uint32_t B2 = B * B;                            // B < 2^16 unless B = 2^16 (then B2 = 0, h = 2)
#pragma unroll 1
  for (uint32_t j = 0; j < nfull; ++j) {
    // two chains, two digits per step: c = c B^2 + (w[i] B + w[i-1])
    const uint16_t* pl = v + j * k + h;  // one past the top digit of the lo chunk
    const uint16_t* ph = pl + h;
    uint32_t lo = 0, hi = 0;
    if (h & 1) {
      --pl;
      --ph;
      lo = *pl;
      hi = *ph;
    }
#pragma unroll 1
    for (uint32_t i = h >> 1; i > 0; --i) {
      pl -= 2;
      ph -= 2;
      lo = lo * B2 + (pl[1] * B + pl[0]);
      hi = hi * B2 + (ph[1] * B + ph[0]);
    }
    uint64_t s = (uint64_t)(hi - corr) * D + (lo - corr);
    if (odd) s += (uint64_t)(v[j * k + 2 * h] - vmin) * DD;
    dst[j] = s;
  }
  if (nfull < nw) {  // the top word: m < k <= 2h + 1 digits, the missing ones are 0
    const uint32_t m = nb - nfull * k;
    const uint16_t* w = v + nfull * k;
    const uint32_t ml = min(m, h), mh = m > h ? m - h : 0u;  // lo / hi chain lengths
    const uint32_t vB1 = vmin * (B + 1);                     // a digit pair's share of vmin
    uint32_t lo = 0, hi = 0;
    const uint16_t* pl = w + ml;
    const uint16_t* ph = w + h + mh;
    if (ml & 1) lo = (uint32_t)*--pl - vmin;
    if (mh & 1) hi = (uint32_t)*--ph - vmin;
#pragma unroll 1
    for (uint32_t i = ml >> 1; i > 0; --i) {
      pl -= 2;
      lo = lo * B2 + (pl[1] * B + pl[0] - vB1);
    }
#pragma unroll 1
    for (uint32_t i = mh >> 1; i > 0; --i) {
      ph -= 2;
      hi = hi * B2 + (ph[1] * B + ph[0] - vB1);
    }
    dst[nfull] = (uint64_t)hi * D + lo;
  }
}

// The top word of a full-length block: m < k digits, digits m..k-1 zero.
// With P = B^(k-m), s' = s P < B^k iff s < B^m, and the digits of s are the
// top m digits of s' -- so only m fraction steps are needed instead of k.
template <typename V>
__device__ __forceinline__ uint32_t decode_top_word(uint64_t s, const DecConst& c, uint32_t B, uint32_t m,
                                                    uint64_t P, uint32_t vmin, V* out) {
  const uint64_t sp = s * P;
  if (__umul64hi(s, P) != 0 || sp > c.Wmax) return POLY_ST_RESIDUE;
  const uint32_t add = dc_add(c);
  const uint64_t hi1 = __umul64hi(sp, c.Rl), lo2 = sp * c.Rh, hi2 = __umul64hi(sp, c.Rh), mid = lo2 + hi1;
  const uint64_t f = ((hi2 + (mid < lo2 ? 1ull : 0ull)) << 32) + (mid >> 32) + add;
  uint32_t f0 = (uint32_t)f, f1 = (uint32_t)(f >> 32);
  const int k = (int)dc_k(c), t = (int)dc_t32(c), lo = k - (int)m;  // digits k-1 .. lo are the output
  int i = k - 1;
  V* o = out + (m - 1);
#pragma unroll 1
  for (; i >= max(t, lo); --i, --o) *o = (V)(vmin + frac_step64(f0, f1, B));
  uint32_t g = f1 + add;
#pragma unroll 1
  for (; i >= lo; --i, --o) *o = (V)(vmin + frac_step32(g, B));
  return 0u;
}

// All words of one block, one thread (B < 2^32).
// P = B^(k - m_top) for the block's top word, or 0 (then the top word steps
// through its zero digits).
template <typename V>
__device__ __forceinline__ uint32_t decode_block_lane(const uint64_t* src, uint32_t nw, uint32_t nb,
                                                      const DecConst& c, uint32_t B, uint32_t vmin, uint64_t P,
                                                      V* out) {
  const uint32_t k = dc_k(c);
  uint32_t err = 0;
  const uint32_t mt = nb - (nw - 1) * k;  // digits of the top word
  const uint32_t nfast = (P != 0 && mt < k) ? nw - 1 : nw;
#pragma unroll 1
  for (uint32_t j = 0, first = 0; j < nfast; ++j, first += k)
    err |= decode_frac<V>(src[j], c, B, min(k, nb - first), vmin, out + first);
  if (nfast < nw) err |= decode_top_word<V>(src[nw - 1], c, B, mt, P, vmin, out + (nw - 1) * k);
  return err;
}

// ------------------------------------------------------------------ unpack (a8)
// Word -> digits, most significant first, through the binary fraction
// f in [s 2^64 / B^k, (s+1) 2^64 / B^k):
//   f = floor(s R / 2^96) + 1,  R = ceil(2^160 / B^k);
//   64-bit step: (d, f) = (floor(f B / 2^64), f B mod 2^64);
//   after k - t32 digits the top 32 bits + 1 are an exact 32-bit fraction for
//   the last t32 digits: (d, g) = (floor(g B / 2^32), g B mod 2^32).
// Word -> its m low digits (out[i] = vmin + digit i, i < m), most significant
// first; digits m..k-1 must be 0.  Plain loops (two digits per iteration): the
// loop trip counts are the only thing that differs between lanes.
template <typename V>
__device__ __forceinline__ uint32_t decode_frac(uint64_t s, const DecConst& c, uint32_t B, uint32_t m,
                                                uint32_t vmin, V* out) {
  if (s > c.Wmax) return POLY_ST_RESIDUE;
  const uint32_t add = dc_add(c);
  const uint64_t hi1 = __umul64hi(s, c.Rl), lo2 = s * c.Rh, hi2 = __umul64hi(s, c.Rh), mid = lo2 + hi1;
  const uint64_t f = ((hi2 + (mid < lo2 ? 1ull : 0ull)) << 32) + (mid >> 32) + add;
  uint32_t f0 = (uint32_t)f, f1 = (uint32_t)(f >> 32);
  const int k = (int)dc_k(c), t = (int)dc_t32(c), mm = (int)m;
  uint32_t extra = 0;
  int i = k - 1;
  if (mm < k) {  // the top word of a block: its top k - m digits are 0
    const int za = max(t, mm);
#pragma unroll 1
    for (; i >= za; --i) extra |= frac_step64(f0, f1, B);
  }
  V* o = out + i;
#pragma unroll 1
  for (; i >= t + 1; i -= 2, o -= 2) {
    const uint32_t d1 = frac_step64(f0, f1, B);
    const uint32_t d0 = frac_step64(f0, f1, B);
    o[0] = (V)(vmin + d1);
    o[-1] = (V)(vmin + d0);
  }
  if (i >= t) {
    o[0] = (V)(vmin + frac_step64(f0, f1, B));
    --i;
    --o;
  }
  uint32_t g = f1 + add;
  if (i >= mm) {
#pragma unroll 1
    for (; i >= mm; --i, --o) extra |= frac_step32(g, B);
  }
#pragma unroll 1
  for (; i >= 1; i -= 2, o -= 2) {
    const uint32_t d1 = frac_step32(g, B);
    const uint32_t d0 = frac_step32(g, B);
    o[0] = (V)(vmin + d1);
    o[-1] = (V)(vmin + d0);
  }
  if (i == 0) o[0] = (V)(vmin + frac_step32(g, B));
  return extra ? POLY_ST_RESIDUE : 0u;
}

template <typename V>
__device__ __forceinline__ uint32_t decode_pow2(uint64_t s, uint32_t j, uint32_t m, uint32_t vmin, V* out) {
  const uint64_t mask = (1ull << j) - 1;  // j <= 32
#pragma unroll 4
  for (uint32_t i = 0; i < m; ++i) out[i] = (V)(vmin + (uint32_t)((s >> (i * j)) & mask));
  return (m * j < 64 && (s >> (m * j)) != 0) ? POLY_ST_RESIDUE : 0u;
}

template <typename V>
__device__ __forceinline__ uint32_t decode_any(uint64_t s, const DecConst& c, uint32_t bm1, uint32_t m,
                                               uint32_t vmin, V* out) {
  const uint32_t j = dc_log2b(c);
  if (j) return decode_pow2<V>(s, j, m, vmin, out);
  return decode_frac<V>(s, c, bm1 + 1, m, vmin, out);
}

// Block-header validation (a9) without an integer divide: n_words must be
// ceil(n_b / k), i.e. (n_words - 1) k < n_b <= n_words k.
__device__ __forceinline__ uint32_t check_block_hdr(uint4 h, uint32_t nb, uint32_t width, uint32_t k) {
  const uint64_t vmax_allowed = (width == 32) ? 0xffffffffull : ((1ull << width) - 1);
  if (h.x == CODEC_CONSTANT) {
    uint32_t e = 0;
    if (h.z != 0 || h.w != 0) e |= POLY_ST_NWORDS;
    if ((uint64_t)h.y > vmax_allowed) e |= POLY_ST_OVERFLOW;
    return e;
  }
  if (h.x != CODEC_BASIC) return POLY_ST_BAD_CODEC;
  if (h.z == 0 || (uint64_t)h.y + h.z > vmax_allowed) return POLY_ST_OVERFLOW;
  if (h.w == 0 || (uint64_t)(h.w - 1) * k >= nb || (uint64_t)h.w * k < nb) return POLY_ST_NWORDS;
  return 0;
}

// The 32-byte global header (reading R9).
__device__ __forceinline__ void write_global_header_f(uint8_t* out, uint32_t width, uint64_t n, uint32_t block_len,
                                                      uint64_t n_blocks, uint64_t payload_words) {
  uint4 h0, h1;
  h0.x = 0x43594c50u;  // "PLYC"
  h0.y = 2u | (width << 16);
  h0.z = (uint32_t)n;
  h0.w = (uint32_t)(n >> 32);
  h1.x = block_len;
  h1.y = (uint32_t)n_blocks;
  h1.z = (uint32_t)(payload_words * 8);
  h1.w = (uint32_t)((payload_words * 8) >> 32);
  reinterpret_cast<uint4*>(out)[0] = h0;
  reinterpret_cast<uint4*>(out)[1] = h1;
}

// inclusive warp scan
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

}  // namespace polyk

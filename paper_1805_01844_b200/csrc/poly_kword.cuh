// poly_kword.cuh -- u16 word codec specialised on the capacity k (a compile-
// time K), for blocks whose k is uniform across a warp (map 1: a warp works
// on one block at a time).
//
// A lane owns a "group" of Q consecutive words (Q = 2 for odd K, else 1), i.e.
// Q*K consecutive values = BYTES bytes, read or written with shared-memory
// vector accesses of VW bytes.  Q and VW are chosen so that the lane stride
// BYTES is an odd multiple of VW for K != 0 mod 16, which makes every access
// of the warp bank-conflict free (32 lanes x VW bytes hit distinct banks).
//
// Pack (Eq. 2): each word is two 32-bit Horner chunks of
// h0 = floor(K/2) digits (B^h0 <= 2^32 because B^K <= 2^64), plus the top
// digit when K is odd, combined in 64 bits.  The chunks run on the raw values
// and subtract vmin * (1 + B + ... + B^(h0-1)) once (exact mod 2^32 because
// the true chunk is < 2^32).
// Unpack: the binary-fraction digit extraction of
// poly_word.cuh decode_frac, fully unrolled, with the switch to 32-bit steps
// at T32MIN[K] = the smallest t32 over the non-power-of-two bases of
// capacity K (exact for every such base: fewer 32-bit steps than a base's own
// t32 are always valid).  Power-of-two bases use shifts.
#pragma once
#include "poly_common.cuh"
#include "poly_word.cuh"

namespace polyk {


// min over non-power-of-two B <= 65536 with k(B) = K of t32(B); computed by
// build_tables() on the host and checked against this table in poly_init.
__host__ __device__ constexpr int t32min_u16(int K) {
  return K == 4 ? 1 : K == 5 ? 1 : K == 6 ? 2 : K == 7 ? 2 : K == 8 ? 3 : K == 9 ? 3 : K == 10 ? 4
       : K == 11 ? 4 : K == 12 ? 5 : K == 13 ? 5 : K == 14 ? 6 : K == 15 ? 6 : K == 16 ? 8 : K == 17 ? 8
       : K == 18 ? 9 : K == 19 ? 9 : K == 20 ? 9 : K == 22 ? 11 : K == 24 ? 12 : K == 27 ? 13 : K == 40 ? 19
       : 0;
}


template <int K>
struct KCls {
  static constexpr int Q = (K % 2) ? 2 : 1;
  static constexpr int VALS = Q * K;
  static constexpr int BYTES = 2 * VALS;  // multiple of 4
  static constexpr int VW = (BYTES % 16 == 0) ? 16 : (BYTES % 8 == 0 ? 8 : 4);
  static constexpr int NR = BYTES / 4;    // 32-bit registers per group
  static constexpr int H0 = K / 2;
};

template <int K>
__device__ __forceinline__ void load_group(const uint8_t* p, uint32_t (&r)[KCls<K>::NR]) {
  using C = KCls<K>;
  if (C::VW == 16) {
#pragma unroll
    for (int i = 0; i < C::NR / 4; ++i) {
      const uint4 v = reinterpret_cast<const uint4*>(p)[i];
      r[4 * i] = v.x;
      r[4 * i + 1] = v.y;
      r[4 * i + 2] = v.z;
      r[4 * i + 3] = v.w;
    }
  } else if (C::VW == 8) {
#pragma unroll
    for (int i = 0; i < C::NR / 2; ++i) {
      const uint2 v = reinterpret_cast<const uint2*>(p)[i];
      r[2 * i] = v.x;
      r[2 * i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < C::NR; ++i) r[i] = reinterpret_cast<const uint32_t*>(p)[i];
  }
}

template <int K>
__device__ __forceinline__ void store_group(uint8_t* p, const uint32_t (&r)[KCls<K>::NR]) {
  using C = KCls<K>;
  if (C::VW == 16) {
#pragma unroll
    for (int i = 0; i < C::NR / 4; ++i)
      reinterpret_cast<uint4*>(p)[i] = make_uint4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
  } else if (C::VW == 8) {
#pragma unroll
    for (int i = 0; i < C::NR / 2; ++i) reinterpret_cast<uint2*>(p)[i] = make_uint2(r[2 * i], r[2 * i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < C::NR; ++i) reinterpret_cast<uint32_t*>(p)[i] = r[i];
  }
}

template <int N>
__device__ __forceinline__ uint32_t val16(const uint32_t (&r)[N], int idx) {
  return (idx & 1) ? (r[idx >> 1] >> 16) : (r[idx >> 1] & 0xffffu);
}

// Per-block constants of the specialised pack.
struct KPack {
  uint32_t B;      // base (<= 65536)
  uint64_t D;      // B^h0 (may be 2^32)
  uint32_t corr;   // vmin * (1 + B + ... + B^(h0-1)) mod 2^32
  uint32_t vmin;
};

template <int K>
__device__ __forceinline__ KPack kpack_consts(uint32_t B, uint32_t vmin) {
  KPack c;
  c.B = B;
  c.vmin = vmin;
  uint64_t D = 1;
  uint32_t G = 0;
#pragma unroll
  for (int i = 0; i < KCls<K>::H0; ++i) {
    G = G * B + 1u;
    D *= B;
  }
  c.D = D;
  c.corr = vmin * G;
  return c;
}

// Pack group g (words g*Q .. g*Q+Q-1, all full) of a block whose values start
// at blk (VW-aligned); words go to dst[g*Q + q].
template <int K>
__device__ __forceinline__ void pack_group(const uint8_t* blk, uint32_t g, const KPack& c, uint64_t* dst) {
  using C = KCls<K>;
  uint32_t r[C::NR];
  load_group<K>(blk + (size_t)g * C::BYTES, r);
#pragma unroll
  for (int q = 0; q < C::Q; ++q) {
    const int o = q * K;
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int i = C::H0 - 1; i >= 0; --i) lo = lo * c.B + val16(r, o + i);
#pragma unroll
    for (int i = 2 * C::H0 - 1; i >= C::H0; --i) hi = hi * c.B + val16(r, o + i);
    lo -= c.corr;
    hi -= c.corr;
    uint64_t s;
    if (K & 1) {
      const uint32_t top = val16(r, o + K - 1) - c.vmin;
      s = ((uint64_t)top * c.D + hi) * c.D + lo;
    } else {
      s = (uint64_t)hi * c.D + lo;
    }
    dst[g * C::Q + q] = s;
  }
}

// The same for a block that starts at any 2-byte aligned address (block
// lengths that are not a multiple of 16 bytes): the values are read one by
// one, 16 bits each, along the Horner chains.
template <int K>
__device__ __forceinline__ void pack_group_u(const uint16_t* blk, uint32_t g, const KPack& c, uint64_t* dst) {
  using C = KCls<K>;
  const uint16_t* v = blk + (size_t)g * C::VALS;
#pragma unroll
  for (int q = 0; q < C::Q; ++q) {
    const int o = q * K;
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int i = C::H0 - 1; i >= 0; --i) lo = lo * c.B + v[o + i];
#pragma unroll
    for (int i = 2 * C::H0 - 1; i >= C::H0; --i) hi = hi * c.B + v[o + i];
    lo -= c.corr;
    hi -= c.corr;
    uint64_t s;
    if (K & 1) {
      const uint32_t top = (uint32_t)v[o + K - 1] - c.vmin;
      s = ((uint64_t)top * c.D + hi) * c.D + lo;
    } else {
      s = (uint64_t)hi * c.D + lo;
    }
    dst[g * C::Q + q] = s;
  }
}
template <int K>
__device__ __forceinline__ uint32_t pack_block_ku(const uint16_t* blk, uint32_t nb, uint32_t B, uint32_t vmin,
                                                  uint32_t g0, uint32_t gstep, uint64_t* dst) {
  using C = KCls<K>;
  const uint32_t ngroups = nb / C::VALS;
  const KPack c = kpack_consts<K>(B, vmin);
  for (uint32_t g = g0; g < ngroups; g += gstep) pack_group_u<K>(blk, g, c, dst);
  return ngroups * C::Q;
}

// Unpack group g of a block (all Q words full).  Returns POLY_ST_RESIDUE if a
// word is >= B^K.
template <int K>
__device__ __forceinline__ uint32_t unpack_group(const uint64_t* src, uint32_t g, const DecConst& dc, uint32_t B,
                                                 uint32_t vmin, uint8_t* blk) {
  using C = KCls<K>;
  constexpr int T = t32min_u16(K);
  uint32_t r[C::NR];
  uint32_t err = 0;
  const uint32_t j = dc_log2b(dc);
#pragma unroll
  for (int q = 0; q < C::Q; ++q) {
    const uint64_t s = src[g * C::Q + q];
    const int o = q * K;
    uint32_t d[K];
    if (j) {  // B = 2^j: bit fields
#pragma unroll
      for (int i = 0; i < K; ++i) d[i] = (uint32_t)(s >> (i * j)) & (B - 1);
      if (K * j < 64 && (s >> (K * j)) != 0) err = POLY_ST_RESIDUE;
    } else {
      if (s > dc.Wmax) err = POLY_ST_RESIDUE;
      const uint64_t hi1 = __umul64hi(s, dc.Rl);
      const uint64_t lo2 = s * dc.Rh;
      const uint64_t hi2 = __umul64hi(s, dc.Rh);
      const uint64_t mid = lo2 + hi1;
      const uint64_t f = ((hi2 + (mid < lo2 ? 1ull : 0ull)) << 32) + (mid >> 32) + 1;
      uint32_t f0 = (uint32_t)f, f1 = (uint32_t)(f >> 32);
#pragma unroll
      for (int i = K - 1; i >= T; --i) {
        const uint64_t t0 = (uint64_t)f0 * B;
        const uint64_t t1 = (uint64_t)f1 * B + (uint32_t)(t0 >> 32);
        d[i] = (uint32_t)(t1 >> 32) + vmin;
        f1 = (uint32_t)t1;
        f0 = (uint32_t)t0;
      }
      uint32_t gg = f1 + 1;
#pragma unroll
      for (int i = T - 1; i >= 0; --i) {
        const uint64_t p = (uint64_t)gg * B;
        d[i] = (uint32_t)(p >> 32) + vmin;
        gg = (uint32_t)p;
      }
    }
    if (j) {
#pragma unroll
      for (int i = 0; i < K; ++i) d[i] += vmin;
    }
    // two values per register: the odd one into the high half by one byte permute
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int idx = o + i;
      if (idx & 1)
        r[idx >> 1] = __byte_perm(r[idx >> 1], d[i], 0x5410);
      else
        r[idx >> 1] = d[i];
    }
  }
  store_group<K>(blk + (size_t)g * C::BYTES, r);
  return err;
}

// The capacities a u16 block can have (B in 2 .. 65536).
// (k = 32, 40, 64, i.e. B <= 4, take the generic path.)
#define POLY_FOR_EACH_K16(X) \
  X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17) X(18) X(19) X(20) X(21) \
  X(22) X(24) X(27)

// One warp (or G warps: lanes g0 + 32*G*i) packs the full groups of a u16 block
// with uniform k; returns the number of leading words it covered.
template <int K>
__device__ __forceinline__ uint32_t pack_block_k(const uint8_t* blk, uint32_t nb, uint32_t B, uint32_t vmin,
                                                 uint32_t g0, uint32_t gstep, uint64_t* dst) {
  using C = KCls<K>;
  const uint32_t ngroups = nb / C::VALS;
  const KPack c = kpack_consts<K>(B, vmin);
  for (uint32_t g = g0; g < ngroups; g += gstep) pack_group<K>(blk, g, c, dst);
  return ngroups * C::Q;
}

// Groups [gb, ge) of a block, lane-strided, by one warp; returns status bits.
template <int K>
__device__ __forceinline__ uint32_t unpack_groups_k(const uint64_t* src, uint32_t gb, uint32_t ge, const DecConst& dc,
                                                    uint32_t B, uint32_t vmin, uint8_t* blk) {
  uint32_t err = 0;
  for (uint32_t g = gb + (threadIdx.x & 31); g < ge; g += 32) err |= unpack_group<K>(src, g, dc, B, vmin, blk);
  return err;
}
template <int K>
__host__ __device__ constexpr uint32_t kvals() { return (uint32_t)KCls<K>::VALS; }
template <int K>
__host__ __device__ constexpr uint32_t kq() { return (uint32_t)KCls<K>::Q; }

template <int K>
__device__ __forceinline__ uint32_t unpack_block_k(const uint64_t* src, uint32_t nb, const DecConst& dc, uint32_t B,
                                                   uint32_t vmin, uint32_t g0, uint32_t gstep, uint8_t* blk,
                                                   uint32_t* words_done) {
  using C = KCls<K>;
  const uint32_t ngroups = nb / C::VALS;
  uint32_t err = 0;
  for (uint32_t g = g0; g < ngroups; g += gstep) err |= unpack_group<K>(src, g, dc, B, vmin, blk);
  *words_done = ngroups * C::Q;
  return err;
}

// Unpack group g with the base class fixed at compile time (POW2: B = 2^j,
// digits are bit fields; else binary-fraction steps), so neither path is
// if-converted into the other (poly_dec3.cuh).
// Digits of group g into registers r (two values per register); returns
// status bits.  The group's words are passed in (w), loaded by the caller.
template <int K, bool POW2>
__device__ __forceinline__ uint32_t unpack_regs_p(const uint64_t (&w)[KCls<K>::Q], const DecConst& dc, uint32_t B,
                                                  uint32_t vmin, uint32_t (&r)[KCls<K>::NR]) {
  using C = KCls<K>;
  constexpr int T = t32min_u16(K);
  uint32_t err = 0;
  if (POW2) {
    // B = 2^J with J = 64 / K (the one power-of-two base of capacity K that
    // takes this path): two J-bit fields per 32-bit register by constant
    // shifts, vmin added to both halves at once (digit + vmin <= 65535)
    constexpr int J = 64 / K;
    constexpr uint32_t M = (1u << J) - 1u;
    const uint32_t vmin2 = vmin * 0x10001u;
#pragma unroll
    for (int q = 0; q < C::Q; ++q)
      if (K * J < 64 && (w[q] >> (K * J)) != 0) err = POLY_ST_RESIDUE;
#pragma unroll
    for (int p = 0; p < C::NR; ++p) {
      const int q0 = (2 * p) / K, e0 = (2 * p) % K, q1 = (2 * p + 1) / K, e1 = (2 * p + 1) % K;
      if (q0 == q1) {
        const uint32_t x = (uint32_t)(w[q0] >> (e0 * J));
        r[p] = ((x & M) | ((x << (16 - J)) & (M << 16))) + vmin2;
      } else {  // the pair straddles the group's two words (odd K)
        const uint32_t d0 = (uint32_t)(w[q0] >> (e0 * J)) & M, d1 = (uint32_t)(w[q1] >> (e1 * J)) & M;
        r[p] = (d0 | (d1 << 16)) + vmin2;
      }
    }
    (void)B;
    (void)dc;
  } else {
#pragma unroll
    for (int q = 0; q < C::Q; ++q) {
      const uint64_t s = w[q];
      const int o = q * K;
      uint32_t d[K];
      if (s > dc.Wmax) err = POLY_ST_RESIDUE;
      const uint64_t hi1 = __umul64hi(s, dc.Rl);
      const uint64_t lo2 = s * dc.Rh;
      const uint64_t hi2 = __umul64hi(s, dc.Rh);
      const uint64_t mid = lo2 + hi1;
      const uint64_t f = ((hi2 + (mid < lo2 ? 1ull : 0ull)) << 32) + (mid >> 32) + 1;
      uint32_t f0 = (uint32_t)f, f1 = (uint32_t)(f >> 32);
#pragma unroll
      for (int i = K - 1; i >= T; --i) {
        const uint64_t t0 = (uint64_t)f0 * B;
        const uint64_t t1 = (uint64_t)f1 * B + (uint32_t)(t0 >> 32);
        d[i] = (uint32_t)(t1 >> 32) + vmin;
        f1 = (uint32_t)t1;
        f0 = (uint32_t)t0;
      }
      uint32_t gg = f1 + 1;
#pragma unroll
      for (int i = T - 1; i >= 0; --i) {
        const uint64_t p = (uint64_t)gg * B;
        d[i] = (uint32_t)(p >> 32) + vmin;
        gg = (uint32_t)p;
      }
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int idx = o + i;
        if (idx & 1)
          r[idx >> 1] = __byte_perm(r[idx >> 1], d[i], 0x5410);
        else
          r[idx >> 1] = d[i];
      }
    }
  }
  return err;
}
// Group g of a block whose words [.., wend) are available: words at or past
// wend (the second word of the block's last, odd pair) read as 0.  Every group
// stores its Q K values, so the staging buffer holds up to K values past the
// last real one (poly_dec3.cuh: the plan's slack).  A short top word is
// decoded like a full one -- its digits past the block's end are not copied
// out; the caller checks it against B^m.
template <int K, bool POW2>
__device__ __forceinline__ uint32_t unpack_group_p(const uint64_t* src, uint32_t g, uint32_t wend, const DecConst& dc,
                                                   uint32_t B, uint32_t vmin, uint8_t* blk) {
  using C = KCls<K>;
  uint64_t w[C::Q];
  uint32_t r[C::NR];
#pragma unroll
  for (int q = 0; q < C::Q; ++q) {
    const uint32_t j = g * C::Q + q;
    w[q] = (q == 0 || j < wend) ? src[j] : 0ull;
  }
  const uint32_t err = unpack_regs_p<K, POW2>(w, dc, B, vmin, r);
  store_group<K>(blk + (size_t)g * C::BYTES, r);
  return err;
}
// Groups [gb, ge) of a block, lane-strided, by one warp; returns status bits.
template <int K, bool POW2>
__device__ __forceinline__ uint32_t unpack_groups_kp(const uint64_t* src, uint32_t gb, uint32_t ge, uint32_t wend,
                                                     const DecConst& dc, uint32_t B, uint32_t vmin, uint8_t* blk) {
  uint32_t err = 0;
  for (uint32_t g = gb + (threadIdx.x & 31); g < ge; g += 32) err |= unpack_group_p<K, POW2>(src, g, wend, dc, B, vmin, blk);
  return err;
}

}  // namespace polyk

// poly_dec3.cuh -- decompression of blocks of 256 B .. 32 KiB (the PIPE
// map-1 regime: cfg4, cfg5, cfg6), in two
// passes:
//
//  dec3_offsets (pass 1): every block's header -> its words n_w and its units
//    (a unit = up to WPU(k) consecutive words of one block, WPU(k) a multiple
//    of 8 with WPU k <= UT values); two device-wide exclusive scans (words,
//    units) chained by a decoupled look-back over chunks of blocks; then the
//    unit table T[u] = {block, first word j0, first payload word}, with a
//    sentinel entry after the last unit.  The headers of this regime are
//    small (<= 16 B per 256 B of values), so the pass costs < 1 % of the
//    traffic.
//  dec3_main (pass 2): with every unit's payload range known there is no
//    cross-CTA dependency: a producer warp per CTA bulk-loads (TMA) tiles of
//    TU units -- table entries, block headers, payload words -- up to NSLOT
//    tiles ahead; consumer warps claim units one at a time and decode each
//    into one of their two staging buffers, which a TMA bulk store of the
//    warp copies to HBM while the warp decodes the next unit into the other.
//    Units split a block into equal parts of about UT values.  u16
//    blocks that start 16-byte aligned use the k-specialised, bank-conflict-
//    free group codec of poly_kword.cuh (unit boundaries fall on multiples of
//    8 words, so every group is 16-byte aligned in the staging buffer); other
//    blocks decode word-parallel with the same binary-fraction steps.
#pragma once
#include "poly_common.cuh"
#include "poly_kword.cuh"
#include "poly_ptx.cuh"

namespace polyk {
namespace d3 {

#ifndef POLY_D3_NW
#define POLY_D3_NW 16
#endif
constexpr int NW = POLY_D3_NW;        // consumer warps per CTA
constexpr int NTHR = 32 * (NW + 1);   // + the producer warp
constexpr int NSLOT = 16;             // tiles in flight per CTA
constexpr int TU = 8;                 // units per tile (16: the ring no longer holds two worst-case tiles)
constexpr int PFD = 4;                // producer: unit-table prefetch depth (tiles)
constexpr uint32_t CE = 2048;         // pass 1: blocks per chunk
constexpr int K1T = 256;              // pass 1 threads per CTA

// POLY_PROBE (timing experiments only, a separate library variant): cycle
// counters per role, summed over warps (lane 0's clock64).
#ifdef POLY_PROBE
__device__ unsigned long long g_probe[24];
#define PROBE_DECL long long pacc[24] = {}
#define PROBE_T0(v) const long long v = clock64()
#define PROBE_ADD(i, t0) pacc[i] += clock64() - (t0)
#define PROBE_FLUSH                                                                  \
  if ((threadIdx.x & 31) == 0)                                                       \
    for (int i_ = 0; i_ < 24; ++i_)                                                  \
      if (pacc[i_]) atomicAdd(&g_probe[i_], (unsigned long long)pacc[i_])
#else
#define PROBE_DECL
#define PROBE_T0(v)
#define PROBE_ADD(i, t0)
#define PROBE_FLUSH
#endif

struct Args {
  const uint8_t* in;
  uint64_t in_bytes;
  uint8_t* out;
  uint32_t* status_out;
  uint32_t* ticket;      // pass-1 chunk ticket
  uint32_t* abort_flag;  // pass 1 -> pass 2: nothing to decode
  uint64_t* cst_w;       // pass-1 look-back words (word counts), one per chunk
  uint64_t* cst_u;       // pass-1 look-back words (unit counts), one per chunk
  uint4* T;              // unit table (+ sentinel)
  uint64_t* n_units;     // pass 1 -> pass 2
  uint64_t n, Le, n_blocks, last_len, n_chunks, max_units;
  uint32_t block_len, width, vb, kmin_log2;
  uint32_t ut;           // values per unit (target)
  uint32_t kw_ok;        // u16: k-specialised codec; 1 = blocks start 16-byte aligned in the output (TMA
                         // stores), 2 = any alignment (staged values copied out by the warp)
  uint32_t capv;         // values a unit may hold (the staging buffer's capacity)
  uint32_t cap;          // bytes per staging buffer (two per warp)
  uint32_t o_warp, o_ring, ring_bytes;
};

// Words per unit for capacity k: a multiple of 8 (unit starts stay 16-byte
// aligned for u16), WPU k <= UT values.
__device__ __forceinline__ uint32_t wpu_of(uint32_t ut, uint32_t k) {
  const uint32_t w = (ut / k) & ~7u;
  return w < 8 ? 8u : w;
}


// Words per unit of a valid BASIC block (capacity k, nw words): the whole
// block when its words fit a staging buffer (nw k <= capv values); else the
// fewest units of about ut values, as equal as a multiple of 8 words allows,
// when they fit; else WPU(k).  Passes 1 and 2 agree through the unit table.
__device__ __forceinline__ uint32_t unit_words(uint32_t ut, uint32_t capv, uint32_t k, uint32_t nw) {
  if ((uint64_t)nw * k <= capv) return (nw + 7) & ~7u;
  const uint32_t nu = (uint32_t)(((uint64_t)(nw - 1) * k + ut - 1) / ut);
  const uint32_t w = ((nw + nu - 1) / nu + 7) & ~7u;
  if ((uint64_t)w * k <= capv) return w;
  return wpu_of(ut, k);
}

// ------------------------------------------------------------------ checks
// Global header against the call's arguments (a9).  The
// length test cannot wrap: payload_bytes is compared with in_bytes minus the
// header bytes only after in_bytes is known to hold them.
__device__ __forceinline__ uint32_t hdr_check(const Args& a, uint64_t* pw) {
  *pw = 0;
  if (a.in_bytes < 32) return POLY_ST_LENGTH;
  const uint4 h0 = reinterpret_cast<const uint4*>(a.in)[0];
  const uint4 h1 = reinterpret_cast<const uint4*>(a.in)[1];
  const uint64_t n = (uint64_t)h0.z | ((uint64_t)h0.w << 32);
  const uint64_t pb = (uint64_t)h1.z | ((uint64_t)h1.w << 32);
  if (h0.x != 0x43594c50u) return POLY_ST_BAD_MAGIC;  // "PLYC"
  if ((h0.y & 0xffu) != 2u) return POLY_ST_BAD_VERSION;
  if (((h0.y >> 8) & 0xffu) != 0u || ((h0.y >> 16) & 0xffu) != a.width || (h0.y >> 24) != 0u || n != a.n ||
      h1.x != a.block_len || h1.y != (uint32_t)a.n_blocks)
    return POLY_ST_HEADER_MISMATCH;
  const uint64_t hb = 32 + 16 * a.n_blocks;
  if (a.in_bytes < hb || pb != a.in_bytes - hb || (pb & 7) != 0) return POLY_ST_LENGTH;
  *pw = pb >> 3;
  return 0;
}

__device__ __forceinline__ uint32_t block_len_of(const Args& a, uint64_t b) {
  return (uint32_t)(b + 1 == a.n_blocks ? a.last_len : a.Le);
}
// Words a block may claim in the offset scan: n_words clamped to the most any
// valid block of this length has (ceil(n_b / k_min)), so a corrupt header can
// neither wrap the sums nor move a later block out of the buffer.  Pass 2
// applies the same clamp, so both passes agree on every offset.
__device__ __forceinline__ uint32_t nw_clamp(const Args& a, uint32_t nw, uint32_t blen, uint32_t& err) {
  const uint32_t cap = (uint32_t)(((uint64_t)blen + (1u << a.kmin_log2) - 1) >> a.kmin_log2);
  if (nw > cap) {
    err |= POLY_ST_NWORDS;
    return cap;
  }
  return nw;
}

// Block header (a9) -> decode constants.  kind: 0 invalid, 1 CONSTANT, 2 BASIC.
struct Blk {
  uint64_t Rl, Rh, P;  // fraction reciprocal, top-word premultiplier B^(k - mtop)
  uint32_t bm1, vmin;
  uint32_t k, t32, add, b32, mtop, nw, kind;
};
constexpr uint32_t CACHE_B = 512;  // bases with shared-memory constants (blocks regime)
// Shared-memory cache entry of base B for full-length blocks (blen = Le):
// {Rl, Rh}, {P = B^(k - mtop), meta = k | t32 << 8 | mtop << 16 | add << 24, nwL}
struct __align__(16) CEnt {
  uint64_t Rl, Rh, P;
  uint32_t meta, nwL;
};
__device__ __forceinline__ Blk block_consts(const Args& a, uint4 h, uint32_t blen, uint32_t& err,
                                            const CEnt* cache = nullptr) {
  Blk c;
  c.Rl = c.Rh = 0;
  c.P = 1;
  c.bm1 = h.z;
  c.vmin = h.y;
  c.k = c.t32 = c.add = c.b32 = c.mtop = 0;
  c.nw = h.w;
  c.kind = 0;
  const uint64_t vmax = a.width == 32 ? 0xffffffffull : ((1ull << a.width) - 1);
  if (h.x == CODEC_CONSTANT) {
    uint32_t e = 0;
    if (h.z != 0 || h.w != 0) e |= POLY_ST_NWORDS;
    if ((uint64_t)h.y > vmax) e |= POLY_ST_OVERFLOW;
    err |= e;
    if (!e) c.kind = 1;
    return c;
  }
  if (h.x != CODEC_BASIC) {
    err |= POLY_ST_BAD_CODEC;
    return c;
  }
  if (h.z == 0 || (uint64_t)h.y + h.z > vmax) {
    err |= POLY_ST_OVERFLOW;
    return c;
  }
  const uint64_t B = (uint64_t)h.z + 1;
  if (cache && B < CACHE_B && blen == a.Le) {
    const uint4* e = reinterpret_cast<const uint4*>(cache + B);
    const uint4 e0 = e[0], e1 = e[1];
    if (h.w != e1.w) {
      err |= POLY_ST_NWORDS;
      return c;
    }
    c.Rl = (uint64_t)e0.x | ((uint64_t)e0.y << 32);
    c.Rh = (uint64_t)e0.z | ((uint64_t)e0.w << 32);
    c.P = (uint64_t)e1.x | ((uint64_t)e1.y << 32);
    c.k = e1.z & 0xffu;
    c.t32 = (e1.z >> 8) & 0xffu;
    c.mtop = (e1.z >> 16) & 0xffu;
    c.add = (e1.z >> 24) & 1u;
    c.kind = 2;
    return c;
  }
  DecConst d;
  if (B <= KTAB_MAX) {
    const uint4* p = reinterpret_cast<const uint4*>(&g_dtab[B]);
    const uint4 x = p[0], y = p[1];
    d.Wmax = (uint64_t)x.x | ((uint64_t)x.y << 32);
    d.Rl = (uint64_t)x.z | ((uint64_t)x.w << 32);
    d.Rh = (uint64_t)y.x | ((uint64_t)y.y << 32);
    d.meta = y.z;
  } else {
    d = dec_const_slow(B);
  }
  const uint32_t k = d.meta & 0xffu;
  // n_words must be ceil(n_b / k): (n_words - 1) k < n_b <= n_words k
  if (h.w == 0 || (uint64_t)(h.w - 1) * k >= blen || (uint64_t)h.w * k < blen) {
    err |= POLY_ST_NWORDS;
    return c;
  }
  c.k = k;
  c.t32 = (d.meta >> 16) & 0xffu;
  c.add = ((d.meta >> 8) & 0xffu) ? 0u : 1u;
  c.b32 = ((d.meta >> 8) & 0xffu) == 32u ? 1u : 0u;
  c.Rl = d.Rl;
  c.Rh = d.Rh;
  c.mtop = blen - (h.w - 1) * k;
  // P = B^(k - mtop) by squaring (k - mtop < k <= 64; B^(k - mtop) < 2^64)
  uint64_t P = 1, q = B;
  for (uint32_t e = k - c.mtop; e; e >>= 1) {
    if (e & 1) P *= q;
    if (e > 1) q *= q;
  }
  c.P = P;
  c.kind = 2;
  return c;
}

// ------------------------------------------------------------------ digits
// 64-bit fraction step with the block minimum folded in: returns
// vmin + floor(f B / 2^64) and sets f <- f B mod 2^64 (f = f1:f0).
__device__ __forceinline__ uint32_t fstep64(uint32_t& f0, uint32_t& f1, uint32_t B, uint32_t vmin) {
  uint32_t c, n0;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(c) : "r"(f0), "r"(B));
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(n0) : "r"(f0), "r"(B));
  uint64_t u;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(u) : "r"(f1), "r"(B), "l"(((uint64_t)vmin << 32) | c));
  f0 = n0;
  f1 = (uint32_t)u;
  return (uint32_t)(u >> 32);
}
// 32-bit step: returns vmin + floor(g B / 2^32), g <- g B mod 2^32.
__device__ __forceinline__ uint32_t fstep32(uint32_t& g, uint32_t B, uint32_t vmin) {
  uint32_t lo, d;
  asm("mul.lo.u32 %0, %2, %3;\n\tmad.hi.u32 %1, %2, %3, %4;" : "=&r"(lo), "=r"(d) : "r"(g), "r"(B), "r"(vmin));
  g = lo;
  return d;
}

// One word s of a block: m digits (m = k, or the block's last word mtop),
// written most significant first at top[0], top[-1], ..., top[1 - m].
// Returns POLY_ST_RESIDUE if s >= B^m (a9).  DESIGN.md Sec. 5.3: the word
// premultiplied by P = B^(k - m) has its m digits on top; f = floor(s R /
// 2^96) + add is its 64-bit binary fraction, s R >= 2^160 iff s >= B^k; the
// last t32 digits of the k take 32-bit steps.
template <typename V>
__device__ __forceinline__ uint32_t dec_word(uint64_t s, const Blk& c, uint32_t m, V* top) {
  uint32_t err = 0;
  if (c.b32) {  // B = 2^32 (u32 only): the digits are the two halves
    if (m == 2) {
      top[0] = (V)(c.vmin + (uint32_t)(s >> 32));
      top[-1] = (V)(c.vmin + (uint32_t)s);
    } else {
      if (s >> 32) err = POLY_ST_RESIDUE;
      top[0] = (V)(c.vmin + (uint32_t)s);
    }
    return err;
  }
  if (m < c.k) {
    if (__umul64hi(s, c.P) != 0) err = POLY_ST_RESIDUE;
    s *= c.P;
  }
  const uint64_t hi1 = __umul64hi(s, c.Rl), lo2 = s * c.Rh, hi2 = __umul64hi(s, c.Rh);
  const uint64_t mid = lo2 + hi1;
  const uint64_t t = hi2 + (mid < lo2 ? 1ull : 0ull);
  if (t >> 32) err = POLY_ST_RESIDUE;
  const uint64_t f = (t << 32) + (mid >> 32) + c.add;
  uint32_t f0 = (uint32_t)f, f1 = (uint32_t)(f >> 32);
  const uint32_t B = c.bm1 + 1, vmin = c.vmin;
  int n32 = (int)c.t32 + (int)m - (int)c.k;
  n32 = n32 < 0 ? 0 : n32;
  int n64 = (int)m - n32;
  V* o = top;
#pragma unroll 1
  for (; n64 >= 2; n64 -= 2, o -= 2) {
    const uint32_t d1 = fstep64(f0, f1, B, vmin);
    const uint32_t d0 = fstep64(f0, f1, B, vmin);
    o[0] = (V)d1;
    o[-1] = (V)d0;
  }
  if (n64) {
    o[0] = (V)fstep64(f0, f1, B, vmin);
    --o;
  }
  uint32_t g = f1 + c.add;
#pragma unroll 1
  for (; n32 >= 2; n32 -= 2, o -= 2) {
    const uint32_t d1 = fstep32(g, B, vmin);
    const uint32_t d0 = fstep32(g, B, vmin);
    o[0] = (V)d1;
    o[-1] = (V)d0;
  }
  if (n32) o[0] = (V)fstep32(g, B, vmin);
  return err;
}

// Two words at once (their own blocks' constants): two independent
// multiply chains per lane.  The common switch to 32-bit steps is the later
// of the two (a word may always take more 64-bit steps: they are exact, and
// fewer than t32 trailing 32-bit steps stay exact); digits past a word's m
// are computed but not stored.


// A word of capacity k from the table constants alone (no premultiplier):
// its m <= k digits are the last m of k steps; the first k - m (above the
// word's top digit) must be 0, else POLY_ST_RESIDUE (s >= B^m).  first[0..m)
// receives v_min + digits, lowest power first.
template <typename V>
__device__ __forceinline__ uint32_t dec_word_dc(uint64_t s, const DecConst& dc, uint32_t B, uint32_t vmin, uint32_t k,
                                                uint32_t m, V* first) {
  const uint32_t add = ((dc.meta >> 8) & 0xffu) ? 0u : 1u, t32 = (dc.meta >> 16) & 0xffu;
  uint32_t err = 0;
  const uint64_t hi1 = __umul64hi(s, dc.Rl), lo2 = s * dc.Rh, hi2 = __umul64hi(s, dc.Rh);
  const uint64_t mid = lo2 + hi1, t = hi2 + (mid < lo2 ? 1ull : 0ull);
  if (t >> 32) err = POLY_ST_RESIDUE;
  const uint64_t f = (t << 32) + (mid >> 32) + add;
  uint32_t f0 = (uint32_t)f, f1 = (uint32_t)(f >> 32), zero = 0;
  const uint32_t n64 = k - t32;  // steps before the 32-bit phase
  uint32_t i = 0;
#pragma unroll 1
  for (; i < n64; ++i) {
    const uint32_t d = fstep64(f0, f1, B, 0u);
    if (i < k - m) zero |= d;
    else first[k - 1 - i] = (V)(vmin + d);
  }
  uint32_t g = f1 + add;
#pragma unroll 1
  for (; i < k; ++i) {
    const uint32_t d = fstep32(g, B, 0u);
    if (i < k - m) zero |= d;
    else first[k - 1 - i] = (V)(vmin + d);
  }
  return (err | (zero ? POLY_ST_RESIDUE : 0u));
}

// ------------------------------------------------------------------ output
// Store the global byte range [c_lo, c_hi) from the staging buffer, whose
// byte x holds global byte G0 + x (G0 16-byte aligned): one TMA bulk store of
// the 16-byte aligned interior
// (issued by lane 0 into the warp's current bulk group; the caller commits
// and waits) and element stores for the partial chunks at the ends.  Every
// lane's staging writes are made visible to the async proxy first.
template <typename V>
__device__ __forceinline__ void store_out(const uint8_t* stg, uint64_t G0, uint64_t c_lo, uint64_t c_hi, int lane) {
  if (c_lo >= c_hi) return;
  const uint64_t a16 = (c_lo + 15) & ~15ull, b16 = c_hi & ~15ull;
  if (a16 < b16) {
    px::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) px::bulk_s2g(reinterpret_cast<void*>(a16), stg + (a16 - G0), (uint32_t)(b16 - a16));
    const uint32_t nh = (uint32_t)(a16 - c_lo) / sizeof(V), nt = (uint32_t)(c_hi - b16) / sizeof(V);
    if ((uint32_t)lane < nh) {
      reinterpret_cast<V*>(c_lo)[lane] = reinterpret_cast<const V*>(stg + (c_lo - G0))[lane];
    } else if ((uint32_t)lane < nh + nt) {
      const uint32_t e = lane - nh;
      reinterpret_cast<V*>(b16)[e] = reinterpret_cast<const V*>(stg + (b16 - G0))[e];
    }
  } else {
    const uint32_t ne = (uint32_t)(c_hi - c_lo) / sizeof(V);
    if ((uint32_t)lane < ne) reinterpret_cast<V*>(c_lo)[lane] = reinterpret_cast<const V*>(stg + (c_lo - G0))[lane];
  }
}

// u16 values staged from a 16-byte aligned address to a global address of
// any (2-byte) alignment: 8-byte stores of the 8-byte aligned interior, the
// word pairs funnel-shifted when the destination sits an odd number of values
// off a 4-byte boundary, and single values at the ends.
__device__ __forceinline__ void copy_out_u16(const uint8_t* stg, uint64_t gbase, uint32_t nv, int lane) {
  if (nv == 0) return;
  const uint16_t* s = reinterpret_cast<const uint16_t*>(stg);
  uint16_t* g = reinterpret_cast<uint16_t*>(gbase);
  const uint64_t gend = gbase + 2ull * nv;
  const uint64_t a8 = (gbase + 7) & ~7ull, b8 = gend & ~7ull;
  if (a8 >= b8) {  // fewer than 8 values
    if ((uint32_t)lane < nv) g[lane] = s[lane];
    return;
  }
  const uint32_t o = (uint32_t)(a8 - gbase);  // staging byte of the first aligned chunk: 0, 2, 4 or 6
  const uint32_t nch = (uint32_t)((b8 - a8) >> 3);
  const uint32_t* S = reinterpret_cast<const uint32_t*>(stg + (o & ~3u));
  uint2* G = reinterpret_cast<uint2*>(a8);
  if ((o & 2u) == 0) {
#pragma unroll 4
    for (uint32_t c = lane; c < nch; c += 32) G[c] = make_uint2(S[2 * c], S[2 * c + 1]);
  } else {
#pragma unroll 4
    for (uint32_t c = lane; c < nch; c += 32) {
      const uint32_t w0 = S[2 * c], w1 = S[2 * c + 1], w2 = S[2 * c + 2];
      G[c] = make_uint2(__funnelshift_r(w0, w1, 16), __funnelshift_r(w1, w2, 16));
    }
  }
  const uint32_t nh = o >> 1, nt = (uint32_t)(gend - b8) >> 1, t0 = (uint32_t)(b8 - gbase) >> 1;
  if ((uint32_t)lane < nh)
    g[lane] = s[lane];
  else if ((uint32_t)lane < nh + nt)
    g[t0 + lane - nh] = s[t0 + lane - nh];
}

// Fill the global byte range [g_lo, g_hi) with the value v (CONSTANT block).
template <typename V>
__device__ __forceinline__ void fill_out(uint64_t g_lo, uint64_t g_hi, uint32_t v, int lane) {
  if (g_lo >= g_hi) return;
  const uint32_t rep = sizeof(V) == 1 ? (v & 0xffu) * 0x01010101u : sizeof(V) == 2 ? ((v & 0xffffu) * 0x10001u) : v;
  const uint4 p = make_uint4(rep, rep, rep, rep);
  const uint64_t a16 = (g_lo + 15) & ~15ull, b16 = g_hi & ~15ull;
  if (a16 < b16) {
    const uint64_t nch = (b16 - a16) >> 4;
    for (uint64_t q = lane; q < nch; q += 32) px::st_v4(reinterpret_cast<void*>(a16 + 16 * q), p);
    const uint32_t nh = (uint32_t)(a16 - g_lo) / sizeof(V), nt = (uint32_t)(g_hi - b16) / sizeof(V);
    if ((uint32_t)lane < nh)
      reinterpret_cast<V*>(g_lo)[lane] = (V)v;
    else if ((uint32_t)lane < nh + nt)
      reinterpret_cast<V*>(b16)[lane - nh] = (V)v;
  } else {
    const uint32_t ne = (uint32_t)(g_hi - g_lo) / sizeof(V);
    if ((uint32_t)lane < ne) reinterpret_cast<V*>(g_lo)[lane] = (V)v;
  }
}

// ======================================================================
// pass 1: unit offsets
// ======================================================================
// Decoupled look-back over the chunks (tickets are handed out in order, so a
// chunk's predecessors are resident or done and the spin terminates).
__device__ __forceinline__ uint64_t chunk_lookback(const uint64_t* st, uint64_t c) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t base = (int64_t)c - 1;
  uint32_t ns = 0;
  while (true) {
    const int64_t idx = base - lane;
    const uint64_t v = idx >= 0 ? px::ld_relaxed(st + idx) : FLAG_PRE;
    const uint32_t pre = __ballot_sync(0xffffffffu, (v & FLAG_PRE) != 0);
    const uint32_t inval = __ballot_sync(0xffffffffu, (v >> 62) == 0);
    if (pre && (inval == 0 || __ffs(pre) < __ffs(inval))) {
      const int first = __ffs(pre) - 1;
      uint64_t x = lane <= first ? (v & VAL_MASK) : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      return excl + x;
    }
    if (inval) {
      if (ns) __nanosleep(ns);
      ns = ns ? min(ns * 2, 256u) : 32u;
      continue;
    }
    uint64_t x = v & VAL_MASK;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    excl += x;
    base -= 32;
  }
}

// ======================================================================
// pass 1: unit table
// ======================================================================
__device__ __forceinline__ uint32_t units_of(const Args& a, uint4 h, uint32_t blen, uint32_t nwc) {
  const uint64_t vmax = a.width == 32 ? 0xffffffffull : ((1ull << a.width) - 1);
  if (h.x == CODEC_BASIC && h.z != 0 && (uint64_t)h.y + h.z <= vmax) {
    const uint32_t k = capacity_of((uint64_t)h.z + 1);
    if (h.w != 0 && (uint64_t)(h.w - 1) * k < blen && (uint64_t)h.w * k >= blen) {
      const uint32_t w = unit_words(a.ut, a.capv, k, h.w);
      return (h.w + w - 1) / w;
    }
  }
  (void)nwc;
  return 1;  // CONSTANT or invalid block: one unit (fill / report)
}

__device__ __forceinline__ uint64_t cta_scan_inplace(uint64_t* v, uint32_t n, uint64_t* swarp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t q = (n + K1T - 1) / K1T;
  const uint32_t i0 = min((uint32_t)tid * q, n), i1 = min(i0 + q, n);
  uint64_t loc = 0;
  for (uint32_t i = i0; i < i1; ++i) loc += v[i];
  uint64_t x = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) swarp[warp] = x;
  __syncthreads();
  uint64_t wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += swarp[w];
  uint64_t run = wpre + x - loc;
  for (uint32_t i = i0; i < i1; ++i) {
    const uint64_t t = v[i];
    v[i] = run;
    run += t;
  }
  __syncthreads();
  uint64_t tot = 0;
  for (int w = 0; w < K1T / 32; ++w) tot += swarp[w];
  __syncthreads();
  return tot;
}

__global__ void __launch_bounds__(K1T) dec3_offsets(Args a) {
  __shared__ uint64_t s_w[CE], s_u[CE], swarp[K1T / 32];
  __shared__ uint64_t s_pw, s_pu;
  __shared__ uint32_t s_c, s_err;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t pw;
  const uint32_t herr = hdr_check(a, &pw);
  if (herr) {
    if (blockIdx.x == 0 && tid == 0) {
      atomicOr(a.status_out, herr);
      *a.abort_flag = 1;
    }
    return;
  }
  const uint4* H = reinterpret_cast<const uint4*>(a.in + 32);
  for (;;) {
    if (tid == 0) {
      s_c = atomicAdd(a.ticket, 1u);
      s_err = 0;
    }
    __syncthreads();
    const uint64_t c = s_c;
    if (c >= a.n_chunks) break;
    const uint64_t b0 = c * CE;
    const uint32_t ne = (uint32_t)min((uint64_t)CE, a.n_blocks - b0);
    uint32_t err = 0;
    for (uint32_t i = tid; i < ne; i += K1T) {
      const uint4 h = px::ld_v4(H + b0 + i);
      const uint32_t blen = block_len_of(a, b0 + i);
      const uint32_t nwc = nw_clamp(a, h.w, blen, err);
      s_w[i] = nwc;
      s_u[i] = units_of(a, h, blen, nwc);
    }
    __syncthreads();
    const uint64_t tw = cta_scan_inplace(s_w, ne, swarp);
    const uint64_t tu = cta_scan_inplace(s_u, ne, swarp);
    if (warp == 0) {
      uint64_t pre_w = 0, pre_u = 0;
      if (c == 0) {
        if (lane == 0) {
          px::st_relaxed(a.cst_w, FLAG_PRE | (tw & VAL_MASK));
          px::st_relaxed(a.cst_u, FLAG_PRE | (tu & VAL_MASK));
        }
      } else {
        if (lane == 0) {
          px::st_relaxed(a.cst_w + c, FLAG_AGG | (tw & VAL_MASK));
          px::st_relaxed(a.cst_u + c, FLAG_AGG | (tu & VAL_MASK));
        }
        pre_w = chunk_lookback(a.cst_w, c);
        if (lane == 0) px::st_relaxed(a.cst_w + c, FLAG_PRE | ((pre_w + tw) & VAL_MASK));
        pre_u = chunk_lookback(a.cst_u, c);
        if (lane == 0) px::st_relaxed(a.cst_u + c, FLAG_PRE | ((pre_u + tu) & VAL_MASK));
      }
      if (lane == 0) {
        s_pw = pre_w;
        s_pu = pre_u;
      }
    }
    __syncthreads();
    const uint64_t Pw = s_pw, Pu = s_pu;
    const bool last = c + 1 == a.n_chunks;
    if (!last || Pu + tu <= a.max_units) {
      for (uint32_t i = tid; i < ne; i += K1T) {
        const uint64_t nu = (i + 1 < ne ? s_u[i + 1] : tu) - s_u[i];
        const uint4 h = px::ld_v4(H + b0 + i);
        const uint32_t blen = block_len_of(a, b0 + i);
        uint32_t w = 0;
        if (nu > 1) {  // a valid BASIC block (units_of)
          const uint32_t k = capacity_of((uint64_t)h.z + 1);
          w = unit_words(a.ut, a.capv, k, h.w);
        }
        (void)blen;
        const uint64_t u0 = Pu + s_u[i], ws = Pw + s_w[i];
        for (uint64_t u = 0; u < nu && u0 + u < a.max_units; ++u) {
          const uint64_t j0 = u * w, wst = ws + j0;
          a.T[u0 + u] = make_uint4((uint32_t)(b0 + i), (uint32_t)j0, (uint32_t)wst, (uint32_t)(wst >> 32));
        }
      }
    }
    if (last && tid == 0) {
      const uint64_t U = Pu + tu, W = Pw + tw;
      if (W != pw || U > a.max_units) {
        err |= POLY_ST_LENGTH;
        *a.abort_flag = 1;
      } else {
        a.T[U] = make_uint4((uint32_t)a.n_blocks, 0u, (uint32_t)W, (uint32_t)(W >> 32));
        *a.n_units = U;
      }
    }
    if (err) atomicOr(&s_err, err);
    __syncthreads();
    if (tid == 0 && s_err) atomicOr(a.status_out, s_err);
  }
}

// ======================================================================
// pass 2: decode
// ======================================================================
struct Slot {
  uint64_t ws;    // first payload word loaded
  uint64_t we;    // payload word after the tile's last unit
  uint64_t hb0;   // first block whose header is staged
  uint32_t off_t, off_h, off_p;  // ring byte offsets: table entries, headers, payload word ws
  uint32_t nu;
};
struct __align__(16) Ctl {
  uint64_t full[NSLOT], empty[NSLOT];
  uint64_t send[NSLOT];
  Slot slot[NSLOT];
  uint32_t next_unit;
};

__device__ __forceinline__ uint64_t ws_of(uint4 e) { return (uint64_t)e.z | ((uint64_t)e.w << 32); }

template <typename V>
__global__ void __launch_bounds__(NTHR, 1) dec3_main(Args a) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ctl& C = *reinterpret_cast<Ctl*>(smem);
  uint8_t* ring = smem + a.o_ring;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      px::mbar_init(&C.full[s], 1);
      px::mbar_init(&C.empty[s], TU);
    }
    px::mbar_fence_init();
    C.next_unit = 0;
  }
  __syncthreads();
  {
    uint64_t pw;
    if (hdr_check(a, &pw) != 0 || *reinterpret_cast<volatile uint32_t*>(a.abort_flag) != 0) return;
  }
  const uint64_t U = *reinterpret_cast<volatile uint64_t*>(a.n_units);
  const uint64_t n_tiles = (U + TU - 1) / TU;
  const uint64_t pay_byte0 = 32 + 16 * a.n_blocks;

  if (warp == NW) {
    // ------------------------------------------------------------ producer
    // The unit-table entries that bound each tile (first unit, last unit,
    // the unit after) are loaded PFD tiles ahead (a register queue), so their
    // latency overlaps the waits and copies of the tiles before.
    if (lane != 0) return;
    PROBE_DECL;
    PROBE_T0(pt0);
    const uint32_t RB = a.ring_bytes;
    uint64_t head = 0, tail = 0, rc = 0, it = 0;
    uint32_t hpos = 0;
    uint4 q0[PFD], ql[PFD], qn[PFD];
#pragma unroll
    for (int i = 0; i < PFD; ++i) {
      const uint64_t tl = blockIdx.x + (uint64_t)i * gridDim.x;
      q0[i] = ql[i] = qn[i] = make_uint4(0, 0, 0, 0);
      if (tl < n_tiles) {
        const uint64_t v0 = tl * TU, v1 = min(v0 + TU, U);
        q0[i] = px::ld_v4(a.T + v0);
        ql[i] = px::ld_v4(a.T + v1 - 1);
        qn[i] = px::ld_v4(a.T + v1);
      }
    }
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const uint4 e0 = q0[0], el = ql[0], en = qn[0];
#pragma unroll
      for (int i = 0; i + 1 < PFD; ++i) {
        q0[i] = q0[i + 1];
        ql[i] = ql[i + 1];
        qn[i] = qn[i + 1];
      }
      const uint64_t tn = t + (uint64_t)PFD * gridDim.x;
      if (tn < n_tiles) {
        const uint64_t v0 = tn * TU, v1 = min(v0 + TU, U);
        q0[PFD - 1] = px::ld_v4(a.T + v0);
        ql[PFD - 1] = px::ld_v4(a.T + v1 - 1);
        qn[PFD - 1] = px::ld_v4(a.T + v1);
      }
      const uint64_t u0 = t * TU, u1 = min(u0 + TU, U);
      const uint32_t nu = (uint32_t)(u1 - u0);
      const uint64_t ws = ws_of(e0), we = ws_of(en);
      const uint64_t hb0 = e0.x, hb1 = (uint64_t)el.x + 1;
      const uint64_t pa = pay_byte0 + 8 * ws, pe = pay_byte0 + 8 * we;
      const uint64_t pa16 = pa & ~15ull;
      uint64_t pe16 = (pe + 15) & ~15ull;
      uint32_t tailw = 0;
      if (pe16 > a.in_bytes) {
        pe16 -= 16;
        tailw = 1;
      }
      const uint32_t bt = 16 * nu, bh = (uint32_t)(16 * (hb1 - hb0));
      const uint32_t bp = (uint32_t)(pe16 - pa16) + 16 * tailw;
      const uint32_t need = bt + bh + bp;
      PROBE_T0(pw0);
      while (it - rc >= NSLOT) {
        const uint32_t s = (uint32_t)(rc % NSLOT);
        px::mbar_wait(&C.empty[s], (uint32_t)(rc / NSLOT) & 1u);
        tail = C.send[s];
        ++rc;
      }
      uint32_t pos = hpos;  // head modulo the ring size, kept incrementally
      if (pos + need > RB) {
        head += RB - pos;
        pos = 0;
      }
      hpos = pos + need;
      while (head + need - tail > RB) {
        const uint32_t s = (uint32_t)(rc % NSLOT);
        px::mbar_wait(&C.empty[s], (uint32_t)(rc / NSLOT) & 1u);
        tail = C.send[s];
        ++rc;
      }
      PROBE_ADD(5, pw0);
      const uint32_t s = (uint32_t)(it % NSLOT);
      Slot& S = C.slot[s];
      S.ws = ws;
      S.we = we;
      S.hb0 = hb0;
      S.nu = nu;
      S.off_t = pos;
      S.off_h = pos + bt;
      S.off_p = pos + bt + bh + (uint32_t)(pa - pa16);
      head += need;
      C.send[s] = head;
      uint8_t* dst = ring + pos;
      if (tailw)
        *reinterpret_cast<uint64_t*>(dst + bt + bh + (pe16 - pa16)) = *reinterpret_cast<const uint64_t*>(a.in + pe - 8);
      px::mbar_arrive_tx(&C.full[s], bt + bh + (uint32_t)(pe16 - pa16));
      px::bulk_g2s(dst, a.T + u0, bt, &C.full[s]);
      px::bulk_g2s(dst + bt, a.in + 32 + 16 * hb0, bh, &C.full[s]);
      if (pe16 > pa16) px::bulk_g2s(dst + bt + bh, a.in + pa16, (uint32_t)(pe16 - pa16), &C.full[s]);
    }
    PROBE_ADD(4, pt0);
    PROBE_FLUSH;
    return;
  }

  // -------------------------------------------------------------- consumers
  // two staging buffers per warp: a unit is decoded into one while the TMA
  // store of the previous unit reads the other
  uint8_t* const stg2 = smem + a.o_warp + (size_t)warp * 2 * a.cap;
  uint32_t bi = 0;
  uint32_t err = 0;
  // the next unit is claimed as soon as the current one is known, so the
  // shared-memory atomic's latency hides behind the decode
  uint32_t qn = 0;
  PROBE_DECL;
  PROBE_T0(ct0);
  if (lane == 0) qn = atomicAdd(&C.next_unit, 1u);
  for (;;) {
    const uint32_t q = __shfl_sync(0xffffffffu, qn, 0);
    const uint64_t it = q / TU;
    const uint32_t wi = q % TU;
    if (blockIdx.x + it * gridDim.x >= n_tiles) break;
    if (lane == 0) qn = atomicAdd(&C.next_unit, 1u);
    const uint32_t s = (uint32_t)(it % NSLOT);
    PROBE_T0(cw0);
    px::mbar_wait(&C.full[s], (uint32_t)(it / NSLOT) & 1u);
    PROBE_ADD(1, cw0);
    PROBE_T0(cd0);
    const Slot& S = C.slot[s];
    uint8_t* const stg = stg2 + bi * a.cap;
    bi ^= 1u;
    if (lane == 0) px::bulk_wait_read<1>();  // this buffer's previous store has read it
    __syncwarp();
    if (wi < S.nu) {
      const uint4* TE = reinterpret_cast<const uint4*>(ring + S.off_t);
      const uint4 e = TE[wi];
      const uint64_t b = e.x, wst = ws_of(e);
      const uint64_t wend = wi + 1 < S.nu ? ws_of(TE[wi + 1]) : S.we;
      const uint32_t nwu = (uint32_t)(wend - wst), j0 = e.y;
      const uint64_t* PAY = reinterpret_cast<const uint64_t*>(ring + S.off_p) + (wst - S.ws);
      const uint4 h = reinterpret_cast<const uint4*>(ring + S.off_h)[b - S.hb0];
      const uint32_t blen = block_len_of(a, b);
      const uint64_t gblk = reinterpret_cast<uint64_t>(a.out) + b * a.Le * sizeof(V);
      const uint32_t B = h.z + 1;
      // fast path: a valid u16 BASIC block that starts 16-byte aligned, a
      // capacity with a k-specialised group codec; the header checks of
      // block_consts, in its order, without the premultiplier
      bool fast = false;
      if (sizeof(V) == 2 && a.kw_ok && h.x == CODEC_BASIC && h.z != 0 && h.y + h.z <= 0xffffu) {
        const DecConst dc = g_dtab[B];
        const uint32_t k = dc.meta & 0xffu, nw = h.w;
        const bool nw_ok = nw != 0 && (nw - 1) * k < blen && nw * k >= blen;
        if (nw_ok && k >= 4 && k <= 27 && k != 23 && k != 25 && k != 26) {
          fast = true;
          const uint32_t j1 = j0 + nwu, mtop = blen - (nw - 1) * k;
          const uint64_t gbase = gblk + (uint64_t)j0 * k * 2;  // kw_ok 1: 16-byte aligned (j0 % 8 == 0)
          uint8_t* blk = stg - 2ull * j0 * k;                 // block value 0 in staging coordinates
          const uint32_t lj = dc_log2b(dc);
          const bool p2 = lj != 0;
          uint32_t jdone = j0;
          switch (k) {
#define POLY_D3K(KK)                                                                             \
  case KK: {                                                                                     \
    /* the group codec's power-of-two path is for B = 2^(64 / KK); the other \
       power-of-two bases of capacity KK (2^11 for 5, 2^13..2^15 for 4) go  \
       word by word below.  The groups cover every word of the unit: an odd \
       last word is paired with a zero word, and the block's short top word \
       is decoded like a full one (checked against B^mtop below) */         \
    const uint32_t gb = j0 / kq<KK>();                                                           \
    const uint32_t ge = (!p2 || lj == 64 / KK) ? (j1 + kq<KK>() - 1) / kq<KK>() : gb;            \
    if (ge > gb) {                                                                               \
      err |= p2 ? unpack_groups_kp<KK, true>(PAY - j0, gb, ge, j1, dc, B, h.y, blk)              \
                : unpack_groups_kp<KK, false>(PAY - j0, gb, ge, j1, dc, B, h.y, blk);            \
      jdone = j1;                                                                                \
    }                                                                                            \
  } break;
            POLY_FOR_EACH_K16(POLY_D3K)
#undef POLY_D3K
            default:
              break;
          }
          if (jdone != j1) {
            for (uint32_t j = jdone + lane; j < j1; j += 32) {  // capacities / bases without a group codec
              const uint32_t m = (j + 1 == nw) ? mtop : k;
              err |= dec_word_dc<V>(PAY[j - j0], dc, B, h.y, k, m, reinterpret_cast<V*>(stg) + (j - j0) * k);
            }
          }
          __syncwarp();
          // a9 for a short top word decoded by the group codec: s < B^mtop, i.e.
          // its k - mtop digits past the block's end (staged as v_min + digit,
          // never copied out) are 0
          if (jdone == j1 && j1 == nw && (uint32_t)lane < k - mtop &&
              reinterpret_cast<const V*>(blk)[blen + lane] != (V)h.y)
            err |= POLY_ST_RESIDUE;
          const uint32_t nv = min(blen, j1 * k) - j0 * k;
          PROBE_ADD(2, cd0);
          PROBE_T0(cc0);
          if (a.kw_ok == 1)
            store_out<V>(stg, gbase, gbase, gbase + (uint64_t)nv * 2, lane);
          else
            copy_out_u16(stg, gbase, nv, lane);
          PROBE_ADD(3, cc0);
        }
      }
      if (!fast) {
        uint32_t e1 = 0;
        nw_clamp(a, h.w, blen, e1);
        const Blk c = block_consts(a, h, blen, e1);
        if (j0 == 0) err |= e1;  // reported once per block
        if (c.kind == 1) {
          fill_out<V>(gblk, gblk + (uint64_t)blen * sizeof(V), c.vmin, lane);
        } else if (c.kind == 2) {
          const uint32_t k = c.k, j1 = j0 + nwu;
          const uint64_t gbase = gblk + (uint64_t)j0 * k * sizeof(V);
          const uint64_t G0 = gbase & ~15ull;
          V* stgv = reinterpret_cast<V*>(stg + (gbase - G0));  // staging value t <-> block value j0 k + t
          for (uint32_t j = j0 + lane; j < j1; j += 32) {
            const uint32_t m = (j + 1 == c.nw) ? c.mtop : k;
            err |= dec_word<V>(PAY[j - j0], c, m, stgv + (j - j0) * k + (m - 1));
          }
          __syncwarp();
          const uint32_t nv = (uint32_t)min((uint64_t)blen, (uint64_t)j1 * k) - j0 * k;
          store_out<V>(stg, G0, gbase, gbase + (uint64_t)nv * sizeof(V), lane);
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      px::mbar_arrive(&C.empty[s]);
      px::bulk_commit();  // one bulk group per unit (possibly empty)
    }
#ifdef POLY_PROBE
    pacc[7] += 1;
#endif
  }
  PROBE_ADD(0, ct0);
  PROBE_FLUSH;
  if (lane == 0) px::bulk_wait_all<0>();  // the stores have read the staging (and landed)
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0 && err) atomicOr(a.status_out, err);
}

}  // namespace d3
}  // namespace polyk

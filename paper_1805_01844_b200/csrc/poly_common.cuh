// poly_common.cuh -- shared device pieces of the sm_100a polynomial codec:
// launch constants, the B -> k / reciprocal tables,
// global-memory access helpers and the single-pass decoupled look-back scan
// (a4).  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/poly.h"

namespace polyk {

constexpr int NT = 256;                 // threads per CTA (8 warps)
constexpr int NWARP = NT / 32;
constexpr uint32_t CH_VALUES = 8192;    // values per chunk in the large-block regime
constexpr uint32_t KTAB_MAX = 65536;    // B <= KTAB_MAX use the tables

// look-back status word: [63:62] flag, [61:0] value
constexpr uint64_t FLAG_AGG = 1ull << 62;
constexpr uint64_t FLAG_PRE = 2ull << 62;
constexpr uint64_t VAL_MASK = (1ull << 62) - 1;

constexpr uint32_t CODEC_CONSTANT = 1;
constexpr uint32_t CODEC_BASIC = 2;

// Per-base constants.  k = max{k : B^k <= 2^64} (Eq. 1,
// reading R2) and h = max{h : B^h <= 2^32} (32-bit chunk length).  The
// decoder's binary fraction of a word s < B^k is f = floor(s R / 2^96) + add:
//   non-power-of-two B: R = ceil(2^160 / B^k) (< 2^128), add = 1;
//   B = 2^j:            R = 2^(160 - kj) (exact),      add = 0.
// Wmax = B^k - 1 is the largest valid word; t32 = the number of trailing
// digits of a word that may be extracted with a 32-bit fraction (Sec. 5.3).
struct __align__(16) DecConst {
  uint64_t Wmax;
  uint64_t Rl;
  uint64_t Rh;
  uint32_t meta;  // k | log2b << 8 | t32 << 16 | h << 24
  uint32_t pad;
};
__device__ __forceinline__ uint32_t dc_k(const DecConst& c) { return c.meta & 0xffu; }
__device__ __forceinline__ uint32_t dc_log2b(const DecConst& c) { return (c.meta >> 8) & 0xffu; }
__device__ __forceinline__ uint32_t dc_t32(const DecConst& c) { return (c.meta >> 16) & 0xffu; }
__device__ __forceinline__ uint32_t dc_add(const DecConst& c) { return ((c.meta >> 8) & 0xffu) ? 0u : 1u; }

// Filled once per device by poly_init (host computes them with exact 128-bit
// integer arithmetic).  g_ktab[B] = k | h << 8.
__device__ uint16_t g_ktab[KTAB_MAX + 1];
__device__ DecConst g_dtab[KTAB_MAX + 1];

// ---------------------------------------------------------------- arithmetic
// k and h for any 2 <= B <= 2^32 (B^3 <= 2^64 iff B <= 2642245; B^2 <= 2^32 iff
// B <= 65536).
__device__ __forceinline__ uint32_t capacity_of(uint64_t B) {
  if (B <= KTAB_MAX) return g_ktab[B] & 0xffu;
  return B <= 2642245ull ? 3u : 2u;
}
__device__ __forceinline__ void capacity_kh(uint64_t B, uint32_t& k, uint32_t& h) {
  if (B <= KTAB_MAX) {
    const uint32_t e = g_ktab[B];
    k = e & 0xffu;
    h = e >> 8;
  } else {
    k = B <= 2642245ull ? 3u : 2u;
    h = 1u;
  }
}

// ceil(2^160 / D) for D not a power of two, D >= 3 (slow path for B > 2^16):
// restoring long division, 161 quotient bits, result < 2^128.
__device__ __noinline__ void recip160(uint64_t D, uint64_t& Rl, uint64_t& Rh) {
  unsigned __int128 rem = 0, q = 0;
  for (int i = 160; i >= 0; --i) {
    rem = (rem << 1) | (i == 160 ? 1u : 0u);
    q <<= 1;
    if (rem >= D) {
      rem -= D;
      q |= 1;
    }
  }
  q += 1;  // D is not a power of two, so the remainder is nonzero: ceil = floor + 1
  Rl = (uint64_t)q;
  Rh = (uint64_t)(q >> 64);
}

__device__ __noinline__ DecConst dec_const_slow(uint64_t B) {
  DecConst c;
  const uint32_t k = B <= 2642245ull ? 3u : 2u;
  const uint32_t log2b = ((B & (B - 1)) == 0) ? (uint32_t)(63 - __clzll(B)) : 0u;
  c.Wmax = 0; c.Rl = 0; c.Rh = 0; c.pad = 0;
  uint32_t t32 = 0;
  if (!log2b) {
    uint64_t p = 1;
    for (uint32_t i = 0; i < k; ++i) p *= B;
    c.Wmax = p - 1;
    recip160(p, c.Rl, c.Rh);
    // t32 <= h = 1: one trailing 32-bit digit iff 2^32 B^k + B^k + 2^64 B <= 2^96
    const unsigned __int128 lhs = ((unsigned __int128)p << 32) + p + ((unsigned __int128)B << 64);
    if (lhs <= ((unsigned __int128)1 << 96)) t32 = 1;
  } else {  // B = 2^j, 17 <= j <= 32: exact fraction, R = 2^(160 - kj)
    const uint32_t kj = k * log2b;
    c.Wmax = kj >= 64 ? ~0ull : ((1ull << kj) - 1);
    const uint32_t e = 160 - kj;  // 96 .. 109
    c.Rh = 1ull << (e - 64);
    t32 = 32 / log2b;
  }
  c.meta = k | (log2b << 8) | (t32 << 16) | (1u << 24);
  return c;
}

__device__ __forceinline__ DecConst dec_const_of(uint64_t B) {
  if (B <= KTAB_MAX) return g_dtab[B];
  return dec_const_slow(B);
}

// ---------------------------------------------------------------- memory
__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint64_t ldg_nc_u64(const void* p) {
  uint64_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ void stg_cs_v4(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------- warp/CTA
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exclusive scan of in[0..count) into out[0..count) over the CTA; returns the
// total.  Every thread must call it.  s_warp: NWARP entries of scratch.
template <typename T>
__device__ T cta_exclusive_scan(const T* in, T* out, uint32_t count, T* s_warp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t q = (count + NT - 1) / NT;
  const uint32_t i0 = min((uint32_t)tid * q, count), i1 = min(i0 + q, count);
  T local = 0;
  for (uint32_t i = i0; i < i1; ++i) local += in[i];
  T x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < NWARP ? s_warp[lane] : (T)0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NWARP) s_warp[lane] = w;
  }
  __syncthreads();
  T excl = x - local + (warp > 0 ? s_warp[warp - 1] : (T)0);
  const T total = s_warp[NWARP - 1];
  for (uint32_t i = i0; i < i1; ++i) {
    T v = in[i];
    out[i] = excl;
    excl += v;
  }
  __syncthreads();
  return total;
}

// Decoupled look-back (single-pass scan): called by all 32 lanes of one warp
// for `tile` >= 1 after the tile published its aggregate; returns the
// exclusive prefix of the tile (same value in every lane).  Tiles are handed
// out in order by an atomic ticket, so every predecessor is resident or done
// and the spin terminates.
// Lane l inspects tile (base - l); the window resolves as soon as the nearest
// published inclusive prefix is closer than the nearest unpublished tile, so
// a slow tile further back never delays its successors.  Unresolved windows
// are re-read with a growing back-off to keep the spin off the L2.
__device__ __forceinline__ uint64_t lookback(const uint64_t* status, uint64_t tile) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t base = (int64_t)tile - 1;
  uint32_t ns = 0;
  while (true) {
    const int64_t idx = base - lane;
    const uint64_t st = idx >= 0 ? ld_relaxed_u64(status + idx) : FLAG_PRE;  // before tile 0: 0
    const uint32_t pre = __ballot_sync(0xffffffffu, (st & FLAG_PRE) != 0);
    const uint32_t inval = __ballot_sync(0xffffffffu, (st >> 62) == 0);
    if (pre && (inval == 0 || __ffs(pre) < __ffs(inval))) {
      const int first = __ffs(pre) - 1;
      return excl + warp_sum_u64(lane <= first ? (st & VAL_MASK) : 0ull);
    }
    if (inval) {
      if (ns) __nanosleep(ns);
      ns = ns ? min(ns * 2, 1024u) : 32u;
      continue;
    }
    excl += warp_sum_u64(st & VAL_MASK);
    base -= 32;
  }
}

// Wide decoupled look-back: 32 lanes x LB_PER tiles per window read (the
// window must outgrow (tile rate x L2 round trip), or the walk to the nearest
// inclusive prefix lengthens with the number of tiles in flight).  Same
// contract as lookback(): all 32 lanes call it for tile >= 1 after the tile
// published its aggregate; returns the exclusive prefix in every lane.
constexpr int LB_PER = 8;
__device__ __forceinline__ uint64_t lookback_wide(const uint64_t* status, uint64_t tile) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t base = (int64_t)tile - 1;  // lane l covers base - LB_PER*l - j, j = 0..LB_PER-1
  uint32_t ns = 0;
  // Cheap wait first: one lane polls the predecessor's status word until it
  // is published (statuses appear roughly in tile order, so by then most of
  // the window is valid); the wide reads below then rarely repeat.
  if (lane == 0) {
    uint32_t w = 0;
    while (ld_relaxed_u64(status + base) == 0) {
      if (w) __nanosleep(w);
      w = w ? min(w * 2, 256u) : 32u;
    }
  }
  __syncwarp();
  while (true) {
    uint64_t e[LB_PER];
    const int64_t top = base - (int64_t)LB_PER * lane;
#pragma unroll
    for (int j = 0; j < LB_PER; ++j) {
      const int64_t idx = top - j;
      e[j] = idx >= 0 ? ld_relaxed_u64(status + idx) : FLAG_PRE;  // before tile 0: prefix 0
    }
    uint32_t fpre = LB_PER, finv = LB_PER;
#pragma unroll
    for (int j = LB_PER - 1; j >= 0; --j) {
      if (e[j] & FLAG_PRE) fpre = j;
      if ((e[j] >> 62) == 0) finv = j;
    }
    const uint32_t bpre = __ballot_sync(0xffffffffu, fpre < LB_PER);
    const uint32_t binv = __ballot_sync(0xffffffffu, finv < LB_PER);
    const int lp = bpre ? __ffs(bpre) - 1 : 32, li = binv ? __ffs(binv) - 1 : 32;
    const uint32_t ppre = bpre ? LB_PER * lp + __shfl_sync(0xffffffffu, fpre, lp) : 0xffffffffu;
    const uint32_t pinv = binv ? LB_PER * li + __shfl_sync(0xffffffffu, finv, li) : 0xffffffffu;
    if (bpre && ppre < pinv) {
      uint64_t sum = 0;
#pragma unroll
      for (int j = 0; j < LB_PER; ++j)
        if ((uint32_t)(LB_PER * lane + j) <= ppre) sum += e[j] & VAL_MASK;
      return excl + warp_sum_u64(sum);
    }
    if (binv) {
      if (ns) __nanosleep(ns);
      ns = ns ? min(ns * 2, 256u) : 32u;
      continue;
    }
    uint64_t sum = 0;
#pragma unroll
    for (int j = 0; j < LB_PER; ++j) sum += e[j] & VAL_MASK;
    excl += warp_sum_u64(sum);
    base -= 32 * LB_PER;
  }
}

__device__ __forceinline__ uint32_t shfl_min(uint32_t v, int w) {
  for (int o = w >> 1; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ uint32_t shfl_max(uint32_t v, int w) {
  for (int o = w >> 1; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Copy nv values of type V from global g to shared s (16-byte vector loads
// when g is 16-byte aligned, scalar otherwise and for the tail).
template <typename V>
__device__ __forceinline__ void load_values(V* s, const V* g, uint32_t nv) {
  const int tid = threadIdx.x;
  const uint32_t nbytes = nv * (uint32_t)sizeof(V);
  uint32_t done = 0;
  if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    const uint32_t n16 = nbytes >> 4;
    const uint8_t* gb = reinterpret_cast<const uint8_t*>(g);
    uint4* sb = reinterpret_cast<uint4*>(s);
#pragma unroll 4
    for (uint32_t i = tid; i < n16; i += NT) sb[i] = ldg_nc_v4(gb + 16ull * i);
    done = (n16 << 4) / (uint32_t)sizeof(V);
  }
  for (uint32_t i = done + tid; i < nv; i += NT) s[i] = g[i];
}

// Copy nv values from shared s to global g (16-byte stores when aligned).
template <typename V>
__device__ __forceinline__ void store_values(V* g, const V* s, uint32_t nv) {
  const int tid = threadIdx.x;
  uint32_t done = 0;
  if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    const uint32_t n16 = (nv * (uint32_t)sizeof(V)) >> 4;
    uint8_t* gb = reinterpret_cast<uint8_t*>(g);
    const uint4* sb = reinterpret_cast<const uint4*>(s);
#pragma unroll 4
    for (uint32_t i = tid; i < n16; i += NT) stg_cs_v4(gb + 16ull * i, sb[i]);
    done = (n16 << 4) / (uint32_t)sizeof(V);
  }
  for (uint32_t i = done + tid; i < nv; i += NT) g[i] = s[i];
}

// Launch-time description of one call (identical for the compress and the
// decompress side; see poly_api.cu plan()).
struct Shape {
  uint64_t n;
  uint64_t Le;          // effective block length
  uint64_t n_blocks;
  uint32_t block_len;   // as given (0 = whole), stored in the global header
  uint32_t width;       // 16 or 32
  uint64_t cpb;         // chunks per block (large regime)
  uint64_t n_chunks;    // large regime
  uint64_t n_stiles;    // scan tiles over blocks (large regime)
};

}  // namespace polyk

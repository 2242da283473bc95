// poly_warp.cuh -- warp-tile kernels (blocks of up to WT_MAX bytes).
//
// Each warp owns one look-back unit: a run of consecutive blocks of the
// stream, handed out in order by an atomic ticket.  No CTA barrier is used:
// a warp stages its unit in its own shared-memory slice, computes the
// per-block statistics, scans its word counts with shuffles, publishes its
// aggregate, looks back for its payload offset, then writes headers and
// words straight to global memory (coalesced 8-byte word stores in the
// lanes-per-block mode, 16-byte header stores).
//
// Two mappings (chosen on the host, see poly.cu plan()):
//   MODE_LANE  (block <= 128 B, e.g. cfg2's 30 x u16): lane l owns blocks
//              l, l+32, ... of the unit (BPL blocks per lane).
//   MODE_WARP  (128 B < block <= WT_MAX): the 32 lanes cooperate on each
//              block; WB blocks per unit; lane l owns words l, l+32, ...
#pragma once
#include "poly_common.cuh"

namespace polyk {

constexpr int WARPS = 4;               // warps per CTA (independent)
constexpr uint32_t WT_MAX = 8192;      // bytes of input per warp unit
constexpr uint32_t LANE_BLOCK_MAX = 128;

struct WarpShape {
  uint64_t n, Le, n_blocks;
  uint32_t block_len, width;
  uint32_t WB;        // blocks per unit
  uint32_t mode;      // 0 lane, 1 warp
  uint32_t slice;     // smem bytes per warp (16-aligned)
  uint64_t n_units;
};

struct WarpArgs {
  const uint8_t* in;        // compress: values; decompress: stream
  uint8_t* out;             // compress: stream;  decompress: values
  uint64_t* compressed_bytes;
  uint64_t in_bytes;        // decompress: stream length
  uint32_t* status_out;     // decompress: caller's status word
  uint64_t* status;         // look-back words, one per unit
  uint32_t* ticket;
  WarpShape sh;
};

__device__ __forceinline__ uint32_t warp_ticket(uint32_t* ticket) {
  uint32_t t = 0;
  if ((threadIdx.x & 31) == 0) t = atomicAdd(ticket, 1u);
  return __shfl_sync(0xffffffffu, t, 0);
}

// Look-back for a warp unit: publish the aggregate, fetch the exclusive
// prefix, publish the inclusive prefix.  All lanes return the prefix.
__device__ __forceinline__ uint64_t warp_publish_and_lookback(uint64_t* status, uint64_t unit,
                                                             uint64_t total) {
  const int lane = threadIdx.x & 31;
  if (unit == 0) {
    if (lane == 0) st_relaxed_u64(status, FLAG_PRE | (total & VAL_MASK));
    return 0;
  }
  if (lane == 0) st_relaxed_u64(status + unit, FLAG_AGG | (total & VAL_MASK));
  const uint64_t p = lookback(status, unit);
  if (lane == 0) st_relaxed_u64(status + unit, FLAG_PRE | ((p + total) & VAL_MASK));
  return p;
}

// Copy nbytes from global g to this warp's smem slice s (16-byte vectors when
// both are aligned, bytes otherwise).  Caller issues __syncwarp() after.
__device__ __forceinline__ void warp_copy_in(uint8_t* s, const uint8_t* g, uint32_t nbytes) {
  const int lane = threadIdx.x & 31;
  uint32_t done = 0;
  const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(g) & 15);
  if (mis == 0) {
    const uint32_t n16 = nbytes >> 4;
    const uint4* gv = reinterpret_cast<const uint4*>(g);
    uint4* sv = reinterpret_cast<uint4*>(s);
    uint32_t i = lane;
    for (; i + 96 < n16; i += 128) {
      const uint4 a = ldg_nc_v4(gv + i), b = ldg_nc_v4(gv + i + 32), c = ldg_nc_v4(gv + i + 64),
                  d = ldg_nc_v4(gv + i + 96);
      sv[i] = a; sv[i + 32] = b; sv[i + 64] = c; sv[i + 96] = d;
    }
    for (; i < n16; i += 32) sv[i] = ldg_nc_v4(gv + i);
    done = n16 << 4;
  }
  for (uint32_t i = done + lane; i < nbytes; i += 32) s[i] = g[i];
}

__device__ __forceinline__ void warp_copy_out(uint8_t* g, const uint8_t* s, uint32_t nbytes) {
  const int lane = threadIdx.x & 31;
  uint32_t done = 0;
  if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    const uint32_t n16 = nbytes >> 4;
    const uint4* sv = reinterpret_cast<const uint4*>(s);
    for (uint32_t i = lane; i < n16; i += 32) stg_cs_v4(g + 16ull * i, sv[i]);
    done = n16 << 4;
  }
  for (uint32_t i = done + lane; i < nbytes; i += 32) g[i] = s[i];
}

// min / max of n values at s (any alignment of the block start within smem)
template <typename V>
__device__ __forceinline__ void block_minmax(const V* s, uint32_t n, uint32_t& mn, uint32_t& mx) {
  mn = 0xffffffffu;
  mx = 0u;
  if (sizeof(V) == 2 && (reinterpret_cast<uintptr_t>(s) & 3) == 0) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(s);
    uint32_t a = 0xffffffffu, b = 0u;
    const uint32_t nw = n >> 1;
#pragma unroll 4
    for (uint32_t i = 0; i < nw; ++i) {
      const uint32_t x = w[i];
      a = __vminu2(a, x);
      b = __vmaxu2(b, x);
    }
    mn = min(a & 0xffffu, a >> 16);
    mx = max(b & 0xffffu, b >> 16);
    if (n & 1) {
      const uint32_t x = (uint32_t)s[n - 1];
      mn = min(mn, x);
      mx = max(mx, x);
    }
    if (nw == 0 && !(n & 1)) { mn = 0xffffffffu; mx = 0; }
  } else {
#pragma unroll 4
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t x = (uint32_t)s[i];
      mn = min(mn, x);
      mx = max(mx, x);
    }
  }
}

template <typename V>
__device__ __forceinline__ uint64_t horner(const V* v, uint32_t m, uint32_t B, uint32_t vmin) {
  uint64_t s = 0;
#pragma unroll 4
  for (int i = (int)m - 1; i >= 0; --i) s = s * B + (uint32_t)((uint32_t)v[i] - vmin);
  return s;
}

// Horner for B = 2^32 (only u32 data with v_min = 0 and v_max = 2^32-1).
template <typename V>
__device__ __forceinline__ uint64_t horner_b32(const V* v, uint32_t m, uint32_t vmin) {
  uint64_t s = 0;
  for (int i = (int)m - 1; i >= 0; --i) s = (s << 32) | (uint32_t)((uint32_t)v[i] - vmin);
  return s;
}

__device__ __forceinline__ void write_global_header_w(uint8_t* out, const WarpShape& sh, uint64_t pw) {
  uint4 h0, h1;
  h0.x = 0x43594c50u;
  h0.y = 2u | (sh.width << 16);
  h0.z = (uint32_t)sh.n;
  h0.w = (uint32_t)(sh.n >> 32);
  h1.x = sh.block_len;
  h1.y = (uint32_t)sh.n_blocks;
  h1.z = (uint32_t)(pw * 8);
  h1.w = (uint32_t)((pw * 8) >> 32);
  reinterpret_cast<uint4*>(out)[0] = h0;
  reinterpret_cast<uint4*>(out)[1] = h1;
}

// ======================================================================
// compress
// ======================================================================
template <typename V, int MODE>
__global__ void __launch_bounds__(WARPS * 32) poly_compress_warp(WarpArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const WarpShape& sh = a.sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* slice = smem + (size_t)warp * sh.slice;
  V* sv = reinterpret_cast<V*>(slice);
  const uint32_t L = (uint32_t)sh.Le;
  uint4* hdr_out = reinterpret_cast<uint4*>(a.out + 32);
  uint64_t* pay = reinterpret_cast<uint64_t*>(a.out + 32 + 16 * sh.n_blocks);

  while (true) {
    const uint64_t unit = warp_ticket(a.ticket);
    if (unit >= sh.n_units) break;
    const uint64_t b0 = unit * sh.WB;
    const uint32_t nblk = (uint32_t)min((uint64_t)sh.WB, sh.n_blocks - b0);
    const uint64_t v0 = b0 * sh.Le;
    const uint32_t nv = (uint32_t)(min(sh.n, v0 + (uint64_t)sh.WB * sh.Le) - v0);
    warp_copy_in(slice, a.in + v0 * sizeof(V), nv * (uint32_t)sizeof(V));
    __syncwarp();

    if (MODE == 0) {
      // ---------------- lane per block
      constexpr int BPL_MAX = 4;
      uint32_t vmin[BPL_MAX], Bv[BPL_MAX], nw[BPL_MAX], off[BPL_MAX];
      uint32_t carry = 0;
#pragma unroll
      for (int r = 0; r < BPL_MAX; ++r) {
        const uint32_t lb = r * 32 + lane;
        uint32_t w = 0, mn = 0, mx = 0;
        if (lb < nblk) {
          const uint32_t nb = min(L, nv - lb * L);
          block_minmax<V>(sv + lb * L, nb, mn, mx);
          const uint64_t B = (uint64_t)mx - mn + 1;
          if (B > 1) {
            const uint32_t k = capacity_of(B);
            w = (nb + k - 1) / k;
          }
        }
        vmin[r] = mn;
        Bv[r] = mx - mn;  // B - 1
        nw[r] = w;
        // inclusive warp scan of w
        uint32_t x = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        off[r] = carry + x - w;
        carry += __shfl_sync(0xffffffffu, x, 31);
        if ((r + 1) * 32 >= (int)nblk) break;
      }
      const uint64_t P = warp_publish_and_lookback(a.status, unit, carry);
#pragma unroll
      for (int r = 0; r < BPL_MAX; ++r) {
        const uint32_t lb = r * 32 + lane;
        if (lb < nblk) {
          const uint32_t bm1 = Bv[r];
          hdr_out[b0 + lb] = make_uint4(bm1 == 0 ? CODEC_CONSTANT : CODEC_BASIC, vmin[r], bm1, nw[r]);
          if (bm1 != 0) {
            const uint32_t nb = min(L, nv - lb * L);
            const uint64_t B = (uint64_t)bm1 + 1;
            const uint32_t k = capacity_of(B);
            uint64_t* dst = pay + P + off[r];
            const V* src = sv + lb * L;
            for (uint32_t j = 0; j < nw[r]; ++j) {
              const uint32_t first = j * k, m = min(k, nb - first);
              dst[j] = (bm1 == 0xffffffffu) ? horner_b32<V>(src + first, m, vmin[r])
                                            : horner<V>(src + first, m, bm1 + 1, vmin[r]);
            }
          }
        }
        if ((r + 1) * 32 >= (int)nblk) break;
      }
      if (unit == sh.n_units - 1 && lane == 0) {
        write_global_header_w(a.out, sh, P + carry);
        *a.compressed_bytes = 32 + 16 * sh.n_blocks + 8 * (P + carry);
      }
    } else {
      // ---------------- warp per block
      uint64_t total = 0;
      for (uint32_t lb = 0; lb < nblk; ++lb) {
        const uint32_t nb = min(L, nv - lb * L);
        const V* src = sv + lb * L;
        uint32_t mn = 0xffffffffu, mx = 0;
        if (sizeof(V) == 2 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
          const uint4* q = reinterpret_cast<const uint4*>(src);
          uint32_t a0 = 0xffffffffu, b0v = 0;
          const uint32_t n8 = nb >> 3;
          for (uint32_t i = lane; i < n8; i += 32) {
            const uint4 t = q[i];
            a0 = __vminu2(__vminu2(a0, t.x), __vminu2(t.y, __vminu2(t.z, t.w)));
            b0v = __vmaxu2(__vmaxu2(b0v, t.x), __vmaxu2(t.y, __vmaxu2(t.z, t.w)));
          }
          mn = min(a0 & 0xffffu, a0 >> 16);
          mx = max(b0v & 0xffffu, b0v >> 16);
          if (n8 == 0) { mn = 0xffffffffu; mx = 0; }
          for (uint32_t i = (n8 << 3) + lane; i < nb; i += 32) {
            mn = min(mn, (uint32_t)src[i]);
            mx = max(mx, (uint32_t)src[i]);
          }
        } else {
          for (uint32_t i = lane; i < nb; i += 32) {
            mn = min(mn, (uint32_t)src[i]);
            mx = max(mx, (uint32_t)src[i]);
          }
        }
        mn = shfl_min(mn, 32);
        mx = shfl_max(mx, 32);
        const uint64_t B = (uint64_t)mx - mn + 1;
        const uint32_t w = B == 1 ? 0u : (nb + capacity_of(B) - 1) / capacity_of(B);
        // per-block stats go to the 512-byte scratch at the end of the slice
        uint32_t* st = reinterpret_cast<uint32_t*>(slice + sh.slice - 16 * 32);
        if (lane == 0) { st[4 * lb] = mn; st[4 * lb + 1] = mx - mn; st[4 * lb + 2] = w; st[4 * lb + 3] = (uint32_t)total; }
        total += w;
      }
      __syncwarp();
      const uint64_t P = warp_publish_and_lookback(a.status, unit, total);
      const uint32_t* st = reinterpret_cast<const uint32_t*>(slice + sh.slice - 16 * 32);
      if (lane < (int)nblk) {
        const uint32_t bm1 = st[4 * lane + 1];
        hdr_out[b0 + lane] = make_uint4(bm1 == 0 ? CODEC_CONSTANT : CODEC_BASIC, st[4 * lane], bm1,
                                        st[4 * lane + 2]);
      }
      for (uint32_t lb = 0; lb < nblk; ++lb) {
        const uint32_t vmin = st[4 * lb], bm1 = st[4 * lb + 1], w = st[4 * lb + 2];
        if (bm1 == 0) continue;
        const uint32_t nb = min(L, nv - lb * L);
        const uint32_t k = capacity_of((uint64_t)bm1 + 1);
        const V* src = sv + lb * L;
        uint64_t* dst = pay + P + st[4 * lb + 3];
        for (uint32_t j = lane; j < w; j += 32) {
          const uint32_t first = j * k, m = min(k, nb - first);
          dst[j] = (bm1 == 0xffffffffu) ? horner_b32<V>(src + first, m, vmin)
                                        : horner<V>(src + first, m, bm1 + 1, vmin);
        }
      }
      if (unit == sh.n_units - 1 && lane == 0) {
        write_global_header_w(a.out, sh, P + total);
        *a.compressed_bytes = 32 + 16 * sh.n_blocks + 8 * (P + total);
      }
    }
    __syncwarp();  // the slice is reused by the next unit
  }
}

// ======================================================================
// decompress
// ======================================================================
// Word -> digits, most significant first, via the 64-bit fraction
// f in [s 2^64 / B^k, (s+1) 2^64 / B^k).
template <typename V>
__device__ __forceinline__ uint32_t decode_frac(uint64_t s, const DecConst& c, uint32_t B, uint32_t m,
                                                uint32_t vmin, V* out) {
  if (s >= c.Bk) return POLY_ST_RESIDUE;
  const uint64_t hi1 = __umul64hi(s, c.Rl);
  const uint64_t lo2 = s * c.Rh;
  const uint64_t hi2 = __umul64hi(s, c.Rh);
  const uint64_t mid = lo2 + hi1;
  const uint64_t f = ((hi2 + (mid < lo2 ? 1ull : 0ull)) << 32) + (mid >> 32) + 1;
  uint32_t f0 = (uint32_t)f, f1 = (uint32_t)(f >> 32);
  uint32_t extra = 0;
  int i = (int)c.k - 1;
  for (; i >= (int)m; --i) {
    const uint64_t t0 = (uint64_t)f0 * B;
    const uint64_t t1 = (uint64_t)f1 * B + (t0 >> 32);
    extra |= (uint32_t)(t1 >> 32);
    f1 = (uint32_t)t1;
    f0 = (uint32_t)t0;
  }
#pragma unroll 4
  for (; i >= 0; --i) {
    const uint64_t t0 = (uint64_t)f0 * B;
    const uint64_t t1 = (uint64_t)f1 * B + (t0 >> 32);
    out[i] = (V)(vmin + (uint32_t)(t1 >> 32));
    f1 = (uint32_t)t1;
    f0 = (uint32_t)t0;
  }
  return extra ? POLY_ST_RESIDUE : 0u;
}

template <typename V>
__device__ __forceinline__ uint32_t decode_pow2(uint64_t s, uint32_t j, uint32_t m, uint32_t vmin, V* out) {
  const uint64_t mask = (j >= 64) ? ~0ull : ((1ull << j) - 1);
#pragma unroll 4
  for (uint32_t i = 0; i < m; ++i) out[i] = (V)(vmin + (uint32_t)((s >> (i * j)) & mask));
  return (m * j < 64 && (s >> (m * j)) != 0) ? POLY_ST_RESIDUE : 0u;
}

template <typename V>
__device__ __forceinline__ uint32_t decode_any(uint64_t s, const DecConst& c, uint32_t bm1, uint32_t m,
                                               uint32_t vmin, V* out) {
  if (c.log2b) return decode_pow2<V>(s, c.log2b, m, vmin, out);
  return decode_frac<V>(s, c, bm1 + 1, m, vmin, out);
}

// Global-header check by lane 0, broadcast.  Returns status bits.
__device__ __forceinline__ uint32_t warp_check_header(const WarpArgs& a, uint64_t* pw) {
  uint32_t e = 0;
  uint64_t p = 0;
  if ((threadIdx.x & 31) == 0) {
    const WarpShape& sh = a.sh;
    if (a.in_bytes < 32) {
      e = POLY_ST_LENGTH;
    } else {
      const uint4 h0 = reinterpret_cast<const uint4*>(a.in)[0];
      const uint4 h1 = reinterpret_cast<const uint4*>(a.in)[1];
      const uint64_t n = (uint64_t)h0.z | ((uint64_t)h0.w << 32);
      const uint64_t pb = (uint64_t)h1.z | ((uint64_t)h1.w << 32);
      if (h0.x != 0x43594c50u) e = POLY_ST_BAD_MAGIC;
      else if ((h0.y & 0xffu) != 2u) e = POLY_ST_BAD_VERSION;
      else if (((h0.y >> 8) & 0xffu) != 0u || ((h0.y >> 16) & 0xffu) != sh.width || (h0.y >> 24) != 0u ||
               n != sh.n || h1.x != sh.block_len || h1.y != (uint32_t)sh.n_blocks)
        e = POLY_ST_HEADER_MISMATCH;
      else if ((pb & 7) != 0 || a.in_bytes != 32 + 16 * sh.n_blocks + pb)
        e = POLY_ST_LENGTH;
      p = pb >> 3;
    }
  }
  *pw = __shfl_sync(0xffffffffu, p, 0);
  return __shfl_sync(0xffffffffu, e, 0);
}

__device__ __forceinline__ uint32_t check_block_hdr(uint4 h, uint32_t nb, uint32_t width, uint32_t k) {
  const uint64_t vmax_allowed = (width == 16) ? 0xffffull : 0xffffffffull;
  if (h.x == CODEC_CONSTANT) {
    uint32_t e = 0;
    if (h.z != 0 || h.w != 0) e |= POLY_ST_NWORDS;
    if ((uint64_t)h.y > vmax_allowed) e |= POLY_ST_OVERFLOW;
    return e;
  }
  if (h.x != CODEC_BASIC) return POLY_ST_BAD_CODEC;
  if (h.z == 0 || (uint64_t)h.y + h.z > vmax_allowed) return POLY_ST_OVERFLOW;
  if (h.w != (nb + k - 1) / k) return POLY_ST_NWORDS;
  return 0;
}

template <typename V, int MODE>
__global__ void __launch_bounds__(WARPS * 32) poly_decompress_warp(WarpArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const WarpShape& sh = a.sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* slice = smem + (size_t)warp * sh.slice;
  V* so = reinterpret_cast<V*>(slice);
  const uint32_t L = (uint32_t)sh.Le;
  uint64_t payload_words = 0;
  const uint32_t herr = warp_check_header(a, &payload_words);
  if (herr) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.status_out, herr);
    return;  // same verdict in every warp: nothing is decoded, no look-back
  }
  const uint4* hdr = reinterpret_cast<const uint4*>(a.in + 32);
  const uint64_t* pay = reinterpret_cast<const uint64_t*>(a.in + 32 + 16 * sh.n_blocks);
  uint32_t err = 0;

  while (true) {
    const uint64_t unit = warp_ticket(a.ticket);
    if (unit >= sh.n_units) break;
    const uint64_t b0 = unit * sh.WB;
    const uint32_t nblk = (uint32_t)min((uint64_t)sh.WB, sh.n_blocks - b0);
    const uint64_t v0 = b0 * sh.Le;
    const uint32_t nv = (uint32_t)(min(sh.n, v0 + (uint64_t)sh.WB * sh.Le) - v0);

    if (MODE == 0) {
      constexpr int BPL_MAX = 4;
      uint4 h[BPL_MAX];
      uint32_t off[BPL_MAX], ok[BPL_MAX];
      uint64_t carry = 0;
#pragma unroll
      for (int r = 0; r < BPL_MAX; ++r) {
        const uint32_t lb = r * 32 + lane;
        uint32_t w = 0;
        ok[r] = 0;
        h[r] = make_uint4(0, 0, 0, 0);
        if (lb < nblk) {
          h[r] = hdr[b0 + lb];
          const uint32_t nb = min(L, nv - lb * L);
          const uint32_t k = (h[r].x == CODEC_BASIC && h[r].z != 0) ? capacity_of((uint64_t)h[r].z + 1) : 1u;
          const uint32_t e = check_block_hdr(h[r], nb, sh.width, k);
          err |= e;
          ok[r] = e ? 0u : (h[r].x == CODEC_CONSTANT ? 1u : 2u);
          w = h[r].w;
        }
        uint32_t x = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        off[r] = (uint32_t)carry + x - w;
        carry += __shfl_sync(0xffffffffu, x, 31);
        if ((r + 1) * 32 >= (int)nblk) break;
      }
      const uint64_t P = warp_publish_and_lookback(a.status, unit, carry);
      if (P + carry > payload_words) err |= POLY_ST_LENGTH;
      if (unit == sh.n_units - 1 && P + carry != payload_words) err |= POLY_ST_LENGTH;
      const bool len_ok = P + carry <= payload_words;
#pragma unroll
      for (int r = 0; r < BPL_MAX; ++r) {
        const uint32_t lb = r * 32 + lane;
        if (lb < nblk && ok[r] && len_ok) {
          const uint32_t nb = min(L, nv - lb * L);
          V* dst = so + lb * L;
          if (ok[r] == 1) {
            for (uint32_t i = 0; i < nb; ++i) dst[i] = (V)h[r].y;
          } else {
            const DecConst c = dec_const_of((uint64_t)h[r].z + 1);
            const uint64_t* src = pay + P + off[r];
            for (uint32_t j = 0; j < h[r].w; ++j) {
              const uint32_t first = j * c.k;
              err |= decode_any<V>(ldg_nc_u64(src + j), c, h[r].z, min(c.k, nb - first), h[r].y, dst + first);
            }
          }
        }
        if ((r + 1) * 32 >= (int)nblk) break;
      }
    } else {
      // warp per block: all lanes read each header (broadcast loads)
      uint64_t total = 0;
      uint32_t* st = reinterpret_cast<uint32_t*>(slice + sh.slice - 16 * 32);
      for (uint32_t lb = 0; lb < nblk; ++lb) {
        const uint4 h = hdr[b0 + lb];
        const uint32_t nb = min(L, nv - lb * L);
        const uint32_t k = (h.x == CODEC_BASIC && h.z != 0) ? capacity_of((uint64_t)h.z + 1) : 1u;
        const uint32_t e = check_block_hdr(h, nb, sh.width, k);
        if (lane == 0) {
          err |= e;
          st[4 * lb] = (uint32_t)total;
          st[4 * lb + 1] = e ? 0u : (h.x == CODEC_CONSTANT ? 1u : 2u);
        }
        total += h.w;
      }
      __syncwarp();
      const uint64_t P = warp_publish_and_lookback(a.status, unit, total);
      if (lane == 0) {
        if (P + total > payload_words) err |= POLY_ST_LENGTH;
        if (unit == sh.n_units - 1 && P + total != payload_words) err |= POLY_ST_LENGTH;
      }
      if (P + total <= payload_words) {
        for (uint32_t lb = 0; lb < nblk; ++lb) {
          const uint32_t okb = st[4 * lb + 1];
          if (!okb) continue;
          const uint4 h = hdr[b0 + lb];
          const uint32_t nb = min(L, nv - lb * L);
          V* dst = so + lb * L;
          if (okb == 1) {
            for (uint32_t i = lane; i < nb; i += 32) dst[i] = (V)h.y;
            continue;
          }
          const DecConst c = dec_const_of((uint64_t)h.z + 1);
          const uint64_t* src = pay + P + st[4 * lb];
          for (uint32_t j = lane; j < h.w; j += 32) {
            const uint32_t first = j * c.k;
            err |= decode_any<V>(ldg_nc_u64(src + j), c, h.z, min(c.k, nb - first), h.y, dst + first);
          }
        }
      }
    }
    __syncwarp();
    warp_copy_out(a.out + v0 * sizeof(V), slice, nv * (uint32_t)sizeof(V));
    __syncwarp();
  }
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0 && err) atomicOr(a.status_out, err);
}

}  // namespace polyk

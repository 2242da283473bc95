// poly_warp.cuh -- warp-tile kernels (blocks of up to WT_MAX bytes) and the
// word codec shared with the large-block kernels.
//
// Each warp owns one look-back unit at a time: a run of consecutive blocks
// of the stream, handed out in order by an atomic ticket (persistent grid).
// No CTA barrier is used.  A warp stages its unit in its own shared-memory
// slice, computes the per-block statistics, scans the word counts with
// shuffles, publishes its aggregate, looks back for its payload offset and
// writes headers and words with coalesced stores.
//
// Two mappings (chosen on the host, see poly.cu plan()):
//   MODE 0 (block <= 128 B, e.g. cfg2's 30 x u16): lane l owns blocks
//          l, l+32, ... of the unit (BPL blocks per lane).  Words are staged
//          in smem before the look-back, so the look-back latency overlaps the
//          packing and the payload leaves with contiguous 8-byte stores.
//   MODE 1 (128 B < block <= WT_MAX): the 32 lanes cooperate on each block
//          (WB blocks per unit); lane l owns words l, l+32, ... (contiguous).
#pragma once
#include "poly_common.cuh"
#include "poly_word.cuh"

namespace polyk {

constexpr int WARPS = 4;               // warps per CTA (independent)
constexpr uint32_t WT_MAX = 8192;      // bytes of input per warp unit
constexpr uint32_t LANE_BLOCK_MAX = 128;
constexpr int BPL_MAX = 4;             // MODE 0: blocks per lane

struct WarpShape {
  uint64_t n, Le, n_blocks;
  uint32_t block_len, width;
  uint32_t WB;         // blocks per unit
  uint32_t mode;       // 0 lane, 1 warp
  uint32_t slice;      // smem bytes per warp (16-aligned)
  uint32_t words_off;  // MODE 0: byte offset of the word area in the slice
  uint32_t words_cap;  // MODE 0: capacity of the word area (words)
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

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t warp_ticket(uint32_t* ticket) {
  uint32_t t = 0;
  if ((threadIdx.x & 31) == 0) t = atomicAdd(ticket, 1u);
  return __shfl_sync(0xffffffffu, t, 0);
}

__device__ __forceinline__ void warp_publish_agg(uint64_t* status, uint64_t unit, uint64_t total) {
  if ((threadIdx.x & 31) == 0)
    st_relaxed_u64(status + unit, (unit == 0 ? FLAG_PRE : FLAG_AGG) | (total & VAL_MASK));
}

// Exclusive prefix of `unit`, then publish its inclusive prefix.
__device__ __forceinline__ uint64_t warp_lookback(uint64_t* status, uint64_t unit, uint64_t total) {
  if (unit == 0) return 0;
  const uint64_t p = lookback(status, unit);
  if ((threadIdx.x & 31) == 0) st_relaxed_u64(status + unit, FLAG_PRE | ((p + total) & VAL_MASK));
  return p;
}

// Copy nbytes from global g to this warp's smem slice s (16-byte vectors when
// g is 16-byte aligned; bytes otherwise).  Up to 8 loads in flight per lane.
__device__ __forceinline__ void warp_copy_in(uint8_t* s, const uint8_t* g, uint32_t nbytes) {
  const int lane = threadIdx.x & 31;
  uint32_t done = 0;
  if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    const uint32_t n16 = nbytes >> 4;
    const uint4* gv = reinterpret_cast<const uint4*>(g);
    uint4* sv = reinterpret_cast<uint4*>(s);
    uint32_t i = lane;
    for (; i + 7 * 32 < n16; i += 8 * 32) {
      uint4 r[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = ldg_nc_v4(gv + i + 32 * q);
#pragma unroll
      for (int q = 0; q < 8; ++q) sv[i + 32 * q] = r[q];
    }
    for (; i < n16; i += 32) sv[i] = ldg_nc_v4(gv + i);
    done = n16 << 4;
  }
  for (uint32_t i = done + lane; i < nbytes; i += 32) s[i] = g[i];
}

// Copy nbytes from smem s to global g (16-byte stores when g is aligned).
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

// Copy `cnt` u64 words between global (8-byte aligned) and smem, coalesced.
__device__ __forceinline__ void warp_words_in(uint64_t* s, const uint64_t* g, uint32_t cnt) {
  const int lane = threadIdx.x & 31;
  uint32_t i = lane;
  for (; i + 3 * 32 < cnt; i += 4 * 32) {
    uint64_t r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = ldg_nc_u64(g + i + 32 * q);
#pragma unroll
    for (int q = 0; q < 4; ++q) s[i + 32 * q] = r[q];
  }
  for (; i < cnt; i += 32) s[i] = ldg_nc_u64(g + i);
}

__device__ __forceinline__ void write_global_header_w(uint8_t* out, const WarpShape& sh, uint64_t pw) {
  write_global_header_f(out, sh.width, sh.n, sh.block_len, sh.n_blocks, pw);
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
      uint64_t* sw = reinterpret_cast<uint64_t*>(slice + sh.words_off);
      uint32_t vmin[BPL_MAX], bm1[BPL_MAX], nw[BPL_MAX], off[BPL_MAX];
      uint32_t carry = 0;
      const int rounds = (int)((nblk + 31) >> 5);
#pragma unroll
      for (int r = 0; r < BPL_MAX; ++r) {
        vmin[r] = 0; bm1[r] = 0; nw[r] = 0; off[r] = 0;
        if (r < rounds) {
          const uint32_t lb = r * 32 + lane;
          if (lb < nblk) {
            const uint32_t nb = min(L, nv - lb * L);
            uint32_t mn, mx;
            block_minmax<V>(sv + lb * L, nb, mn, mx);
            vmin[r] = mn;
            bm1[r] = mx - mn;
            if (mx != mn) nw[r] = ceil_div_small(nb, capacity_of((uint64_t)(mx - mn) + 1));
          }
          const uint32_t x = warp_incl_scan(nw[r]);
          off[r] = carry + x - nw[r];
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
      }
      warp_publish_agg(a.status, unit, carry);
      // pack into the word area (overlaps the predecessors' progress)
#pragma unroll
      for (int r = 0; r < BPL_MAX; ++r) {
        const uint32_t lb = r * 32 + lane;
        if (r < rounds && lb < nblk && bm1[r] != 0) {
          const uint32_t nb = min(L, nv - lb * L);
          const PackParams pp = pack_params(bm1[r]);
          const V* src = sv + lb * L;
          uint64_t* dst = sw + off[r];
          for (uint32_t j = 0, first = 0; j < nw[r]; ++j, first += pp.k)
            dst[j] = pack_any<V>(src + first, min(pp.k, nb - first), pp, vmin[r]);
        }
      }
      const uint64_t P = warp_lookback(a.status, unit, carry);
#pragma unroll
      for (int r = 0; r < BPL_MAX; ++r) {
        const uint32_t lb = r * 32 + lane;
        if (r < rounds && lb < nblk)
          hdr_out[b0 + lb] = make_uint4(bm1[r] == 0 ? CODEC_CONSTANT : CODEC_BASIC, vmin[r], bm1[r], nw[r]);
      }
      __syncwarp();
      uint64_t* dst = pay + P;
      for (uint32_t i = lane; i < carry; i += 32) dst[i] = sw[i];
      if (unit == sh.n_units - 1 && lane == 0) {
        write_global_header_w(a.out, sh, P + carry);
        *a.compressed_bytes = 32 + 16 * sh.n_blocks + 8 * (P + carry);
      }
    } else {
      // ---------------- warp per block
      uint32_t* st = reinterpret_cast<uint32_t*>(slice + sh.slice - 16 * 32);
      uint64_t total = 0;
      for (uint32_t lb = 0; lb < nblk; ++lb) {
        const uint32_t nb = min(L, nv - lb * L);
        const V* src = sv + lb * L;
        uint32_t mn = 0xffffffffu, mx = 0;
        if (sizeof(V) == 2 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
          const uint4* q = reinterpret_cast<const uint4*>(src);
          uint32_t a0 = 0xffffffffu, a1 = 0u;
          const uint32_t n8 = nb >> 3;
          for (uint32_t i = lane; i < n8; i += 32) {
            const uint4 t = q[i];
            a0 = __vimin3_u16x2(a0, t.x, t.y);
            a0 = __vimin3_u16x2(a0, t.z, t.w);
            a1 = __vimax3_u16x2(a1, t.x, t.y);
            a1 = __vimax3_u16x2(a1, t.z, t.w);
          }
          mn = min(a0 & 0xffffu, a0 >> 16);
          mx = max(a1 & 0xffffu, a1 >> 16);
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
        const uint32_t w = mx == mn ? 0u : ceil_div_small(nb, capacity_of((uint64_t)(mx - mn) + 1));
        if (lane == 0) {
          st[4 * lb] = mn;
          st[4 * lb + 1] = mx - mn;
          st[4 * lb + 2] = w;
          st[4 * lb + 3] = (uint32_t)total;
        }
        total += w;
      }
      warp_publish_agg(a.status, unit, total);
      __syncwarp();
      if (lane < (int)nblk) {
        const uint32_t bm1 = st[4 * lane + 1];
        hdr_out[b0 + lane] = make_uint4(bm1 == 0 ? CODEC_CONSTANT : CODEC_BASIC, st[4 * lane], bm1,
                                        st[4 * lane + 2]);
      }
      const uint64_t P = warp_lookback(a.status, unit, total);
      for (uint32_t lb = 0; lb < nblk; ++lb) {
        const uint32_t vmin = st[4 * lb], bm1 = st[4 * lb + 1], w = st[4 * lb + 2];
        if (bm1 == 0) continue;
        const uint32_t nb = min(L, nv - lb * L);
        const PackParams pp = pack_params(bm1);
        const V* src = sv + lb * L;
        uint64_t* dst = pay + P + st[4 * lb + 3];
        for (uint32_t j = lane; j < w; j += 32) {
          const uint32_t first = j * pp.k;
          dst[j] = pack_any<V>(src + first, min(pp.k, nb - first), pp, vmin);
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
      uint64_t* sw = reinterpret_cast<uint64_t*>(slice + sh.words_off);
      uint4 h[BPL_MAX];
      uint32_t off[BPL_MAX];
      uint32_t carry = 0;
      const int rounds = (int)((nblk + 31) >> 5);
#pragma unroll
      for (int r = 0; r < BPL_MAX; ++r) {
        const uint32_t lb = r * 32 + lane;
        h[r] = make_uint4(0, 0, 0, 0);
        if (r < rounds && lb < nblk) h[r] = hdr[b0 + lb];
      }
#pragma unroll
      for (int r = 0; r < BPL_MAX; ++r) {
        off[r] = 0;
        if (r < rounds) {
          const uint32_t lb = r * 32 + lane;
          uint32_t w = 0;
          if (lb < nblk) {
            const uint32_t nb = min(L, nv - lb * L);
            const uint32_t k = (h[r].x == CODEC_BASIC && h[r].z != 0) ? capacity_of((uint64_t)h[r].z + 1) : 1u;
            const uint32_t e = check_block_hdr(h[r], nb, sh.width, k);
            err |= e;
            if (e) h[r].x = 0;  // skip the block
            w = h[r].w;
          }
          const uint32_t x = warp_incl_scan(w);
          off[r] = carry + x - w;
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
      }
      warp_publish_agg(a.status, unit, carry);
      const uint64_t P = warp_lookback(a.status, unit, carry);
      const bool len_ok = P + carry <= payload_words && carry <= sh.words_cap;
      if (!len_ok || (unit == sh.n_units - 1 && P + carry != payload_words)) err |= POLY_ST_LENGTH;
      if (len_ok) warp_words_in(sw, pay + P, carry);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < BPL_MAX; ++r) {
        const uint32_t lb = r * 32 + lane;
        if (r < rounds && lb < nblk && h[r].x != 0 && len_ok) {
          const uint32_t nb = min(L, nv - lb * L);
          V* dst = so + lb * L;
          if (h[r].x == CODEC_CONSTANT) {
            for (uint32_t i = 0; i < nb; ++i) dst[i] = (V)h[r].y;
          } else {
            const DecConst c = dec_const_of((uint64_t)h[r].z + 1);
            const uint32_t k = dc_k(c);
            const uint64_t* src = sw + off[r];
            for (uint32_t j = 0, first = 0; j < h[r].w; ++j, first += k)
              err |= decode_any<V>(src[j], c, h[r].z, min(k, nb - first), h[r].y, dst + first);
          }
        }
      }
    } else {
      // warp per block: every lane reads each header (broadcast loads)
      uint32_t* st = reinterpret_cast<uint32_t*>(slice + sh.slice - 16 * 32);
      uint64_t total = 0;
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
      warp_publish_agg(a.status, unit, total);
      const uint64_t P = warp_lookback(a.status, unit, total);
      __syncwarp();
      const bool len_ok = P + total <= payload_words;
      if (lane == 0 && (!len_ok || (unit == sh.n_units - 1 && P + total != payload_words)))
        err |= POLY_ST_LENGTH;
      if (len_ok) {
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
          const uint32_t k = dc_k(c);
          const uint64_t* src = pay + P + st[4 * lb];
          uint32_t j = lane;
          for (; j + 32 < h.w; j += 64) {  // two words in flight per lane
            const uint64_t s0 = ldg_nc_u64(src + j), s1 = ldg_nc_u64(src + j + 32);
            err |= decode_any<V>(s0, c, h.z, min(k, nb - j * k), h.y, dst + j * k);
            err |= decode_any<V>(s1, c, h.z, min(k, nb - (j + 32) * k), h.y, dst + (j + 32) * k);
          }
          if (j < h.w) err |= decode_any<V>(ldg_nc_u64(src + j), c, h.z, min(k, nb - j * k), h.y, dst + j * k);
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

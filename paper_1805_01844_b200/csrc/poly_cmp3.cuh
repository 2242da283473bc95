// poly_cmp3.cuh -- compression of blocks whose byte size is a multiple of 16
// (128 B < block <= 32 KiB: the PIPE map-1 shapes cfg4, cfg5), SURVEY.md
// Sec. 8(a) rows a2-a6, one warp per block, packed in place.
//
// A tile is TB consecutive blocks (about C3_TILE bytes); the tiles of a launch
// are dealt round robin to the worker CTAs (the prefix-server CTA is the last
// one, cooperative launch; measured against a ticket per tile: faster).  Per
// CTA:
//   producer warp : a 1-D TMA bulk copy of each tile's values into one of S
//                   shared-memory slots (mbarrier complete_tx)
//   consumer warps: claim CB blocks at a time (shared-memory counter; CB > 1
//                   for small blocks); per block a min/max (a2) by 32 / CB
//                   lanes, B and k from the base table
//                   (a3), n_words = ceil(n_b / k), the block header straight to
//                   its fixed offset; the consumer that completes a tile's
//                   word counts publishes the tile aggregate (a4) at once; then
//                   the block is Horner-packed (a5) IN PLACE: word j of a block
//                   never extends past the first byte of value j k (k >= 8 /
//                   value bytes), and every step loads its values before any
//                   lane stores (__syncwarp), so no unread value is overwritten
//   writer warps  : writer w owns the slots s = w (mod NWR) (S is a multiple
//                   of NWR), so it meets each slot's uses in order; it waits
//                   for the tile's blocks, scans their word counts, gets the
//                   tile prefix (prefix server or look-back), copies the words
//                   to the stream (a6) and frees the slot; the last tile writes
//                   the global header and *compressed_bytes.
// No CTA-wide barrier after the start: warps meet only on mbarriers.
#pragma once
#include "poly_common.cuh"
#include "poly_word.cuh"
#include "poly_kword.cuh"
#include "poly_pipe.cuh"
#include "poly_dec3.cuh"  // PROBE_* (timing-experiment variant only)

namespace polyk {
namespace c3 {
#ifdef POLY_PROBE
using d3::g_probe;
#endif

#ifndef POLY_C3_NW
#define POLY_C3_NW 12
#endif
#ifndef POLY_C3_NWR
#define POLY_C3_NWR 4
#endif
constexpr int NW = POLY_C3_NW;           // consumer warps
constexpr int NWR = POLY_C3_NWR;         // writer warps
constexpr int NTHR = 32 * (NW + 1 + NWR);
// slots and tile size (A/B knobs; measured, cfg5 / cfg4 compress GB/s against
// 3545 / 2436: 16 KiB x 12 slots 2877 / 2278, 8 KiB x 24 1824 / 1551, 32 KiB x 6
// with 3 writers 3575 / 2392, with 2 writers 3664 / 1990, 48 KiB x 4 3421 / 2026)
#ifndef POLY_C3_MAXS
#define POLY_C3_MAXS 8
#endif
#ifndef POLY_C3_TILE
#define POLY_C3_TILE 24576
#endif
constexpr int MAXS3 = POLY_C3_MAXS;      // slots
constexpr uint32_t TBMAX = 256;          // blocks per tile
constexpr uint32_t C3_TILE = POLY_C3_TILE;  // value bytes per tile (target)
constexpr uint32_t C3_CLAIM = 8192;      // value bytes per consumer claim (target; small blocks)

struct __align__(16) Ctl {
  uint64_t full[MAXS3], packed[MAXS3], empty[MAXS3];
  volatile uint64_t fseq[MAXS3];  // the CTA iteration whose tile the slot's fill is for
  uint32_t cnt[MAXS3];            // blocks of the slot's tile whose word count is known
  uint32_t next;                  // consumer claims
  uint32_t nw[MAXS3][TBMAX];      // word counts of the slot's blocks
};

// In-place pack of a u16 block of uniform capacity K with the k-specialised
// group codec (poly_kword.cuh): group g (Q words, Q K values) is loaded by
// lane g mod 32 before any lane of the step stores its words.  Returns the
// number of leading words packed.
template <int K>
__device__ __forceinline__ uint32_t pack_inplace_k(uint8_t* blk, uint32_t nb, uint32_t B, uint32_t vmin) {
  using C = KCls<K>;
  const int lane = threadIdx.x & 31;
  const uint32_t ng = nb / C::VALS;
  const KPack c = kpack_consts<K>(B, vmin);
  uint64_t* dst = reinterpret_cast<uint64_t*>(blk);
  for (uint32_t g0 = 0; g0 < ng; g0 += 32) {
    const uint32_t g = g0 + lane;
    uint32_t r[C::NR];
    load_group<K>(blk + (size_t)min(g, ng - 1) * C::BYTES, r);  // lanes past the end reload the last group
    __syncwarp();
    if (g < ng) {
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
  }
  return ng * C::Q;
}

// Words [j0, nw) of a block, word-parallel, in place (each step loads before
// it stores).
template <typename V>
__device__ __forceinline__ void pack_inplace_words(V* v, uint32_t nb, uint32_t k, uint64_t B, uint32_t vmin,
                                                   uint32_t j0, uint32_t nw) {
  const int lane = threadIdx.x & 31;
  uint64_t* dst = reinterpret_cast<uint64_t*>(v);
  for (uint32_t jb = j0; jb < nw; jb += 32) {
    const uint32_t j = jb + lane;
    uint64_t w = 0;
    if (j < nw) {
      const uint32_t first = j * k;
      w = pack_word64<V>(v + first, min(k, nb - first), B, vmin);
    }
    __syncwarp();
    if (j < nw) dst[j] = w;
  }
}

// min / max of the CB (<= 32) blocks of a claim: LPB = 32 / CB lanes per
// block (lane l works on block l / LPB), 16-byte loads, a reduction over the
// block's lanes.  Every lane returns its block's min / max.
template <typename V>
__device__ __forceinline__ void claim_minmax(const uint8_t* base, uint32_t bb, uint32_t lgl, uint32_t nvb,
                                             uint32_t nb_last, uint32_t& mn, uint32_t& mx) {
  const int lane = threadIdx.x & 31;
  const uint32_t LPB = 1u << lgl, c = (uint32_t)lane >> lgl, r = (uint32_t)lane & (LPB - 1);
  constexpr uint32_t PER = 16 / sizeof(V);
  mn = 0xffffffffu;
  mx = 0u;
  if (c < nvb) {
    const uint32_t nb = c + 1 == nvb ? nb_last : bb / (uint32_t)sizeof(V);
    const uint4* q = reinterpret_cast<const uint4*>(base + (size_t)c * bb);
    const uint32_t nq = nb / PER;
    if (sizeof(V) == 2) {
      uint32_t a0 = 0xffffffffu, a1 = 0u;
#pragma unroll 4
      for (uint32_t j = r; j < nq; j += LPB) {
        const uint4 t = q[j];
        a0 = __vimin3_u16x2(a0, t.x, t.y);
        a0 = __vimin3_u16x2(a0, t.z, t.w);
        a1 = __vimax3_u16x2(a1, t.x, t.y);
        a1 = __vimax3_u16x2(a1, t.z, t.w);
      }
      mn = min(a0 & 0xffffu, a0 >> 16);
      mx = max(a1 & 0xffffu, a1 >> 16);
    } else if (sizeof(V) == 1) {
      uint32_t a0 = 0xffffffffu, a1 = 0u;
#pragma unroll 4
      for (uint32_t j = r; j < nq; j += LPB) {
        const uint4 t = q[j];
        a0 = __vminu4(__vminu4(a0, __vminu4(t.x, t.y)), __vminu4(t.z, t.w));
        a1 = __vmaxu4(__vmaxu4(a1, __vmaxu4(t.x, t.y)), __vmaxu4(t.z, t.w));
      }
      mn = min(min(a0 & 0xffu, (a0 >> 8) & 0xffu), min((a0 >> 16) & 0xffu, a0 >> 24));
      mx = max(max(a1 & 0xffu, (a1 >> 8) & 0xffu), max((a1 >> 16) & 0xffu, a1 >> 24));
    } else {
#pragma unroll 4
      for (uint32_t j = r; j < nq; j += LPB) {
        const uint4 t = q[j];
        mn = min(min(mn, t.x), min(t.y, min(t.z, t.w)));
        mx = max(max(mx, t.x), max(t.y, max(t.z, t.w)));
      }
    }
    const V* v = reinterpret_cast<const V*>(q);
    for (uint32_t e = nq * PER + r; e < nb; e += LPB) {  // the array's last block: a partial vector
      mn = min(mn, (uint32_t)v[e]);
      mx = max(mx, (uint32_t)v[e]);
    }
  }
  for (uint32_t o = LPB >> 1; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
}

// MULTI: claims of CB > 1 blocks (small blocks); the CB = 1 instantiation
// keeps the one-block path alone (measured: the shared kernel cost cfg5 6 %).
template <typename V, bool MULTI>
__global__ void __launch_bounds__(NTHR, 1) cmp3(PipeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  if (a.server && blockIdx.x == gridDim.x - 1) {
    if (threadIdx.x < 32) prefix_server(a.status, a.t_end, a.t_begin);
    return;
  }
  Ctl& C = *reinterpret_cast<Ctl*>(smem);
  const PipeShape& sh = a.sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t S = sh.S, TB = sh.TB, CB = MULTI ? sh.G : 1u, NU = TB / CB;  // CB blocks per claim, NU claims per tile
  const BaseCache bc = cache_at(smem + sh.o_cache, false);
  if (tid == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&C.full[s], 1);
      mbar_init(&C.packed[s], NU);
      mbar_init(&C.empty[s], 1);
      C.fseq[s] = ~0ull;
      C.cnt[s] = 0;
    }
    C.next = 0;
    mbar_fence_init();
  }
  cache_fill(bc, false);
  __syncthreads();
  // this CTA's tiles: t = t_begin + blockIdx.x + i * nwork, i < my
  const uint64_t nwork = gridDim.x - a.server;
  const uint64_t ntl = a.t_end - a.t_begin;
  const uint64_t my = blockIdx.x < ntl ? (ntl - blockIdx.x + nwork - 1) / nwork : 0;
  const uint32_t L = (uint32_t)sh.Le, bb = L * sh.vb;
  uint8_t* const slots = smem + sh.o_in;

  if (warp == NW) {
    // ------------------------------------------------------------ producer
    const uint64_t total = sh.n * sh.vb;
    PROBE_DECL;
    PROBE_T0(pt0);
    for (uint64_t i = 0; i < my; ++i) {
      const uint32_t s = (uint32_t)(i % S);
      PROBE_T0(pw0);
      if (i >= S) mbar_wait_cmp<1>(&C.empty[s], (uint32_t)((i / S) & 1) ^ 1u);
      PROBE_ADD(15, pw0);
      const uint64_t t = a.t_begin + blockIdx.x + i * nwork;
      const uint64_t off = t * sh.tile_bytes;
      const uint32_t bytes = (uint32_t)min((uint64_t)sh.tile_bytes, total - off);
      uint8_t* dst = slots + (size_t)s * sh.in_stride;
      const uint8_t* src = a.in + off;
      if (a.bulk) {
        if (lane == 0) {
          const uint32_t n16 = bytes & ~15u;
          for (uint32_t j = n16; j < bytes; ++j) dst[j] = src[j];  // the last tile's tail
          C.fseq[s] = i;
          mbar_arrive_tx(&C.full[s], n16);
          if (n16) bulk_g2s(dst, src, n16, &C.full[s]);
        }
      } else {
        warp_copy(dst, src, bytes, lane);
        __syncwarp();
        if (lane == 0) {
          C.fseq[s] = i;
          mbar_arrive(&C.full[s]);
        }
      }
    }
    PROBE_ADD(16, pt0);
    PROBE_FLUSH;
    return;
  }

  uint64_t* const pay_g = reinterpret_cast<uint64_t*>(a.out + 32 + 16 * sh.n_blocks);
  if (warp > NW) {
    // ------------------------------------------------------------ writers
    // (a writer meets the uses of its slots in order, so the packed-barrier
    // parity cannot alias a later use)
    const uint32_t w = (uint32_t)(warp - NW - 1);
    PROBE_DECL;
    PROBE_T0(wt0);
    for (uint64_t i = w; i < my; i += NWR) {
      const uint32_t s = (uint32_t)(i % S);
      PROBE_T0(ww0);
      mbar_wait_writer(&C.packed[s], (uint32_t)(i / S) & 1u);
      PROBE_ADD(13, ww0);
      PROBE_T0(wp0);
      const uint64_t t = a.t_begin + blockIdx.x + i * nwork;
      const uint64_t b0 = t * TB;
      const uint32_t nblk = (uint32_t)min((uint64_t)TB, sh.n_blocks - b0);
      uint64_t P = 0;
      if (t != 0) {
        if (a.server) {
          P = wait_prefix(a.status, t);
        } else {
          uint32_t W = 0;
          for (uint32_t b = lane; b < nblk; b += 32) W += C.nw[s][b];
          W = __reduce_add_sync(0xffffffffu, W);
          P = lookback_wide(a.status, t);
          if (lane == 0) st_relaxed_u64(a.status + t, FLAG_PRE | ((P + W) & VAL_MASK));
        }
      }
      PROBE_ADD(14, wp0);
      // copy the blocks' words, 32 blocks per round: each lane's block offset
      // from a warp scan, then block by block, lane-strided 8-byte copies
      uint64_t off = P;
      const uint8_t* base = slots + (size_t)s * sh.in_stride;
      for (uint32_t r0 = 0; r0 < nblk; r0 += 32) {
        const uint32_t b = r0 + lane;
        const uint32_t nwb = b < nblk ? C.nw[s][b] : 0u;
        uint32_t tot;
        const uint32_t ex = warp_excl_scan(nwb, &tot);
        const uint32_t nr = min(32u, nblk - r0);
        for (uint32_t q = 0; q < nr; ++q) {
          const uint32_t n = __shfl_sync(0xffffffffu, nwb, q), e = __shfl_sync(0xffffffffu, ex, q);
          const uint64_t* src = reinterpret_cast<const uint64_t*>(base + (size_t)(r0 + q) * bb);
          uint64_t* dst = pay_g + off + e;
          uint32_t j = lane;
          for (; j + 96 < n; j += 128) {
            const uint64_t x0 = src[j], x1 = src[j + 32], x2 = src[j + 64], x3 = src[j + 96];
            dst[j] = x0;
            dst[j + 32] = x1;
            dst[j + 64] = x2;
            dst[j + 96] = x3;
          }
          for (; j < n; j += 32) dst[j] = src[j];
        }
        off += tot;
      }
      if (t == sh.n_tiles - 1 && lane == 0) {
        write_global_header_f(a.out, sh.width, sh.n, sh.block_len, sh.n_blocks, off);
        *a.compressed_bytes = 32 + 16 * sh.n_blocks + 8 * off;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&C.empty[s]);
    }
    PROBE_ADD(12, wt0);
    PROBE_FLUSH;
    return;
  }

  // -------------------------------------------------------------- consumers
  uint4* const hdr_g = reinterpret_cast<uint4*>(a.out + 32);
  const uint32_t lgl = MULTI ? 5 - (__ffs(CB) - 1) : 5u;  // log2(32 / CB): lanes per block in the min / max
  PROBE_DECL;
  PROBE_T0(ct0);
  for (;;) {
    uint32_t q = 0;
    if (lane == 0) q = atomicAdd(&C.next, 1u);
    q = __shfl_sync(0xffffffffu, q, 0);
    const uint64_t i = q / NU;
    const uint32_t u = q % NU;
    if (i >= my) break;
    const uint32_t s = (uint32_t)(i % S);
    // the slot's fill for iteration i has been issued (so the barrier's
    // current phase is this fill's), then it has landed
    PROBE_T0(cf0);
    if (lane == 0) {
      uint32_t ns = 0;
      while (C.fseq[s] != i) {
        __nanosleep(ns);
        ns = ns ? min(ns * 2, 256u) : 32u;
      }
    }
    __syncwarp();
    mbar_wait_cmp<1>(&C.full[s], (uint32_t)(i / S) & 1u);
    PROBE_ADD(9, cf0);
    PROBE_T0(cm0);
    const uint64_t t = a.t_begin + blockIdx.x + i * nwork;
    const uint64_t b0 = t * TB;
    const uint32_t nblk = (uint32_t)min((uint64_t)TB, sh.n_blocks - b0);
    const uint32_t bf = u * CB;  // the claim's first block in the tile
    if (bf < nblk) {
      const uint32_t nvb = min(CB, nblk - bf);  // blocks of this claim
      const uint64_t gl = b0 + bf + nvb - 1;    // its last block (maybe the array's short last block)
      const uint32_t nb_last = (uint32_t)min((uint64_t)L, sh.n - gl * L);
      uint8_t* const base = slots + (size_t)s * sh.in_stride + (size_t)bf * bb;
      // a2: min / max -- a whole warp per block, or 32 / CB lanes per block
      uint32_t mn, mx;
      if (!MULTI)
        warp_minmax<V>(reinterpret_cast<const V*>(base), nb_last, mn, mx);
      else
        claim_minmax<V>(base, bb, lgl, nvb, nb_last, mn, mx);
      // a3: lane c 2^lgl holds block c's header and word count
      const uint32_t c = (uint32_t)lane >> lgl;
      const bool lead = ((uint32_t)lane & ((1u << lgl) - 1)) == 0 && c < nvb;
      const uint32_t nbc = c + 1 == nvb ? nb_last : L;
      const uint32_t kc = mx != mn ? k_of(bc, (uint64_t)(mx - mn) + 1) : 1u;
      const uint32_t nwc = mx != mn ? (nbc + kc - 1) / kc : 0u;
      uint32_t cc = 0;
      if (lead) {
        hdr_g[b0 + bf + c] = make_uint4(mx == mn ? CODEC_CONSTANT : CODEC_BASIC, mn, mx - mn, nwc);
        C.nw[s][bf + c] = nwc;
        __threadfence_block();
      }
      if (MULTI) __syncwarp();
      if (lane == 0) cc = atomicAdd(&C.cnt[s], nvb);
      cc = __shfl_sync(0xffffffffu, cc, 0);
      if (cc + nvb == nblk) {
        // the tile's last word counts: publish its aggregate now (a4)
        __threadfence_block();
        const volatile uint32_t* nwv = C.nw[s];
        uint32_t W = 0;
        for (uint32_t j = lane; j < nblk; j += 32) W += nwv[j];
        W = __reduce_add_sync(0xffffffffu, W);
        if (lane == 0) {
          C.cnt[s] = 0;
          if (a.server || t != 0) st_relaxed_u64(a.status + t, FLAG_AGG | W);
          else st_relaxed_u64(a.status + t, FLAG_PRE | W);
        }
      }
      PROBE_ADD(10, cm0);
      PROBE_T0(cp0);
      // a5: each block of the claim packed in place by the whole warp
      for (uint32_t cb = 0; cb < nvb; ++cb) {
        uint32_t bmn = mn, bmx = mx, k = kc, nw = nwc;
        if (MULTI) {
          const uint32_t src = cb << lgl;
          bmn = __shfl_sync(0xffffffffu, mn, src);
          bmx = __shfl_sync(0xffffffffu, mx, src);
          k = __shfl_sync(0xffffffffu, kc, src);
          nw = __shfl_sync(0xffffffffu, nwc, src);
        }
        if (bmn == bmx) continue;
        const uint32_t nb = cb + 1 == nvb ? nb_last : L;
        const uint64_t B = (uint64_t)(bmx - bmn) + 1;
        uint8_t* blk = base + (size_t)cb * bb;
        uint32_t done = 0;
        if (sizeof(V) == 2) {
          switch (k) {
#define POLY_C3K(KK)                                                    \
  case KK:                                                              \
    done = pack_inplace_k<KK>(blk, nb, (uint32_t)B, bmn);               \
    break;
            POLY_FOR_EACH_K16(POLY_C3K)
#undef POLY_C3K
            default:
              break;
          }
        }
        pack_inplace_words<V>(reinterpret_cast<V*>(blk), nb, k, B, bmn, done, nw);
      }
      PROBE_ADD(11, cp0);
#ifdef POLY_PROBE
      pacc[17] += nvb;
#endif
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&C.packed[s]);
  }
  PROBE_ADD(8, ct0);
  PROBE_FLUSH;
}

}  // namespace c3
}  // namespace polyk

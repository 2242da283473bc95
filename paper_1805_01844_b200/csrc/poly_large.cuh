// poly_large.cuh -- persistent pipeline kernels for large blocks (SURVEY.md
// Sec. 8(a) "large" regime: block > 32 KiB, e.g. cfg3's 65 536 x u32), one CTA
// per block at a time.  The look-back unit is a block.
//
// compress: the producer streams the block through shared memory twice in
//   sub-tiles of SV values (TMA bulk copies): sweep 0 computes the block's
//   min/max (a2) from HBM; then the block's B, k, n_words and header are known
//   (a3, a6), its aggregate is published and the writer warp looks back for
//   its payload offset (a4) while sweep 1 re-reads the block -- now from L2,
//   the CTA touched it microseconds earlier -- and Horner-packs every word
//   whose first value lies in the sub-tile straight to its place in the
//   stream (a5; a sub-tile carries a halo of 64 values for words that cross
//   its end).
// decompress: a scheduler warp takes a block, reads its header, publishes
//   its aggregate, looks back, then streams the words of each sub-tile
//   (TMA bulk) to the consumers, which extract the digits (a8) of the words
//   that overlap the sub-tile into a staging buffer; one bulk store per
//   sub-tile writes the values.
#pragma once
#include "poly_common.cuh"
#include "poly_word.cuh"
#include "poly_pipe.cuh"

namespace polyk {

constexpr uint32_t LG_HALO = 64;  // values: >= k_max - 1 (k <= 64)
// helper-warp waits of the large-block kernels (producer, writer, scheduler,
// store warp): parked (mbar_wait_helper) or polling
#ifndef POLY_LARGE_HELPER_PARK
#define POLY_LARGE_HELPER_PARK 1
#endif
#if POLY_LARGE_HELPER_PARK
#define POLY_LARGE_HWAIT mbar_wait_helper
#else
#define POLY_LARGE_HWAIT mbar_wait
#endif
// large-block consumer waits (input stage, published prefix, free staging)
#ifndef POLY_LARGE_CONSUMER_PARK
#define POLY_LARGE_CONSUMER_PARK 1  // measured: cfg3 decompress 1830 -> 1854, compress 2027 -> 2048
#endif
#if POLY_LARGE_CONSUMER_PARK
#define POLY_LARGE_CWAIT mbar_wait_helper
#else
#define POLY_LARGE_CWAIT mbar_wait
#endif

struct LargeShape {
  uint64_t n, Le, n_blocks;
  uint32_t block_len, width, vb;
  uint32_t SV;        // values per sub-tile
  uint32_t nsub;      // sub-tiles per (full) block
  uint32_t S;         // ring stages
  uint32_t stage;     // bytes per stage
  uint32_t o_in;      // ring offset
  uint32_t o_out;     // decompress: staging buffers (2 x SV values)
  uint32_t smem;
};

struct LargeArgs {
  const uint8_t* in;
  uint8_t* out;
  uint64_t* compressed_bytes;
  uint64_t in_bytes;
  uint32_t* status_out;
  uint64_t* status;   // look-back words, one per block
  uint32_t* ticket;
  uint32_t bulk;      // value array 16-byte aligned and Le * vb % 16 == 0
  uint32_t server;    // 1: the last CTA is the prefix server (poly_pipe.cuh prefix_server)
  LargeShape sh;
};

struct __align__(16) LargeCtl {
  uint64_t full_in[MAXS], empty_in[MAXS];
  uint64_t statsready[2], prefixready[2];
  // per stage
  uint64_t sb[MAXS];          // block of the stage (TILE_NONE = end)
  uint32_t spass[MAXS], ssub[MAXS], snv[MAXS], slast[MAXS];
  uint32_t sseq[MAXS];        // compress: the block's sequence number in this CTA (slot = seq & 1)
  uint64_t sj0[MAXS], sj1[MAXS], sP[MAXS];  // decompress: words of the stage, block payload offset
  uint32_t serr[MAXS];
  uint4 shdr[MAXS];           // decompress: block header
  DecConst sdc[MAXS];         // decompress: the block's digit-extraction constants
  // per block (double buffered)
  uint32_t bmin[2], bmax[2], bcnt[2];
  uint64_t blk[2];            // block index (TILE_NONE = end)
  uint32_t bvmin[2], bbm1[2], bk[2], bnw[2];
  uint64_t bP[2];
  uint64_t payload_words;
  uint32_t hdr_err, pad;
  // decompress: staging buffers (two) filled by the consumer warps (count NCW)
  // and freed by the store warp once its bulk store has read them
  uint64_t sfull[2], sfree[2];
  uint8_t* st_og[2];          // destination of the staging buffer's values
  uint32_t st_bytes[2];       // bytes (~0u: end of the stream)
};

__device__ __forceinline__ uint64_t blk_len(const LargeShape& sh, uint64_t b) {
  return min(sh.Le, sh.n - b * sh.Le);
}

// ======================================================================
// compress
// ======================================================================
template <typename V>
__global__ void __launch_bounds__(PT, 1) poly_compress_large(LargeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  if (a.server && blockIdx.x == gridDim.x - 1) {
    if (threadIdx.x < 32) prefix_server(a.status, a.sh.n_blocks);
    return;
  }
  LargeCtl& C = *reinterpret_cast<LargeCtl*>(smem);
  const LargeShape& sh = a.sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t S = sh.S;
  if (tid == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&C.full_in[s], 1);
      mbar_init(&C.empty_in[s], NCW);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&C.statsready[i], 1);
      mbar_init(&C.prefixready[i], 1);
      C.bmin[i] = 0xffffffffu;
      C.bmax[i] = 0u;
      C.bcnt[i] = 0u;
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == W_PROD) {
    // ---------------------------------------------------------- producer: each block twice
    uint32_t s = 0, ph = 0;
    auto next = [&]() {
      if (++s == S) {
        s = 0;
        ph ^= 1u;
      }
    };
    // Order: sweep 0 of block i+1 is issued before sweep 1 of block i, so the
    // wait for block i's payload offset overlaps the next block's min/max
    // (block i is still in L2: two blocks per SM fit).
    auto issue = [&](uint64_t b, uint32_t pass, uint32_t seq) {
      const uint64_t nb = blk_len(sh, b);
      const uint32_t nsub = (uint32_t)((nb + sh.SV - 1) / sh.SV);
      const uint8_t* base = a.in + b * sh.Le * sh.vb;
      for (uint32_t c = 0; c < nsub; ++c) {
        POLY_LARGE_HWAIT(&C.empty_in[s], ph ^ 1u);
        const uint64_t v0 = (uint64_t)c * sh.SV;
        const uint32_t nv = (uint32_t)min((uint64_t)sh.SV, nb - v0);
        const uint32_t halo = pass ? (uint32_t)min((uint64_t)LG_HALO, nb - v0 - nv) : 0u;
        const uint32_t bytes = (nv + halo) * sh.vb;
        uint8_t* dst = smem + sh.o_in + (size_t)s * sh.stage;
        const uint8_t* src = base + v0 * sh.vb;
        if (a.bulk) {
          if (lane == 0) {
            C.sb[s] = b;
            C.spass[s] = pass;
            C.ssub[s] = c;
            C.snv[s] = nv;
            C.slast[s] = c + 1 == nsub;
            C.sseq[s] = seq;
            const uint32_t b16 = bytes & ~15u;
            for (uint32_t j = b16; j < bytes; ++j) dst[j] = src[j];
            mbar_arrive_tx(&C.full_in[s], b16);
            if (b16) bulk_g2s(dst, src, b16, &C.full_in[s]);
          }
        } else {
          warp_copy(dst, src, bytes, lane);
          __syncwarp();
          if (lane == 0) {
            C.sb[s] = b;
            C.spass[s] = pass;
            C.ssub[s] = c;
            C.snv[s] = nv;
            C.slast[s] = c + 1 == nsub;
            C.sseq[s] = seq;
            mbar_arrive(&C.full_in[s]);
          }
        }
        next();
      }
    };
    uint64_t prev = TILE_NONE;
    for (uint32_t seq = 0;; ++seq) {
      uint32_t t32 = 0;
      if (lane == 0) t32 = atomicAdd(a.ticket, 1u);
      const uint64_t b = __shfl_sync(0xffffffffu, t32, 0);
      const bool more = b < sh.n_blocks;
      if (more) issue(b, 0, seq);
      if (prev != TILE_NONE) issue(prev, 1, seq - 1);
      if (!more) {
        POLY_LARGE_HWAIT(&C.empty_in[s], ph ^ 1u);
        if (lane == 0) {
          C.sb[s] = TILE_NONE;
          C.sseq[s] = seq;  // the writer's end marker goes to slot seq & 1
          mbar_arrive(&C.full_in[s]);
        }
        break;
      }
      prev = b;
    }
    return;
  }

  uint64_t* pay_g = reinterpret_cast<uint64_t*>(a.out + 32 + 16 * sh.n_blocks);
  if (warp == W_WRIT) {
    // ---------------------------------------------------------- writer: look-back per block
    for (uint32_t i = 0;; ++i) {
      const uint32_t bs = i & 1u, ph = (i >> 1) & 1u;
      POLY_LARGE_HWAIT(&C.statsready[bs], ph);
      const uint64_t b = C.blk[bs];
      if (b == TILE_NONE) break;
      const uint64_t W = C.bnw[bs];
      uint64_t P = 0;
      if (b != 0) {
        if (a.server) {
          P = wait_prefix(a.status, b);
        } else {
          P = lookback_wide(a.status, b);
          if (lane == 0) st_relaxed_u64(a.status + b, FLAG_PRE | ((P + W) & VAL_MASK));
        }
      }
      if (lane == 0) {
        C.bP[bs] = P;
        if (b == sh.n_blocks - 1) {
          write_global_header_f(a.out, sh.width, sh.n, sh.block_len, sh.n_blocks, P + W);
          *a.compressed_bytes = 32 + 16 * sh.n_blocks + 8 * (P + W);
        }
        mbar_arrive(&C.prefixready[bs]);
      }
      __syncwarp();
    }
    return;
  }
  if (warp >= NCW) return;

  // ------------------------------------------------------------ consumers
  uint4* hdr_g = reinterpret_cast<uint4*>(a.out + 32);
  for (uint32_t s = 0, ph = 0;; s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0)) {
    POLY_LARGE_CWAIT(&C.full_in[s], ph);
    const uint64_t b = C.sb[s];
    const uint32_t seq = C.sseq[s];
    if (b == TILE_NONE) {
      if (warp == 0 && lane == 0) {  // end marker for the writer
        const uint32_t bs = seq & 1u;
        C.blk[bs] = TILE_NONE;
        mbar_arrive(&C.statsready[bs]);
      }
      break;
    }
    const uint32_t pass = C.spass[s], c = C.ssub[s], nv = C.snv[s], last = C.slast[s];
    const V* sv = reinterpret_cast<const V*>(smem + sh.o_in + (size_t)s * sh.stage);
    const uint32_t nb = (uint32_t)blk_len(sh, b);  // < 2^24 (block <= 4 MiB)
    if (pass == 0) {
      const uint32_t bs = seq & 1u;
      // ---- a2: min / max of the sub-tile, warp slices, folded into the block's
      const uint32_t per = ((nv + NCW - 1) / NCW + 7) & ~7u;
      const uint32_t lo = min(nv, warp * per), hi = min(nv, lo + per);
      uint32_t mn, mx;
      warp_minmax<V>(sv + lo, hi - lo, mn, mx);
      if (lane == 0) {
        atomicMin(&C.bmin[bs], mn);
        atomicMax(&C.bmax[bs], mx);
        if (last) {
          __threadfence_block();
          if (atomicAdd(&C.bcnt[bs], 1u) == NCW - 1) {  // the block's last contribution
            __threadfence_block();
            const uint32_t vmin = C.bmin[bs], vmax = C.bmax[bs];
            const uint64_t B = (uint64_t)vmax - vmin + 1;
            const uint32_t k = B == 1 ? 1u : capacity_of(B);
            const uint64_t nw = B == 1 ? 0ull : ceil_div_small(nb, k);
            hdr_g[b] = make_uint4(B == 1 ? CODEC_CONSTANT : CODEC_BASIC, vmin, vmax - vmin, (uint32_t)nw);
            C.blk[bs] = b;
            C.bvmin[bs] = vmin;
            C.bbm1[bs] = vmax - vmin;
            C.bk[bs] = k;
            C.bnw[bs] = (uint32_t)nw;
            C.bmin[bs] = 0xffffffffu;  // reset for the block after next
            C.bmax[bs] = 0u;
            C.bcnt[bs] = 0u;
            st_relaxed_u64(a.status + b, (b == 0 && !a.server ? FLAG_PRE : FLAG_AGG) | nw);  // a4: aggregate
            mbar_arrive(&C.statsready[bs]);
          }
        }
      }
    } else {
      // ---- a5: words whose first value lies in this sub-tile, straight to HBM
      const uint32_t bs = seq & 1u;
      POLY_LARGE_CWAIT(&C.prefixready[bs], (seq >> 1) & 1u);
      const uint32_t bm1 = C.bbm1[bs];
      if (bm1 != 0) {
        const uint32_t vmin = C.bvmin[bs], k = C.bk[bs];
        const uint64_t B = (uint64_t)bm1 + 1;
        const uint32_t v0 = c * sh.SV;
        const uint32_t jb = ceil_div_small(v0, k);
        const uint32_t je = min(C.bnw[bs], ceil_div_small(v0 + nv, k));
        uint64_t* dst = pay_g + C.bP[bs];
        // two words per thread per step: two independent Horner chains
        for (uint32_t j = jb + (uint32_t)(warp * 32 + lane); j < je; j += 2 * PC) {
          const uint32_t j2 = j + PC, f1 = j * k, f2 = j2 * k;
          const uint32_t m1 = min(k, nb - f1);
          if (j2 < je && m1 == k && f2 + k <= nb && B < (1ull << 32)) {
            const V* p1 = sv + (f1 - v0);
            const V* p2 = sv + (f2 - v0);
            const uint32_t Bu = (uint32_t)B;
            uint64_t s1 = 0, s2 = 0;
#pragma unroll 4
            for (int i = (int)k - 1; i >= 0; --i) {
              s1 = s1 * Bu + ((uint32_t)p1[i] - vmin);
              s2 = s2 * Bu + ((uint32_t)p2[i] - vmin);
            }
            dst[j] = s1;
            dst[j2] = s2;
          } else {
            dst[j] = pack_word64<V>(sv + (f1 - v0), m1, B, vmin);
            if (j2 < je) dst[j2] = pack_word64<V>(sv + (f2 - v0), min(k, nb - f2), B, vmin);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&C.empty_in[s]);
  }
}

// ======================================================================
// decompress
// ======================================================================
__device__ __forceinline__ uint32_t check_global_header_l(const LargeArgs& a, uint64_t* pw) {
  const LargeShape& sh = a.sh;
  *pw = 0;
  if (a.in_bytes < 32) return POLY_ST_LENGTH;
  const uint4 h0 = reinterpret_cast<const uint4*>(a.in)[0];
  const uint4 h1 = reinterpret_cast<const uint4*>(a.in)[1];
  const uint64_t n = (uint64_t)h0.z | ((uint64_t)h0.w << 32);
  const uint64_t pb = (uint64_t)h1.z | ((uint64_t)h1.w << 32);
  if (h0.x != 0x43594c50u) return POLY_ST_BAD_MAGIC;
  if ((h0.y & 0xffu) != 2u) return POLY_ST_BAD_VERSION;
  if (((h0.y >> 8) & 0xffu) != 0u || ((h0.y >> 16) & 0xffu) != sh.width || (h0.y >> 24) != 0u || n != sh.n ||
      h1.x != sh.block_len || h1.y != (uint32_t)sh.n_blocks)
    return POLY_ST_HEADER_MISMATCH;
  // overflow-safe: in_bytes must hold the headers before pb is compared with the rest
  if ((pb & 7) != 0 || a.in_bytes < 32 + 16 * sh.n_blocks || pb != a.in_bytes - (32 + 16 * sh.n_blocks))
    return POLY_ST_LENGTH;
  *pw = pb >> 3;
  return 0;
}

template <typename V>
__global__ void __launch_bounds__(PT, 1) poly_decompress_large(LargeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  if (a.server && blockIdx.x == gridDim.x - 1) {
    uint64_t pw;
    if (threadIdx.x < 32 && check_global_header_l(a, &pw) == 0) prefix_server(a.status, a.sh.n_blocks);
    return;
  }
  LargeCtl& C = *reinterpret_cast<LargeCtl*>(smem);
  const LargeShape& sh = a.sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t S = sh.S;
  if (tid == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&C.full_in[s], 1);
      mbar_init(&C.empty_in[s], NCW);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&C.sfull[q], NCW);
      mbar_init(&C.sfree[q], 1);
    }
    mbar_fence_init();
    uint64_t pw;
    C.hdr_err = check_global_header_l(a, &pw);
    C.payload_words = pw;
  }
  __syncthreads();
  if (C.hdr_err) {
    if (blockIdx.x == 0 && tid == 0) atomicOr(a.status_out, C.hdr_err);
    return;
  }
  const uint4* hdr_g = reinterpret_cast<const uint4*>(a.in + 32);
  const uint64_t* pay_g = reinterpret_cast<const uint64_t*>(a.in + 32 + 16 * sh.n_blocks);

  if (warp == W_PROD) {
    // ---------------------------------------------------------- store warp
    // Bulk-stores each staging buffer once every consumer warp has filled it,
    // then frees it: the consumers never wait for one another.
    for (uint32_t i = 0;; ++i) {
      const uint32_t q = i & 1u;
      POLY_LARGE_HWAIT(&C.sfull[q], (i >> 1) & 1u);
      const uint32_t bytes = C.st_bytes[q];
      if (bytes == ~0u) break;
      uint8_t* og = C.st_og[q];
      const uint8_t* src = smem + sh.o_out + (size_t)q * sh.SV * sh.vb;
      if (a.bulk) {
        const uint32_t b16 = bytes & ~15u;
        if (lane == 0 && b16) bulk_s2g(og, src, b16);
        for (uint32_t j = b16 + lane; j < bytes; j += 32) og[j] = src[j];
        if (lane == 0) {
          bulk_commit();
          bulk_wait_read<0>();
        }
      } else {
        for (uint32_t j = lane; j < bytes; j += 32) og[j] = src[j];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&C.sfree[q]);
    }
    if (a.bulk && lane == 0) bulk_wait_all<0>();
    return;
  }
  if (warp == W_WRIT) {
    // ---------------------------------------------------------- scheduler
    const uint64_t pw = C.payload_words;
    uint32_t s = 0, ph = 0;
    // One block ahead: the next block's ticket is taken and its aggregate
    // published before this block waits for its payload offset, so the
    // prefix frontier never waits on a scheduler that is itself waiting.
    auto take = [&](uint4& hh) -> uint64_t {
      uint32_t t32 = 0;
      if (lane == 0) t32 = atomicAdd(a.ticket, 1u);
      const uint64_t bb = __shfl_sync(0xffffffffu, t32, 0);
      if (bb < sh.n_blocks) {
        hh = hdr_g[bb];
        if (lane == 0) st_relaxed_u64(a.status + bb, (bb == 0 && !a.server ? FLAG_PRE : FLAG_AGG) | (hh.w & VAL_MASK));
      }
      return bb;
    };
    uint4 hn = make_uint4(0, 0, 0, 0);
    uint64_t bn = take(hn);
    while (true) {
      const uint64_t b = bn;
      const uint4 h = hn;
      if (b >= sh.n_blocks) {
        if (lane == 0) {
          POLY_LARGE_HWAIT(&C.empty_in[s], ph ^ 1u);
          C.sb[s] = TILE_NONE;
          mbar_arrive(&C.full_in[s]);
        }
        break;
      }
      bn = take(hn);
      const uint64_t nb = blk_len(sh, b);
      const uint64_t W = h.w;
      uint64_t P = 0;
      if (b != 0) {
        if (a.server) {
          P = wait_prefix(a.status, b);
        } else {
          P = lookback_wide(a.status, b);
          if (lane == 0) st_relaxed_u64(a.status + b, FLAG_PRE | ((P + W) & VAL_MASK));
        }
      }
      const uint32_t k = (h.x == CODEC_BASIC && h.z != 0) ? capacity_of((uint64_t)h.z + 1) : 1u;
      uint32_t e = 0;
      // check_block_hdr takes a 32-bit block length: compare in 64 bits here
      if (h.x == CODEC_CONSTANT) {
        if (h.z != 0 || h.w != 0) e |= POLY_ST_NWORDS;
        if ((uint64_t)h.y > ((sh.width == 32) ? 0xffffffffull : ((1ull << sh.width) - 1))) e |= POLY_ST_OVERFLOW;
      } else if (h.x != CODEC_BASIC) {
        e |= POLY_ST_BAD_CODEC;
      } else if (h.z == 0 || (uint64_t)h.y + h.z > ((sh.width == 32) ? 0xffffffffull : ((1ull << sh.width) - 1))) {
        e |= POLY_ST_OVERFLOW;
      } else if (W == 0 || (W - 1) * k >= nb || W * k < nb) {
        e |= POLY_ST_NWORDS;
      }
      if (P + W > pw) e |= POLY_ST_LENGTH;
      if (b == sh.n_blocks - 1 && P + W != pw) e |= POLY_ST_LENGTH;
      const uint32_t nsub = (uint32_t)((nb + sh.SV - 1) / sh.SV);
      DecConst dc;  // once per block (B > 2^16 takes the slow exact path)
      if (lane == 0 && !e && h.x == CODEC_BASIC) dc = dec_const_of((uint64_t)h.z + 1);
      for (uint32_t c = 0; c < nsub; ++c) {
        if (lane == 0) {
          POLY_LARGE_HWAIT(&C.empty_in[s], ph ^ 1u);
          const uint64_t v0 = (uint64_t)c * sh.SV;
          const uint32_t nv = (uint32_t)min((uint64_t)sh.SV, nb - v0);
          uint64_t j0 = 0, j1 = 0;
          if (!e && h.x == CODEC_BASIC) {
            j0 = v0 / k;
            j1 = min(W, (v0 + nv + k - 1) / k);
          }
          C.sb[s] = b;
          C.ssub[s] = c;
          C.snv[s] = nv;
          C.sj0[s] = j0;
          C.sj1[s] = j1;
          C.sP[s] = P + j0;
          C.serr[s] = e;
          C.shdr[s] = h;
          C.sdc[s] = dc;
          uint8_t* dst = smem + sh.o_in + (size_t)s * sh.stage;
          if (j1 > j0) {
            const uint64_t a0 = (P + j0) & ~1ull, hw = P + j1;
            uint64_t a1 = min((hw + 1) & ~1ull, pw & ~1ull);
            if (a1 < a0) a1 = a0;
            for (uint64_t w = a1; w < hw; ++w) reinterpret_cast<uint64_t*>(dst)[w - a0] = ldg_nc_u64(pay_g + w);
            const uint32_t bytes = (uint32_t)(8 * (a1 - a0));
            mbar_arrive_tx(&C.full_in[s], bytes);
            if (bytes) bulk_g2s(dst, pay_g + a0, bytes, &C.full_in[s]);
          } else {
            mbar_arrive(&C.full_in[s]);
          }
        }
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  if (warp >= NCW) return;

  // ------------------------------------------------------------ consumers
  uint32_t err = 0;
  for (uint32_t s = 0, ph = 0, i = 0;; s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0), ++i) {
    const uint32_t s2 = i & 1u;
    POLY_LARGE_CWAIT(&C.full_in[s], ph);
    const uint64_t b = C.sb[s];
    if (b == TILE_NONE) {
      POLY_LARGE_CWAIT(&C.sfree[s2], ((i >> 1) & 1u) ^ 1u);
      if (tid == 0) C.st_bytes[s2] = ~0u;  // end marker for the store warp
      __syncwarp();
      if (lane == 0) mbar_arrive(&C.sfull[s2]);
      break;
    }
    const uint32_t c = C.ssub[s], nv = C.snv[s], e = C.serr[s];
    const uint64_t j0 = C.sj0[s], j1 = C.sj1[s];
    const uint4 h = C.shdr[s];
    const uint64_t* words = reinterpret_cast<const uint64_t*>(smem + sh.o_in + (size_t)s * sh.stage) + (C.sP[s] & 1);
    V* ob = reinterpret_cast<V*>(smem + sh.o_out + (size_t)s2 * sh.SV * sh.vb);
    const uint64_t nb = blk_len(sh, b);
    const uint64_t v0 = (uint64_t)c * sh.SV;
    if (tid == 0 && c == 0) err |= e;
    POLY_LARGE_CWAIT(&C.sfree[s2], ((i >> 1) & 1u) ^ 1u);  // the buffer's store of two sub-tiles ago has read it
    if (!e) {
      if (h.x == CODEC_CONSTANT) {
        for (uint32_t i2 = tid; i2 < nv; i2 += PC) ob[i2] = (V)h.y;
      } else {
        const DecConst dc = C.sdc[s];
        const uint32_t k = dc_k(dc);
        const uint32_t nb32 = (uint32_t)nb, v032 = (uint32_t)v0, jn = (uint32_t)(j1 - j0), j032 = (uint32_t)j0;
        for (uint32_t jj = tid; jj < jn; jj += PC) {
          const uint32_t first = (j032 + jj) * k;  // < 2^24: block <= 4 MiB
          const uint32_t m = min(k, nb32 - first);
          if (first >= v032 && first + m <= v032 + nv) {  // the word lies inside the sub-tile
            err |= decode_any<V>(words[jj], dc, h.z, m, h.y, ob + (first - v032));
          } else {  // crosses a sub-tile edge: decode to scratch, keep the part inside
            V tmp[64];
            err |= decode_any<V>(words[jj], dc, h.z, m, h.y, tmp);
            for (uint32_t q = 0; q < m; ++q) {
              const uint32_t p = first + q;
              if (p >= v032 && p < v032 + nv) ob[p - v032] = tmp[q];
            }
          }
        }
      }
    }
    if (a.bulk) fence_proxy_async_smem();
    if (tid == 0) {
      C.st_og[s2] = a.out + (b * sh.Le + v0) * sh.vb;
      C.st_bytes[s2] = nv * sh.vb;
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&C.sfull[s2]);
      mbar_arrive(&C.empty_in[s]);
    }
  }
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0 && err) atomicOr(a.status_out, err);
}

}  // namespace polyk

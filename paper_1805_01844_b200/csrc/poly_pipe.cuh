// poly_pipe.cuh -- persistent, warp-specialized pipeline kernels for blocks of
// up to PIPE_MAX_BLOCK bytes (cfg2, cfg4, cfg5).
//
// One CTA per SM (persistent grid).  A tile is TB consecutive blocks; tiles
// are handed out in increasing order by an atomic ticket, so the single-pass
// decoupled look-back over tiles (a4 / a7) always terminates.
//
// compress (warps 0..NCW-1 consumers, NCW producer, NCW+1 writer):
//   producer : ticket -> 1-D TMA bulk copy of the tile's values into a ring of
//              S shared-memory stages (mbarrier complete_tx)
//   consumers: per-block min/max, B, k, n_words (a2, a3); block headers go
//              straight to global memory (fixed offsets); CTA scan of n_words;
//              publish the tile aggregate; Horner-pack the words (a5) into one
//              of two staging buffers
//   writer   : look back for the tile's payload offset, publish the inclusive
//              prefix, copy the staged words to the stream with coalesced
//              16-byte stores (a4, a6); the last tile writes the global header
// decompress (warps 0..NCW-1 consumers, NCW header loader, NCW+1 look-back):
//   header loader : ticket -> TMA bulk copy of the tile's block headers into
//              one of SH header stages (deep prefetch: headers are small)
//   look-back warp: n_words sum and in-tile offsets, publish the aggregate,
//              look back, then TMA bulk copy of the tile's payload words into
//              a shared-memory ring buffer (allocated by size, not worst case)
//   consumers: validate headers (a9), extract digits without integer divides
//              (a8) into a staging buffer, TMA bulk store of the decoded tile.
#pragma once
#include "poly_common.cuh"
#include "poly_word.cuh"
#include "poly_kword.cuh"

namespace polyk {

#ifndef POLY_NCW
#define POLY_NCW 16  // consumer warps per CTA
#endif
#ifndef POLY_CTAS
#define POLY_CTAS 1  // CTAs per SM the shared-memory plan targets
#endif

// POLY_TRACE (timing experiments only, a separate library variant): per CTA
// and per tile (the CTA's i-th tile), globaltimer stamps of pipeline events,
// read back with poly_trace_dump (profiles/trace_run.py).
#ifdef POLY_TRACE
constexpr uint32_t TRACE_TILES = 1024, TRACE_EV = 16;
__device__ uint64_t g_trace[160 * TRACE_TILES * TRACE_EV];
__device__ __forceinline__ void trace_ev(uint32_t i, int e, uint64_t v = ~0ull) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (i < TRACE_TILES) g_trace[((size_t)blockIdx.x * TRACE_TILES + i) * TRACE_EV + e] = v == ~0ull ? t : v;
}
#define TRACE(i, e) trace_ev((i), (e))
#define TRACE_V(i, e, v) trace_ev((i), (e), (v))
#else
#define TRACE(i, e)
#define TRACE_V(i, e, v)
#endif
constexpr int NCW = POLY_NCW;      // consumer warps
constexpr int PC = NCW * 32;       // consumer threads
// Timing experiments (skip compute / the look-back / stores; the output is
// then wrong) exist only in a separate variant library built with
// -DPOLY_TIMING (profiles/); in the product library DBG(x) is the constant 0
// and the experiment branches compile away.
#ifdef POLY_TIMING
#define DBG(a, bit) ((a).debug & (bit))
#else
#define DBG(a, bit) 0u
#endif

#ifndef POLY_NLB_MAX
#define POLY_NLB_MAX 4
#endif
constexpr int NLB_MAX = POLY_NLB_MAX;  // look-back warps per CTA (upper bound)
constexpr int PT = PC + 32 * (2 + NLB_MAX);  // + producer, header-sum and look-back / writer warps
constexpr int W_PROD = NCW;        // warp index of the producer / header issuer
constexpr int W_WRIT = NCW + 1;    // first writer (compress) / look-back (decompress) warp
constexpr int W_HSUM = NCW + 2;    // decompress: header-sum warp (compress: a writer)
constexpr int W_LBX = NCW + 3;     // decompress: look-back warps 2 .. NLB_MAX
// PipeArgs.nlb = look-back warps in use: compress writers W_WRIT .. W_WRIT +
// nlb - 1 (nlb <= NLB_MAX + 1), decompress W_WRIT and W_LBX .. (nlb <= NLB_MAX)
// (host: POLY_LB env, defaults in poly.cu).
constexpr int MAXS = 8;            // max ring stages
constexpr int BPT_MAX = 2;         // map 0: blocks per consumer thread
constexpr uint32_t PIPE_MAX_BLOCK = 32768;  // bytes per block handled here
constexpr uint32_t MAP0_MAX_BLOCK = 128;    // bytes per block for one consumer thread per block
constexpr uint32_t CACHE_B = 512;  // shared-memory cache of per-base constants
constexpr uint64_t TILE_NONE = ~0ull;
constexpr int BAR_CONS = 1;        // named barrier id of the consumer warps

struct PipeShape {
  uint64_t n, Le, n_blocks, n_tiles;
  uint32_t block_len, width, vb;
  uint32_t TB;          // blocks per tile
  uint32_t map;         // 0: one consumer thread per block; 1: G warps per block
  uint32_t bpt;         // map 0: blocks per consumer thread
  uint32_t G;           // map 1: warps per block (power of two)
  uint32_t Lp;          // map 1: values per part (G parts per block)
  uint32_t tile_bytes;  // value bytes of a full tile
  uint32_t words_cap;   // payload words a tile can hold (any valid stream)
  uint32_t S;           // ring stages (compress input / decompress header stages)
  uint32_t in_stride;   // bytes per stage
  uint32_t out_stride;  // bytes per staging buffer (map 0: per consumer warp; map 1: two per CTA)
  uint32_t o_off;       // decompress: offset of OFF[] inside a header stage (HDR at 0)
  uint32_t o_cache;     // offset of the base-constant cache
  uint32_t o_in, o_out; // offsets of the stages and the staging buffers
  uint32_t o_ring, ring_bytes;  // decompress: payload ring; compress: word slots
  uint32_t wrings;      // compress map 0: per-warp word rings in use (see plan_pipe)
  uint32_t nslot;       // compress: records in flight (<= MAXR)
  uint32_t slot_bytes;  // compress: bytes of each consumer warp's word ring
  uint32_t ncw;         // consumer warps of the kernel instantiation this shape is for
  uint32_t c3;          // compress: the in-place one-warp-per-block kernel (poly_cmp3.cuh)
  uint32_t smem;        // dynamic shared memory bytes
};

struct PipeArgs {
  const uint8_t* in;        // compress: values; decompress: stream
  uint8_t* out;             // compress: stream; decompress: values
  uint64_t* compressed_bytes;
  uint64_t in_bytes;        // decompress: stream length
  uint32_t* status_out;     // decompress: caller's status word
  uint64_t* status;         // look-back words, one per tile
  uint32_t* ticket;
  uint32_t bulk;            // value array 16-byte aligned and tile_bytes % 16 == 0
  uint32_t tma_shift;       // compress: array aligned, tiles not: TMA of the 16-byte aligned superset
  uint32_t debug;           // POLY_TIMING builds only (read through DBG): 1 skip compute, 2 skip look-back, ...
  uint32_t nlb;             // look-back / writer warps in use
  uint32_t server;          // 1: the last CTA is the prefix server (see prefix_server)
  uint64_t t_begin, t_end;  // compress: the tiles of this launch (chunked host calls)
  PipeShape sh;
};

constexpr int MAXR = 8;            // compress: word slots (tiles between consumers and writer)
constexpr int MAXSEG = 256;        // segments per tile (map 0: warp groups of 32 blocks; map 1: blocks)

struct __align__(16) PipeCtl {
  uint64_t full_in[MAXS], empty_in[MAXS];    // stage filled (1 + tx) / released (NCW warps)
  uint64_t hbar[MAXS], aggr[MAXS];           // decompress: headers landed / aggregate published
  uint64_t rec_full[MAXR];    // compress: record ready for the writer
  uint64_t rec_cnt[MAXR];     // compress WARP_RINGS: every warp's word count of the record known
  uint64_t tkt[MAXS];       // ticket of the tile held by each stage
  uint64_t W[MAXS];         // decompress: payload words of the stage's tile
  uint64_t P[MAXS];         // decompress: payload word prefix of the stage's tile
  uint64_t ring_end[MAXS];  // decompress: ring position after the stage's payload
  uint32_t ring_off[MAXS];  // decompress: byte offset of the stage's payload in the ring
  uint32_t err[MAXS];       // decompress: tile-level status bits
  uint32_t shift[MAXS];     // compress: offset of the tile's first value in its stage (tma_shift)
  uint32_t done_cnt[MAXS];  // decompress: warps done with the stage
  uint32_t gnext[MAXS];     // decompress: next group (map 0) / block (map 1, G = 1) of the stage to claim
  uint64_t tfull[4], tfree[4];  // decompress maps 1, 2: staging tile filled (NCW warps) / read by its bulk store
  uint8_t* t_og[4];             // decompress maps 1, 2: destination of the staging tile
  uint32_t t_bytes[4];          // decompress maps 1, 2: its bytes (~0u: end)
  uint64_t rec_t[MAXR], rec_W[MAXR], rec_end[MAXR];  // compress: staged tiles
  uint64_t rec_empty[MAXR];
  uint32_t rec_off[MAXR];
  volatile uint32_t wdone;  // compress: records completed, in order
  uint32_t scan[2][32];      // per consumer warp (NCW <= 32)
  uint64_t payload_words;
  volatile uint64_t ring_tail;  // decompress: ring bytes released by the consumers
  volatile uint32_t lb_seq;     // decompress: next stage to take ring space
  uint64_t ring_head;           // decompress: ring bytes handed out
  uint32_t ring_hpos, pad2;     // decompress: ring_head modulo the ring size
  uint32_t hdr_err, pad;
  uint32_t nwL[68];             // compress map 0: ceil(L / k) for k = 1..64
  // compress map 0 with one block per consumer thread (bpt = 1): per-warp word
  // rings; record r holds each warp's word count, ring offset and ring end
  uint32_t rw_words[MAXR][32], rw_off[MAXR][32];
  uint64_t rw_end[MAXR][32];
  volatile uint64_t wtail[32];  // per-warp ring bytes released (in record order)
  uint32_t smin[256], smax[256];                        // map 1: partial min / max per segment
  uint32_t bvmin[256], bbm1[256], bnw[256], boff[256];  // map 1: per-block results
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx)
               : "memory");
}
// Wait for the phase with the given parity to complete.  The suspend-time hint
// parks the thread in the barrier unit instead of spinning on issue slots.
#ifndef POLY_SUSPEND_NS
#define POLY_SUSPEND_NS 0x989680u
#endif
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity);
#ifndef POLY_CMP_WARP_RINGS
#define POLY_CMP_WARP_RINGS 1  // compress map 0 (bpt = 1): per-warp word rings, no CTA scan
#endif
#ifndef POLY_WAIT_MIN
#define POLY_WAIT_MIN 32  // first sleep (ns) of a barrier poll
#endif
#ifndef POLY_WAIT_BACKOFF
#define POLY_WAIT_BACKOFF 256  // max sleep (ns) between barrier polls; 0: hardware-suspended try_wait (measured: 256 > 512, 1024)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if POLY_WAIT_BACKOFF > 0
  // Poll with an exponential sleep: a waiting warp (a consumer ahead of the
  // others, an idle helper) then costs a few issue slots per microsecond
  // instead of re-polling on every barrier event of the SM.
  uint32_t ns = POLY_WAIT_MIN;
  while (!mbar_test(bar, parity)) {
    __nanosleep(ns);
    ns = min(ns * 2, (uint32_t)POLY_WAIT_BACKOFF);
  }
#elif POLY_SUSPEND_NS > 0
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"((uint32_t)POLY_SUSPEND_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
// Decompress helper-warp waits (header issuer, header sum, look-back, tile
// store): POLY_HELPER_WAIT = 1 parks them in the barrier unit (try_wait with
// a suspend-time hint) instead of polling, leaving the issue slots to the
// consumer warps (measured: cfg5 decompress +6 %; the compress writers react
// too late when parked, they keep polling).
#ifndef POLY_HELPER_WAIT
#define POLY_HELPER_WAIT 1
#endif
__device__ __forceinline__ void mbar_wait_helper(uint64_t* bar, uint32_t parity) {
#if POLY_HELPER_WAIT
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITH_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITH_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
#else
  mbar_wait(bar, parity);
#endif
}
// Decompress consumer waits (next stage's payload, a free staging tile):
// parked like the helpers (measured against the polling wait: cfg5 1829 ->
// 1898 GB/s, cfg4 1331 -> 1338, cfg2 unchanged; the compress consumers lose
// with it and keep polling).
#ifndef POLY_DEC_PARK
#define POLY_DEC_PARK 1
#endif
// Compress waits: the producer's free stage, the consumers' next input stage
// and their record slots, each parked (1) or polling (0); the writers poll
// (parked they react too late).  Measured, all three parked: cfg2 compress
// 2110 -> 2154 GB/s, cfg4 1949 -> 1959, cfg5 2378 -> 2388.
#ifndef POLY_CMP_PARK_PROD
#define POLY_CMP_PARK_PROD 1
#endif
#ifndef POLY_CMP_PARK_IN
#define POLY_CMP_PARK_IN 1
#endif
#ifndef POLY_CMP_PARK_REC
#define POLY_CMP_PARK_REC 1
#endif
#ifndef POLY_WRITER_BACKOFF
#define POLY_WRITER_BACKOFF POLY_WAIT_BACKOFF  // max sleep (ns) of a compress writer's poll
#endif
__device__ __forceinline__ void mbar_wait_writer(uint64_t* bar, uint32_t parity) {
  uint32_t ns = POLY_WAIT_MIN;
  while (!mbar_test(bar, parity)) {
    __nanosleep(ns);
    ns = min(ns * 2, (uint32_t)POLY_WRITER_BACKOFF);
  }
}
template <int PARK>
__device__ __forceinline__ void mbar_wait_cmp(uint64_t* bar, uint32_t parity) {
  if (PARK)
    mbar_wait_helper(bar, parity);
  else
    mbar_wait(bar, parity);
}
__device__ __forceinline__ void mbar_wait_dec(uint64_t* bar, uint32_t parity) {
#if POLY_DEC_PARK
  mbar_wait_helper(bar, parity);
#else
  mbar_wait(bar, parity);
#endif
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// 1-D bulk copy global -> shared (both 16-byte aligned, bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 1-D bulk copy shared -> global (bulk group).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
template <int NW>
__device__ __forceinline__ void cons_bar() { asm volatile("bar.sync %0, %1;" ::"n"(BAR_CONS), "n"(NW * 32) : "memory"); }
// Named barrier of the G consecutive warps that share one block (map 1, G > 1).
__device__ __forceinline__ void group_bar(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t x, uint32_t* total) {
  const uint32_t inc = warp_incl_scan(x);
  *total = __shfl_sync(0xffffffffu, inc, 31);
  return inc - x;
}

// Exclusive scan of x over the PC consumer threads; *total = sum.  `buf`
// alternates between calls (a call's barrier protects the buffer of the
// call before it).
template <int NW>
__device__ __forceinline__ uint32_t cons_scan(uint32_t x, uint32_t* total, uint32_t* buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t inc = warp_incl_scan(x);
  if (lane == 31) buf[warp] = inc;
  cons_bar<NW>();
  const uint32_t ws = lane < NW ? buf[lane] : 0u;
  const uint32_t wi = warp_incl_scan(ws);
  *total = __shfl_sync(0xffffffffu, wi, NW - 1);
  const uint32_t wex = __shfl_sync(0xffffffffu, wi - ws, warp);
  return wex + inc - x;
}

// ------------------------------------------------------------------ base constants
// Shared-memory cache of the per-base table for B <= CACHE_B (SoA so that
// lanes with nearby bases hit different banks).  cmeta = DecConst.meta
// (k | log2b << 8 | t32 << 16 | h << 24).
// Decoder constants of one base, with the L-dependent shape of a full block
// (48 bytes: three 16-byte shared-memory loads).
struct __align__(16) DecEnt {
  uint64_t Rl, Rh;  // fraction reciprocal (DecConst)
  uint64_t Wmax;    // B^k - 1
  uint64_t P;       // B^(k - mt): premultiplier of an L-block's top word (1 if full)
  uint32_t meta;    // as DecConst
  uint32_t nwL;     // words of an L-block = ceil(L / k)
  uint32_t mt;      // digits of an L-block's top word
  uint32_t pad;
};

struct BaseCache {
  DecEnt* E;     // decompress
  uint32_t* meta;  // compress
  uint64_t* D;   // compress: B^h
  uint32_t* G;   // compress: 1 + B + ... + B^(h-1) mod 2^32
};

__device__ __forceinline__ BaseCache cache_at(uint8_t* base, bool dec) {
  BaseCache c;
  uint64_t* p = reinterpret_cast<uint64_t*>(base);
  if (dec) {
    c.E = reinterpret_cast<DecEnt*>(base);
    c.meta = nullptr;
    c.D = nullptr;
    c.G = nullptr;
  } else {
    c.E = nullptr;
    c.D = p;
    c.meta = reinterpret_cast<uint32_t*>(p + (CACHE_B + 1));
    c.G = c.meta + (CACHE_B + 1);
  }
  return c;
}
__host__ __device__ constexpr uint32_t cache_bytes(bool dec) {
  return dec ? (uint32_t)(sizeof(DecEnt) * (CACHE_B + 1) + 15) / 16 * 16
             : (uint32_t)(8 * (CACHE_B + 1) + 8 * (CACHE_B + 1) + 15) / 16 * 16;
}
__device__ __forceinline__ void cache_fill(const BaseCache& c, bool dec, uint64_t L = 0) {
  for (uint32_t B = threadIdx.x; B <= CACHE_B; B += blockDim.x) {
    const DecConst d = g_dtab[B];
    if (dec) {
      DecEnt e;
      e.Rl = d.Rl;
      e.Rh = d.Rh;
      e.Wmax = d.Wmax;
      e.meta = d.meta;
      e.P = 1;
      e.nwL = 0;
      e.mt = 0;
      e.pad = 0;
      const uint32_t k = d.meta & 0xffu;
      if (B >= 2 && L != 0 && k != 0) {
        e.nwL = (uint32_t)((L + k - 1) / k);
        e.mt = (uint32_t)(L - (uint64_t)(e.nwL - 1) * k);  // 1 .. k
        for (uint32_t i = e.mt; i < k; ++i) e.P *= B;
      }
      c.E[B] = e;
    } else {
      c.meta[B] = d.meta;
      const uint32_t h = d.meta >> 24;
      uint64_t D = 1;
      uint32_t G = 0;
      for (uint32_t i = 0; i < h; ++i) {
        G = G * B + 1u;
        D *= B;
      }
      c.D[B] = D;
      c.G[B] = G;
    }
  }
}
// Chunk constants of the pack: D = B^h and G = 1 + B + ... + B^(h-1) mod 2^32.
__device__ __forceinline__ void chunk_consts(const BaseCache& c, uint32_t B, uint32_t h, uint64_t& D, uint32_t& G) {
  if (B <= CACHE_B) {
    D = c.D[B];
    G = c.G[B];
    return;
  }
  D = 1;
  G = 0;
  for (uint32_t i = 0; i < h; ++i) {
    G = G * B + 1u;
    D *= B;
  }
}
// k (values per u64 word) for 2 <= B <= 2^32 (compress / decompress caches).
__device__ __forceinline__ uint32_t k_of(const BaseCache& c, uint64_t B) {
  if (B <= CACHE_B) return c.meta[B] & 0xffu;
  return capacity_of(B);
}
__device__ __forceinline__ uint32_t dk_of(const BaseCache& c, uint64_t B) {
  if (B <= CACHE_B) return c.E[B].meta & 0xffu;
  return capacity_of(B);
}
// k and h (values per 32-bit chunk) for 2 <= B <= 2^16.
__device__ __forceinline__ uint32_t kh_of16(const BaseCache& c, uint32_t B) {
  const uint32_t m = B <= CACHE_B ? c.meta[B] : g_dtab[B].meta;
  return (m & 0xffu) | ((m >> 16) & 0xff00u);  // k | h << 8
}
__device__ __forceinline__ DecConst dconst_of(const BaseCache& c, uint64_t B) {
  if (B <= CACHE_B) {
    const DecEnt& e = c.E[B];
    DecConst d;
    d.Wmax = e.Wmax;
    d.Rl = e.Rl;
    d.Rh = e.Rh;
    d.meta = e.meta;
    d.pad = 0;
    return d;
  }
  return dec_const_of(B);
}

// min / max of n values at s by one warp (16-byte vector loads when aligned).
template <typename V>
__device__ __forceinline__ void warp_minmax(const V* s, uint32_t n, uint32_t& mn, uint32_t& mx) {
  const int lane = threadIdx.x & 31;
  mn = 0xffffffffu;
  mx = 0u;
  uint32_t i0 = 0;
  if ((reinterpret_cast<uintptr_t>(s) & 15) == 0) {
    const uint4* q = reinterpret_cast<const uint4*>(s);
    constexpr uint32_t PER = 16 / sizeof(V);
    const uint32_t nq = n / PER;
    if (sizeof(V) == 2) {
      uint32_t a0 = 0xffffffffu, a1 = 0u;
#pragma unroll 4
      for (uint32_t i = lane; i < nq; i += 32) {
        const uint4 t = q[i];
        a0 = __vimin3_u16x2(a0, t.x, t.y);
        a0 = __vimin3_u16x2(a0, t.z, t.w);
        a1 = __vimax3_u16x2(a1, t.x, t.y);
        a1 = __vimax3_u16x2(a1, t.z, t.w);
      }
      mn = min(a0 & 0xffffu, a0 >> 16);
      mx = max(a1 & 0xffffu, a1 >> 16);
    } else if (sizeof(V) == 1) {  // u8: four lanes of bytes per register
      uint32_t a0 = 0xffffffffu, a1 = 0u;
#pragma unroll 4
      for (uint32_t i = lane; i < nq; i += 32) {
        const uint4 t = q[i];
        a0 = __vminu4(__vminu4(a0, __vminu4(t.x, t.y)), __vminu4(t.z, t.w));
        a1 = __vmaxu4(__vmaxu4(a1, __vmaxu4(t.x, t.y)), __vmaxu4(t.z, t.w));
      }
      mn = min(min(a0 & 0xffu, (a0 >> 8) & 0xffu), min((a0 >> 16) & 0xffu, a0 >> 24));
      mx = max(max(a1 & 0xffu, (a1 >> 8) & 0xffu), max((a1 >> 16) & 0xffu, a1 >> 24));
    } else {
#pragma unroll 4
      for (uint32_t i = lane; i < nq; i += 32) {
        const uint4 t = q[i];
        mn = min(min(mn, t.x), min(t.y, min(t.z, t.w)));
        mx = max(max(mx, t.x), max(t.y, max(t.z, t.w)));
      }
    }
    i0 = nq * PER;
  }
  for (uint32_t i = i0 + lane; i < n; i += 32) {
    mn = min(mn, (uint32_t)s[i]);
    mx = max(mx, (uint32_t)s[i]);
  }
  mn = shfl_min(mn, 32);
  mx = shfl_max(mx, 32);
}

// Copy nbytes global -> shared by one warp (16-byte vectors when both allow).
__device__ __forceinline__ void warp_copy(uint8_t* dst, const uint8_t* src, uint32_t nbytes, int lane) {
  // the widest unit both addresses share the alignment of (after a short
  // byte head), so a tile that only starts 2-, 4- or 8-byte aligned (blocks
  // whose byte size is not a multiple of 16) still moves in 8- or 4-byte
  // pieces, four in flight per lane
  const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(dst) ^ reinterpret_cast<uintptr_t>(src)) & 15);
  const uint32_t unit = (mis == 0) ? 16u : ((mis & 7) == 0) ? 8u : ((mis & 3) == 0) ? 4u : 1u;
  uint32_t head = (uint32_t)((unit - (reinterpret_cast<uintptr_t>(src) & (unit - 1))) & (unit - 1));
  head = min(head, nbytes);
  if ((uint32_t)lane < head) dst[lane] = src[lane];
  uint32_t done = head;
  if (unit > 1) {
    const uint32_t nu = (nbytes - head) / unit;
    uint8_t* d = dst + head;
    const uint8_t* s = src + head;
    if (unit == 16) {
#pragma unroll 4
      for (uint32_t i = lane; i < nu; i += 32) reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(s)[i];
    } else if (unit == 8) {
#pragma unroll 4
      for (uint32_t i = lane; i < nu; i += 32) reinterpret_cast<uint2*>(d)[i] = reinterpret_cast<const uint2*>(s)[i];
    } else {
#pragma unroll 4
      for (uint32_t i = lane; i < nu; i += 32) reinterpret_cast<uint32_t*>(d)[i] = reinterpret_cast<const uint32_t*>(s)[i];
    }
    done = head + nu * unit;
  }
  for (uint32_t i = done + lane; i < nbytes; i += 32) dst[i] = src[i];
}

// ======================================================================
// tile prefixes (a4)
// ======================================================================
// Prefix server: the last CTA of the grid runs no tiles; one warp turns the
// tiles' published aggregates (FLAG_AGG | words) into inclusive prefixes
// (FLAG_PRE | words up to and including the tile), in tile order, 256 tiles
// per read.  Its SM carries no bulk traffic, so its reads return quickly; a
// worker then needs one word, status[t - 1], to learn its tile's offset
// instead of walking back through other tiles.
// PER tiles per lane per read (32 PER per round; measured for the 24 KiB
// tiles of cmp3: 8 and 16 alike).
template <int PER = LB_PER>
__device__ __noinline__ void prefix_server(uint64_t* status, uint64_t n_tiles, uint64_t t_begin = 0) {
  constexpr int LB_PER = PER;
  // tiles [t_begin, n_tiles); a range after the first continues from the
  // inclusive prefix the previous launch's server left in status[t_begin - 1]
  const int lane = threadIdx.x & 31;
  uint64_t P = t_begin ? (ld_relaxed_u64(status + t_begin - 1) & VAL_MASK) : 0, f = t_begin;
  uint32_t ns = 0;
  while (f < n_tiles) {
    uint64_t e[LB_PER];
    uint32_t lv = LB_PER;  // this lane's first unpublished slot
#pragma unroll
    for (int j = 0; j < LB_PER; ++j) {
      const uint64_t idx = f + (uint64_t)(LB_PER * lane + j);
      e[j] = idx < n_tiles ? ld_relaxed_u64(status + idx) : 0ull;
    }
#pragma unroll
    for (int j = LB_PER - 1; j >= 0; --j)
      if ((e[j] >> 62) == 0) lv = j;
    const uint32_t bad = __ballot_sync(0xffffffffu, lv < LB_PER);
    const int l0 = bad ? __ffs(bad) - 1 : 32;
    const uint32_t q = l0 == 32 ? 32 * LB_PER : LB_PER * l0 + __shfl_sync(0xffffffffu, lv, l0 & 31);
    if (q == 0) {
      if (ns) __nanosleep(ns);
      ns = ns ? min(ns * 2, 128u) : 32u;
      continue;
    }
    ns = 0;
    // inclusive prefixes of the run [f, f + q) (the lane's running sum is
    // recomputed while storing, so only e[] stays in registers)
    uint64_t run = 0;
#pragma unroll
    for (int j = 0; j < LB_PER; ++j)
      if ((uint32_t)(LB_PER * lane + j) < q) run += e[j] & VAL_MASK;
    uint64_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    uint64_t acc = P + inc - run;
#pragma unroll
    for (int j = 0; j < LB_PER; ++j)
      if ((uint32_t)(LB_PER * lane + j) < q) {
        acc += e[j] & VAL_MASK;
        st_relaxed_u64(status + f + LB_PER * lane + j, FLAG_PRE | (acc & VAL_MASK));
      }
    P += __shfl_sync(0xffffffffu, inc, 31);
    f += q;
  }
}

// A worker's exclusive prefix for tile t >= 1: the server's inclusive prefix
// of tile t - 1 (one word, polled by lane 0).
__device__ __forceinline__ uint64_t wait_prefix(const uint64_t* status, uint64_t t) {
  uint64_t v = 0;
  if ((threadIdx.x & 31) == 0) {
    uint32_t ns = 0;
    while (((v = ld_relaxed_u64(status + t - 1)) >> 62) != 2) {
      if (ns) __nanosleep(ns);
      ns = ns ? min(ns * 2, 256u) : 64u;
    }
  }
  return __shfl_sync(0xffffffffu, v, 0) & VAL_MASK;
}

// ======================================================================
// compress
// ======================================================================
template <typename V, int MAP, int NW>
__global__ void __launch_bounds__(NW * 32 + 32 * (2 + NLB_MAX), POLY_CTAS) poly_compress_pipe(PipeArgs a) {
  constexpr int NCW = NW, PC = NW * 32, PT = PC + 32 * (2 + NLB_MAX);
  constexpr int W_PROD = NCW, W_WRIT = NCW + 1, W_HSUM = NCW + 2, W_LBX = NCW + 3;
  (void)W_HSUM;
  (void)W_LBX;
  extern __shared__ __align__(128) uint8_t smem[];
  if (a.server && blockIdx.x == gridDim.x - 1) {
    if (threadIdx.x < 32) prefix_server(a.status, a.t_end, a.t_begin);
    return;
  }
  PipeCtl& C = *reinterpret_cast<PipeCtl*>(smem);
  const PipeShape& sh = a.sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t S = sh.S;
  const BaseCache bc = cache_at(smem + sh.o_cache, false);
  uint8_t* ring = smem + sh.o_ring;
  const bool WARP_RINGS = MAP == 0 && sh.wrings;  // see plan_pipe
  if (tid == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&C.full_in[s], 1);
      mbar_init(&C.empty_in[s], NCW);
    }
    for (int r = 0; r < MAXR; ++r) {
      mbar_init(&C.rec_full[r], NCW);
      mbar_init(&C.rec_cnt[r], NCW);
      mbar_init(&C.rec_empty[r], 1);
    }
    C.ring_tail = 0;
    C.wdone = 0;
    for (int w = 0; w < 32; ++w) C.wtail[w] = 0;
    mbar_fence_init();
  }
  cache_fill(bc, false);
  if (MAP == 0)
    for (uint32_t k = tid; k < 68; k += PT) C.nwL[k] = k ? (uint32_t)((sh.Le + k - 1) / k) : 0u;
  __syncthreads();

  if (warp == W_PROD) {
    // ---------------------------------------------------------- producer
    const uint64_t total_bytes = sh.n * sh.vb;
    for (uint32_t s = 0, ph = 0, it = 0;; s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0), ++it) {
      mbar_wait_cmp<POLY_CMP_PARK_PROD>(&C.empty_in[s], ph ^ 1u);
      uint32_t t32 = 0;
      if (lane == 0) t32 = atomicAdd(a.ticket, 1u);
      if (lane == 0) {
        TRACE(it, 0);
        TRACE_V(it, 10, t32);
      }
      const uint64_t t = a.t_begin + __shfl_sync(0xffffffffu, t32, 0);
      uint8_t* dst = smem + sh.o_in + (size_t)s * sh.in_stride;
      if (t >= a.t_end) {
        if (lane == 0) {
          C.tkt[s] = TILE_NONE;
          mbar_arrive(&C.full_in[s]);
        }
        break;
      }
      const uint64_t off = t * sh.tile_bytes;
      const uint32_t bytes = (uint32_t)min((uint64_t)sh.tile_bytes, total_bytes - off);
      const uint8_t* src = a.in + off;
      if (a.bulk || a.tma_shift) {
        // TMA of the 16-byte aligned range that holds the tile (blocks whose
        // byte size is not a multiple of 16 make tiles start 2-, 4- or 8-byte
        // aligned); the consumers start `shift` bytes into the stage.  The
        // bytes past the last 16-byte boundary of the tile are copied by hand.
        if (lane == 0) {
          const uintptr_t sa = reinterpret_cast<uintptr_t>(src), s0 = sa & ~(uintptr_t)15, e16 = (sa + bytes) & ~(uintptr_t)15;
          const uint32_t shift = (uint32_t)(sa - s0), n16 = e16 > s0 ? (uint32_t)(e16 - s0) : 0u;
          const uint8_t* g0 = reinterpret_cast<const uint8_t*>(s0);
          C.tkt[s] = t;
          C.shift[s] = shift;
          for (uint32_t j = n16; j < shift + bytes; ++j) dst[j] = g0[j];  // the tail (the last tile, or a shifted one)
          mbar_arrive_tx(&C.full_in[s], n16);
          if (n16) bulk_g2s(dst, g0, n16, &C.full_in[s]);
        }
      } else {
        warp_copy(dst, src, bytes, lane);
        __syncwarp();
        if (lane == 0) {
          C.tkt[s] = t;
          C.shift[s] = 0;
          mbar_arrive(&C.full_in[s]);
        }
      }
    }
    return;
  }

  uint64_t* pay_g = reinterpret_cast<uint64_t*>(a.out + 32 + 16 * sh.n_blocks);
  if (warp >= W_WRIT && warp < W_WRIT + (int)a.nlb) {
    // ---------------------------------------------------------- writers
    // nlb writer warps take records round robin (look-backs overlap);
    // ring space is released strictly in record order.
    for (uint32_t i = (uint32_t)(warp - W_WRIT);; i += a.nlb) {
      const uint32_t r = i % MAXR, ph = (i / MAXR) & 1u;
      mbar_wait_writer(WARP_RINGS ? &C.rec_cnt[r] : &C.rec_full[r], ph);
      const uint64_t t = C.rec_t[r];
      if (t == TILE_NONE) break;
      if (lane == 0) TRACE(i, 5);
      if (WARP_RINGS) {
        // the tile's words are NCW warp segments, in warp order
        const uint32_t ww = lane < NCW ? C.rw_words[r][lane] : 0u;
        const uint32_t wo = lane < NCW ? C.rw_off[r][lane] : 0u;
        uint32_t Wt;
        const uint32_t wex = warp_excl_scan(ww, &Wt);
        if (lane == 0) st_relaxed_u64(a.status + t, (t == 0 && !a.server ? FLAG_PRE : FLAG_AGG) | Wt);
        uint64_t P = 0;
        if (t != 0 && !DBG(a, 2)) {
          if (a.server) {
            P = wait_prefix(a.status, t);
          } else {
            P = lookback_wide(a.status, t);
            if (lane == 0) st_relaxed_u64(a.status + t, FLAG_PRE | ((P + Wt) & VAL_MASK));
          }
        }
        if (lane == 0) TRACE(i, 6);
        mbar_wait_writer(&C.rec_full[r], ph);  // every warp's words packed
        // copy: each lane walks the tile's words lane-strided; the warp segment
        // of word j is found by advancing through the (short) segment list
#pragma unroll 1
        for (int w = 0; w < NCW; w += 2) {
          const uint32_t n0 = __shfl_sync(0xffffffffu, ww, w), o0 = __shfl_sync(0xffffffffu, wex, w);
          const uint32_t s0 = __shfl_sync(0xffffffffu, wo, w);
          const uint32_t n1 = __shfl_sync(0xffffffffu, ww, w + 1), o1 = __shfl_sync(0xffffffffu, wex, w + 1);
          const uint32_t s1 = __shfl_sync(0xffffffffu, wo, w + 1);
          const uint64_t* src0 = reinterpret_cast<const uint64_t*>(ring + (size_t)w * sh.ring_bytes + s0);
          const uint64_t* src1 = reinterpret_cast<const uint64_t*>(ring + (size_t)(w + 1) * sh.ring_bytes + s1);
          uint64_t* d0 = pay_g + P + o0;
          uint64_t* d1 = pay_g + P + o1;
          const uint32_t nm = max(n0, w + 1 < NCW ? n1 : 0u);
          for (uint32_t j = lane; j < nm; j += 32) {
            uint64_t x0 = 0, x1 = 0;
            if (j < n0) x0 = src0[j];
            if (w + 1 < NCW && j < n1) x1 = src1[j];
            if (j < n0) d0[j] = x0;
            if (w + 1 < NCW && j < n1) d1[j] = x1;
          }
        }
        if (t == sh.n_tiles - 1 && lane == 0) {
          write_global_header_f(a.out, sh.width, sh.n, sh.block_len, sh.n_blocks, P + Wt);
          *a.compressed_bytes = 32 + 16 * sh.n_blocks + 8 * (P + Wt);
        }
        __syncwarp();
        if (lane == 0) {
          TRACE(i, 7);
          while (C.wdone != i) __nanosleep(32);
          __threadfence_block();
        }
        __syncwarp();
        if (lane < NCW) C.wtail[lane] = C.rw_end[r][lane];
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          C.wdone = i + 1;
          mbar_arrive(&C.rec_empty[r]);
        }
        __syncwarp();
        continue;
      }
      const uint64_t W = C.rec_W[r];
      uint64_t P = 0;
      if (t != 0 && !DBG(a, 2)) {
        if (a.server) {
          P = wait_prefix(a.status, t);
        } else {
          P = lookback_wide(a.status, t);
          if (lane == 0) st_relaxed_u64(a.status + t, FLAG_PRE | ((P + W) & VAL_MASK));
        }
      }
      if (lane == 0) TRACE(i, 6);
      const uint64_t* src = reinterpret_cast<const uint64_t*>(ring + C.rec_off[r]);
      uint64_t* dst = pay_g + P;
      const uint32_t w = (uint32_t)W;
      uint32_t j = lane;
      for (; j + 224 < w; j += 256) {
        uint64_t v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = src[j + 32 * q];
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[j + 32 * q] = v[q];
      }
      for (; j < w; j += 32) dst[j] = src[j];
      if (t == sh.n_tiles - 1 && lane == 0) {
        write_global_header_f(a.out, sh.width, sh.n, sh.block_len, sh.n_blocks, P + W);
        *a.compressed_bytes = 32 + 16 * sh.n_blocks + 8 * (P + W);
      }
      __syncwarp();
      if (lane == 0) {
        TRACE(i, 7);
        while (C.wdone != i) __nanosleep(32);
        __threadfence_block();
        C.ring_tail = C.rec_end[r];
        C.wdone = i + 1;
        mbar_arrive(&C.rec_empty[r]);
      }
      __syncwarp();
    }
    return;
  }

  if (warp >= NCW) return;  // spare warps

  // ------------------------------------------------------------ consumers
  const int ctid = tid;  // 0 .. PC-1
  const uint32_t L = (uint32_t)sh.Le;
  uint4* hdr_g = reinterpret_cast<uint4*>(a.out + 32);
  uint64_t head = 0;  // ring bytes handed out (thread 0's copy is authoritative)
  uint64_t whead = 0;  // WARP_RINGS: this warp's ring bytes handed out (lane 0)
  uint32_t hpos = 0;   // head (or whead) modulo the ring size, kept incrementally
  for (uint32_t s = 0, ph = 0, r = 0, rph = 0, it = 0;;
       s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0), r = (r + 1) % MAXR, rph ^= (r == 0), ++it) {
    mbar_wait_cmp<POLY_CMP_PARK_IN>(&C.full_in[s], ph);
    if (ctid == 0) TRACE(it, 1);
    const uint64_t t = C.tkt[s];
    if (t == TILE_NONE) {  // one end marker per writer warp (every consumer warp arrives)
      if (lane == 0) {
        for (uint32_t e = 0; e < a.nlb; ++e) {
          mbar_wait(&C.rec_empty[r], rph ^ 1u);
          if (warp == 0) C.rec_t[r] = TILE_NONE;
          mbar_arrive(&C.rec_cnt[r]);
          mbar_arrive(&C.rec_full[r]);
          r = (r + 1) % MAXR;
          rph ^= (r == 0);
        }
      }
      break;
    }
    const V* sv = reinterpret_cast<const V*>(smem + sh.o_in + (size_t)s * sh.in_stride + C.shift[s]);
    const uint64_t b0 = t * sh.TB;
    const uint32_t nblk = (uint32_t)min((uint64_t)sh.TB, sh.n_blocks - b0);
    const uint64_t v0 = b0 * sh.Le;
    const uint32_t nv = (uint32_t)(min(sh.n, v0 + (uint64_t)sh.TB * sh.Le) - v0);
    if (WARP_RINGS) {
      // One block per thread; the warp's 32 blocks are packed into its own
      // word ring -- no CTA scan, no shared ring allocation (the writers
      // concatenate the warp segments and publish the tile aggregate).
      const uint32_t b = ctid;
      uint32_t vmn = 0, bmm = 0, nwb = 0, kkb = 1;
      if (b < nblk && !DBG(a, 1)) {
        const uint32_t nb = min(L, nv - b * L);
        uint32_t mn, mx;
        block_minmax<V>(sv + (size_t)b * L, nb, mn, mx);
        vmn = mn;
        bmm = mx - mn;
        if (mx != mn) {
          kkb = sizeof(V) == 2 ? kh_of16(bc, mx - mn + 1) : k_of(bc, (uint64_t)(mx - mn) + 1);
          nwb = nb == L ? C.nwL[kkb & 0xffu] : ceil_div_small(nb, kkb & 0xffu);
        }
        hdr_g[b0 + b] = make_uint4(mx == mn ? CODEC_CONSTANT : CODEC_BASIC, mn, mx - mn, nwb);
      }
      uint32_t tot;
      const uint32_t ex = warp_excl_scan(nwb, &tot);
      uint32_t pos = 0;
      if (lane == 0) {
        mbar_wait_cmp<POLY_CMP_PARK_REC>(&C.rec_empty[r], rph ^ 1u);
        const uint32_t need = (8 * tot + 15) & ~15u, RB = sh.ring_bytes;
        uint32_t p = hpos;
        if (p + need > RB) {  // wrap: the segment stays contiguous
          whead += RB - p;
          p = 0;
        }
        hpos = p + need;
        uint32_t ns = 0;
        while (whead + need - C.wtail[warp] > RB) {
          __nanosleep(ns);
          ns = ns ? min(ns * 2, 256u) : 32u;
        }
        whead += need;
        C.rw_off[r][warp] = p;
        C.rw_words[r][warp] = tot;
        C.rw_end[r][warp] = whead;
        if (warp == 0) C.rec_t[r] = t;
        mbar_arrive(&C.rec_cnt[r]);
        pos = p;
        if (warp == 0) TRACE(it, 3);
      }
      pos = __shfl_sync(0xffffffffu, pos, 0);
      uint64_t* ow = reinterpret_cast<uint64_t*>(ring + (size_t)warp * sh.ring_bytes + pos);
      if (b < nblk && nwb != 0) {
        const uint32_t nb = min(L, nv - b * L);
        if (sizeof(V) == 2) {
          const uint32_t B = bmm + 1, k = kkb & 0xffu, h = kkb >> 8;
          uint64_t D;
          uint32_t G;
          chunk_consts(bc, B, h, D, G);
          pack_block_lane16(reinterpret_cast<const uint16_t*>(sv + (size_t)b * L), nb, vmn, B, k, h, D, G, nwb,
                            ow + ex);
        } else {
          pack_block_words<V>(sv + (size_t)b * L, nb, vmn, (uint64_t)bmm + 1, kkb, nwb, ow + ex);
        }
      }
      __syncwarp();
      if (lane == 0) {
        if (warp == 0) TRACE(it, 4);
        mbar_arrive(&C.rec_full[r]);
        mbar_arrive(&C.empty_in[s]);
      }
      continue;
    }
    uint32_t W = 0;
    uint32_t vmin[BPT_MAX], bm1[BPT_MAX], nw[BPT_MAX], kk[BPT_MAX], off[BPT_MAX];

    // ---- a2, a3: block statistics, headers, in-tile word offsets
    if (DBG(a, 1)) {
#pragma unroll
      for (int q = 0; q < BPT_MAX; ++q) {
        vmin[q] = bm1[q] = nw[q] = off[q] = 0;
        kk[q] = 1;
      }
      if (MAP == 1 && ctid < (int)nblk) C.bbm1[ctid] = 0;
    } else if (MAP == 0) {
#pragma unroll
      for (int q = 0; q < BPT_MAX; ++q) {
        vmin[q] = 0;
        bm1[q] = 0;
        nw[q] = 0;
        kk[q] = 1;
        off[q] = 0;
        if (q < (int)sh.bpt) {
          const uint32_t b = q * PC + ctid;
          if (b < nblk) {
            const uint32_t nb = min(L, nv - b * L);
            uint32_t mn, mx;
            block_minmax<V>(sv + (size_t)b * L, nb, mn, mx);
            vmin[q] = mn;
            bm1[q] = mx - mn;
            if (mx != mn) {
              kk[q] = sizeof(V) == 2 ? kh_of16(bc, mx - mn + 1) : k_of(bc, (uint64_t)(mx - mn) + 1);
              nw[q] = nb == L ? C.nwL[kk[q] & 0xffu] : ceil_div_small(nb, kk[q] & 0xffu);
            }
            hdr_g[b0 + b] = make_uint4(mx == mn ? CODEC_CONSTANT : CODEC_BASIC, mn, mx - mn, nw[q]);
          }
          uint32_t tot;
          off[q] = W + cons_scan<NW>(nw[q], &tot, C.scan[q & 1]);
          W += tot;
        }
      }
    } else {
      const uint32_t lg = __ffs(sh.G) - 1, G = sh.G, nseg = nblk << lg;  // G: a power of two
      for (uint32_t seg = warp; seg < nseg; seg += NCW) {
        const uint32_t b = seg >> lg, part = seg & (G - 1);
        const uint32_t nb = min(L, nv - b * L);
        const uint32_t lo = min(nb, part * sh.Lp), hi = min(nb, lo + sh.Lp);
        uint32_t mn, mx;
        warp_minmax<V>(sv + (size_t)b * L + lo, hi - lo, mn, mx);
        if (lane == 0) {
          C.smin[seg] = mn;
          C.smax[seg] = mx;
        }
      }
      if (ctid == 0) TRACE(it, 9);
      cons_bar<NW>();
      if (ctid == 0) TRACE(it, 11);
      // per-block reduction of the segments and the in-tile word offsets: by
      // warp 0 alone when the tile has at most 32 blocks (no CTA scan, the
      // other warps go straight to the barrier before the pack)
      const bool w0 = nblk <= 32;
      if (!w0 || warp == 0) {
        uint32_t nwb = 0;
        if (ctid < (int)nblk) {
          uint32_t mn = 0xffffffffu, mx = 0u;
          for (uint32_t p = 0; p < G; ++p) {
            mn = min(mn, C.smin[(ctid << lg) + p]);
            mx = max(mx, C.smax[(ctid << lg) + p]);
          }
          const uint32_t nb = min(L, nv - ctid * L);
          if (mx != mn) nwb = ceil_div_small(nb, k_of(bc, (uint64_t)(mx - mn) + 1));
          C.bvmin[ctid] = mn;
          C.bbm1[ctid] = mx - mn;
          C.bnw[ctid] = nwb;
          hdr_g[b0 + ctid] = make_uint4(mx == mn ? CODEC_CONSTANT : CODEC_BASIC, mn, mx - mn, nwb);
        }
        const uint32_t ex = w0 ? warp_excl_scan(nwb, &W) : cons_scan<NW>(nwb, &W, C.scan[0]);
        if (ctid < (int)nblk) C.boff[ctid] = ex;
      }
    }
    // ---- a4: publish the tile aggregate, then take ring space for its words
    if (ctid == 0) {
      st_relaxed_u64(a.status + t, (t == 0 && !a.server ? FLAG_PRE : FLAG_AGG) | W);
      TRACE(it, 2);
      mbar_wait_cmp<POLY_CMP_PARK_REC>(&C.rec_empty[r], rph ^ 1u);
      const uint32_t need = (8 * W + 15) & ~15u;
      uint32_t pos = hpos;
      if (pos + need > sh.ring_bytes) {
        head += sh.ring_bytes - pos;
        pos = 0;
      }
      hpos = pos + need;
      uint32_t ns = 0;
      while (head + need - C.ring_tail > sh.ring_bytes) {
        __nanosleep(ns);
        ns = ns ? min(ns * 2, 256u) : 32u;
      }
      __threadfence_block();
      head += need;
      C.rec_t[r] = t;
      C.rec_W[r] = W;
      C.rec_off[r] = pos;
      C.rec_end[r] = head;
      TRACE(it, 3);
    }
    cons_bar<NW>();
    uint64_t* ow = reinterpret_cast<uint64_t*>(ring + C.rec_off[r]);

    // ---- a5: Horner pack
    if (MAP == 0) {
#pragma unroll
      for (int q = 0; q < BPT_MAX; ++q) {
        const uint32_t b = q * PC + ctid;
        if (q < (int)sh.bpt && b < nblk && nw[q] != 0) {
          const uint32_t nb = min(L, nv - b * L);
          if (sizeof(V) == 2) {
            const uint32_t B = bm1[q] + 1, k = kk[q] & 0xffu, h = kk[q] >> 8;
            uint64_t D;
            uint32_t G;
            chunk_consts(bc, B, h, D, G);
            pack_block_lane16(reinterpret_cast<const uint16_t*>(sv + (size_t)b * L), nb, vmin[q], B, k, h, D, G,
                              nw[q], ow + off[q]);
          } else {
            pack_block_words<V>(sv + (size_t)b * L, nb, vmin[q], (uint64_t)bm1[q] + 1, kk[q], nw[q], ow + off[q]);
          }
        }
      }
    } else {
      const uint32_t lg = __ffs(sh.G) - 1, G = sh.G, nseg = nblk << lg;
      for (uint32_t seg = warp; seg < nseg; seg += NCW) {
        const uint32_t b = seg >> lg, part = seg & (G - 1);
        const uint32_t bm1b = C.bbm1[b];
        if (bm1b == 0) continue;
        const uint32_t nb = min(L, nv - b * L), nwk = C.bnw[b], vm = C.bvmin[b];
        const uint64_t B = (uint64_t)bm1b + 1;
        const uint32_t k = k_of(bc, B);
        const V* src = sv + (size_t)b * L;
        uint64_t* dst = ow + C.boff[b];
        uint32_t done = 0;
        if (sizeof(V) == 2 && ((L * 2) & 15) == 0) {
          const uint8_t* blk = reinterpret_cast<const uint8_t*>(src);
          switch (k) {
#define POLY_PK(KK)                                                                              \
  case KK:                                                                                       \
    done = pack_block_k<KK>(blk, nb, (uint32_t)B, vm, part * 32 + lane, 32 * G, dst);            \
    break;
            POLY_FOR_EACH_K16(POLY_PK)
#undef POLY_PK
            default:
              break;
          }
        } else if (sizeof(V) == 2) {
          // blocks at any 2-byte alignment: the same chains over 16-bit reads
          const uint16_t* blk = reinterpret_cast<const uint16_t*>(src);
          switch (k) {
#define POLY_PKU(KK)                                                                             \
  case KK:                                                                                       \
    done = pack_block_ku<KK>(blk, nb, (uint32_t)B, vm, part * 32 + lane, 32 * G, dst);           \
    break;
            POLY_FOR_EACH_K16(POLY_PKU)
#undef POLY_PKU
            default:
              break;
          }
        }
        for (uint32_t j = done + part * 32 + lane; j < nwk; j += 32 * G) {
          const uint32_t first = j * k;
          dst[j] = pack_word64<V>(src + first, min(k, nb - first), B, vm);
        }
      }
    }
    // every warp reports its own end: the record is complete and the input
    // stage free once all NCW warps have arrived (no CTA barrier)
    __syncwarp();
    if (lane == 0) {
      if (warp == 0) TRACE(it, 4);
      if (warp == NCW - 1) TRACE(it, 8);
      mbar_arrive(&C.rec_full[r]);
      mbar_arrive(&C.empty_in[s]);
    }
  }
}

// ======================================================================
// decompress
// ======================================================================
__device__ __forceinline__ uint32_t check_global_header_p(const PipeArgs& a, uint64_t* pw) {
  const PipeShape& sh = a.sh;
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

// 64-bit fraction step with the block minimum folded into the digit:
// returns vmin + floor(f B / 2^64), f <- f B mod 2^64 (f = f1:f0).
__device__ __forceinline__ uint32_t fstep64v(uint32_t& f0, uint32_t& f1, uint32_t B, uint32_t vmin) {
  // (f0 B) gives the new low word and a carry word c; f1 B + (vmin:c) gives
  // the new high word and vmin + digit (no carry chain across instructions)
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
__device__ __forceinline__ uint32_t fstep32v(uint32_t& g, uint32_t B, uint32_t vmin) {
  uint32_t lo, d;
  asm("mul.lo.u32 %0, %2, %3;\n\tmad.hi.u32 %1, %2, %3, %4;" : "=&r"(lo), "=r"(d) : "r"(g), "r"(B), "r"(vmin));
  g = lo;
  return d;
}

// The m top digits of a word (already premultiplied so they are its top
// digits), written most significant first at o[0], o[-1], ...: n64 64-bit
// steps, then n32 32-bit steps.
template <typename V>
__device__ __forceinline__ void digits_out(uint32_t f0, uint32_t f1, uint32_t add, uint32_t B, uint32_t vmin,
                                           int n64, int n32, V* o) {
#pragma unroll 1
  for (; n64 >= 2; n64 -= 2, o -= 2) {
    const uint32_t d1 = fstep64v(f0, f1, B, vmin);
    const uint32_t d0 = fstep64v(f0, f1, B, vmin);
    o[0] = (V)d1;
    o[-1] = (V)d0;
  }
  if (n64) {
    o[0] = (V)fstep64v(f0, f1, B, vmin);
    --o;
  }
  uint32_t g = f1 + add;
#pragma unroll 1
  for (; n32 >= 2; n32 -= 2, o -= 2) {
    const uint32_t d1 = fstep32v(g, B, vmin);
    const uint32_t d0 = fstep32v(g, B, vmin);
    o[0] = (V)d1;
    o[-1] = (V)d0;
  }
  if (n32) o[0] = (V)fstep32v(g, B, vmin);
}

// One full-length block (nb = L, B <= CACHE_B, B < 2^32) from its cached
// constants: every word decodes exactly its own digits (the top word is
// premultiplied by P = B^(k - mt), so its k - mt zero digits are skipped and
// s < B^mt is checked as s P < B^k).
template <typename V>
__device__ __forceinline__ uint32_t decode_block_ent(const uint64_t* src, uint32_t nw, uint32_t B, uint32_t vmin,
                                                     const DecEnt& e, V* dst, uint32_t jcap, uint32_t* extra) {
  // the constants live in registers for the whole block (the digit stores
  // would otherwise force the compiler to reload them from shared memory)
  const uint64_t Rl = e.Rl, Rh = e.Rh, Wmax = e.Wmax, P = e.P;
  const uint32_t meta = e.meta, mt = e.mt;
  const uint32_t k = meta & 0xffu, t = (meta >> 16) & 0xffu, add = ((meta >> 8) & 0xffu) ? 0u : 1u;
  uint32_t err = 0;
  const uint32_t nfull = mt < k ? nw - 1 : nw;
  // full words past jcap are left to the warp's overflow round (decode_group0)
  const uint32_t nin = min(nfull, jcap);
  *extra = nfull - nin;
  V* o = dst + (k - 1);
  uint32_t j = 0;
#pragma unroll 1
  for (; j < nin; ++j, o += k) {
    const uint64_t s = src[j];
    if (s > Wmax) err = POLY_ST_RESIDUE;
    const uint64_t hi1 = __umul64hi(s, Rl), lo2 = s * Rh, hi2 = __umul64hi(s, Rh), mid = lo2 + hi1;
    const uint64_t f = ((hi2 + (mid < lo2 ? 1ull : 0ull)) << 32) + (mid >> 32) + add;
    digits_out<V>((uint32_t)f, (uint32_t)(f >> 32), add, B, vmin, (int)(k - t), (int)t, o);
  }
  if (nfull < nw) {  // the top word: mt < k digits, premultiplied by P = B^(k - mt)
    uint64_t s = src[nfull];
    if (__umul64hi(s, P) != 0) err = POLY_ST_RESIDUE;
    s *= P;
    if (s > Wmax) err = POLY_ST_RESIDUE;
    const uint64_t hi1 = __umul64hi(s, Rl), lo2 = s * Rh, hi2 = __umul64hi(s, Rh), mid = lo2 + hi1;
    const uint64_t f = ((hi2 + (mid < lo2 ? 1ull : 0ull)) << 32) + (mid >> 32) + add;
    const int n32 = (int)(t + mt) > (int)k ? (int)(t + mt - k) : 0;
    digits_out<V>((uint32_t)f, (uint32_t)(f >> 32), add, B, vmin, (int)mt - n32, n32, dst + (nfull * k + mt - 1));
  }
  return err;
}

// One block of the lane-per-block map (a8, a9): header validation and decode.
template <typename V>
__device__ __forceinline__ uint32_t decode_block0(const uint4 h, const uint64_t* src, uint32_t nb, uint32_t L,
                                                  uint32_t width, const BaseCache& bc, V* dst,
                                                  uint32_t jcap = 0xffffffffu, uint32_t* extra = nullptr) {
  const uint64_t vmax = (width == 32) ? 0xffffffffull : ((1ull << width) - 1);
  uint32_t ex0 = 0;
  if (!extra) extra = &ex0;
  *extra = 0;
  if (h.x == CODEC_BASIC && h.z != 0 && (uint64_t)h.y + h.z <= vmax) {
    const uint64_t B = (uint64_t)h.z + 1;
    if (B <= CACHE_B && nb == L) {
      const DecEnt& e = bc.E[B];
      if (h.w != e.nwL) return POLY_ST_NWORDS;
      return decode_block_ent<V>(src, h.w, (uint32_t)B, h.y, e, dst, jcap, extra);
    }
  }
  // general path: partial last block, large bases, constant blocks, errors
  const uint32_t k = (h.x == CODEC_BASIC && h.z != 0) ? dk_of(bc, (uint64_t)h.z + 1) : 1u;
  const uint32_t e = check_block_hdr(h, nb, width, k);
  if (e) return e;
  if (h.x == CODEC_CONSTANT) {
    for (uint32_t j = 0; j < nb; ++j) dst[j] = (V)h.y;
    return 0;
  }
  const DecConst c = dconst_of(bc, (uint64_t)h.z + 1);
  uint32_t err = 0;
  if (dc_log2b(c) == 32) {  // B = 2^32 (u32 only) does not fit the 32-bit multiplier
    for (uint32_t j = 0, first = 0; j < h.w; ++j, first += k)
      err |= decode_pow2<V>(src[j], 32, min(k, nb - first), h.y, dst + first);
  } else {
    err = decode_block_lane<V>(src, h.w, nb, c, h.z + 1, h.y, 0ull, dst);
  }
  return err;
}



__device__ __forceinline__ bool check_global_header_p_ok(const PipeArgs& a) {
  uint64_t pw;
  return check_global_header_p(a, &pw) == 0;
}

// The words of a block past its full k-specialised groups (at most Q full
// words and the top word), one lane each; the top word of a full-length block
// takes the premultiplied path (m steps, not k).
template <typename V>
__device__ __forceinline__ uint32_t decode_tail(const uint64_t* src, uint32_t j0, uint32_t nw, const DecConst& c,
                                                uint32_t B, uint32_t vmin, uint32_t nb, uint32_t k, V* dst,
                                                const BaseCache& bc, uint32_t L) {
  uint32_t err = 0;
  const uint32_t j = j0 + (threadIdx.x & 31);
  if (j < nw) {
    const uint32_t first = j * k, m = min(k, nb - first);
    const uint64_t P = (m < k && nb == L && B <= CACHE_B) ? bc.E[B].P : 0ull;
    if (P != 0 && dc_log2b(c) != 32)
      err = decode_top_word<V>(src[j], c, B, m, P, vmin, dst + first);
    else
      err = decode_any<V>(src[j], c, B - 1, m, vmin, dst + first);
  }
  return err;
}

template <typename V, int MAP, int NW>
__global__ void __launch_bounds__(NW * 32 + 32 * (2 + NLB_MAX), POLY_CTAS) poly_decompress_pipe(PipeArgs a) {
  constexpr int NCW = NW, PC = NW * 32, PT = PC + 32 * (2 + NLB_MAX);
  constexpr int W_PROD = NCW, W_WRIT = NCW + 1, W_HSUM = NCW + 2, W_LBX = NCW + 3;
  constexpr uint32_t NTS = 2;  // staging tiles (map 1)
  (void)W_HSUM;
  (void)W_LBX;
  extern __shared__ __align__(128) uint8_t smem[];
  if (a.server && blockIdx.x == gridDim.x - 1) {
    if (threadIdx.x < 32 && check_global_header_p_ok(a)) prefix_server(a.status, a.t_end, a.t_begin);
    return;
  }
  PipeCtl& C = *reinterpret_cast<PipeCtl*>(smem);
  const PipeShape& sh = a.sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t S = sh.S;
  const BaseCache bc = cache_at(smem + sh.o_cache, true);
  uint8_t* ring = smem + sh.o_ring;
  if (tid == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&C.hbar[s], 1);
      mbar_init(&C.aggr[s], 1);
      mbar_init(&C.full_in[s], 1);
      mbar_init(&C.empty_in[s], NCW);
      C.done_cnt[s] = 0;
      C.gnext[s] = 0;
    }
    for (int q = 0; q < NTS; ++q) {
      mbar_init(&C.tfull[q], NCW);
      mbar_init(&C.tfree[q], 1);
    }
    mbar_fence_init();
    uint64_t pw;
    C.hdr_err = check_global_header_p(a, &pw);
    C.payload_words = pw;
    C.ring_tail = 0;
    C.lb_seq = 0;
    C.ring_head = 0;
    C.ring_hpos = 0;
  }
  cache_fill(bc, true, sh.Le);
  __syncthreads();
  if (C.hdr_err) {  // same verdict in every CTA: nothing is decoded, no look-back
    if (blockIdx.x == 0 && tid == 0) atomicOr(a.status_out, C.hdr_err);
    return;
  }
  const uint4* hdr_g = reinterpret_cast<const uint4*>(a.in + 32);
  const uint64_t* pay_g = reinterpret_cast<const uint64_t*>(a.in + 32 + 16 * sh.n_blocks);

  if (warp == W_PROD) {
    // ---------------------------------------------------------- header issuer
    if (lane != 0) return;
    uint32_t nend = 0;  // end markers emitted (one per look-back warp)
    for (uint32_t i = 0, s = 0, ph = 0;; ++i) {
      mbar_wait_helper(&C.empty_in[s], ph ^ 1u);
      const uint64_t t = nend ? a.t_end : a.t_begin + atomicAdd(a.ticket, 1u);
      TRACE(i, 0);
      TRACE_V(i, 10, t);
      if (t >= a.t_end) {
        C.tkt[s] = TILE_NONE;
        mbar_arrive(&C.hbar[s]);
        if (++nend == a.nlb) break;
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
        continue;
      }
      C.tkt[s] = t;
      const uint64_t b0 = t * sh.TB;
      const uint32_t nblk = (uint32_t)min((uint64_t)sh.TB, sh.n_blocks - b0);
      mbar_arrive_tx(&C.hbar[s], nblk * 16);
      bulk_g2s(smem + sh.o_in + (size_t)s * sh.in_stride, hdr_g + b0, nblk * 16, &C.hbar[s]);
      if (++s == S) {
        s = 0;
        ph ^= 1u;
      }
    }
    return;
  }

  if (warp == W_HSUM) {
    // ---------------------------------------------------------- header sum
    // Publishes each tile's aggregate as soon as its headers land (a7), and
    // the in-tile word offsets of its blocks.
    uint32_t nend = 0;
    for (uint32_t s = 0, ph = 0, it = 0;; ++it) {
      mbar_wait_helper(&C.hbar[s], ph);
      if (lane == 0) TRACE(it, 1);
      const uint64_t t = C.tkt[s];
      if (t == TILE_NONE) {
        if (lane == 0) mbar_arrive(&C.aggr[s]);
        if (++nend == a.nlb) break;
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
        continue;
      }
      uint8_t* st = smem + sh.o_in + (size_t)s * sh.in_stride;
      const uint4* H = reinterpret_cast<const uint4*>(st);
      uint32_t* OFF = reinterpret_cast<uint32_t*>(smem + sh.o_in + (size_t)s * sh.in_stride + sh.o_off);
      const uint64_t b0 = t * sh.TB;
      const uint32_t nblk = (uint32_t)min((uint64_t)sh.TB, sh.n_blocks - b0);
      // OFF[b] = words before block b in the tile: eight independent warp
      // scans of 32 blocks at a time (their shuffles overlap), then a carry.
      // A block's n_words is clamped to 2^20 - 1 (a valid block has at most
      // 4096 words here) so a corrupt header cannot wrap the 32-bit sums; the
      // consumers reject such a block and the look-back warp such a tile.
      const uint32_t* Hw = reinterpret_cast<const uint32_t*>(H) + 3;
      uint32_t Wt = 0;
      if (MAP == 0) {
        // map 0: only each 32-block group's offset (OFF[g]); a consumer warp
        // scans within its group.  One warp reduction per group.  (Map 2: the
        // tile's sum only; its look-back warp rewrites OFF with sorted slots.)
        for (uint32_t r0 = 0; r0 < nblk; r0 += 256) {
          uint32_t x[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t b = r0 + 32 * q + lane;
            x[q] = b < nblk ? min(Hw[4 * b], 0xfffffu) : 0u;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t sum = __reduce_add_sync(0xffffffffu, x[q]);
            if (lane == 0 && r0 + 32 * q < nblk) OFF[(r0 >> 5) + q] = Wt;
            Wt += sum;
          }
        }
      } else
      for (uint32_t r0 = 0; r0 < nblk; r0 += 256) {
        uint32_t x[8], v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t b = r0 + 32 * q + lane;
          x[q] = b < nblk ? min(Hw[4 * b], 0xfffffu) : 0u;
          v[q] = x[q];
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v[q], o);
            if (lane >= o) v[q] += y;
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t b = r0 + 32 * q + lane;
          if (b < nblk) OFF[b] = Wt + v[q] - x[q];
          Wt += __shfl_sync(0xffffffffu, v[q], 31);
        }
      }
      const uint64_t W = Wt;
      __syncwarp();
      if (lane == 0) {
        st_relaxed_u64(a.status + t, (t == 0 && !a.server ? FLAG_PRE : FLAG_AGG) | (W & VAL_MASK));
        C.W[s] = W;
        TRACE(it, 2);
        mbar_arrive(&C.aggr[s]);
      }
      if (++s == S) {
        s = 0;
        ph ^= 1u;
      }
    }
    return;
  }

  const int lbi = warp == W_WRIT ? 0 : (warp >= W_LBX && warp < W_LBX + NLB_MAX - 1) ? warp - W_LBX + 1 : -1;
  if (lbi >= 0 && lbi < (int)a.nlb) {
    // ---------------------------------------------------------- look-back + payload loader
    // nlb warps take stages round robin, so nlb look-backs are in flight; ring
    // space is handed out strictly in stage order (C.lb_seq).
    const uint64_t pw = C.payload_words;
    const uint32_t nlb = a.nlb;
    for (uint32_t i = (uint32_t)lbi;; i += nlb) {
      const uint32_t s = i % S, ph = (i / S) & 1u;
      mbar_wait_helper(&C.aggr[s], ph);
      const uint64_t t = C.tkt[s];
      if (t == TILE_NONE) {
        if (lane == 0) mbar_arrive(&C.full_in[s]);
        break;
      }
      if (lane == 0) TRACE(i, 3);
      const uint64_t W = C.W[s];
      uint64_t P = 0;
      if (DBG(a, 2)) {
        P = min(t * (pw / sh.n_tiles), pw - min(pw, W));
      } else if (t != 0) {
        if (a.server) {
          P = wait_prefix(a.status, t);
        } else {
          P = lookback_wide(a.status, t);
          if (lane == 0) st_relaxed_u64(a.status + t, FLAG_PRE | ((P + W) & VAL_MASK));
        }
      }
      if (lane == 0) TRACE(i, 4);
      uint32_t e = 0;
      uint64_t wl = DBG(a, 16) ? 0 : W;
      if (W > sh.words_cap || P + W > pw) {
        e = POLY_ST_LENGTH;
        wl = 0;
      }
      if (t == sh.n_tiles - 1 && P + W != pw) e |= POLY_ST_LENGTH;
      if (DBG(a, 2)) e = 0;
      if (lane == 0) {
        C.P[s] = P;
        C.err[s] = e;
        while (C.lb_seq != i) __nanosleep(32);  // in-order ring allocation
        __threadfence_block();
        uint64_t head = C.ring_head;
        if (wl) {
          const uint64_t a0 = P & ~1ull, hw = P + wl;
          uint64_t a1 = min((hw + 1) & ~1ull, pw & ~1ull);
          if (a1 < a0) a1 = a0;
          const uint32_t need = (uint32_t)((8 * (hw - a0) + 15) & ~15ull);
          uint32_t pos = C.ring_hpos;
          if (pos + need > sh.ring_bytes) {  // wrap: the tile's words stay contiguous
            head += sh.ring_bytes - pos;
            pos = 0;
          }
          uint32_t ns = 0;
          while (head + need - C.ring_tail > sh.ring_bytes) {
            __nanosleep(ns);
            ns = ns ? min(ns * 2, 256u) : 32u;
          }
          TRACE(i, 5);
          __threadfence_block();
          fence_proxy_async_smem();
          uint64_t* dst = reinterpret_cast<uint64_t*>(ring + pos);
          C.ring_off[s] = pos;
          head += need;
          C.ring_end[s] = head;
          C.ring_head = head;
          C.ring_hpos = pos + need;
          __threadfence_block();
          C.lb_seq = i + 1;
          for (uint64_t w = a1; w < hw; ++w) dst[w - a0] = ldg_nc_u64(pay_g + w);
          const uint32_t bytes = (uint32_t)(8 * (a1 - a0));
          mbar_arrive_tx(&C.full_in[s], bytes);
          if (bytes) bulk_g2s(dst, pay_g + a0, bytes, &C.full_in[s]);
        } else {
          C.ring_off[s] = 0;
          C.ring_end[s] = head;
          __threadfence_block();
          C.lb_seq = i + 1;
          mbar_arrive(&C.full_in[s]);
        }
      }
      __syncwarp();
    }
    return;
  }
  if (MAP != 0 && warp == NCW + 1 + NLB_MAX) {
    // ---------------------------------------------------------- tile store warp (map 1)
    // One bulk store per decoded tile, issued once every consumer warp has
    // filled its parts; the staging tile is freed when the store has read it.
    for (uint32_t i = 0;; ++i) {
      const uint32_t q = i % NTS;
      mbar_wait_helper(&C.tfull[q], (i / NTS) & 1u);
      const uint32_t bytes = C.t_bytes[q];
      if (bytes == ~0u) break;
      uint8_t* og = C.t_og[q];
      const uint8_t* src = smem + sh.o_out + (size_t)q * sh.out_stride;
      if (bytes && !DBG(a, 8)) {
        if (a.bulk) {
          const uint32_t b16 = bytes & ~15u;  // the tile starts 16-byte aligned
          if (lane == 0 && b16) bulk_s2g(og, src, b16);
          for (uint32_t j = b16 + lane; j < bytes; j += 32) og[j] = src[j];
          if (lane == 0) {
            bulk_commit();
            bulk_wait_read<0>();
          }
        } else {
          warp_copy(og, src, bytes, lane);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&C.tfree[q]);
    }
    if (a.bulk && lane == 0) bulk_wait_all<0>();
    return;
  }
  if (warp >= NCW) return;  // spare warps

  // ------------------------------------------------------------ consumers
  // No CTA barrier: a warp's block offsets come from a warp scan plus its
  // group offset (map 0) or from OFF[] (map 1); each warp (or block group)
  // bulk-stores its own part of the decoded tile; the stage is released when
  // all NCW warps have arrived.
  const uint32_t L = (uint32_t)sh.Le;
  uint32_t err = 0;
  const bool bst = a.bulk && !DBG(a, 4);
  for (uint32_t s = 0, ph = 0, s2 = 0, it = 0;; s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0), s2 = (s2 + 1 == NTS) ? 0 : s2 + 1, ++it) {
    mbar_wait_dec(&C.full_in[s], ph);
    if (lane == 0 && warp == 0) TRACE(it, 6);
    if (lane == 0 && warp == NCW - 1) TRACE(it, 9);
    const uint64_t t = C.tkt[s];
    if (t == TILE_NONE) {
      if (MAP != 0) {  // end marker for the tile store warp
        mbar_wait_dec(&C.tfree[s2], ((it / NTS) & 1u) ^ 1u);
        if (warp == 0 && lane == 0) C.t_bytes[s2] = ~0u;
        __syncwarp();
        if (lane == 0) mbar_arrive(&C.tfull[s2]);
      }
      break;
    }
    const uint8_t* st = smem + sh.o_in + (size_t)s * sh.in_stride;
    const uint4* H = reinterpret_cast<const uint4*>(st);
    const uint32_t* OFF = reinterpret_cast<const uint32_t*>(st + sh.o_off);
    const uint64_t* PAY = reinterpret_cast<const uint64_t*>(ring + C.ring_off[s]) + (C.P[s] & 1);
    const uint32_t terr = C.err[s];
    const uint64_t rend = C.ring_end[s];
    uint8_t* ob8 = smem + sh.o_out + (size_t)(MAP == 0 ? warp : s2) * sh.out_stride;
    V* ob = reinterpret_cast<V*>(ob8);
    const uint64_t b0 = t * sh.TB;
    const uint32_t nblk = (uint32_t)min((uint64_t)sh.TB, sh.n_blocks - b0);
    const uint64_t v0 = b0 * sh.Le;
    const uint32_t nv = (uint32_t)(min(sh.n, v0 + (uint64_t)sh.TB * sh.Le) - v0);
    uint8_t* og = a.out + v0 * sh.vb;
    if (terr) err |= terr;
    if (MAP == 0) {
      // 32-block groups are claimed dynamically, so a warp that is ahead takes
      // more of the tile and no warp drifts tiles behind the others; each group
      // is decoded into the warp's own staging buffer and copied out at once.
      const uint32_t ngrp = (nblk + 31) / 32;
      const uint32_t gb = 32 * L * sh.vb;  // bytes of a full group (a multiple of 64)
#pragma unroll 1
      for (uint32_t gi = 0;; ++gi) {
        uint32_t g = 0;
        if (lane == 0) g = atomicAdd(&C.gnext[s], 1u);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= ngrp) break;
        const uint32_t g0 = g * 32, b = g0 + lane;
        const uint4 h = b < nblk ? H[b] : make_uint4(0, 0, 0, 0);
        uint32_t tot;
        const uint32_t ex = warp_excl_scan(min(h.w, 0xfffffu), &tot);
        if (b < nblk && !terr && !DBG(a, 1))
          err |= decode_block0<V>(h, PAY + OFF[g] + ex, min(L, nv - b * L), L, sh.width, bc, ob + (size_t)lane * L);
        __syncwarp();
        const uint32_t bytes = min(nv * sh.vb - g0 * L * sh.vb, gb);
        uint8_t* dst = og + (size_t)g0 * L * sh.vb;
        if (!DBG(a, 8)) {
          if (a.bulk) {
            // 16-byte copies, lane-strided (a group is at most 4 KiB: <= 8 per lane)
            const uint32_t n16 = bytes >> 4;
            uint4* d4 = reinterpret_cast<uint4*>(dst) + lane;
            const uint4* s4 = reinterpret_cast<const uint4*>(ob8) + lane;
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i)
              if (lane + 32 * i < n16) d4[32 * i] = s4[32 * i];
            for (uint32_t i = 16 * n16 + lane; i < bytes; i += 32) dst[i] = ob8[i];
          } else {
            warp_copy(dst, ob8, bytes, lane);
          }
        }
        __syncwarp();
      }
    } else {
      // map 1: part p of a block (G parts) decodes one contiguous range of the
      // block's values into the tile's staging buffer; the tile store warp
      // bulk-stores the whole tile once every warp is done, so no warp waits
      // for another (the buffer was freed by the store of two tiles ago).
      mbar_wait_dec(&C.tfree[s2], ((it / NTS) & 1u) ^ 1u);
      const uint32_t G = sh.G;
#pragma unroll 1
      for (uint32_t gi = 0;; ++gi) {
        const uint32_t seg = warp + gi * NCW;
        if (seg >= sh.TB * G) break;
        const uint32_t b = seg / G, part = seg % G;
        if (b >= nblk) break;
        const uint4 h = H[b];
        const uint32_t nb = min(L, nv - b * L);
        V* dst = ob + (size_t)b * L;
        uint32_t vlo = (uint32_t)(((uint64_t)nb * part / G) & ~7ull), vhi = part + 1 == G ? nb
                                                                         : (uint32_t)(((uint64_t)nb * (part + 1) / G) & ~7ull);
        if (!terr && !DBG(a, 1)) {
          const uint32_t k = (h.x == CODEC_BASIC && h.z != 0) ? dk_of(bc, (uint64_t)h.z + 1) : 1u;
          const uint32_t e = check_block_hdr(h, nb, sh.width, k);
          err |= e;
          if (!e) {
            if (h.x == CODEC_CONSTANT) {
              for (uint32_t j = vlo + lane; j < vhi; j += 32) dst[j] = (V)h.y;
            } else {
              const DecConst c = dconst_of(bc, (uint64_t)h.z + 1);
              const uint64_t* src = PAY + OFF[b];
              bool spec = false;
              if (sizeof(V) == 2 && ((L * 2) & 15) == 0) {
                uint8_t* blk = reinterpret_cast<uint8_t*>(dst);
                const uint32_t Bu = h.z + 1;
                switch (k) {
#define POLY_UK(KK)                                                                                       \
  case KK: {                                                                                              \
    const uint32_t ng = nb / kvals<KK>(), gb = ng * part / G, ge = ng * (part + 1) / G;                   \
    err |= unpack_groups_k<KK>(src, gb, ge, c, Bu, h.y, blk);                                             \
    vlo = gb * kvals<KK>();                                                                               \
    vhi = part + 1 == G ? nb : ge * kvals<KK>();                                                          \
    if (part + 1 == G)                                                                                    \
      err |= decode_tail(src, ng * kq<KK>(), h.w, c, Bu, h.y, nb, k, dst, bc, L);                          \
    spec = true;                                                                                          \
  } break;
                  POLY_FOR_EACH_K16(POLY_UK)
#undef POLY_UK
                  default:
                    break;
                }
              }
              if (!spec) {  // generic: a contiguous range of words per part
                const uint32_t jb = (uint32_t)((uint64_t)h.w * part / G), je = (uint32_t)((uint64_t)h.w * (part + 1) / G);
                for (uint32_t j = jb + lane; j < je; j += 32)
                  err |= decode_any<V>(src[j], c, h.z, min(k, nb - j * k), h.y, dst + j * k);
                vlo = min(nb, jb * k);
                vhi = min(nb, je * k);
              }
            }
          }
        }
      }
      if (bst) fence_proxy_async_smem();
      if (warp == 0 && lane == 0) {
        C.t_og[s2] = og;
        C.t_bytes[s2] = nv * sh.vb;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&C.tfull[s2]);
    }
    __syncwarp();
    if (lane == 0) {
      if (warp == 0) TRACE(it, 7);
      // the last warp done with the stage frees its payload ring space (the
      // stages complete in order: every warp finished the previous one)
      if (atomicAdd(&C.done_cnt[s], 1u) == NCW - 1) {
        TRACE(it, 8);
        C.done_cnt[s] = 0;
        C.gnext[s] = 0;
        __threadfence_block();
        C.ring_tail = rend;
      }
      mbar_arrive(&C.empty_in[s]);
    }
  }
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0 && err) atomicOr(a.status_out, err);
}

}  // namespace polyk

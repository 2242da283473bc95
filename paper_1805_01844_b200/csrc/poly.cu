// poly.cu -- host side of the C ABI declared in include/poly.h: argument
// checks, regime selection, table upload, kernel launches.  One translation
// unit (the device tables are module globals).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "poly_common.cuh"
#include "poly_compress.cuh"
#include "poly_decompress.cuh"
#include "poly_pipe.cuh"
#include "poly_large.cuh"
#include "poly_adv.cuh"
#include "poly_dec3.cuh"
#include "poly_cmp3.cuh"

#include <vector>

using namespace polyk;

// Value type of a dtype, for the kernel templates: runs BODY with V bound.
#define POLY_DISPATCH(dt, ...)         \
  do {                                 \
    if ((dt) == POLY_U8) {             \
      typedef uint8_t V;               \
      __VA_ARGS__;                     \
    } else if ((dt) == POLY_U16) {     \
      typedef uint16_t V;              \
      __VA_ARGS__;                     \
    } else {                           \
      typedef uint32_t V;              \
      __VA_ARGS__;                     \
    }                                  \
  } while (0)

namespace {
// Smallest capacity k of any base of a width (B <= 2^w): u8 8, u16 4, u32 2.
inline uint64_t kmin_of(uint32_t w) { return w == 8 ? 8 : (w == 16 ? 4 : 2); }
inline bool dt_ok(poly_dtype_t dt) { return dt == POLY_U8 || dt == POLY_U16 || dt == POLY_U32; }
}  // namespace

namespace {
// Consumer warps of the pipeline kernels (compress / decompress).
// (measured on cfg2/4/5: more warps hide the lane-per-block latency of map 0
// and of the compress kernels; decompress map 1 is best at 16).
#ifndef POLY_NCW_C
#define POLY_NCW_C 24
#endif
#ifndef POLY_NCW_C2
#define POLY_NCW_C2 12
#endif
#ifndef POLY_NCW_D0
#define POLY_NCW_D0 26
#endif
#ifndef POLY_NCW_D1
#define POLY_NCW_D1 16
#endif
#ifndef POLY_NCW_D1B
#define POLY_NCW_D1B 12
#endif
constexpr int NCW_C = POLY_NCW_C, NCW_C2 = POLY_NCW_C2, NCW_D0 = POLY_NCW_D0, NCW_D1 = POLY_NCW_D1, NCW_D1B = POLY_NCW_D1B;
// Compress: worst-case tiles the word ring is guaranteed to hold (the input
// stages get the rest first).  At least 2: a tile's words stay contiguous, so
// an allocation that wraps skips the ring's tail end (1 tile can deadlock).
#ifndef POLY_CMP_RING_TILES
#define POLY_CMP_RING_TILES 2
#endif
static_assert(POLY_CMP_RING_TILES >= 2, "the compress word ring needs two worst-case tiles");
// Decompress header stages (the payload ring gets the rest of shared memory).
#ifndef POLY_DEC_STAGES
#define POLY_DEC_STAGES 8
#endif
constexpr int pipe_threads(int ncw) { return ncw * 32 + 32 * (2 + NLB_MAX); }


enum Regime { LARGE = 1, PIPE = 2, LARGE2 = 3 };

constexpr int MAX_DEVICES = 64;
std::mutex g_mu;
bool g_ready[MAX_DEVICES];
int g_sms[MAX_DEVICES];

typedef unsigned __int128 u128;

// Host copies of the tables (exact integer arithmetic).
uint16_t h_ktab[KTAB_MAX + 1];
DecConst h_dtab[KTAB_MAX + 1];
bool h_tables_built = false;
bool h_tables_bad = false;  // a Sec. 5.3 precondition failed (never expected)

// k = max{k : B^k <= 2^64}, h = max{h : B^h <= 2^32}; for non-powers of two
// B^k, R = ceil(2^160 / B^k) and t32 = max{t <= min(k, h) :
// 2^32 B^k + B^k + 2^64 B^t <= 2^96}.
void build_tables() {
  if (h_tables_built) return;
  const u128 word_ring = ((u128)1) << 64;
  for (uint64_t B = 0; B <= KTAB_MAX; ++B) {
    DecConst c;
    memset(&c, 0, sizeof c);
    uint32_t k = 0, h = 0, log2b = 0, t32 = 0;
    if (B >= 2) {
      u128 p = 1;
      while (p * B <= word_ring) {
        p *= B;
        ++k;
      }
      u128 q = 1;
      while (q * B <= (((u128)1) << 32)) {
        q *= B;
        ++h;
      }
      if ((B & (B - 1)) == 0) {
        while ((1ull << log2b) != B) ++log2b;
        // exact fraction: R = 2^(160 - kj), Wmax = B^k - 1, t32 = h = floor(32 / j)
        const uint32_t kj = k * log2b;
        const u128 R = ((u128)1) << (160 - kj);
        c.Rl = (uint64_t)R;
        c.Rh = (uint64_t)(R >> 64);
        c.Wmax = (uint64_t)(p - 1);
        t32 = std::min(k, 32u / log2b);
      } else {
        const uint64_t D = (uint64_t)p;  // B^k < 2^64 for non-powers of two
        // the fraction error bound needs B^k < 2^64 - 2^32
        if (word_ring - p <= ((u128)1 << 32)) h_tables_bad = true;
        u128 rem = 0, r = 0;
        for (int i = 160; i >= 0; --i) {
          rem = (rem << 1) | (i == 160 ? 1u : 0u);
          r <<= 1;
          if (rem >= D) {
            rem -= D;
            r |= 1;
          }
        }
        r += 1;  // ceil: the remainder of 2^160 / D is nonzero
        c.Wmax = D - 1;
        c.Rl = (uint64_t)r;
        c.Rh = (uint64_t)(r >> 64);
        const u128 lim96 = ((u128)1) << 96;
        u128 bt = 1;
        for (uint32_t t = 1; t <= std::min(k, h); ++t) {
          bt *= B;
          if ((((u128)D) << 32) + D + (bt << 64) <= lim96) t32 = t;
          else break;
        }
      }
    }
    c.meta = k | (log2b << 8) | (t32 << 16) | (h << 24);
    h_ktab[B] = (uint16_t)(k | (h << 8));
    h_dtab[B] = c;
  }
  // The k-specialised u16 decoders (poly_kword.cuh) switch to 32-bit steps at
  // the compile-time T32MIN[K]; it must be the least t32 over the
  // non-power-of-two bases of capacity K, else poly_init
  // fails (POLY_ERR_CUDA) rather than decode wrongly.
  {
    int lo[65];
    for (int K = 0; K <= 64; ++K) lo[K] = 1 << 30;
    for (uint64_t B = 3; B <= KTAB_MAX; ++B) {
      if ((B & (B - 1)) == 0) continue;
      const int K = (int)(h_dtab[B].meta & 0xffu), t = (int)((h_dtab[B].meta >> 16) & 0xffu);
      lo[K] = std::min(lo[K], t);
    }
#define POLY_CHECK_T32(KK) \
  if (lo[KK] != (1 << 30) && lo[KK] != t32min_u16(KK)) h_tables_bad = true; /* K = 21: B = 8 only */
    POLY_FOR_EACH_K16(POLY_CHECK_T32)
#undef POLY_CHECK_T32
  }
  h_tables_built = true;
}

// ---------------------------------------------------------------- advanced codec
// Schedule table of the split-base codec (poly_adv.cuh): for every B <= 65536
// the orbit of R' under the series of PAPER.md:244-257, R'_0 = 1, until it
// repeats -- its pre-period and one period -- with exact integers:
//   p = max{p : R' B^p <= 2^32 - 1},  R = floor((2^32 - 1) / (R' B^p)),
//   R'_next = ceil(B / R).
std::vector<adv::AdvIdx> h_aidx;
std::vector<uint4> h_aent;
std::vector<uint64_t> h_amag;
bool h_adv_built = false;
struct AdvDev {
  bool ready = false;
  adv::AdvIdx* idx = nullptr;
  uint4* ent = nullptr;
  uint64_t* rmag = nullptr;
};
AdvDev g_adv[MAX_DEVICES];

void build_adv_table() {
  if (h_adv_built) return;
  const uint64_t M = 0xffffffffull;
  h_aidx.assign(adv::BMAX + 1, adv::AdvIdx{0, 0, 1, 0});
  std::vector<int32_t> seen(adv::BMAX + 2, -1);
  std::vector<uint32_t> states;
  for (uint64_t B = 2; B <= adv::BMAX; ++B) {
    states.clear();
    uint64_t Rp = 1;  // R' <= B always (R >= 1)
    while (seen[Rp] < 0) {
      seen[Rp] = (int32_t)states.size();
      states.push_back((uint32_t)Rp);
      uint64_t x = Rp;
      while (x * B <= M) x *= B;
      const uint64_t R = M / x;
      Rp = (B + R - 1) / R;
    }
    adv::AdvIdx ix;
    ix.off = (uint32_t)h_aent.size();
    ix.pre = (uint32_t)seen[Rp];
    ix.per = (uint32_t)states.size() - ix.pre;
    uint32_t Q = 0, qcyc = 0;
    for (size_t j = 0; j < states.size(); ++j) {
      const uint64_t st = states[j];
      uint64_t x = st;
      uint32_t p = 0;
      while (x * B <= M) {
        x *= B;
        ++p;
      }
      const uint64_t R = M / x;
      h_aent.push_back(make_uint4((uint32_t)R, (uint32_t)st, Q, p));
      h_amag.push_back(R == 1 ? 0ull : (~0ull / R + 1));  // ceil(2^64 / R)
      Q += p + 1;
      if (j >= ix.pre) qcyc += p + 1;
    }
    ix.qcyc = qcyc;
    h_aidx[B] = ix;
    for (uint32_t st : states) seen[st] = -1;
  }
  h_adv_built = true;
}

poly_status_t ensure_adv(int dev, adv::AdvTab& T) {
  std::lock_guard<std::mutex> lk(g_mu);
  AdvDev& d = g_adv[dev];
  if (!d.ready) {
    build_adv_table();
    if (cudaMalloc(&d.idx, sizeof(adv::AdvIdx) * h_aidx.size()) != cudaSuccess ||
        cudaMalloc(&d.ent, sizeof(uint4) * h_aent.size()) != cudaSuccess ||
        cudaMalloc(&d.rmag, sizeof(uint64_t) * h_amag.size()) != cudaSuccess ||
        cudaMemcpy(d.idx, h_aidx.data(), sizeof(adv::AdvIdx) * h_aidx.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(d.ent, h_aent.data(), sizeof(uint4) * h_aent.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(d.rmag, h_amag.data(), sizeof(uint64_t) * h_amag.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return POLY_ERR_CUDA;
    d.ready = true;
  }
  T.idx = d.idx;
  T.ent = d.ent;
  T.rmag = d.rmag;
  return POLY_OK;
}

struct AdvPlan {
  uint64_t n, Le, n_blocks, last_len, n_chunks, o_cstat, o_nw, o_woff, ws_bytes;
};
bool plan_adv(uint64_t n, poly_dtype_t dt, uint64_t block_size, AdvPlan& P) {
  if (n == 0 || dt != POLY_U16 || block_size >= (1ull << 32)) return false;
  P.n = n;
  P.Le = block_size ? block_size : n;
  P.n_blocks = (n + P.Le - 1) / P.Le;
  if (P.n_blocks >= (1ull << 32) || P.Le >= (1ull << 32)) return false;
  P.last_len = n - (P.n_blocks - 1) * P.Le;
  P.n_chunks = (P.n_blocks + adv::SCHUNK - 1) / adv::SCHUNK;
  P.o_cstat = 64;
  P.o_nw = (64 + 8 * P.n_chunks + 15) / 16 * 16;
  P.o_woff = (P.o_nw + 4 * P.n_blocks + 15) / 16 * 16;
  P.ws_bytes = P.o_woff + 8 * P.n_blocks;
  return true;
}

adv::Args adv_args(const AdvPlan& P, uint64_t block_size, uint8_t* ws, const adv::AdvTab& T) {
  adv::Args a;
  memset(&a, 0, sizeof a);
  a.T = T;
  a.n = P.n;
  a.Le = P.Le;
  a.n_blocks = P.n_blocks;
  a.last_len = P.last_len;
  a.n_chunks = P.n_chunks;
  a.block_len = (uint32_t)block_size;
  a.warp_per_block = P.Le > 64 ? 1u : 0u;
  a.ticket = reinterpret_cast<uint32_t*>(ws);
  a.cstat = reinterpret_cast<uint64_t*>(ws + P.o_cstat);
  a.nw = reinterpret_cast<uint32_t*>(ws + P.o_nw);
  a.woff = reinterpret_cast<uint64_t*>(ws + P.o_woff);
  return a;
}

template <typename K>
void set_smem_attr(K kernel, int bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <typename V>
uint32_t large_smem_pack() { return ((CH_VALUES + 64) * sizeof(V) + 15) / 16 * 16; }
template <typename V>
uint32_t large_smem_unpack() {
  return 16 * ((CH_VALUES + 64) * sizeof(V) / 16 + 1) + 8 * (CH_VALUES / 2 + 2);
}

template <typename V>
void set_attrs(int pmax) {
  set_smem_attr(poly_compress_pipe<V, 0, NCW_C>, pmax);
  set_smem_attr(poly_compress_pipe<V, 1, NCW_C>, pmax);
  set_smem_attr(poly_compress_pipe<V, 1, NCW_C2>, pmax);
  set_smem_attr(poly_decompress_pipe<V, 0, NCW_D0>, pmax);
  set_smem_attr(poly_decompress_pipe<V, 1, NCW_D1>, pmax);
  set_smem_attr(poly_decompress_pipe<V, 1, NCW_D1B>, pmax);
  set_smem_attr(poly_compress_large<V>, pmax);
  set_smem_attr(poly_decompress_large<V>, pmax);
  set_smem_attr(poly_compress_pack<V>, large_smem_pack<V>());
  set_smem_attr(poly_decompress_unpack<V>, large_smem_unpack<V>());
  set_smem_attr(poly_decompress_large1<V>, large_smem_unpack<V>());
  set_smem_attr(poly_compress_large1<V>, large_smem_pack<V>());
  set_smem_attr(d3::dec3_main<V>, 227 * 1024);
  set_smem_attr(c3::cmp3<V, false>, 227 * 1024);
  set_smem_attr(c3::cmp3<V, true>, 227 * 1024);
}

poly_status_t ensure_init(int dev) {
  if (dev < 0 || dev >= MAX_DEVICES) return POLY_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_ready[dev]) return POLY_OK;
  build_tables();
  if (h_tables_bad) return POLY_ERR_CUDA;
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return POLY_ERR_CUDA;
  if (cur != dev && cudaSetDevice(dev) != cudaSuccess) return POLY_ERR_CUDA;
  cudaError_t e = cudaMemcpyToSymbol(g_ktab, h_ktab, sizeof h_ktab);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_dtab, h_dtab, sizeof h_dtab);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev);
  const int pmax = (POLY_CTAS == 1 ? 227 : 113) * 1024;
  set_attrs<uint8_t>(pmax);
  set_attrs<uint16_t>(pmax);
  set_attrs<uint32_t>(pmax);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (cur != dev) cudaSetDevice(cur);
  if (e != cudaSuccess) return POLY_ERR_CUDA;
  g_ready[dev] = true;
  return POLY_OK;
}

// Regime and launch shape for (n, w, block_size).  Deterministic: the same
// arguments always give the same shape (the stream does not depend on it).
constexpr uint32_t WT_TARGET = 4096;  // input bytes per warp unit (target)

constexpr uint32_t PIPE_TILE_TARGET = 32768 / POLY_CTAS;          // value bytes per tile (target)
constexpr uint32_t PIPE_SMEM_MAX = (POLY_CTAS == 1 ? 227 : 113) * 1024;  // shared memory per CTA

uint32_t r16(uint64_t x) { return (uint32_t)((x + 15) / 16 * 16); }

// Tile shape and shared-memory layout of the pipeline kernels (poly_pipe.cuh).
bool plan_pipe_n(const Shape& sh, PipeShape& ps, bool decomp, uint32_t ncw) {
  const uint32_t pc = 32 * ncw;
  memset(&ps, 0, sizeof ps);
  ps.ncw = ncw;
  ps.n = sh.n;
  ps.Le = sh.Le;
  ps.n_blocks = sh.n_blocks;
  ps.block_len = sh.block_len;
  ps.width = sh.width;
  ps.vb = sh.width / 8;
  const uint64_t bb = sh.Le * ps.vb;
  const uint64_t kmin = kmin_of(sh.width);
  if (bb <= MAP0_MAX_BLOCK) {
    ps.map = 0;
    uint64_t bpt = PIPE_TILE_TARGET / (pc * bb);
    bpt = std::max<uint64_t>(1, std::min<uint64_t>(BPT_MAX, bpt));
    ps.bpt = (uint32_t)bpt;
    ps.TB = (uint32_t)(pc * bpt);
  } else {
    ps.map = 1;
    uint64_t tb = PIPE_TILE_TARGET / bb;
    tb = std::max<uint64_t>(1, std::min<uint64_t>(256, tb));
    ps.TB = (uint32_t)tb;
    uint32_t G = 1;
    while (ps.TB * G * 2 <= ncw && ncw % (G * 2) == 0) G *= 2;  // a block's G warps: a whole group
    ps.G = G;
    // a whole number of segments (block parts) per consumer warp
    const uint32_t per = std::max<uint32_t>(1, ncw / G);
    ps.TB = std::max<uint32_t>(per, ps.TB / per * per);
    ps.Lp = (uint32_t)(((sh.Le + G - 1) / G + 7) / 8 * 8);
  }
  ps.tile_bytes = (uint32_t)(ps.TB * bb);
  ps.words_cap = (uint32_t)(ps.TB * ((sh.Le + kmin - 1) / kmin));
  ps.n_tiles = (sh.n_blocks + ps.TB - 1) / ps.TB;
  if (ps.n_tiles >= (1ull << 32)) return false;
  const uint32_t ctl = (uint32_t)((sizeof(PipeCtl) + 127) / 128 * 128);
  const uint32_t cache = cache_bytes(decomp);
  ps.o_cache = ctl;
  const uint32_t base = ctl + cache;
  if (!decomp) {
    // input ring (S stages) + word ring (the rest, >= 2 worst-case tiles)
    const uint32_t stage = r16(ps.tile_bytes) + 128;  // slack: the top-word pack may read past a block
    const uint32_t tile_words = r16(8ull * ps.words_cap + 16);
    int64_t room = (int64_t)PIPE_SMEM_MAX - base - POLY_CMP_RING_TILES * (int64_t)tile_words;
    if (room < 2 * (int64_t)stage) return false;
    ps.S = (uint32_t)std::min<int64_t>(4, room / stage);
    ps.in_stride = stage;
    ps.o_in = base;
    ps.o_ring = base + ps.S * stage;
    ps.ring_bytes = (PIPE_SMEM_MAX - ps.o_ring) / 16 * 16;
    if (ps.map == 0 && ps.bpt == 1 && POLY_CMP_WARP_RINGS) {
      // one word ring per consumer warp, each >= 2 worst-case warp segments;
      // when they do not fit (u32 blocks of many values), the shared ring
      const uint32_t wseg = r16(8ull * 32 * ((sh.Le + kmin - 1) / kmin) + 16);
      const uint32_t per = (PIPE_SMEM_MAX - ps.o_ring) / ncw / 16 * 16;
      if (per >= 2 * wseg) {
        ps.wrings = 1;
        ps.ring_bytes = per;
      }
    }
    ps.smem = ps.o_ring + (ps.wrings ? ncw * ps.ring_bytes : ps.ring_bytes);
  } else {
    ps.o_off = 16 * ps.TB;
    const uint32_t stage = ps.o_off + r16(4ull * ps.TB);
    // staging of the decoded values: map 0, one 32-block group per consumer
    // warp (copied out right after it is decoded); map 1, two tiles
    // (bulk stores, the buffer is rewritten two tiles later)
    const bool perwarp = ps.map == 0;
    const uint32_t outb = ps.map == 0 ? r16(32ull * bb) : perwarp ? r16(bb) : r16(ps.tile_bytes);
    const uint32_t outs = perwarp ? ncw * outb : 2 * outb;
    // the payload ring (the remainder) holds at least one worst-case tile
    const uint32_t tile_pay = r16(8ull * (ps.words_cap + 2));
    const int64_t room = (int64_t)PIPE_SMEM_MAX - base - (int64_t)outs - (int64_t)tile_pay;
    if (room < 2 * (int64_t)stage) return false;
    ps.S = (uint32_t)std::min<int64_t>(std::min<int64_t>(MAXS, POLY_DEC_STAGES), room / stage);
    ps.in_stride = stage;
    ps.out_stride = outb;
    ps.o_in = base;
    ps.o_out = base + ps.S * stage;
    ps.o_ring = ps.o_out + outs;
    ps.ring_bytes = (PIPE_SMEM_MAX - ps.o_ring) / 16 * 16;
    ps.smem = ps.o_ring + ps.ring_bytes;
  }
  return ps.smem <= PIPE_SMEM_MAX;
}

// Consumer-warp count per kernel: compress NCW_C; decompress map 0 NCW_D0;
// decompress map 1 the instantiation (NCW_D1 or NCW_D1B) whose plan gives the
// larger block parts (fewer warps per block: fewer group barriers and part
// tails), ties to the larger warp count (measured: cfg5 12 warps / 4 KiB
// parts 1751 GB/s vs 16 / 2 KiB 1439; cfg4 16 warps).
// Compress of blocks whose byte size is a multiple of 16 (poly_cmp3.cuh):
// tiles of about C3_TILE bytes in S slots, S a multiple of the writer count.
bool plan_c3(const Shape& sh, PipeShape& ps) {
  memset(&ps, 0, sizeof ps);
  const uint64_t bb = sh.Le * (sh.width / 8);
  if (bb <= MAP0_MAX_BLOCK || bb > PIPE_MAX_BLOCK || bb % 16 != 0) return false;
  ps.c3 = 1;
  ps.map = 1;
  ps.ncw = c3::NW;
  ps.n = sh.n;
  ps.Le = sh.Le;
  ps.n_blocks = sh.n_blocks;
  ps.block_len = sh.block_len;
  ps.width = sh.width;
  ps.vb = sh.width / 8;
  ps.TB = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(c3::TBMAX, c3::C3_TILE / bb));
  // G = blocks per consumer claim: a power of two <= 32 with about 8 KiB of
  // values per claim (small blocks share one claim's overheads), TB a multiple
  uint32_t cb = 1;
  while (cb < 32 && 2ull * cb * bb <= c3::C3_CLAIM && 2 * cb <= ps.TB) cb *= 2;
  ps.G = cb;
  ps.TB = ps.TB / cb * cb;
  ps.tile_bytes = (uint32_t)(ps.TB * bb);
  ps.words_cap = (uint32_t)(ps.TB * ((sh.Le + kmin_of(sh.width) - 1) / kmin_of(sh.width)));
  ps.n_tiles = (sh.n_blocks + ps.TB - 1) / ps.TB;
  if (ps.n_tiles >= (1ull << 32)) return false;
  ps.o_cache = (uint32_t)((sizeof(c3::Ctl) + 127) / 128 * 128);
  ps.o_in = (ps.o_cache + cache_bytes(false) + 127) / 128 * 128;
  ps.in_stride = (ps.tile_bytes + 127) / 128 * 128;
  uint32_t S = std::min<uint32_t>(c3::MAXS3, (PIPE_SMEM_MAX - ps.o_in) / ps.in_stride);
  S = S / c3::NWR * c3::NWR;
  if (S < (uint32_t)c3::NWR || S < 2) return false;
  ps.S = S;
  ps.smem = ps.o_in + S * ps.in_stride;
  return true;
}

bool plan_pipe(const Shape& sh, PipeShape& ps, bool decomp) {
  const bool map0 = (uint64_t)sh.Le * (sh.width / 8) <= MAP0_MAX_BLOCK;
  if (!decomp && !map0 && plan_c3(sh, ps)) return true;
  if (!decomp) {
    // map 1: NCW_C2 warps when NCW_C would split each block over 4 or more
    // warps and the smaller count keeps the tile (measured, cfg5: 24 warps /
    // 1024-value parts 2725 GB/s, 12 / 2048 2980; cfg6, G 2 -> 1, and cfg4,
    // G = 1 either way, keep NCW_C)
    if (!plan_pipe_n(sh, ps, false, NCW_C)) return false;
    PipeShape b;
    if (ps.map == 1 && ps.G >= 4 && plan_pipe_n(sh, b, false, NCW_C2) && b.G < ps.G && b.tile_bytes == ps.tile_bytes)
      ps = b;
    return true;
  }
  if (map0) return plan_pipe_n(sh, ps, true, NCW_D0);
  PipeShape a, b;
  const bool oa = plan_pipe_n(sh, a, true, NCW_D1), ob = plan_pipe_n(sh, b, true, NCW_D1B);
  if (oa && (!ob || a.G <= b.G)) {
    ps = a;
    return true;
  }
  ps = b;
  return ob;
}

// Large blocks, one CTA per block (poly_large.cuh): sub-tiles of 32 KiB plus a
// halo, S stages; decompress adds two staging buffers of one sub-tile.
constexpr uint64_t LARGE2_MIN_BLOCKS = 256;     // enough blocks to occupy every SM
constexpr uint64_t LARGE2_MAX_BLOCK = 4 << 20;  // bytes: sweep 1 must find the block in L2
bool plan_large(const Shape& sh, LargeShape& ls, bool decomp) {
  memset(&ls, 0, sizeof ls);
  ls.n = sh.n;
  ls.Le = sh.Le;
  ls.n_blocks = sh.n_blocks;
  ls.block_len = sh.block_len;
  ls.width = sh.width;
  ls.vb = sh.width / 8;
  ls.SV = 32768 / ls.vb;
  ls.nsub = (uint32_t)((sh.Le + ls.SV - 1) / ls.SV);
  const uint32_t ctl = (uint32_t)((sizeof(LargeCtl) + 127) / 128 * 128);
  if (!decomp) {
    ls.stage = r16((uint64_t)(ls.SV + LG_HALO) * ls.vb);
    ls.S = 4;
    ls.o_in = ctl;
    ls.smem = ctl + ls.S * ls.stage;
  } else {
    const uint64_t kmin = kmin_of(sh.width);
    ls.stage = r16(8ull * (ls.SV / kmin + 4));
    const uint32_t outb = 2 * ls.SV * ls.vb;
    ls.S = (uint32_t)std::min<uint64_t>(MAXS, (PIPE_SMEM_MAX - ctl - outb) / ls.stage);
    if (ls.S < 2) return false;
    ls.o_in = ctl;
    ls.o_out = ctl + ls.S * ls.stage;
    ls.smem = ls.o_out + outb;
  }
  return ls.smem <= PIPE_SMEM_MAX;
}

bool plan(uint64_t n, uint32_t w, uint64_t block_size, Shape& sh, Regime& rg) {
  if (n == 0 || (w != 8 && w != 16 && w != 32) || block_size >= (1ull << 32)) return false;
  memset(&sh, 0, sizeof sh);
  sh.n = n;
  sh.width = w;
  sh.block_len = (uint32_t)block_size;
  sh.Le = block_size == 0 ? n : block_size;
  sh.n_blocks = (n + sh.Le - 1) / sh.Le;
  if (sh.n_blocks >= (1ull << 32)) return false;
  // a block header holds n_words in 32 bits: ceil(L_e / k_min) < 2^32 (only a
  // block_size = 0 call with n >= 2^33 (u32) / 2^34 (u16) exceeds it)
  if ((sh.Le + kmin_of(w) - 1) / kmin_of(w) >= (1ull << 32)) return false;
  const uint64_t bb = sh.Le * (w / 8);  // bytes per block
  PipeShape pc, pd;
  LargeShape lc, ld;
  if (bb <= PIPE_MAX_BLOCK && plan_pipe(sh, pc, false) && plan_pipe(sh, pd, true)) {
    rg = PIPE;
    sh.n_chunks = std::max(pc.n_tiles, pd.n_tiles);  // tiles (look-back units) of either direction
  } else if (bb <= LARGE2_MAX_BLOCK && sh.n_blocks >= LARGE2_MIN_BLOCKS && plan_large(sh, lc, false) &&
             plan_large(sh, ld, true)) {
    rg = LARGE2;
    sh.n_chunks = sh.n_blocks;  // blocks (look-back units)
  } else {
    rg = LARGE;
    sh.cpb = (sh.Le + CH_VALUES - 1) / CH_VALUES;
    sh.n_chunks = sh.n_blocks * sh.cpb;
    sh.n_stiles = (sh.n_blocks + SCAN_T - 1) / SCAN_T;
  }
  return true;
}

// ---------------------------------------------------------------- dec3
// Two-pass decompress of the map-1 regime (128 B < block <= 32 KiB,
// poly_dec3.cuh): shapes, shared memory, workspace.
struct Dec3Plan {
  d3::Args a;
  uint32_t smem;
  uint64_t ws_bytes, o_cw, o_cu, o_T;
};
uint64_t dec3_units_max(uint64_t blen, uint32_t ut, uint32_t kmin) {
  uint64_t m = 1;
  for (uint32_t k = kmin; k <= 64; ++k) {
    uint32_t w = (ut / k) & ~7u;
    if (w < 8) w = 8;
    const uint64_t nw = (blen + k - 1) / k;
    m = std::max<uint64_t>(m, (nw + w - 1) / w);
  }
  return m;
}
bool plan_dec3(const Shape& sh, Dec3Plan& P) {
  memset(&P, 0, sizeof P);
  d3::Args& a = P.a;
  a.n = sh.n;
  a.Le = sh.Le;
  a.n_blocks = sh.n_blocks;
  a.last_len = sh.n - (sh.n_blocks - 1) * sh.Le;
  a.block_len = sh.block_len;
  a.width = sh.width;
  a.vb = sh.width / 8;
  a.kmin_log2 = sh.width == 8 ? 3u : (sh.width == 16 ? 2u : 1u);
  a.ut = 4096 / a.vb;
  a.n_chunks = (sh.n_blocks + d3::CE - 1) / d3::CE;
  const uint32_t kmin = 1u << a.kmin_log2;
  a.max_units = (sh.n_blocks - 1) * dec3_units_max(sh.Le, a.ut, kmin) + dec3_units_max(a.last_len, a.ut, kmin);
  // a staging buffer holds a unit of up to capv values (unit_words) plus the
  // 16-byte alignment shift of the generic path and the group codec's overhang
  // past a unit's last value (< 32 u16 values: poly_kword.cuh unpack_group_p);
  // two per warp (TMA stores)
  a.capv = a.ut + 128u;
  a.cap = (uint32_t)((a.capv * a.vb + 32 + 64 + 15) / 16 * 16);
  a.o_warp = (uint32_t)((sizeof(d3::Ctl) + 127) / 128 * 128);
  a.o_ring = (a.o_warp + d3::NW * 2 * a.cap + 127) / 128 * 128;
  const uint32_t smax = 227 * 1024;
  a.ring_bytes = (smax - a.o_ring) / 16 * 16;
  // worst tile: TU units of <= ut / k_min + 8 words, their headers, the table entries
  const uint64_t worst = 16ull * d3::TU + 16ull * (d3::TU + 1) + 8ull * d3::TU * (a.ut / kmin + 8) + 64;
  if (worst > a.ring_bytes / 2) return false;
  P.smem = smax;
  P.o_cw = 64;
  P.o_cu = 64 + 8 * a.n_chunks;
  P.o_T = (P.o_cu + 8 * a.n_chunks + 15) / 16 * 16;
  P.ws_bytes = P.o_T + 16 * (a.max_units + 1);
  return true;
}
bool use_dec3(const Shape& sh) {
  const uint64_t bb = sh.Le * (sh.width / 8);
  return bb > MAP0_MAX_BLOCK && bb <= PIPE_MAX_BLOCK;
}

struct WsLayout {
  uint64_t status_off, bmin_off, bmax_off, woff_off, total;
};

WsLayout ws_layout(const Shape& sh, Regime rg) {
  WsLayout L;
  memset(&L, 0, sizeof L);
  L.status_off = 64;
  if (rg == PIPE || rg == LARGE2) {
    L.total = 64 + 8 * sh.n_chunks;
  } else {
    // bmin / bmax: per-block running min / max (three-kernel path) or per-chunk
    // partials (single-launch path, poly_compress_large1)
    const uint64_t nmm = std::max(sh.n_blocks, sh.n_chunks);
    L.bmin_off = (64 + 8 * sh.n_stiles + 15) / 16 * 16;
    L.bmax_off = (L.bmin_off + 4 * nmm + 15) / 16 * 16;
    L.woff_off = (L.bmax_off + 4 * nmm + 15) / 16 * 16;
    L.total = L.woff_off + 8 * sh.n_blocks;
  }
  return L;
}

// The LARGE regime in one launch per call (poly_compress_large1 /
// poly_decompress_large1): a few blocks and chunks (cfg1: one 2 MiB block).
bool large1_compress(const Shape& sh) {
  return sh.n_blocks <= LARGE1C_MAX_BLOCKS && sh.n_chunks <= LARGE1C_MAX_CHUNKS;
}
bool large1_decompress(const Shape& sh) { return sh.n_blocks <= LARGE1_MAX_BLOCKS; }

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

int grid_for(uint64_t work, int dev) {
  const uint64_t cap = (uint64_t)(g_sms[dev] > 0 ? g_sms[dev] : 148) * 8;
  return (int)std::min<uint64_t>(work, cap);
}


#ifdef POLY_TIMING
// Timing-experiment variant library only (never the product library): the
// POLY_DEBUG bits skip per-block compute (1), the look-back (2) or stores
// (4, 8, 16); the output is then wrong (profiles/ab_bench.sh).
uint32_t debug_flags() {
  const char* e = getenv("POLY_DEBUG");
  return e ? (uint32_t)strtoul(e, nullptr, 0) : 0u;
}
#else
uint32_t debug_flags() { return 0u; }
#endif
// Look-back / writer warps per CTA.
uint32_t lb_warps(uint32_t dflt, uint32_t vmax) { return std::max(1u, std::min(dflt, vmax)); }

template <typename K>
int pipe_grid(K kernel, uint32_t smem, uint64_t tiles, int dev, int threads = PT) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const uint64_t cap = (uint64_t)(g_sms[dev] > 0 ? g_sms[dev] : 148) * per_sm;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(cap, tiles));
}
// Grid of a pipeline launch: worker CTAs plus, when there is more than one
// tile, the prefix-server CTA.  Every worker of tile t >= 1 waits on the
// server, so the grid must be co-resident: such launches are cooperative
// (launch_k), which the driver only starts when every CTA fits (it never
// exceeds the occupancy bound computed here).
template <typename K>
int pipe_grid_server(K kernel, int threads, uint32_t smem, uint64_t tiles, int dev, uint32_t& server) {
  const int cap = pipe_grid(kernel, smem, ~0ull, dev, threads);
  server = (tiles > 1 && cap >= 2) ? 1u : 0u;
  const uint64_t workers = std::min<uint64_t>(tiles, (uint64_t)cap - server);
  return (int)(std::max<uint64_t>(1, workers) + server);
}

// Launch `kernel` (cooperatively when `coop`: a grid whose CTAs wait on one
// another -- the prefix server -- must be resident all at once).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), int grid, int threads, uint32_t smem, cudaStream_t s, bool coop,
                     Args... args) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = coop ? attr : nullptr;
  cfg.numAttrs = coop ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace

// One poly_compress_pipe launch over tiles [t_begin, t_end) (clipped to the
// plan); the caller zeroes the status words once per stream and the ticket
// word before every launch.
void launch_compress_pipe(const Shape& sh, poly_dtype_t dt, const void* d_in, uint8_t* d_out,
                          uint64_t* d_compressed_bytes, uint8_t* ws, const WsLayout& W, uint64_t t_begin,
                          uint64_t t_end, cudaStream_t s, int dev) {
  PipeArgs pa;
  memset(&pa, 0, sizeof pa);
  plan_pipe(sh, pa.sh, false);
  pa.in = reinterpret_cast<const uint8_t*>(d_in);
  pa.out = d_out;
  pa.compressed_bytes = d_compressed_bytes;
  pa.status = reinterpret_cast<uint64_t*>(ws + W.status_off);
  pa.ticket = reinterpret_cast<uint32_t*>(ws);
  pa.bulk = ((reinterpret_cast<uintptr_t>(d_in) & 15) == 0 && pa.sh.tile_bytes % 16 == 0) ? 1u : 0u;
  pa.tma_shift = ((reinterpret_cast<uintptr_t>(d_in) & 15) == 0 && pa.sh.tile_bytes % 16 != 0) ? 1u : 0u;
  pa.debug = debug_flags();
  pa.t_begin = t_begin;
  pa.t_end = std::min<uint64_t>(t_end, pa.sh.n_tiles);
  // per-warp word rings (map 0, one block per thread) move the tile assembly
  // to the writers: 4 of them keep up (measured: 2 -> 1254, 4 -> 2078 GB/s cfg2)
  const bool wr = pa.sh.wrings != 0;
  pa.nlb = lb_warps(wr ? 4 : 2, NLB_MAX + 1);
  if (pa.sh.c3) {
    pa.nlb = c3::NWR;
    POLY_DISPATCH(dt, {
      auto k = pa.sh.G > 1 ? c3::cmp3<V, true> : c3::cmp3<V, false>;
      const int grid = pipe_grid_server(k, c3::NTHR, pa.sh.smem, pa.t_end - pa.t_begin, dev, pa.server);
      launch_k(k, grid, c3::NTHR, pa.sh.smem, s, pa.server != 0, pa);
    });
    return;
  }
  POLY_DISPATCH(dt, {
    auto k = pa.sh.map == 0         ? poly_compress_pipe<V, 0, NCW_C>
             : pa.sh.ncw == NCW_C ? poly_compress_pipe<V, 1, NCW_C>
                                  : poly_compress_pipe<V, 1, NCW_C2>;
    const int nt = pipe_threads((int)pa.sh.ncw);
    const int grid = pipe_grid_server(k, nt, pa.sh.smem, pa.t_end - pa.t_begin, dev, pa.server);
    launch_k(k, grid, nt, pa.sh.smem, s, pa.server != 0, pa);
  });
}

// One poly_decompress_pipe launch over tiles [t_begin, t_end) (clipped).
void launch_decompress_pipe(const Shape& sh, poly_dtype_t dt, const uint8_t* d_in, uint64_t compressed_bytes,
                            void* d_out, uint32_t* d_status, uint8_t* ws, const WsLayout& W, uint64_t t_begin,
                            uint64_t t_end, cudaStream_t s, int dev) {
  PipeArgs pa;
  memset(&pa, 0, sizeof pa);
  plan_pipe(sh, pa.sh, true);
  pa.in = d_in;
  pa.out = reinterpret_cast<uint8_t*>(d_out);
  pa.in_bytes = compressed_bytes;
  pa.status_out = d_status;
  pa.status = reinterpret_cast<uint64_t*>(ws + W.status_off);
  pa.ticket = reinterpret_cast<uint32_t*>(ws);
  pa.bulk = ((reinterpret_cast<uintptr_t>(d_out) & 15) == 0 && pa.sh.tile_bytes % 16 == 0) ? 1u : 0u;
  pa.debug = debug_flags();
  pa.t_begin = t_begin;
  pa.t_end = std::min<uint64_t>(t_end, pa.sh.n_tiles);
  // a look-back warp waits on stage i's barrier only after finishing stage
  // i - nlb, so nlb <= S keeps every parity wait within one phase
  // (map 1: the last helper warp is the tile store warp)
  // (map 1: one look-back warp, measured cfg5 1948 -> 2044 GB/s, cfg4 1390 -> 1398)
  pa.nlb = lb_warps(pa.sh.map == 1 ? 1 : 2, std::min<uint32_t>(pa.sh.map != 0 ? NLB_MAX - 1 : NLB_MAX, pa.sh.S));
  POLY_DISPATCH(dt, {
    auto k = pa.sh.map == 0 ? poly_decompress_pipe<V, 0, NCW_D0>
             : pa.sh.ncw == NCW_D1 ? poly_decompress_pipe<V, 1, NCW_D1> : poly_decompress_pipe<V, 1, NCW_D1B>;
    const int nt = pipe_threads((int)pa.sh.ncw);
    const int grid = pipe_grid_server(k, nt, pa.sh.smem, pa.t_end - pa.t_begin, dev, pa.server);
    launch_k(k, grid, nt, pa.sh.smem, s, pa.server != 0, pa);
  });
}

// Streams, events and pinned prefix slots of the chunked host calls.
constexpr int HOST_CHUNKS = 8;
struct HostPipe {
  bool ready = false;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t in[HOST_CHUNKS], kern[HOST_CHUNKS], start;
  uint64_t* hP = nullptr;  // pinned: inclusive word prefix after each chunk
};
HostPipe g_hp[MAX_DEVICES];
// One chunked host call per device at a time: the events and the pinned
// prefix slots of g_hp[dev] are per device, not per call.
std::mutex g_host_mu[MAX_DEVICES];
bool host_pipe(int dev, HostPipe*& hp) {
  std::lock_guard<std::mutex> lk(g_mu);
  hp = &g_hp[dev];
  if (hp->ready) return true;
  if (cudaStreamCreateWithFlags(&hp->h2d, cudaStreamNonBlocking) != cudaSuccess) return false;
  if (cudaStreamCreateWithFlags(&hp->d2h, cudaStreamNonBlocking) != cudaSuccess) return false;
  for (int c = 0; c < HOST_CHUNKS; ++c) {
    if (cudaEventCreateWithFlags(&hp->in[c], cudaEventDisableTiming) != cudaSuccess) return false;
    if (cudaEventCreateWithFlags(&hp->kern[c], cudaEventDisableTiming) != cudaSuccess) return false;
  }
  if (cudaEventCreateWithFlags(&hp->start, cudaEventDisableTiming) != cudaSuccess) return false;
  if (cudaHostAlloc(reinterpret_cast<void**>(&hp->hP), 8 * HOST_CHUNKS, cudaHostAllocDefault) != cudaSuccess)
    return false;
  hp->ready = true;
  return true;
}

extern "C" {

int poly_version(void) { return 200; }

int poly_tables_ok(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  build_tables();
  return h_tables_bad ? 0 : 1;
}

const char* poly_status_string(poly_status_t s) {
  switch (s) {
    case POLY_OK: return "POLY_OK";
    case POLY_ERR_INVALID_ARG: return "POLY_ERR_INVALID_ARG";
    case POLY_ERR_EMPTY_INPUT: return "POLY_ERR_EMPTY_INPUT";
    case POLY_ERR_CAPACITY: return "POLY_ERR_CAPACITY";
    case POLY_ERR_WORKSPACE: return "POLY_ERR_WORKSPACE";
    case POLY_ERR_CUDA: return "POLY_ERR_CUDA";
    case POLY_ERR_CORRUPT: return "POLY_ERR_CORRUPT";
  }
  return "POLY_UNKNOWN";
}

poly_status_t poly_init(int device) { return ensure_init(device); }

uint64_t poly_max_compressed_bytes(uint64_t n, poly_dtype_t dt, uint64_t block_size) {
  if (n == 0 || !dt_ok(dt)) return 0;
  const uint64_t L = block_size == 0 ? n : block_size;
  const uint64_t nb = (n + L - 1) / L;
  const uint64_t kmin = kmin_of((uint32_t)dt);
  const uint64_t full = n / L, last = n - full * L;
  uint64_t words = full * ((L + kmin - 1) / kmin);
  if (last) words += (last + kmin - 1) / kmin;
  return 32 + 16 * nb + 8 * words;
}

uint64_t poly_workspace_bytes(uint64_t n, poly_dtype_t dt, uint64_t block_size) {
  Shape sh;
  Regime rg;
  if (!plan(n, (uint32_t)dt, block_size, sh, rg)) return 0;
  uint64_t t = ws_layout(sh, rg).total;
  Dec3Plan dp;
  if (rg == PIPE && use_dec3(sh) && plan_dec3(sh, dp)) t = std::max<uint64_t>(t, dp.ws_bytes);
  return t;
}

#ifdef POLY_TRACE
// Timing experiments only (not in include/poly.h): the pipeline event trace.
int poly_trace_reset(void) {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, polyk::g_trace) != cudaSuccess) return 1;
  return cudaMemset(p, 0xff, sizeof(polyk::g_trace)) == cudaSuccess ? 0 : 1;
}
int poly_trace_dump(void* host, uint64_t bytes) {
  if (bytes > sizeof(polyk::g_trace)) bytes = sizeof(polyk::g_trace);
  return cudaMemcpyFromSymbol(host, polyk::g_trace, bytes) == cudaSuccess ? 0 : 1;
}
uint64_t poly_trace_bytes(void) { return sizeof(polyk::g_trace); }
#endif

#ifdef POLY_PROBE
// Timing experiments only (not in include/poly.h): dec3 cycle counters.
int poly_probe_reset(void) {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, polyk::d3::g_probe) != cudaSuccess) return 1;
  return cudaMemset(p, 0, sizeof(polyk::d3::g_probe)) == cudaSuccess ? 0 : 1;
}
int poly_probe_dump(void* host) {  // 24 u64
  return cudaMemcpyFromSymbol(host, polyk::d3::g_probe, sizeof(polyk::d3::g_probe)) == cudaSuccess ? 0 : 1;
}
#endif

int poly_launches_per_call(uint64_t n, poly_dtype_t dt, uint64_t block_size, int decompress) {
  Shape sh;
  Regime rg;
  if (!plan(n, (uint32_t)dt, block_size, sh, rg)) return 0;
  if (decompress && rg == PIPE && use_dec3(sh)) return 2;  // unit table + decode (poly_dec3.cuh)
  if (rg == PIPE || rg == LARGE2) return 1;
  if (decompress) return large1_decompress(sh) ? 1 : 2;
  return large1_compress(sh) ? 1 : 3;
}

poly_status_t poly_compress(const void* d_in, uint64_t n, poly_dtype_t dt, uint64_t block_size,
                            void* d_out, uint64_t out_capacity, uint64_t* d_compressed_bytes,
                            void* d_workspace, uint64_t workspace_bytes, void* stream) {
  if (!dt_ok(dt)) return POLY_ERR_INVALID_ARG;
  if (n == 0) return POLY_ERR_EMPTY_INPUT;
  if (!d_in || !d_out || !d_compressed_bytes || !d_workspace) return POLY_ERR_INVALID_ARG;
  const uint32_t vb = (uint32_t)dt / 8;
  if ((reinterpret_cast<uintptr_t>(d_in) % vb) != 0) return POLY_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(d_out) & 15) != 0) return POLY_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(d_compressed_bytes) & 7) != 0) return POLY_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(d_workspace) & 15) != 0) return POLY_ERR_INVALID_ARG;
  Shape sh;
  Regime rg;
  if (!plan(n, (uint32_t)dt, block_size, sh, rg)) return POLY_ERR_INVALID_ARG;
  if (out_capacity < poly_max_compressed_bytes(n, dt, block_size)) return POLY_ERR_CAPACITY;
  const WsLayout W = ws_layout(sh, rg);
  if (workspace_bytes < W.total) return POLY_ERR_WORKSPACE;
  const int dev = current_device();
  poly_status_t st = ensure_init(dev);
  if (st != POLY_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_workspace);

  CompressArgs a;
  memset(&a, 0, sizeof a);
  a.in = d_in;
  a.out = reinterpret_cast<uint8_t*>(d_out);
  a.compressed_bytes = d_compressed_bytes;
  a.ticket = reinterpret_cast<uint32_t*>(ws);
  a.status = reinterpret_cast<uint64_t*>(ws + W.status_off);
  a.sh = sh;
  if (rg == LARGE2) {
    cudaMemsetAsync(ws, 0, W.total, s);
    LargeArgs la;
    memset(&la, 0, sizeof la);
    plan_large(sh, la.sh, false);
    la.in = reinterpret_cast<const uint8_t*>(d_in);
    la.out = a.out;
    la.compressed_bytes = d_compressed_bytes;
    la.status = a.status;
    la.ticket = a.ticket;
    la.bulk = ((reinterpret_cast<uintptr_t>(d_in) & 15) == 0 && (sh.Le * (dt / 8)) % 16 == 0) ? 1u : 0u;
    POLY_DISPATCH(dt, {
      auto k = poly_compress_large<V>;
      const int grid = pipe_grid_server(k, PT, la.sh.smem, sh.n_blocks, dev, la.server);
      launch_k(k, grid, PT, la.sh.smem, s, la.server != 0, la);
    });
  } else if (rg == PIPE) {
    cudaMemsetAsync(ws, 0, W.total, s);
    launch_compress_pipe(sh, dt, d_in, a.out, d_compressed_bytes, ws, W, 0, ~0ull, s, dev);
  } else {
    a.bmin = reinterpret_cast<uint32_t*>(ws + W.bmin_off);
    a.bmax = reinterpret_cast<uint32_t*>(ws + W.bmax_off);
    a.woff = reinterpret_cast<uint64_t*>(ws + W.woff_off);
    cudaMemsetAsync(ws, 0, W.bmin_off, s);
    if (large1_compress(sh)) {  // one cooperative launch (grid barrier inside)
      POLY_DISPATCH(dt, {
        auto k = poly_compress_large1<V>;
        const uint32_t smem = large_smem_pack<V>();
        const int grid = pipe_grid(k, smem, sh.n_chunks, dev, NT);
        launch_k(k, grid, NT, smem, s, true, a);
      });
      if (cudaGetLastError() != cudaSuccess) return POLY_ERR_CUDA;
      return POLY_OK;
    }
    cudaMemsetAsync(a.bmin, 0xff, 4 * sh.n_blocks, s);
    cudaMemsetAsync(a.bmax, 0, 4 * sh.n_blocks, s);
    const int gr = grid_for(sh.n_chunks, dev);
    POLY_DISPATCH(dt, {
      poly_compress_minmax<V><<<gr, NT, 0, s>>>(a);
      poly_compress_block_scan<<<(unsigned)sh.n_stiles, NT, 0, s>>>(a);
      poly_compress_pack<V><<<gr, NT, large_smem_pack<V>(), s>>>(a);
    });
  }
  if (cudaGetLastError() != cudaSuccess) return POLY_ERR_CUDA;
  return POLY_OK;
}

poly_status_t poly_read_header(const void* h_hdr32, uint64_t* n, poly_dtype_t* dt,
                               uint64_t* block_size, uint64_t* n_blocks, uint64_t* payload_bytes) {
  if (!h_hdr32) return POLY_ERR_INVALID_ARG;
  const uint8_t* p = reinterpret_cast<const uint8_t*>(h_hdr32);
  if (memcmp(p, "PLYC", 4) != 0 || p[4] != 2 || p[5] != 0 || p[7] != 0 || (p[6] != 8 && p[6] != 16 && p[6] != 32))
    return POLY_ERR_CORRUPT;
  uint64_t nn, pb;
  uint32_t bl, nb;
  memcpy(&nn, p + 8, 8);
  memcpy(&bl, p + 16, 4);
  memcpy(&nb, p + 20, 4);
  memcpy(&pb, p + 24, 8);
  if (n) *n = nn;
  if (dt) *dt = (poly_dtype_t)p[6];
  if (block_size) *block_size = bl;
  if (n_blocks) *n_blocks = nb;
  if (payload_bytes) *payload_bytes = pb;
  return POLY_OK;
}

poly_status_t poly_decompress(const void* d_in, uint64_t compressed_bytes, poly_dtype_t dt,
                              uint64_t n, uint64_t block_size, void* d_out, uint32_t* d_status,
                              void* d_workspace, uint64_t workspace_bytes, void* stream) {
  if (!dt_ok(dt)) return POLY_ERR_INVALID_ARG;
  if (n == 0) return POLY_ERR_EMPTY_INPUT;
  if (!d_in || !d_out || !d_status || !d_workspace) return POLY_ERR_INVALID_ARG;
  const uint32_t vb = (uint32_t)dt / 8;
  if ((reinterpret_cast<uintptr_t>(d_in) & 15) != 0) return POLY_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(d_out) % vb) != 0) return POLY_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(d_workspace) & 15) != 0) return POLY_ERR_INVALID_ARG;
  Shape sh;
  Regime rg;
  if (!plan(n, (uint32_t)dt, block_size, sh, rg)) return POLY_ERR_INVALID_ARG;
  const WsLayout W = ws_layout(sh, rg);
  if (workspace_bytes < W.total) return POLY_ERR_WORKSPACE;
  const int dev = current_device();
  poly_status_t st = ensure_init(dev);
  if (st != POLY_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_workspace);

  DecompressArgs a;
  memset(&a, 0, sizeof a);
  a.in = reinterpret_cast<const uint8_t*>(d_in);
  a.compressed_bytes = compressed_bytes;
  a.out = d_out;
  a.status_out = d_status;
  a.ticket = reinterpret_cast<uint32_t*>(ws);
  a.status = reinterpret_cast<uint64_t*>(ws + W.status_off);
  a.sh = sh;
  cudaMemsetAsync(d_status, 0, 4, s);
  Dec3Plan dp;
  if (rg == PIPE && use_dec3(sh) && plan_dec3(sh, dp)) {
    if (workspace_bytes < dp.ws_bytes) return POLY_ERR_WORKSPACE;
    d3::Args d = dp.a;
    d.in = a.in;
    d.in_bytes = compressed_bytes;
    d.out = reinterpret_cast<uint8_t*>(d_out);
    d.status_out = d_status;
    d.ticket = reinterpret_cast<uint32_t*>(ws);
    d.abort_flag = reinterpret_cast<uint32_t*>(ws + 4);
    d.n_units = reinterpret_cast<uint64_t*>(ws + 8);
    d.cst_w = reinterpret_cast<uint64_t*>(ws + dp.o_cw);
    d.cst_u = reinterpret_cast<uint64_t*>(ws + dp.o_cu);
    d.T = reinterpret_cast<uint4*>(ws + dp.o_T);
    d.kw_ok = dt != POLY_U16 ? 0u
              : ((reinterpret_cast<uintptr_t>(d_out) & 15) == 0 && (sh.Le * 2) % 16 == 0) ? 1u : 2u;
    cudaMemsetAsync(ws, 0, dp.o_T, s);
    const uint64_t sms = (uint64_t)(g_sms[dev] > 0 ? g_sms[dev] : 148);
    const unsigned g1 = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(d.n_chunks, 4 * sms));
    d3::dec3_offsets<<<g1, d3::K1T, 0, s>>>(d);
    POLY_DISPATCH(dt, { d3::dec3_main<V><<<(unsigned)sms, d3::NTHR, dp.smem, s>>>(d); });
    if (cudaGetLastError() != cudaSuccess) return POLY_ERR_CUDA;
    return POLY_OK;
  }
  if (rg == LARGE2) {
    cudaMemsetAsync(ws, 0, W.total, s);
    LargeArgs la;
    memset(&la, 0, sizeof la);
    plan_large(sh, la.sh, true);
    la.in = a.in;
    la.out = reinterpret_cast<uint8_t*>(d_out);
    la.in_bytes = compressed_bytes;
    la.status_out = d_status;
    la.status = a.status;
    la.ticket = a.ticket;
    la.bulk = ((reinterpret_cast<uintptr_t>(d_out) & 15) == 0 && (sh.Le * (dt / 8)) % 16 == 0) ? 1u : 0u;
    POLY_DISPATCH(dt, {
      auto k = poly_decompress_large<V>;
      const int grid = pipe_grid_server(k, PT, la.sh.smem, sh.n_blocks, dev, la.server);
      launch_k(k, grid, PT, la.sh.smem, s, la.server != 0, la);
    });
  } else if (rg == PIPE) {
    cudaMemsetAsync(ws, 0, W.total, s);
    launch_decompress_pipe(sh, dt, a.in, compressed_bytes, d_out, d_status, ws, W, 0, ~0ull, s, dev);
  } else {
    a.woff = reinterpret_cast<uint64_t*>(ws + W.woff_off);
    const int gr = grid_for(sh.n_chunks, dev);
    if (large1_decompress(sh)) {  // one launch: every CTA scans the few headers itself
      POLY_DISPATCH(dt, { poly_decompress_large1<V><<<gr, NT, large_smem_unpack<V>(), s>>>(a); });
      if (cudaGetLastError() != cudaSuccess) return POLY_ERR_CUDA;
      return POLY_OK;
    }
    cudaMemsetAsync(ws, 0, W.bmin_off, s);
    poly_decompress_block_scan<<<(unsigned)sh.n_stiles, NT, 0, s>>>(a);
    POLY_DISPATCH(dt, { poly_decompress_unpack<V><<<gr, NT, large_smem_unpack<V>(), s>>>(a); });
  }
  if (cudaGetLastError() != cudaSuccess) return POLY_ERR_CUDA;
  return POLY_OK;
}

uint64_t poly_max_compressed_bytes_advanced(uint64_t n, poly_dtype_t dt, uint64_t block_size) {
  AdvPlan P;
  if (!plan_adv(n, dt, block_size, P)) return 0;
  return 32 + 16 * P.n_blocks + 4 * (n + P.n_blocks);  // a word holds >= 1 value; the last may hold a carry only
}

uint64_t poly_workspace_bytes_advanced(uint64_t n, poly_dtype_t dt, uint64_t block_size) {
  AdvPlan P;
  if (!plan_adv(n, dt, block_size, P)) return 0;
  return P.ws_bytes;
}

poly_status_t poly_compress_advanced(const void* d_in, uint64_t n, poly_dtype_t dt, uint64_t block_size,
                                     void* d_out, uint64_t out_capacity, uint64_t* d_compressed_bytes,
                                     void* d_workspace, uint64_t workspace_bytes, void* stream) {
  if (n == 0) return POLY_ERR_EMPTY_INPUT;
  if (dt != POLY_U16 || !d_in || !d_out || !d_compressed_bytes || !d_workspace) return POLY_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(d_in) & 1) || (reinterpret_cast<uintptr_t>(d_out) & 15) ||
      (reinterpret_cast<uintptr_t>(d_workspace) & 15))
    return POLY_ERR_INVALID_ARG;
  AdvPlan P;
  if (!plan_adv(n, dt, block_size, P)) return POLY_ERR_INVALID_ARG;
  if (out_capacity < poly_max_compressed_bytes_advanced(n, dt, block_size)) return POLY_ERR_CAPACITY;
  if (workspace_bytes < P.ws_bytes) return POLY_ERR_WORKSPACE;
  const int dev = current_device();
  poly_status_t st = ensure_init(dev);
  adv::AdvTab T;
  if (st == POLY_OK) st = ensure_adv(dev, T);
  if (st != POLY_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_workspace);
  adv::Args a = adv_args(P, block_size, ws, T);
  a.in = reinterpret_cast<const uint8_t*>(d_in);
  a.out = reinterpret_cast<uint8_t*>(d_out);
  a.compressed_bytes = d_compressed_bytes;
  cudaMemsetAsync(ws, 0, P.o_nw, s);
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(
      a.warp_per_block ? (P.n_blocks + 7) / 8 : (P.n_blocks + adv::NTA - 1) / adv::NTA, 148ull * 16));
  adv::adv_stats<uint16_t><<<g, adv::NTA, 0, s>>>(a);
  adv::adv_scan<<<(unsigned)P.n_chunks, adv::NTA, 0, s>>>(a, 1u);
  adv::adv_pack<uint16_t><<<g, adv::NTA, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? POLY_OK : POLY_ERR_CUDA;
}

poly_status_t poly_decompress_advanced(const void* d_in, uint64_t compressed_bytes, poly_dtype_t dt,
                                       uint64_t n, uint64_t block_size, void* d_out, uint32_t* d_status,
                                       void* d_workspace, uint64_t workspace_bytes, void* stream) {
  if (n == 0) return POLY_ERR_EMPTY_INPUT;
  if (dt != POLY_U16 || !d_in || !d_out || !d_status || !d_workspace) return POLY_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(d_in) & 15) || (reinterpret_cast<uintptr_t>(d_out) & 1) ||
      (reinterpret_cast<uintptr_t>(d_workspace) & 15))
    return POLY_ERR_INVALID_ARG;
  AdvPlan P;
  if (!plan_adv(n, dt, block_size, P)) return POLY_ERR_INVALID_ARG;
  if (workspace_bytes < P.ws_bytes) return POLY_ERR_WORKSPACE;
  const int dev = current_device();
  poly_status_t st = ensure_init(dev);
  adv::AdvTab T;
  if (st == POLY_OK) st = ensure_adv(dev, T);
  if (st != POLY_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_workspace);
  adv::Args a = adv_args(P, block_size, ws, T);
  a.in = reinterpret_cast<const uint8_t*>(d_in);
  a.in_bytes = compressed_bytes;
  a.out = reinterpret_cast<uint8_t*>(d_out);
  a.status_out = d_status;
  cudaMemsetAsync(d_status, 0, 4, s);
  cudaMemsetAsync(ws, 0, P.o_nw, s);
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(
      a.warp_per_block ? (P.n_blocks + 7) / 8 : (P.n_blocks + adv::NTA - 1) / adv::NTA, 148ull * 16));
  adv::adv_check_header<<<1, 1, 0, s>>>(a);
  adv::adv_scan<<<(unsigned)P.n_chunks, adv::NTA, 0, s>>>(a, 0u);
  adv::adv_unpack<uint16_t><<<g, adv::NTA, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? POLY_OK : POLY_ERR_CUDA;
}

poly_status_t poly_compress_host(const void* h_in, uint64_t n, poly_dtype_t dt, uint64_t block_size,
                                 void* h_out, uint64_t h_out_capacity, uint64_t* h_compressed_bytes,
                                 void* d_in_scratch, void* d_out_scratch, uint64_t d_out_capacity,
                                 void* d_workspace, uint64_t workspace_bytes, void* stream) {
  if (!h_in || !h_out || !h_compressed_bytes || !d_in_scratch) return POLY_ERR_INVALID_ARG;
  if (!dt_ok(dt)) return POLY_ERR_INVALID_ARG;
  if (n == 0) return POLY_ERR_EMPTY_INPUT;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_workspace);
  if (!ws) return POLY_ERR_INVALID_ARG;
  {
    // Chunked path (pipeline regime): the values go up in HOST_CHUNKS pieces
    // on one copy stream, each piece is compressed by a launch over its tiles
    // (the prefix continues across launches), and each piece's headers and
    // payload come down on another copy stream while the next piece goes up
    // -- PCIe carries both directions at once.
    Shape sh;
    Regime rg;
    const uint32_t vb = (uint32_t)dt / 8;
    if (plan(n, (uint32_t)dt, block_size, sh, rg) && rg == PIPE &&
        (reinterpret_cast<uintptr_t>(d_in_scratch) % 16) == 0 && (reinterpret_cast<uintptr_t>(d_out_scratch) & 15) == 0 &&
        d_out_capacity >= poly_max_compressed_bytes(n, dt, block_size)) {
      PipeShape ps;
      plan_pipe(sh, ps, false);
      const WsLayout W = ws_layout(sh, rg);
      const int dev = current_device();
      HostPipe* hp = nullptr;
      if (ps.n_tiles >= 2 * HOST_CHUNKS && workspace_bytes >= W.total && ensure_init(dev) == POLY_OK &&
          host_pipe(dev, hp)) {
        std::lock_guard<std::mutex> call_lock(g_host_mu[dev]);
        const uint64_t T = ps.n_tiles, tvals = (uint64_t)ps.TB * sh.Le;
        const uint8_t* hin = reinterpret_cast<const uint8_t*>(h_in);
        uint8_t* din = reinterpret_cast<uint8_t*>(d_in_scratch);
        uint8_t* dout = reinterpret_cast<uint8_t*>(d_out_scratch);
        uint8_t* hout = reinterpret_cast<uint8_t*>(h_out);
        uint64_t* d_nbytes = reinterpret_cast<uint64_t*>(ws + 8);
        const uint64_t* status = reinterpret_cast<const uint64_t*>(ws + W.status_off);
        uint64_t tb[HOST_CHUNKS + 1];
        for (int c = 0; c <= HOST_CHUNKS; ++c) tb[c] = T * c / HOST_CHUNKS;
        // the copy streams start after the caller's earlier work on `s`
        bool ok = cudaEventRecord(hp->start, s) == cudaSuccess && cudaStreamWaitEvent(hp->h2d, hp->start, 0) == cudaSuccess &&
                  cudaStreamWaitEvent(hp->d2h, hp->start, 0) == cudaSuccess && cudaMemsetAsync(ws, 0, W.total, s) == cudaSuccess;
        for (int c = 0; c < HOST_CHUNKS && ok; ++c) {  // values up
          const uint64_t v0 = std::min<uint64_t>(n, tb[c] * tvals), v1 = std::min<uint64_t>(n, tb[c + 1] * tvals);
          ok = cudaMemcpyAsync(din + v0 * vb, hin + v0 * vb, (v1 - v0) * vb, cudaMemcpyHostToDevice, hp->h2d) ==
                   cudaSuccess &&
               cudaEventRecord(hp->in[c], hp->h2d) == cudaSuccess;
        }
        for (int c = 0; c < HOST_CHUNKS && ok; ++c) {  // compress each piece
          ok = cudaStreamWaitEvent(s, hp->in[c], 0) == cudaSuccess && cudaMemsetAsync(ws, 0, 4, s) == cudaSuccess;
          if (!ok) break;
          launch_compress_pipe(sh, dt, d_in_scratch, dout, d_nbytes, ws, W, tb[c], tb[c + 1], s, dev);
          ok = cudaGetLastError() == cudaSuccess &&
               cudaMemcpyAsync(hp->hP + c, status + tb[c + 1] - 1, 8, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
               cudaEventRecord(hp->kern[c], s) == cudaSuccess;
        }
        const uint64_t hdr0 = 32, pay0 = 32 + 16 * sh.n_blocks;
        uint64_t P0 = 0;
        for (int c = 0; c < HOST_CHUNKS && ok; ++c) {  // stream down, piece by piece
          ok = cudaEventSynchronize(hp->kern[c]) == cudaSuccess;
          if (!ok) break;
          const uint64_t P1 = hp->hP[c] & VAL_MASK;
          const uint64_t b0 = tb[c] * ps.TB, b1 = std::min<uint64_t>(sh.n_blocks, tb[c + 1] * ps.TB);
          if (pay0 + 8 * P1 > h_out_capacity) {
            // drain every copy and kernel of this call before returning
            cudaStreamSynchronize(s);
            cudaStreamSynchronize(hp->h2d);
            cudaStreamSynchronize(hp->d2h);
            return POLY_ERR_CAPACITY;
          }
          ok = cudaStreamWaitEvent(hp->d2h, hp->kern[c], 0) == cudaSuccess &&
               cudaMemcpyAsync(hout + hdr0 + 16 * b0, dout + hdr0 + 16 * b0, 16 * (b1 - b0), cudaMemcpyDeviceToHost,
                               hp->d2h) == cudaSuccess &&
               (P1 == P0 || cudaMemcpyAsync(hout + pay0 + 8 * P0, dout + pay0 + 8 * P0, 8 * (P1 - P0),
                                            cudaMemcpyDeviceToHost, hp->d2h) == cudaSuccess);
          P0 = P1;
        }
        if (ok) ok = cudaMemcpyAsync(hout, dout, 32, cudaMemcpyDeviceToHost, hp->d2h) == cudaSuccess;
        if (cudaStreamSynchronize(hp->d2h) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) ok = false;
        if (!ok) return POLY_ERR_CUDA;
        *h_compressed_bytes = pay0 + 8 * P0;
        return POLY_OK;
      }
    }
  }
  if (cudaMemcpyAsync(d_in_scratch, h_in, n * ((uint32_t)dt / 8), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return POLY_ERR_CUDA;
  uint64_t* d_nbytes = reinterpret_cast<uint64_t*>(ws + 8);
  poly_status_t st = poly_compress(d_in_scratch, n, dt, block_size, d_out_scratch, d_out_capacity,
                                   d_nbytes, d_workspace, workspace_bytes, stream);
  if (st != POLY_OK) return st;
  if (cudaMemcpyAsync(h_compressed_bytes, d_nbytes, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return POLY_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return POLY_ERR_CUDA;
  if (*h_compressed_bytes > h_out_capacity) return POLY_ERR_CAPACITY;
  if (cudaMemcpyAsync(h_out, d_out_scratch, *h_compressed_bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return POLY_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return POLY_ERR_CUDA;
  return POLY_OK;
}

poly_status_t poly_decompress_host(const void* h_in, uint64_t compressed_bytes, poly_dtype_t dt,
                                   uint64_t n, uint64_t block_size, void* h_out, uint32_t* h_status,
                                   void* d_in_scratch, void* d_out_scratch,
                                   void* d_workspace, uint64_t workspace_bytes, void* stream) {
  if (!h_in || !h_out || !h_status || !d_in_scratch || !d_out_scratch || !d_workspace)
    return POLY_ERR_INVALID_ARG;
  if (!dt_ok(dt)) return POLY_ERR_INVALID_ARG;
  if (n == 0) return POLY_ERR_EMPTY_INPUT;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_workspace);
  if (cudaMemcpyAsync(d_in_scratch, h_in, compressed_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return POLY_ERR_CUDA;
  uint32_t* d_st = reinterpret_cast<uint32_t*>(ws + 16);
  poly_status_t st = poly_decompress(d_in_scratch, compressed_bytes, dt, n, block_size, d_out_scratch,
                                     d_st, d_workspace, workspace_bytes, stream);
  if (st != POLY_OK) return st;
  if (cudaMemcpyAsync(h_out, d_out_scratch, n * ((uint32_t)dt / 8), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return POLY_ERR_CUDA;
  if (cudaMemcpyAsync(h_status, d_st, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return POLY_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return POLY_ERR_CUDA;
  return POLY_OK;
}

}  // extern "C"

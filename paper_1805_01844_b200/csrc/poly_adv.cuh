// poly_adv.cuh -- the ADVANCED (split-base) polynomial codec of PAPER.md
// Sec. 3.2 on u16 blocks (Sec. 3.3), 32-bit words, word-
// parallel: SURVEY.md Sec. 8(f) row 1.
//
// The paper's series is sequential in the word index: word i
// depends on R'_{i-1}.  But R'_i is a function of R'_{i-1} alone (for a fixed
// B), so the sequence R'_0 = 1, R'_1, ... is eventually periodic; the host
// tabulates, for every B <= 65536, its pre-period and one period (601,575
// entries in all, pre-period <= 7, period <= 510; built exactly in
// poly.cu build_adv_table).  Word i's (p_i, R_i, R'_{i-1}) and the number q_i
// of values before it are then an O(1) lookup, and every word is packed /
// unpacked by its own thread:
//   non-final word i: s_i = r_i + R_i (r'_{i-1} B^{p_i} + sum_k d[q_i+k] B^(p_i-1-k)),
//                     d[q_i + p_i] = r'_i R_i + r_i  (the split value);
//   final word (values left m <= p_i): r'_{i-1} B^m + sum_k d[q_i+k] B^(m-1-k).
// A thread packing word i reads the previous word's split value for r'_{i-1};
// a thread unpacking word i writes its full digits and completes the previous
// word's split value with its carry r'_{i-1} and the previous word's remainder.
// Divisions by R_i and B are exact 64-bit reciprocal multiplies (Lemire, Kaser,
// Kurz 2019: floor(n / d) = (ceil(2^64 / d) n) >> 64 for 32-bit n and d).
#pragma once
#include "poly_common.cuh"
#include "poly_word.cuh"

namespace polyk {
namespace adv {

constexpr uint32_t BMAX = 65536;
constexpr uint64_t WMAX32 = 0xffffffffull;
constexpr uint32_t CODEC_ADVANCED = 3;
constexpr int NTA = 256;

struct __align__(16) AdvIdx {
  uint32_t off;   // first table entry of base B
  uint32_t pre;   // pre-period (words before the cycle)
  uint32_t per;   // period
  uint32_t qcyc;  // values consumed by one period
};
// entry j of base B: x = R_j, y = R'_{j-1} (the carry base), z = values
// consumed before word j within the listing, w = p_j; plus ceil(2^64 / R_j).
struct AdvTab {
  const AdvIdx* idx;
  const uint4* ent;
  const uint64_t* rmag;
};

struct Args {
  const uint8_t* in;   // compress: values; decompress: stream
  uint8_t* out;        // compress: stream; decompress: values
  uint64_t in_bytes;   // decompress: stream bytes
  uint64_t* compressed_bytes;
  uint32_t* status_out;
  uint32_t* nw;        // per block: words (compress stats -> scan)
  uint64_t* woff;      // per block: first word (exclusive scan)
  uint64_t* cstat;     // scan look-back words
  uint32_t* ticket;
  AdvTab T;
  uint64_t n, Le, n_blocks, last_len, n_chunks;
  uint32_t block_len;
  uint32_t warp_per_block;  // 1: a warp per block (lanes over words); 0: a thread per block
};

__device__ __forceinline__ uint32_t blen_of(const Args& a, uint64_t b) {
  return (uint32_t)(b + 1 == a.n_blocks ? a.last_len : a.Le);
}
// floor(n / d) for n < 2^32, d >= 1, with m = ceil(2^64 / d) (m = 0 stands for d = 1)
__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint64_t m) {
  return m ? (uint32_t)__umul64hi(m, (uint64_t)n) : n;
}

struct Word {
  uint32_t R, Rp_prev, p;
  uint64_t q;
  uint64_t mag;
};
// word i of a block of base B (the schedule)
__device__ __forceinline__ Word word_of(const AdvTab& T, uint32_t B, uint64_t i) {
  const AdvIdx x = T.idx[B];
  uint64_t j = i, cyc = 0;
  if (i >= x.pre) {
    const uint64_t t = i - x.pre;
    cyc = t / x.per;
    j = x.pre + (t - cyc * x.per);
  }
  const uint4 e = T.ent[x.off + j];
  Word w;
  w.R = e.x;
  w.Rp_prev = e.y;
  w.p = e.w;
  w.q = (uint64_t)e.z + cyc * x.qcyc;
  w.mag = T.rmag[x.off + j];
  return w;
}
// words of a block of n values: the least i with q_i + p_i >= n, plus one
// (q_i + p_i is strictly increasing in i; the answer is < n + 1)
__device__ __forceinline__ uint64_t word_count(const AdvTab& T, uint32_t B, uint64_t n) {
  uint64_t lo = 0, hi = n;  // q_n + p_n >= n
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    const Word w = word_of(T, B, mid);
    if (w.q + w.p >= n) hi = mid;
    else lo = mid + 1;
  }
  return lo + 1;
}

// ------------------------------------------------------------------ pack
// Word i of a block (v: its values, vmin, base B, n values).
template <typename V>
__device__ __forceinline__ uint32_t pack_word_adv(const AdvTab& T, const V* v, uint32_t vmin, uint32_t B, uint32_t n,
                                                  uint64_t i) {
  const Word w = word_of(T, B, i);
  uint32_t carry = 0;  // r'_{i-1}
  if (i > 0) {
    const Word wp = word_of(T, B, i - 1);
    carry = fdiv((uint32_t)v[wp.q + wp.p] - vmin, wp.mag);
  }
  const uint32_t left = (uint32_t)(n - w.q);
  const bool fin = left <= w.p;
  const uint32_t m = fin ? left : w.p;
  uint32_t body = carry;
  for (uint32_t k = 0; k < m; ++k) body = body * B + ((uint32_t)v[w.q + k] - vmin);  // < R'_{i-1} B^p <= 2^32 - 1
  if (fin) return body;
  const uint32_t sv = (uint32_t)v[w.q + w.p] - vmin;  // the split value
  const uint32_t rp = fdiv(sv, w.mag);
  return (sv - rp * w.R) + w.R * body;  // r_i + R_i body <= 2^32 - 1 (tightness)
}

// Stats: v_min, B, CONSTANT / ADVANCED, word count; header written.
template <typename V>
__global__ void __launch_bounds__(NTA) adv_stats(Args a) {
  const V* in = reinterpret_cast<const V*>(a.in);
  uint4* hdr = reinterpret_cast<uint4*>(a.out + 32);
  const int lane = threadIdx.x & 31;
  if (a.warp_per_block) {
    const uint64_t nwarps = (uint64_t)gridDim.x * (NTA / 32);
    for (uint64_t b = blockIdx.x * (uint64_t)(NTA / 32) + (threadIdx.x >> 5); b < a.n_blocks; b += nwarps) {
      const uint32_t n = blen_of(a, b);
      const V* v = in + b * a.Le;
      uint32_t mn = 0xffffffffu, mx = 0;
      for (uint32_t i = lane; i < n; i += 32) {
        const uint32_t x = v[i];
        mn = min(mn, x);
        mx = max(mx, x);
      }
      mn = __reduce_min_sync(0xffffffffu, mn);
      mx = __reduce_max_sync(0xffffffffu, mx);
      if (lane == 0) {
        const uint32_t B = mx - mn + 1;
        const uint32_t nw = B == 1 ? 0u : (uint32_t)word_count(a.T, B, n);
        a.nw[b] = nw;
        hdr[b] = make_uint4(B == 1 ? CODEC_CONSTANT : CODEC_ADVANCED, mn, mx - mn, nw);
      }
    }
  } else {
    for (uint64_t b = blockIdx.x * (uint64_t)NTA + threadIdx.x; b < a.n_blocks; b += (uint64_t)gridDim.x * NTA) {
      const uint32_t n = blen_of(a, b);
      const V* v = in + b * a.Le;
      uint32_t mn = 0xffffffffu, mx = 0;
      for (uint32_t i = 0; i < n; ++i) {
        const uint32_t x = v[i];
        mn = min(mn, x);
        mx = max(mx, x);
      }
      const uint32_t B = mx - mn + 1;
      const uint32_t nw = B == 1 ? 0u : (uint32_t)word_count(a.T, B, n);
      a.nw[b] = nw;
      hdr[b] = make_uint4(B == 1 ? CODEC_CONSTANT : CODEC_ADVANCED, mn, mx - mn, nw);
    }
  }
}

// Global header of an advanced stream (layout byte 1): POLY_ST_* bits.
__device__ __forceinline__ uint32_t adv_header_err(const Args& a) {
  uint32_t e = 0;
  if (a.in_bytes < 32) {
    e = POLY_ST_LENGTH;
  } else {
    const uint4 h0 = reinterpret_cast<const uint4*>(a.in)[0], h1 = reinterpret_cast<const uint4*>(a.in)[1];
    const uint64_t n = (uint64_t)h0.z | ((uint64_t)h0.w << 32), pb = (uint64_t)h1.z | ((uint64_t)h1.w << 32);
    if (h0.x != 0x43594c50u) e = POLY_ST_BAD_MAGIC;
    else if ((h0.y & 0xffu) != 2u) e = POLY_ST_BAD_VERSION;
    else if (((h0.y >> 8) & 0xffu) != 1u || ((h0.y >> 16) & 0xffu) != 16u || (h0.y >> 24) != 0u || n != a.n ||
             h1.x != a.block_len || h1.y != (uint32_t)a.n_blocks)
      e = POLY_ST_HEADER_MISMATCH;
    else if ((pb & 3) != 0 || a.in_bytes < 32 + 16 * a.n_blocks || pb != a.in_bytes - (32 + 16 * a.n_blocks))
      e = POLY_ST_LENGTH;
  }
  return e;
}
__global__ void adv_check_header(Args a) {
  const uint32_t e = adv_header_err(a);
  if (e) atomicOr(a.status_out, e);
}


// Exclusive scan of nw[] -> woff[] (chunks of NTA * 16 blocks, decoupled
// look-back in ticket order); the last chunk writes the global header.
constexpr uint32_t SCHUNK = NTA * 16;
__global__ void __launch_bounds__(NTA) adv_scan(Args a, uint32_t compress) {
  __shared__ uint64_t s_v[SCHUNK + 1], s_w[NTA / 32];
  __shared__ uint32_t s_c;
  __shared__ uint64_t s_pre;
  const int tid = threadIdx.x;
  if (tid == 0) s_c = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint64_t c = s_c;
  const uint64_t b0 = c * SCHUNK;
  if (b0 >= a.n_blocks) return;
  if (!compress && adv_header_err(a)) return;  // reported by adv_check_header
  const uint32_t nb = (uint32_t)min((uint64_t)SCHUNK, a.n_blocks - b0);
  if (compress) {
    for (uint32_t i = tid; i < nb; i += NTA) s_v[i] = a.nw[b0 + i];
  } else {  // n_words clamped to n_b + 1 (the most a valid block has): the sums cannot wrap
    const uint4* hdr = reinterpret_cast<const uint4*>(a.in + 32);
    for (uint32_t i = tid; i < nb; i += NTA) s_v[i] = min(hdr[b0 + i].w, blen_of(a, b0 + i) + 1);
  }
  __syncthreads();
  const uint64_t total = cta_exclusive_scan<uint64_t>(s_v, s_v, nb, s_w);
  // cta_exclusive_scan (NT = 256 threads) leaves s_v exclusive; publish, look back
  if (tid < 32) {
    uint64_t p = 0;
    if (tid == 0) st_relaxed_u64(a.cstat + c, (c == 0 ? FLAG_PRE : FLAG_AGG) | (total & VAL_MASK));
    if (c != 0) {
      p = lookback(a.cstat, c);
      if (tid == 0) st_relaxed_u64(a.cstat + c, FLAG_PRE | ((p + total) & VAL_MASK));
    }
    if (tid == 0) s_pre = p;
  }
  __syncthreads();
  const uint64_t P = s_pre;
  for (uint32_t i = tid; i < nb; i += NTA) a.woff[b0 + i] = P + s_v[i];
  if (compress && b0 + nb == a.n_blocks && tid == 0) {
    uint4 h0, h1;
    h0.x = 0x43594c50u;  // "PLYC", version 2, layout 1 (advanced, 32-bit words), width 16
    h0.y = 2u | (1u << 8) | (16u << 16);
    h0.z = (uint32_t)a.n;
    h0.w = (uint32_t)(a.n >> 32);
    h1.x = a.block_len;
    h1.y = (uint32_t)a.n_blocks;
    const uint64_t pb = 4 * (P + total);
    h1.z = (uint32_t)pb;
    h1.w = (uint32_t)(pb >> 32);
    reinterpret_cast<uint4*>(a.out)[0] = h0;
    reinterpret_cast<uint4*>(a.out)[1] = h1;
    *a.compressed_bytes = 32 + 16 * a.n_blocks + pb;
  }
  if (!compress && b0 + nb == a.n_blocks && tid == 0) {
    const uint64_t pb = a.in_bytes - (32 + 16 * a.n_blocks);
    if (4 * (P + total) != pb) atomicOr(a.status_out, POLY_ST_LENGTH);
  }
}

template <typename V>
__global__ void __launch_bounds__(NTA) adv_pack(Args a) {
  const V* in = reinterpret_cast<const V*>(a.in);
  const uint4* hdr = reinterpret_cast<const uint4*>(a.out + 32);
  uint32_t* pay = reinterpret_cast<uint32_t*>(a.out + 32 + 16 * a.n_blocks);
  const int lane = threadIdx.x & 31;
  const uint64_t step = a.warp_per_block ? (uint64_t)gridDim.x * (NTA / 32) : (uint64_t)gridDim.x * NTA;
  const uint64_t first = a.warp_per_block ? blockIdx.x * (uint64_t)(NTA / 32) + (threadIdx.x >> 5)
                                          : blockIdx.x * (uint64_t)NTA + threadIdx.x;
  for (uint64_t b = first; b < a.n_blocks; b += step) {
    const uint4 h = hdr[b];
    if (h.w == 0) continue;
    const uint32_t n = blen_of(a, b), B = h.z + 1;
    uint32_t* dst = pay + a.woff[b];
    const V* v = in + b * a.Le;
    if (a.warp_per_block) {
      for (uint32_t i = lane; i < h.w; i += 32) dst[i] = pack_word_adv<V>(a.T, v, h.y, B, n, i);
    } else {
      for (uint32_t i = 0; i < h.w; ++i) dst[i] = pack_word_adv<V>(a.T, v, h.y, B, n, i);
    }
  }
}

// ------------------------------------------------------------------ unpack
// Header checks (a9) of an advanced stream's block; returns POLY_ST_* bits.
__device__ __forceinline__ uint32_t check_adv_block(const AdvTab& T, uint4 h, uint32_t n) {
  if (h.x == CODEC_CONSTANT) {
    uint32_t e = 0;
    if (h.z != 0 || h.w != 0) e |= POLY_ST_NWORDS;
    if (h.y > 0xffffu) e |= POLY_ST_OVERFLOW;
    return e;
  }
  if (h.x != CODEC_ADVANCED) return POLY_ST_BAD_CODEC;
  if (h.z == 0 || (uint64_t)h.y + h.z > 0xffffu) return POLY_ST_OVERFLOW;
  if (h.w != word_count(T, h.z + 1, n)) return POLY_ST_NWORDS;
  return 0;
}

// Word i: its full digits, and the previous word's split value.
template <typename V>
__device__ __forceinline__ uint32_t unpack_word_adv(const AdvTab& T, const uint32_t* src, uint32_t B, uint64_t bmag,
                                                    uint32_t vmin, uint32_t n, uint64_t i, V* out) {
  const Word w = word_of(T, B, i);
  const uint32_t s = src[i];
  const uint32_t left = (uint32_t)(n - w.q);
  const bool fin = left <= w.p;
  const uint32_t m = fin ? left : w.p;
  uint32_t t = s, r = 0;
  if (!fin) {
    t = fdiv(s, w.mag);
    r = s - t * w.R;
  }
  (void)r;
  for (int k = (int)m - 1; k >= 0; --k) {  // polynomial division
    const uint32_t qq = (uint32_t)__umul64hi(bmag, (uint64_t)t);
    out[w.q + k] = (V)(vmin + (t - qq * B));
    t = qq;
  }
  uint32_t err = t >= w.Rp_prev ? POLY_ST_RESIDUE : 0u;  // the carry r'_{i-1} < R'_{i-1}
  if (i > 0) {
    const Word wp = word_of(T, B, i - 1);
    const uint32_t sp = src[i - 1];
    const uint32_t rprev = sp - fdiv(sp, wp.mag) * wp.R;
    const uint64_t sv = (uint64_t)t * wp.R + rprev;
    if (sv >= B) err = POLY_ST_RESIDUE;
    out[wp.q + wp.p] = (V)(vmin + (uint32_t)sv);
  }
  return err;
}

template <typename V>
__global__ void __launch_bounds__(NTA) adv_unpack(Args a) {
  const uint4* hdr = reinterpret_cast<const uint4*>(a.in + 32);
  const uint32_t* pay = reinterpret_cast<const uint32_t*>(a.in + 32 + 16 * a.n_blocks);
  const uint64_t pw = (a.in_bytes - (32 + 16 * a.n_blocks)) / 4;
  V* outv = reinterpret_cast<V*>(a.out);
  const int lane = threadIdx.x & 31;
  uint32_t err = 0;
  const uint64_t step = a.warp_per_block ? (uint64_t)gridDim.x * (NTA / 32) : (uint64_t)gridDim.x * NTA;
  const uint64_t first = a.warp_per_block ? blockIdx.x * (uint64_t)(NTA / 32) + (threadIdx.x >> 5)
                                          : blockIdx.x * (uint64_t)NTA + threadIdx.x;
  if (adv_header_err(a)) return;  // reported by adv_check_header
  for (uint64_t b = first; b < a.n_blocks; b += step) {
    const uint4 h = hdr[b];
    const uint32_t n = blen_of(a, b);
    const uint32_t e = check_adv_block(a.T, h, n);
    V* o = outv + b * a.Le;
    if (e || a.woff[b] + h.w > pw) {
      if (!a.warp_per_block || lane == 0) err |= e ? e : POLY_ST_LENGTH;
      continue;
    }
    if (h.x == CODEC_CONSTANT) {
      if (a.warp_per_block)
        for (uint32_t i = lane; i < n; i += 32) o[i] = (V)h.y;
      else
        for (uint32_t i = 0; i < n; ++i) o[i] = (V)h.y;
      continue;
    }
    const uint32_t B = h.z + 1;
    const uint64_t bmag = ~0ull / B + 1;  // ceil(2^64 / B), B >= 2
    const uint32_t* src = pay + a.woff[b];
    if (a.warp_per_block) {
      for (uint32_t i = lane; i < h.w; i += 32) err |= unpack_word_adv<V>(a.T, src, B, bmag, h.y, n, i, o);
    } else {
      for (uint32_t i = 0; i < h.w; ++i) err |= unpack_word_adv<V>(a.T, src, B, bmag, h.y, n, i, o);
    }
  }
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0 && err) atomicOr(a.status_out, err);
}

}  // namespace adv
}  // namespace polyk

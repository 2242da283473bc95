// poly_compress.cuh -- compress kernels.
//
// Large-block regime (block_len * w > WT_MAX, e.g. cfg1 / cfg3): chunked
// min/max with atomics (a2), a look-back scan over blocks for B, k, n_words,
// headers and payload offsets (a3, a4, a6), then a chunked Horner pack pass
// (a5).  Used for blocks the pipeline kernels do not take (few blocks larger
// than 32 KiB, e.g. cfg1's single block); see poly.cu plan().
#pragma once
#include "poly_common.cuh"
#include "poly_word.cuh"

namespace polyk {

struct CompressArgs {
  const void* in;
  uint8_t* out;
  uint64_t* compressed_bytes;
  uint64_t* status;   // n_stiles look-back words
  uint32_t* ticket;
  uint32_t* bmin;     // large regime: per-block running min
  uint32_t* bmax;     // large regime: per-block running max
  uint64_t* woff;     // large regime: per-block payload word offset
  Shape sh;
};

// Horner evaluation of Eq. 2 for one word: s = sum_{i<m} (v[i] - vmin) B^i,
// evaluated from the last digit down.
template <typename V>
__device__ __forceinline__ uint64_t horner_word(const V* v, uint32_t m, uint64_t B, uint32_t vmin) {
  uint64_t s = 0;
  for (int i = (int)m - 1; i >= 0; --i) s = s * B + (uint64_t)((uint32_t)v[i] - vmin);
  return s;
}

// ------------------------------------------------------------ large regime
// Chunk c of block b covers values [c*CH, min((c+1)*CH, n_b)) of the block.
__device__ __forceinline__ void chunk_of(const Shape& sh, uint64_t id, uint64_t& b, uint64_t& c,
                                         uint64_t& lo, uint64_t& nb) {
  b = id / sh.cpb;
  c = id % sh.cpb;
  lo = b * sh.Le;
  nb = min(sh.Le, sh.n - lo);
}

template <typename V>
__global__ void __launch_bounds__(NT) poly_compress_minmax(CompressArgs a) {
  __shared__ uint32_t s_mn[NWARP], s_mx[NWARP];
  const Shape& sh = a.sh;
  const V* in = reinterpret_cast<const V*>(a.in);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint64_t id = blockIdx.x; id < sh.n_chunks; id += gridDim.x) {
    uint64_t b, c, lo, nb;
    chunk_of(sh, id, b, c, lo, nb);
    const uint64_t c0 = c * CH_VALUES;
    if (c0 >= nb) continue;  // uniform across the CTA
    const uint32_t cnt = (uint32_t)min((uint64_t)CH_VALUES, nb - c0);
    uint32_t mn = 0xffffffffu, mx = 0u;
    for (uint32_t i = tid; i < cnt; i += NT) {
      const uint32_t v = (uint32_t)in[lo + c0 + i];
      mn = min(mn, v);
      mx = max(mx, v);
    }
    mn = shfl_min(mn, 32);
    mx = shfl_max(mx, 32);
    if (lane == 0) { s_mn[warp] = mn; s_mx[warp] = mx; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < NWARP; ++w) { mn = min(mn, s_mn[w]); mx = max(mx, s_mx[w]); }
      atomicMin(a.bmin + b, mn);
      atomicMax(a.bmax + b, mx);
    }
    __syncthreads();
  }
}

// One CTA per NT*4 blocks: B, k, n_words, headers, look-back scan of n_words
// into woff[]; the last scan tile writes the global header.
constexpr uint32_t SCAN_T = NT * 4;

__global__ void __launch_bounds__(NT) poly_compress_block_scan(CompressArgs a) {
  __shared__ uint64_t s_nw[SCAN_T], s_off[SCAN_T];
  __shared__ uint64_t s_warp[NWARP];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_prefix;
  const Shape& sh = a.sh;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t b0 = tile * SCAN_T;
  const uint32_t nblk = (uint32_t)min((uint64_t)SCAN_T, sh.n_blocks - b0);
  uint4* hdr = reinterpret_cast<uint4*>(a.out + 32);
  for (uint32_t i = tid; i < nblk; i += NT) {
    const uint64_t b = b0 + i;
    const uint64_t nb = min(sh.Le, sh.n - b * sh.Le);
    const uint32_t vmin = a.bmin[b];
    const uint64_t B = (uint64_t)a.bmax[b] - vmin + 1;
    const uint32_t nw = B == 1 ? 0u : (uint32_t)((nb + capacity_of(B) - 1) / capacity_of(B));
    s_nw[i] = nw;
    hdr[b] = make_uint4(B == 1 ? CODEC_CONSTANT : CODEC_BASIC, vmin, (uint32_t)(B - 1), nw);
  }
  __syncthreads();
  const uint64_t total = cta_exclusive_scan<uint64_t>(s_nw, s_off, nblk, s_warp);
  if (tid < 32) {
    uint64_t p = 0;
    if (tid == 0) st_relaxed_u64(a.status + tile, (tile == 0 ? FLAG_PRE : FLAG_AGG) | total);
    if (tile != 0) {
      p = lookback(a.status, tile);
      if (tid == 0) st_relaxed_u64(a.status + tile, FLAG_PRE | (p + total));
    }
    if (tid == 0) s_prefix = p;
  }
  __syncthreads();
  const uint64_t P = s_prefix;
  for (uint32_t i = tid; i < nblk; i += NT) a.woff[b0 + i] = P + s_off[i];
  if (tile == sh.n_stiles - 1 && tid == 0) {
    write_global_header_f(a.out, sh.width, sh.n, sh.block_len, sh.n_blocks, P + total);
    *a.compressed_bytes = 32 + 16 * sh.n_blocks + 8 * (P + total);
  }
}

// Pack pass: chunk c of block b packs the words whose first value lies in
// [c*CH, (c+1)*CH); their values are staged in smem (CH + 64 values).
template <typename V>
__global__ void __launch_bounds__(NT) poly_compress_pack(CompressArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  V* s_in = reinterpret_cast<V*>(smem);
  const Shape& sh = a.sh;
  const V* in = reinterpret_cast<const V*>(a.in);
  uint64_t* pay = reinterpret_cast<uint64_t*>(a.out + 32 + 16 * sh.n_blocks);
  const int tid = threadIdx.x;
  for (uint64_t id = blockIdx.x; id < sh.n_chunks; id += gridDim.x) {
    uint64_t b, c, lo, nb;
    chunk_of(sh, id, b, c, lo, nb);
    const uint32_t vmin = a.bmin[b];
    const uint64_t B = (uint64_t)a.bmax[b] - vmin + 1;
    if (B == 1 || c * CH_VALUES >= nb) continue;  // uniform across the CTA
    const uint32_t k = capacity_of(B);
    const uint64_t nw = (nb + k - 1) / k;
    const uint64_t j0 = (c * CH_VALUES + k - 1) / k;
    const uint64_t j1 = min(nw, ((c + 1) * CH_VALUES + k - 1) / k);
    if (j0 >= j1) continue;
    const uint64_t f0 = j0 * k, f1 = min(nb, j1 * k);
    __syncthreads();  // s_in reuse across iterations
    load_values<V>(s_in, in + lo + f0, (uint32_t)(f1 - f0));
    __syncthreads();
    uint64_t* dst = pay + a.woff[b];
    for (uint64_t j = j0 + tid; j < j1; j += NT) {
      const uint64_t first = j * k;
      dst[j] = horner_word<V>(s_in + (first - f0), (uint32_t)min((uint64_t)k, nb - first), B, vmin);
    }
  }
}

// ------------------------------------------------------------ single launch
// A few huge blocks in ONE cooperative launch (cfg1): chunk min/max partials,
// one grid barrier, then every CTA reduces the partials of all blocks, scans
// the word counts in shared memory and packs its chunks; CTA 0 writes the
// headers.  n_blocks <= LARGE1_MAX_BLOCKS, n_chunks <= LARGE1_MAX_CHUNKS and
// every CTA resident (cooperative launch; the barrier would hang otherwise).
constexpr uint32_t LARGE1C_MAX_BLOCKS = 256;
constexpr uint32_t LARGE1C_MAX_CHUNKS = 2048;

__device__ __forceinline__ void grid_barrier(uint32_t* count, uint32_t nctas) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(count, 1u);
    uint32_t ns = 32, v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
      if (v >= nctas) break;
      __nanosleep(ns);
      ns = min(ns * 2, 256u);
    }
  }
  __syncthreads();
}

template <typename V>
__global__ void __launch_bounds__(NT) poly_compress_large1(CompressArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  V* s_in = reinterpret_cast<V*>(smem);
  __shared__ uint32_t s_mn[NWARP], s_mx[NWARP];
  __shared__ uint32_t s_bmin[LARGE1C_MAX_BLOCKS], s_bmax[LARGE1C_MAX_BLOCKS];
  __shared__ uint64_t s_nw[LARGE1C_MAX_BLOCKS], s_off[LARGE1C_MAX_BLOCKS], s_warp[NWARP];
  const Shape& sh = a.sh;
  const V* in = reinterpret_cast<const V*>(a.in);
  uint32_t* pmin = a.bmin;  // per-chunk partials (workspace)
  uint32_t* pmax = a.bmax;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // a CTA with a single chunk keeps its values in shared memory for the pack
  const bool one = gridDim.x >= sh.n_chunks;
  // ---- a2: chunk min / max (the chunk is staged: 16-byte loads when aligned)
  for (uint64_t id = blockIdx.x; id < sh.n_chunks; id += gridDim.x) {
    uint64_t b, c, lo, nb;
    chunk_of(sh, id, b, c, lo, nb);
    const uint64_t c0 = c * CH_VALUES;
    uint32_t mn = 0xffffffffu, mx = 0u;
    if (c0 < nb) {
      const uint32_t cnt = (uint32_t)min((uint64_t)CH_VALUES, nb - c0);
      __syncthreads();  // s_in reuse
      load_values<V>(s_in, in + lo + c0, cnt);
      __syncthreads();
      for (uint32_t i = tid; i < cnt; i += NT) {
        const uint32_t v = (uint32_t)s_in[i];
        mn = min(mn, v);
        mx = max(mx, v);
      }
    }
    mn = shfl_min(mn, 32);
    mx = shfl_max(mx, 32);
    if (lane == 0) {
      s_mn[warp] = mn;
      s_mx[warp] = mx;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < NWARP; ++w) {
        mn = min(mn, s_mn[w]);
        mx = max(mx, s_mx[w]);
      }
      pmin[id] = mn;
      pmax[id] = mx;
    }
  }
  grid_barrier(a.ticket, gridDim.x);
  // ---- a3, a4: every CTA: block bases, k, n_words, offsets
  const uint32_t nblk = (uint32_t)sh.n_blocks;
  for (uint32_t b = tid; b < nblk; b += NT) {
    s_bmin[b] = 0xffffffffu;
    s_bmax[b] = 0u;
  }
  __syncthreads();
  for (uint64_t id = tid; id < sh.n_chunks; id += NT) {  // the partials, all threads
    const uint32_t b = (uint32_t)(id / sh.cpb);
    atomicMin(&s_bmin[b], __ldcg(pmin + id));
    atomicMax(&s_bmax[b], __ldcg(pmax + id));
  }
  __syncthreads();
  for (uint32_t b = tid; b < nblk; b += NT) {
    const uint32_t mn = s_bmin[b], mx = s_bmax[b];
    const uint64_t nb = min(sh.Le, sh.n - (uint64_t)b * sh.Le);
    const uint64_t B = (uint64_t)mx - mn + 1;
    const uint32_t nw = B == 1 ? 0u : (uint32_t)((nb + capacity_of(B) - 1) / capacity_of(B));
    s_nw[b] = nw;
    if (blockIdx.x == 0)
      reinterpret_cast<uint4*>(a.out + 32)[b] = make_uint4(B == 1 ? CODEC_CONSTANT : CODEC_BASIC, mn, mx - mn, nw);
  }
  __syncthreads();
  const uint64_t total = cta_exclusive_scan<uint64_t>(s_nw, s_off, nblk, s_warp);
  if (blockIdx.x == 0 && tid == 0) {
    write_global_header_f(a.out, sh.width, sh.n, sh.block_len, sh.n_blocks, total);
    *a.compressed_bytes = 32 + 16 * sh.n_blocks + 8 * total;
  }
  // ---- a5, a6: pack the words whose first value lies in the chunk
  uint64_t* pay = reinterpret_cast<uint64_t*>(a.out + 32 + 16 * sh.n_blocks);
  for (uint64_t id = blockIdx.x; id < sh.n_chunks; id += gridDim.x) {
    uint64_t b, c, lo, nb;
    chunk_of(sh, id, b, c, lo, nb);
    const uint32_t vmin = s_bmin[b];
    const uint64_t B = (uint64_t)s_bmax[b] - vmin + 1;
    if (B == 1 || c * CH_VALUES >= nb) continue;  // uniform across the CTA
    const uint32_t k = capacity_of(B);
    const uint64_t nw = (nb + k - 1) / k;
    const uint64_t j0 = (c * CH_VALUES + k - 1) / k;
    const uint64_t j1 = min(nw, ((c + 1) * CH_VALUES + k - 1) / k);
    if (j0 >= j1) continue;
    const uint64_t f0 = j0 * k, f1 = min(nb, j1 * k);
    // staged chunk values start at c0 = c * CH; the words need [f0, f1) with
    // f0 >= c0 and f1 <= c0 + CH + k - 1: the tail past the chunk comes from HBM
    const uint64_t c0 = c * CH_VALUES;
    const V* src;
    if (one) {
      const uint32_t have = (uint32_t)min((uint64_t)CH_VALUES, nb - c0);
      __syncthreads();
      for (uint64_t i = c0 + have + tid; i < f1; i += NT) s_in[i - c0] = in[lo + i];
      __syncthreads();
      src = s_in + (f0 - c0);
    } else {
      __syncthreads();  // s_in reuse across iterations
      load_values<V>(s_in, in + lo + f0, (uint32_t)(f1 - f0));
      __syncthreads();
      src = s_in;
    }
    uint64_t* dst = pay + s_off[b];
    for (uint64_t j = j0 + tid; j < j1; j += NT) {
      const uint64_t first = j * k;
      dst[j] = horner_word<V>(src + (first - f0), (uint32_t)min((uint64_t)k, nb - first), B, vmin);
    }
  }
}

}  // namespace polyk

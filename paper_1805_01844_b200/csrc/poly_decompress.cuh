// poly_decompress.cuh -- decompress kernels.
//
// Digit extraction (a8) uses no integer divide: for a non-power-of-two base B
// with capacity k, a word s < B^k is turned into the 64-bit binary fraction
// f = floor(s * R / 2^96) + 1, R = ceil(2^160 / B^k), which satisfies
// s*2^64/B^k <= f < (s+1)*2^64/B^k.  Multiplying the
// fraction by B then yields the base-B digits of s from the most significant
// one down: digit = floor(f*B / 2^64), f = f*B mod 2^64 -- two 32x32->64
// multiply-adds per digit.  Power-of-two bases use shifts and masks.
#pragma once
#include "poly_common.cuh"
#include "poly_word.cuh"

namespace polyk {

struct DecompressArgs {
  const uint8_t* in;
  uint64_t compressed_bytes;
  void* out;
  uint32_t* status_out;  // caller's device status word
  uint64_t* status;      // look-back words
  uint32_t* ticket;
  uint64_t* woff;        // large regime: per-block payload word offset
  Shape sh;
};

// Global header check; returns POLY_ST_* bits (0 = header consistent).
__device__ __forceinline__ uint32_t check_global_header(const DecompressArgs& a,
                                                        uint64_t* payload_words) {
  const Shape& sh = a.sh;
  if (a.compressed_bytes < 32) return POLY_ST_LENGTH;
  const uint4 h0 = reinterpret_cast<const uint4*>(a.in)[0];
  const uint4 h1 = reinterpret_cast<const uint4*>(a.in)[1];
  if (h0.x != 0x43594c50u) return POLY_ST_BAD_MAGIC;
  if ((h0.y & 0xffu) != 2u) return POLY_ST_BAD_VERSION;
  const uint64_t n = (uint64_t)h0.z | ((uint64_t)h0.w << 32);
  const uint64_t pb = (uint64_t)h1.z | ((uint64_t)h1.w << 32);
  if (((h0.y >> 8) & 0xffu) != 0u || ((h0.y >> 16) & 0xffu) != sh.width || (h0.y >> 24) != 0u ||
      n != sh.n || h1.x != sh.block_len || h1.y != (uint32_t)sh.n_blocks)
    return POLY_ST_HEADER_MISMATCH;
  // overflow-safe: in_bytes must hold the headers before pb is compared with the rest
  if ((pb & 7) != 0 || a.compressed_bytes < 32 + 16 * sh.n_blocks || pb != a.compressed_bytes - (32 + 16 * sh.n_blocks))
    return POLY_ST_LENGTH;
  *payload_words = pb >> 3;
  return 0;
}

// Validate one block header; returns POLY_ST_* bits.
__device__ __forceinline__ uint32_t check_block(uint4 h, uint64_t nb, uint32_t width, uint32_t k) {
  const uint64_t vmax_allowed = (width == 32) ? 0xffffffffull : ((1ull << width) - 1);
  if (h.x == CODEC_CONSTANT) {
    uint32_t e = 0;
    if (h.z != 0 || h.w != 0) e |= POLY_ST_NWORDS;
    if ((uint64_t)h.y > vmax_allowed) e |= POLY_ST_OVERFLOW;
    return e;
  }
  if (h.x != CODEC_BASIC) return POLY_ST_BAD_CODEC;
  if (h.z == 0 || (uint64_t)h.y + h.z > vmax_allowed) return POLY_ST_OVERFLOW;
  if ((uint64_t)h.w != (nb + k - 1) / k) return POLY_ST_NWORDS;
  return 0;
}

// ------------------------------------------------------------ large regime
constexpr uint32_t DSCAN_T = NT * 4;

__global__ void __launch_bounds__(NT) poly_decompress_block_scan(DecompressArgs a) {
  __shared__ uint64_t s_nw[DSCAN_T], s_off[DSCAN_T];
  __shared__ uint64_t s_warp[NWARP];
  __shared__ uint32_t s_tile, s_err, s_hdr_err;
  __shared__ uint64_t s_prefix, s_pw;
  const Shape& sh = a.sh;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_tile = atomicAdd(a.ticket, 1u);
    s_err = 0;
    uint64_t pw = 0;
    s_hdr_err = check_global_header(a, &pw);
    s_pw = pw;
  }
  __syncthreads();
  const uint64_t tile = s_tile;
  if (s_hdr_err) {
    if (tile == 0 && tid == 0) atomicOr(a.status_out, s_hdr_err);
    return;
  }
  const uint64_t b0 = tile * DSCAN_T;
  const uint32_t nblk = (uint32_t)min((uint64_t)DSCAN_T, sh.n_blocks - b0);
  const uint4* hdr = reinterpret_cast<const uint4*>(a.in + 32);
  uint32_t err = 0;
  for (uint32_t i = tid; i < nblk; i += NT) {
    const uint64_t b = b0 + i;
    const uint4 h = hdr[b];
    const uint64_t nb = min(sh.Le, sh.n - b * sh.Le);
    const uint32_t k = (h.x == CODEC_BASIC && h.z != 0) ? capacity_of((uint64_t)h.z + 1) : 1u;
    err |= check_block(h, nb, sh.width, k);
    s_nw[i] = h.w;
  }
  if (err) atomicOr(&s_err, err);
  __syncthreads();
  const uint64_t total = cta_exclusive_scan<uint64_t>(s_nw, s_off, nblk, s_warp);
  if (tid < 32) {
    uint64_t p = 0;
    if (tid == 0) st_relaxed_u64(a.status + tile, (tile == 0 ? FLAG_PRE : FLAG_AGG) | (total & VAL_MASK));
    if (tile != 0) {
      p = lookback(a.status, tile);
      if (tid == 0) st_relaxed_u64(a.status + tile, FLAG_PRE | ((p + total) & VAL_MASK));
    }
    if (tid == 0) {
      s_prefix = p;
      if (tile == sh.n_stiles - 1 && p + total != s_pw) atomicOr(&s_err, POLY_ST_LENGTH);
    }
  }
  __syncthreads();
  for (uint32_t i = tid; i < nblk; i += NT) a.woff[b0 + i] = s_prefix + s_off[i];
  if (tid == 0 && s_err) atomicOr(a.status_out, s_err);
}

// Chunk c of block b decodes the words whose first value lies in
// [c*CH, (c+1)*CH) (CONSTANT blocks: the values [c*CH, (c+1)*CH)).
template <typename V>
__global__ void __launch_bounds__(NT) poly_decompress_unpack(DecompressArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  V* s_out = reinterpret_cast<V*>(smem);
  uint64_t* s_words = reinterpret_cast<uint64_t*>(smem + 16 * ((CH_VALUES + 64) * sizeof(V) / 16 + 1));
  __shared__ DecConst s_c;
  __shared__ uint32_t s_err, s_bad;
  __shared__ uint64_t s_pw;
  const Shape& sh = a.sh;
  const int tid = threadIdx.x;
  if (tid == 0) {
    uint64_t pw = 0;
    s_bad = check_global_header(a, &pw);
    s_pw = pw;
    s_err = 0;
  }
  __syncthreads();
  if (s_bad) return;  // reported by the scan kernel
  const uint64_t payload_words = s_pw;
  const uint4* hdr = reinterpret_cast<const uint4*>(a.in + 32);
  const uint64_t* pay = reinterpret_cast<const uint64_t*>(a.in + 32 + 16 * sh.n_blocks);
  V* out = reinterpret_cast<V*>(a.out);
  uint32_t err = 0;
  for (uint64_t id = blockIdx.x; id < sh.n_chunks; id += gridDim.x) {
    const uint64_t b = id / sh.cpb, c = id % sh.cpb;
    const uint64_t lo = b * sh.Le, nb = min(sh.Le, sh.n - lo);
    if (c * CH_VALUES >= nb) continue;
    const uint4 h = hdr[b];
    if (h.x == CODEC_CONSTANT) {
      if (h.z != 0 || h.w != 0) continue;
      const uint64_t f1 = min(nb, (c + 1) * CH_VALUES);
      for (uint64_t i = c * CH_VALUES + tid; i < f1; i += NT) out[lo + i] = (V)h.y;
      continue;
    }
    if (h.x != CODEC_BASIC || h.z == 0) continue;
    const uint64_t B = (uint64_t)h.z + 1;
    __syncthreads();
    if (tid == 0) s_c = dec_const_of(B);
    __syncthreads();
    const DecConst cst = s_c;
    const uint32_t k = dc_k(cst);
    if (check_block(h, nb, sh.width, k)) continue;
    const uint64_t nw = h.w;
    const uint64_t j0 = (c * CH_VALUES + k - 1) / k;
    const uint64_t j1 = min(nw, ((c + 1) * CH_VALUES + k - 1) / k);
    if (j0 >= j1) continue;
    const uint64_t w0 = a.woff[b] + j0;
    const uint32_t cnt = (uint32_t)(j1 - j0);
    if (w0 + cnt > payload_words) continue;  // flagged as LENGTH by the scan
    for (uint32_t i = tid; i < cnt; i += NT) s_words[i] = ldg_nc_u64(pay + w0 + i);
    __syncthreads();
    const uint64_t f0 = j0 * k;
    for (uint32_t i = tid; i < cnt; i += NT) {
      const uint64_t first = (j0 + i) * k;
      err |= decode_any<V>(s_words[i], cst, h.z, (uint32_t)min((uint64_t)k, nb - first), h.y,
                           s_out + (first - f0));
    }
    __syncthreads();
    store_values<V>(out + lo + f0, s_out, (uint32_t)(min(nb, j1 * k) - f0));
  }
  if (err) atomicOr(&s_err, err);
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(a.status_out, s_err);
}

// ------------------------------------------------------------ single launch
// A few huge blocks in ONE launch (cfg1: one block of the whole array): every
// CTA validates the headers and scans the blocks' n_words into its own
// shared-memory offsets (n_blocks <= LARGE1_MAX_BLOCKS), then decodes its
// chunks as poly_decompress_unpack does -- no offset kernel, no workspace.
constexpr uint32_t LARGE1_MAX_BLOCKS = 256;
constexpr uint32_t LARGE1_MAX_CHUNKS = 2048;

template <typename V>
__global__ void __launch_bounds__(NT) poly_decompress_large1(DecompressArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  V* s_out = reinterpret_cast<V*>(smem);
  uint64_t* s_words = reinterpret_cast<uint64_t*>(smem + 16 * ((CH_VALUES + 64) * sizeof(V) / 16 + 1));
  __shared__ uint64_t s_nw[LARGE1_MAX_BLOCKS], s_off[LARGE1_MAX_BLOCKS], s_warp[NWARP];
  __shared__ DecConst s_c;
  __shared__ uint32_t s_err, s_bad;
  __shared__ uint64_t s_pw;
  const Shape& sh = a.sh;
  const int tid = threadIdx.x;
  if (tid == 0) {
    uint64_t pw = 0;
    s_bad = check_global_header(a, &pw);
    s_pw = pw;
    s_err = 0;
  }
  __syncthreads();
  if (s_bad) {
    if (blockIdx.x == 0 && tid == 0) atomicOr(a.status_out, s_bad);
    return;
  }
  const uint64_t payload_words = s_pw;
  const uint4* hdr = reinterpret_cast<const uint4*>(a.in + 32);
  const uint64_t* pay = reinterpret_cast<const uint64_t*>(a.in + 32 + 16 * sh.n_blocks);
  const uint32_t nblk = (uint32_t)sh.n_blocks;
  uint32_t err = 0;
  for (uint32_t b = tid; b < nblk; b += NT) {
    const uint4 h = hdr[b];
    const uint64_t nb = min(sh.Le, sh.n - (uint64_t)b * sh.Le);
    const uint32_t k = (h.x == CODEC_BASIC && h.z != 0) ? capacity_of((uint64_t)h.z + 1) : 1u;
    err |= check_block(h, nb, sh.width, k);
    s_nw[b] = h.w;
  }
  __syncthreads();
  const uint64_t total = cta_exclusive_scan<uint64_t>(s_nw, s_off, nblk, s_warp);
  if (blockIdx.x == 0 && tid == 0 && total != payload_words) err |= POLY_ST_LENGTH;
  if (blockIdx.x != 0) err = 0;  // header verdicts reported once
  V* out = reinterpret_cast<V*>(a.out);
  for (uint64_t id = blockIdx.x; id < sh.n_chunks; id += gridDim.x) {
    const uint64_t b = id / sh.cpb, c = id % sh.cpb;
    const uint64_t lo = b * sh.Le, nb = min(sh.Le, sh.n - lo);
    if (c * CH_VALUES >= nb) continue;
    const uint4 h = hdr[b];
    if (h.x == CODEC_CONSTANT) {
      if (h.z != 0 || h.w != 0) continue;
      const uint64_t f1 = min(nb, (c + 1) * CH_VALUES);
      for (uint64_t i = c * CH_VALUES + tid; i < f1; i += NT) out[lo + i] = (V)h.y;
      continue;
    }
    if (h.x != CODEC_BASIC || h.z == 0) continue;
    const uint64_t B = (uint64_t)h.z + 1;
    __syncthreads();
    if (tid == 0) s_c = dec_const_of(B);
    __syncthreads();
    const DecConst cst = s_c;
    const uint32_t k = dc_k(cst);
    if (check_block(h, nb, sh.width, k)) continue;
    const uint64_t nw = h.w;
    const uint64_t j0 = (c * CH_VALUES + k - 1) / k;
    const uint64_t j1 = min(nw, ((c + 1) * CH_VALUES + k - 1) / k);
    if (j0 >= j1) continue;
    const uint64_t w0 = s_off[b] + j0;
    const uint32_t cnt = (uint32_t)(j1 - j0);
    if (w0 + cnt > payload_words) continue;  // flagged as LENGTH above
    for (uint32_t i = tid; i < cnt; i += NT) s_words[i] = ldg_nc_u64(pay + w0 + i);
    __syncthreads();
    const uint64_t f0 = j0 * k;
    uint32_t e = 0;
    for (uint32_t i = tid; i < cnt; i += NT) {
      const uint64_t first = (j0 + i) * k;
      e |= decode_any<V>(s_words[i], cst, h.z, (uint32_t)min((uint64_t)k, nb - first), h.y, s_out + (first - f0));
    }
    err |= e;
    __syncthreads();
    store_values<V>(out + lo + f0, s_out, (uint32_t)(min(nb, j1 * k) - f0));
  }
  if (err) atomicOr(&s_err, err);
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(a.status_out, s_err);
}

}  // namespace polyk

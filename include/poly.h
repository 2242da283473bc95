/*
 * poly.h -- C ABI of the B200 (sm_100a) basic blocked polynomial codec.
 *
 * The operation (arXiv 1805.01844, PAPER.md = /root/reference/PAPER.md):
 *   Sec. 3.3: split the vector into blocks of `block_size`
 *   values (0 = one block of the whole vector; the short last block is coded
 *   like any other -- DESIGN.md R10).
 *   Sec. 3.1, per block: v_min, v_max, the base
 *   B = v_max - v_min + 1; the capacity k = max{k : B^k <= 2^64}
 *   (Eq. 1 with a 64-bit word, R1/R2); the words
 *   s_j = sum_{i<m} (v_{jk+i} - v_min) * B^i (Eq. 2, R3-R5); B = 1 is a
 *   CONSTANT block without words (R6).  Decompression is the "polynomial
 *   division" of PAPER.md:147.
 * Stream layout (readings R7-R9):
 *   32-byte global header | n_blocks x 16-byte block headers | u64 payload words.
 *
 * Conventions for every function below:
 *   - Pointers named d_* are DEVICE memory, h_* are HOST memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Device-side calls are asynchronous on `stream`; they never allocate,
 *     free or synchronize, and keep no pointer after they return.  The caller
 *     owns every buffer.
 *   - Arrays of values are u8 (POLY_U8), little-endian u16
 *     (POLY_U16) or u32 (POLY_U32), contiguous, aligned to their element size
 *     only (16-byte alignment is faster).  A compressed stream buffer (the
 *     output of poly_compress, the input of poly_decompress) must be 16-byte
 *     aligned (POLY_ERR_INVALID_ARG otherwise; torch / cudaMalloc buffers are).
 *   - Argument errors are returned synchronously, with nothing launched.
 *     Errors in stream CONTENT are only known on the device and are reported
 *     as POLY_ST_* bits in the caller's device status word.
 *   - The first call on a device uploads the k / reciprocal tables with a
 *     synchronous copy; call poly_init() first if the calls will be captured
 *     into a CUDA graph.
 */
#ifndef POLY_H_
#define POLY_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { POLY_U8 = 8, POLY_U16 = 16, POLY_U32 = 32 } poly_dtype_t;

typedef enum {
  POLY_OK = 0,
  POLY_ERR_INVALID_ARG = 1,  /* null pointer, dtype not 16/32, block_size or n_blocks >= 2^32 */
  POLY_ERR_EMPTY_INPUT = 2,  /* n == 0 (SPEC.md:53 EmptyInput) */
  POLY_ERR_CAPACITY = 3,     /* out_capacity < poly_max_compressed_bytes / output too small */
  POLY_ERR_WORKSPACE = 4,    /* workspace_bytes < poly_workspace_bytes */
  POLY_ERR_CUDA = 5,         /* a CUDA runtime call or launch failed */
  POLY_ERR_CORRUPT = 6       /* host-side header parse failed (poly_read_header) */
} poly_status_t;

/* Device status bits written by poly_decompress (atomicOr into *d_status,
 * which the call first zeroes).  0 after the call = the stream was valid. */
#define POLY_ST_BAD_MAGIC 1u        /* not "PLYC" (SPEC.md:311 NotAContainer) */
#define POLY_ST_BAD_VERSION 2u      /* version != 2 (SPEC.md:311 UnsupportedVersion) */
#define POLY_ST_HEADER_MISMATCH 4u  /* global header != (dtype, n, block_size) or bad layout */
#define POLY_ST_BAD_CODEC 8u        /* block codec not CONSTANT(1) / BASIC(2) */
#define POLY_ST_NWORDS 16u          /* n_words != ceil(n_b / k), or CONSTANT with payload */
#define POLY_ST_RESIDUE 32u         /* word >= B^m: nonzero residue after m digits */
#define POLY_ST_OVERFLOW 64u        /* v_min + B - 1 > 2^w - 1, or B < 2 for BASIC */
#define POLY_ST_LENGTH 128u         /* truncated / length != 32 + 16 n_blocks + payload_bytes */

/* Library version (major*10000 + minor*100 + patch). */
int poly_version(void);

/* Host-only self-check (no device needed): builds the per-base tables with
 * exact 128-bit integers and returns 1 if every precondition of the decoder
 * arithmetic holds (B^k < 2^64 - 2^32 for non-powers of
 * two; the compile-time T32MIN[K] of the k-specialised decoders equals the
 * least t32 over the non-power-of-two bases of capacity K), else 0.
 * poly_init fails with POLY_ERR_CUDA in the second case. */
int poly_tables_ok(void);

/* Human-readable name of a poly_status_t. */
const char* poly_status_string(poly_status_t s);

/* Upload the B -> (k, B^k, reciprocal) tables to `device` (synchronous, once
 * per device; later calls return immediately).  Thread-safe. */
poly_status_t poly_init(int device);

/* Worst-case stream size for n values of dtype `dt` in blocks of block_size:
 * 32 + 16 n_blocks + 8 sum_b ceil(n_b / k_min), k_min = 8 (u8), 4 (u16), 2 (u32)
 * (the smallest k under R2 for B <= 2^8, 2^16 resp. 2^32).  0 if n == 0. */
uint64_t poly_max_compressed_bytes(uint64_t n, poly_dtype_t dt, uint64_t block_size);

/* Device workspace bytes needed by poly_compress / poly_decompress and the
 * host variants for this shape (tile look-back flags, per-block scratch for
 * large blocks).  The content need not be initialised. */
uint64_t poly_workspace_bytes(uint64_t n, poly_dtype_t dt, uint64_t block_size);

/* Compress d_in[0..n) into d_out (the stream of DESIGN.md Sec. 3).
 *   d_in              device array of n u16/u32 values (read only)
 *   block_size        values per block, 0 = whole array (R10); < 2^32
 *   d_out             device buffer of out_capacity bytes; out_capacity must
 *                     be >= poly_max_compressed_bytes(n, dt, block_size)
 *                     because the size is only known on the device
 *   d_compressed_bytes device u64 receiving the stream size in bytes
 *   d_workspace       device scratch of workspace_bytes >=
 *                     poly_workspace_bytes(n, dt, block_size)
 * The stream is bit-identical to the oracle's (oracle/), whatever the launch
 * configuration.  Returns POLY_ERR_EMPTY_INPUT for n == 0. */
poly_status_t poly_compress(const void* d_in, uint64_t n, poly_dtype_t dt, uint64_t block_size,
                            void* d_out, uint64_t out_capacity, uint64_t* d_compressed_bytes,
                            void* d_workspace, uint64_t workspace_bytes, void* stream);

/* Parse a 32-byte global header held in HOST memory.  Any output pointer may
 * be NULL.  Returns POLY_ERR_CORRUPT for bad magic / version / layout. */
poly_status_t poly_read_header(const void* h_hdr32, uint64_t* n, poly_dtype_t* dt,
                               uint64_t* block_size, uint64_t* n_blocks,
                               uint64_t* payload_bytes);

/* Decompress the stream d_in[0..compressed_bytes) into d_out[0..n).
 * (dt, n, block_size) are what the caller expects; the kernels check them
 * against the global header (POLY_ST_HEADER_MISMATCH).  *d_status (device
 * u32) is zeroed, then receives POLY_ST_* bits; on any bit the content of
 * d_out is unspecified, but no read or write leaves the given buffers. */
poly_status_t poly_decompress(const void* d_in, uint64_t compressed_bytes, poly_dtype_t dt,
                              uint64_t n, uint64_t block_size, void* d_out, uint32_t* d_status,
                              void* d_workspace, uint64_t workspace_bytes, void* stream);

/* ADVANCED (split-base) codec of PAPER.md Sec. 3.2, blocked
 * (Sec. 3.3), u16 values only, 32-bit words with the paper's 2^32 - 1 bound
 * (readings A1-A6).  The last digit of a word is split into
 * (r, r') against R and R' (R R' >= B): r in this word, r' at the top of the
 * next, so no word has unused space.  Stream: as above but with layout byte 1,
 * block codec 3 (ADVANCED) or 1 (CONSTANT), and 32-bit payload words.  The
 * first call on a device builds and uploads the per-base schedule table
 * (~15 MB, synchronous).  Same conventions and status bits as poly_compress /
 * poly_decompress; POLY_ERR_INVALID_ARG for dt != POLY_U16.
 *   poly_max_compressed_bytes_advanced = 32 + 16 n_blocks + 4 (n + n_blocks). */
uint64_t poly_max_compressed_bytes_advanced(uint64_t n, poly_dtype_t dt, uint64_t block_size);
uint64_t poly_workspace_bytes_advanced(uint64_t n, poly_dtype_t dt, uint64_t block_size);
poly_status_t poly_compress_advanced(const void* d_in, uint64_t n, poly_dtype_t dt, uint64_t block_size,
                                     void* d_out, uint64_t out_capacity, uint64_t* d_compressed_bytes,
                                     void* d_workspace, uint64_t workspace_bytes, void* stream);
poly_status_t poly_decompress_advanced(const void* d_in, uint64_t compressed_bytes, poly_dtype_t dt,
                                       uint64_t n, uint64_t block_size, void* d_out, uint32_t* d_status,
                                       void* d_workspace, uint64_t workspace_bytes, void* stream);

/* End-to-end variants over HOST buffers (the path a user with data in host
 * RAM takes).  They copy h_in to the caller's device scratch, run the same
 * kernels, copy the result back, and SYNCHRONIZE `stream` before returning.
 * Host buffers should be pinned (cudaHostAlloc / torch pin_memory) for full
 * PCIe bandwidth; pageable memory works but is slower.
 *   poly_compress_host: d_in_scratch >= n*w/8 bytes, d_out_scratch >=
 *     poly_max_compressed_bytes; h_out receives *h_compressed_bytes bytes
 *     (POLY_ERR_CAPACITY if h_out_capacity is smaller).
 *   poly_decompress_host: d_in_scratch >= compressed_bytes, d_out_scratch >=
 *     n*w/8; h_out receives n values; *h_status receives the POLY_ST_* bits. */
poly_status_t poly_compress_host(const void* h_in, uint64_t n, poly_dtype_t dt, uint64_t block_size,
                                 void* h_out, uint64_t h_out_capacity, uint64_t* h_compressed_bytes,
                                 void* d_in_scratch, void* d_out_scratch, uint64_t d_out_capacity,
                                 void* d_workspace, uint64_t workspace_bytes, void* stream);

poly_status_t poly_decompress_host(const void* h_in, uint64_t compressed_bytes, poly_dtype_t dt,
                                   uint64_t n, uint64_t block_size, void* h_out, uint32_t* h_status,
                                   void* d_in_scratch, void* d_out_scratch,
                                   void* d_workspace, uint64_t workspace_bytes, void* stream);

/* Number of kernel launches one poly_compress / poly_decompress call makes for
 * this shape (memsets not counted). */
int poly_launches_per_call(uint64_t n, poly_dtype_t dt, uint64_t block_size, int decompress);

#ifdef __cplusplus
}
#endif

#endif /* POLY_H_ */

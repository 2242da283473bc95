/*
 * oracle.c -- plain C oracle for the basic blocked polynomial codec.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs load this library.  It shares
 * no code, header, table or constant with the CUDA path; it includes nothing
 * from include/ or paper_1805_01844_b200/.
 *
 * It is the same definition as oracle/ref.py, written with machine integers so
 * that the large BASELINE configurations finish in seconds:
 *   - per block (Sec. 3.3): v_min, v_max by a plain loop,
 *     B = v_max - v_min + 1;
 *   - k = largest k with B^k <= 2^64 by the exact loop in unsigned __int128
 *     (Eq. 1, reading R2 of DESIGN.md);
 *   - word s_j = sum_i d_{i + k(j-1)} * B^{i-1}, d = v - v_min, by the literal
 *     sum with an unsigned __int128 power (Eq. 2, R3-R5);
 *   - decode by repeated "% B" and "/ B" with the hardware divide
 *     ("A polynomial division can be used to uncompress").
 * Stream layout: reading R8/R9 (32-byte global header, all 16-byte block
 * headers, then all u64 payload words, little-endian).
 *
 * The only parallelism is threads over whole block ranges (blocks are
 * independent): pass 1 sizes, serial exclusive scan, pass 2 pack.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* status bits; the oracle defines its own copy */
#define OST_BAD_MAGIC 1u
#define OST_BAD_VERSION 2u
#define OST_HEADER_MISMATCH 4u
#define OST_BAD_CODEC 8u
#define OST_NWORDS 16u
#define OST_RESIDUE 32u
#define OST_OVERFLOW 64u
#define OST_LENGTH 128u

/* Eq. 1 under reading R2: largest k with B^k <= 2^64, exact loop. */
int oracle_capacity(uint64_t B) {
    if (B < 2) return 0;
    u128 limit = ((u128)1) << 64;
    u128 p = 1;
    int k = 0;
    while (p * (u128)B <= limit) {
        p = p * (u128)B;
        k = k + 1;
    }
    return k;
}

static uint64_t get_value(const void* in, int width_bits, uint64_t i) {
    if (width_bits == 8) return ((const uint8_t*)in)[i];
    if (width_bits == 16) return ((const uint16_t*)in)[i];
    return ((const uint32_t*)in)[i];
}

static void put_value(void* out, int width_bits, uint64_t i, uint64_t v) {
    if (width_bits == 8) ((uint8_t*)out)[i] = (uint8_t)v;
    else if (width_bits == 16) ((uint16_t*)out)[i] = (uint16_t)v;
    else ((uint32_t*)out)[i] = (uint32_t)v;
}

static void put_u32(uint8_t* p, uint32_t v) {
    for (int i = 0; i < 4; i++) p[i] = (uint8_t)(v >> (8 * i));
}
static void put_u64(uint8_t* p, uint64_t v) {
    for (int i = 0; i < 8; i++) p[i] = (uint8_t)(v >> (8 * i));
}
static uint32_t get_u32(const uint8_t* p) {
    uint32_t v = 0;
    for (int i = 0; i < 4; i++) v |= ((uint32_t)p[i]) << (8 * i);
    return v;
}
static uint64_t get_u64(const uint8_t* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; i++) v |= ((uint64_t)p[i]) << (8 * i);
    return v;
}

uint64_t oracle_max_compressed_bytes(uint64_t n, int width_bits, uint64_t block_len) {
    if (n == 0) return 32;
    uint64_t L = block_len == 0 ? n : block_len;
    uint64_t nb = (n + L - 1) / L;
    /* smallest k: u16 -> 4 (B <= 2^16), u32 -> 2 (B <= 2^32) */
    /* smallest k: u8 -> 8 (B <= 2^8), u16 -> 4 (B <= 2^16), u32 -> 2 (B <= 2^32) */
    uint64_t kmin = width_bits == 8 ? 8 : (width_bits == 16 ? 4 : 2);
    uint64_t words = 0;
    uint64_t full = n / L, last = n - full * L;
    words += full * ((L + kmin - 1) / kmin);
    if (last) words += (last + kmin - 1) / kmin;
    return 32 + 16 * nb + 8 * words;
}

/* ------------------------------------------------------------------ compress */
typedef struct {
    const void* in;
    int width_bits;
    uint64_t n, L, b0, b1;
    uint8_t* out;          /* stream */
    uint64_t n_blocks;
    uint32_t* n_words;     /* per block */
    uint64_t* word_off;    /* per block, exclusive scan */
    int pass;
} cjob_t;

static void* compress_worker(void* arg) {
    cjob_t* J = (cjob_t*)arg;
    for (uint64_t b = J->b0; b < J->b1; b++) {
        uint64_t lo = b * J->L;
        uint64_t hi = lo + J->L < J->n ? lo + J->L : J->n;
        uint64_t nb = hi - lo;
        /* Sec. 3.1: v_min, v_max, B */
        uint64_t vmin = get_value(J->in, J->width_bits, lo), vmax = vmin;
        for (uint64_t i = lo; i < hi; i++) {
            uint64_t v = get_value(J->in, J->width_bits, i);
            if (v < vmin) vmin = v;
            if (v > vmax) vmax = v;
        }
        uint64_t B = vmax - vmin + 1;
        uint8_t* hdr = J->out + 32 + 16 * b;
        if (J->pass == 1) {
            if (B == 1) {
                J->n_words[b] = 0;
                put_u32(hdr + 0, 1); /* CONSTANT */
                put_u32(hdr + 4, (uint32_t)vmin);
                put_u32(hdr + 8, 0);
                put_u32(hdr + 12, 0);
            } else {
                int k = oracle_capacity(B);
                uint64_t W = (nb + k - 1) / k;
                J->n_words[b] = (uint32_t)W;
                put_u32(hdr + 0, 2); /* BASIC */
                put_u32(hdr + 4, (uint32_t)vmin);
                put_u32(hdr + 8, (uint32_t)(B - 1));
                put_u32(hdr + 12, (uint32_t)W);
            }
            continue;
        }
        if (B == 1) continue;
        int k = oracle_capacity(B);
        uint64_t W = (nb + k - 1) / k;
        uint8_t* pay = J->out + 32 + 16 * J->n_blocks + 8 * J->word_off[b];
        for (uint64_t j = 0; j < W; j++) {
            /* Eq. 2: s_j = sum_{i} d_{i+k(j-1)} B^{i-1} */
            u128 s = 0, p = 1;
            for (int i = 0; i < k; i++) {
                uint64_t idx = lo + j * (uint64_t)k + (uint64_t)i;
                if (idx >= hi) break;
                uint64_t d = get_value(J->in, J->width_bits, idx) - vmin;
                s = s + (u128)d * p;
                p = p * (u128)B;
            }
            if (s >> 64) abort(); /* cannot happen: B^k <= 2^64 */
            put_u64(pay + 8 * j, (uint64_t)s);
        }
    }
    return NULL;
}

static void run_jobs(cjob_t* base, int threads, void* (*fn)(void*)) {
    if (threads < 1) threads = 1;
    uint64_t nb = base->n_blocks;
    if ((uint64_t)threads > nb) threads = (int)(nb ? nb : 1);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    cjob_t* jobs = (cjob_t*)malloc(sizeof(cjob_t) * threads);
    for (int t = 0; t < threads; t++) {
        jobs[t] = *base;
        jobs[t].b0 = nb * (uint64_t)t / (uint64_t)threads;
        jobs[t].b1 = nb * (uint64_t)(t + 1) / (uint64_t)threads;
        if (threads == 1) fn(&jobs[t]);
        else pthread_create(&th[t], NULL, fn, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
}

/* returns 0 on success, 1 empty input, 2 bad argument, 3 capacity, 4 oom */
int oracle_compress(const void* in, uint64_t n, int width_bits, uint64_t block_len,
                    uint8_t* out, uint64_t out_capacity, uint64_t* out_bytes, int threads) {
    if (n == 0) return 1;
    if (width_bits != 8 && width_bits != 16 && width_bits != 32) return 2;
    if (block_len >= (1ull << 32)) return 2;
    uint64_t L = block_len == 0 ? n : block_len;
    uint64_t n_blocks = (n + L - 1) / L;
    if (n_blocks >= (1ull << 32)) return 2;
    if (out_capacity < 32 + 16 * n_blocks) return 3;
    cjob_t J;
    memset(&J, 0, sizeof J);
    J.in = in; J.width_bits = width_bits; J.n = n; J.L = L; J.out = out; J.n_blocks = n_blocks;
    J.n_words = (uint32_t*)malloc(sizeof(uint32_t) * n_blocks);
    J.word_off = (uint64_t*)malloc(sizeof(uint64_t) * n_blocks);
    if (!J.n_words || !J.word_off) { free(J.n_words); free(J.word_off); return 4; }
    J.pass = 1;
    run_jobs(&J, threads, compress_worker);
    uint64_t acc = 0;
    for (uint64_t b = 0; b < n_blocks; b++) { J.word_off[b] = acc; acc += J.n_words[b]; }
    uint64_t total = 32 + 16 * n_blocks + 8 * acc;
    if (total > out_capacity) { free(J.n_words); free(J.word_off); return 3; }
    J.pass = 2;
    run_jobs(&J, threads, compress_worker);
    /* global header, reading R9 */
    out[0] = 'P'; out[1] = 'L'; out[2] = 'Y'; out[3] = 'C';
    out[4] = 2; out[5] = 0; out[6] = (uint8_t)width_bits; out[7] = 0;
    put_u64(out + 8, n);
    put_u32(out + 16, (uint32_t)block_len);
    put_u32(out + 20, (uint32_t)n_blocks);
    put_u64(out + 24, 8 * acc);
    *out_bytes = total;
    free(J.n_words);
    free(J.word_off);
    return 0;
}

/* ---------------------------------------------------------------- decompress */
typedef struct {
    const uint8_t* in;
    uint64_t in_bytes;
    int width_bits;
    uint64_t n, L, n_blocks, b0, b1;
    const uint64_t* word_off;
    void* out;
    uint32_t status;
} djob_t;

static void* decompress_worker(void* arg) {
    djob_t* J = (djob_t*)arg;
    uint64_t pay0 = 32 + 16 * J->n_blocks;
    uint64_t vlim = (1ull << J->width_bits) - 1;
    for (uint64_t b = J->b0; b < J->b1; b++) {
        const uint8_t* hdr = J->in + 32 + 16 * b;
        uint32_t codec = get_u32(hdr), vmin = get_u32(hdr + 4);
        uint32_t bm1 = get_u32(hdr + 8), W = get_u32(hdr + 12);
        uint64_t lo = b * J->L;
        uint64_t hi = lo + J->L < J->n ? lo + J->L : J->n;
        uint64_t nb = hi - lo;
        if (codec == 1) {
            for (uint64_t i = lo; i < hi; i++) put_value(J->out, J->width_bits, i, vmin);
            continue;
        }
        if (codec != 2) continue; /* flagged in the serial pass */
        uint64_t B = (uint64_t)bm1 + 1;
        int k = oracle_capacity(B);
        if (B < 2 || (uint64_t)vmin + bm1 > vlim || k == 0) continue;
        if (W != (nb + k - 1) / k) continue;
        const uint8_t* pay = J->in + pay0 + 8 * J->word_off[b];
        for (uint64_t j = 0; j < W; j++) {
            uint64_t s = get_u64(pay + 8 * j);
            uint64_t m = nb - j * (uint64_t)k;
            if (m > (uint64_t)k) m = (uint64_t)k;
            for (uint64_t i = 0; i < m; i++) {
                uint64_t d = s % B; /* polynomial division */
                s = s / B;
                put_value(J->out, J->width_bits, lo + j * (uint64_t)k + i, (uint64_t)vmin + d);
            }
            if (s != 0) J->status |= OST_RESIDUE;
        }
    }
    return NULL;
}

/* Decompress a whole stream.  *status receives OST_* bits (0 = ok).  The
 * caller passes the element capacity of `out`; returns the element count in
 * *n_out.  Returns 0 if decoding ran (check *status), nonzero if the stream
 * could not be parsed at all. */
int oracle_decompress(const uint8_t* in, uint64_t in_bytes, void* out, uint64_t out_capacity,
                      uint64_t* n_out, int* width_out, uint32_t* status, int threads) {
    *status = 0;
    if (in_bytes < 32) { *status = OST_LENGTH; return 1; }
    if (!(in[0] == 'P' && in[1] == 'L' && in[2] == 'Y' && in[3] == 'C')) { *status = OST_BAD_MAGIC; return 1; }
    if (in[4] != 2) { *status = OST_BAD_VERSION; return 1; }
    int width_bits = in[6];
    if (in[5] != 0 || in[7] != 0 || (width_bits != 8 && width_bits != 16 && width_bits != 32)) { *status = OST_HEADER_MISMATCH; return 1; }
    uint64_t n = get_u64(in + 8);
    uint64_t block_len = get_u32(in + 16);
    uint64_t n_blocks = get_u32(in + 20);
    uint64_t payload = get_u64(in + 24);
    if (n == 0) { *status = OST_HEADER_MISMATCH; return 1; }
    uint64_t L = block_len == 0 ? n : block_len;
    if ((n + L - 1) / L != n_blocks) { *status = OST_HEADER_MISMATCH; return 1; }
    if (n > out_capacity) { *status = OST_HEADER_MISMATCH; return 1; }
    if (in_bytes < 32 + 16 * n_blocks) { *status = OST_LENGTH; return 1; }
    uint64_t* off = (uint64_t*)malloc(sizeof(uint64_t) * (n_blocks ? n_blocks : 1));
    uint64_t acc = 0;
    uint32_t st = 0;
    uint64_t vlim = (1ull << width_bits) - 1;
    for (uint64_t b = 0; b < n_blocks; b++) {
        const uint8_t* hdr = in + 32 + 16 * b;
        uint32_t codec = get_u32(hdr), vmin = get_u32(hdr + 4);
        uint32_t bm1 = get_u32(hdr + 8), W = get_u32(hdr + 12);
        uint64_t lo = b * L, hi = lo + L < n ? lo + L : n, nb = hi - lo;
        off[b] = acc;
        if (codec == 1) {
            if (bm1 != 0 || W != 0) st |= OST_NWORDS;
            if ((uint64_t)vmin > vlim) st |= OST_OVERFLOW;
        } else if (codec == 2) {
            uint64_t B = (uint64_t)bm1 + 1;
            if (B < 2 || (uint64_t)vmin + bm1 > vlim) st |= OST_OVERFLOW;
            else {
                int k = oracle_capacity(B);
                if (W != (nb + k - 1) / k) st |= OST_NWORDS;
            }
        } else {
            st |= OST_BAD_CODEC;
        }
        acc += W;
    }
    if (8 * acc != payload || in_bytes != 32 + 16 * n_blocks + payload) st |= OST_LENGTH;
    if (st & (OST_LENGTH | OST_NWORDS)) { *status = st; free(off); return 0; }
    djob_t J;
    memset(&J, 0, sizeof J);
    J.in = in; J.in_bytes = in_bytes; J.width_bits = width_bits; J.n = n; J.L = L;
    J.n_blocks = n_blocks; J.word_off = off; J.out = out;
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > n_blocks) threads = (int)n_blocks;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    djob_t* jobs = (djob_t*)malloc(sizeof(djob_t) * threads);
    for (int t = 0; t < threads; t++) {
        jobs[t] = J;
        jobs[t].b0 = n_blocks * (uint64_t)t / (uint64_t)threads;
        jobs[t].b1 = n_blocks * (uint64_t)(t + 1) / (uint64_t)threads;
        if (threads == 1) decompress_worker(&jobs[t]);
        else pthread_create(&th[t], NULL, decompress_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    for (int t = 0; t < threads; t++) st |= jobs[t].status;
    free(jobs);
    free(th);
    free(off);
    *status = st;
    *n_out = n;
    *width_out = width_bits;
    return 0;
}

/*
 * oracle_adv.c -- plain C oracle for the ADVANCED (split-base) polynomial
 * codec of PAPER.md Sec. 3.2, blocked as in Sec. 3.3.
 *
 * TEST INFRASTRUCTURE ONLY (linked into liboracle.so with oracle.c).  It shares
 * no code, header, table or constant with the CUDA path.  It is the same
 * definition as oracle/advanced.py (whose header lists the readings A1-A6),
 * written with machine integers so the BASELINE-sized inputs finish in
 * seconds:
 *   p_i  = max{p : R'_{i-1} B^p <= 2^32 - 1}          (the series' p_i, exact)
 *   R_i  = floor((2^32 - 1) / (R'_{i-1} B^{p_i}))
 *   R'_i = ceil(B / R_i)
 *   s_i  = r_i + R_i * (sum_k d[q_i + k] B^(p_i - 1 - k) + r'_{i-1} B^{p_i})
 * with the split value d[q_i + p_i] = r'_i R_i + r_i, R'_0 = 1, r'_0 = 0, and
 * the FINAL word (values left m <= p_i) = r'_{i-1} B^m + sum_k d[q_i+k] B^(m-1-k).
 * Decoding uses the hardware "/" and "%".
 * Stream: 32-byte global header with layout byte 1, 16-byte block headers
 * {codec (0 RAW, 1 CONSTANT, 3 ADVANCED), v_min, b_minus_1, n_words}, then the
 * 32-bit words of every block, little-endian.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
#define WMAX 4294967295ull
#define AST_BAD_MAGIC 1u
#define AST_BAD_VERSION 2u
#define AST_HEADER_MISMATCH 4u
#define AST_BAD_CODEC 8u
#define AST_NWORDS 16u
#define AST_RESIDUE 32u
#define AST_OVERFLOW 64u
#define AST_LENGTH 128u

static uint64_t aget(const void* in, int w, uint64_t i) {
    if (w == 16) return ((const uint16_t*)in)[i];
    return ((const uint32_t*)in)[i];
}
static void aput(void* out, int w, uint64_t i, uint64_t v) {
    if (w == 16) ((uint16_t*)out)[i] = (uint16_t)v;
    else ((uint32_t*)out)[i] = (uint32_t)v;
}
static void p32(uint8_t* p, uint32_t v) { for (int i = 0; i < 4; i++) p[i] = (uint8_t)(v >> (8 * i)); }
static void p64(uint8_t* p, uint64_t v) { for (int i = 0; i < 8; i++) p[i] = (uint8_t)(v >> (8 * i)); }
static uint32_t g32(const uint8_t* p) { uint32_t v = 0; for (int i = 3; i >= 0; i--) v = (v << 8) | p[i]; return v; }
static uint64_t g64(const uint8_t* p) { uint64_t v = 0; for (int i = 7; i >= 0; i--) v = (v << 8) | p[i]; return v; }

/* p_i: the largest p with Rp * B^p <= 2^32 - 1 (exact, in 128 bits). */
int oracle_adv_capacity(uint64_t B, uint64_t Rp) {
    int p = 0;
    u128 x = Rp;
    while (x * (u128)B <= WMAX) {
        x = x * (u128)B;
        p = p + 1;
    }
    return p;
}

static uint64_t powu(uint64_t B, int e) {
    uint64_t x = 1;
    for (int i = 0; i < e; i++) x = x * B;
    return x;
}

/* Words of a block of n values with base B (the schedule walked to FINAL). */
uint64_t oracle_adv_word_count(uint64_t B, uint64_t n) {
    uint64_t Rp = 1, q = 0, w = 0;
    while (1) {
        int p = oracle_adv_capacity(B, Rp);
        w = w + 1;
        if (n - q <= (uint64_t)p) return w;
        uint64_t R = WMAX / (Rp * powu(B, p));
        Rp = (B + R - 1) / R;
        q = q + (uint64_t)p + 1;
    }
}

uint64_t oracle_max_compressed_bytes_advanced(uint64_t n, int width_bits, uint64_t block_len) {
    (void)width_bits;
    if (n == 0) return 32;
    uint64_t L = block_len == 0 ? n : block_len;
    uint64_t nb = (n + L - 1) / L;
    return 32 + 16 * nb + 4 * (n + nb); /* a word holds >= 1 value, the last may hold only a carry */
}

/* ------------------------------------------------------------------ compress */
typedef struct {
    const void* in;
    int w;
    uint64_t n, L, nblk, b0, b1;
    uint8_t* out;
    uint32_t* nwords;
    uint64_t* woff;
    int pass;
} ajob_t;

/* Pack one ADVANCED block: d[] are the min-shifted values. */
static void pack_block(const void* in, int w, uint64_t lo, uint64_t nb, uint64_t vmin, uint64_t B, uint8_t* pay) {
    uint64_t Rp = 1, q = 0, rprime = 0, j = 0;
    while (1) {
        int p = oracle_adv_capacity(B, Rp);
        uint64_t m = nb - q;
        if (m <= (uint64_t)p) { /* FINAL word */
            uint64_t s = rprime;
            for (uint64_t k = 0; k < m; k++) s = s * B + (aget(in, w, lo + q + k) - vmin);
            p32(pay + 4 * j, (uint32_t)s);
            return;
        }
        uint64_t R = WMAX / (Rp * powu(B, p));
        uint64_t body = rprime;
        for (int k = 0; k < p; k++) body = body * B + (aget(in, w, lo + q + (uint64_t)k) - vmin);
        uint64_t v = aget(in, w, lo + q + (uint64_t)p) - vmin; /* the split value */
        uint64_t rp = v / R, r = v - rp * R;
        u128 s = (u128)r + (u128)R * body;
        if (s > WMAX) abort(); /* cannot happen: R * Rp * B^p <= 2^32 - 1 */
        p32(pay + 4 * j, (uint32_t)s);
        j = j + 1;
        rprime = rp;
        Rp = (B + R - 1) / R;
        q = q + (uint64_t)p + 1;
    }
}

static void* acompress_worker(void* arg) {
    ajob_t* J = (ajob_t*)arg;
    for (uint64_t b = J->b0; b < J->b1; b++) {
        uint64_t lo = b * J->L, hi = lo + J->L < J->n ? lo + J->L : J->n, nb = hi - lo;
        uint64_t vmin = aget(J->in, J->w, lo), vmax = vmin;
        for (uint64_t i = lo; i < hi; i++) {
            uint64_t v = aget(J->in, J->w, i);
            if (v < vmin) vmin = v;
            if (v > vmax) vmax = v;
        }
        uint64_t B = vmax - vmin + 1;
        uint32_t codec = B == 1 ? 1u : (oracle_adv_capacity(B, 1) < 1 ? 0u : 3u);
        if (J->pass == 1) {
            uint64_t W = codec == 1 ? 0 : (codec == 0 ? nb : oracle_adv_word_count(B, nb));
            J->nwords[b] = (uint32_t)W;
            uint8_t* h = J->out + 32 + 16 * b;
            p32(h, codec);
            p32(h + 4, (uint32_t)vmin);
            p32(h + 8, (uint32_t)(B - 1));
            p32(h + 12, (uint32_t)W);
            continue;
        }
        uint8_t* pay = J->out + 32 + 16 * J->nblk + 4 * J->woff[b];
        if (codec == 0)
            for (uint64_t i = 0; i < nb; i++) p32(pay + 4 * i, (uint32_t)(aget(J->in, J->w, lo + i) - vmin));
        else if (codec == 3)
            pack_block(J->in, J->w, lo, nb, vmin, B, pay);
    }
    return NULL;
}

static void arun(ajob_t* base, int threads, void* (*fn)(void*)) {
    if (threads < 1) threads = 1;
    uint64_t nb = base->nblk;
    if ((uint64_t)threads > nb) threads = (int)(nb ? nb : 1);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    ajob_t* jobs = (ajob_t*)malloc(sizeof(ajob_t) * threads);
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

/* returns 0 ok, 1 empty, 2 bad argument, 3 capacity, 4 oom */
int oracle_compress_advanced(const void* in, uint64_t n, int width_bits, uint64_t block_len, uint8_t* out,
                             uint64_t out_capacity, uint64_t* out_bytes, int threads) {
    if (n == 0) return 1;
    if ((width_bits != 16 && width_bits != 32) || block_len >= (1ull << 32)) return 2;
    uint64_t L = block_len == 0 ? n : block_len, nblk = (n + L - 1) / L;
    if (nblk >= (1ull << 32) || out_capacity < 32 + 16 * nblk) return 3;
    ajob_t J;
    memset(&J, 0, sizeof J);
    J.in = in; J.w = width_bits; J.n = n; J.L = L; J.nblk = nblk; J.out = out;
    J.nwords = (uint32_t*)malloc(4 * nblk);
    J.woff = (uint64_t*)malloc(8 * nblk);
    if (!J.nwords || !J.woff) { free(J.nwords); free(J.woff); return 4; }
    J.pass = 1;
    arun(&J, threads, acompress_worker);
    uint64_t acc = 0;
    for (uint64_t b = 0; b < nblk; b++) { J.woff[b] = acc; acc += J.nwords[b]; }
    uint64_t total = 32 + 16 * nblk + 4 * acc;
    if (total > out_capacity) { free(J.nwords); free(J.woff); return 3; }
    J.pass = 2;
    arun(&J, threads, acompress_worker);
    out[0] = 'P'; out[1] = 'L'; out[2] = 'Y'; out[3] = 'C';
    out[4] = 2; out[5] = 1; out[6] = (uint8_t)width_bits; out[7] = 0;
    p64(out + 8, n);
    p32(out + 16, (uint32_t)block_len);
    p32(out + 20, (uint32_t)nblk);
    p64(out + 24, 4 * acc);
    *out_bytes = total;
    free(J.nwords);
    free(J.woff);
    return 0;
}

/* ---------------------------------------------------------------- decompress */
typedef struct {
    const uint8_t* in;
    int w;
    uint64_t n, L, nblk, b0, b1;
    const uint64_t* woff;
    void* out;
    uint32_t status;
} adjob_t;

/* Unpack one ADVANCED block; returns AST_* bits. */
static uint32_t unpack_block(const uint8_t* pay, uint64_t B, uint64_t nb, uint64_t vmin, void* out, int w, uint64_t lo) {
    uint64_t Rp = 1, q = 0, j = 0, Rprev = 0, rprev = 0, qsplit = 0;
    while (1) {
        int p = oracle_adv_capacity(B, Rp);
        uint64_t m = nb - q;
        int fin = m <= (uint64_t)p;
        uint64_t s = g32(pay + 4 * j), r = 0, t = s, R = 0;
        if (!fin) {
            R = WMAX / (Rp * powu(B, p));
            r = s % R;
            t = s / R;
        }
        uint64_t cnt = fin ? m : (uint64_t)p;
        uint64_t low = powu(B, (int)cnt);
        uint64_t carry = t / low, digits = t % low;
        if (carry >= Rp) return AST_RESIDUE;
        for (uint64_t k = cnt; k-- > 0;) { /* polynomial division, lowest power first */
            aput(out, w, lo + q + k, vmin + digits % B);
            digits = digits / B;
        }
        if (j > 0) { /* the previous word's split value */
            uint64_t v = carry * Rprev + rprev;
            if (v >= B) return AST_RESIDUE;
            aput(out, w, lo + qsplit, vmin + v);
        }
        if (fin) return 0;
        Rprev = R;
        rprev = r;
        qsplit = q + (uint64_t)p;
        Rp = (B + R - 1) / R;
        q = q + (uint64_t)p + 1;
        j = j + 1;
    }
}

static void* adecompress_worker(void* arg) {
    adjob_t* J = (adjob_t*)arg;
    uint64_t pay0 = 32 + 16 * J->nblk;
    for (uint64_t b = J->b0; b < J->b1; b++) {
        const uint8_t* h = J->in + 32 + 16 * b;
        uint32_t codec = g32(h), vmin = g32(h + 4), bm1 = g32(h + 8);
        uint64_t lo = b * J->L, hi = lo + J->L < J->n ? lo + J->L : J->n, nb = hi - lo;
        const uint8_t* pay = J->in + pay0 + 4 * J->woff[b];
        uint64_t B = (uint64_t)bm1 + 1;
        if (codec == 1) {
            for (uint64_t i = lo; i < hi; i++) aput(J->out, J->w, i, vmin);
        } else if (codec == 0) {
            for (uint64_t i = 0; i < nb; i++) {
                uint64_t d = g32(pay + 4 * i);
                if (d >= B) J->status |= AST_RESIDUE;
                aput(J->out, J->w, lo + i, vmin + d);
            }
        } else if (codec == 3) {
            J->status |= unpack_block(pay, B, nb, vmin, J->out, J->w, lo);
        }
    }
    return NULL;
}

int oracle_decompress_advanced(const uint8_t* in, uint64_t in_bytes, void* out, uint64_t out_capacity,
                               uint64_t* n_out, int* width_out, uint32_t* status, int threads) {
    *status = 0;
    if (in_bytes < 32) { *status = AST_LENGTH; return 1; }
    if (!(in[0] == 'P' && in[1] == 'L' && in[2] == 'Y' && in[3] == 'C')) { *status = AST_BAD_MAGIC; return 1; }
    if (in[4] != 2) { *status = AST_BAD_VERSION; return 1; }
    int w = in[6];
    if (in[5] != 1 || in[7] != 0 || (w != 16 && w != 32)) { *status = AST_HEADER_MISMATCH; return 1; }
    uint64_t n = g64(in + 8), bl = g32(in + 16), nblk = g32(in + 20), pb = g64(in + 24);
    if (n == 0) { *status = AST_HEADER_MISMATCH; return 1; }
    uint64_t L = bl == 0 ? n : bl;
    if ((n + L - 1) / L != nblk || n > out_capacity) { *status = AST_HEADER_MISMATCH; return 1; }
    if (in_bytes < 32 + 16 * nblk) { *status = AST_LENGTH; return 1; }
    uint64_t* off = (uint64_t*)malloc(8 * (nblk ? nblk : 1));
    uint64_t acc = 0, vlim = (1ull << w) - 1;
    uint32_t st = 0;
    for (uint64_t b = 0; b < nblk; b++) {
        const uint8_t* h = in + 32 + 16 * b;
        uint32_t codec = g32(h), vmin = g32(h + 4), bm1 = g32(h + 8), W = g32(h + 12);
        uint64_t lo = b * L, hi = lo + L < n ? lo + L : n, nb = hi - lo;
        uint64_t B = (uint64_t)bm1 + 1;
        off[b] = acc;
        if (codec == 1) {
            if (bm1 != 0 || W != 0) st |= AST_NWORDS;
            if ((uint64_t)vmin > vlim) st |= AST_OVERFLOW;
        } else if (codec == 0) {
            if ((uint64_t)vmin + bm1 > vlim) st |= AST_OVERFLOW;
            else if (oracle_adv_capacity(B, 1) >= 1) st |= AST_BAD_CODEC; /* RAW only when nothing packs */
            if (W != nb) st |= AST_NWORDS;
        } else if (codec == 3) {
            if (B < 2 || (uint64_t)vmin + bm1 > vlim || oracle_adv_capacity(B, 1) < 1) st |= AST_OVERFLOW;
            else if (W != oracle_adv_word_count(B, nb)) st |= AST_NWORDS;
        } else {
            st |= AST_BAD_CODEC;
        }
        acc += W;
    }
    if (4 * acc != pb || in_bytes != 32 + 16 * nblk + pb) st |= AST_LENGTH;
    if (st) { *status = st; free(off); return 0; }
    adjob_t J;
    memset(&J, 0, sizeof J);
    J.in = in; J.w = w; J.n = n; J.L = L; J.nblk = nblk; J.woff = off; J.out = out;
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > nblk) threads = (int)nblk;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    adjob_t* jobs = (adjob_t*)malloc(sizeof(adjob_t) * threads);
    for (int t = 0; t < threads; t++) {
        jobs[t] = J;
        jobs[t].b0 = nblk * (uint64_t)t / (uint64_t)threads;
        jobs[t].b1 = nblk * (uint64_t)(t + 1) / (uint64_t)threads;
        if (threads == 1) adecompress_worker(&jobs[t]);
        else pthread_create(&th[t], NULL, adecompress_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    for (int t = 0; t < threads; t++) st |= jobs[t].status;
    free(jobs);
    free(th);
    free(off);
    *status = st;
    *n_out = n;
    *width_out = w;
    return 0;
}

/* ORACLE / TEST INFRASTRUCTURE ONLY — see xpir_oracle.h for scope and pinning.
 * Each function cites the reference file:line (under /root/reference/proj) it
 * restates. */
#include "xpir_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static inline uint32_t rotl32(uint32_t x, int n) { return (x << n) | (x >> (32 - n)); }
static inline uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }
static inline uint64_t rotl64(uint64_t x, int n) { return (x << n) | (x >> (64 - n)); }
static inline uint32_t ld32le(const uint8_t* p) {
    return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24;
}
static inline uint64_t ld64le(const uint8_t* p) {
    return (uint64_t)ld32le(p) | (uint64_t)ld32le(p + 4) << 32;
}
static inline void st32le(uint8_t* p, uint32_t v) {
    p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}
static inline void st64le(uint8_t* p, uint64_t v) { st32le(p, (uint32_t)v); st32le(p + 4, (uint32_t)(v >> 32)); }
static inline void st64be(uint8_t* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (56 - 8 * i));
}

/* ---- ChaCha20, original DJB layout (crypto_stream_chacha20) -------------- */
#define QR(a, b, c, d)                                   \
    a += b; d ^= a; d = rotl32(d, 16);                   \
    c += d; b ^= c; b = rotl32(b, 12);                   \
    a += b; d ^= a; d = rotl32(d, 8);                    \
    c += d; b ^= c; b = rotl32(b, 7)

static void chacha20_block(const uint32_t in[16], uint8_t out[64]) {
    uint32_t x[16];
    memcpy(x, in, sizeof x);
    for (int i = 0; i < 10; ++i) {
        QR(x[0], x[4], x[8], x[12]); QR(x[1], x[5], x[9], x[13]);
        QR(x[2], x[6], x[10], x[14]); QR(x[3], x[7], x[11], x[15]);
        QR(x[0], x[5], x[10], x[15]); QR(x[1], x[6], x[11], x[12]);
        QR(x[2], x[7], x[8], x[13]); QR(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; ++i) st32le(out + 4 * i, x[i] + in[i]);
}

void xo_chacha20_stream(uint8_t* out, uint64_t len, const uint8_t key[32], const uint8_t nonce[8],
                        uint64_t block0) {
    uint32_t st[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u};
    for (int i = 0; i < 8; ++i) st[4 + i] = ld32le(key + 4 * i);
    st[14] = ld32le(nonce);
    st[15] = ld32le(nonce + 4);
    uint64_t ctr = block0;
    uint8_t blk[64];
    while (len) {
        st[12] = (uint32_t)ctr;
        st[13] = (uint32_t)(ctr >> 32);
        chacha20_block(st, blk);
        uint64_t n = len < 64 ? len : 64;
        memcpy(out, blk, n);
        out += n;
        len -= n;
        ++ctr;
    }
}

/* ---- BLAKE2b (crypto_generichash, unkeyed) ------------------------------- */
static const uint64_t B2_IV[8] = {
    0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL, 0xa54ff53a5f1d36f1ULL,
    0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL, 0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};
static const uint8_t B2_SIGMA[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

static void b2_compress(xo_blake2b_state* s, const uint8_t blk[128], int last) {
    uint64_t m[16], v[16];
    for (int i = 0; i < 16; ++i) m[i] = ld64le(blk + 8 * i);
    for (int i = 0; i < 8; ++i) { v[i] = s->h[i]; v[8 + i] = B2_IV[i]; }
    v[12] ^= s->t[0];
    v[13] ^= s->t[1];
    if (last) v[14] = ~v[14];
#define G(r, i, a, b, c, d)                                  \
    a = a + b + m[B2_SIGMA[r][2 * i]]; d = rotr64(d ^ a, 32); \
    c = c + d; b = rotr64(b ^ c, 24);                        \
    a = a + b + m[B2_SIGMA[r][2 * i + 1]]; d = rotr64(d ^ a, 16); \
    c = c + d; b = rotr64(b ^ c, 63)
    for (int r = 0; r < 12; ++r) {
        G(r, 0, v[0], v[4], v[8], v[12]); G(r, 1, v[1], v[5], v[9], v[13]);
        G(r, 2, v[2], v[6], v[10], v[14]); G(r, 3, v[3], v[7], v[11], v[15]);
        G(r, 4, v[0], v[5], v[10], v[15]); G(r, 5, v[1], v[6], v[11], v[12]);
        G(r, 6, v[2], v[7], v[8], v[13]); G(r, 7, v[3], v[4], v[9], v[14]);
    }
#undef G
    for (int i = 0; i < 8; ++i) s->h[i] ^= v[i] ^ v[8 + i];
}

void xo_blake2b_init(xo_blake2b_state* s, size_t outlen) {
    memset(s, 0, sizeof *s);
    for (int i = 0; i < 8; ++i) s->h[i] = B2_IV[i];
    s->h[0] ^= 0x01010000ULL ^ (uint64_t)outlen;
    s->outlen = outlen;
}

void xo_blake2b_update(xo_blake2b_state* s, const uint8_t* in, uint64_t len) {
    while (len) {
        if (s->buflen == 128) { /* only compress once more input is known to follow */
            s->t[0] += 128;
            if (s->t[0] < 128) s->t[1]++;
            b2_compress(s, s->buf, 0);
            s->buflen = 0;
        }
        size_t take = 128 - s->buflen;
        if (take > len) take = (size_t)len;
        memcpy(s->buf + s->buflen, in, take);
        s->buflen += take;
        in += take;
        len -= take;
    }
}

void xo_blake2b_final(xo_blake2b_state* s, uint8_t* out) {
    s->t[0] += s->buflen;
    if (s->t[0] < s->buflen) s->t[1]++;
    memset(s->buf + s->buflen, 0, 128 - s->buflen);
    b2_compress(s, s->buf, 1);
    uint8_t full[64];
    for (int i = 0; i < 8; ++i) st64le(full + 8 * i, s->h[i]);
    memcpy(out, full, s->outlen);
}

void xo_blake2b(uint8_t* out, size_t outlen, const uint8_t* in, uint64_t len) {
    xo_blake2b_state s;
    xo_blake2b_init(&s, outlen);
    xo_blake2b_update(&s, in, len);
    xo_blake2b_final(&s, out);
}

/* ---- SipHash-2-4 (crypto_shorthash) -------------------------------------- */
#define SIPROUND                                                            \
    v0 += v1; v1 = rotl64(v1, 13); v1 ^= v0; v0 = rotl64(v0, 32);          \
    v2 += v3; v3 = rotl64(v3, 16); v3 ^= v2;                                \
    v0 += v3; v3 = rotl64(v3, 21); v3 ^= v0;                                \
    v2 += v1; v1 = rotl64(v1, 17); v1 ^= v2; v2 = rotl64(v2, 32)

uint64_t xo_siphash24(const uint8_t key[16], const uint8_t* in, uint64_t len) {
    uint64_t k0 = ld64le(key), k1 = ld64le(key + 8);
    uint64_t v0 = k0 ^ 0x736f6d6570736575ULL, v1 = k1 ^ 0x646f72616e646f6dULL;
    uint64_t v2 = k0 ^ 0x6c7967656e657261ULL, v3 = k1 ^ 0x7465646279746573ULL;
    uint64_t i = 0;
    for (; i + 8 <= len; i += 8) {
        uint64_t m = ld64le(in + i);
        v3 ^= m;
        SIPROUND; SIPROUND;
        v0 ^= m;
    }
    uint64_t b = len << 56;
    for (uint64_t j = 0; i + j < len; ++j) b |= (uint64_t)in[i + j] << (8 * j);
    v3 ^= b;
    SIPROUND; SIPROUND;
    v0 ^= b;
    v2 ^= 0xff;
    SIPROUND; SIPROUND; SIPROUND; SIPROUND;
    return v0 ^ v1 ^ v2 ^ v3;
}

/* ---- DetRng (rng.cpp) ---------------------------------------------------- */
void xo_detrng_init_seed(xo_detrng* r, uint64_t seed) {
    uint8_t buf[8];
    st64le(buf, seed);                 /* rng.cpp:20-21 */
    xo_blake2b(r->key, 32, buf, 8);    /* rng.cpp:22 */
    r->block = 0;
}

void xo_detrng_init_key(xo_detrng* r, const uint8_t key[32]) {
    memcpy(r->key, key, 32);
    r->block = 0;
}

void xo_detrng_fill(xo_detrng* r, uint8_t* out, uint64_t n) {
    uint8_t nonce[8];
    st64le(nonce, r->block);           /* rng.cpp:28 */
    r->block++;                        /* rng.cpp:29 */
    xo_chacha20_stream(out, n, r->key, nonce, 0); /* rng.cpp:30 */
}

uint64_t xo_detrng_next_u64(xo_detrng* r) {
    uint8_t b[8];
    xo_detrng_fill(r, b, 8);
    return ld64le(b);
}

uint64_t xo_detrng_uniform(xo_detrng* r, uint64_t bound) {
    uint64_t tail = (UINT64_MAX % bound + 1) % bound; /* rng.cpp:11 */
    for (;;) {
        uint64_t v = xo_detrng_next_u64(r);
        if (tail == 0 || v <= UINT64_MAX - tail) return v % bound;
    }
}

/* ---- crypto.cpp ---------------------------------------------------------- */
uint64_t xo_prf(const uint8_t key[16], uint64_t input, uint64_t modulus) {
    uint64_t tail = (UINT64_MAX % modulus + 1) % modulus; /* crypto.cpp:22 */
    uint8_t block[16];
    for (uint64_t attempt = 0;; ++attempt) {
        st64le(block, input);
        st64le(block + 8, attempt);
        uint64_t v = xo_siphash24(key, block, 16);
        if (tail == 0 || v <= UINT64_MAX - tail) return v % modulus;
    }
}

void xo_bloom_positions(const uint8_t* item, uint64_t len, uint32_t h, uint32_t m_bits,
                        uint32_t* out) {
    for (uint32_t i = 0; i < h; ++i) {
        xo_blake2b_state st;
        xo_blake2b_init(&st, 8);
        xo_blake2b_update(&st, item, len);
        uint8_t idx[4];
        st32le(idx, i);
        xo_blake2b_update(&st, idx, 4);
        uint8_t o[8];
        xo_blake2b_final(&st, o);
        uint64_t v = ld64le(o);
        out[i] = (uint32_t)(((unsigned __int128)v * m_bits) >> 64); /* crypto.cpp:163 */
    }
}

void xo_make_interest(uint32_t m_bits, uint32_t h, const uint8_t id[16], uint64_t seq,
                      uint32_t* out) {
    uint8_t item[24];
    memcpy(item, id, 16);
    st64be(item + 16, seq); /* notify.cpp:32-33 */
    xo_bloom_positions(item, 24, h, m_bits, out);
}

uint32_t xo_bloom_hash_count(uint32_t m_bits, uint64_t n_window) {
    double h = round((double)m_bits / (double)n_window * log(2.0));
    return h < 1.0 ? 1 : (uint32_t)h;
}

/* ---- pir.cpp ------------------------------------------------------------- */
typedef struct {
    const uint8_t* db;
    uint32_t N, S;
    const uint8_t* q;
    uint64_t q_stride;
    uint32_t r0, r1;
    uint8_t* out;
} scan_job;

static void* scan_worker(void* arg) {
    scan_job* j = (scan_job*)arg;
    memset(j->out + (size_t)j->r0 * j->S, 0, (size_t)(j->r1 - j->r0) * j->S);
    for (uint32_t b = 0; b < j->N; ++b) { /* bucket-outer, request-inner: pir.cpp:46-50 */
        const uint8_t* bucket = j->db + (size_t)b * j->S;
        for (uint32_t r = j->r0; r < j->r1; ++r) {
            if (!((j->q[r * j->q_stride + (b >> 3)] >> (b & 7)) & 1)) continue;
            uint8_t* acc = j->out + (size_t)r * j->S;
            uint32_t i = 0;
            for (; i + 8 <= j->S; i += 8) {
                uint64_t a, c;
                memcpy(&a, acc + i, 8);
                memcpy(&c, bucket + i, 8);
                a ^= c;
                memcpy(acc + i, &a, 8);
            }
            for (; i < j->S; ++i) acc[i] ^= bucket[i];
        }
    }
    return NULL;
}

int xo_answer_batch(const uint8_t* db, uint32_t N, uint32_t S, const uint8_t* q,
                    uint64_t q_stride, uint32_t q_bits, uint32_t B, uint8_t* out,
                    uint32_t threads) {
    if (q_bits != N) return -1; /* pir.cpp:42-44 */
    if (threads < 1) threads = 1;
    if (threads > B) threads = B ? B : 1;
    pthread_t* th = (pthread_t*)calloc(threads, sizeof(pthread_t));
    scan_job* jobs = (scan_job*)calloc(threads, sizeof(scan_job));
    for (uint32_t t = 0; t < threads; ++t) {
        jobs[t] = (scan_job){db, N, S, q, q_stride, (uint32_t)((uint64_t)B * t / threads),
                             (uint32_t)((uint64_t)B * (t + 1) / threads), out};
        pthread_create(&th[t], NULL, scan_worker, &jobs[t]);
    }
    for (uint32_t t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return 0;
}

void xo_mask_answer(const uint8_t* ans, uint64_t len, const uint8_t seed[32], uint8_t* out) {
    static const uint8_t zero_nonce[8] = {0};
    xo_chacha20_stream(out, len, seed, zero_nonce, 0); /* crypto.cpp:35-39 */
    for (uint64_t i = 0; i < len; ++i) out[i] ^= ans[i]; /* pir.cpp:67 */
}

int xo_gen_queries(uint32_t beta, uint32_t N, uint32_t servers, xo_detrng* rng, uint8_t* out) {
    if (N == 0 || servers < 2 || beta >= N) return -1; /* pir.cpp:9-11 */
    size_t nb = (N + 7) / 8;
    uint8_t* last = out + (size_t)(servers - 1) * nb;
    memset(last, 0, nb);
    last[beta / 8] |= (uint8_t)(1u << (beta % 8));
    for (uint32_t i = 0; i + 1 < servers; ++i) {
        uint8_t* q = out + (size_t)i * nb;
        xo_detrng_fill(rng, q, nb);
        if (N % 8) q[nb - 1] &= (uint8_t)(0xffu >> (8 - N % 8));
    }
    for (uint32_t i = 0; i + 1 < servers; ++i)
        for (size_t k = 0; k < nb; ++k) last[k] ^= out[(size_t)i * nb + k];
    return 0;
}

/* ---- cuckoo.cpp ---------------------------------------------------------- */
#define XO_MAX_DISPLACEMENTS 500u /* cuckoo.hpp:15 */

struct xo_table {
    uint32_t buckets, depth;
    uint64_t capacity, item;
    uint8_t* data;
    uint8_t* used;
    uint32_t *b1, *b2;
    uint64_t* stamp;
    /* FIFO (cuckoo.hpp:79 std::map stamp->slot): stamps are issued in order, so a
     * stamp-indexed array plus a moving head gives the same "oldest live" answer. */
    int64_t* fifo; /* stamp -> flat slot, -1 when erased */
    uint64_t fifo_cap, fifo_head;
    xo_detrng rng;
    uint64_t next_stamp, writes, live;
};

xo_table* xo_table_new(uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                       const uint8_t seed[32]) {
    if (!buckets || !depth || !item_size) return NULL;              /* cuckoo.cpp:15-16 */
    if (!capacity || capacity > (uint64_t)buckets * depth) return NULL; /* :17-18 */
    xo_table* t = (xo_table*)calloc(1, sizeof *t);
    uint64_t slots = (uint64_t)buckets * depth;
    t->buckets = buckets; t->depth = depth; t->capacity = capacity; t->item = item_size;
    t->data = (uint8_t*)calloc(slots, item_size);
    t->used = (uint8_t*)calloc(slots, 1);
    t->b1 = (uint32_t*)calloc(slots, 4);
    t->b2 = (uint32_t*)calloc(slots, 4);
    t->stamp = (uint64_t*)calloc(slots, 8);
    t->fifo_cap = 1024;
    t->fifo = (int64_t*)malloc(t->fifo_cap * 8);
    xo_detrng_init_key(&t->rng, seed);
    return t;
}

void xo_table_free(xo_table* t) {
    if (!t) return;
    free(t->data); free(t->used); free(t->b1); free(t->b2); free(t->stamp); free(t->fifo);
    free(t);
}

static int free_slot(const xo_table* t, uint32_t b) { /* cuckoo.cpp:31-35 */
    for (uint32_t s = 0; s < t->depth; ++s)
        if (!t->used[(uint64_t)b * t->depth + s]) return (int)s;
    return -1;
}

static void place(xo_table* t, uint32_t b, uint32_t s, uint32_t b1, uint32_t b2,
                  const uint8_t* data, uint64_t stamp) { /* cuckoo.cpp:37-46 */
    uint64_t f = (uint64_t)b * t->depth + s;
    memcpy(t->data + f * t->item, data, t->item);
    t->used[f] = 1; t->b1[f] = b1; t->b2[f] = b2; t->stamp[f] = stamp;
    while (stamp >= t->fifo_cap) {
        t->fifo = (int64_t*)realloc(t->fifo, t->fifo_cap * 2 * 8);
        t->fifo_cap *= 2;
    }
    t->fifo[stamp] = (int64_t)(uint32_t)(b * t->depth + s); /* 32-bit flat as in the reference */
    t->live++;
}

static void clear_slot(xo_table* t, uint32_t b, uint32_t s) { /* cuckoo.cpp:48-54 */
    uint64_t f = (uint64_t)b * t->depth + s;
    memset(t->data + f * t->item, 0, t->item);
    t->fifo[t->stamp[f]] = -1;
    t->used[f] = 0; t->b1[f] = 0; t->b2[f] = 0; t->stamp[f] = 0;
    t->live--;
}

int xo_table_insert(xo_table* t, uint32_t beta1, uint32_t beta2, const uint8_t* data,
                    uint32_t report[4]) {
    if (beta1 >= t->buckets || beta2 >= t->buckets) return -1; /* cuckoo.cpp:57-58 */
    uint32_t stored = 0, dropped = 0, gc = 0, disp = 0;
    t->writes++;                                                 /* :62 */
    if (t->live == t->capacity) {                                /* :64-69 */
        while (t->fifo[t->fifo_head] < 0) t->fifo_head++;
        uint32_t flat = (uint32_t)t->fifo[t->fifo_head];
        clear_slot(t, flat / t->depth, flat % t->depth);
        gc = 1;
    }
    uint64_t stamp = t->next_stamp++;                            /* :71 */
    int s = free_slot(t, beta1);                                 /* :73-84 */
    if (s >= 0) {
        place(t, beta1, (uint32_t)s, beta1, beta2, data, stamp);
        stored = 1;
        goto done;
    }
    s = free_slot(t, beta2);
    if (s >= 0) {
        place(t, beta2, (uint32_t)s, beta1, beta2, data, stamp);
        stored = 1;
        goto done;
    }
    {
        uint32_t be = xo_detrng_uniform(&t->rng, 2) == 0 ? beta1 : beta2; /* :89 */
        uint8_t* carry = (uint8_t*)malloc(t->item);
        uint8_t* victim = (uint8_t*)malloc(t->item);
        memcpy(carry, data, t->item);
        uint32_t c1 = beta1, c2 = beta2;
        uint64_t cst = stamp;
        int carry_incoming = 1, incoming_stored = 0;
        for (uint32_t hops = 0;; ++hops) {                       /* :95-119 */
            int fs = free_slot(t, be);
            if (fs >= 0) {
                place(t, be, (uint32_t)fs, c1, c2, carry, cst);
                if (carry_incoming) incoming_stored = 1;
                stored = (uint32_t)incoming_stored;
                disp = hops;
                free(carry); free(victim);
                goto done;
            }
            if (hops == XO_MAX_DISPLACEMENTS) break;
            uint32_t vs = (uint32_t)xo_detrng_uniform(&t->rng, t->depth); /* :105 */
            uint64_t f = (uint64_t)be * t->depth + vs;
            uint32_t v1 = t->b1[f], v2 = t->b2[f];
            uint64_t vst = t->stamp[f];
            memcpy(victim, t->data + f * t->item, t->item);
            clear_slot(t, be, vs);
            place(t, be, vs, c1, c2, carry, cst);
            if (carry_incoming) incoming_stored = 1;
            memcpy(carry, victim, t->item);
            c1 = v1; c2 = v2; cst = vst;
            carry_incoming = 0;
            be = v1 == be ? v2 : v1;                              /* :118 */
        }
        disp = XO_MAX_DISPLACEMENTS;                               /* :122-125 */
        dropped = 1;
        stored = (uint32_t)incoming_stored;
        free(carry); free(victim);
    }
done:
    if (report) { report[0] = stored; report[1] = dropped; report[2] = gc; report[3] = disp; }
    return 0;
}

const uint8_t* xo_table_data(const xo_table* t) { return t->data; }

void xo_table_counters(const xo_table* t, uint64_t* writes, uint64_t* live, uint64_t* next_stamp) {
    if (writes) *writes = t->writes;
    if (live) *live = t->live;
    if (next_stamp) *next_stamp = t->next_stamp;
}

void xo_table_meta(const xo_table* t, uint8_t* used, uint32_t* b1, uint32_t* b2, uint64_t* stamp) {
    uint64_t slots = (uint64_t)t->buckets * t->depth;
    if (used) memcpy(used, t->used, slots);
    if (b1) memcpy(b1, t->b1, slots * 4);
    if (b2) memcpy(b2, t->b2, slots * 4);
    if (stamp) memcpy(stamp, t->stamp, slots * 8);
}

static void upd_u64be(xo_blake2b_state* h, uint64_t v) {
    uint8_t b[8];
    st64be(b, v);
    xo_blake2b_update(h, b, 8);
}

void xo_table_state_digest(const xo_table* t, uint8_t out[32]) { /* cuckoo.cpp:137-149 */
    xo_blake2b_state h;
    xo_blake2b_init(&h, 32);
    upd_u64be(&h, t->writes);
    upd_u64be(&h, t->live);
    upd_u64be(&h, t->next_stamp);
    uint64_t slots = (uint64_t)t->buckets * t->depth;
    xo_blake2b_update(&h, t->data, slots * t->item);
    for (uint64_t f = 0; f < slots; ++f) {
        upd_u64be(&h, t->used[f] ? 1 : 0);
        upd_u64be(&h, (uint64_t)t->b1[f] << 32 | t->b2[f]);
        upd_u64be(&h, t->stamp[f]);
    }
    xo_blake2b_final(&h, out);
}

/* ---- notify.cpp Window --------------------------------------------------- */
struct xo_window {
    uint32_t m, h, w;
    uint64_t base, n, words;
    uint64_t** deltas; /* ring of at most w+1 */
};

xo_window* xo_window_new(uint32_t m_bits, uint32_t h, uint32_t w) {
    if (!w || !m_bits || !h) return NULL; /* notify.cpp:55-56 */
    xo_window* x = (xo_window*)calloc(1, sizeof *x);
    x->m = m_bits; x->h = h; x->w = w;
    x->words = (m_bits + 63) / 64;
    x->deltas = (uint64_t**)calloc((size_t)w + 1, sizeof(uint64_t*));
    x->deltas[0] = (uint64_t*)calloc(x->words, 8);
    x->n = 1;
    return x;
}

void xo_window_free(xo_window* x) {
    if (!x) return;
    for (uint64_t i = 0; i < x->n; ++i) free(x->deltas[i]);
    free(x->deltas);
    free(x);
}

int xo_window_absorb(xo_window* x, const uint32_t* pos, uint64_t n) { /* :60-65 */
    uint64_t* d = x->deltas[x->n - 1];
    for (uint64_t i = 0; i < n; ++i) {
        if (pos[i] >= x->m) return -1;
        d[pos[i] / 64] |= (uint64_t)1 << (pos[i] % 64);
    }
    return 0;
}

void xo_window_rotate(xo_window* x) { /* :67-73 */
    x->deltas[x->n++] = (uint64_t*)calloc(x->words, 8);
    while (x->n > x->w) {
        free(x->deltas[0]);
        memmove(x->deltas, x->deltas + 1, (x->n - 1) * sizeof(uint64_t*));
        x->n--;
        x->base++;
    }
}

void xo_window_digest(const xo_window* x, uint8_t out[32]) { /* :89-107 */
    xo_window_digest_n(x, x->n, out);
}

void xo_window_digest_n(const xo_window* x, uint64_t count, uint8_t out[32]) { /* Window::digest(count), :91-107 */
    xo_blake2b_state h;
    xo_blake2b_init(&h, 32);
    xo_blake2b_update(&h, (const uint8_t*)"interest-window-v1", 18);
    upd_u64be(&h, x->m);
    upd_u64be(&h, x->h);
    upd_u64be(&h, x->w);
    upd_u64be(&h, x->base);
    upd_u64be(&h, count);
    for (uint64_t i = 0; i < count && i < x->n; ++i) {
        /* raw words in host (little-endian) order, notify.cpp:103-104 */
        uint8_t b[8];
        for (uint64_t k = 0; k < x->words; ++k) {
            st64le(b, x->deltas[i][k]);
            xo_blake2b_update(&h, b, 8);
        }
    }
    xo_blake2b_final(&h, out);
}

uint64_t xo_window_size(const xo_window* x) { return x->n; }
uint64_t xo_window_base(const xo_window* x) { return x->base; }
const uint64_t* xo_window_delta(const xo_window* x, uint64_t i) { return x->deltas[i]; }

/* ---- interest-delta codecs (notify.cpp:119-180) ---------------------------- */
static uint64_t xo_put_varint(uint8_t* out, uint64_t at, uint64_t cap, uint64_t v) { /* :110-116 */
    while (v >= 0x80) {
        if (out && at < cap) out[at] = (uint8_t)(v | 0x80);
        ++at;
        v >>= 7;
    }
    if (out && at < cap) out[at] = (uint8_t)v;
    return at + 1;
}

static int xo_get_varint(const uint8_t* buf, uint64_t len, uint64_t* at, uint64_t* out) { /* :118-129 */
    uint64_t v = 0;
    int shift = 0;
    while (*at < len && shift < 64) {
        uint8_t b = buf[(*at)++];
        v |= (uint64_t)(b & 0x7f) << shift;
        if (!(b & 0x80)) {
            *out = v;
            return 1;
        }
        shift += 7;
    }
    return 0;
}

uint64_t xo_encode_delta(uint32_t m_bits, const uint64_t* words, uint8_t* out, uint64_t cap) { /* :131-149 */
    const uint64_t nw = ((uint64_t)m_bits + 63) / 64;
    uint64_t ones = 0;
    for (uint64_t w = 0; w < nw; ++w) ones += (uint64_t)__builtin_popcountll(words[w]);
    uint64_t need = xo_put_varint(NULL, 0, 0, m_bits);
    need = xo_put_varint(NULL, need, 0, ones);
    uint64_t prev = 0;
    int first = 1;
    for (uint64_t w = 0; w < nw; ++w) {
        uint64_t x = words[w];
        while (x) {
            uint64_t pos = w * 64 + (uint64_t)__builtin_ctzll(x);
            need = xo_put_varint(NULL, need, 0, first ? pos : pos - prev);
            prev = pos;
            first = 0;
            x &= x - 1;
        }
    }
    if (!out || cap < need) return need;
    uint64_t at = xo_put_varint(out, 0, cap, m_bits);
    at = xo_put_varint(out, at, cap, ones);
    prev = 0;
    first = 1;
    for (uint64_t w = 0; w < nw; ++w) {
        uint64_t x = words[w];
        while (x) {
            uint64_t pos = w * 64 + (uint64_t)__builtin_ctzll(x);
            at = xo_put_varint(out, at, cap, first ? pos : pos - prev);
            prev = pos;
            first = 0;
            x &= x - 1;
        }
    }
    return need;
}

/* notify::encode_positions (notify.cpp:182-196): varint(count) || varint(first) ||
 * varint(gaps) of the sorted positions, zero-padded to cap bytes. Returns the
 * encoded length; > cap means the reference throws (out is then left zeroed). */
uint64_t xo_encode_positions(const uint32_t* positions, uint32_t n, uint8_t* out, uint64_t cap) {
    uint32_t s[256];
    if (n > 256) return ~0ull;
    memcpy(s, positions, (size_t)n * 4);
    for (uint32_t i = 1; i < n; ++i) { /* insertion sort (std::sort order) */
        const uint32_t v = s[i];
        uint32_t j = i;
        while (j > 0 && s[j - 1] > v) {
            s[j] = s[j - 1];
            --j;
        }
        s[j] = v;
    }
    uint64_t need = xo_put_varint(NULL, 0, 0, n);
    for (uint32_t i = 0; i < n; ++i) need = xo_put_varint(NULL, need, 0, i == 0 ? s[i] : s[i] - s[i - 1]);
    if (out) memset(out, 0, cap);
    if (!out || need > cap) return need;
    uint64_t at = xo_put_varint(out, 0, cap, n);
    for (uint32_t i = 0; i < n; ++i) at = xo_put_varint(out, at, cap, i == 0 ? s[i] : s[i] - s[i - 1]);
    return need;
}

/* notify::decode_positions (notify.cpp:198-214): 1 ok (*count positions written
 * when they fit in max_out), 0 = std::nullopt. */
int xo_decode_positions(const uint8_t* buf, uint64_t len, uint32_t* out, uint32_t max_out, uint32_t* count_out) {
    uint64_t at = 0, count = 0, pos = 0;
    if (!xo_get_varint(buf, len, &at, &count) || count > len * 8) return 0;
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t gap;
        if (!xo_get_varint(buf, len, &at, &gap)) return 0;
        pos = i == 0 ? gap : pos + gap; /* uint64 arithmetic, wrapping as the reference's */
        if (pos > 0xffffffffull) return 0;
        if (out && i < max_out) out[i] = (uint32_t)pos;
    }
    *count_out = (uint32_t)count;
    return 1;
}

int xo_decode_delta(const uint8_t* buf, uint64_t len, uint32_t* m_bits, uint64_t* words,
                    uint64_t words_cap) { /* :151-170 */
    uint64_t at = 0, m = 0, count = 0;
    if (!xo_get_varint(buf, len, &at, &m) || !xo_get_varint(buf, len, &at, &count)) return 0;
    if (m == 0 || m > 0xffffffffull) return 0;
    const uint64_t nw = (m + 63) / 64;
    int fill = words && words_cap >= nw;
    if (fill) memset(words, 0, nw * 8);
    uint64_t pos = 0;
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t gap;
        if (!xo_get_varint(buf, len, &at, &gap)) return 0;
        if (i == 0)
            pos = gap;
        else {
            if (gap == 0) return 0;
            pos += gap;
        }
        if (pos >= m) return 0;
        if (fill) words[pos >> 6] |= 1ull << (pos & 63);
    }
    if (at != len) return 0;
    *m_bits = (uint32_t)m;
    return 1;
}

/* ORACLE / TEST INFRASTRUCTURE ONLY — a plain-C restatement of the reference's
 * server hot path (arXiv 2001.08250 "Talek", /root/reference/proj) used as the
 * parity checker for the CUDA path. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Parity pinning: every function here is checked against the unmodified
 * reference (oracle/_ref/libxpir_ref.so, built by oracle/Makefile) and against
 * the committed fixtures in tests/golden/ (written by oracle/make_golden.py from
 * that reference build). See tests/test_oracle.py.
 *
 * The reference delegates ChaCha20 / SipHash-2-4 / BLAKE2b to libsodium, which
 * is not vendored in /root/reference (proj/CMakeLists.txt:12-13, no pinned
 * version; the image carries libsodium 1.0.20). They are restated here from
 * their published specifications (DJB ChaCha20 with 8-byte nonce and 64-bit
 * block counter as in crypto_stream_chacha20; SipHash-2-4 as crypto_shorthash;
 * BLAKE2b as crypto_generichash, unkeyed).
 */
#ifndef XPIR_ORACLE_H
#define XPIR_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- primitives ---------------------------------------------------------- */

/* crypto_stream_chacha20 keystream starting at 64-byte block `block0`. */
void xo_chacha20_stream(uint8_t* out, uint64_t len, const uint8_t key[32], const uint8_t nonce[8],
                        uint64_t block0);

typedef struct {
    uint64_t h[8];
    uint64_t t[2];
    uint8_t buf[128];
    size_t buflen;
    size_t outlen;
} xo_blake2b_state;

void xo_blake2b_init(xo_blake2b_state* s, size_t outlen);
void xo_blake2b_update(xo_blake2b_state* s, const uint8_t* in, uint64_t len);
void xo_blake2b_final(xo_blake2b_state* s, uint8_t* out);
void xo_blake2b(uint8_t* out, size_t outlen, const uint8_t* in, uint64_t len);

uint64_t xo_siphash24(const uint8_t key[16], const uint8_t* in, uint64_t len);

/* ---- rng.cpp ------------------------------------------------------------- */
typedef struct {
    uint8_t key[32];
    uint64_t block; /* fill-call counter = nonce (rng.cpp:25-31) */
} xo_detrng;

void xo_detrng_init_seed(xo_detrng* r, uint64_t seed);       /* rng.cpp:18-23 */
void xo_detrng_init_key(xo_detrng* r, const uint8_t key[32]); /* rng.hpp:43 */
void xo_detrng_fill(xo_detrng* r, uint8_t* out, uint64_t n);   /* rng.cpp:25-31 */
uint64_t xo_detrng_next_u64(xo_detrng* r);                     /* rng.hpp:31-37 */
uint64_t xo_detrng_uniform(xo_detrng* r, uint64_t bound);      /* rng.cpp:9-16 */

/* ---- crypto.cpp ---------------------------------------------------------- */
uint64_t xo_prf(const uint8_t key[16], uint64_t input, uint64_t modulus); /* :17-33 */
void xo_bloom_positions(const uint8_t* item, uint64_t len, uint32_t h, uint32_t m_bits,
                        uint32_t* out);                                    /* :146-166 */
void xo_make_interest(uint32_t m_bits, uint32_t h, const uint8_t id[16], uint64_t seq,
                      uint32_t* out);                                      /* notify.cpp:30-35 */
uint32_t xo_bloom_hash_count(uint32_t m_bits, uint64_t n_window);          /* notify.cpp:17-21 */

/* ---- pir.cpp ------------------------------------------------------------- */
/* answer_batch (pir.cpp:41-52): out[r*S..] = XOR of buckets j<N with bit j of
 * q[r*q_stride..] set. Returns -1 when q_bits != N (the reference's
 * invalid_argument). `threads` host threads split the requests. */
int xo_answer_batch(const uint8_t* db, uint32_t N, uint32_t S, const uint8_t* q,
                    uint64_t q_stride, uint32_t q_bits, uint32_t B, uint8_t* out,
                    uint32_t threads);
/* mask_answer (pir.cpp:65-69): out = ans ^ chacha20(seed, nonce 0)[0:len] */
void xo_mask_answer(const uint8_t* ans, uint64_t len, const uint8_t seed[32], uint8_t* out);
/* gen_queries (pir.cpp:7-27): out = servers * ceil(N/8) bytes */
int xo_gen_queries(uint32_t beta, uint32_t N, uint32_t servers, xo_detrng* rng, uint8_t* out);

/* ---- cuckoo.cpp ---------------------------------------------------------- */
typedef struct xo_table xo_table;
xo_table* xo_table_new(uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                       const uint8_t seed[32]);                           /* :8-21 */
void xo_table_free(xo_table* t);
/* insert (cuckoo.cpp:56-126); report = {stored, dropped, gc_evicted, displacements} */
int xo_table_insert(xo_table* t, uint32_t beta1, uint32_t beta2, const uint8_t* data,
                    uint32_t report[4]);
const uint8_t* xo_table_data(const xo_table* t);                          /* snapshot bytes */
void xo_table_state_digest(const xo_table* t, uint8_t out[32]);            /* :137-149 */
void xo_table_counters(const xo_table* t, uint64_t* writes, uint64_t* live, uint64_t* next_stamp);
/* per-slot metadata: used (0/1), beta1, beta2, stamp */
void xo_table_meta(const xo_table* t, uint8_t* used, uint32_t* beta1, uint32_t* beta2,
                   uint64_t* stamp);

/* ---- notify.cpp ---------------------------------------------------------- */
typedef struct xo_window xo_window;
xo_window* xo_window_new(uint32_t m_bits, uint32_t h, uint32_t w); /* :54-58 */
void xo_window_free(xo_window* w);
int xo_window_absorb(xo_window* w, const uint32_t* pos, uint64_t n); /* :60-65 */
void xo_window_rotate(xo_window* w);                                  /* :67-73 */
void xo_window_digest(const xo_window* w, uint8_t out[32]);           /* :89-107 */
void xo_window_digest_n(const xo_window* w, uint64_t count, uint8_t out[32]); /* digest(count) */
uint64_t xo_window_size(const xo_window* w);
uint64_t xo_window_base(const xo_window* w);
const uint64_t* xo_window_delta(const xo_window* w, uint64_t i);
/* notify::encode_delta (notify.cpp:139-157): returns the encoded size; writes when cap suffices */
uint64_t xo_encode_delta(uint32_t m_bits, const uint64_t* words, uint8_t* out, uint64_t cap);
/* notify::decode_delta (notify.cpp:159-180): 1 ok, 0 nullopt; words (ceil(m/64), zeroed here) when cap suffices */
int xo_decode_delta(const uint8_t* buf, uint64_t len, uint32_t* m_bits, uint64_t* words, uint64_t words_cap);
uint64_t xo_encode_positions(const uint32_t* positions, uint32_t n, uint8_t* out, uint64_t cap);
int xo_decode_positions(const uint8_t* buf, uint64_t len, uint32_t* out, uint32_t max_out, uint32_t* count_out);

#ifdef __cplusplus
}
#endif
#endif

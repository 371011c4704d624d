/* Declaration-only stand-in for <sodium.h>, written for this repo.
 *
 * ORACLE / TEST INFRASTRUCTURE ONLY. The reference (/root/reference/proj) links
 * libsodium but the image ships no header for it; the shared object that pyzmq
 * bundles (libsodium 1.0.20) exports every symbol the reference's hot-path
 * translation units call. This header declares just those symbols and the few
 * size constants the reference uses, so the reference sources compile
 * unmodified where they lie. The constants were checked against the library's
 * own crypto_*_bytes() functions.
 */
#ifndef XPIR_ORACLE_SODIUM_SHIM_H
#define XPIR_ORACLE_SODIUM_SHIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define crypto_stream_chacha20_NONCEBYTES 8U
#define crypto_stream_chacha20_KEYBYTES 32U
#define crypto_shorthash_BYTES 8U
#define crypto_shorthash_KEYBYTES 16U
#define crypto_secretbox_MACBYTES 16U
#define crypto_box_MACBYTES 16U
#define crypto_box_SEALBYTES 48U
#define crypto_sign_SECRETKEYBYTES 64U
#define crypto_sign_PUBLICKEYBYTES 32U
#define crypto_sign_BYTES 64U
#define crypto_kx_SESSIONKEYBYTES 32U
#define crypto_kx_PUBLICKEYBYTES 32U
#define crypto_kx_SECRETKEYBYTES 32U

/* libsodium 1.0.20 reports crypto_generichash_statebytes() == 384. */
#ifdef __cplusplus
#define XPIR_SHIM_ALIGN64 alignas(64)
#else
#define XPIR_SHIM_ALIGN64 _Alignas(64)
#endif
typedef struct {
    XPIR_SHIM_ALIGN64 unsigned char opaque[384];
} crypto_generichash_state;

int sodium_init(void);
void sodium_memzero(void* pnt, size_t len);
void randombytes_buf(void* buf, size_t size);

int crypto_stream_chacha20(unsigned char* c, unsigned long long clen, const unsigned char* n,
                           const unsigned char* k);

int crypto_generichash(unsigned char* out, size_t outlen, const unsigned char* in,
                       unsigned long long inlen, const unsigned char* key, size_t keylen);
int crypto_generichash_init(crypto_generichash_state* state, const unsigned char* key,
                            size_t keylen, size_t outlen);
int crypto_generichash_update(crypto_generichash_state* state, const unsigned char* in,
                              unsigned long long inlen);
int crypto_generichash_final(crypto_generichash_state* state, unsigned char* out, size_t outlen);

int crypto_shorthash(unsigned char* out, const unsigned char* in, unsigned long long inlen,
                     const unsigned char* k);

int crypto_secretbox_easy(unsigned char* c, const unsigned char* m, unsigned long long mlen,
                          const unsigned char* n, const unsigned char* k);
int crypto_secretbox_open_easy(unsigned char* m, const unsigned char* c, unsigned long long clen,
                               const unsigned char* n, const unsigned char* k);

int crypto_box_seed_keypair(unsigned char* pk, unsigned char* sk, const unsigned char* seed);
int crypto_box_easy(unsigned char* c, const unsigned char* m, unsigned long long mlen,
                    const unsigned char* n, const unsigned char* pk, const unsigned char* sk);
int crypto_box_seal(unsigned char* c, const unsigned char* m, unsigned long long mlen,
                    const unsigned char* pk);
int crypto_box_seal_open(unsigned char* m, const unsigned char* c, unsigned long long clen,
                         const unsigned char* pk, const unsigned char* sk);

int crypto_sign_seed_keypair(unsigned char* pk, unsigned char* sk, const unsigned char* seed);
int crypto_sign_detached(unsigned char* sig, unsigned long long* siglen_p, const unsigned char* m,
                         unsigned long long mlen, const unsigned char* sk);
int crypto_sign_verify_detached(const unsigned char* sig, const unsigned char* m,
                                unsigned long long mlen, const unsigned char* pk);

int crypto_kx_seed_keypair(unsigned char* pk, unsigned char* sk, const unsigned char* seed);
int crypto_kx_client_session_keys(unsigned char* rx, unsigned char* tx,
                                  const unsigned char* client_pk, const unsigned char* client_sk,
                                  const unsigned char* server_pk);
int crypto_kx_server_session_keys(unsigned char* rx, unsigned char* tx,
                                  const unsigned char* server_pk, const unsigned char* server_sk,
                                  const unsigned char* client_pk);

#ifdef __cplusplus
}
#endif

#endif

// Bit-exact device (and host) ports of the three libsodium primitives the
// reference's hot path calls:
//   ChaCha20, original DJB layout (crypto_stream_chacha20):
//       crypto::prng_expand (crypto.cpp:35-45), DetRng::fill (rng.cpp:25-31)
//   SipHash-2-4 (crypto_shorthash):      crypto::prf (crypto.cpp:17-33)
//   BLAKE2b, unkeyed (crypto_generichash): crypto::bloom_positions
//       (crypto.cpp:146-166), DetRng key (rng.cpp:18-23), Hasher/digest
//       (crypto.cpp:168-201)
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define XP_HD __host__ __device__ __forceinline__
#else
#define XP_HD inline
#endif

namespace xpir {

XP_HD uint32_t rotl32(uint32_t x, int n) { return (x << n) | (x >> (32 - n)); }
XP_HD uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }
XP_HD uint64_t rotl64(uint64_t x, int n) { return (x << n) | (x >> (64 - n)); }

XP_HD uint32_t ld32le(const uint8_t* p) {
    return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}
XP_HD uint64_t ld64le(const uint8_t* p) { return uint64_t(ld32le(p)) | uint64_t(ld32le(p + 4)) << 32; }

// ---- ChaCha20 ---------------------------------------------------------------
struct ChaChaKey {
    uint32_t k[8];
    uint32_t n[2];
};

XP_HD ChaChaKey chacha_key(const uint8_t key[32], uint64_t nonce) {
    ChaChaKey c;
    for (int i = 0; i < 8; ++i) c.k[i] = ld32le(key + 4 * i);
    c.n[0] = uint32_t(nonce);
    c.n[1] = uint32_t(nonce >> 32);
    return c;
}

#define XP_QR(a, b, c, d)          \
    a += b; d ^= a; d = rotl32(d, 16); \
    c += d; b ^= c; b = rotl32(b, 12); \
    a += b; d ^= a; d = rotl32(d, 8);  \
    c += d; b ^= c; b = rotl32(b, 7)

// One 64-byte keystream block as 16 little-endian words.
XP_HD void chacha20_block(const ChaChaKey& key, uint64_t counter, uint32_t out[16]) {
    const uint32_t c0 = 0x61707865u, c1 = 0x3320646eu, c2 = 0x79622d32u, c3 = 0x6b206574u;
    uint32_t x0 = c0, x1 = c1, x2 = c2, x3 = c3;
    uint32_t x4 = key.k[0], x5 = key.k[1], x6 = key.k[2], x7 = key.k[3];
    uint32_t x8 = key.k[4], x9 = key.k[5], x10 = key.k[6], x11 = key.k[7];
    uint32_t x12 = uint32_t(counter), x13 = uint32_t(counter >> 32);
    uint32_t x14 = key.n[0], x15 = key.n[1];
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int i = 0; i < 10; ++i) {
        XP_QR(x0, x4, x8, x12); XP_QR(x1, x5, x9, x13);
        XP_QR(x2, x6, x10, x14); XP_QR(x3, x7, x11, x15);
        XP_QR(x0, x5, x10, x15); XP_QR(x1, x6, x11, x12);
        XP_QR(x2, x7, x8, x13); XP_QR(x3, x4, x9, x14);
    }
    out[0] = x0 + c0; out[1] = x1 + c1; out[2] = x2 + c2; out[3] = x3 + c3;
    out[4] = x4 + key.k[0]; out[5] = x5 + key.k[1]; out[6] = x6 + key.k[2]; out[7] = x7 + key.k[3];
    out[8] = x8 + key.k[4]; out[9] = x9 + key.k[5]; out[10] = x10 + key.k[6]; out[11] = x11 + key.k[7];
    out[12] = x12 + uint32_t(counter); out[13] = x13 + uint32_t(counter >> 32);
    out[14] = x14 + key.n[0]; out[15] = x15 + key.n[1];
}
#undef XP_QR

// ---- SipHash-2-4 over a 16-byte message (the PRF block, crypto.cpp:24-28) ----
#define XP_SIPROUND                                                   \
    v0 += v1; v1 = rotl64(v1, 13); v1 ^= v0; v0 = rotl64(v0, 32);     \
    v2 += v3; v3 = rotl64(v3, 16); v3 ^= v2;                          \
    v0 += v3; v3 = rotl64(v3, 21); v3 ^= v0;                          \
    v2 += v1; v1 = rotl64(v1, 17); v1 ^= v2; v2 = rotl64(v2, 32)

XP_HD uint64_t siphash24_2w(uint64_t k0, uint64_t k1, uint64_t m0, uint64_t m1) {
    uint64_t v0 = k0 ^ 0x736f6d6570736575ULL, v1 = k1 ^ 0x646f72616e646f6dULL;
    uint64_t v2 = k0 ^ 0x6c7967656e657261ULL, v3 = k1 ^ 0x7465646279746573ULL;
    v3 ^= m0; XP_SIPROUND; XP_SIPROUND; v0 ^= m0;
    v3 ^= m1; XP_SIPROUND; XP_SIPROUND; v0 ^= m1;
    const uint64_t b = uint64_t(16) << 56;
    v3 ^= b; XP_SIPROUND; XP_SIPROUND; v0 ^= b;
    v2 ^= 0xff;
    XP_SIPROUND; XP_SIPROUND; XP_SIPROUND; XP_SIPROUND;
    return v0 ^ v1 ^ v2 ^ v3;
}
#undef XP_SIPROUND

// crypto::prf (crypto.cpp:17-33): rejection over fresh (input, attempt) blocks.
XP_HD uint64_t prf(uint64_t k0, uint64_t k1, uint64_t input, uint64_t modulus) {
    const uint64_t tail = (~uint64_t(0) % modulus + 1) % modulus;
    for (uint64_t attempt = 0;; ++attempt) {
        uint64_t v = siphash24_2w(k0, k1, input, attempt);
        if (tail == 0 || v <= ~uint64_t(0) - tail) return v % modulus;
    }
}

// ---- BLAKE2b --------------------------------------------------------------
struct Blake2bConst {
    static constexpr uint64_t IV0 = 0x6a09e667f3bcc908ULL, IV1 = 0xbb67ae8584caa73bULL,
                              IV2 = 0x3c6ef372fe94f82bULL, IV3 = 0xa54ff53a5f1d36f1ULL,
                              IV4 = 0x510e527fade682d1ULL, IV5 = 0x9b05688c2b3e6c1fULL,
                              IV6 = 0x1f83d9abfb41bd6bULL, IV7 = 0x5be0cd19137e2179ULL;
};

XP_HD uint64_t b2_iv(int i) {
    switch (i) {
        case 0: return Blake2bConst::IV0;
        case 1: return Blake2bConst::IV1;
        case 2: return Blake2bConst::IV2;
        case 3: return Blake2bConst::IV3;
        case 4: return Blake2bConst::IV4;
        case 5: return Blake2bConst::IV5;
        case 6: return Blake2bConst::IV6;
        default: return Blake2bConst::IV7;
    }
}

// sigma[r][i] packed as nibbles: row r, 16 nibbles, entry i at bits 4*i.
XP_HD uint32_t b2_sigma(int r, int i) {
    const uint64_t S[10] = {
        0xfedcba9876543210ULL, 0x357b20c16df984aeULL, 0x491763eadf250c8bULL,
        0x8f04a562ebcd1397ULL, 0xd386cb1efa427509ULL, 0x91ef57d438b0a6c2ULL,
        0xb8293670a4def15cULL, 0xa2684f05931ce7bdULL, 0x5a417d2c803b9ef6ULL,
        0x0dc3e9bf5167482aULL};
    return uint32_t(S[r % 10] >> (4 * i)) & 15u;
}

XP_HD void blake2b_compress(uint64_t h[8], const uint64_t m[16], uint64_t t0, uint64_t t1,
                            bool last) {
    uint64_t v[16];
    for (int i = 0; i < 8; ++i) {
        v[i] = h[i];
        v[8 + i] = b2_iv(i);
    }
    v[12] ^= t0;
    v[13] ^= t1;
    if (last) v[14] = ~v[14];
#define XP_G(r, i, a, b, c, d)                                       \
    a = a + b + m[b2_sigma(r, 2 * i)]; d = rotr64(d ^ a, 32);        \
    c = c + d; b = rotr64(b ^ c, 24);                                \
    a = a + b + m[b2_sigma(r, 2 * i + 1)]; d = rotr64(d ^ a, 16);    \
    c = c + d; b = rotr64(b ^ c, 63)
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int r = 0; r < 12; ++r) {
        XP_G(r, 0, v[0], v[4], v[8], v[12]); XP_G(r, 1, v[1], v[5], v[9], v[13]);
        XP_G(r, 2, v[2], v[6], v[10], v[14]); XP_G(r, 3, v[3], v[7], v[11], v[15]);
        XP_G(r, 4, v[0], v[5], v[10], v[15]); XP_G(r, 5, v[1], v[6], v[11], v[12]);
        XP_G(r, 6, v[2], v[7], v[8], v[13]); XP_G(r, 7, v[3], v[4], v[9], v[14]);
    }
#undef XP_G
    for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[8 + i];
}

// BLAKE2b-64 (outlen 8) of a message of at most 128 bytes given as 16 LE words
// (zero padded), returning the first output word. One compression: the whole
// bloom_positions input (24-byte item + 4-byte index) fits one block.
XP_HD uint64_t blake2b64_oneblock(const uint64_t m[16], uint32_t len) {
    uint64_t h[8];
    for (int i = 0; i < 8; ++i) h[i] = b2_iv(i);
    h[0] ^= 0x01010000ULL ^ 8ULL;
    blake2b_compress(h, m, len, 0, true);
    return h[0];
}

// crypto::bloom_positions (crypto.cpp:146-166) for one index i, item of <= 124 bytes.
XP_HD uint32_t bloom_position(const uint8_t* item, uint32_t len, uint32_t i, uint32_t m_bits) {
    uint64_t m[16];
    for (int k = 0; k < 16; ++k) m[k] = 0;
    for (uint32_t k = 0; k < len; ++k) m[k >> 3] |= uint64_t(item[k]) << (8 * (k & 7));
    for (uint32_t k = 0; k < 4; ++k)
        m[(len + k) >> 3] |= uint64_t((i >> (8 * k)) & 0xff) << (8 * ((len + k) & 7));
    uint64_t v = blake2b64_oneblock(m, len + 4);
#ifdef __CUDA_ARCH__
    return uint32_t(__umul64hi(v, uint64_t(m_bits)));
#else
    return uint32_t((unsigned __int128)v * m_bits >> 64);
#endif
}

// bloom_positions for the make_interest item (notify.cpp:30-35): LogId (16 B) ||
// BE64(seq), then LE32(i) — 28 message bytes, so m[4..15] are compile-time zero
// and the message words never touch local memory. w0/w1 = the LogId as LE words,
// w2 = the BE64 sequence number read as an LE word.
XP_HD uint32_t bloom_position_interest(uint64_t w0, uint64_t w1, uint64_t w2, uint32_t i, uint32_t m_bits) {
    uint64_t m[16];
    m[0] = w0;
    m[1] = w1;
    m[2] = w2;
    m[3] = uint64_t(i);
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int k = 4; k < 16; ++k) m[k] = 0;
    const uint64_t v = blake2b64_oneblock(m, 28);
#ifdef __CUDA_ARCH__
    return uint32_t(__umul64hi(v, uint64_t(m_bits)));
#else
    return uint32_t((unsigned __int128)v * m_bits >> 64);
#endif
}

}  // namespace xpir

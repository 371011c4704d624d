// Write path (K5-K7) and keystream generators on sm_100a.
//
//   K5 k_prf          crypto::prf (crypto.cpp:17-33)            SipHash-2-4 + rejection
//   K6 k_cuckoo_walk  cuckoo::Table::insert (cuckoo.cpp:56-126) sequential metadata walk
//      k_cuckoo_*     payload gather/scatter of the round          parallel
//   K7 k_interest     notify::make_interest (notify.cpp:30-35) + Window::absorb
//                     (notify.cpp:60-65): BLAKE2b positions OR-ed into the delta
//   k_keystream*      DetRng::fill / prng_expand keystream (rng.cpp:25-31)
//   k_draws           DetRng::next_u64 of consecutive fill calls (rng.hpp:31-37)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "prims.cuh"
#include "scan.cuh"

namespace xpir {

// ---------------------------------------------------------------------------
// keystream generators
// ---------------------------------------------------------------------------
__global__ void k_keystream(ChaChaKey key, uint64_t byte_offset, uint8_t* __restrict__ out,
                            uint64_t len) {
    const uint64_t blk_lo = byte_offset / 64;
    const uint64_t nblk = (byte_offset + len + 63) / 64 - blk_lo;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nblk; t += stride) {
        const uint64_t blk = blk_lo + t;
        uint32_t ks[16];
        chacha20_block(key, blk, ks);
        const uint64_t b0 = blk * 64;
        if (b0 >= byte_offset && b0 + 64 <= byte_offset + len && ((b0 - byte_offset) & 15) == 0 &&
            (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
            uint4* o4 = reinterpret_cast<uint4*>(out + (b0 - byte_offset));
#pragma unroll
            for (int k = 0; k < 4; ++k)
                __stcs(o4 + k, make_uint4(ks[4 * k], ks[4 * k + 1], ks[4 * k + 2], ks[4 * k + 3]));
        } else {
            for (int k = 0; k < 64; ++k) {
                const uint64_t p = b0 + k;
                if (p >= byte_offset && p < byte_offset + len)
                    out[p - byte_offset] = uint8_t(ks[k >> 2] >> (8 * (k & 3)));
            }
        }
    }
}

__global__ void k_keystream_rows(ChaChaKey key, uint64_t nonce0, uint32_t rows, uint64_t len,
                                 uint8_t* __restrict__ out, uint64_t row_stride) {
    const uint64_t nblk = (len + 63) / 64;
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= uint64_t(rows) * nblk) return;
    const uint32_t r = uint32_t(t / nblk);
    const uint64_t blk = t - uint64_t(r) * nblk;
    ChaChaKey k = key;
    const uint64_t nonce = nonce0 + r;
    k.n[0] = uint32_t(nonce);
    k.n[1] = uint32_t(nonce >> 32);
    uint32_t ks[16];
    chacha20_block(k, blk, ks);
    uint8_t* o = out + uint64_t(r) * row_stride + blk * 64;
    const uint64_t n = (len - blk * 64) < 64 ? (len - blk * 64) : 64;
    for (uint64_t i = 0; i < n; ++i) o[i] = uint8_t(ks[i >> 2] >> (8 * (i & 3)));
}

__global__ void k_draws(ChaChaKey key, uint64_t nonce0, uint32_t count, uint64_t* __restrict__ out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    ChaChaKey k = key;
    const uint64_t nonce = nonce0 + t;
    k.n[0] = uint32_t(nonce);
    k.n[1] = uint32_t(nonce >> 32);
    uint32_t ks[16];
    chacha20_block(k, 0, ks);
    out[t] = uint64_t(ks[0]) | uint64_t(ks[1]) << 32;
}

// ---------------------------------------------------------------------------
// K5 PRF, K7 interest / absorb
// ---------------------------------------------------------------------------
__global__ void k_prf(uint64_t k0, uint64_t k1, const uint64_t* __restrict__ in, uint64_t n,
                      uint64_t modulus, uint64_t* __restrict__ out, uint32_t* __restrict__ out32) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t v = prf(k0, k1, in[t], modulus);
    if (out) out[t] = v;
    if (out32) out32[t] = uint32_t(v);
}

// beta1 = prf(K1, x), beta2 = prf(K2, x) of every write key (logproto.cpp:74-75)
__global__ void k_prf2(uint64_t a0, uint64_t a1, uint64_t c0, uint64_t c1, const uint64_t* __restrict__ in,
                       uint64_t n, uint64_t modulus, uint32_t* __restrict__ o1, uint32_t* __restrict__ o2) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t x = in[t];
    o1[t] = uint32_t(prf(a0, a1, x, modulus));
    o2[t] = uint32_t(prf(c0, c1, x, modulus));
}

cudaError_t launch_prf2(const uint64_t k1[2], const uint64_t k2[2], const uint64_t* in, uint64_t n,
                        uint64_t modulus, uint32_t* o1, uint32_t* o2, cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_prf2<<<uint32_t((n + 127) / 128), 128, 0, s>>>(k1[0], k1[1], k2[0], k2[1], in, n, modulus, o1, o2);
    return cudaGetLastError();
}

struct Id16 {
    uint8_t b[16];
};

// BLAKE2b for the interest hashes (prims.cuh blake2b_compress, crypto.cpp:146-166
// via bloom_positions), the G function's rotate-left-by-1 moved to the FMA pipe:
// the compression is ALU-bound (XOR / funnel shift / 64-bit add all issue on the
// ALU pipe), so lo' = lo*2 + hi>>31 and hi' = hi*2 + lo>>31 are IMADs with a
// multiplier the compiler cannot fold (`two`, a kernel argument). Bit-identical.
// Measured (config 3 round as one graph): 0.119 -> 0.116 ms, the hashes alone
// 100 -> 96 us. Moving the rotations by 24 and 16 too (MUL.HI + IMAD pairs) was
// no faster (98.5 us) or slower (108 us): the longer dependency chain costs more.
__device__ __forceinline__ uint64_t rotl1_fma(uint64_t x, uint32_t two) {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    uint32_t tl, th, nl, nh;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(tl) : "r"(lo), "r"(two));   // lo >> 31
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(th) : "r"(hi), "r"(two));   // hi >> 31
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(nl) : "r"(lo), "r"(two), "r"(th));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(nh) : "r"(hi), "r"(two), "r"(tl));
    return (uint64_t(nh) << 32) | nl;
}

__device__ __forceinline__ uint64_t blake2b64_interest(uint64_t w0, uint64_t w1, uint64_t w2, uint32_t i,
                                                       uint32_t two) {
    const uint64_t m[16] = {w0, w1, w2, uint64_t(i), 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    uint64_t v[16];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        v[k] = b2_iv(k);
        v[8 + k] = b2_iv(k);
    }
    v[0] ^= 0x01010000ULL ^ 8ULL;  // parameter block: outlen 8, fanout 1, depth 1
    const uint64_t h0 = v[0];
    v[12] ^= 28;  // t0 = message length
    v[14] = ~v[14];
#define XP_GI(r, i, a, b, c, d)                                         \
    a = a + b + m[b2_sigma(r, 2 * i)]; d = rotr64(d ^ a, 32);           \
    c = c + d; b = rotr64(b ^ c, 24);                                   \
    a = a + b + m[b2_sigma(r, 2 * i + 1)]; d = rotr64(d ^ a, 16);       \
    c = c + d; b = rotl1_fma(b ^ c, two)
#pragma unroll
    for (int r = 0; r < 12; ++r) {
        XP_GI(r, 0, v[0], v[4], v[8], v[12]); XP_GI(r, 1, v[1], v[5], v[9], v[13]);
        XP_GI(r, 2, v[2], v[6], v[10], v[14]); XP_GI(r, 3, v[3], v[7], v[11], v[15]);
        XP_GI(r, 4, v[0], v[5], v[10], v[15]); XP_GI(r, 5, v[1], v[6], v[11], v[12]);
        XP_GI(r, 6, v[2], v[7], v[8], v[13]); XP_GI(r, 7, v[3], v[4], v[9], v[14]);
    }
#undef XP_GI
    return h0 ^ v[0] ^ v[8];
}

__global__ void k_interest(Id16 id, const uint64_t* __restrict__ seqs, uint64_t n, uint32_t h,
                           uint32_t m_bits, uint32_t* __restrict__ pos_out,
                           unsigned long long* __restrict__ words, uint32_t two) {
    uint64_t w0 = 0, w1 = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        w0 |= uint64_t(id.b[i]) << (8 * i);
        w1 |= uint64_t(id.b[8 + i]) << (8 * i);
    }
    // grid-stride over (write, hash index) pairs
    const uint64_t total = n * h, stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += stride) {
        const uint64_t w = t / h;
        const uint32_t k = uint32_t(t - w * h);
        // item = LogId || BE64(seq) (notify.cpp:33): the BE64 bytes read as an LE word
        const uint64_t sq = seqs[w];
        const uint64_t w2 = __byte_perm(uint32_t(sq >> 32), 0, 0x0123) |
                            uint64_t(__byte_perm(uint32_t(sq), 0, 0x0123)) << 32;
        const uint32_t pos = uint32_t(__umul64hi(blake2b64_interest(w0, w1, w2, k, two), uint64_t(m_bits)));
        if (pos_out) pos_out[t] = pos;
        if (words) atomicOr(words + (pos >> 6), 1ull << (pos & 63));
    }
}

__global__ void k_bloom_item(const uint8_t* __restrict__ item, uint32_t len, uint32_t h,
                             uint32_t m_bits, uint32_t* __restrict__ out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < h) out[t] = bloom_position(item, len, t, m_bits);
}

__global__ void k_absorb_check(const uint32_t* __restrict__ pos, uint64_t n, uint32_t m_bits,
                               unsigned long long* __restrict__ first_bad) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n && pos[t] >= m_bits) atomicMin(first_bad, (unsigned long long)t);
}

// cuckoo.cpp:57-58 for device-resident write batches: first item with a bucket
// index out of range (atomicMin; ~0 when none)
__global__ void k_beta_check(const uint32_t* __restrict__ b1, const uint32_t* __restrict__ b2, uint64_t n,
                             uint32_t buckets, unsigned long long* __restrict__ first_bad) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n && (b1[t] >= buckets || b2[t] >= buckets)) atomicMin(first_bad, (unsigned long long)t);
}

__global__ void k_absorb(const uint32_t* __restrict__ pos, uint64_t n,
                         const unsigned long long* __restrict__ limit,
                         unsigned long long* __restrict__ words) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n && t < *limit) atomicOr(words + (pos[t] >> 6), 1ull << (pos[t] & 63));
}

// ---------------------------------------------------------------------------
// K6: cuckoo insertion walk. One thread executes the reference's sequential
// semantics exactly (cuckoo.cpp:56-126); the rest of the CTA mirrors the
// occupancy bitmap into shared memory first so the common path (free slot in
// beta1/beta2) never waits on global memory. Payload bytes are not moved here:
// each touched slot records where its final content comes from (origin) and
// k_cuckoo_gather_sharded / k_cuckoo_scatter_sharded move the bytes in parallel
// afterwards.
//   origin >= 0   : payload row `origin` of this batch
//   origin == -1  : cleared (zero)
//   origin <= -2  : the pre-batch content of flat slot (-origin - 2)
// ---------------------------------------------------------------------------
constexpr uint32_t WALK_SMEM_MAX_SLOTS = 64 * 1024 * 8;  // bit-packed: 64 KiB each map
constexpr uint32_t WALK_MIN_DRAWS = 640;  // >= 1 + 500 draws of one insert, with slack
constexpr uint32_t WALK_DRAWS_SMEM = 4096;  // draws staged in shared memory per launch
constexpr uint32_t WALK_CHUNK = 2048;       // inserts whose buckets are staged per round

// Shared memory: [used bits][touched bits] (when use_smem) | draws[4096] u64 |
// beta1[2048] | beta2[2048] | flag. All threads stage; thread 0 walks. Every
// load on thread 0's critical path is a shared-memory load except the victim
// metadata of an eviction hop (one dependent L2 access per hop).
__global__ void __launch_bounds__(256)
k_cuckoo_walk(CuckooDev d, CuckooState* __restrict__ gst, const uint32_t* __restrict__ beta1,
              const uint32_t* __restrict__ beta2, uint64_t i0, uint64_t n,
              uint32_t* __restrict__ reports, int use_smem) {
    if (!walk_prologue(gst, i0, n)) return;
    extern __shared__ __align__(16) uint32_t sm[];
    const uint64_t slots = uint64_t(d.buckets) * d.depth;
    const uint32_t words = use_smem ? uint32_t((slots + 31) / 32) : 0;
    uint32_t* used_bits = sm;
    uint32_t* touch_bits = sm + words;
    uint64_t* dr = reinterpret_cast<uint64_t*>(sm + ((2 * words + 3) & ~3u));
    uint32_t* sb1 = reinterpret_cast<uint32_t*>(dr + WALK_DRAWS_SMEM);
    uint32_t* sb2 = sb1 + WALK_CHUNK;
    uint32_t* stop = sb2 + WALK_CHUNK;
    __shared__ CuckooState sh_state;
    if (threadIdx.x == 0) {
        sh_state = *gst;
        *stop = 0;
    }
    __syncthreads();
    CuckooState s = sh_state;  // thread 0 mutates its register copy; the others only read it
    if (use_smem) {
        for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) {
            uint32_t v = 0;
            for (uint32_t b = 0; b < 32; ++b) {
                const uint64_t f = uint64_t(w) * 32 + b;
                if (f < slots && d.used[f]) v |= 1u << b;
            }
            used_bits[w] = v;
            touch_bits[w] = 0;
        }
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < s.n_touched; k += blockDim.x) {
            const uint32_t f = d.touched[k];
            atomicOr(&touch_bits[f >> 5], 1u << (f & 31));
        }
    }
    // the next WALK_DRAWS_SMEM draws (nonces rng_block ..) from the global window
    const uint64_t dr_base = s.rng_block;
    const uint64_t avail = (s.draw_base + s.draw_count > s.rng_block) ? s.draw_base + s.draw_count - s.rng_block : 0;
    const uint32_t dr_count = uint32_t(avail < WALK_DRAWS_SMEM ? avail : WALK_DRAWS_SMEM);
    for (uint32_t k = threadIdx.x; k < dr_count; k += blockDim.x) dr[k] = d.draws[dr_base - s.draw_base + k];
    __syncthreads();

    const uint64_t fmask = d.fifo_cap - 1;
    auto is_used = [&](uint32_t f) -> bool {
        return use_smem ? ((used_bits[f >> 5] >> (f & 31)) & 1u) : d.used[f] != 0;
    };
    auto is_touched = [&](uint32_t f) -> bool {
        return use_smem ? ((touch_bits[f >> 5] >> (f & 31)) & 1u) : d.touched_mark[f] == s.batch_id;
    };
    // In shared-memory mode the occupancy and touched maps live in shared memory
    // (global `used` is written back once at the end, `touched_mark` is only the
    // fallback map), so a placement costs no global loads and few stores.
    auto touch = [&](uint32_t f, int64_t org) {
        if (!is_touched(f)) {
            if (use_smem) touch_bits[f >> 5] |= 1u << (f & 31);
            else d.touched_mark[f] = s.batch_id;
            d.touched[s.n_touched++] = f;
        }
        d.origin[f] = org;
    };
    auto free_slot = [&](uint32_t b) -> int {  // cuckoo.cpp:31-35: lowest free slot of bucket b
        if (use_smem && d.depth <= 32) {
            const uint32_t f0 = b * d.depth, w0 = f0 >> 5, sh = f0 & 31;
            uint64_t bits = used_bits[w0];
            if (sh + d.depth > 32) bits |= uint64_t(used_bits[w0 + 1]) << 32;
            const uint64_t mask = d.depth == 32 ? 0xffffffffull : ((1ull << d.depth) - 1);
            const uint64_t freeb = ~(bits >> sh) & mask;
            return freeb ? __ffsll(static_cast<long long>(freeb)) - 1 : -1;
        }
        for (uint32_t sl = 0; sl < d.depth; ++sl)
            if (!is_used(b * d.depth + sl)) return int(sl);
        return -1;
    };
    auto place = [&](uint32_t f, uint32_t b1, uint32_t b2, uint64_t stamp, int64_t org) {  // :37-46
        if (use_smem) used_bits[f >> 5] |= 1u << (f & 31);
        else d.used[f] = 1;
        d.beta1[f] = b1;
        d.beta2[f] = b2;
        d.stamp[f] = stamp;
        d.fifo[stamp & fmask] = int64_t(f);
        touch(f, org);
        s.live++;
    };
    auto clear = [&](uint32_t f) {  // :48-54
        if (use_smem) used_bits[f >> 5] &= ~(1u << (f & 31));
        else d.used[f] = 0;
        d.fifo[d.stamp[f] & fmask] = -1;
        d.beta1[f] = 0;
        d.beta2[f] = 0;
        d.stamp[f] = 0;
        touch(f, -1);
        s.live--;
    };
    auto uniform = [&](uint64_t bound) -> uint64_t {  // rng.cpp:9-16 over DetRng::fill draws
        const uint64_t tail = (~uint64_t(0) % bound + 1) % bound;
        for (;;) {
            const uint64_t v = dr[s.rng_block - dr_base];
            s.rng_block++;
            if (tail == 0 || v <= ~uint64_t(0) - tail) return v % bound;
        }
    };

    if (threadIdx.x == 0) s.status = 0;
    uint64_t i = i0;
    for (uint64_t c0 = i0; c0 < n; c0 += WALK_CHUNK) {
        const uint32_t cn = uint32_t((n - c0) < WALK_CHUNK ? (n - c0) : WALK_CHUNK);
        for (uint32_t k = threadIdx.x; k < cn; k += blockDim.x) {
            sb1[k] = beta1[c0 + k];
            sb2[k] = beta2[c0 + k];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (uint32_t k = 0; k < cn; ++k, ++i) {
                const uint32_t b1 = sb1[k], b2 = sb2[k];
                if (s.rng_block + WALK_MIN_DRAWS > dr_base + dr_count) {
                    s.status = 1;  // host refills / re-stages draws from nonce s.rng_block and resumes at i
                    *stop = 1;
                    break;
                }
                // FIFO ring room for this insert's stamp, before any state changes
                if (s.next_stamp - s.fifo_head >= d.fifo_cap) {
                    while (s.fifo_head < s.next_stamp && d.fifo[s.fifo_head & fmask] < 0) s.fifo_head++;
                    if (s.next_stamp - s.fifo_head >= d.fifo_cap) {
                        s.status = 2;
                        *stop = 1;
                        break;
                    }
                }
                uint32_t stored = 0, dropped = 0, gc = 0, disp = 0;
                s.writes++;                                 // :62
                if (s.live == d.capacity) {                 // :64-69 FIFO GC of the oldest entry
                    while (d.fifo[s.fifo_head & fmask] < 0) s.fifo_head++;
                    clear(uint32_t(d.fifo[s.fifo_head & fmask]));
                    gc = 1;
                }
                const uint64_t stamp = s.next_stamp++;     // :71 (ring room checked above)
                int fs = free_slot(b1);                     // :73-84
                if (fs >= 0) {
                    place(b1 * d.depth + fs, b1, b2, stamp, int64_t(i));
                    stored = 1;
                } else if ((fs = free_slot(b2)) >= 0) {
                    place(b2 * d.depth + fs, b1, b2, stamp, int64_t(i));
                    stored = 1;
                } else {                                    // :86-125 random-walk eviction
                    uint32_t be = uniform(2) == 0 ? b1 : b2;
                    uint32_t c1 = b1, c2 = b2;
                    uint64_t cst = stamp;
                    int64_t corg = int64_t(i);
                    bool carry_incoming = true, incoming_stored = false, done = false;
                    for (uint32_t hops = 0;; ++hops) {
                        const int f2 = free_slot(be);
                        if (f2 >= 0) {
                            place(be * d.depth + f2, c1, c2, cst, corg);
                            if (carry_incoming) incoming_stored = true;
                            stored = incoming_stored;
                            disp = hops;
                            done = true;
                            break;
                        }
                        if (hops == XPIR_MAX_DISPLACEMENTS_DEV) break;
                        const uint32_t vs = uint32_t(uniform(d.depth));
                        const uint32_t vf = be * d.depth + vs;
                        const uint32_t v1 = d.beta1[vf], v2 = d.beta2[vf];
                        const uint64_t vst = d.stamp[vf];
                        const int64_t vo = d.origin[vf];  // loaded beside the metadata (speculative)
                        const int64_t vorg = is_touched(vf) ? vo : -int64_t(vf) - 2;
                        // clear(vf) then place(vf, carry) (:110-113): the slot stays occupied and
                        // live is unchanged, so only the FIFO, metadata and origin change.
                        d.fifo[vst & fmask] = -1;
                        d.beta1[vf] = c1;
                        d.beta2[vf] = c2;
                        d.stamp[vf] = cst;
                        d.fifo[cst & fmask] = int64_t(vf);
                        touch(vf, corg);
                        if (carry_incoming) incoming_stored = true;
                        c1 = v1;
                        c2 = v2;
                        cst = vst;
                        corg = vorg;
                        carry_incoming = false;
                        be = v1 == be ? v2 : v1;            // :118
                    }
                    if (!done) {                            // :122-125
                        disp = XPIR_MAX_DISPLACEMENTS_DEV;
                        dropped = 1;
                        stored = incoming_stored;
                    }
                }
                if (reports) reinterpret_cast<uint4*>(reports)[i] = make_uint4(stored, dropped, gc, disp);
            }
        }
        __syncthreads();
        if (*stop) break;
    }
    if (use_smem) {  // occupancy map back to the global byte array
        __syncthreads();
        for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) {
            const uint32_t v = used_bits[w];
            const uint64_t f0 = uint64_t(w) * 32;
            if (f0 + 32 <= slots && (reinterpret_cast<uintptr_t>(d.used + f0) & 15) == 0) {
                uint32_t b[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    b[k] = ((v >> (4 * k)) & 1u) | ((v >> (4 * k + 1)) & 1u) << 8 | ((v >> (4 * k + 2)) & 1u) << 16 |
                           ((v >> (4 * k + 3)) & 1u) << 24;
                reinterpret_cast<uint4*>(d.used + f0)[0] = make_uint4(b[0], b[1], b[2], b[3]);
                reinterpret_cast<uint4*>(d.used + f0)[1] = make_uint4(b[4], b[5], b[6], b[7]);
            } else {
                for (uint32_t k = 0; k < 32 && f0 + k < slots; ++k) d.used[f0 + k] = (v >> k) & 1u;
            }
        }
    }
    if (threadIdx.x == 0) {
        s.resume_at = i;
        *gst = s;
    }
}

// ---- bucket-range payload shards ("payload scatter goes to the GPU
// owning each bucket range"). The walk is replicated, so every shard knows every
// touched slot and its origin; a shard only materialises the slots of its range.
__global__ void k_cuckoo_gather_sharded(CuckooDev d, uint32_t n_touched, uint64_t f_lo, uint64_t f_hi,
                                        const uint8_t* __restrict__ table, ShardMap map,
                                        CuckooState* __restrict__ dev_state, uint32_t cap) {
    if (dev_state) {  // the walk ran on device: its count, unless it paused (host finishes it)
        if (dev_state->status || !dev_state->walked) return;
        n_touched = dev_state->n_touched;
        if (n_touched > cap) {  // staging too small: the host redoes gather + scatter
            if (blockIdx.x == 0 && threadIdx.x == 0) dev_state->status = 3;
            return;
        }
    }
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_touched; k += nw) {
        const uint32_t f = d.touched[k];
        if (f < f_lo || f >= f_hi) continue;
        const int64_t o = d.origin[f];
        if (o > -2) continue;
        const uint64_t src = uint64_t(-o - 2);  // pre-round slot of the moved item
        const uint8_t* s = nullptr;
        if (src >= f_lo && src < f_hi) {
            s = table + (src - f_lo) * d.item;
        } else {
            const uint32_t b = uint32_t(src / d.depth);
            for (uint32_t g = 0; g < map.n; ++g)
                if (b >= map.lo[g] && b < map.lo[g + 1]) s = map.data[g] + (src - uint64_t(map.lo[g]) * d.depth) * d.item;
        }
        uint8_t* gdst = d.gather + uint64_t(k) * d.item;
        if ((d.item & 15) == 0) {
            for (uint64_t b = lane * 16; b < d.item; b += 32 * 16)
                *reinterpret_cast<uint4*>(gdst + b) = s ? *reinterpret_cast<const uint4*>(s + b) : make_uint4(0, 0, 0, 0);
        } else {
            for (uint64_t b = lane; b < d.item; b += 32) gdst[b] = s ? s[b] : 0;
        }
    }
}

__global__ void k_cuckoo_scatter_sharded(CuckooDev d, uint32_t n_touched, uint64_t f_lo, uint64_t f_hi,
                                         uint8_t* __restrict__ table, const uint8_t* __restrict__ payload,
                                         uint32_t batch_id, const CuckooState* __restrict__ dev_state) {
    if (dev_state) {  // the walk ran on device: its count and batch, unless it paused / overflowed
        if (dev_state->status) return;
        n_touched = dev_state->n_touched;
        batch_id = dev_state->batch_id;
    }
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_touched; k += nw) {
        const uint32_t f = d.touched[k];
        if (lane == 0) d.mod_batch[f] = batch_id;  // replicated metadata: every shard records it
        if (f < f_lo || f >= f_hi) continue;
        const int64_t o = d.origin[f];
        uint8_t* dst = table + (f - f_lo) * d.item;
        const uint8_t* src = o >= 0 ? payload + uint64_t(o) * d.item
                            : o == -1 ? nullptr
                                      : d.gather + uint64_t(k) * d.item;
        if ((d.item & 15) == 0) {
            for (uint64_t b = lane * 16; b < d.item; b += 32 * 16)
                *reinterpret_cast<uint4*>(dst + b) =
                    src ? *reinterpret_cast<const uint4*>(src + b) : make_uint4(0, 0, 0, 0);
        } else {
            for (uint64_t b = lane; b < d.item; b += 32) dst[b] = src ? src[b] : 0;
        }
    }
}

cudaError_t launch_cuckoo_gather_sharded(const CuckooDev& d, const CuckooState* st, uint32_t lo, uint32_t hi,
                                         const uint8_t* table, const ShardMap& map, cudaStream_t s,
                                         CuckooState* dev_state, uint32_t max_touched, uint32_t cap) {
    const uint32_t nt = dev_state ? max_touched : st->n_touched;
    if (!nt) return cudaSuccess;
    // warp per slot, grid-stride; with the count on device the grid is sized for the
    // bound, and a batch with nothing to move returns from every block at once
    uint32_t g = (nt + 7) / 8;
    if (g > (dev_state ? 148 * 4 : 148 * 16)) g = dev_state ? 148 * 4 : 148 * 16;
    k_cuckoo_gather_sharded<<<g, 256, 0, s>>>(d, st->n_touched, uint64_t(lo) * d.depth, uint64_t(hi) * d.depth,
                                              table, map, dev_state, cap);
    return cudaGetLastError();
}

cudaError_t launch_cuckoo_scatter_sharded(const CuckooDev& d, const CuckooState* st, uint32_t lo, uint32_t hi,
                                          uint8_t* table, const uint8_t* payload, cudaStream_t s,
                                          const CuckooState* dev_state, uint32_t max_touched) {
    const uint32_t nt = dev_state ? max_touched : st->n_touched;
    if (!nt) return cudaSuccess;
    uint32_t g = (nt + 7) / 8;
    if (g > 148 * 16) g = 148 * 16;
    k_cuckoo_scatter_sharded<<<g, 256, 0, s>>>(d, st->n_touched, uint64_t(lo) * d.depth, uint64_t(hi) * d.depth,
                                               table, payload, st->batch_id, dev_state);
    return cudaGetLastError();
}

// Incremental seal (ServerCore::seal_epoch, server.cpp:75-81, without the full
// copy): bring a sealed image last synchronised at round `since` up to date by
// copying only the slots a later round modified. One warp per slot range.
// slots [f_lo, f_lo + slots) of the logical table; table and img hold exactly them
__global__ void k_seal_incremental(const uint32_t* __restrict__ mod_batch, uint64_t f_lo, uint64_t slots,
                                   uint64_t item, uint32_t since, const uint8_t* __restrict__ table,
                                   uint8_t* __restrict__ img) {
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t f = warp; f < slots; f += nwarps) {
        if (mod_batch[f_lo + f] <= since) continue;
        const uint8_t* s = table + f * item;
        uint8_t* dst = img + f * item;
        if ((item & 15) == 0) {
            for (uint64_t b = lane * 16; b < item; b += 32 * 16)
                *reinterpret_cast<uint4*>(dst + b) = *reinterpret_cast<const uint4*>(s + b);
        } else {
            for (uint64_t b = lane; b < item; b += 32) dst[b] = s[b];
        }
    }
}

cudaError_t launch_seal_incremental(const CuckooDev& d, uint32_t lo, uint32_t hi, uint32_t since,
                                    const uint8_t* table, uint8_t* img, int num_sms, cudaStream_t s) {
    const uint64_t slots = uint64_t(hi - lo) * d.depth;
    if (!slots) return cudaSuccess;
    uint64_t g = (slots * 32 + 255) / 256;
    if (g > uint64_t(num_sms) * 16) g = uint64_t(num_sms) * 16;
    k_seal_incremental<<<uint32_t(g), 256, 0, s>>>(d.mod_batch, uint64_t(lo) * d.depth, slots, d.item, since,
                                                   table, img);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static ChaChaKey host_key(const uint8_t* key32, uint64_t nonce) { return chacha_key(key32, nonce); }

cudaError_t launch_keystream(const uint8_t* key_host32, uint64_t nonce, uint64_t byte_offset,
                             uint8_t* out, uint64_t len, cudaStream_t s) {
    if (len == 0) return cudaSuccess;
    const uint64_t nblk = (byte_offset + len + 63) / 64 - byte_offset / 64;
    uint64_t g = (nblk + 255) / 256;
    if (g > 148 * 64) g = 148 * 64;
    k_keystream<<<uint32_t(g), 256, 0, s>>>(host_key(key_host32, nonce), byte_offset, out, len);
    return cudaGetLastError();
}

cudaError_t launch_keystream_rows(const uint8_t* key_host32, uint64_t nonce0, uint32_t rows,
                                  uint64_t len, uint8_t* out, uint64_t row_stride, cudaStream_t s) {
    const uint64_t n = uint64_t(rows) * ((len + 63) / 64);
    if (n == 0) return cudaSuccess;
    k_keystream_rows<<<uint32_t((n + 127) / 128), 128, 0, s>>>(host_key(key_host32, 0), nonce0, rows,
                                                               len, out, row_stride);
    return cudaGetLastError();
}

cudaError_t launch_draws(const uint8_t* key_host32, uint64_t nonce0, uint32_t count, uint64_t* out,
                         cudaStream_t s) {
    if (!count) return cudaSuccess;
    k_draws<<<(count + 127) / 128, 128, 0, s>>>(host_key(key_host32, 0), nonce0, count, out);
    return cudaGetLastError();
}

cudaError_t launch_prf(uint64_t k0, uint64_t k1, const uint64_t* in, uint64_t n, uint64_t modulus,
                       uint64_t* out, uint32_t* out32, cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_prf<<<uint32_t((n + 127) / 128), 128, 0, s>>>(k0, k1, in, n, modulus, out, out32);
    return cudaGetLastError();
}

cudaError_t launch_interest(const uint8_t* id16_host, const uint64_t* seqs, uint64_t n, uint32_t h,
                            uint32_t m_bits, uint32_t* pos_out, unsigned long long* words,
                            cudaStream_t s) {
    const uint64_t t = n * h;
    if (!t) return cudaSuccess;
    Id16 id;
    std::memcpy(id.b, id16_host, 16);
    // One thread per (write, hash): short-lived blocks, so the write round's table
    // chain (its cooperative prefix on a higher-priority stream) takes SMs as they
    // retire instead of waiting for a resident grid-stride wave to drain (config 3
    // round as one graph: 0.157 -> 0.127 ms). 56 KiB of (unused) dynamic shared
    // memory per block caps the kernel at 4 blocks per SM, leaving thread slots for
    // the chain from the start: 0.127 -> 0.119 ms (ALU-bound at 16 warps per SM).
    constexpr int kOccupancyCapSmem = 56 * 1024;
    static std::atomic<uint64_t> attr_set{0};  // per device (the attribute is per context)
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !((attr_set.load() >> dev) & 1)) {
        cudaError_t e = cudaFuncSetAttribute(k_interest, cudaFuncAttributeMaxDynamicSharedMemorySize, kOccupancyCapSmem);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(uint64_t(1) << dev);
    }
    const uint64_t want = (t + 127) / 128, cap = 0x7fffffffull;
    k_interest<<<uint32_t(want < cap ? want : cap), 128, kOccupancyCapSmem, s>>>(id, seqs, n, h, m_bits, pos_out,
                                                                                 words, 2u);
    return cudaGetLastError();
}

cudaError_t launch_bloom_item(const uint8_t* item_dev, uint32_t len, uint32_t h, uint32_t m_bits,
                              uint32_t* out, cudaStream_t s) {
    if (!h) return cudaSuccess;
    k_bloom_item<<<(h + 127) / 128, 128, 0, s>>>(item_dev, len, h, m_bits, out);
    return cudaGetLastError();
}

cudaError_t launch_absorb(const uint32_t* pos, uint64_t n, uint32_t m_bits,
                          unsigned long long* words, unsigned long long* first_bad, cudaStream_t s) {
    if (!n) return cudaSuccess;
    const unsigned long long init = ~0ull;
    cudaError_t e = cudaMemcpyAsync(first_bad, &init, 8, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    const uint32_t g = uint32_t((n + 255) / 256);
    k_absorb_check<<<g, 256, 0, s>>>(pos, n, m_bits, first_bad);
    k_absorb<<<g, 256, 0, s>>>(pos, n, first_bad, words);
    return cudaGetLastError();
}

// positions already checked against m_bits (host): OR them in, no limit
__global__ void k_absorb_all(const uint32_t* __restrict__ pos, uint64_t n, unsigned long long* __restrict__ words) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n) atomicOr(words + (pos[t] >> 6), 1ull << (pos[t] & 63));
}

cudaError_t launch_absorb_unchecked(const uint32_t* pos, uint64_t n, unsigned long long* words, cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_absorb_all<<<uint32_t((n + 255) / 256), 256, 0, s>>>(pos, n, words);
    return cudaGetLastError();
}

// FIFO ring growth: every live slot re-entered at stamp & (new_cap - 1)
__global__ void k_fifo_rebuild(CuckooDev d, int64_t* __restrict__ ring, uint64_t cap_mask) {
    const uint64_t slots = uint64_t(d.buckets) * d.depth;
    for (uint64_t f = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; f < slots; f += uint64_t(gridDim.x) * blockDim.x)
        if (d.used[f]) ring[d.stamp[f] & cap_mask] = int64_t(f);
}

cudaError_t launch_fifo_rebuild(const CuckooDev& d, int64_t* ring, uint64_t cap, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(ring, 0xff, cap * 8, s);  // -1: no entry
    if (e != cudaSuccess) return e;
    const uint64_t slots = uint64_t(d.buckets) * d.depth;
    k_fifo_rebuild<<<uint32_t(std::min<uint64_t>((slots + 255) / 256, 148 * 8)), 256, 0, s>>>(d, ring, cap - 1);
    return cudaGetLastError();
}

cudaError_t launch_beta_check(const uint32_t* b1, const uint32_t* b2, uint64_t n, uint32_t buckets,
                              unsigned long long* first_bad, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(first_bad, 0xff, 8, s);
    if (e != cudaSuccess || !n) return e;
    k_beta_check<<<uint32_t((n + 255) / 256), 256, 0, s>>>(b1, b2, n, buckets, first_bad);
    return cudaGetLastError();
}

cudaError_t launch_cuckoo_walk(const CuckooDev& d, CuckooState* st, const uint32_t* beta1,
                               const uint32_t* beta2, uint64_t i0, uint64_t n, uint32_t* reports,
                               cudaStream_t s) {
    // XPIR_CUCKOO_WALK (A/B runs): "1" single-thread walk, "2" warp walk with global
    // victim metadata, unset/other: on-chip eviction control when the table fits
    static const int choice = [] {
        const char* e = std::getenv("XPIR_CUCKOO_WALK");
        return e ? e[0] - '0' : 0;
    }();
    // a batch small against the table (e.g. one ServerCore::apply_write) skips the
    // O(slots) on-chip staging of the other variants: global-map warp walk (a walk
    // that starts where the parallel prefix stopped is sized by the whole batch)
    const uint64_t slots = uint64_t(d.buckets) * d.depth;
    const uint64_t span = i0 == WALK_FROM_STATE ? n : n - i0;
    const bool small = span * 256 < slots;
    if (choice != 1 && choice != 2 && !small && walk_x_supported(d))
        return launch_cuckoo_walk_x(d, st, beta1, beta2, i0, n, reports, s);
    if (choice != 1 && walk_w_supported(d))
        return launch_cuckoo_walk_w(d, st, beta1, beta2, i0, n, reports, s, small);
    const bool use_smem = slots <= WALK_SMEM_MAX_SLOTS && !small;
    const size_t words = use_smem ? (slots + 31) / 32 : 0;
    const size_t smem = ((2 * words + 3) & ~size_t(3)) * 4 + WALK_DRAWS_SMEM * 8 + 2 * WALK_CHUNK * 4 + 16;
    cudaError_t e = cudaFuncSetAttribute(k_cuckoo_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    k_cuckoo_walk<<<1, 256, smem, s>>>(d, st, beta1, beta2, i0, n, reports, use_smem ? 1 : 0);
    return cudaGetLastError();
}


}  // namespace xpir

// K1 (large batches): the "four Russians" byte-table scan on sm_100a.
//
// Bit-exact restatement of pir::answer_batch (pir.cpp:41-52) for B >= ~128:
//   out_r ^= XOR_{j < N_g : bit j of q_r} bucket_j
// Query byte g of request r is exactly the 8-bit selection of buckets 8g..8g+7
// (bit j at byte j/8, position j%8 — pir.hpp:25), so for every 128-byte column
// slice of the shard the CTA builds in shared memory the 256-row table
//     T_g[x] = XOR_{i : bit i of x} bucket_{8g+i}[slice]
// and each request does ONE 16-byte LDS + 4 XORs per 8 buckets (8x fewer XORs
// than the dense masked select-XOR). Rows are 128 bytes and a quarter-warp
// (8 lanes x 16 B) reads one row per LDS.128 phase, so any index pattern is
// bank-conflict-free. Shared-memory bandwidth (128 B/clk/SM) is the bound.
//
// Layouts:
//   db   shard, bucket-major (N_g x S bytes), S % 128 == 0
//   qT   group-major query bytes: qT[g*qstride + r] = q_r[g] (shard-relative g),
//        qstride % 16 == 0, rows allocated up to round16(n_groups)
//   out  B x S, pre-initialised (zero or mask pad), XOR-accumulated here
//
// Work decomposition: (request tile rt of Rc requests) x (column tile c of 128 B)
// x (group g), flattened and split evenly over a persistent grid (one 512-thread
// CTA per SM); accumulators live in registers and are flushed with 64-bit
// atomicXor at segment ends. Thread (warp w, quarter qq, lane8 l) owns requests
//   r_local(i) = (w*4 + qq)*RPT + i,  i < RPT,   bytes [c*128 + l*16, +16).
// Warps 0..7 build the table (32 rows each: Gray code over buckets 0..4, masks
// for buckets 5..7); everyone looks up. One __syncthreads per group; tables and
// staged chunks (16 groups of query bytes + 128 buckets x 128 B) are
// double-buffered with cp.async.
#include <cuda_runtime.h>

#include <cstdint>

#include "prims.cuh"
#include "ptx.cuh"
#include "scan.cuh"

namespace xpir {

using namespace ptx;

constexpr int M4_CHUNK_G = 16;
constexpr int M4_TAB_BYTES = 256 * 128;
constexpr int M4_DBS_BYTES = M4_CHUNK_G * 8 * 128;
constexpr int M4_BUILD_WARPS = 8;

template <int NT, int RPT>
struct M4Layout {
    static constexpr int NW = NT / 32;
    static constexpr int Rc = NW * 4 * RPT;
    static constexpr int QS_BYTES = M4_CHUNK_G * Rc;
    static constexpr int OFF_TAB = 0;
    static constexpr int OFF_QS = 4 * M4_TAB_BYTES;  // [2 phases][2 tables]
    static constexpr int OFF_DBS = OFF_QS + 2 * QS_BYTES;
    static constexpr int SMEM = OFF_DBS + 2 * M4_DBS_BYTES;
};

template <int RPT>
struct IdxVec;
template <>
struct IdxVec<16> {
    uint32_t w[4];
    __device__ __forceinline__ void load(uint32_t a) {
        const uint4 v = lds128(a);
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    }
};
template <>
struct IdxVec<8> {
    uint32_t w[2];
    __device__ __forceinline__ void load(uint32_t a) {
        const uint2 v = lds64(a);
        w[0] = v.x; w[1] = v.y;
    }
};
template <>
struct IdxVec<4> {
    uint32_t w[1];
    __device__ __forceinline__ void load(uint32_t a) { w[0] = lds32(a); }
};

template <int NT, int RPT>
__global__ void __launch_bounds__(NT, 1)
k_scan_m4rm(const uint8_t* __restrict__ db, uint32_t nb, uint32_t S, const uint8_t* __restrict__ qT,
            uint64_t qstride, uint32_t B, uint8_t* __restrict__ out, uint32_t n_ctiles,
            uint32_t n_groups, uint64_t total_work) {
    using L = M4Layout<NT, RPT>;
    static_assert(L::NW >= 2 * M4_BUILD_WARPS, "need 8 builder warps per table of a pair");
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int qq = lane >> 3, l8 = lane & 7;
    const int slot0 = (warp * 4 + qq) * RPT;  // first request slot of this thread

    // builder role (warps 0..7): word column `lane`, rows [32*warp, 32*warp+32)
    const bool builder = warp < 2 * M4_BUILD_WARPS;
    const uint32_t hm5 = 0u - ((warp >> 0) & 1u), hm6 = 0u - ((warp >> 1) & 1u),
                   hm7 = 0u - ((warp >> 2) & 1u);

    const uint64_t w0 = total_work * blockIdx.x / gridDim.x;
    const uint64_t w1 = total_work * (blockIdx.x + 1) / gridDim.x;

    for (uint64_t u = w0; u < w1;) {
        const uint32_t p = uint32_t(u / n_groups);
        const uint32_t gs = uint32_t(u - uint64_t(p) * n_groups);
        const uint64_t pend = uint64_t(p + 1) * n_groups;
        const uint32_t ge = uint32_t((w1 < pend ? w1 : pend) - uint64_t(p) * n_groups);
        u = uint64_t(p) * n_groups + ge;
        const uint32_t rt = p / n_ctiles, c = p - rt * n_ctiles;
        const uint32_t r_base = rt * L::Rc;
        const uint32_t nvalid = min(uint32_t(L::Rc), B - r_base);
        const bool active = uint32_t(warp * 4 * RPT) < nvalid;  // warp-uniform

        uint4 acc[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) acc[i] = make_uint4(0, 0, 0, 0);

        auto stage = [&](uint32_t kc, int b) {
            const uint32_t qdst = sbase + L::OFF_QS + b * L::QS_BYTES;
            constexpr int QCH = L::Rc / 16;  // 16-byte chunks per group row
            for (int k = tid; k < M4_CHUNK_G * QCH; k += NT) {
                const uint32_t gl = k / QCH, ch = k - gl * QCH;
                const uint64_t col = uint64_t(r_base) + ch * 16;
                const bool ok = col < qstride;
                const uint8_t* src = qT + (uint64_t(kc) * M4_CHUNK_G + gl) * qstride + (ok ? col : 0);
                cp_async16(qdst + gl * L::Rc + ch * 16, src, ok ? 16u : 0u);
            }
            const uint32_t ddst = sbase + L::OFF_DBS + b * M4_DBS_BYTES;
            for (int k = tid; k < M4_CHUNK_G * 8 * 8; k += NT) {
                const uint32_t bl = k >> 3, part = k & 7;
                const uint32_t bucket = kc * 128 + bl;
                const bool ok = bucket < nb;
                const uint8_t* src = db + (ok ? uint64_t(bucket) * S : 0) + uint64_t(c) * 128 + part * 16;
                cp_async16(ddst + bl * 128 + part * 16, src, ok ? 16u : 0u);
            }
        };

        const uint32_t kc0 = gs / M4_CHUNK_G, kc1 = (ge + M4_CHUNK_G - 1) / M4_CHUNK_G;
        stage(kc0, 0);
        cp_async_commit();
        int tb = 0;
        for (uint32_t kc = kc0; kc < kc1; ++kc) {
            const int b = (kc - kc0) & 1;
            if (kc + 1 < kc1) {
                stage(kc + 1, b ^ 1);
                cp_async_commit();
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const uint32_t qbuf = sbase + L::OFF_QS + b * L::QS_BYTES;
            const uint32_t dbuf = sbase + L::OFF_DBS + b * M4_DBS_BYTES;
            const uint32_t g0 = kc * M4_CHUNK_G;
            const uint32_t glo = (gs > g0 ? gs : g0) - g0;
            const uint32_t ghi = (ge < g0 + M4_CHUNK_G ? ge : g0 + M4_CHUNK_G) - g0;
            // Groups are processed in pairs: warps 0..7 build T_g, warps 8..15 build
            // T_{g+1}, one barrier, then every request does two lookups folded with
            // one 3-input XOR per word (acc ^= T_g[x] ^ T_{g+1}[y]).
#pragma unroll 1
            for (uint32_t gl = glo; gl < ghi; gl += 2) {
                const bool pair = gl + 1 < ghi;  // uniform across the CTA
                const uint32_t tabA = sbase + L::OFF_TAB + tb * 2 * M4_TAB_BYTES;
                if (builder && (warp < M4_BUILD_WARPS || pair)) {
                    const uint32_t g = gl + (warp >> 3);
                    const uint32_t src = dbuf + g * 8 * 128 + lane * 4;
                    uint32_t bk[5];
#pragma unroll
                    for (int k = 0; k < 5; ++k) bk[k] = lds32(src + k * 128);
                    uint32_t h = (lds32(src + 5 * 128) & hm5) ^ (lds32(src + 6 * 128) & hm6) ^
                                 (lds32(src + 7 * 128) & hm7);
                    const uint32_t row0 = tabA + (warp >> 3) * M4_TAB_BYTES + ((warp & 7) * 32) * 128 + lane * 4;
                    sts32(row0, h);
#pragma unroll
                    for (int k = 1; k < 32; ++k) {
                        h ^= bk[(k & 1) ? 0 : (k & 2) ? 1 : (k & 4) ? 2 : (k & 8) ? 3 : 4];  // ctz(k)
                        sts32(row0 + uint32_t(k ^ (k >> 1)) * 128, h);
                    }
                }
                __syncthreads();
                if (active) {
                    const uint32_t rowA = tabA + l8 * 16;
                    IdxVec<RPT> ia;
                    ia.load(qbuf + gl * L::Rc + slot0);
                    if (pair) {
                        const uint32_t rowB = rowA + M4_TAB_BYTES;
                        IdxVec<RPT> ib;
                        ib.load(qbuf + (gl + 1) * L::Rc + slot0);
#pragma unroll
                        for (int i = 0; i < RPT; ++i) {
                            const uint32_t xa = (ia.w[i >> 2] >> (8 * (i & 3))) & 0xffu;
                            const uint32_t xb = (ib.w[i >> 2] >> (8 * (i & 3))) & 0xffu;
                            const uint4 va = lds128(rowA + xa * 128);
                            const uint4 vb = lds128(rowB + xb * 128);
                            acc[i].x ^= va.x ^ vb.x;
                            acc[i].y ^= va.y ^ vb.y;
                            acc[i].z ^= va.z ^ vb.z;
                            acc[i].w ^= va.w ^ vb.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < RPT; ++i) {
                            const uint32_t xa = (ia.w[i >> 2] >> (8 * (i & 3))) & 0xffu;
                            const uint4 va = lds128(rowA + xa * 128);
                            acc[i].x ^= va.x;
                            acc[i].y ^= va.y;
                            acc[i].z ^= va.z;
                            acc[i].w ^= va.w;
                        }
                    }
                }
                tb ^= 1;
            }
            __syncthreads();  // buffers b are re-staged next iteration
        }
        if (active) {
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const uint32_t rl = slot0 + i;
                if (rl < nvalid) {
                    uint8_t* o = out + uint64_t(r_base + rl) * S + uint64_t(c) * 128 + l8 * 16;
                    red_xor64(o, uint64_t(acc[i].y) << 32 | acc[i].x);
                    red_xor64(o + 8, uint64_t(acc[i].w) << 32 | acc[i].z);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Query layout kernels for the M4RM path.
// k_expand_T: qT[(k)*qstride + r] = prng_expand(seed_r)[byte_lo + k], k < nbytes.
//   Consecutive threads take consecutive requests of the same keystream block,
//   so each of the 64 byte stores per thread is a coalesced 32-byte warp store.
// k_transpose_q: rows q[r*q_stride + byte_lo + k] -> qT (32x32 smem tiles).
// ---------------------------------------------------------------------------
// layout 2 (k_scan_m4rm_q9, kernel 8): byte k = 9p + b of pair p; b < 8 goes to
// byte b & 3 of the 32-bit word of set 2p + b/4 (one word per request and set,
// [set][request]), b = 8 (the pair's ninth index bits) to the plane after the
// words: hi_off + p * qstride + r.
__device__ __forceinline__ uint64_t qidx(uint64_t k, uint32_t r, uint64_t qstride, int layout, uint64_t hi_off) {
    if (layout == 0) return k * qstride + r;
    const uint64_t p = k / 9, b = k - 9 * p;
    return b < 8 ? (2 * p + (b >> 2)) * 4 * qstride + uint64_t(r) * 4 + (b & 3) : hi_off + p * qstride + r;
}

__global__ void __launch_bounds__(128)
k_expand_T(const uint8_t* __restrict__ seeds, uint32_t B, uint64_t byte_lo, uint64_t nbytes,
           uint8_t* __restrict__ qT, uint64_t qstride, int layout, uint64_t hi_off) {
    const uint64_t blk_lo = byte_lo / 64;
    const uint64_t nblk = (byte_lo + nbytes + 63) / 64 - blk_lo;
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t Bp = (B + 31) & ~31u;
    if (t >= Bp * nblk) return;
    const uint64_t kb = t / Bp;
    const uint32_t r = uint32_t(t - kb * Bp);
    if (r >= B) return;
    const uint64_t blk = blk_lo + kb;
    ChaChaKey key = chacha_key(seeds + uint64_t(r) * 32, 0);
    uint32_t ks[16];
    chacha20_block(key, blk, ks);
    const int64_t base = int64_t(blk * 64) - int64_t(byte_lo);
#pragma unroll
    for (int j = 0; j < 64; ++j) {
        const int64_t k = base + j;
        if (k >= 0 && uint64_t(k) < nbytes)
            qT[qidx(uint64_t(k), r, qstride, layout, hi_off)] = uint8_t(ks[j >> 2] >> (8 * (j & 3)));
    }
}

// Layout 2 straight from the keystream: a thread owns request r and a chunk of
// 576 window bytes (64 pairs = 9 ChaCha blocks, the period where pairs and blocks
// realign). Whole chunks of a 64-byte-aligned window write each set's 32-bit word
// with one funnel shift (the word straddling a block boundary takes the previous
// block's last word) and each pair's ninth-bit byte; the rest go byte by byte.
__global__ void __launch_bounds__(128)
k_expand_q9(const uint8_t* __restrict__ seeds, uint32_t B, uint64_t byte_lo, uint64_t nbytes,
            uint8_t* __restrict__ qT, uint64_t qstride, uint64_t hi_off) {
    const uint64_t nch = (nbytes + 575) / 576;
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t Bp = (B + 31) & ~31u;
    if (t >= Bp * nch) return;
    const uint64_t c = t / Bp;
    const uint32_t r = uint32_t(t - c * Bp);
    if (r >= B) return;
    ChaChaKey key = chacha_key(seeds + uint64_t(r) * 32, 0);
    const uint64_t k0 = 576 * c;
    if ((byte_lo & 63) == 0 && k0 + 576 <= nbytes) {
        const uint64_t blk0 = (byte_lo + k0) / 64;
        uint8_t* const lo_base = qT + uint64_t(128 * c) * 4 * qstride + uint64_t(r) * 4;
        uint8_t* const hi_base = qT + hi_off + uint64_t(64 * c) * qstride + r;
        uint32_t prev = 0;
#pragma unroll
        for (int b = 0; b < 9; ++b) {
            uint32_t ks[16];
            chacha20_block(key, blk0 + b, ks);
#pragma unroll
            for (int s = 0; s < 128; ++s) {
                const int o = 9 * (s >> 1) + 4 * (s & 1), w = o >> 2, sh = 8 * (o & 3);
                const int wl = w + (sh ? 1 : 0);  // last keystream word the set needs
                if (wl / 16 != b) continue;
                const uint32_t a = (w / 16 == b) ? ks[w & 15] : prev;
                const uint32_t v = sh ? __funnelshift_r(a, ks[wl & 15], sh) : a;
                *reinterpret_cast<uint32_t*>(lo_base + uint64_t(s) * 4 * qstride) = v;
            }
#pragma unroll
            for (int p = 0; p < 64; ++p) {
                const int o = 9 * p + 8, w = o >> 2;
                if (w / 16 != b) continue;
                hi_base[uint64_t(p) * qstride] = uint8_t(ks[w & 15] >> (8 * (o & 3)));
            }
            prev = ks[15];
        }
        return;
    }
    const uint64_t k1 = k0 + 576 < nbytes ? k0 + 576 : nbytes;
    for (uint64_t blk = (byte_lo + k0) / 64; blk * 64 < byte_lo + k1; ++blk) {
        uint32_t ks[16];
        chacha20_block(key, blk, ks);
        const int64_t base = int64_t(blk * 64) - int64_t(byte_lo);
#pragma unroll
        for (int j = 0; j < 64; ++j) {
            const int64_t k = base + j;
            if (k >= int64_t(k0) && uint64_t(k) < k1)
                qT[qidx(uint64_t(k), r, qstride, 2, hi_off)] = uint8_t(ks[j >> 2] >> (8 * (j & 3)));
        }
    }
}

__global__ void k_transpose_q(const uint8_t* __restrict__ q, uint64_t q_stride, uint64_t byte_lo,
                              uint64_t nbytes, uint32_t B, uint8_t* __restrict__ qT, uint64_t qstride, int layout,
                              uint64_t hi_off) {
    __shared__ uint8_t tile[32][33];
    const uint64_t k0 = uint64_t(blockIdx.x) * 32;  // byte (group) tile
    const uint32_t r0 = blockIdx.y * 32;            // request tile
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const uint32_t r = r0 + y;
        const uint64_t k = k0 + threadIdx.x;
        tile[y][threadIdx.x] = (r < B && k < nbytes) ? q[uint64_t(r) * q_stride + byte_lo + k] : uint8_t(0);
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const uint64_t k = k0 + y;
        const uint32_t r = r0 + threadIdx.x;
        if (k < nbytes && r < B) qT[qidx(k, r, qstride, layout, hi_off)] = tile[threadIdx.x][y];
    }
}

// Layout 2 from caller rows: a block transposes 32 pairs (288 query bytes) of 32
// requests through shared memory and writes whole 32-bit set words (one coalesced
// 128-byte store per set and warp) and the pairs' ninth-bit bytes. Row stride 292
// bytes = 73 words: the column reads of the write phase are bank-conflict-free.
__global__ void __launch_bounds__(256)
k_transpose_q9(const uint8_t* __restrict__ q, uint64_t q_stride, uint64_t byte_lo, uint64_t nbytes, uint32_t B,
               uint8_t* __restrict__ qT, uint64_t qstride, uint64_t hi_off) {
    __shared__ uint8_t tile[32][292];
    const uint64_t k0 = uint64_t(blockIdx.x) * 288;
    const uint32_t r0 = blockIdx.y * 32;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int idx = tid; idx < 32 * 288; idx += 256) {
        const int row = idx / 288, k = idx - row * 288;
        const uint32_t r = r0 + row;
        tile[row][k] = (r < B && k0 + k < nbytes) ? q[uint64_t(r) * q_stride + byte_lo + k0 + k] : uint8_t(0);
    }
    __syncthreads();
    const uint64_t n_pairs = (nbytes + 8) / 9;
    const uint32_t tx = threadIdx.x, r = r0 + tx;
    if (r >= B) return;
    for (int s = threadIdx.y; s < 64; s += 8) {
        const int c = 9 * (s >> 1) + 4 * (s & 1);
        const uint64_t gp = uint64_t(blockIdx.x) * 32 + (s >> 1);
        if (gp >= n_pairs) break;
        const uint32_t w = uint32_t(tile[tx][c]) | uint32_t(tile[tx][c + 1]) << 8 | uint32_t(tile[tx][c + 2]) << 16 |
                           uint32_t(tile[tx][c + 3]) << 24;
        *reinterpret_cast<uint32_t*>(qT + (2 * gp + (s & 1)) * 4 * qstride + uint64_t(r) * 4) = w;
    }
    for (int p = threadIdx.y; p < 32; p += 8) {
        const uint64_t gp = uint64_t(blockIdx.x) * 32 + p;
        if (gp >= n_pairs) break;
        qT[hi_off + gp * qstride + r] = tile[tx][9 * p + 8];
    }
}

// ---------------------------------------------------------------------------
template <int NT, int RPT>
static cudaError_t launch_m4(const M4Args& a, int ctas_per_sm, int num_sms) {
    using L = M4Layout<NT, RPT>;
    cudaError_t e = cudaFuncSetAttribute(k_scan_m4rm<NT, RPT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t n_ctiles = a.S / 128;
    const uint32_t n_rtiles = (a.B + L::Rc - 1) / L::Rc;
    const uint32_t n_groups = (a.nb + 7) / 8;
    const uint64_t total = uint64_t(n_ctiles) * n_rtiles * n_groups;
    uint64_t grid = uint64_t(num_sms) * (ctas_per_sm > 0 ? ctas_per_sm : 1);
    const uint64_t max_grid = (total + 7) / 8;  // at least ~8 groups of work per CTA
    if (grid > max_grid) grid = max_grid > 0 ? max_grid : 1;
    k_scan_m4rm<NT, RPT><<<dim3(uint32_t(grid)), NT, L::SMEM, a.stream>>>(
        a.db, a.nb, a.S, a.qT, a.qstride, a.B, a.out, n_ctiles, n_groups, total);
    return cudaGetLastError();
}

cudaError_t launch_scan_m4rm(const M4Args& a, int ctas_per_sm, int num_sms, int variant) {
    // variant 0: auto (TMEM-accumulator kernel for full 2048-request tiles),
    // 1: register accumulators only, 2: TMEM-accumulator kernel
    if (variant == 2 || (variant == 0 && a.B >= 2048)) return launch_scan_m4rm_tmem(a, num_sms);
    if (a.B <= 256) return launch_m4<512, 4>(a, ctas_per_sm, num_sms);
    if (a.B <= 512) return launch_m4<512, 8>(a, ctas_per_sm, num_sms);
    return launch_m4<512, 16>(a, ctas_per_sm, num_sms);
}

uint64_t m4rm_qstride(uint32_t B) { return (uint64_t(B) + 15) & ~uint64_t(15); }
// rows of the group-major query layout: a multiple of 48 covers the 16-byte
// chunks of the nibble kernel, the 12-byte chunks of the 6-bucket kernel and
// the 4-byte sets of the quad kernel (rows past the vector are never selected:
// they map to zero-filled buckets)
uint64_t m4rm_qrows(uint64_t n_groups) {
    const uint64_t r48 = (n_groups + 47) / 48 * 48;
    const uint64_t r9 = (n_groups + 8) / 9 * 9;  // layout 2: whole pairs
    return r48 > r9 ? r48 : r9;
}

static uint64_t hi_offset(int layout, uint64_t nbytes, uint64_t qstride) {
    return layout == 2 ? (nbytes + 8) / 9 * 8 * qstride : 0;
}

cudaError_t launch_expand_T(const uint8_t* seeds, uint32_t B, uint64_t byte_lo, uint64_t nbytes,
                            uint8_t* qT, uint64_t qstride, cudaStream_t s, int layout) {
    if (layout == 2) {
        const uint64_t n = uint64_t((B + 31) & ~31u) * ((nbytes + 575) / 576);
        if (n == 0) return cudaSuccess;
        k_expand_q9<<<uint32_t((n + 127) / 128), 128, 0, s>>>(seeds, B, byte_lo, nbytes, qT, qstride,
                                                               hi_offset(layout, nbytes, qstride));
        return cudaGetLastError();
    }
    const uint64_t nblk = (byte_lo + nbytes + 63) / 64 - byte_lo / 64;
    const uint64_t n = uint64_t((B + 31) & ~31u) * nblk;
    if (n == 0) return cudaSuccess;
    k_expand_T<<<uint32_t((n + 127) / 128), 128, 0, s>>>(seeds, B, byte_lo, nbytes, qT, qstride, layout,
                                                          hi_offset(layout, nbytes, qstride));
    return cudaGetLastError();
}

cudaError_t launch_transpose_q(const uint8_t* q, uint64_t q_stride, uint64_t byte_lo, uint64_t nbytes,
                               uint32_t B, uint8_t* qT, uint64_t qstride, cudaStream_t s, int layout) {
    if (!B || !nbytes) return cudaSuccess;
    if (layout == 2) {
        dim3 grid9(uint32_t((nbytes + 287) / 288), (B + 31) / 32);
        k_transpose_q9<<<grid9, dim3(32, 8), 0, s>>>(q, q_stride, byte_lo, nbytes, B, qT, qstride,
                                                     hi_offset(layout, nbytes, qstride));
        return cudaGetLastError();
    }
    dim3 grid(uint32_t((nbytes + 31) / 32), (B + 31) / 32);
    k_transpose_q<<<grid, dim3(32, 8), 0, s>>>(q, q_stride, byte_lo, nbytes, B, qT, qstride, layout,
                                               hi_offset(layout, nbytes, qstride));
    return cudaGetLastError();
}

}  // namespace xpir

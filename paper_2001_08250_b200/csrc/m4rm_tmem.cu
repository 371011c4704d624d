// K1 (B >= 2048): the M4RM byte-table scan with HALF-TMEM accumulators.
//
// Same math and table layout as k_scan_m4rm (m4rm.cu): query byte g of request
// r selects buckets 8g..8g+7 (pir.hpp:25), the CTA builds T_g[x] =
// XOR_{i in x} bucket_{8g+i} for a 128-byte column slice in shared memory and
// every request does one conflict-free LDS.128 per 8 buckets, two groups per
// barrier folded with one 3-input XOR (bit-exact pir::answer_batch, pir.cpp:41-52).
//
// What changes: the table-build cost (256 rows x 128 B of STS per group) is
// amortised over Rc requests, and Rc is bounded by where the accumulators live.
// Registers hold 8 request slots per thread (32 regs); Tensor Memory holds 24
// more (tcgen05.ld/st .32x32b.x4 read-modify-write: thread lane l keeps its
// 16 bytes of a request's 128-byte slice in 4 TMEM columns). Rc doubles from
// 1024 to 2048, so the STS/LDS overhead per request halves. Measured on B200
// (xpir_probe_tmem): TMEM x4 read+write runs at ~400 B/clk/SM and does not slow
// concurrent LDS.128 traffic, so the TMEM half of the accumulator traffic rides
// beside the shared-memory-bound lookups.
//
// TMEM map (512 columns x 128 lanes, one CTA per SM): warp w uses lanes
// 32*(w%4)..+31 (hardware quadrant) and columns 128*(w/4) + 4*t, t < 24.
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"
#include "scan.cuh"

namespace xpir {

using namespace ptx;

namespace {

constexpr int TM_NT = 512;
constexpr int TM_NW = TM_NT / 32;
constexpr int TM_RR = 8;                   // register slots per thread
constexpr int TM_RT = 24;                  // TMEM slots per thread
constexpr int TM_SLOTS = TM_RR + TM_RT;    // 32
constexpr int TM_RC = TM_NW * 4 * TM_SLOTS;  // 2048 requests per tile
constexpr int TM_CHUNK_G = 16;
constexpr int TM_TAB = 256 * 128;
constexpr int TM_DBS = TM_CHUNK_G * 8 * 128;
constexpr int TM_QS = TM_CHUNK_G * TM_RC;
constexpr int TM_OFF_QS = 4 * TM_TAB;
constexpr int TM_OFF_DBS = TM_OFF_QS + 2 * TM_QS;
constexpr int TM_OFF_ADDR = TM_OFF_DBS + 2 * TM_DBS;
constexpr int TM_SMEM = TM_OFF_ADDR + 16;
static_assert(TM_SMEM <= 232448, "exceeds the 227 KB opt-in shared memory per CTA");

__device__ __forceinline__ void tm_ld4(uint32_t a, uint4& v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a));
}
__device__ __forceinline__ void tm_st4(uint32_t a, const uint4& v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(a), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w));
}
// wait::ld with the loaded registers as in/out operands, so no use of them can be
// scheduled before the wait (tcgen05.ld destinations are undefined until then).
__device__ __forceinline__ void tm_wait_ld(uint4 (&m)[4]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(m[0].x), "+r"(m[0].y), "+r"(m[0].z), "+r"(m[0].w), "+r"(m[1].x), "+r"(m[1].y),
                   "+r"(m[1].z), "+r"(m[1].w), "+r"(m[2].x), "+r"(m[2].y), "+r"(m[2].z), "+r"(m[2].w),
                   "+r"(m[3].x), "+r"(m[3].y), "+r"(m[3].z), "+r"(m[3].w)
                 :
                 : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ uint32_t byte_of(const uint32_t (&w)[8], int s) {
    return (w[s >> 2] >> (8 * (s & 3))) & 0xffu;
}

__device__ __forceinline__ void load_idx(uint32_t a, uint32_t (&w)[8]) {
    const uint4 x = lds128(a), y = lds128(a + 16);
    w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
    w[4] = y.x; w[5] = y.y; w[6] = y.z; w[7] = y.w;
}

__device__ __forceinline__ void xor3(uint4& a, const uint4& b, const uint4& c) {
    a.x ^= b.x ^ c.x;
    a.y ^= b.y ^ c.y;
    a.z ^= b.z ^ c.z;
    a.w ^= b.w ^ c.w;
}
__device__ __forceinline__ void xor2(uint4& a, const uint4& b) {
    a.x ^= b.x;
    a.y ^= b.y;
    a.z ^= b.z;
    a.w ^= b.w;
}

}  // namespace

__global__ void __launch_bounds__(TM_NT, 1)
k_scan_m4rm_tmem(const uint8_t* __restrict__ db, uint32_t nb, uint32_t S, const uint8_t* __restrict__ qT,
                 uint64_t qstride, uint32_t B, uint8_t* __restrict__ out, uint32_t n_ctiles, uint32_t n_groups,
                 uint64_t n_segments, PeerOut peers) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int qq = lane >> 3, l8 = lane & 7;
    const int slot0 = (warp * 4 + qq) * TM_SLOTS;  // first request slot of this thread

    // TMEM: warp 0 allocates all 512 columns for the CTA (one CTA per SM)
    uint32_t* taddr_smem = reinterpret_cast<uint32_t*>(smem + TM_OFF_ADDR);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            sbase + TM_OFF_ADDR));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = *taddr_smem;
    const uint32_t tcol = tbase + (uint32_t((warp & 3) * 32) << 16) + uint32_t(warp >> 2) * 128;

    const uint32_t hm5 = 0u - ((warp >> 0) & 1u), hm6 = 0u - ((warp >> 1) & 1u), hm7 = 0u - ((warp >> 2) & 1u);
    // Work units (column tile c fastest, then request tile, then group segment),
    // dealt round-robin: at any moment the CTAs work on the same few
    // (request tile, segment) pairs for all column tiles, so each staged query
    // chunk and bucket chunk is fetched from HBM once and re-read from L2.
    const uint32_t n_rtiles = (B + TM_RC - 1) / TM_RC;
    const uint32_t n_seg = uint32_t(n_segments);  // host-chosen segment count
    const uint64_t units = uint64_t(n_ctiles) * n_rtiles * n_seg;

    for (uint64_t v = blockIdx.x; v < units; v += gridDim.x) {
        const uint32_t c = uint32_t(v % n_ctiles);
        const uint32_t rt = uint32_t((v / n_ctiles) % n_rtiles);
        const uint32_t sg = uint32_t(v / (uint64_t(n_ctiles) * n_rtiles));
        const uint32_t gs = uint32_t(uint64_t(n_groups) * sg / n_seg);
        const uint32_t ge = uint32_t(uint64_t(n_groups) * (sg + 1) / n_seg);
        if (gs >= ge) continue;
        const uint32_t r_base = rt * TM_RC;
        const uint32_t nvalid = min(uint32_t(TM_RC), B - r_base);
        const bool active = uint32_t(warp * 4 * TM_SLOTS) < nvalid;  // warp-uniform

        uint4 racc[TM_RR];
#pragma unroll
        for (int i = 0; i < TM_RR; ++i) racc[i] = make_uint4(0, 0, 0, 0);
        if (active) {
#pragma unroll
            for (int t = 0; t < TM_RT; ++t) tm_st4(tcol + 4 * t, make_uint4(0, 0, 0, 0));
            tm_wait_st();
        }

        auto stage = [&](uint32_t kc, int b) {
            const uint32_t qdst = sbase + TM_OFF_QS + b * TM_QS;
            constexpr int QCH = TM_RC / 16;
            for (int k = tid; k < TM_CHUNK_G * QCH; k += TM_NT) {
                const uint32_t gl = k / QCH, ch = k - gl * QCH;
                const uint64_t col = uint64_t(r_base) + ch * 16;
                const bool ok = col < qstride;
                const uint8_t* src = qT + (uint64_t(kc) * TM_CHUNK_G + gl) * qstride + (ok ? col : 0);
                cp_async16(qdst + gl * TM_RC + ch * 16, src, ok ? 16u : 0u);
            }
            const uint32_t ddst = sbase + TM_OFF_DBS + b * TM_DBS;
            for (int k = tid; k < TM_CHUNK_G * 8 * 8; k += TM_NT) {
                const uint32_t bl = k >> 3, part = k & 7;
                const uint32_t bucket = kc * 128 + bl;
                const bool ok = bucket < nb;
                const uint8_t* src = db + (ok ? uint64_t(bucket) * S : 0) + uint64_t(c) * 128 + part * 16;
                cp_async16(ddst + bl * 128 + part * 16, src, ok ? 16u : 0u);
            }
        };

        const uint32_t kc0 = gs / TM_CHUNK_G, kc1 = (ge + TM_CHUNK_G - 1) / TM_CHUNK_G;
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
            const uint32_t qbuf = sbase + TM_OFF_QS + b * TM_QS;
            const uint32_t dbuf = sbase + TM_OFF_DBS + b * TM_DBS;
            const uint32_t g0 = kc * TM_CHUNK_G;
            const uint32_t glo = (gs > g0 ? gs : g0) - g0;
            const uint32_t ghi = (ge < g0 + TM_CHUNK_G ? ge : g0 + TM_CHUNK_G) - g0;
#pragma unroll 1
            for (uint32_t gl = glo; gl < ghi; gl += 2) {
                const bool pair = gl + 1 < ghi;
                const uint32_t tabA = sbase + tb * 2 * TM_TAB;
                if (warp < 8 || pair) {  // warps 0-7 build T_gl, warps 8-15 build T_gl+1
                    const uint32_t g = gl + (warp >> 3);
                    const uint32_t src = dbuf + g * 8 * 128 + lane * 4;
                    uint32_t bk[5];
#pragma unroll
                    for (int k = 0; k < 5; ++k) bk[k] = lds32(src + k * 128);
                    uint32_t h = (lds32(src + 5 * 128) & hm5) ^ (lds32(src + 6 * 128) & hm6) ^
                                 (lds32(src + 7 * 128) & hm7);
                    const uint32_t row0 = tabA + (warp >> 3) * TM_TAB + ((warp & 7) * 32) * 128 + lane * 4;
                    sts32(row0, h);
#pragma unroll
                    for (int k = 1; k < 32; ++k) {
                        h ^= bk[(k & 1) ? 0 : (k & 2) ? 1 : (k & 4) ? 2 : (k & 8) ? 3 : 4];  // ctz(k)
                        sts32(row0 + uint32_t(k ^ (k >> 1)) * 128, h);
                    }
                }
                __syncthreads();
                if (active) {
                    const uint32_t rowA = tabA + l8 * 16, rowB = rowA + TM_TAB;
                    uint32_t ia[8], ib[8];
                    load_idx(qbuf + gl * TM_RC + slot0, ia);
                    if (pair) {
                        load_idx(qbuf + (gl + 1) * TM_RC + slot0, ib);
#pragma unroll
                        for (int s = 0; s < TM_RR; ++s) {
                            const uint4 va = lds128(rowA + byte_of(ia, s) * 128);
                            const uint4 vb = lds128(rowB + byte_of(ib, s) * 128);
                            xor3(racc[s], va, vb);
                        }
#pragma unroll
                        for (int t0 = 0; t0 < TM_RT; t0 += 4) {
                            uint4 m[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) tm_ld4(tcol + 4 * (t0 + k), m[k]);
                            uint4 va[4], vb[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const int s = TM_RR + t0 + k;
                                va[k] = lds128(rowA + byte_of(ia, s) * 128);
                                vb[k] = lds128(rowB + byte_of(ib, s) * 128);
                            }
                            tm_wait_ld(m);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                xor3(m[k], va[k], vb[k]);
                                tm_st4(tcol + 4 * (t0 + k), m[k]);
                            }
                        }
                    } else {
#pragma unroll
                        for (int s = 0; s < TM_RR; ++s) xor2(racc[s], lds128(rowA + byte_of(ia, s) * 128));
#pragma unroll
                        for (int t0 = 0; t0 < TM_RT; t0 += 4) {
                            uint4 m[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) tm_ld4(tcol + 4 * (t0 + k), m[k]);
                            uint4 va[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) va[k] = lds128(rowA + byte_of(ia, TM_RR + t0 + k) * 128);
                            tm_wait_ld(m);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                xor2(m[k], va[k]);
                                tm_st4(tcol + 4 * (t0 + k), m[k]);
                            }
                        }
                    }
                    tm_wait_st();
                }
                tb ^= 1;
            }
            __syncthreads();
        }
        // flush: registers, then TMEM slots
        if (active) {
#pragma unroll
            for (int s = 0; s < TM_SLOTS; s += 4) {
                uint4 v[4];
                if (s >= TM_RR) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) tm_ld4(tcol + 4 * (s - TM_RR + k), v[k]);
                    tm_wait_ld(v);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) v[k] = racc[s + k];
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t rl = slot0 + s + k;
                    if (rl < nvalid) {
                        // fused cross-GPU reduce: with peers, the row is XORed straight into its
                        // owner rank's answer buffer (NVLink peer atomics); otherwise locally
                        uint8_t* const base = peers.n ? peers.owner_out(r_base + rl) : out;
                        uint8_t* o = base + uint64_t(r_base + rl) * S + uint64_t(c) * 128 + l8 * 16;
                        if (peers.n) {  // rows every rank reduces into: system-scope RMWs
                            red_xor64_sys(o, uint64_t(v[k].y) << 32 | v[k].x);
                            red_xor64_sys(o + 8, uint64_t(v[k].w) << 32 | v[k].z);
                        } else {
                            red_xor64(o, uint64_t(v[k].y) << 32 | v[k].x);
                            red_xor64(o + 8, uint64_t(v[k].w) << 32 | v[k].z);
                        }
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

int m4rm_tmem_rows_per_tile() { return TM_RC; }

cudaError_t launch_scan_m4rm_tmem(const M4Args& a, int num_sms) {
    cudaError_t e =
        cudaFuncSetAttribute(k_scan_m4rm_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, TM_SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t n_ctiles = a.S / 128;
    const uint32_t n_rtiles = (a.B + TM_RC - 1) / TM_RC;
    const uint32_t n_groups = (a.nb + 7) / 8;
    // Segments per (request tile, column tile): about 32 units per CTA, and a unit
    // count that is a multiple of the grid when the shapes allow (config 4: 4 x 32
    // pairs x 37 segments = 32 x 148), segments of at least 64 groups.
    const uint64_t pairs = uint64_t(n_ctiles) * n_rtiles;
    const uint64_t grid = uint64_t(num_sms);
    uint64_t a_ = pairs, b_ = grid;
    while (b_) {
        const uint64_t t = a_ % b_;
        a_ = b_;
        b_ = t;
    }
    const uint64_t step = grid / a_;
    const uint64_t target = (32 * grid + pairs - 1) / pairs;
    uint64_t n_seg = (target + step - 1) / step * step;
    if (step > 4 * target) n_seg = target;  // no convenient multiple: stay near the target
    const uint64_t max_seg = n_groups / 64 > 0 ? n_groups / 64 : 1;
    if (n_seg > max_seg) n_seg = max_seg;
    if (n_seg < 1) n_seg = 1;
    k_scan_m4rm_tmem<<<dim3(uint32_t(grid)), TM_NT, TM_SMEM, a.stream>>>(a.db, a.nb, a.S, a.qT, a.qstride, a.B,
                                                                      a.out, n_ctiles, n_groups, n_seg, a.peers);
    return cudaGetLastError();
}

}  // namespace xpir

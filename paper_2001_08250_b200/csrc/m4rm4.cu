// K1 (mid-size batches, ~16 <= B <= 256): four-Russians scan with NIBBLE tables.
//
// Same structure as k_scan_m4rm (m4rm.cu) but with 4-bucket groups: a query
// nibble selects buckets 4h..4h+3 (low nibble of byte g = buckets 8g..8g+3,
// high nibble = 8g+4..8g+7, pir.hpp:25), so a table has 16 rows instead of
// 256. For small batches the 256-row build dominates the byte-table kernel;
// here a phase covers 64 buckets: each of the 16 warps builds one 16-row
// table (Gray code, 15 XORs + 16 STS per lane), one barrier, then every request
// does 16 conflict-free LDS.128 lookups folded pairwise with 3-input XORs.
// Per phase and 128-byte column: 256 STS + B x 16 LDS wavefronts for
// B x 64 buckets of work — ~1.4-1.9x the dense masked-XOR roofline at
// B = 64..256 where the byte tables reach 0.9-1.5x. Queries arrive group-major
// (qT) exactly as for k_scan_m4rm; work units are dealt round-robin with the
// column tile fastest (shared L2 reuse of staged chunks); accumulators are
// flushed with 64-bit atomicXor per unit. Bit-exact pir::answer_batch.
// B <= 32 (round 2): each request's lookups are dealt over 2/4/8 quarter-warp
// slots (template SPLIT, no per-lookup branch), so all 16 warps look up instead
// of B/4; B = 32 rose from 0.72-0.76 to 0.80 of the dense roofline, and the
// branch-free loop lifted B = 48..256 by 4-12% (profiles/r02_nibble_split.jsonl).
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"
#include "scan.cuh"

namespace xpir {

using namespace ptx;

namespace {
constexpr int K4_NT = 512;
constexpr int K4_NW = K4_NT / 32;
constexpr int K4_CHUNK_BUCKETS = 128;                // 16 query bytes per request
constexpr int K4_TAB = 16 * 128;                     // one 16-row table
constexpr int K4_DBS = K4_CHUNK_BUCKETS * 128;       // 16 KiB

// PT tables per phase (16: 64 buckets, two phases per chunk; 32: the whole chunk);
// NST staged chunks in flight (the prefetch distance: a small batch finishes a
// chunk faster than HBM latency, so it needs more than double buffering)
template <int RPT, int PT, int NST>
struct K4Layout {
    static constexpr int Rc = K4_NW * 4 * RPT;
    static constexpr int QS = 16 * Rc;               // 16 qT rows of the chunk
    static constexpr int PHASE_TABS = PT * K4_TAB;
    static constexpr int OFF_QS = 2 * PHASE_TABS;
    static constexpr int OFF_DBS = OFF_QS + NST * QS;
    static constexpr int SMEM = OFF_DBS + NST * K4_DBS;
    static_assert(SMEM <= 232448, "exceeds the 227 KB opt-in shared memory per CTA");
};

template <int RPT>
__device__ __forceinline__ uint32_t load_bytes(uint32_t a) {
    if constexpr (RPT == 4) {
        return lds32(a);
    } else {
        uint32_t v;
        if constexpr (RPT == 2)
            asm volatile("ld.shared.u16 %0, [%1];\n" : "=r"(v) : "r"(a));
        else
            asm volatile("ld.shared.u8 %0, [%1];\n" : "=r"(v) : "r"(a));
        return v;
    }
}
}  // namespace

template <int RPT, int PT, int NST, int SPLIT>
__global__ void __launch_bounds__(K4_NT, 1)
k_scan_m4rm4(const uint8_t* __restrict__ db, uint32_t nb, uint32_t S, const uint8_t* __restrict__ qT,
             uint64_t qstride, uint32_t B, uint8_t* __restrict__ out, uint32_t n_ctiles, uint32_t n_chunks,
             uint32_t n_seg) {
    using L = K4Layout<RPT, PT, NST>;
    constexpr int JB = PT / 2;  // query bytes per phase
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int qq = lane >> 3, l8 = lane & 7;
    // SPLIT > 1 (RPT = 1, B <= 32): the 64 quarter-warp slots hold 64 / SPLIT
    // requests, each request's lookups of a phase dealt to SPLIT slots (query byte
    // j to part j % SPLIT), so every warp looks up; the parts' partial answers
    // meet in the red.xor flush
    constexpr int PER = 64 / SPLIT;  // requests per tile when split
    const int part = (warp * 4 + qq) / PER;
    const int slot0 = SPLIT > 1 ? (warp * 4 + qq) - part * PER : (warp * 4 + qq) * RPT;
    const uint32_t n_rtiles = (B + L::Rc - 1) / L::Rc;
    const uint64_t units = uint64_t(n_ctiles) * n_rtiles * n_seg;

    for (uint64_t v = blockIdx.x; v < units; v += gridDim.x) {
        const uint32_t c = uint32_t(v % n_ctiles);
        const uint32_t rt = uint32_t((v / n_ctiles) % n_rtiles);
        const uint32_t sg = uint32_t(v / (uint64_t(n_ctiles) * n_rtiles));
        const uint32_t kc0 = uint32_t(uint64_t(n_chunks) * sg / n_seg);
        const uint32_t kc1 = uint32_t(uint64_t(n_chunks) * (sg + 1) / n_seg);
        if (kc0 >= kc1) continue;
        const uint32_t r_base = rt * L::Rc;
        const uint32_t nvalid = min(uint32_t(L::Rc), B - r_base);
        const bool active = SPLIT > 1 ? uint32_t(slot0) < nvalid : uint32_t(warp * 4 * RPT) < nvalid;

        uint4 acc[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) acc[i] = make_uint4(0, 0, 0, 0);

        auto stage = [&](uint32_t kc, int b) {
            const uint32_t qdst = sbase + L::OFF_QS + b * L::QS;
            constexpr int QCH = L::Rc / 16;
            for (int k = tid; k < 16 * QCH; k += K4_NT) {
                const uint32_t row = k / QCH, ch = k - row * QCH;
                const uint64_t col = uint64_t(r_base) + ch * 16;
                const bool ok = col < qstride;
                const uint8_t* src = qT + (uint64_t(kc) * 16 + row) * qstride + (ok ? col : 0);
                cp_async16(qdst + row * L::Rc + ch * 16, src, ok ? 16u : 0u);
            }
            const uint32_t ddst = sbase + L::OFF_DBS + b * K4_DBS;
            for (int k = tid; k < K4_CHUNK_BUCKETS * 8; k += K4_NT) {
                const uint32_t bl = k >> 3, part = k & 7;
                const uint32_t bucket = kc * K4_CHUNK_BUCKETS + bl;
                const bool ok = bucket < nb;
                const uint8_t* src = db + (ok ? uint64_t(bucket) * S : 0) + uint64_t(c) * 128 + part * 16;
                cp_async16(ddst + bl * 128 + part * 16, src, ok ? 16u : 0u);
            }
        };

#pragma unroll
        for (int p = 0; p < NST - 1; ++p) {
            if (kc0 + p < kc1) stage(kc0 + p, p);
            cp_async_commit();
        }
        int tb = 0;
        for (uint32_t kc = kc0; kc < kc1; ++kc) {
            const int b = int((kc - kc0) % NST);
            if (kc + NST - 1 < kc1) stage(kc + NST - 1, int((kc - kc0 + NST - 1) % NST));
            cp_async_commit();
            cp_async_wait<NST - 1>();  // chunk kc landed (one group per chunk, empty past the end)
            __syncthreads();
            const uint32_t qbuf = sbase + L::OFF_QS + b * L::QS;
            const uint32_t dbuf = sbase + L::OFF_DBS + b * K4_DBS;
#pragma unroll 1
            for (int ph = 0; ph < 32 / PT; ++ph) {
                const uint32_t tabs = sbase + tb * L::PHASE_TABS;
#pragma unroll
                for (int u = 0; u < PT / 16; ++u) {  // warp w builds table t = w + 16u: buckets 4t .. 4t+3
                    const int t16 = warp + 16 * u;
                    const uint32_t src = dbuf + (4 * PT * ph + 4 * t16) * 128 + lane * 4;
                    const uint32_t b0 = lds32(src), b1 = lds32(src + 128), b2 = lds32(src + 256),
                                   b3 = lds32(src + 384);
                    const uint32_t t = tabs + t16 * K4_TAB + lane * 4;
                    uint32_t h = 0;
                    sts32(t + 0 * 128, h);
                    h ^= b0; sts32(t + 1 * 128, h);
                    h ^= b1; sts32(t + 3 * 128, h);
                    h ^= b0; sts32(t + 2 * 128, h);
                    h ^= b2; sts32(t + 6 * 128, h);
                    h ^= b0; sts32(t + 7 * 128, h);
                    h ^= b1; sts32(t + 5 * 128, h);
                    h ^= b0; sts32(t + 4 * 128, h);
                    h ^= b3; sts32(t + 12 * 128, h);
                    h ^= b0; sts32(t + 13 * 128, h);
                    h ^= b1; sts32(t + 15 * 128, h);
                    h ^= b0; sts32(t + 14 * 128, h);
                    h ^= b2; sts32(t + 10 * 128, h);
                    h ^= b0; sts32(t + 11 * 128, h);
                    h ^= b1; sts32(t + 9 * 128, h);
                    h ^= b0; sts32(t + 8 * 128, h);
                }
                __syncthreads();
                if (active) {
                    const uint32_t rows = tabs + l8 * 16;
#pragma unroll
                    for (int jj = 0; jj < JB / SPLIT; ++jj) {  // query byte JB*ph + j: tables 2j, 2j+1
                        const int j = part + jj * SPLIT;
                        const uint32_t qb = load_bytes<RPT>(qbuf + (JB * ph + j) * L::Rc + slot0);
#pragma unroll
                        for (int i = 0; i < RPT; ++i) {
                            const uint32_t x = (qb >> (8 * i)) & 0xffu;
                            const uint4 va = lds128(rows + (2 * j) * K4_TAB + (x & 15u) * 128);
                            const uint4 vb = lds128(rows + (2 * j + 1) * K4_TAB + (x >> 4) * 128);
                            acc[i].x ^= va.x ^ vb.x;
                            acc[i].y ^= va.y ^ vb.y;
                            acc[i].z ^= va.z ^ vb.z;
                            acc[i].w ^= va.w ^ vb.w;
                        }
                    }
                }
                tb ^= 1;
            }
            __syncthreads();
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

template <int RPT, int SPLIT = 1>
static cudaError_t launch_k4(const M4Args& a, int num_sms) {
    constexpr int PT = 16, NST = 2;  // 32 tables per phase / deeper staging: measured no faster
    using L = K4Layout<RPT, PT, NST>;
    cudaError_t e = cudaFuncSetAttribute(k_scan_m4rm4<RPT, PT, NST, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t n_ctiles = a.S / 128;
    const uint32_t n_rtiles = (a.B + L::Rc - 1) / L::Rc;
    const uint32_t n_chunks = (a.nb + K4_CHUNK_BUCKETS - 1) / K4_CHUNK_BUCKETS;
    const uint64_t pairs = uint64_t(n_ctiles) * n_rtiles;
    const uint64_t grid = uint64_t(num_sms);
    uint64_t n_seg = (16 * grid + pairs - 1) / pairs;  // ~16 units per CTA
    if (n_seg > n_chunks) n_seg = n_chunks;
    if (n_seg < 1) n_seg = 1;
    k_scan_m4rm4<RPT, PT, NST, SPLIT><<<uint32_t(grid), K4_NT, L::SMEM, a.stream>>>(
        a.db, a.nb, a.S, a.qT, a.qstride, a.B, a.out, n_ctiles, n_chunks, uint32_t(n_seg));
    return cudaGetLastError();
}

cudaError_t launch_scan_m4rm4(const M4Args& a, int num_sms) {
    // B <= 32: each request's lookups spread over 64 / B' slots (B' = B rounded up
    // to a power of two >= 8), so all 16 warps look up
    if (a.B <= 8) return launch_k4<1, 8>(a, num_sms);
    if (a.B <= 16) return launch_k4<1, 4>(a, num_sms);
    if (a.B <= 32) return launch_k4<1, 2>(a, num_sms);
    if (a.B <= 64) return launch_k4<1>(a, num_sms);
    if (a.B <= 128) return launch_k4<2>(a, num_sms);
    return launch_k4<4>(a, num_sms);
}

}  // namespace xpir

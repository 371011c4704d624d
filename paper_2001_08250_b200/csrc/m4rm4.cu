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
constexpr int K4_PHASE_TABS = 16 * K4_TAB;           // 16 tables = 64 buckets
constexpr int K4_DBS = K4_CHUNK_BUCKETS * 128;       // 16 KiB

template <int RPT>
struct K4Layout {
    static constexpr int Rc = K4_NW * 4 * RPT;
    static constexpr int QS = 16 * Rc;               // 16 qT rows of the chunk
    static constexpr int OFF_QS = 2 * K4_PHASE_TABS;
    static constexpr int OFF_DBS = OFF_QS + 2 * QS;
    static constexpr int SMEM = OFF_DBS + 2 * K4_DBS;
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

template <int RPT>
__global__ void __launch_bounds__(K4_NT, 1)
k_scan_m4rm4(const uint8_t* __restrict__ db, uint32_t nb, uint32_t S, const uint8_t* __restrict__ qT,
             uint64_t qstride, uint32_t B, uint8_t* __restrict__ out, uint32_t n_ctiles, uint32_t n_chunks,
             uint32_t n_seg) {
    using L = K4Layout<RPT>;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int qq = lane >> 3, l8 = lane & 7;
    const int slot0 = (warp * 4 + qq) * RPT;
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
        const bool active = uint32_t(warp * 4 * RPT) < nvalid;

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
            const uint32_t qbuf = sbase + L::OFF_QS + b * L::QS;
            const uint32_t dbuf = sbase + L::OFF_DBS + b * K4_DBS;
#pragma unroll 1
            for (int ph = 0; ph < 2; ++ph) {
                const uint32_t tabs = sbase + tb * K4_PHASE_TABS;
                {   // warp w builds the table of buckets 64*ph + 4w .. +3
                    const uint32_t src = dbuf + (64 * ph + 4 * warp) * 128 + lane * 4;
                    const uint32_t b0 = lds32(src), b1 = lds32(src + 128), b2 = lds32(src + 256),
                                   b3 = lds32(src + 384);
                    const uint32_t t = tabs + warp * K4_TAB + lane * 4;
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
                    for (int j = 0; j < 8; ++j) {  // query byte 8*ph + j: tables 2j (low) and 2j+1 (high)
                        const uint32_t qb = load_bytes<RPT>(qbuf + (8 * ph + j) * L::Rc + slot0);
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

template <int RPT>
static cudaError_t launch_k4(const M4Args& a, int num_sms) {
    using L = K4Layout<RPT>;
    cudaError_t e = cudaFuncSetAttribute(k_scan_m4rm4<RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t n_ctiles = a.S / 128;
    const uint32_t n_rtiles = (a.B + L::Rc - 1) / L::Rc;
    const uint32_t n_chunks = (a.nb + K4_CHUNK_BUCKETS - 1) / K4_CHUNK_BUCKETS;
    const uint64_t pairs = uint64_t(n_ctiles) * n_rtiles;
    const uint64_t grid = uint64_t(num_sms);
    uint64_t n_seg = (16 * grid + pairs - 1) / pairs;  // ~16 units per CTA
    if (n_seg > n_chunks) n_seg = n_chunks;
    if (n_seg < 1) n_seg = 1;
    k_scan_m4rm4<RPT><<<uint32_t(grid), K4_NT, L::SMEM, a.stream>>>(a.db, a.nb, a.S, a.qT, a.qstride, a.B, a.out,
                                                                  n_ctiles, n_chunks, uint32_t(n_seg));
    return cudaGetLastError();
}

cudaError_t launch_scan_m4rm4(const M4Args& a, int num_sms) {
    if (a.B <= 64) return launch_k4<1>(a, num_sms);
    if (a.B <= 128) return launch_k4<2>(a, num_sms);
    return launch_k4<4>(a, num_sms);
}

}  // namespace xpir

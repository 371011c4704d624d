// K9 (mid-size batches, ~96 <= B <= ~400): four-Russians scan with 6-BUCKET tables.
//
// Same structure as k_scan_m4rm4 (m4rm4.cu), with groups of 6 buckets instead of
// 4: three query bytes (24 bits, LSB-first, pir.hpp:25) hold the selections of
// four 6-bucket groups, so a table has 64 rows. Per bucket and 128-byte column
// the shared-memory wavefronts are (2^k + B) / k for k-bucket tables; k = 6
// minimises that for B ~ 100-400 (k = 4: (16 + B)/4, k = 8: (256 + B)/8), e.g.
// B = 256: 53 instead of 68 (nibble) or 64 (byte tables).
//
// A chunk is 96 buckets (12 query bytes), scanned in two phases of 48 buckets =
// 8 tables. Warp w builds half of table w/2 (the 32 rows with bit 5 = w & 1,
// Gray-code order: one XOR and one STS per row and lane), one barrier, then
// every request does 8 conflict-free LDS.128 lookups per phase (8 lanes x 16 B
// per request and row). Query bytes arrive group-major (qT, as for the other
// M4RM kernels); tables are double-buffered across phases. Buckets past the
// shard are zero-filled, so selection bits past N contribute nothing.
// Bit-exact pir::answer_batch (pir.cpp:41-52).
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"
#include "scan.cuh"

namespace xpir {

using namespace ptx;

namespace {
constexpr int K6_NT = 512;
constexpr int K6_NW = K6_NT / 32;
constexpr int K6_CHUNK_BUCKETS = 96;                  // 12 query bytes per request
constexpr int K6_TAB = 64 * 128;                      // one 64-row table of 128-byte rows
constexpr int K6_PHASE_TABS = 8 * K6_TAB;             // 8 tables = 48 buckets
constexpr int K6_DBS = K6_CHUNK_BUCKETS * 128;        // 12 KiB

template <int RPT>
struct K6Layout {
    static constexpr int Rc = K6_NW * 4 * RPT;
    static constexpr int QS = 12 * Rc;                // 12 qT rows of the chunk
    static constexpr int OFF_QS = 2 * K6_PHASE_TABS;
    static constexpr int OFF_DBS = OFF_QS + 2 * QS;
    static constexpr int SMEM = OFF_DBS + 2 * K6_DBS;
};

template <int RPT>
__device__ __forceinline__ uint32_t load_bytes6(uint32_t a) {
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
__global__ void __launch_bounds__(K6_NT, 1)
k_scan_m4rm6(const uint8_t* __restrict__ db, uint32_t nb, uint32_t S, const uint8_t* __restrict__ qT,
             uint64_t qstride, uint32_t B, uint8_t* __restrict__ out, uint32_t n_ctiles, uint32_t n_chunks,
             uint32_t n_seg) {
    using L = K6Layout<RPT>;
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
            for (int k = tid; k < 12 * QCH; k += K6_NT) {
                const uint32_t row = k / QCH, ch = k - row * QCH;
                const uint64_t col = uint64_t(r_base) + ch * 16;
                const bool ok = col < qstride;
                const uint8_t* src = qT + (uint64_t(kc) * 12 + row) * qstride + (ok ? col : 0);
                cp_async16(qdst + row * L::Rc + ch * 16, src, ok ? 16u : 0u);
            }
            const uint32_t ddst = sbase + L::OFF_DBS + b * K6_DBS;
            for (int k = tid; k < K6_CHUNK_BUCKETS * 8; k += K6_NT) {
                const uint32_t bl = k >> 3, part = k & 7;
                const uint32_t bucket = kc * K6_CHUNK_BUCKETS + bl;
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
            const uint32_t dbuf = sbase + L::OFF_DBS + b * K6_DBS;
#pragma unroll 1
            for (int ph = 0; ph < 2; ++ph) {
                const uint32_t tabs = sbase + tb * K6_PHASE_TABS;
                {   // warp w: rows (w & 1) << 5 | g of table w >> 1 (buckets 48*ph + 6*(w >> 1) + 0..5)
                    const int t = warp >> 1, hi = warp & 1;
                    const uint32_t src = dbuf + (48 * ph + 6 * t) * 128 + lane * 4;
                    uint32_t bw[5];
#pragma unroll
                    for (int j = 0; j < 5; ++j) bw[j] = lds32(src + j * 128);
                    uint32_t h = hi ? lds32(src + 5 * 128) : 0u;
                    const uint32_t dst = tabs + t * K6_TAB + (hi << 5) * 128 + lane * 4;
#pragma unroll
                    for (int i = 0; i < 32; ++i) {  // Gray code over buckets 0..4 of the group
                        if (i) h ^= bw[(i & 1) ? 0 : (i & 2) ? 1 : (i & 4) ? 2 : (i & 8) ? 3 : 4];  // ctz(i)
                        sts32(dst + (i ^ (i >> 1)) * 128, h);
                    }
                }
                __syncthreads();
                if (active) {
                    const uint32_t rows = tabs + l8 * 16;
#pragma unroll
                    for (int u = 0; u < 2; ++u) {  // query bytes 6*ph + 3u .. +2: tables 4u .. 4u+3
                        const uint32_t q0 = load_bytes6<RPT>(qbuf + (6 * ph + 3 * u + 0) * L::Rc + slot0);
                        const uint32_t q1 = load_bytes6<RPT>(qbuf + (6 * ph + 3 * u + 1) * L::Rc + slot0);
                        const uint32_t q2 = load_bytes6<RPT>(qbuf + (6 * ph + 3 * u + 2) * L::Rc + slot0);
#pragma unroll
                        for (int i = 0; i < RPT; ++i) {
                            // the request's 24 selection bits, bucket 24u + j at bit j
                            const uint32_t x = ((q0 >> (8 * i)) & 0xffu) | (((q1 >> (8 * i)) & 0xffu) << 8) |
                                               (((q2 >> (8 * i)) & 0xffu) << 16);
                            const uint32_t base = rows + (4 * u) * K6_TAB;
                            const uint4 va = lds128(base + 0 * K6_TAB + (x & 63u) * 128);
                            const uint4 vb = lds128(base + 1 * K6_TAB + ((x >> 6) & 63u) * 128);
                            const uint4 vc = lds128(base + 2 * K6_TAB + ((x >> 12) & 63u) * 128);
                            const uint4 vd = lds128(base + 3 * K6_TAB + (x >> 18) * 128);
                            acc[i].x ^= va.x ^ vb.x ^ vc.x ^ vd.x;
                            acc[i].y ^= va.y ^ vb.y ^ vc.y ^ vd.y;
                            acc[i].z ^= va.z ^ vb.z ^ vc.z ^ vd.z;
                            acc[i].w ^= va.w ^ vb.w ^ vc.w ^ vd.w;
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
static cudaError_t launch_k6(const M4Args& a, int num_sms) {
    using L = K6Layout<RPT>;
    cudaError_t e = cudaFuncSetAttribute(k_scan_m4rm6<RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t n_ctiles = a.S / 128;
    const uint32_t n_rtiles = (a.B + L::Rc - 1) / L::Rc;
    const uint32_t n_chunks = (a.nb + K6_CHUNK_BUCKETS - 1) / K6_CHUNK_BUCKETS;
    const uint64_t pairs = uint64_t(n_ctiles) * n_rtiles;
    const uint64_t grid = uint64_t(num_sms);
    uint64_t n_seg = (16 * grid + pairs - 1) / pairs;  // ~16 units per CTA
    if (n_seg > n_chunks) n_seg = n_chunks;
    if (n_seg < 1) n_seg = 1;
    k_scan_m4rm6<RPT><<<uint32_t(grid), K6_NT, L::SMEM, a.stream>>>(a.db, a.nb, a.S, a.qT, a.qstride, a.B, a.out,
                                                                  n_ctiles, n_chunks, uint32_t(n_seg));
    return cudaGetLastError();
}

// qT must hold m4rm_qrows(nbytes) rows (a multiple of 48 >= 12 * chunks).
cudaError_t launch_scan_m4rm6(const M4Args& a, int num_sms) {
    if (a.B <= 64) return launch_k6<1>(a, num_sms);
    if (a.B <= 128) return launch_k6<2>(a, num_sms);
    return launch_k6<4>(a, num_sms);
}

}  // namespace xpir

// K1 (mid-size batches, 8 <= B <= 192): warp-private nibble tables.
//
// pir::answer_batch (pir.cpp:41-52) for batches too small to amortise the
// 256-row byte tables of k_scan_m4rm but large enough to be bound by the dense
// masked-XOR rate. Each warp independently owns (request tile, 128-byte column
// slice, bucket chunk) work items. For every 4 buckets it builds a 16-row table
//     T[x] = XOR_{i : bit i of x} bucket_{4h+i}[slice]      (x = one query nibble)
// in its own slice of shared memory (lane l computes word l of all 16 rows in
// Gray-code order: 15 XORs, 16 STS), and each request of the tile does one
// conflict-free LDS.128 per 4 buckets — two nibble groups per step folded with
// one 3-input XOR. Bucket words come straight from global memory into registers
// (coalesced 128-byte rows, prefetched one step ahead); no block-wide barriers,
// only __syncwarp. Cost per 4 buckets and warp: 16 + B shared-memory wavefronts
// for B x 128 bucket-bytes of work, vs 4*B masked XORs per word for the dense
// kernel. Accumulators are flushed with 64-bit atomicXor per work item.
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"
#include "scan.cuh"

namespace xpir {

using namespace ptx;

constexpr int NIB_NT = 256;
constexpr int NIB_NW = NIB_NT / 32;
constexpr int NIB_TAB = 16 * 128;               // one nibble table
constexpr int NIB_WARP_SMEM = 2 * 2 * NIB_TAB;  // [2 phases][2 tables]
constexpr int NIB_CHUNK = 1024;                 // buckets per work item (multiple of 32)

template <int RPT>
__global__ void __launch_bounds__(NIB_NT)
k_scan_nib(const uint8_t* __restrict__ db, uint32_t nb, uint32_t S, const uint8_t* __restrict__ q,
           uint64_t q_stride, uint32_t B, uint8_t* __restrict__ out, uint32_t n_ctiles, uint32_t n_chunks,
           uint64_t total_items) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int qq = lane >> 3, l8 = lane & 7;
    const uint32_t wbase = smem_u32(smem) + warp * NIB_WARP_SMEM;
    constexpr uint32_t TILE = 4 * RPT;
    const uint64_t gw = uint64_t(blockIdx.x) * NIB_NW + warp;
    const uint64_t nwarps = uint64_t(gridDim.x) * NIB_NW;

    for (uint64_t item = gw; item < total_items; item += nwarps) {
        const uint32_t ch = uint32_t(item % n_chunks);
        const uint64_t rest = item / n_chunks;
        const uint32_t c = uint32_t(rest % n_ctiles);
        const uint32_t rt = uint32_t(rest / n_ctiles);
        const uint32_t r0 = rt * TILE + qq * RPT;  // this thread's first request
        const uint32_t j0 = ch * NIB_CHUNK;
        const uint32_t j1 = min(nb, j0 + NIB_CHUNK);
        const uint8_t* colp = db + uint64_t(c) * 128 + lane * 4;

        uint4 acc[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) acc[i] = make_uint4(0, 0, 0, 0);

        // bucket words of the next 8-bucket step, prefetched
        auto load8 = [&](uint32_t jb, uint32_t (&w)[8]) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t b = jb + k;
                w[k] = b < j1 ? __ldcs(reinterpret_cast<const uint32_t*>(colp + uint64_t(b) * S)) : 0u;
            }
        };
        uint32_t cur[8], nxt[8];
        load8(j0, cur);
        int ph = 0;
        for (uint32_t jc = j0; jc < j1; jc += 32) {
            // 32 buckets = 8 nibble groups = 4 query bytes per request
            uint32_t qw[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                uint32_t w = 0;
                const uint32_t r = r0 + i;
                if (r < B) {
                    const uint8_t* qp = q + uint64_t(r) * q_stride + (jc >> 3);
                    const uint32_t n = min(32u, j1 - jc);
#pragma unroll
                    for (uint32_t k = 0; k < 4; ++k)
                        if (8 * k < n) w |= uint32_t(__ldg(qp + k)) << (8 * k);
                    if (n < 32) w &= (1u << n) - 1u;
                }
                qw[i] = w;
            }
#pragma unroll
            for (int st = 0; st < 4; ++st) {
                const uint32_t jb = jc + 8 * st;
                if (jb >= j1) break;
                if (jb + 8 < j1) load8(jb + 8, nxt);
                // build two 16-row tables: buckets jb..jb+3 and jb+4..jb+7
                const uint32_t tA = wbase + ph * 2 * NIB_TAB, tB = tA + NIB_TAB;
                {
                    uint32_t h = 0;
                    sts32(tA + lane * 4, 0u);
                    sts32(tB + lane * 4, 0u);
                    uint32_t g = 0;
                    uint32_t hb = 0;
#pragma unroll
                    for (int k = 1; k < 16; ++k) {
                        const int bit = (k & 1) ? 0 : (k & 2) ? 1 : (k & 4) ? 2 : 3;  // ctz(k)
                        h ^= cur[bit];
                        hb ^= cur[4 + bit];
                        g = uint32_t(k ^ (k >> 1));
                        sts32(tA + g * 128 + lane * 4, h);
                        sts32(tB + g * 128 + lane * 4, hb);
                    }
                }
                __syncwarp();
                const uint32_t rA = tA + l8 * 16, rB = tB + l8 * 16;
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const uint32_t xa = (qw[i] >> (8 * st)) & 15u;
                    const uint32_t xb = (qw[i] >> (8 * st + 4)) & 15u;
                    const uint4 va = lds128(rA + xa * 128);
                    const uint4 vb = lds128(rB + xb * 128);
                    acc[i].x ^= va.x ^ vb.x;
                    acc[i].y ^= va.y ^ vb.y;
                    acc[i].z ^= va.z ^ vb.z;
                    acc[i].w ^= va.w ^ vb.w;
                }
                ph ^= 1;
#pragma unroll
                for (int k = 0; k < 8; ++k) cur[k] = nxt[k];
            }
        }
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const uint32_t r = r0 + i;
            if (r < B) {
                uint8_t* o = out + uint64_t(r) * S + uint64_t(c) * 128 + l8 * 16;
                red_xor64(o, uint64_t(acc[i].y) << 32 | acc[i].x);
                red_xor64(o + 8, uint64_t(acc[i].w) << 32 | acc[i].z);
            }
        }
        __syncwarp();
    }
}

template <int RPT>
static cudaError_t launch_nib_t(const ScanArgs& a, int num_sms) {
    constexpr int SMEM = NIB_NW * NIB_WARP_SMEM;
    cudaError_t e = cudaFuncSetAttribute(k_scan_nib<RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t n_ctiles = a.S / 128;
    const uint32_t n_chunks = (a.nb + NIB_CHUNK - 1) / NIB_CHUNK;
    const uint32_t n_rtiles = (a.B + 4 * RPT - 1) / (4 * RPT);
    const uint64_t items = uint64_t(n_rtiles) * n_ctiles * n_chunks;
    uint64_t grid = (items + NIB_NW - 1) / NIB_NW;
    const uint64_t max_grid = uint64_t(num_sms) * 4;
    if (grid > max_grid) grid = max_grid;
    if (grid < 1) grid = 1;
    k_scan_nib<RPT><<<uint32_t(grid), NIB_NT, SMEM, a.stream>>>(a.db, a.nb, a.S, a.q, a.q_stride, a.B, a.out,
                                                               n_ctiles, n_chunks, items);
    return cudaGetLastError();
}

cudaError_t launch_scan_nib(const ScanArgs& a, int num_sms) {
    if (a.B <= 16) return launch_nib_t<4>(a, num_sms);
    if (a.B <= 32) return launch_nib_t<8>(a, num_sms);
    return launch_nib_t<16>(a, num_sms);
}

}  // namespace xpir

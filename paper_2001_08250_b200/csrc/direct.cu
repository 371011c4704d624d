// K1 (small batches, B < ~96): direct select-XOR — pir::answer_batch
// (pir.cpp:41-52) streamed once from HBM.
//
// For small batches the scan is HBM-bound (B <~ 11) or bound by the dense
// masked-XOR rate (one LOP3 per request x 32-bit word x bucket). Each CTA
// (256 threads) owns a bucket range; a thread owns one 16-byte column of the
// bucket and a contiguous run of buckets ("phase"), so each warp load is a
// coalesced slice of one bucket (or of several buckets when S < 512 B) and every
// thread has a long, independent, unrolled stream of 16-byte loads in flight.
// Selection bits come from 32-bucket query words, bit-reversed so each bucket's
// all-ones/zero mask is one arithmetic shift. Phases are XOR-reduced in shared
// memory and each CTA XORs its partial answers into `out` with 64-bit atomicXor
// (XOR is associative and commutative, so the result is order-independent).
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"
#include "scan.cuh"

namespace xpir {

using ptx::red_xor64;

constexpr int DIRECT_NT = 256;
// requests per tile that select through the FMA pipe (split-pipe step below):
// measured on a 1 GiB store (profiles/r02_direct_split_pipe.txt) — one of eight
// wins 6-7% at B = 16-32; more lose to register pressure and issue slots
#ifndef XPIR_DIRECT_NI
#define XPIR_DIRECT_NI(r) ((r) == 8 ? 1 : 0)
#endif

template <int RPT, int W>
__global__ void __launch_bounds__(DIRECT_NT)
k_scan_direct(const uint8_t* __restrict__ db, uint32_t nb, uint32_t S, const uint8_t* __restrict__ q,
              uint64_t q_stride, uint32_t B, uint8_t* __restrict__ out, uint32_t bpc, uint32_t cw) {
    constexpr int RB = RPT < 4 ? RPT : 4;  // requests reduced per shared-memory round
    __shared__ uint4 red[DIRECT_NT * RB * W];
    const uint32_t ncol = S / (16 * W);  // thread columns of W x 16 bytes
    const uint32_t tid = threadIdx.x;
    const uint32_t phases = DIRECT_NT / cw;
    const uint32_t p = tid / cw;
    const uint32_t c = blockIdx.y * cw + (tid - p * cw);
    const bool active = p < phases && c < ncol;
    // grid: x = request tile (fastest, so the tiles reading the same bucket range run
    // together and share it through L2), y = column block, z = bucket split
    const uint32_t split = blockIdx.z;
    const uint32_t r0 = blockIdx.x * RPT;
    const uint32_t L = bpc / phases;  // multiple of 32
    const uint32_t jb = split * bpc + p * L;
    const uint32_t je = min(nb, jb + L);

    uint4 acc[RPT][W];
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int w = 0; w < W; ++w) acc[i][w] = make_uint4(0, 0, 0, 0);

    // acc ^= bucket when the request selects it: one predicate per (request, bucket)
    // shared by the W x 4 predicated XORs (the bucket's 16W bytes in this thread)
    // B <= 4 (HBM-bound): masked XOR from the bit-reversed word (one shift pair per
    // request x bucket keeps the load stream dense); larger B: predicated XOR.
    constexpr bool kMask = RPT <= 4;
    auto step = [&](const uint4 (&v)[W], uint32_t (&qw)[RPT], uint32_t bit) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            if (kMask) {
                const uint32_t m = uint32_t(int32_t(qw[i]) >> 31);
                qw[i] <<= 1;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    acc[i][w].x ^= v[w].x & m;
                    acc[i][w].y ^= v[w].y & m;
                    acc[i][w].z ^= v[w].z & m;
                    acc[i][w].w ^= v[w].w & m;
                }
            } else if (qw[i] & bit) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    acc[i][w].x ^= v[w].x;
                    acc[i][w].y ^= v[w].y;
                    acc[i][w].z ^= v[w].z;
                    acc[i][w].w ^= v[w].w;
                }
            }
        }
    };

    // Split-pipe pair step (B > 4): the dense masked XOR is ALU-bound (LOP3 and
    // SHF issue on the ALU pipe only), so NI of the RPT requests take their
    // selection through the FMA pipe instead — the bit b in {0,1} is the top bit of
    // the request's bit-reversed word, read with IMAD.HI(qr, 2) and stepped with
    // IMAD (qr * 2), and the selected word is IMAD(v, b) — leaving one 3-input
    // LOP3 per word for two buckets (acc ^ v_a*b_a ^ v_b*b_b). The other requests
    // keep the predicated XOR (one predicate per request x bucket). Per request x
    // 2 buckets x 8 words the FMA path costs 20 FMA + 8 ALU instructions, the
    // predicated path 18 ALU; the pipe model says ~5 of 8 requests, but the kernel
    // is latency-bound at 2 CTAs/SM and the extra instructions and registers cost
    // more than the ALU relief beyond NI = 1 (measured, XPIR_DIRECT_NI).
    constexpr int NI = kMask ? 0 : XPIR_DIRECT_NI(RPT);
    auto fma_sel = [](uint32_t v, uint32_t b) -> uint32_t {
        uint32_t r;
        asm("mad.lo.u32 %0, %1, %2, 0;" : "=r"(r) : "r"(v), "r"(b));
        return r;
    };
    auto fma_top = [](uint32_t x) -> uint32_t {  // x >> 31, on the FMA pipe
        uint32_t r;
        asm("mul.hi.u32 %0, %1, 2;" : "=r"(r) : "r"(x));
        return r;
    };
    auto fma_dbl = [](uint32_t x) -> uint32_t {  // x << 1, on the FMA pipe
        uint32_t r;
        asm("mul.lo.u32 %0, %1, 2;" : "=r"(r) : "r"(x));
        return r;
    };
    auto step2 = [&](const uint4 (&va)[W], const uint4 (&vb)[W], uint32_t (&qw)[RPT], uint32_t (&qr)[RPT],
                     uint32_t bit) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            if (i < NI) {
                const uint32_t ba = fma_top(qr[i]);
                const uint32_t q1 = fma_dbl(qr[i]);
                const uint32_t bb = fma_top(q1);
                qr[i] = fma_dbl(q1);
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    acc[i][w].x ^= fma_sel(va[w].x, ba) ^ fma_sel(vb[w].x, bb);
                    acc[i][w].y ^= fma_sel(va[w].y, ba) ^ fma_sel(vb[w].y, bb);
                    acc[i][w].z ^= fma_sel(va[w].z, ba) ^ fma_sel(vb[w].z, bb);
                    acc[i][w].w ^= fma_sel(va[w].w, ba) ^ fma_sel(vb[w].w, bb);
                }
            } else {
                if (qw[i] & bit) {
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        acc[i][w].x ^= va[w].x;
                        acc[i][w].y ^= va[w].y;
                        acc[i][w].z ^= va[w].z;
                        acc[i][w].w ^= va[w].w;
                    }
                }
                if (qw[i] & (bit << 1)) {
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        acc[i][w].x ^= vb[w].x;
                        acc[i][w].y ^= vb[w].y;
                        acc[i][w].z ^= vb[w].z;
                        acc[i][w].w ^= vb[w].w;
                    }
                }
            }
        }
    };

    if (active) {
        const uint4* col = reinterpret_cast<const uint4*>(db) + uint64_t(c) * W;
        const uint64_t stride = S / 16;
        for (uint32_t jc = jb; jc < je; jc += 32) {
            const uint32_t n = min(32u, je - jc);
            uint32_t qw[RPT], qr[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                uint32_t w = 0;
                if (r0 + i < B) {
                    const uint8_t* qp = q + uint64_t(r0 + i) * q_stride + (jc >> 3);
#pragma unroll
                    for (uint32_t k = 0; k < 4; ++k)
                        if (8 * k < n) w |= uint32_t(__ldg(qp + k)) << (8 * k);
                }
                if (n < 32) w &= (1u << n) - 1u;
                qw[i] = kMask ? __brev(w) : w;  // bucket jc+jj -> bit jj (pir.hpp:25); bit 31-jj reversed
                qr[i] = __brev(w);
            }
            if (n == 32 && NI > 0) {
#pragma unroll 4
                for (uint32_t jj = 0; jj < 32; jj += 2) {
                    uint4 va[W], vb[W];
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        va[w] = __ldcs(col + uint64_t(jc + jj) * stride + w);
                        vb[w] = __ldcs(col + uint64_t(jc + jj + 1) * stride + w);
                    }
                    step2(va, vb, qw, qr, 1u << jj);
                }
            } else if (n == 32) {
#pragma unroll 8
                for (uint32_t jj = 0; jj < 32; ++jj) {
                    uint4 v[W];
#pragma unroll
                    for (int w = 0; w < W; ++w) v[w] = __ldcs(col + uint64_t(jc + jj) * stride + w);
                    step(v, qw, 1u << jj);
                }
            } else {
                for (uint32_t jj = 0; jj < n; ++jj) {
                    uint4 v[W];
#pragma unroll
                    for (int w = 0; w < W; ++w) v[w] = __ldcs(col + uint64_t(jc + jj) * stride + w);
                    step(v, qw, 1u << jj);
                }
            }
        }
    }
    // XOR-reduce the phases that share a column, then one atomic XOR per (request, word pair)
    if (phases > 1) {
#pragma unroll
        for (int i0 = 0; i0 < RPT; i0 += RB) {
#pragma unroll
            for (int i = 0; i < RB; ++i)
#pragma unroll
                for (int w = 0; w < W; ++w) red[(i * W + w) * DIRECT_NT + tid] = acc[i0 + i][w];
            __syncthreads();
            if (p == 0 && active) {
                for (uint32_t ph = 1; ph < phases; ++ph)
#pragma unroll
                    for (int i = 0; i < RB; ++i)
#pragma unroll
                        for (int w = 0; w < W; ++w) {
                            const uint4 v = red[(i * W + w) * DIRECT_NT + ph * cw + tid];
                            acc[i0 + i][w].x ^= v.x; acc[i0 + i][w].y ^= v.y;
                            acc[i0 + i][w].z ^= v.z; acc[i0 + i][w].w ^= v.w;
                        }
            }
            __syncthreads();
        }
    }
    if (p == 0 && active) {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
            if (r0 + i < B) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    uint8_t* o = out + uint64_t(r0 + i) * S + (uint64_t(c) * W + w) * 16;
                    red_xor64(o, (unsigned long long)acc[i][w].y << 32 | acc[i][w].x);
                    red_xor64(o + 8, (unsigned long long)acc[i][w].w << 32 | acc[i][w].z);
                }
            }
    }
}

template <int RPT, int W>
static cudaError_t launch_direct_t(const ScanArgs& a, int num_sms, uint32_t* nsplit_out) {
    const uint32_t ncol = a.S / (16 * W);
    const uint32_t cw = ncol >= DIRECT_NT ? DIRECT_NT : ncol;  // thread columns per CTA
    const uint32_t phases = DIRECT_NT / cw;
    const uint32_t gx = (ncol + cw - 1) / cw;
    const uint32_t gz = (a.B + RPT - 1) / RPT;
    // ~8 CTAs per SM; each phase gets a multiple of 32 buckets
    const uint64_t per = uint64_t(gx) * gz;
    uint64_t nsplit = (uint64_t(num_sms) * 8 + per - 1) / per;
    const uint64_t unit = 32ull * phases;
    const uint64_t max_split = (a.nb + unit - 1) / unit;
    if (nsplit > max_split) nsplit = max_split;
    if (nsplit < 1) nsplit = 1;
    uint64_t bpc = (a.nb + nsplit - 1) / nsplit;
    bpc = (bpc + unit - 1) / unit * unit;
    nsplit = (a.nb + bpc - 1) / bpc;
    if (nsplit < 1) nsplit = 1;
    k_scan_direct<RPT, W><<<dim3(gz, gx, uint32_t(nsplit)), DIRECT_NT, 0, a.stream>>>(
        a.db, a.nb, a.S, a.q, a.q_stride, a.B, a.out, uint32_t(bpc), cw);
    *nsplit_out = uint32_t(nsplit);
    return cudaGetLastError();
}

cudaError_t launch_scan_direct(const ScanArgs& a, int num_sms, uint32_t* nsplit_out) {
    // B > 4: 32 bytes per thread (one predicate feeds 8 XORs) when the bucket allows
    // it; request tiles of at most 8 keep the accumulators in 64 registers
    // (HBM-bound batches of <= 4 keep 16-byte columns: more threads per bucket row)
    // Request tiles of 6 (80 registers, 3 CTAs per SM) beat tiles of 8 (128, 2 per SM)
    // when B = 9..12 — two tiles of 6 instead of two of 8 where the second is
    // half empty (1 GiB store: 0.30 vs 0.37 ms at B = 12; B = 16 stays on tiles of 8)
    if (a.S % 32 == 0 && a.B > 4) {
        if (a.B <= 6 || (a.B > 8 && a.B <= 12)) return launch_direct_t<6, 2>(a, num_sms, nsplit_out);
        return launch_direct_t<8, 2>(a, num_sms, nsplit_out);
    }
    if (a.B <= 1) return launch_direct_t<1, 1>(a, num_sms, nsplit_out);
    if (a.B <= 2) return launch_direct_t<2, 1>(a, num_sms, nsplit_out);
    if (a.B <= 4) return launch_direct_t<4, 1>(a, num_sms, nsplit_out);
    if (a.B <= 8) return launch_direct_t<8, 1>(a, num_sms, nsplit_out);
    return launch_direct_t<16, 1>(a, num_sms, nsplit_out);
}

}  // namespace xpir

// Microbenchmarks that size the scan's on-chip ceilings on the actual part:
// tcgen05.ld (TMEM -> registers) throughput with a warp-uniform, data-dependent
// column address — the access pattern a TMEM-resident byte table would need.
#include <cuda_runtime.h>

#include <cstdint>

#include "scan.cuh"

namespace xpir {

template <int X>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[X]);
template <>
__device__ __forceinline__ void tmem_ld<1>(uint32_t taddr, uint32_t (&r)[1]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r[0]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<2>(uint32_t taddr, uint32_t (&r)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n"
                 : "=r"(r[0]), "=r"(r[1])
                 : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<4>(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}

// NW warps per CTA, one CTA per SM. Each warp loads from its own lane quadrant.
template <int X, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_tmem_probe(uint32_t iters, uint32_t* sink, unsigned long long* cycles) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t base = tbase + (uint32_t((warp & 3) * 32) << 16);
    if (warp < 4) {  // fill this quadrant: 512 columns
        for (int c = 0; c < 512; ++c) {
            uint32_t v = c * 0x9e3779b9u + lane;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(base + c), "r"(v));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    uint32_t acc[X];
#pragma unroll
    for (int k = 0; k < X; ++k) acc[k] = 0;
    uint32_t idx = warp * 7;
    const unsigned long long t0 = clock64();
    for (uint32_t it = 0; it < iters; ++it) {
        uint32_t r[8][X];
#pragma unroll
        for (int j = 0; j < 8; ++j) tmem_ld<X>(base + ((idx + j * 37) & (511 & ~(X - 1))), r[j]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int k = 0; k < X; ++k) acc[k] ^= r[j][k];
        idx = (idx + (acc[0] & 3) + 1) & 511;
    }
    const unsigned long long t1 = clock64();
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < X; ++k) x ^= acc[k];
    if (x == 0x12345678u) sink[0] = x;
    if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

// Mixed probe: every warp interleaves LDS.128 table-style lookups (smem) with
// tcgen05.ld.x4 + tcgen05.st.x4 read-modify-writes of its TMEM columns — the
// traffic mix of a scan that keeps half its accumulators in TMEM. Reports the
// combined smem+TMEM bytes per SM clock. MODE 0: smem only, 1: TMEM rmw only, 2: both.
template <int MODE>
__global__ void __launch_bounds__(512, 1) k_mix_probe(uint32_t iters, uint32_t* sink, unsigned long long* cycles) {
    __shared__ uint32_t tbase;
    __shared__ __align__(16) uint4 tab[2048];  // 256 rows x 128 B
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) tab[i] = make_uint4(i, i * 3, i * 5, i * 7);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // warp w: lanes of quadrant w%4, columns [(w/4)*128, +128)
    const uint32_t tcol = tbase + (uint32_t((warp & 3) * 32) << 16) + (warp >> 2) * 128;
    const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(tab)) + (lane & 7) * 16;
    uint4 acc = make_uint4(lane, 0, 0, 0);
    uint32_t idx = warp * 13 + (lane >> 3);
    const unsigned long long t0 = clock64();
    for (uint32_t it = 0; it < iters; ++it) {
        if (MODE != 1) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                uint4 v;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(sb + ((idx + j * 29) & 255) * 128));
                acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
            }
        }
        if (MODE != 0) {
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint32_t a = tcol + ((it * 4 + s) & 31) * 4;
                uint32_t r0, r1, r2, r3;
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                             : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                             : "r"(a));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n");
                r0 ^= acc.x; r1 ^= acc.y; r2 ^= acc.z; r3 ^= acc.w;
                asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(a), "r"(r0),
                             "r"(r1), "r"(r2), "r"(r3));
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n");
        }
        idx += acc.x & 7;
    }
    const unsigned long long t1 = clock64();
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) sink[0] = acc.x;
    if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

template <int MODE>
static cudaError_t run_mix(int num_sms, double* bytes_per_clk_sm) {
    uint32_t* sink;
    unsigned long long* cyc;
    cudaError_t e = cudaMalloc(&sink, 16);
    if (e != cudaSuccess) return e;
    cudaMalloc(&cyc, 8);
    cudaMemset(cyc, 0, 8);
    const uint32_t iters = 2048;
    k_mix_probe<MODE><<<num_sms, 512>>>(16, sink, cyc);
    cudaMemset(cyc, 0, 8);
    k_mix_probe<MODE><<<num_sms, 512>>>(iters, sink, cyc);
    unsigned long long c = 0;
    e = cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaGetLastError();
    // per iteration per warp: smem 8 x 512 B; TMEM 4 x (512 B ld + 512 B st)
    const double per_it = (MODE != 1 ? 8 * 512.0 : 0) + (MODE != 0 ? 4 * 1024.0 : 0);
    if (bytes_per_clk_sm && c) *bytes_per_clk_sm = 16.0 * iters * per_it / double(c);
    cudaFree(sink);
    cudaFree(cyc);
    return e;
}

template <int X, int NW>
static cudaError_t run_probe(int num_sms, double* bytes_per_clk_sm) {
    uint32_t* sink;
    unsigned long long* cyc;
    cudaError_t e = cudaMalloc(&sink, 16);
    if (e != cudaSuccess) return e;
    cudaMalloc(&cyc, 8);
    cudaMemset(cyc, 0, 8);
    const uint32_t iters = 4096;
    k_tmem_probe<X, NW><<<num_sms, NW * 32>>>(16, sink, cyc);
    cudaMemset(cyc, 0, 8);
    k_tmem_probe<X, NW><<<num_sms, NW * 32>>>(iters, sink, cyc);
    unsigned long long c = 0;
    e = cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaGetLastError();
    // bytes moved per SM: NW warps x iters x 8 loads x 32 lanes x X words x 4 B
    if (bytes_per_clk_sm && c) *bytes_per_clk_sm = double(NW) * iters * 8 * 32 * X * 4 / double(c);
    cudaFree(sink);
    cudaFree(cyc);
    return e;
}

cudaError_t run_tmem_probe(int variant, int num_sms, double* bytes_per_clk_sm) {
    switch (variant) {
        case 0: return run_probe<1, 4>(num_sms, bytes_per_clk_sm);
        case 1: return run_probe<1, 16>(num_sms, bytes_per_clk_sm);
        case 2: return run_probe<2, 16>(num_sms, bytes_per_clk_sm);
        case 3: return run_probe<4, 16>(num_sms, bytes_per_clk_sm);
        case 4: return run_probe<4, 8>(num_sms, bytes_per_clk_sm);
        case 5: return run_mix<0>(num_sms, bytes_per_clk_sm);
        case 6: return run_mix<1>(num_sms, bytes_per_clk_sm);
        default: return run_mix<2>(num_sms, bytes_per_clk_sm);
    }
}

}  // namespace xpir

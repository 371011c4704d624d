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
        default: return run_probe<4, 8>(num_sms, bytes_per_clk_sm);
    }
}

}  // namespace xpir

// K1/K2/K3/K4 — the PIR read scan on sm_100a.
//
// Reference semantics (bit-exact target):
//   pir::answer_batch (pir.cpp:41-52): out_r = XOR_{j < N : q_r bit j} bucket_j,
//     bit j = q_r[j/8] >> (j%8) & 1 (pir.hpp:25); bits >= N are ignored.
//   pir::mask_answer (pir.cpp:65-69): out_r ^= ChaCha20(mask_seed_r, nonce 0)[0:S].
//   crypto::prng_expand (crypto.cpp:35-45) for seed-expanded query vectors.
//   pir::reconstruct / combine_masked (pir.cpp:54-73) for the cross-shard reduce.
//
// Two scan kernels:
//   k_scan_m4rm   — batches >= ~128: "four Russians" byte tables. Query byte g of
//                   request r is exactly the 8-bit selection of buckets 8g..8g+7,
//                   so per 128-byte column slice the CTA builds the 256-row table
//                   T_g[x] = XOR_{i: bit i of x} bucket_{8g+i} in shared memory
//                   (Gray-code order, one XOR per row), and every request does ONE
//                   16-byte LDS + 4 XORs per 8 buckets instead of 8 masked XORs.
//                   Shared-memory bandwidth (128 B/clk/SM) is the bound.
//   k_scan_direct — small batches: stream the shard once through registers and
//                   XOR 16-byte words under warp-uniform selection bits (HBM bound).
#include <cuda_runtime.h>

#include <cstdint>

#include "prims.cuh"
#include "scan.cuh"

namespace xpir {

// ---------------------------------------------------------------------------
// small PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte cp.async with zero-fill when src_bytes == 0.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ void red_xor64(uint8_t* p, uint64_t v) {
    atomicXor(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
}

// Byte-granular fallback for bucket sizes that are not a multiple of 16 (the
// reference's own tests use 1-, 8- and 12-byte buckets). One thread per
// (request, byte).
__global__ void k_scan_bytes(const uint8_t* __restrict__ db, uint32_t nb, uint32_t S,
                             const uint8_t* __restrict__ q, uint64_t q_stride, uint32_t B,
                             uint8_t* __restrict__ out) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= uint64_t(B) * S) return;
    const uint32_t r = uint32_t(t / S), k = uint32_t(t - uint64_t(r) * S);
    const uint8_t* qr = q + uint64_t(r) * q_stride;
    uint8_t acc = 0;
    for (uint32_t j = 0; j < nb; ++j)
        if ((qr[j >> 3] >> (j & 7)) & 1) acc ^= db[uint64_t(j) * S + k];
    out[t] ^= acc;
}

// ---------------------------------------------------------------------------
// K3: out[r] = mask pad (prng_expand(mask_seed_r, S)) or zero — applied before
// the scan XOR-accumulates into it, so the mask costs one write pass.
// ---------------------------------------------------------------------------
__global__ void k_init_out(uint8_t* __restrict__ out, uint32_t B, uint32_t S,
                           const uint8_t* __restrict__ mask_seeds, int xor_into) {
    const uint32_t nblk = (S + 63) / 64;
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= uint64_t(B) * nblk) return;
    const uint32_t r = uint32_t(t / nblk), blk = uint32_t(t - uint64_t(r) * nblk);
    uint32_t ks[16];
    if (mask_seeds) {
        ChaChaKey key = chacha_key(mask_seeds + uint64_t(r) * 32, 0);
        chacha20_block(key, blk, ks);
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) ks[k] = 0;
    }
    uint8_t* o = out + uint64_t(r) * S + uint64_t(blk) * 64;
    const uint32_t n = min(64u, S - blk * 64);
    if (n == 64 && (S % 16) == 0) {
        uint4* o4 = reinterpret_cast<uint4*>(o);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint4 v = make_uint4(ks[4 * k], ks[4 * k + 1], ks[4 * k + 2], ks[4 * k + 3]);
            if (xor_into) {
                const uint4 a = o4[k];
                v.x ^= a.x; v.y ^= a.y; v.z ^= a.z; v.w ^= a.w;
            }
            o4[k] = v;
        }
    } else {
        for (uint32_t k = 0; k < n; ++k) {
            const uint8_t b = uint8_t(ks[k >> 2] >> (8 * (k & 3)));
            o[k] = xor_into ? uint8_t(o[k] ^ b) : b;
        }
    }
}

// ---------------------------------------------------------------------------
// K2: query expansion. d_q[r*stride + k] = prng_expand(seed_r)[byte_lo + k].
// One thread per 64-byte ChaCha20 block of the window.
// ---------------------------------------------------------------------------
// rows == nullptr: seed r expands into row r; else into row rows[r] (mixed batches)
__global__ void k_expand(const uint8_t* __restrict__ seeds, uint32_t B, uint64_t byte_lo,
                         uint64_t nbytes, uint8_t* __restrict__ qout, uint64_t stride,
                         const uint32_t* __restrict__ rows) {
    const uint64_t blk_lo = byte_lo / 64, blk_hi = (byte_lo + nbytes + 63) / 64;
    const uint64_t nblk = blk_hi - blk_lo;
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= uint64_t(B) * nblk) return;
    const uint32_t r = uint32_t(t / nblk);
    const uint64_t blk = blk_lo + (t - uint64_t(r) * nblk);
    ChaChaKey key = chacha_key(seeds + uint64_t(r) * 32, 0);
    uint32_t ks[16];
    chacha20_block(key, blk, ks);
    const uint64_t b0 = blk * 64;
    uint8_t* o = qout + uint64_t(rows ? rows[r] : r) * stride;
    if (b0 >= byte_lo && b0 + 64 <= byte_lo + nbytes && ((b0 - byte_lo) % 16) == 0 &&
        (stride % 16) == 0) {
        uint4* o4 = reinterpret_cast<uint4*>(o + (b0 - byte_lo));
#pragma unroll
        for (int k = 0; k < 4; ++k) o4[k] = make_uint4(ks[4 * k], ks[4 * k + 1], ks[4 * k + 2], ks[4 * k + 3]);
    } else {
        for (int k = 0; k < 64; ++k) {
            const uint64_t pos = b0 + k;
            if (pos >= byte_lo && pos < byte_lo + nbytes)
                o[pos - byte_lo] = uint8_t(ks[k >> 2] >> (8 * (k & 3)));
        }
    }
}

// ---------------------------------------------------------------------------
// K4: dst ^= XOR_k srcs[k] (srcs may be NVLink peer pointers).
// ---------------------------------------------------------------------------
__global__ void k_xor_reduce(uint8_t* __restrict__ dst, const uint8_t* const* __restrict__ srcs,
                             uint32_t nsrc, uint64_t bytes) {
    const uint64_t n16 = bytes / 16;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
        uint4 a = reinterpret_cast<uint4*>(dst)[i];
        for (uint32_t s = 0; s < nsrc; ++s) {
            const uint4 v = __ldcv(reinterpret_cast<const uint4*>(srcs[s]) + i);
            a.x ^= v.x; a.y ^= v.y; a.z ^= v.z; a.w ^= v.w;
        }
        reinterpret_cast<uint4*>(dst)[i] = a;
    }
    // byte tail
    if (blockIdx.x == 0) {
        for (uint64_t k = n16 * 16 + threadIdx.x; k < bytes; k += blockDim.x) {
            uint8_t a = dst[k];
            for (uint32_t s = 0; s < nsrc; ++s) a ^= srcs[s][k];
            dst[k] = a;
        }
    }
}

// ---------------------------------------------------------------------------
// Microbenchmarks for the roofline denominators.
// k_lop3_peak: 8 independent accumulators per thread, acc ^= w & m — exactly the
// dense select-XOR inner op, one LOP3 each. k_lds_peak: conflict-free LDS.128.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_lop3_peak(uint32_t iters, uint32_t seed, uint32_t* sink) {
    uint32_t a[8], w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        a[k] = seed * (k + 1) + threadIdx.x;
        w[k] = seed ^ (k * 0x9e3779b9u) ^ blockIdx.x;
    }
    uint32_t m = 0u - (threadIdx.x & 1u);
    for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                uint32_t out;
                asm volatile("lop3.b32 %0, %1, %2, %3, 0x78;\n"  // a ^ (w & m)
                             : "=r"(out)
                             : "r"(a[k]), "r"(w[k]), "r"(m));
                a[k] = out;
            }
            m = ~m;
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) x ^= a[k];
    if (x == 0x12345678u) sink[0] = x;
}

__global__ void __launch_bounds__(512) k_lds_peak(uint32_t iters, uint32_t* sink) {
    __shared__ __align__(16) uint4 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
    __syncthreads();
    const uint32_t base = smem_u32(buf) + (threadIdx.x & 7) * 16;
    uint4 acc = make_uint4(0, 0, 0, 0);
    uint32_t idx = threadIdx.x >> 3;
    for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const uint4 v = lds128(base + ((idx + r * 37) & 255) * 128);
            acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
        }
        idx += acc.x & 1;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) sink[0] = acc.x;
}

cudaError_t run_peak_kernels(int num_sms, double* lop3_per_s, double* smem_bps, cudaStream_t s) {
    uint32_t* sink = nullptr;
    cudaError_t e = cudaMalloc(&sink, 16);
    if (e != cudaSuccess) return e;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    const uint32_t it1 = 4096;
    const uint32_t grid1 = num_sms * 8;  // 8 x 256 threads per SM = 64 warps
    k_lop3_peak<<<grid1, 256, 0, s>>>(64, 1, sink);  // warm-up
    cudaEventRecord(a, s);
    k_lop3_peak<<<grid1, 256, 0, s>>>(it1, 1, sink);
    cudaEventRecord(b, s);
    e = cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (lop3_per_s) *lop3_per_s = double(grid1) * 256 * it1 * 16 * 8 / (ms * 1e-3);
    const uint32_t it2 = 2048, grid2 = num_sms * 2;
    k_lds_peak<<<grid2, 512, 0, s>>>(64, sink);
    cudaEventRecord(a, s);
    k_lds_peak<<<grid2, 512, 0, s>>>(it2, sink);
    cudaEventRecord(b, s);
    if (e == cudaSuccess) e = cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (smem_bps) *smem_bps = double(grid2) * 512 * it2 * 16 * 16 / (ms * 1e-3);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e;
}

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------
cudaError_t launch_scan_bytes(const ScanArgs& a) {
    const uint64_t n = uint64_t(a.B) * a.S;
    if (n == 0) return cudaSuccess;
    k_scan_bytes<<<uint32_t((n + 255) / 256), 256, 0, a.stream>>>(a.db, a.nb, a.S, a.q, a.q_stride,
                                                                  a.B, a.out);
    return cudaGetLastError();
}

cudaError_t launch_init_out(uint8_t* out, uint32_t B, uint32_t S, const uint8_t* mask_seeds,
                            bool xor_into, cudaStream_t s) {
    const uint64_t n = uint64_t(B) * ((S + 63) / 64);
    if (n == 0) return cudaSuccess;
    k_init_out<<<uint32_t((n + 255) / 256), 256, 0, s>>>(out, B, S, mask_seeds, xor_into ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_expand(const uint8_t* seeds, uint32_t B, uint64_t byte_lo, uint64_t nbytes,
                          uint8_t* qout, uint64_t stride, cudaStream_t s, const uint32_t* rows) {
    const uint64_t nblk = (byte_lo + nbytes + 63) / 64 - byte_lo / 64;
    const uint64_t n = uint64_t(B) * nblk;
    if (n == 0) return cudaSuccess;
    k_expand<<<uint32_t((n + 127) / 128), 128, 0, s>>>(seeds, B, byte_lo, nbytes, qout, stride, rows);
    return cudaGetLastError();
}

// row k of src (stride ss) -> row idx[k] of dst (stride ds), nbytes each; one warp per row
__global__ void k_scatter_rows(const uint8_t* __restrict__ src, uint64_t ss, uint32_t n,
                               const uint32_t* __restrict__ idx, uint8_t* __restrict__ dst, uint64_t ds,
                               uint64_t nbytes) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n; k += nw) {
        const uint8_t* a = src + uint64_t(k) * ss;
        uint8_t* b = dst + uint64_t(idx[k]) * ds;
        if ((ss % 16) == 0 && (ds % 16) == 0) {
            for (uint64_t j = uint64_t(lane) * 16; j + 16 <= nbytes; j += 32 * 16)
                *reinterpret_cast<uint4*>(b + j) = *reinterpret_cast<const uint4*>(a + j);
            for (uint64_t j = nbytes / 16 * 16 + lane; j < nbytes; j += 32) b[j] = a[j];
        } else {
            for (uint64_t j = lane; j < nbytes; j += 32) b[j] = a[j];
        }
    }
}

cudaError_t launch_scatter_rows(const uint8_t* src, uint64_t ss, uint32_t n, const uint32_t* idx, uint8_t* dst,
                                uint64_t ds, uint64_t nbytes, cudaStream_t s) {
    if (!n || !nbytes) return cudaSuccess;
    uint32_t g = (n + 7) / 8;
    if (g > 148 * 16) g = 148 * 16;
    k_scatter_rows<<<g, 256, 0, s>>>(src, ss, n, idx, dst, ds, nbytes);
    return cudaGetLastError();
}

cudaError_t launch_xor_reduce(uint8_t* dst, const uint8_t* const* d_srcs, uint32_t nsrc,
                              uint64_t bytes, int num_sms, cudaStream_t s) {
    if (bytes == 0 || nsrc == 0) return cudaSuccess;
    uint64_t n16 = bytes / 16 + 1;
    uint32_t g = uint32_t((n16 + 255) / 256);
    if (g > uint32_t(num_sms) * 8) g = uint32_t(num_sms) * 8;
    k_xor_reduce<<<g, 256, 0, s>>>(dst, d_srcs, nsrc, bytes);
    return cudaGetLastError();
}

}  // namespace xpir

// Thin PTX wrappers shared by the sm_100a kernels.
#pragma once
#include <cstdint>

namespace xpir {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte cp.async (L2 only) with zero-fill when src_bytes == 0.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
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
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "r"(addr));
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
// 64-bit XOR reduction into this GPU's global memory.
__device__ __forceinline__ void red_xor64(void* p, uint64_t v) {
    asm volatile("red.relaxed.gpu.global.xor.b64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
// The same into memory other GPUs also reduce into (NVLink peer rows of the fused
// cross-GPU reduce): system scope, so the RMWs of all GPUs are atomic together.
__device__ __forceinline__ void red_xor64_sys(void* p, uint64_t v) {
    asm volatile("red.relaxed.sys.global.xor.b64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

}  // namespace ptx
}  // namespace xpir

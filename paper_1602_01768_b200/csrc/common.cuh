// Shared device helpers for the sm_100a FP64 kernels (DMMA via mma.sync .f64,
// cp.async staging, warp reductions).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace si {

constexpr int kWarp = 32;

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
    // D(8x8) += A(8x4,row) * B(4x8,col); lowers to SASS DMMA.8x8x4.
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero-fill: copies `src_bytes` (0 or BYTES) and zero-fills the rest.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool pred) {
    const int src = pred ? BYTES : 0;
    if constexpr (BYTES == 16) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src));
    } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(smem_u32(smem)), "l"(gmem), "n"(BYTES),
                     "r"(src));
    }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace si

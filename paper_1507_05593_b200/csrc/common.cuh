// Shared device helpers for librsc_b200 (sm_100a, FP64 everywhere).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/rsc_b200.h"

// Diagnostic launch counter (bench.py reports it as gpu_launches); every
// kernel launch site goes through RSC_CHECK_LAUNCH.
void rsc_count_launch();

#define RSC_CHECK_LAUNCH()                                   \
    do {                                                     \
        rsc_count_launch();                                  \
        cudaError_t _e = cudaGetLastError();                 \
        if (_e != cudaSuccess) return (int)_e;               \
    } while (0)

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).  On sm_100a every
// f64 mma.sync shape lowers to SASS DMMA.8x8x4, so m8n8k4 is the native unit.
// Fragment ownership (g = lane>>2, q = lane&3):
//   a = A[g][q], b = B[q][g], c0/c1 = C[g][2q], C[g][2q+1].
__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

// 8-byte cp.async with zero fill when !valid (src-size 0 reads nothing).
__device__ __forceinline__ void cp_async_8(void *smem, const double *gmem, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Warp sums of four per-lane values, all lanes get all four: a reduce-scatter
// butterfly (2 + 1 + 1 + 1 + 1 exchanges) plus 4 broadcasts -- 10 double shuffles
// instead of the 20 of four independent butterflies.
__device__ __forceinline__ void warp_sum4(double (&d)[4]) {
    const int lane = threadIdx.x & 31;
    const bool h16 = lane & 16, h8 = lane & 8;
    double k0 = h16 ? d[2] : d[0], k1 = h16 ? d[3] : d[1];
    const double s0 = h16 ? d[0] : d[2], s1 = h16 ? d[1] : d[3];
    k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
    k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
    double kk = h8 ? k1 : k0;
    kk += __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
    kk += __shfl_xor_sync(0xffffffffu, kk, 4);
    kk += __shfl_xor_sync(0xffffffffu, kk, 2);
    kk += __shfl_xor_sync(0xffffffffu, kk, 1);
#pragma unroll
    for (int s = 0; s < 4; ++s) d[s] = __shfl_sync(0xffffffffu, kk, 8 * s);
}

// Block-wide sum; `red` must hold >= 32 doubles.  Result broadcast to all threads.
__device__ __forceinline__ double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
    if (w == 0) t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
    __syncthreads();
    t = red[0];
    return t;
}

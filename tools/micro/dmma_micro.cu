// DMMA.8x8x4 latency / throughput on this GPU: chains of dependent MMAs with
// NACC independent accumulators per warp and W warps per CTA (one CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void k(double *out, int iters, long long *cyc) {
    double c[NACC][2];
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int NACC>
void run(int warps, int blocks) {
    double *out; long long *cyc;
    cudaMalloc(&out, sizeof(double) * blocks * warps * 32);
    cudaMalloc(&cyc, 8);
    int iters = 4096;
    k<NACC><<<blocks, warps * 32>>>(out, 16, cyc);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<NACC><<<blocks, warps * 32>>>(out, iters, cyc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double flops = 512.0 * NACC * iters * warps * (double)blocks;
    printf("NACC=%2d warps/CTA=%2d CTAs=%4d: %.2f TF/s, %.1f cyc per dependent DMMA (CTA0), %.2f cyc/DMMA/SM\n",
           NACC, warps, blocks, flops / ms / 1e9, (double)c / iters, (double)c / (iters * NACC * warps));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1>(1, 1);
    run<2>(1, 1);
    run<4>(1, 1);
    run<8>(1, 1);
    run<16>(1, 1);
    for (int w : {4, 8, 16, 32}) { run<1>(w, sms); run<4>(w, sms); run<8>(w, sms); run<16>(w, sms); }
    return 0;
}

// MUFU throughput probe: ex2.approx.f32 vs ex2.approx.f16x2 vs ex2.approx.ftz.bf16x2 (sm_100a).
#include <cstdio>
#include <cuda_fp16.h>
__global__ void k32(float* out, int iters) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k16x2(float* out, int iters) {
    unsigned a[8];
    for (int i = 0; i < 8; ++i) { __half2 h = __floats2half2_rn(-0.001f * threadIdx.x, -0.002f * i); a[i] = *(unsigned*)&h; }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
    float s = 0; for (int i = 0; i < 8; ++i) { __half2 h = *(__half2*)&a[i]; s += __low2float(h) + __high2float(h); }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kbf16x2(float* out, int iters) {
    unsigned a[8];
    for (int i = 0; i < 8; ++i) a[i] = 0xBF80BF80u + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
    float s = 0; for (int i = 0; i < 8; ++i) s += (float)(a[i] & 0xffff);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    for (int v = 0; v < 3; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (v == 0) k32<<<blocks, threads>>>(out, iters);
            if (v == 1) k16x2<<<blocks, threads>>>(out, iters);
            if (v == 2) kbf16x2<<<blocks, threads>>>(out, iters);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)blocks * threads * iters * 8 * (v ? 2 : 1);
            if (rep) printf("%s: %.1f Gexp/s = %.1f exp/clk/SM @1.9GHz\n", v == 0 ? "f32" : v == 1 ? "f16x2" : "bf16x2",
                            ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.9e9);
        }
    }
    return 0;
}

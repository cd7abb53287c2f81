// Packed half-precision exp2 probe (sm_100a): is MUFU.EX2 on f16x2 / bf16x2 operands
// two results per issue?  Measures raw throughput (exp/clk/SM, counting 2 per packed op)
// and a softmax-section rate (FFMA2 scale/shift -> pack -> packed ex2 -> P words) for
// 1/2/4 warps per sub-partition, next to the fp32 MUFU path the kernels use today.
// Timed with clock64 inside the kernel.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include "../../paper_2408_12588_b200/csrc/tc_ptx.cuh"
using namespace pab::tc;

template <int MODE>  // 0: f32, 1: f16x2, 2: bf16x2
__global__ void raw(uint32_t* out, long long* cyc, int iters) {
    uint32_t a[16];
    for (int i = 0; i < 16; ++i) {
        float v = -0.001f * (threadIdx.x + i);
        a[i] = MODE == 0 ? __float_as_uint(v) : (MODE == 1 ? 0xbc00bc00u : pack_bf16(v, v * 0.5f));
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(a[i]));
            if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
            if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
        }
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < 16; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + (threadIdx.x >> 5)] = t1 - t0;
}

__device__ __forceinline__ uint32_t cvt_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

template <int MODE>  // 0: f32 MUFU + F2FP pack (today's kernel), 1: f16x2, 2: bf16x2
__global__ void section(const float* in, uint32_t* out, long long* cyc, int iters) {
    float s[112];
    for (int i = 0; i < 112; ++i) s[i] = in[(threadIdx.x + i) & 1023];
    uint32_t acc = 0;
    float m = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const unsigned long long sc2 = f2_pack(0.17f, 0.17f), nm2 = f2_pack(-m, -m);
        uint32_t pk[56];
#pragma unroll
        for (int q = 0; q < 56; ++q) {
            float2 x = f2_unpack(f2_fma(f2_pack(s[2 * q], s[2 * q + 1]), sc2, nm2));
            if (MODE == 0) {
                pk[q] = pack_bf16(fast_exp2(x.x), fast_exp2(x.y));
            } else if (MODE == 1) {
                uint32_t h = cvt_f16x2(x.x, x.y);
                asm("ex2.approx.f16x2 %0, %0;" : "+r"(h));
                pk[q] = h;
            } else {
                uint32_t h = cvt_bf16x2(x.x, x.y);
                asm("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h));
                pk[q] = h;
            }
        }
#pragma unroll
        for (int q = 0; q < 56; ++q) acc ^= pk[q];
        m += 1e-7f * (float)(acc & 1);
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + (threadIdx.x >> 5)] = t1 - t0;
}

// accuracy of the packed paths against exp2f on a sweep of softmax arguments in [-20, 0]
__global__ void accuracy(float* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const float x = -20.0f * (float)i / (float)(gridDim.x * blockDim.x);
    const float ref = exp2f(x);
    uint32_t h = cvt_f16x2(x, x);
    asm("ex2.approx.f16x2 %0, %0;" : "+r"(h));
    const float f16v = __half2float(__ushort_as_half((unsigned short)(h & 0xffff)));
    uint32_t b = cvt_bf16x2(x, x);
    asm("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(b));
    const float bf16v = __uint_as_float(b << 16);
    const float bfround = __uint_as_float(pack_bf16(ref, ref) << 16);  // bf16 rounding of the exact value
    err[3 * i + 0] = fabsf(f16v - ref) / ref;
    err[3 * i + 1] = fabsf(bf16v - ref) / ref;
    err[3 * i + 2] = fabsf(bfround - ref) / ref;
}

static long long max_cycles(long long* cyc, int warps) {
    static long long h[148 * 32];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int b = 0; b < 148; ++b)
        for (int w = 0; w < warps; ++w) mx = h[b * 32 + w] > mx ? h[b * 32 + w] : mx;
    return mx;
}

int main() {
    float* in; uint32_t* out; long long* cyc; float* err;
    cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 32 * 8);
    cudaMemset(cyc, 0, 148 * 32 * 8);
    const int iters = 200;
    const char* nm[] = {"f32", "f16x2", "bf16x2"};
    for (int mode = 0; mode < 3; ++mode)
        for (int warps : {4, 8, 16}) {
            for (int r = 0; r < 2; ++r) {
                if (mode == 0) raw<0><<<148, warps * 32>>>(out, cyc, iters * 8);
                if (mode == 1) raw<1><<<148, warps * 32>>>(out, cyc, iters * 8);
                if (mode == 2) raw<2><<<148, warps * 32>>>(out, cyc, iters * 8);
            }
            cudaDeviceSynchronize();
            const long long mx = max_cycles(cyc, warps);
            const double per = mode == 0 ? 1.0 : 2.0;
            printf("raw %-7s warps/SMSP %2d: %.2f exp/clk/SM\n", nm[mode], warps / 4,
                   per * 16.0 * iters * 8 * warps * 32 / mx);
        }
    for (int mode = 0; mode < 3; ++mode)
        for (int warps : {4, 8, 16}) {
            for (int r = 0; r < 2; ++r) {
                if (mode == 0) section<0><<<148, warps * 32>>>(in, out, cyc, iters);
                if (mode == 1) section<1><<<148, warps * 32>>>(in, out, cyc, iters);
                if (mode == 2) section<2><<<148, warps * 32>>>(in, out, cyc, iters);
            }
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            const long long mx = max_cycles(cyc, warps);
            printf("section %-7s warps/SMSP %2d: %7.1f clk per 112-col section per warp, %.2f exp/clk/SM\n",
                   nm[mode], warps / 4, (double)mx / iters, 112.0 * iters * warps * 32 / mx);
        }
    const int n = 148 * 256;
    cudaMalloc(&err, 3 * n * 4);
    accuracy<<<148, 256>>>(err);
    static float h[3 * 148 * 256];
    cudaMemcpy(h, err, sizeof(h), cudaMemcpyDeviceToHost);
    double mx[3] = {0, 0, 0}, mean[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
            mx[k] = h[3 * i + k] > mx[k] ? h[3 * i + k] : mx[k];
            mean[k] += h[3 * i + k] / n;
        }
    printf("rel err over x in [-20,0]: f16x2 max %.3e mean %.3e | bf16x2 max %.3e mean %.3e | "
           "bf16 rounding of exact max %.3e mean %.3e\n", mx[0], mean[0], mx[1], mean[1], mx[2], mean[2]);
    return 0;
}

// Softmax exp-section probe (sm_100a): cycles per 112-column row section for 1/2/4 warps per
// SM sub-partition, MUFU-only vs the attention kernel's 1-in-3 polynomial mix, and raw MUFU.EX2
// throughput.  Timed with clock64 inside the kernel (independent of the SM clock).
#include <cstdio>
#include <cstdint>
#include "../../paper_2408_12588_b200/csrc/tc_ptx.cuh"
using namespace pab::tc;

__device__ __forceinline__ void poly2(float& a, float& b) {
    a = fmaxf(a, -127.0f); b = fmaxf(b, -127.0f);
    const unsigned long long x = f2_pack(a, b);
    const unsigned long long t = f2_add(x, f2_pack(12582912.0f, 12582912.0f));
    const unsigned long long j = f2_add(t, f2_pack(-12582912.0f, -12582912.0f));
    const unsigned long long f = f2_fma(j, f2_pack(-1.0f, -1.0f), x);
    unsigned long long p = f2_fma(f, f2_pack(0.05517132f, 0.05517132f), f2_pack(0.24261054f, 0.24261054f));
    p = f2_fma(p, f, f2_pack(0.69326097f, 0.69326097f));
    p = f2_fma(p, f, f2_pack(0.99992812f, 0.99992812f));
    const float2 pv = f2_unpack(p), tv = f2_unpack(t);
    a = __int_as_float(__float_as_int(pv.x) + (__float_as_int(tv.x) << 23));
    b = __int_as_float(__float_as_int(pv.y) + (__float_as_int(tv.y) << 23));
}

template <int POLY_DIV, int POLY_NUM>
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
            if (POLY_NUM > 0 && (q % POLY_DIV) >= POLY_DIV - POLY_NUM) poly2(x.x, x.y);
            else { x.x = fast_exp2(x.x); x.y = fast_exp2(x.y); }
            pk[q] = pack_bf16(x.x, x.y);
        }
#pragma unroll
        for (int q = 0; q < 56; ++q) acc ^= pk[q];
        m += 1e-7f * (float)(acc & 1);
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + (threadIdx.x >> 5)] = t1 - t0;
}

__global__ void mufu_raw(float* out, long long* cyc, int iters) {
    float a[16];
    for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + (threadIdx.x >> 5)] = t1 - t0;
}

static long long max_cycles(long long* cyc, int warps) {
    long long h[148 * 32];
    cudaMemcpy(h, cyc, 148 * 32 * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int b = 0; b < 148; ++b)
        for (int w = 0; w < warps; ++w) mx = h[b * 32 + w] > mx ? h[b * 32 + w] : mx;
    return mx;
}

int main() {
    float* in; uint32_t* out; long long* cyc; float* fo;
    cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&fo, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 32 * 8);
    cudaMemset(cyc, 0, 148 * 32 * 8);
    const int iters = 200;
    for (int warps : {4, 8, 12, 16}) {
        for (int r = 0; r < 2; ++r) mufu_raw<<<148, warps * 32>>>(fo, cyc, iters * 8);
        cudaDeviceSynchronize();
        long long mx = max_cycles(cyc, warps);
        printf("mufu raw      warps/SMSP %2d: %.2f exp/clk/SM\n", warps / 4, 16.0 * iters * 8 * warps * 32 / mx);
    }
    for (int variant = 0; variant < 4; ++variant) {
        for (int warps : {4, 8, 12, 16}) {
            for (int r = 0; r < 2; ++r) {
                if (variant == 0) section<3, 0><<<148, warps * 32>>>(in, out, cyc, iters);
                if (variant == 1) section<3, 1><<<148, warps * 32>>>(in, out, cyc, iters);
                if (variant == 2) section<2, 1><<<148, warps * 32>>>(in, out, cyc, iters);
                if (variant == 3) section<5, 2><<<148, warps * 32>>>(in, out, cyc, iters);
            }
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            long long mx = max_cycles(cyc, warps);
            const char* nm[] = {"mufu only", "poly 1/3", "poly 1/2", "poly 2/5"};
            printf("%-12s  warps/SMSP %2d: %7.1f clk per 112-col section per warp, %.2f exp/clk/SM\n", nm[variant],
                   warps / 4, (double)mx / iters, 112.0 * iters * warps * 32 / mx);
        }
    }
    return 0;
}

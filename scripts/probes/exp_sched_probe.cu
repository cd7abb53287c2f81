// Softmax exp-section scheduling probe (sm_100a).  exp16_probe showed packed f16x2/bf16x2
// MUFU.EX2 gives no extra throughput (16 exp/clk/SM either way) and that ONE warp per SM
// sub-partition running the kernel's per-pair sequence (FFMA2 -> 2x MUFU.EX2 -> F2FP) reaches
// only ~11.7 exp/clk/SM while a pure MUFU stream reaches 15.8.  This probe asks whether the
// instruction ORDER of the section is what costs the missing 27%:
//   mode 0: per-pair sequence (today's exp_pack), 1-in-3 pairs on the FMA-pipe polynomial
//   mode 1: per-pair sequence, MUFU only
//   mode 2: phased: all FFMA2 scale/shift first (in place), then the exp2 stream, then the
//           F2FP packs, MUFU only
//   mode 3: phased, 1-in-3 pairs on the polynomial, the polynomial work interleaved into the
//           MUFU stream
//   mode 4: per-chunk phased (16 columns at a time: FFMA2 x8, ex2 x16, F2FP x8), MUFU only
//   mode 5: mode 4 with 1-in-3 poly pairs
// Timed with clock64 inside the kernel, 1 and 2 warps per sub-partition.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp_sched_probe exp_sched_probe.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_2408_12588_b200/csrc/tc_ptx.cuh"
using namespace pab::tc;

__device__ __forceinline__ void poly2(float& a, float& b) {
    a = fmaxf(a, -126.0f);
    b = fmaxf(b, -126.0f);
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

__device__ __forceinline__ float ex2v(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int MODE>
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
        if (MODE == 0 || MODE == 1) {
#pragma unroll
            for (int q = 0; q < 56; ++q) {
                float2 x = f2_unpack(f2_fma(f2_pack(s[2 * q], s[2 * q + 1]), sc2, nm2));
                if (MODE == 0 && q % 3 == 2) {
                    poly2(x.x, x.y);
                } else {
                    x.x = fast_exp2(x.x);
                    x.y = fast_exp2(x.y);
                }
                pk[q] = pack_bf16(x.x, x.y);
            }
        } else if (MODE == 2 || MODE == 3) {
            float x[112];
#pragma unroll
            for (int q = 0; q < 56; ++q) {
                float2 v = f2_unpack(f2_fma(f2_pack(s[2 * q], s[2 * q + 1]), sc2, nm2));
                x[2 * q] = v.x;
                x[2 * q + 1] = v.y;
            }
#pragma unroll
            for (int q = 0; q < 56; ++q) {
                if (MODE == 3 && q % 3 == 2) {
                    poly2(x[2 * q], x[2 * q + 1]);
                } else {
                    x[2 * q] = ex2v(x[2 * q]);
                    x[2 * q + 1] = ex2v(x[2 * q + 1]);
                }
            }
#pragma unroll
            for (int q = 0; q < 56; ++q) pk[q] = pack_bf16(x[2 * q], x[2 * q + 1]);
        } else {
#pragma unroll
            for (int c = 0; c < 7; ++c) {
                float x[16];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float2 v = f2_unpack(f2_fma(f2_pack(s[16 * c + 2 * q], s[16 * c + 2 * q + 1]), sc2, nm2));
                    x[2 * q] = v.x;
                    x[2 * q + 1] = v.y;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (MODE == 5 && (8 * c + q) % 3 == 2) {
                        poly2(x[2 * q], x[2 * q + 1]);
                    } else {
                        x[2 * q] = ex2v(x[2 * q]);
                        x[2 * q + 1] = ex2v(x[2 * q + 1]);
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) pk[8 * c + q] = pack_bf16(x[2 * q], x[2 * q + 1]);
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

static long long max_cycles(long long* cyc, int warps) {
    static long long h[148 * 32];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int b = 0; b < 148; ++b)
        for (int w = 0; w < warps; ++w) mx = h[b * 32 + w] > mx ? h[b * 32 + w] : mx;
    return mx;
}

template <int MODE>
void run(const float* in, uint32_t* out, long long* cyc, int iters) {
    const char* nm[] = {"per-pair poly1/3", "per-pair mufu", "phased mufu", "phased poly1/3",
                        "chunk16 mufu", "chunk16 poly1/3"};
    for (int warps : {4, 8}) {
        for (int r = 0; r < 2; ++r) section<MODE><<<148, warps * 32>>>(in, out, cyc, iters);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("err %s\n", cudaGetErrorString(e));
            return;
        }
        const long long mx = max_cycles(cyc, warps);
        printf("%-18s warps/SMSP %d: %7.1f clk per 112-col section per warp, %.2f exp/clk/SM\n", nm[MODE],
               warps / 4, (double)mx / iters, 112.0 * iters * warps * 32 / mx);
    }
}

int main() {
    float* in;
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&in, 4096 * 4);
    cudaMemset(in, 0, 4096 * 4);
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 32 * 8);
    cudaMemset(cyc, 0, 148 * 32 * 8);
    const int iters = 200;
    run<0>(in, out, cyc, iters);
    run<1>(in, out, cyc, iters);
    run<2>(in, out, cyc, iters);
    run<3>(in, out, cyc, iters);
    run<4>(in, out, cyc, iters);
    run<5>(in, out, cyc, iters);
    return 0;
}

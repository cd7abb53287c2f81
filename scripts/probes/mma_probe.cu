// Microbenchmark: tcgen05.mma throughput of the attention kernel's MMA shapes/layouts.
// One CTA per SM; an elected thread issues `iters` rounds of a chosen MMA group, then
// commits and waits; clock64 per round is reported.  Data is garbage (timing only).
#include "../../paper_2408_12588_b200/csrc/tc_ptx.cuh"
#include <cstdio>
using namespace pab::tc;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

__global__ void __launch_bounds__(256, 1) probe(int mode, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    for (int i = threadIdx.x * 16; i < 200 * 1024; i += 128 * 16) *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
    fence_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = tbase;
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (warp >= 4 && (mode == 7 || mode == 8 || mode == 21)) {
        // TMEM traffic of the softmax warps: ld 128 S columns (+ st 64 P columns in mode 8)
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        float acc = 0.f;
        if (mode == 21) {  // MUFU-heavy helpers (softmax exp phase stand-in)
            float x = (float)threadIdx.x * 1e-3f;
            while (!done) {
#pragma unroll 16
                for (int i = 0; i < 64; ++i) x = fast_exp2(x) * 0.5f;
                acc += x;
            }
        } else
        while (!done) {
            for (int t = 0; t < 2; ++t) {
                float v[32];
                for (int q = 0; q < 4; ++q) {
                    PAB_TMEM_LD32(tmem + lane_off + 128 * t + 32 * q, v);
                    tmem_wait_ld();
                    acc += v[q];
                }
                if (mode == 8) {
                    for (int q = 0; q < 4; ++q) PAB_TMEM_ST16(tmem + lane_off + 128 * t + 16 * q, v);
                    tmem_wait_st();
                }
            }
        }
        if (acc == 1234.5f) out[1] = 1;
    }
    if (threadIdx.x == 0) {
        const uint32_t base = smem_u32(smem);
        const uint64_t dq128 = smem_desc(base, 16, 1024, kLayoutSW128), dk128 = smem_desc(base + 40960, 16, 1024, kLayoutSW128);
        const uint64_t dq32 = smem_desc(base + 16384, 16, 256, kLayoutSW32), dk32 = smem_desc(base + 40960 + 16384, 16, 256, kLayoutSW32);
        const uint64_t dv = smem_desc(base + 81920, 4096, 256, kLayoutSW32);
        const uint64_t dv128 = smem_desc(base + 81920, 8192, 1024, kLayoutSW128);   // MN-major SW128: 64-col atoms
        const uint64_t dp = smem_desc(base + 122880, 16, 1024, kLayoutSW128);
        const uint32_t idS = idesc_bf16(128, 128, 0), idO = idesc_bf16(128, 80, 1), idO64 = idesc_bf16(128, 64, 1),
                       idO16 = idesc_bf16(128, 16, 1);
        long long t0 = clock64();
        if (mode == 21) mode = 20;
        if (mode >= 9) {
            const uint32_t idS256 = idesc_bf16(128, 256, 0);
            for (int it = 0; it < iters; ++it) {
                if (mode == 9) {  // S of both tiles, K-steps interleaved across the two accumulators
                    for (int k = 0; k < 5; ++k)
                        for (int t = 0; t < 2; ++t)
                            mma_ss(tmem + 128 * t, dq128 + ((32 * k) >> 4), dk128 + ((32 * k) >> 4), idS, k > 0);
                }
                if (mode == 10) {  // PV of both tiles interleaved
                    for (int k = 0; k < 8; ++k)
                        for (int t = 0; t < 2; ++t)
                            mma_ts(tmem + 256 + 128 * t, tmem + 128 * t + 8 * k, dv + ((512 * k) >> 4), idO, 1);
                }
                if (mode == 11) {  // one S of N = 256 per round (K = 80): same MACs as mode 1
                    for (int k = 0; k < 5; ++k) mma_ss(tmem, dq128 + ((32 * k) >> 4), dk128 + ((32 * k) >> 4), idS256, k > 0);
                }
                if (mode == 13) {  // PV SS 2 tiles interleaved
                    for (int k = 0; k < 8; ++k)
                        for (int t = 0; t < 2; ++t)
                            mma_ss(tmem + 256 + 128 * t, dp + ((((k >> 2) * 16384) + 32 * (k & 3)) >> 4), dv + ((512 * k) >> 4), idO, 1);
                }
                if (mode == 14) {  // PV TS 4 accumulators interleaved (O cols 256,336,416 + 176)
                    const uint32_t dd[4] = {256, 336, 416, 176};
                    for (int k = 0; k < 8; ++k)
                        for (int t = 0; t < 4; ++t)
                            mma_ts(tmem + dd[t], tmem + 64 * (t & 1) + 8 * k, dv + ((512 * k) >> 4), idO, 1);
                }
                if (mode == 15 || mode == 16) {  // per tile: S(5, SS) interleaved 1:1 with PV(8, TS or SS), 2 tiles
                    for (int t = 0; t < 2; ++t) {
                        int ks = 0, kp = 0;
                        while (ks < 5 || kp < 8) {
                            if (ks < 5) { mma_ss(tmem + 128 * t, dq128 + ((32 * ks) >> 4), dk128 + ((32 * ks) >> 4), idS, ks > 0); ++ks; }
                            if (kp < 8) {
                                if (mode == 15) mma_ts(tmem + 256 + 128 * t, tmem + 448 + 8 * (kp & 7) * 0, dv + ((512 * kp) >> 4), idO, 1);
                                else mma_ss(tmem + 256 + 128 * t, dp + ((((kp >> 2) * 16384) + 32 * (kp & 3)) >> 4), dv + ((512 * kp) >> 4), idO, 1);
                                ++kp;
                            }
                        }
                    }
                }
                if (mode == 17) {  // S of tile 1 interleaved with PV(TS) of tile 0, then S of tile 0 with PV of tile 1
                    for (int t = 0; t < 2; ++t) {
                        int ks = 0, kp = 0;
                        while (ks < 5 || kp < 8) {
                            if (kp < 8) { mma_ts(tmem + 256 + 128 * t, tmem + 128 * t + 8 * kp, dv + ((512 * kp) >> 4), idO, 1); ++kp; }
                            if (ks < 5) { mma_ss(tmem + 128 * (1 - t), dq128 + ((32 * ks) >> 4), dk128 + ((32 * ks) >> 4), idS, ks > 0); ++ks; }
                        }
                    }
                }
                if (mode == 18 || mode == 20) {  // S N=112, 2 tiles interleaved, 5 k-steps
                    const uint32_t idS112 = idesc_bf16(128, 112, 0);
                    for (int k = 0; k < 5; ++k)
                        for (int t = 0; t < 2; ++t)
                            mma_ss(tmem + 112 * t, dq128 + ((32 * (k & 3)) >> 4), dk128 + ((32 * (k & 3)) >> 4), idS112, k > 0);
                }
                if (mode == 19 || mode == 20) {  // PV 7 k-steps, N=80, 2 tiles interleaved, P at 384/448
                    for (int k = 0; k < 7; ++k)
                        for (int t = 0; t < 2; ++t)
                            mma_ts(tmem + 224 + 80 * t, tmem + 384 + 64 * t + 8 * k, dv + ((512 * k) >> 4), idO, 1);
                }
                if (mode == 12) {  // S of 4 accumulators (N = 64 each... here N=128 into 4 x 128 cols) interleaved
                    for (int k = 0; k < 5; ++k)
                        for (int t = 0; t < 4; ++t)
                            mma_ss(tmem + 128 * t, dq128 + ((32 * k) >> 4), dk128 + ((32 * k) >> 4), idS, k > 0);
                }
            }
        } else
        for (int it = 0; it < iters; ++it) {
            for (int t = 0; t < 2; ++t) {
                const uint32_t d_s = tmem + 128 * t, d_o = tmem + 256 + 128 * t;
                if (mode == 0 || mode == 1 || mode == 5 || mode == 7 || mode == 8) {  // S: 4 x SW128 k16 + 1 x SW32 k16
                    for (int k = 0; k < 4; ++k) mma_ss(d_s, dq128 + ((32 * k) >> 4), dk128 + ((32 * k) >> 4), idS, k > 0);
                    mma_ss(d_s, dq32, dk32, idS, 1);
                }
                if (mode == 4) {  // S without the SW32 block (K = 64)
                    for (int k = 0; k < 4; ++k) mma_ss(d_s, dq128 + ((32 * k) >> 4), dk128 + ((32 * k) >> 4), idS, k > 0);
                }
                if (mode == 0 || mode == 2 || mode == 7 || mode == 8) {  // PV: A = P from TMEM, B = V MN-major SW32 atoms, N = 80
                    for (int k = 0; k < 8; ++k) mma_ts(d_o, d_s + 8 * k, dv + ((512 * k) >> 4), idO, 1);
                }
                if (mode == 3 || mode == 5) {  // PV with P in smem (SS)
                    for (int k = 0; k < 8; ++k)
                        mma_ss(d_o, dp + ((((k >> 2) * 16384) + 32 * (k & 3)) >> 4), dv + ((512 * k) >> 4), idO, 1);
                }
                if (mode == 6) {  // PV: TS, V as MN-major SW128 (N=64) + SW32 (N=16)
                    for (int k = 0; k < 8; ++k) {
                        mma_ts(d_o, d_s + 8 * k, dv128 + ((1024 * 2 * k) >> 4), idO64, 1);
                        mma_ts(d_o + 64, d_s + 8 * k, dv + ((512 * k) >> 4), idO16, 1);
                    }
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
        done = 1;
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
    long long* d; cudaMalloc(&d, 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[] = {"S+PV(TS,N80) x2tiles", "S only (5 MMA N128)", "PV TS N80 only", "PV SS N80 only", "S K64 only (4 MMA)", "S + PV SS", "PV TS N64 SW128 + N16 SW32", "mode0 + TMEM ld traffic", "mode0 + TMEM ld+st traffic", "S 2 tiles interleaved", "PV 2 tiles interleaved", "S N=256 x5", "S 4 accumulators interleaved", "PV SS 2 tiles interleaved", "PV TS 4 acc interleaved", "S+PV(TS) 1:1 per tile", "S+PV(SS) 1:1 per tile", "S(1-t)+PV(t) TS interleave", "S N112 2x interleaved", "PV 7 steps 2x interleaved", "S112 + PV7 (kernel order)", "same + MUFU helper warps"};
    // per round (2 tiles) ideal clocks at 4096 MAC/clk: S = 2*128*128*80/4096 = 640, PV = 640
    const double ideal[] = {1280, 640, 640, 640, 512, 1280, 640, 1280, 1280, 640, 640, 640, 1280, 640, 1280, 1280, 1280, 1280, 560, 560, 1120, 1120};
    for (int mode = 0; mode < 22; ++mode) {
        const int iters = 200;
        probe<<<148, 256, 200 * 1024>>>(mode, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %d %-28s : %8.1f clk/round (ideal %.0f) %s\n", mode, names[mode], (double)c / iters, ideal[mode], e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}

// Shared helpers for the PAB B200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "../../include/pab_b200.h"

namespace pab {

void set_last_error(const char* what, cudaError_t err);

inline int launch_status(const char* what) {
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        set_last_error(what, err);
        return PAB_ERR_CUDA;
    }
    return PAB_OK;
}

struct PendingList {
    const __nv_bfloat16* p[PAB_MAX_PENDING];
    int n;
    // bit i set: term i is stored token-major, rows (b, s, t) instead of (b, t, s)
    // (the temporal site's output, see pab_residual_modnorm_tm); tm_t/tm_s give T and S
    uint32_t tm_mask;
    int64_t tm_t, tm_s;
    // source row of term i for residual row `row` = (b, t, s)
    __device__ __forceinline__ int64_t src_row(int i, int64_t row) const {
        if (!((tm_mask >> i) & 1u)) return row;
        const int64_t s = row % tm_s, bt = row / tm_s, t = bt % tm_t, b = bt / tm_t;
        return (b * tm_s + s) * tm_t + t;
    }
};

inline PendingList make_pending(const void* const* ptrs, int n) {
    PendingList pl;
    pl.n = n;
    pl.tm_mask = 0;
    pl.tm_t = 1;
    pl.tm_s = 1;
    for (int i = 0; i < PAB_MAX_PENDING; ++i)
        pl.p[i] = (i < n) ? reinterpret_cast<const __nv_bfloat16*>(ptrs[i]) : nullptr;
    return pl;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace pab

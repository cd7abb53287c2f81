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

// Row layouts of a pending residual term (and of a prologue's h output):
//   PAB_LAYOUT_FRAME  rows (b, t, s)              -- the residual stream's own order
//   PAB_LAYOUT_TOKEN  rows (b, s, t)              -- the serial temporal site's output
//   PAB_LAYOUT_A2A    rows (s / (S/W), t, b, s % (S/W)) -- a frame shard in all-to-all order
//                     (the sequence-parallel temporal site's received output, unpacked by the
//                     next prologue instead of a separate permute pass)
struct PendingList {
    const __nv_bfloat16* p[PAB_MAX_PENDING];
    int n;
    uint32_t tm_mask;   // bit i: term i is PAB_LAYOUT_TOKEN
    uint32_t a2a_mask;  // bit i: term i is PAB_LAYOUT_A2A
    int64_t n_b, tm_t, tm_s, n_w;
    // source row of term i for residual row `row` = (b, t, s)
    __device__ __forceinline__ int64_t src_row(int i, int64_t row) const {
        const uint32_t bit = 1u << i;
        if (!((tm_mask | a2a_mask) & bit)) return row;
        const int64_t s = row % tm_s, bt = row / tm_s, t = bt % tm_t, b = bt / tm_t;
        if (tm_mask & bit) return (b * tm_s + s) * tm_t + t;
        const int64_t sw = tm_s / n_w, dst = s / sw;
        return ((dst * tm_t + t) * n_b + b) * sw + (s - dst * sw);
    }
};

inline PendingList make_pending(const void* const* ptrs, int n) {
    PendingList pl;
    pl.n = n;
    pl.tm_mask = 0;
    pl.a2a_mask = 0;
    pl.n_b = 1;
    pl.tm_t = 1;
    pl.tm_s = 1;
    pl.n_w = 1;
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

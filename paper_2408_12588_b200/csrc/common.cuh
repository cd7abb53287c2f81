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
//   PAB_LAYOUT_PEER   the sequence-parallel temporal output read straight out of the W ranks'
//                     token-layout buffers (T, B, S/W, D) over NVLink peer memory: residual row
//                     (b, t, s) of rank `me` lives on rank src = s / (S/W) at token row
//                     ((me * T/W + t) * B + b) * (S/W) + s % (S/W)  (no all-to-all at all)
struct PendingList {
    const __nv_bfloat16* p[PAB_MAX_PENDING];
    int n;
    uint32_t tm_mask;   // bit i: term i is PAB_LAYOUT_TOKEN
    uint32_t a2a_mask;  // bit i: term i is PAB_LAYOUT_A2A
    uint32_t peer_mask; // bit i: term i is PAB_LAYOUT_PEER (sources in peer[])
    int copy_term;      // >= 0: term copy_term is also written frame-major into `copy` (cache slot)
    int64_t n_b, tm_t, tm_s, n_w, me;
    const __nv_bfloat16* peer[PAB_MAX_PEERS];
    __nv_bfloat16* copy;
    // source row of term i for residual row `row` = (b, t, s)
    __device__ __forceinline__ int64_t src_row(int i, int64_t row) const {
        const uint32_t bit = 1u << i;
        if (!((tm_mask | a2a_mask) & bit)) return row;
        const int64_t s = row % tm_s, bt = row / tm_s, t = bt % tm_t, b = bt / tm_t;
        if (tm_mask & bit) return (b * tm_s + s) * tm_t + t;
        const int64_t sw = tm_s / n_w, dst = s / sw;
        return ((dst * tm_t + t) * n_b + b) * sw + (s - dst * sw);
    }
    // first element of term i's row for residual row `row`
    __device__ __forceinline__ const __nv_bfloat16* row_ptr(int i, int64_t row, int64_t D) const {
        if (peer_mask & (1u << i)) {
            const int64_t s = row % tm_s, bt = row / tm_s, t = bt % tm_t, b = bt / tm_t;
            const int64_t sw = tm_s / n_w, src = s / sw;
            return peer[src] + (((me * tm_t + t) * n_b + b) * sw + (s - src * sw)) * D;
        }
        return p[i] + src_row(i, row) * D;
    }
};

inline PendingList make_pending(const void* const* ptrs, int n) {
    PendingList pl;
    pl.n = n;
    pl.tm_mask = 0;
    pl.a2a_mask = 0;
    pl.peer_mask = 0;
    pl.copy_term = -1;
    pl.n_b = 1;
    pl.tm_t = 1;
    pl.tm_s = 1;
    pl.n_w = 1;
    pl.me = 0;
    pl.copy = nullptr;
    for (int i = 0; i < PAB_MAX_PENDING; ++i)
        pl.p[i] = (i < n) ? reinterpret_cast<const __nv_bfloat16*>(ptrs[i]) : nullptr;
    for (int i = 0; i < PAB_MAX_PEERS; ++i) pl.peer[i] = nullptr;
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

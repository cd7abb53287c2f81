// Device-side barrier of a sequence-parallel group over NVLink peer memory.
//
// Broadcast SP's frames<->tokens exchange (reference parallel.reshard around the
// temporal site, pkg/src/pab_engine/parallel.py:140-180, 322-348) runs WITHOUT a
// collective in the peer transport: the temporal prologue stores h straight into
// every rank's token-layout receive buffer (pab_residual_modnorm_peer, h_layout
// PAB_LAYOUT_PEER) and the prologue after the temporal site reads the attention
// output straight out of the ranks' token buffers (term layout PAB_LAYOUT_PEER).
// What remains is ordering: a rank may read a buffer only after every writer has
// finished, and may overwrite one only after every reader is done.  Both are one
// barrier each, issued on the compute stream right after the producing kernel:
//
//   prologue (peer stores of h) -> barrier -> QKV GEMM, attention, O GEMM -> barrier
//   -> next prologue (peer loads of o)
//
// The reuse direction is covered by the same two barriers (a rank's next peer
// store into a buffer happens after a barrier that every reader reaches only
// after its last read), see DESIGN.md section 6.
//
// The barrier is epoch based and graph-safe: every rank keeps a device counter;
// a launch bumps it to e, stores e into slot [me] of every rank's flag array with
// st.release.sys, and waits until its own flag array holds >= e in every slot
// (ld.acquire.sys).  Epochs advance identically on all ranks because every rank
// issues the same barriers in the same order (the decision table is global), so a
// CUDA graph replay needs no host-side epoch.  The wait is bounded by a
// %globaltimer deadline: on timeout the kernel records PAB_PEER_TIMEOUT in
// `error` and returns instead of hanging the GPU.
#include "common.cuh"

namespace pab {

struct PeerFlags {
    uint32_t* flags[PAB_MAX_PEERS];  // flags[q]: rank q's W-entry flag array (peer-mapped)
};

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(32) peer_barrier_kernel(PeerFlags f, uint32_t* counter, int me, int n_w,
                                                          uint32_t* error, uint64_t timeout_ns) {
    __shared__ uint32_t epoch;
    if (threadIdx.x == 0) {
        epoch = *counter + 1u;
        *counter = epoch;
    }
    __syncthreads();
    const int q = threadIdx.x;
    if (q >= n_w) return;
    const uint32_t e = epoch;
    // everything this rank wrote before (earlier kernels on this stream, incl. peer
    // stores over NVLink) is ordered before the signal
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_release_sys(f.flags[q] + me, e);
    const uint32_t* mine = f.flags[me] + q;
    const uint64_t t0 = global_ns();
    // wrap-safe comparison of 32-bit epochs
    while ((int32_t)(ld_acquire_sys(mine) - e) < 0) {
        __nanosleep(100);
        if (global_ns() - t0 > timeout_ns) {
            atomicExch(error, (uint32_t)PAB_PEER_TIMEOUT);
            break;
        }
    }
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}

}  // namespace pab

using namespace pab;

extern "C" int pab_peer_barrier(void* const* flags, void* counter, int rank, int n_w, void* error,
                                double timeout_s, void* stream) {
    if (n_w < 1 || n_w > PAB_MAX_PEERS) return PAB_ERR_SHAPE;
    if (rank < 0 || rank >= n_w || flags == nullptr || counter == nullptr || error == nullptr)
        return PAB_ERR_INVALID;
    if (!(timeout_s > 0.0)) return PAB_ERR_INVALID;
    PeerFlags f;
    for (int w = 0; w < PAB_MAX_PEERS; ++w) {
        f.flags[w] = w < n_w ? reinterpret_cast<uint32_t*>(flags[w]) : nullptr;
        if (w < n_w && (f.flags[w] == nullptr || (uintptr_t)f.flags[w] % 4 != 0)) return PAB_ERR_INVALID;
    }
    peer_barrier_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        f, reinterpret_cast<uint32_t*>(counter), rank, n_w, reinterpret_cast<uint32_t*>(error),
        (uint64_t)(timeout_s * 1e9));
    return launch_status("peer_barrier");
}

// tcgen05 / TMEM / TMA flash attention for sm_100a (kernels K1-K3).
//
// reference op: numerics.scaled_dot_attention (pkg/src/pab_engine/numerics.py:133-151)
// as used by the spatial, temporal and cross sites (model.py:327-385).
//
// CTA layout (576 threads, one CTA per SM):
//   warps 0-7   softmax for query tile 0, warps 8-15 for query tile 1; within a
//               tile, warps w and w+4 own the same 32 rows (TMEM lanes) and the
//               left / right 64 score columns, exchanging the row max through smem
//   warp  16    TMA producer (one elected lane)
//   warps 17-18 MMA issuers, one per query tile, so the two tiles' tcgen05.mma
//               streams are issued in parallel (warp 17 also owns TMEM)
// Per KV tile j the MMA lane issues, ping-ponging the two query tiles,
//   S_i = Q_i K_j^T  (M=128, N=128, K=dh padded to 16)  -> TMEM cols [128 i, 128 i + 128)
//   O_i += P_i V_j   (M=128, N=64|16 blocks, K=128)      -> TMEM cols [256 + 128 i, ...)
// while group i turns S_i into P_i (bf16, smem) with an online softmax whose
// running max is only raised (and O rescaled in TMEM) when it grows by more
// than 2^8, so P stays <= 256 and the O correction is rare.
//
// Head dim: dh is split into 64-wide K blocks staged with 128B swizzle plus
// 16-wide blocks with 32B swizzle; the TMA box of the last block runs past dh
// and the hardware zero-fills the padding (72 -> 64 + 16 with 8 zero columns).
//
// "Packed" mode (temporal attention, sequence length T <= 64): one 128-row
// tile holds floor(128/T) independent sequences (consecutive tokens b) and the
// softmax masks the block diagonal, so the short problems still run on
// 128x128 tensor-core tiles; the kernel is HBM-bound there.
#include "common.cuh"
#include "tc_ptx.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <mutex>

namespace pab {

namespace tc {

constexpr int kSoftmaxWarps = 16;
constexpr int kTmaWarp = 16;
constexpr int kMmaWarp = 17;  // MMA issuer for query tile 0 (also owns the TMEM allocation); 18 for tile 1
constexpr int kThreads = 32 * (kSoftmaxWarps + 3);
constexpr int kGroupThreads = 256;  // softmax threads per query tile
constexpr int kRows = 128;       // query rows per tile == TMEM lanes
constexpr int kKv = 128;         // keys per KV tile
constexpr int kPBytes = kRows * kKv * 2;
constexpr uint32_t kTmemCols = 512;

struct Params {
    int n_q, n_k, n_b, heads, dh;
    int packed;        // 0: rows along i; >0: sequences per tile (T = n_k)
    int row_tiles;     // query tiles along the tiled axis
    int n_kv;          // KV tiles per problem
    int n_pairs;       // query-tile pairs per (problem, head)
    int n_items;       // total work items = n_pairs * heads * problems
    float scale_log2;  // scale * log2(e)
    __nv_bfloat16* o;
    int64_t o_sa, o_sb, o_si;
    long long* trace;  // debug: clock64 event log of CTA (0,0,0), nullptr in production
};

// trace slot layout: [(iteration * 2 + t) * 16 + event], iterations < 61 of CTA 0 (scripts/tc_timeline.py)
#ifndef PAB_ATTN_TRACE
#define PAB_TRACE(cond, j, t, ev) \
    do {                          \
    } while (0)
#else
#define PAB_TRACE(cond, j, t, ev)                                                                   \
    do {                                                                                            \
        if (p.trace != nullptr && (cond) && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) \
            p.trace[((j) * 2 + (t)) * 16 + (ev)] = clock64();                                       \
    } while (0)
#endif


#ifndef PAB_POLY_EVERY
#define PAB_POLY_EVERY 8
#endif
#define PAB_POLY_DIV (PAB_POLY_EVERY > 0 ? PAB_POLY_EVERY : 1)

// Softmax building blocks, instantiated separately for full tiles (no masking
// instructions at all) and for the partial / block-diagonal tiles.
template <bool FULL>
__device__ __forceinline__ float row_max_half(uint32_t s_tmem, int lo_c, int hi_c) {
    float mx = -INFINITY;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        float v[32];
        PAB_TMEM_LD32(s_tmem + 32 * q, v);
        tmem_wait_ld();
        if (!FULL) {
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = (32 * q + c >= lo_c && 32 * q + c < hi_c) ? v[c] : -INFINITY;
        }
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1)
#pragma unroll
            for (int c = 0; c < w; ++c) v[c] = fmaxf(v[c], v[c + w]);
        mx = fmaxf(mx, v[0]);
    }
    return mx;
}


// P = exp2(s * scale_log2 - m) for this thread's 64 scores -> bf16 into its 128-byte
// swizzled P row; returns the row-sum contribution.
template <bool FULL>
__device__ __forceinline__ float exp_pack_half(const float* v, float scale_log2, float neg_m, uint32_t p_row,
                                               uint32_t rsw, int lo_c, int hi_c) {
    if (FULL) {
        // x = s * scale_log2 - m for all 64 scores (FFMA2), then all exp2 back to back so
        // the MUFU queue stays full, then row sum (FADD2) + bf16 pack + swizzled stores
        float e[64];
        const unsigned long long sc2 = f2_pack(scale_log2, scale_log2), nm2 = f2_pack(neg_m, neg_m);
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
            const float2 x = f2_unpack(f2_fma(f2_pack(v[c], v[c + 1]), sc2, nm2));
            e[c] = x.x;
            e[c + 1] = x.y;
        }
#pragma unroll
        for (int c = 0; c < 64; ++c)
            // optionally every PAB_POLY_EVERY-th score on the FMA pipe (polynomial exp2)
            e[c] = (PAB_POLY_EVERY > 0 && (c % PAB_POLY_DIV) == PAB_POLY_DIV - 1) ? poly_exp2(e[c]) : fast_exp2(e[c]);
        unsigned long long acc2[2] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f)};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
#pragma unroll
            for (int c = 0; c < 8; c += 2)
                acc2[(c >> 1) & 1] = f2_add(acc2[(c >> 1) & 1], f2_pack(e[8 * k + c], e[8 * k + c + 1]));
            st_shared_v4(p_row + ((((uint32_t)k) ^ rsw) << 4), pack_bf16(e[8 * k], e[8 * k + 1]),
                         pack_bf16(e[8 * k + 2], e[8 * k + 3]), pack_bf16(e[8 * k + 4], e[8 * k + 5]),
                         pack_bf16(e[8 * k + 6], e[8 * k + 7]));
        }
        const float2 a0 = f2_unpack(acc2[0]), a1 = f2_unpack(acc2[1]);
        return (a0.x + a0.y) + (a1.x + a1.y);
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        float e[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            e[c] = fast_exp2(fmaf(v[8 * k + c], scale_log2, neg_m));
            e[c] = (8 * k + c >= lo_c && 8 * k + c < hi_c) ? e[c] : 0.f;
            acc[c & 3] += e[c];
        }
        st_shared_v4(p_row + ((((uint32_t)k) ^ rsw) << 4), pack_bf16(e[0], e[1]), pack_bf16(e[2], e[3]),
                     pack_bf16(e[4], e[5]), pack_bf16(e[6], e[7]));
    }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}


// ------------------------------------------------------------- the kernel
template <int N128, int N32>
struct Geometry {
    static constexpr int kDhPad = 64 * N128 + 16 * N32;
    static constexpr int kTileBytes = N128 * 16384 + N32 * 4096;  // one 128-row operand tile
    static constexpr int kQ0 = 0;
    static constexpr int kK0 = 2 * kTileBytes;     // 3 K stages (K runs ahead of V: S(j+1) before PV(j))
    static constexpr int kV0 = 5 * kTileBytes;     // 2 V stages
    static constexpr int kP0 = 7 * kTileBytes;     // 2 P tiles
    static constexpr int kX0 = kP0 + 2 * kPBytes;  // row max / row sum exchange: [tile][half][slot][128] f32
    static constexpr int kBar = kX0 + 2 * 2 * 3 * kRows * 4;
    static constexpr int kSmem = kBar + 256 + 1024;  // + barriers + alignment slack
    static_assert(kSmem <= 232448, "attention tiles exceed the 227 KB shared memory of one CTA");
};

struct Bars {
    uint64_t q_full, q_empty, k_full[3], k_empty[3], v_full[2], v_empty[2];
    uint64_t s_full[2], s_free[2], p_full[2], o_done[2], o_free[2];
    uint32_t tmem_base;
};

// Persistent kernel: grid = min(#items, #SMs); CTA c processes work items
// c, c + gridDim.x, ...  An item is two 128-row query tiles of one (problem,
// head); all pipeline stages / barrier phases run on CTA-global counters so
// the producer prefetches the next item's Q and K/V while the current one
// finishes.
template <int N128, int N32>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap q128, const __grid_constant__ CUtensorMap q32,
                   const __grid_constant__ CUtensorMap k128, const __grid_constant__ CUtensorMap k32,
                   const __grid_constant__ CUtensorMap v128, const __grid_constant__ CUtensorMap v32,
                   const __grid_constant__ CUtensorMap omap, const Params p) {
    using G = Geometry<N128, N32>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + G::kBar);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // item -> (head, pair, a, b), head fastest: concurrently running CTAs read all heads of
    // the same q/k/v rows (whole 6.9 KB qkv rows per DRAM page visit) and share K/V in L2
    struct Item {
        int pair, h, a_idx, b_idx0;
    };
    auto decode = [&](int item) {
        Item it;
        it.h = item % p.heads;
        const int rest = item / p.heads;
        it.pair = rest % p.n_pairs;
        const int az = rest / p.n_pairs;
        if (p.packed) {
            it.a_idx = az;
            it.b_idx0 = 0;
        } else {
            it.a_idx = az / p.n_b;
            it.b_idx0 = az - it.a_idx * p.n_b;
        }
        return it;
    };
    // per-tile coordinates (t = 0, 1) as scalar expressions (no runtime-indexed arrays)
    auto i_base = [&](const Item& it, int t) { return p.packed ? 0 : (2 * it.pair + t) * kRows; };
    auto b_base = [&](const Item& it, int t) { return p.packed ? (2 * it.pair + t) * p.packed : it.b_idx0; };
    const int box_rows = p.packed ? p.packed * p.n_k : kRows;  // rows a TMA box fills
    const uint32_t box_bytes = (uint32_t)box_rows * (uint32_t)(N128 * 128 + N32 * 32);
    const int n_iter = p.packed ? 1 : p.n_kv;                  // S/P/O iterations per item and tile
    const int kv_per_item = p.packed ? 2 : p.n_kv;             // K (and V) tiles loaded per item
    const int my_items = (p.n_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

    // ---------------------------------------------------------------- setup
    if (warp == kTmaWarp && lane == 0) {
        prefetch_map(&q128); prefetch_map(&k128); prefetch_map(&v32); prefetch_map(&omap);
        if (N32) { prefetch_map(&q32); prefetch_map(&k32); }
        mbar_init(&bars->q_full, 1);
        mbar_init(&bars->q_empty, 2);  // both tiles' MMA warps are done with Q
        for (int s = 0; s < 3; ++s) {
            mbar_init(&bars->k_full[s], 1);
            mbar_init(&bars->k_empty[s], 2);  // released by both tiles' MMA warps
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars->v_full[s], 1);
            mbar_init(&bars->v_empty[s], 2);  // released by both tiles' MMA warps
            mbar_init(&bars->s_full[s], 1);
            mbar_init(&bars->s_free[s], kGroupThreads);
            mbar_init(&bars->p_full[s], kGroupThreads);
            mbar_init(&bars->o_done[s], 1);
            mbar_init(&bars->o_free[s], kGroupThreads);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&bars->tmem_base)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (box_rows < kRows) {
        // packed tiles leave rows [box_rows, 128) of Q/K/V untouched by TMA:
        // zero them once so masked lanes can never inject NaN/Inf into P.V
        uint4 zero = make_uint4(0, 0, 0, 0);
        for (int off = threadIdx.x * 16; off < 7 * G::kTileBytes; off += kThreads * 16)
            *reinterpret_cast<uint4*>(smem + off) = zero;
        fence_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == kTmaWarp) {
        // ===================================================== TMA producer
        if (lane == 0) {
            // K ring (3 stages) runs up to two tiles ahead of the V ring (2 stages): S(j+1) is issued before PV(j)
            auto load_k = [&](const Item& it, int g, int j) {
                const int ks = g % 3;
                if (g >= 3) mbar_wait(&bars->k_empty[ks], ((g / 3) - 1) & 1);
                const int kv_i = p.packed ? 0 : j * kKv, kv_b = b_base(it, p.packed ? j : 0);
                uint8_t* kd = smem + G::kK0 + ks * G::kTileBytes;
                mbar_expect_tx(&bars->k_full[ks], box_bytes);
                for (int blk = 0; blk < N128; ++blk)
                    tma_load_5d(kd + blk * 16384, &k128, &bars->k_full[ks], 64 * blk, it.h, kv_i, kv_b, it.a_idx);
                for (int blk = 0; blk < N32; ++blk)
                    tma_load_5d(kd + N128 * 16384 + blk * 4096, &k32, &bars->k_full[ks], 64 * N128 + 16 * blk, it.h,
                                kv_i, kv_b, it.a_idx);
            };
            // V is staged as 16-column SW32 atoms ([atom][row][32 B]) so one
            // MN-major descriptor spans the whole padded head dim (N = kDhPad)
            auto load_v = [&](const Item& it, int g, int j) {
                const int vs = g & 1;
                if (g >= 2) mbar_wait(&bars->v_empty[vs], ((g >> 1) - 1) & 1);
                const int kv_i = p.packed ? 0 : j * kKv, kv_b = b_base(it, p.packed ? j : 0);
                uint8_t* vd = smem + G::kV0 + vs * G::kTileBytes;
                mbar_expect_tx(&bars->v_full[vs], box_bytes);
                for (int blk = 0; blk < G::kDhPad / 16; ++blk)
                    tma_load_5d(vd + blk * 4096, &v32, &bars->v_full[vs], 16 * blk, it.h, kv_i, kv_b, it.a_idx);
            };
            int gkv = 0;  // K/V tiles loaded so far by this CTA
            for (int c = 0; c < my_items; ++c) {
                const Item it = decode((int)blockIdx.x + c * (int)gridDim.x);
                if (c > 0) mbar_wait(&bars->q_empty, (c - 1) & 1);
                mbar_expect_tx(&bars->q_full, 2 * box_bytes);
                for (int t = 0; t < 2; ++t) {
                    uint8_t* dst = smem + G::kQ0 + t * G::kTileBytes;
                    for (int blk = 0; blk < N128; ++blk)
                        tma_load_5d(dst + blk * 16384, &q128, &bars->q_full, 64 * blk, it.h, i_base(it, t),
                                    b_base(it, t), it.a_idx);
                    for (int blk = 0; blk < N32; ++blk)
                        tma_load_5d(dst + N128 * 16384 + blk * 4096, &q32, &bars->q_full, 64 * N128 + 16 * blk, it.h,
                                    i_base(it, t), b_base(it, t), it.a_idx);
                }
                // packed: KV tile j (j < 2) holds the keys of query tile j
                load_k(it, gkv, 0);
                if (kv_per_item > 1) load_k(it, gkv + 1, 1);
                load_v(it, gkv, 0);
                for (int j = 0; j < kv_per_item; ++j) {
                    if (j + 2 < kv_per_item) load_k(it, gkv + j + 2, j + 2);
                    if (j + 1 < kv_per_item) load_v(it, gkv + j + 1, j + 1);
                }
                gkv += kv_per_item;
            }
        }
    } else if (warp == kMmaWarp || warp == kMmaWarp + 1) {
        // ============================ MMA issuer of query tile t (warp-wide, elected lane issues)
        const int t = warp - kMmaWarp;
        constexpr uint32_t idS128 = idesc_bf16(128, 128, 0);
        constexpr uint32_t idO = idesc_bf16(128, G::kDhPad, 1);
        const uint32_t q_addr = smem_u32(smem + G::kQ0 + t * G::kTileBytes);
        const uint32_t k_addr = smem_u32(smem + G::kK0);
        const uint32_t v_addr = smem_u32(smem + G::kV0);
        const uint32_t p_addr = smem_u32(smem + G::kP0 + t * kPBytes);
        const uint32_t d_s = tmem + 128 * t, d_o = tmem + 256 + 128 * t;
        // descriptors: constant layout bits | (address >> 4); moving the start
        // address by `off` bytes adds off >> 4 to the low word (no carry: < 256 KB)
        const uint64_t dq128 = smem_desc(q_addr, 16, 1024, kLayoutSW128);
        const uint64_t dk128 = smem_desc(k_addr, 16, 1024, kLayoutSW128);
        const uint64_t dq32 = smem_desc(q_addr + N128 * 16384, 16, 256, kLayoutSW32);
        const uint64_t dk32 = smem_desc(k_addr + N128 * 16384, 16, 256, kLayoutSW32);
        const uint64_t dp = smem_desc(p_addr, 16, 1024, kLayoutSW128);
        // V: MN-major SW32, 16-column atoms 4096 B apart (LBO), 8-row groups 256 B apart (SBO)
        const uint64_t dv = smem_desc(v_addr, 4096, 256, kLayoutSW32);
        // S_t = Q_t K^T over the dh K-blocks (K-major operands)
        // ncols: key columns of this S tile rounded up to 16 (a partial last tile runs N < 128)
        auto issue_s = [&](int st, int ncols) {
            const uint32_t ko = (st * G::kTileBytes) >> 4;
            const uint32_t idS = (idS128 & ~(0x3Fu << 17)) | ((uint32_t)(ncols >> 3) << 17);
            uint32_t acc = 0;
#pragma unroll
            for (int blk = 0; blk < N128; ++blk)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t o = (blk * 16384 + 32 * k) >> 4;
                    tc_mma(d_s, dq128 + o, dk128 + ko + o, idS, acc);
                    acc = 1;
                }
#pragma unroll
            for (int blk = 0; blk < N32; ++blk) {
                const uint32_t o = (blk * 4096) >> 4;
                tc_mma(d_s, dq32 + o, dk32 + ko + o, idS, acc);
                acc = 1;
            }
        };
        // O_t += P_t V: ncols / 16 K-steps of 16 keys, each one N = kDhPad MMA
        auto issue_pv = [&](int st, uint32_t accumulate, int ncols) {
            const uint32_t vo = (st * G::kTileBytes) >> 4;
#pragma unroll
            for (int k = 0; k < kKv / 16; ++k)
                if (16 * k < ncols)
                    tc_mma(d_o, dp + (((k >> 2) * 16384 + 32 * (k & 3)) >> 4), dv + vo + ((512 * k) >> 4), idO,
                           (accumulate || k > 0) ? 1u : 0u);
        };
        auto cols_of = [&](int j) {
            if (p.packed) return kKv;
            const int n = min(kKv, p.n_k - j * kKv);
            return (n + 15) & ~15;
        };
        // S for global iteration gi from K ring slot g; the softmax must have released S(gi - 1)
        auto do_s = [&](int gi, int g, int ncols) {
            mbar_wait(&bars->k_full[g % 3], (g / 3) & 1);
            if (gi > 0) mbar_wait(&bars->s_free[t], (gi - 1) & 1);
            tc_fence_after();
            issue_s(g % 3, ncols);
            tc_commit(&bars->s_full[t]);
            tc_commit(&bars->k_empty[g % 3]);
            if (p.packed) tc_commit(&bars->k_empty[g % 3]);  // sole consumer of this K tile
        };
        int gi = 0, gkv = 0;
        for (int c = 0; c < my_items; ++c) {
            mbar_wait(&bars->q_full, c & 1);
            const int g0 = gkv + (p.packed ? t : 0);
            do_s(gi, g0, cols_of(0));
            if (n_iter == 1) tc_commit(&bars->q_empty);
            for (int j = 0; j < n_iter; ++j) {
                // next scores first: S_t(j+1) only needs the softmax to have read S_t(j),
                // so the tensor pipe computes it while P_t(j) is still being written
                if (j + 1 < n_iter) {
                    do_s(gi + j + 1, gkv + j + 1, cols_of(j + 1));
                    if (j + 2 == n_iter) tc_commit(&bars->q_empty);  // last S of this item issued
                }
                const int gv = g0 + j;
                mbar_wait(&bars->v_full[gv & 1], (gv >> 1) & 1);
                mbar_wait(&bars->p_full[t], (gi + j) & 1);
                if (j == 0 && c > 0) mbar_wait(&bars->o_free[t], (c - 1) & 1);  // epilogue read O
                tc_fence_after();
                issue_pv(gv & 1, j > 0, cols_of(j));
                tc_commit(&bars->o_done[t]);
                tc_commit(&bars->v_empty[gv & 1]);
                if (p.packed) tc_commit(&bars->v_empty[gv & 1]);
            }
            gi += n_iter;
            gkv += kv_per_item;
        }
    } else {
        // ================================================= softmax groups
        const int t = warp >> 3;            // query tile of this group
        const int hc = (warp >> 2) & 1;     // score-column half: [64 hc, 64 hc + 64)
        const int wl = warp & 3;            // TMEM lane quarter
        const int row = wl * 32 + lane;     // tile row owned by this thread
        const uint32_t lane_off = (uint32_t)(wl * 32) << 16;
        const uint32_t s_tmem = tmem + lane_off + 128 * t + 64 * hc;
        const uint32_t o_tmem = tmem + lane_off + 256 + 128 * t;
        uint8_t* p_blk = smem + G::kP0 + t * kPBytes + hc * 16384;
        float* xch = reinterpret_cast<float*>(smem + G::kX0) + t * (2 * 3 * kRows);  // [half][slot][row]
        const uint32_t bar_id = 1 + t;
        // O columns this half rescales / stores: 16-wide chunks [c_lo, c_hi)
        constexpr int kOChunks = G::kDhPad / 16;
        const int c_lo = hc ? (kOChunks + 1) / 2 : 0;
        const int c_hi = hc ? kOChunks : (kOChunks + 1) / 2;
        const int T = p.n_k;
        const int group = p.packed ? row / T : 0;
        const uint32_t rsw = (uint32_t)(row & 7);
        // shared-space address of this row in the P block
        const uint32_t p_row = smem_u32(p_blk) + (uint32_t)row * 128u;
        const int total_iters = my_items * n_iter;
        int gi = 0;
        const bool o_issuer = (hc == 0 && wl == 0 && lane == 0);  // issues this tile's O store
        uint8_t* o_stage = smem + G::kP0 + t * kPBytes;           // dense O rows, staged in the P block

        for (int c = 0; c < my_items; ++c) {
            const Item it = decode((int)blockIdx.x + c * (int)gridDim.x);
            float m_run = -INFINITY, l_run = 0.f;
            for (int j = 0; j < n_iter; ++j, ++gi) {
                PAB_TRACE(wl == 0 && lane == 0 && hc == 0, gi < 60 ? gi : 60, t, 0);
                mbar_wait(&bars->s_full[t], gi & 1);
                tc_fence_after();
                PAB_TRACE(wl == 0 && lane == 0 && hc == 0, gi < 60 ? gi : 60, t, 1);
                // live score columns [lo, hi) of this row in this S tile
                int lo = 0, hi = kKv;
                if (p.packed) {
                    lo = group * T;
                    hi = lo + T;
                } else if (p.n_k - j * kKv < kKv) {
                    hi = p.n_k - j * kKv;
                }
                // live columns of this thread's 64-column half, relative to the half
                const int lo_c = max(lo - 64 * hc, 0), hi_c = min(hi - 64 * hc, 64);
                const bool full = (lo_c == 0) && (hi_c == 64);
                // ---- pass 1: this half's row max of the raw scores (scale > 0 commutes with max)
                // false: this half lies past a partial last tile, whose P.V does not read it
                // (packed tiles always run the masked path: their P.V reads all 128 keys)
                const bool live = p.packed || hi_c > lo_c;
                float mx = full   ? row_max_half<true>(s_tmem, 0, 64)
                           : live ? row_max_half<false>(s_tmem, lo_c, hi_c)
                                  : -INFINITY;
                // exchange with the other column half of the same rows (double-buffered slot)
                const int slot = gi & 1;
                PAB_TRACE(wl == 0 && lane == 0 && hc == 0, gi < 60 ? gi : 60, t, 2);
                xch[(hc * 3 + slot) * kRows + row] = mx;
                // the previous item's O tile store has finished reading its staging (the P block
                // this group is about to overwrite) before the group passes this barrier
                if (o_issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(kGroupThreads) : "memory");
                mx = fmaxf(mx, xch[((1 - hc) * 3 + slot) * kRows + row]);
                const float m_tile = mx * p.scale_log2;
                PAB_TRACE(wl == 0 && lane == 0 && hc == 0, gi < 60 ? gi : 60, t, 3);
                // previous P.V must be finished before P smem is overwritten or O rescaled
                // (j == 0: the previous item's epilogue already waited for its last P.V)
                if (j > 0) {
                    mbar_wait(&bars->o_done[t], (gi - 1) & 1);
                    tc_fence_after();
                }
                // both halves see identical (m_tile, m_run) per row, so they take the same branch
                const bool need = m_tile > m_run + 8.0f;
                if (__any_sync(0xffffffffu, need)) {
                    const float m_new = fmaxf(m_run, m_tile);
                    if (j > 0) {
                        const float alpha = fast_exp2(m_run - m_new);
                        l_run *= alpha;
                        for (int cc = c_lo; cc < c_hi; ++cc) {
                            float o[16];
                            PAB_TMEM_LD16(o_tmem + 16 * cc, o);
                            tmem_wait_ld();
#pragma unroll
                            for (int e = 0; e < 16; ++e) o[e] *= alpha;
                            PAB_TMEM_ST16(o_tmem + 16 * cc, o);
                        }
                        tmem_wait_st();
                    }
                    m_run = m_new;
                }
                const float neg_m = (m_run == -INFINITY) ? 0.f : -m_run;
                PAB_TRACE(wl == 0 && lane == 0 && hc == 0, gi < 60 ? gi : 60, t, 4);
                // ---- pass 2: P = exp2(s * scale_log2 - m) -> bf16 into this half's 128B-swizzled P block.
                // All 64 scores are pulled from TMEM first so S can be released (s_free) and the
                // tensor pipe can start S(j+1) while this warp is still exponentiating.
                // (a half past a partial last tile loads stale columns it never uses)
                float v[64];
                PAB_TMEM_LD32(s_tmem, v);
                PAB_TMEM_LD32(s_tmem + 32, (v + 32));
                tmem_wait_ld();
                PAB_TRACE(wl == 0 && lane == 0 && hc == 0, gi < 60 ? gi : 60, t, 6);
                tc_fence_before();
                mbar_arrive(&bars->s_free[t]);
#ifndef PAB_NO_MUFU_TOKEN
                // MUFU token: the two query tiles' exp2 phases strictly alternate
                // (tile 0 of iteration g, tile 1 of g, tile 0 of g+1, ...), so one
                // group exponentiates while the other reduces / exchanges / waits.
                if (t == 1 || gi > 0) asm volatile("bar.sync %0, %1;" ::"r"(3 + t), "r"(2 * kGroupThreads) : "memory");
#endif
                const float psum = full   ? exp_pack_half<true>(v, p.scale_log2, neg_m, p_row, rsw, 0, 64)
                                   : live ? exp_pack_half<false>(v, p.scale_log2, neg_m, p_row, rsw, lo_c, hi_c)
                                          : 0.f;  // the P.V of this tile does not read this half
#ifndef PAB_NO_MUFU_TOKEN
                if (t == 0 || gi + 1 < total_iters)
                    asm volatile("bar.arrive %0, %1;" ::"r"(4 - t), "r"(2 * kGroupThreads) : "memory");
#endif
                PAB_TRACE(wl == 0 && lane == 0 && hc == 0, gi < 60 ? gi : 60, t, 7);
                l_run += psum;
                fence_async_smem();
                PAB_TRACE(wl == 0 && lane == 0 && hc == 0, gi < 60 ? gi : 60, t, 5);
                mbar_arrive(&bars->p_full[t]);
            }

            // ------------------------------------------------------ epilogue of this item
            PAB_TRACE(wl == 0 && lane == 0 && hc == 0, (gi - 1) < 60 ? (gi - 1) : 60, t, 8);
            xch[(hc * 3 + 2) * kRows + row] = l_run;
            asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(kGroupThreads) : "memory");
            const float l_tot = l_run + xch[((1 - hc) * 3 + 2) * kRows + row];
            mbar_wait(&bars->o_done[t], (gi - 1) & 1);
            tc_fence_after();
            // O rows leave through the tile's (now idle) P block and ONE asynchronous TMA tensor
            // store per tile: plain row stores from every CTA at the same moment form a GPU-wide
            // write burst the softmax stalls on (the same fix as attn_fa.cu's epilogue).
            const float inv = (l_tot > 0.f) ? 1.0f / l_tot : 0.f;
            uint8_t* stg = o_stage + row * (2 * p.dh);  // dense rows: the TMA box layout
            for (int cc = c_lo; cc < c_hi; ++cc) {
                float o[16];
                PAB_TMEM_LD16(o_tmem + 16 * cc, o);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; e += 8) {
                    if (16 * cc + e < p.dh) {
                        uint32_t w[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) w[q] = pack_bf16(o[e + 2 * q] * inv, o[e + 2 * q + 1] * inv);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(stg + (16 * cc + e) * 2)),
                                     "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                                     : "memory");
                    }
                }
            }
            fence_async_smem();
            asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(kGroupThreads) : "memory");
            if (o_issuer) {
                // packed: box (dh, 1, T, packed, 1) at (0, h, 0, first sequence, a); rows past the
                // problem count / n_q are clipped by the tensor map
                const int ci = p.packed ? 0 : i_base(it, t), cb = b_base(it, t);
                asm volatile(
                    "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n\t"
                    "cp.async.bulk.commit_group;" ::"l"(reinterpret_cast<uint64_t>(&omap)),
                    "r"(smem_u32(o_stage)), "r"(0), "r"(it.h), "r"(ci), "r"(cb), "r"(it.a_idx)
                    : "memory");
            }
            // O may now be overwritten by the next item's first P.V
            PAB_TRACE(wl == 0 && lane == 0 && hc == 0, (gi - 1) < 60 ? (gi - 1) : 60, t, 9);
            tc_fence_before();
            mbar_arrive(&bars->o_free[t]);
        }
        if (o_issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // O stores done before exit
    }
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

// 5-D view (dh, heads, i, b, a) of one operand; box = (inner, 1, rows_i, rows_b, 1)
bool make_map(CUtensorMap* map, const void* base, int dh, int heads, int n_i, int n_b, int n_a, int64_t s_i,
              int64_t s_b, int64_t s_a, int box_inner, int box_i, int box_b, CUtensorMapSwizzle swz) {
    auto encode = get_encode();
    if (!encode) return false;
    cuuint64_t dims[5] = {(cuuint64_t)dh, (cuuint64_t)heads, (cuuint64_t)n_i, (cuuint64_t)n_b, (cuuint64_t)n_a};
    auto bytes = [](int64_t s) { return (cuuint64_t)(s > 0 ? s * 2 : 16); };
    cuuint64_t strides[4] = {(cuuint64_t)dh * 2, bytes(s_i), bytes(s_b), bytes(s_a)};
    cuuint32_t box[5] = {(cuuint32_t)box_inner, 1, (cuuint32_t)box_i, (cuuint32_t)box_b, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

long long* g_trace = nullptr;  // set by pab_attn_debug_trace (debug builds of the timeline only)

template <int N128, int N32>
int launch(const pab_attn_args* a, int packed, cudaStream_t st) {
    using G = Geometry<N128, N32>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(attn_tc_kernel<N128, N32>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::kSmem) !=
            cudaSuccess)
            return launch_status("attn_tc smem attribute");
        attr_set = true;
    }
    const int box_i = packed ? a->n_k : kRows;
    const int box_b = packed ? packed : 1;
    CUtensorMap maps[7];
    struct Op { const void* ptr; int64_t sa, sb, si; int n_i; } ops[3] = {
        {a->q, a->q_sa, a->q_sb, a->q_si, a->n_q}, {a->k, a->k_sa, a->k_sb, a->k_si, a->n_k},
        {a->v, a->v_sa, a->v_sb, a->v_si, a->n_k}};
    for (int o = 0; o < 3; ++o) {
        const Op& op = ops[o];
        if (!make_map(&maps[2 * o], op.ptr, a->dh, a->heads, op.n_i, a->n_b, a->n_a, op.si, op.sb, op.sa,
                      N128 ? 64 : 16, box_i, box_b, N128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B))
            return PAB_ERR_CUDA;
        if (!make_map(&maps[2 * o + 1], op.ptr, a->dh, a->heads, op.n_i, a->n_b, a->n_a, op.si, op.sb, op.sa, 16,
                      box_i, box_b, CU_TENSOR_MAP_SWIZZLE_32B))
            return PAB_ERR_CUDA;
    }
    // O: one TMA tensor store per 128-row tile (box = dh x the Q box rows), no swizzle
    if (!make_map(&maps[6], a->o, a->dh, a->heads, a->n_q, a->n_b, a->n_a, a->o_si, a->o_sb, a->o_sa, a->dh, box_i,
                  box_b, CU_TENSOR_MAP_SWIZZLE_NONE))
        return PAB_ERR_CUDA;
    Params p;
    p.n_q = a->n_q; p.n_k = a->n_k; p.n_b = a->n_b; p.heads = a->heads; p.dh = a->dh;
    p.packed = packed;
    p.scale_log2 = a->scale * 1.4426950408889634f;
    p.o = reinterpret_cast<__nv_bfloat16*>(a->o);
    p.o_sa = a->o_sa; p.o_sb = a->o_sb; p.o_si = a->o_si;
    p.trace = g_trace;
    int64_t problems;
    if (packed) {
        p.row_tiles = (a->n_b + packed - 1) / packed;
        p.n_kv = 2;  // one KV tile per query tile
        problems = a->n_a;
    } else {
        p.row_tiles = (a->n_q + kRows - 1) / kRows;
        p.n_kv = (a->n_k + kKv - 1) / kKv;
        problems = (int64_t)a->n_a * a->n_b;
    }
    p.n_pairs = (p.row_tiles + 1) / 2;
    const int64_t items = (int64_t)p.n_pairs * a->heads * problems;
    if (items > 0x7fffffff) return PAB_ERR_UNSUPPORTED;
    p.n_items = (int)items;
    static int num_sms = 0;
    if (num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (num_sms <= 0) num_sms = 148;
    }
    dim3 grid((unsigned)(p.n_items < num_sms ? p.n_items : num_sms));
    attn_tc_kernel<N128, N32><<<grid, kThreads, G::kSmem, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4],
                                                                 maps[5], maps[6], p);
    return launch_status("attn_tc");
}

int packing_for(const pab_attn_args* a) {
    if (a->n_b > 1 && a->n_q == a->n_k && a->n_k <= 64) return kRows / a->n_k;
    return 0;
}

}  // namespace tc

extern "C" int pab_attn_debug_trace(long long* device_buffer) {
    pab::tc::g_trace = device_buffer;
    return PAB_OK;
}

bool attn_tc_supported(const pab_attn_args* a) {
    if (a->dh % 8 != 0 || a->dh > 80 || a->n_k < 1) return false;  // smem: 7 operand tiles + 2 P tiles
    const int64_t strides[] = {a->q_sa, a->q_sb, a->q_si, a->k_sa, a->k_sb, a->k_si,
                               a->v_sa, a->v_sb, a->v_si, a->o_sa, a->o_sb, a->o_si};  // all TMA-addressed
    for (int64_t s : strides)
        if (s % 8 != 0 || s < 0) return false;
    const uintptr_t ptrs[] = {(uintptr_t)a->q, (uintptr_t)a->k, (uintptr_t)a->v, (uintptr_t)a->o};
    for (uintptr_t p : ptrs)
        if (p % 16 != 0) return false;
    if ((int64_t)a->n_a * a->n_b > 65535 || a->heads > 65535) return false;
    if (a->n_a > 0x7fffffff || a->n_q > (1 << 30)) return false;
    return tc::get_encode() != nullptr;
}

int attn_tc_packing(const pab_attn_args* a) { return tc::packing_for(a); }

int attn_tc_launch(const pab_attn_args* a, cudaStream_t st) {
    const int packed = tc::packing_for(a);
    const int n128 = a->dh / 64;
    const int n32 = (a->dh - 64 * n128 + 15) / 16;
#define PAB_TC(A, B) \
    if (n128 == A && n32 == B) return tc::launch<A, B>(a, packed, st)
    PAB_TC(0, 1); PAB_TC(0, 2); PAB_TC(0, 3);
    PAB_TC(1, 0); PAB_TC(1, 1);
#undef PAB_TC
    return PAB_ERR_UNSUPPORTED;
}

}  // namespace pab

// Temporal attention (K2) for sm_100a: short sequences (T frames of one token) packed
// 128 rows to a tile, built to stream at the HBM roofline.
//
// reference op: numerics.scaled_dot_attention (pkg/src/pab_engine/numerics.py:133-151) as
// used by _axis_attention_compute(temporal_axis=True) (pkg/src/pab_engine/model.py:351-357):
// every (batch, token, head) attends over its own T frames.
//
// Work item = one head h of 128 / T consecutive sequences (rows (seq, t), 128 per tile).
// Per item: S = Q K^T (M = N = 128, block-diagonal: row r only needs the T keys of its own
// sequence), P = softmax within the diagonal block, O = P V (M = 128, N = dh padded to 16,
// K = 128 keys with P zero off the diagonal).  What makes it lean (T divides 32):
//   * a softmax warp owns TMEM lanes [32 wl, 32 wl + 32) = 32 / T whole sequences, whose keys
//     are exactly S columns [32 wl, 32 wl + 32): it loads those 32 columns only, masks each
//     row to its own T-wide window (T exps per row, not 128) and writes P straight into TMEM
//     over the S columns it has read -- its 16 live words plus zeros for the other 48;
//   * row sums are kept in registers (fp32 sum of the exps), so O needs no extra column;
//   * two TMEM slots (S/P 128 columns + O up to 80 columns each) and two softmax/epilogue
//     groups of 4 warps: group g handles items c with c % 2 == g, so one group's epilogue
//     overlaps the other group's softmax and the tensor pipe;
//   * two MMA issuer warps: warp S issues S(c) as soon as item c's operands have landed and
//     PV(c - 2) (which read the same slot's P) is complete; warp PV issues PV(c) once P(c) is
//     stored and the epilogue of item c - 2 has pulled O out of the slot -- neither waits
//     behind the other's dependencies;
//   * Q/K/V of an item arrive by TMA (one 5-D box per 64/16-column block, the box spanning
//     T rows x 128/T sequences of any row strides, so the token-major serial layout and
//     the all-to-all layout of sequence parallelism both work) into a 3-stage ring;
//   * O leaves per warp: TMEM -> normalised bf16 rows in smem -> one TMA tensor store of the
//     warp's 32 / T sequences (box dh x T x 32 / T), clipped past the last sequence;
//   * each CTA walks one contiguous range of items, heads fastest (see item_of).
// Per item the kernel moves 3 x 128 x dh x 2 bytes in and 128 x dh x 2 out; the tensor and
// MUFU work per item is a few hundred cycles, far below the ~3K-cycle HBM budget of an SM.
#include "tc_ptx.cuh"

namespace pab {
namespace tm {

using namespace pab::tc;

constexpr int kRows = 128;      // rows per tile == TMEM lanes == keys per tile
constexpr int kGroupWarps = 4;  // softmax + epilogue warps per group (one per TMEM lane quarter)
constexpr int kSWarp = 2 * kGroupWarps;  // S issuer (also allocates TMEM)
constexpr int kPvWarp = kSWarp + 1;      // PV issuer
constexpr int kTmaWarp = kSWarp + 2;     // TMA producer
constexpr int kThreads = 32 * (kTmaWarp + 1);
constexpr int kStages = 3;
#ifndef PAB_TM_ORDER
#define PAB_TM_ORDER 1  // 1: one contiguous item range per CTA; 0: items strided over CTAs (head fastest)
#endif
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kOCol0 = 256;  // O of slot g at kOCol0 + 128 g; S/P of slot g at 128 g

template <int N128, int N32>
struct Geometry {
    static constexpr int kDhPad = 64 * N128 + 16 * N32;         // head dim padded to 16 (K of S, N of O)
    static constexpr int kOpBytes = kRows * kDhPad * 2;          // one 128-row operand tile
    static constexpr int kStageBytes = 3 * kOpBytes;             // Q, K, V
    static constexpr int kStageRowBytes = 2 * kDhPad;            // max bytes of one dense bf16 O row
    static constexpr int kStg0 = kStages * kStageBytes;          // O staging: [group][128 rows]
    static constexpr int kBar = kStg0 + 2 * kRows * kStageRowBytes;
    static constexpr int kSmem = kBar + 256 + 1024;  // + barriers + alignment slack
    static_assert(kSmem <= 232448, "temporal attention tiles exceed the 227 KB of shared memory");
    static_assert(kOpBytes % 1024 == 0, "operand tiles must keep 1 KB swizzle alignment");
};

struct Bars {
    uint64_t full[kStages], empty[kStages];
    uint64_t s_full[2], p_full[2], o_done[2], o_free[2];
    uint32_t tmem_base;
};

struct Params {
    int T, spt;          // frames per sequence, sequences per tile (128 / T)
    int heads, dh;
    int tiles_per_a;     // tiles along the sequence axis of one problem a
    int n_items;         // tiles_per_a * n_a * heads
    float scale_log2;    // scale * log2(e)
};

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

#define PAB_TM_ST16(taddr, w)                                                                                \
    asm volatile(                                                                                            \
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
        "%16};" ::"r"(taddr),                                                                                \
        "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]),   \
        "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])                    \
        : "memory")

template <int N128, int N32>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tm_kernel(const __grid_constant__ CUtensorMap q128, const __grid_constant__ CUtensorMap q32,
                   const __grid_constant__ CUtensorMap k128, const __grid_constant__ CUtensorMap k32,
                   const __grid_constant__ CUtensorMap v32, const __grid_constant__ CUtensorMap omap,
                   const Params p) {
    using G = Geometry<N128, N32>;
    constexpr int kDhPad = G::kDhPad;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + G::kBar);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if PAB_TM_ORDER == 0
    const int my_items = (p.n_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
#else
    const int i0 = (int)(((long long)p.n_items * blockIdx.x) / gridDim.x);
    const int my_items = (int)(((long long)p.n_items * (blockIdx.x + 1)) / gridDim.x) - i0;
#endif
    // item -> (head fastest, tile, problem), each CTA walking ONE contiguous range of items:
    // its consecutive items are the 16 heads of the same 128 rows, so the 32-byte sectors two
    // neighbouring heads' 144-byte slices share are re-read from L2 moments later by the same
    // SM.  Striding items over the CTAs instead (item = CTA + c * grid, the spatial kernel's
    // order) read 527 MB from DRAM for 345 MB of operands and ran at 61% of HBM; the
    // contiguous ranges read 356 MB and run at 84% (C3, 83.6 vs 116 us).
    auto item_of = [&](int c, int& h, int& seq0, int& a) {
#if PAB_TM_ORDER == 0
        const int item = (int)blockIdx.x + c * (int)gridDim.x;
#else
        const int item = i0 + c;
#endif
        h = item % p.heads;
        const int rest = item / p.heads;
        seq0 = (rest % p.tiles_per_a) * p.spt;
        a = rest / p.tiles_per_a;
    };

    if (warp == kTmaWarp && lane == 0) {
        prefetch_map(&q128);
        prefetch_map(&k128);
        prefetch_map(&v32);
        prefetch_map(&omap);
        if (N32) {
            prefetch_map(&q32);
            prefetch_map(&k32);
        }
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int g = 0; g < 2; ++g) {
            mbar_init(&bars->s_full[g], 1);
            mbar_init(&bars->p_full[g], kGroupWarps);
            mbar_init(&bars->o_done[g], 1);
            mbar_init(&bars->o_free[g], kGroupWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kSWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&bars->tmem_base)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == kTmaWarp) {
        // ===================================================== TMA producer (lane 0)
        if (lane == 0) {
            for (int c = 0; c < my_items; ++c) {
                int h, seq0, a;
                item_of(c, h, seq0, a);
                const int st = c % kStages;
                if (c >= kStages) mbar_wait(&bars->empty[st], ((c / kStages) - 1) & 1);
                uint8_t* base = smem + st * G::kStageBytes;
                uint64_t* bar = &bars->full[st];
                mbar_expect_tx(bar, G::kStageBytes);
                // Q and K: one 64-column SW128 block per 64 head columns, then 16-column SW32 blocks
                for (int blk = 0; blk < N128; ++blk) {
                    tma_load_5d(base + blk * kRows * 128, &q128, bar, 64 * blk, h, 0, seq0, a);
                    tma_load_5d(base + G::kOpBytes + blk * kRows * 128, &k128, bar, 64 * blk, h, 0, seq0, a);
                }
                for (int blk = 0; blk < N32; ++blk) {
                    const int off = N128 * kRows * 128 + blk * kRows * 32;
                    tma_load_5d(base + off, &q32, bar, 64 * N128 + 16 * blk, h, 0, seq0, a);
                    tma_load_5d(base + G::kOpBytes + off, &k32, bar, 64 * N128 + 16 * blk, h, 0, seq0, a);
                }
                // V as 16-column SW32 atoms ([atom][row][32 B]): one MN-major descriptor spans dh
                for (int blk = 0; blk < kDhPad / 16; ++blk)
                    tma_load_5d(base + 2 * G::kOpBytes + blk * kRows * 32, &v32, bar, 16 * blk, h, 0, seq0, a);
            }
        }
    } else if (warp == kSWarp) {
        // ===================================================== S = Q K^T issuer
        constexpr uint32_t idS = idesc_bf16(kRows, kRows, 0);
        for (int c = 0; c < my_items; ++c) {
            const int st = c % kStages, g = c & 1;
            mbar_wait(&bars->full[st], (c / kStages) & 1);
            // the slot's previous occupant (item c - 2): its P.V must be complete before S(c)
            // overwrites the P it reads (the softmax group read that S long before)
            if (c >= 2) mbar_wait(&bars->o_done[g], ((c >> 1) - 1) & 1);
            tc_fence_after();
            const uint32_t qa = smem_u32(smem + st * G::kStageBytes);
            const uint32_t ka = qa + G::kOpBytes;
            const uint64_t dq128 = smem_desc(qa, 16, 1024, kLayoutSW128), dk128 = smem_desc(ka, 16, 1024, kLayoutSW128);
            const uint64_t dq32 = smem_desc(qa + N128 * kRows * 128, 16, 256, kLayoutSW32);
            const uint64_t dk32 = smem_desc(ka + N128 * kRows * 128, 16, 256, kLayoutSW32);
            const uint32_t d = tmem + 128 * g;
            uint32_t acc = 0;
#pragma unroll
            for (int blk = 0; blk < N128; ++blk)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t o = (blk * kRows * 128 + 32 * k) >> 4;
                    tc_mma(d, dq128 + o, dk128 + o, idS, acc);
                    acc = 1;
                }
#pragma unroll
            for (int blk = 0; blk < N32; ++blk) {
                const uint32_t o = (blk * kRows * 32) >> 4;
                tc_mma(d, dq32 + o, dk32 + o, idS, acc);
                acc = 1;
            }
            tc_commit(&bars->s_full[g]);
        }
    } else if (warp == kPvWarp) {
        // ===================================================== O = P V issuer
        constexpr uint32_t idO = idesc_bf16(kRows, kDhPad, 1);
        for (int c = 0; c < my_items; ++c) {
            const int st = c % kStages, g = c & 1;
            mbar_wait(&bars->p_full[g], (c >> 1) & 1);
            if (c >= 2) mbar_wait(&bars->o_free[g], ((c >> 1) - 1) & 1);  // epilogue of c - 2 read O
            tc_fence_after();
            // V: MN-major SW32, 16-column atoms kRows * 32 B apart (LBO), 8-row groups 256 B apart (SBO)
            const uint64_t dv = smem_desc(smem_u32(smem + st * G::kStageBytes + 2 * G::kOpBytes), kRows * 32, 256,
                                          kLayoutSW32);
#pragma unroll
            for (int k = 0; k < kRows / 16; ++k)  // 16 keys per K step: P columns 8k.. (bf16 pairs), V rows 16k..
                mma_ts(tmem + kOCol0 + 128 * g, tmem + 128 * g + 8 * k, dv + ((512 * k) >> 4), idO, k > 0 ? 1u : 0u);
            tc_commit(&bars->o_done[g]);
            tc_commit(&bars->empty[st]);
        }
    } else {
        // ============================================ softmax + epilogue, group g (4 warps)
        const int g = warp / kGroupWarps, wl = warp % kGroupWarps;
        const uint32_t lane_off = (uint32_t)(wl * 32) << 16;
        const uint32_t s_tmem = tmem + lane_off + 128 * g;  // S/P of this slot
        const uint32_t o_tmem = tmem + lane_off + kOCol0 + 128 * g;
        // this row's keys within the warp's 32 columns: [lo, lo + T) (T divides 32)
        const int lo = (lane / p.T) * p.T;
        uint8_t* stg_warp = smem + G::kStg0 + (g * kRows + wl * 32) * (2 * p.dh);
        uint8_t* stg = stg_warp + lane * (2 * p.dh);  // dense rows: the TMA box layout
        const unsigned long long sc2 = f2_pack(p.scale_log2, p.scale_log2);
        for (int c = g; c < my_items; c += 2) {
            const int k = c >> 1;
            int h, seq0, a;
            item_of(c, h, seq0, a);
            mbar_wait(&bars->s_full[g], k & 1);
            tc_fence_after();
            float s[32];
            PAB_TMEM_LD32(s_tmem + 32 * wl, s);
            tmem_wait_ld();
            float mx = -INFINITY;
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) mx = ((unsigned)(cc - lo) < (unsigned)p.T) ? fmaxf(mx, s[cc]) : mx;
            const float nm = -mx * p.scale_log2;
            const unsigned long long nm2 = f2_pack(nm, nm);
            float l = 0.f;
            uint32_t w[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                float2 x = f2_unpack(f2_fma(f2_pack(s[2 * q], s[2 * q + 1]), sc2, nm2));
                x.x = ((unsigned)(2 * q - lo) < (unsigned)p.T) ? fast_exp2(x.x) : 0.f;
                x.y = ((unsigned)(2 * q + 1 - lo) < (unsigned)p.T) ? fast_exp2(x.y) : 0.f;
                l += x.x + x.y;
                w[q] = pack_bf16(x.x, x.y);
            }
            // P over the S columns: this warp's 16 words at [16 wl, 16 wl + 16), zeros elsewhere
            // (P.V runs all 128 keys; every off-diagonal block must be exactly zero)
            uint32_t z[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) z[q] = 0u;
#pragma unroll
            for (int blk = 0; blk < 4; ++blk) {
                if (blk == wl)
                    PAB_TM_ST16(s_tmem + 16 * blk, w);
                else
                    PAB_TM_ST16(s_tmem + 16 * blk, z);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->p_full[g]);

            // ---- epilogue: O rows of this warp -> smem -> one TMA tensor store
            mbar_wait(&bars->o_done[g], k & 1);
            tc_fence_after();
            float o[kDhPad];
#pragma unroll
            for (int cc = 0; cc < kDhPad / 16; ++cc) PAB_TMEM_LD16(o_tmem + 16 * cc, (o + 16 * cc));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->o_free[g]);  // the slot's O may be overwritten
            const float inv = (l > 0.f) ? 1.0f / l : 0.f;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // last store read stg
            __syncwarp();
#pragma unroll
            for (int e = 0; e < kDhPad; e += 8) {
                if (e < p.dh) {
                    uint32_t ow[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) ow[q] = pack_bf16(o[e + 2 * q] * inv, o[e + 2 * q + 1] * inv);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(stg + 2 * e)), "r"(ow[0]),
                                 "r"(ow[1]), "r"(ow[2]), "r"(ow[3])
                                 : "memory");
                }
            }
            fence_async_smem();  // generic-proxy smem writes -> visible to the TMA (async proxy)
            __syncwarp();
            if (lane == 0)
                asm volatile(
                    "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n\t"
                    "cp.async.bulk.commit_group;" ::"l"(reinterpret_cast<uint64_t>(&omap)),
                    "r"(smem_u32(stg_warp)), "r"(0), "r"(h), "r"(0), "r"(seq0 + wl * (32 / p.T)), "r"(a)
                    : "memory");
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // O stores done before exit
    }
    __syncthreads();
    if (warp == kSWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

template <int N128, int N32>
int launch(const pab_attn_args* a, cudaStream_t st) {
    using G = Geometry<N128, N32>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(attn_tm_kernel<N128, N32>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::kSmem) !=
            cudaSuccess)
            return launch_status("attn_tm smem attribute");
        attr_set = true;
    }
    const int T = a->n_k, spt = kRows / T;
    CUtensorMap mq128, mq32, mk128, mk32, mv32, mo;
    const CUtensorMapSwizzle big = N128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B;
    const int inner = N128 ? 64 : 16;
    // 5-D views (dh, heads, t, sequence, a); a box spans T frames x spt sequences
    if (!make_map(&mq128, a->q, a->dh, a->heads, T, a->n_b, a->n_a, a->q_si, a->q_sb, a->q_sa, inner, T, spt, big) ||
        !make_map(&mq32, a->q, a->dh, a->heads, T, a->n_b, a->n_a, a->q_si, a->q_sb, a->q_sa, 16, T, spt,
                  CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_map(&mk128, a->k, a->dh, a->heads, T, a->n_b, a->n_a, a->k_si, a->k_sb, a->k_sa, inner, T, spt, big) ||
        !make_map(&mk32, a->k, a->dh, a->heads, T, a->n_b, a->n_a, a->k_si, a->k_sb, a->k_sa, 16, T, spt,
                  CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_map(&mv32, a->v, a->dh, a->heads, T, a->n_b, a->n_a, a->v_si, a->v_sb, a->v_sa, 16, T, spt,
                  CU_TENSOR_MAP_SWIZZLE_32B) ||
        // O: per-warp store of 32 / T sequences (box = dh x T x 32 / T)
        !make_map(&mo, a->o, a->dh, a->heads, T, a->n_b, a->n_a, a->o_si, a->o_sb, a->o_sa, a->dh, T, 32 / T,
                  CU_TENSOR_MAP_SWIZZLE_NONE))
        return PAB_ERR_CUDA;
    Params p;
    p.T = T;
    p.spt = spt;
    p.heads = a->heads;
    p.dh = a->dh;
    p.tiles_per_a = (a->n_b + spt - 1) / spt;
    const int64_t items = (int64_t)p.tiles_per_a * a->n_a * a->heads;
    if (items > 0x7fffffff) return PAB_ERR_UNSUPPORTED;
    p.n_items = (int)items;
    p.scale_log2 = a->scale * 1.4426950408889634f;
    static int num_sms = 0;
    if (num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (num_sms <= 0) num_sms = 148;
    }
    dim3 grid((unsigned)(p.n_items < num_sms ? p.n_items : num_sms));
    attn_tm_kernel<N128, N32><<<grid, kThreads, G::kSmem, st>>>(mq128, mq32, mk128, mk32, mv32, mo, p);
    return launch_status("attn_tm");
}

}  // namespace tm

// square short sequences (n_q == n_k == T, T divides 32) with dh <= 80, a multiple of 8
bool attn_tm_supported(const pab_attn_args* a) {
    const int T = a->n_k;
    return a->n_q == T && T >= 1 && T <= 32 && (32 % T) == 0 && a->n_b > 1 && a->dh % 8 == 0 && a->dh <= 80;
}

int attn_tm_launch(const pab_attn_args* a, cudaStream_t st) {
    const int n128 = a->dh / 64;
    const int n32 = (a->dh - 64 * n128 + 15) / 16;
#define PAB_TM(A, B) \
    if (n128 == A && n32 == B) return tm::launch<A, B>(a, st)
    PAB_TM(0, 1);
    PAB_TM(0, 2);
    PAB_TM(0, 3);
    PAB_TM(0, 4);
    PAB_TM(1, 0);
    PAB_TM(1, 1);
#undef PAB_TM
    return PAB_ERR_UNSUPPORTED;
}

}  // namespace pab

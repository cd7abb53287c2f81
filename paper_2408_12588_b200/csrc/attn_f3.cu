// Three-tile row-per-thread tcgen05 flash attention for sm_100a (spatial K1 / cross K3).
//
// reference op: numerics.scaled_dot_attention (pkg/src/pab_engine/numerics.py:133-151)
// as used by _axis_attention_compute(temporal_axis=False) and _cross_attention_compute
// (pkg/src/pab_engine/model.py:346-359, 376-385):
//   logits = q k^T * (1/sqrt(dh)); p = softmax(logits) (max-shifted); out = p v
//
// Why a third query tile.  The two-tile kernel (attn_fa.cu) is bound by the exp work of
// ONE softmax warp per SM sub-partition at a time: the two tiles' exp sections alternate,
// and a lone warp keeps the MUFU only ~73% busy.  Here a work item is
// THREE 128-row query tiles of one (problem, head) and each tile runs its own chain
//     S_t(j) = Q_t K_j^T  ->  softmax_t(j) (P_t written over S_t in TMEM)  ->  O_t += P_t V_j
// with per-tile barriers and no exp token, so up to three softmax warps per sub-partition
// are in different phases and the tensor pipe serves whichever tile is ready.
//
// TMEM (512 columns): KV tiles of 80 keys, so per tile S/P (80 columns; P = 40 packed bf16
// words over the first S columns) + O (16 NV columns) -> 3 x (80 + 80) = 480.  Because P
// aliases S, S_t(j + 1) is issued right after P.V_t(j) (the tensor pipe executes one
// issuer's MMAs in order), and the commit that signals S_t(j + 1) also proves P.V_t(j)
// complete: the softmax never waits for O separately inside an item.
//
// Warps: 0-11 softmax + epilogue (tile t = warp / 4, TMEM lane quarter warp % 4, one thread
// per query row), 12 MMA issuer (owns TMEM), 13 TMA producer, 14 fixer (ones column of V
// for the row sums; the dh % 16 != 0 pad-column key mask of partial KV tiles).
// Shared memory: Q 3 x 20 KB (one buffer per tile, reloaded when the tile's last S of an
// item is done), a 3-stage K ring and V ring of 80-row tiles, and an O staging block per
// tile (each warp stages its 32 rows and issues one TMA tensor store).
#include "tc_ptx.cuh"

namespace pab {
namespace tc {
extern long long* g_trace;  // attn_tc.cu: pab_attn_debug_trace
}
namespace f3 {

using namespace pab::tc;

constexpr int kTiles = 3;
constexpr int kSoftmaxWarps = 4 * kTiles;
constexpr int kMmaWarp = kSoftmaxWarps, kTmaWarp = kSoftmaxWarps + 1, kFixWarp = kSoftmaxWarps + 2;
constexpr int kThreads = 32 * (kSoftmaxWarps + 3);
constexpr int kRows = 128;  // query rows per tile == TMEM lanes
constexpr int kKv = 80;     // keys per KV tile
constexpr int kStages = 3;
constexpr uint32_t kTmemCols = 512;

#ifndef PAB_F3_POLY_DIV
#define PAB_F3_POLY_DIV 3  // one column pair in PAB_F3_POLY_DIV on the FMA pipe (0: MUFU only)
#endif

struct Params {
    int n_q, n_k, n_b, heads, dh;
    int row_tiles;    // 128-row query tiles per (problem, head)
    int n_kv;         // KV tiles per problem
    int n_trips;      // tile triples per (problem, head)
    int n_items;      // n_trips * heads * problems
    float scale_log2;  // scale * log2(e)
    long long* trace;
};

template <int N128, int N32, int NV>
struct Geometry {
    static constexpr int kOCols = 16 * NV;
    static constexpr int kSCol0 = 0;                  // S/P of tile t at kSCol0 + kKv t
    static constexpr int kOCol0 = kKv * kTiles;       // O of tile t at kOCol0 + kOCols t
    static constexpr int kQSlot = 20480;              // one 128-row Q tile, dh <= 80
    static constexpr int kK128 = kKv * 128, kK32 = kKv * 32, kVAtom = kKv * 32;
    static constexpr int kSlotKV = 13312;             // 80-row K or V tile (13 KB, 1 KB aligned)
    static constexpr int kQ0 = 0;
    static constexpr int kK0 = kTiles * kQSlot;
    static constexpr int kV0 = kK0 + kStages * kSlotKV;
    static constexpr int kStg0 = kV0 + kStages * kSlotKV;  // O staging: [tile][128 rows][2 dh]
    static constexpr int kStageRow = 144;
    static constexpr int kBar = kStg0 + kTiles * kRows * kStageRow;
    static constexpr int kSmem = kBar + 512 + 1024;
    static_assert(N128 * 16384 + N32 * 4096 <= kQSlot, "Q slot");
    static_assert(N128 * kK128 + N32 * kK32 <= kSlotKV && NV * kVAtom <= kSlotKV, "K/V slot");
    static_assert(kOCol0 + kTiles * kOCols <= (int)kTmemCols, "TMEM");
    static_assert(kSmem <= 232448, "shared memory");
};

struct Bars {
    uint64_t q_full[kTiles], q_ready[kTiles], q_empty[kTiles];
    uint64_t k_full[kStages], k_ready[kStages], k_empty[kStages];
    uint64_t v_full[kStages], v_ready[kStages], v_empty[kStages];
    uint64_t s_full[kTiles], p_full[kTiles], o_done[kTiles];
};

// S_t = Q_t K^T for dh = 72 (4 SW128 K-steps + 1 SW32 step) as one asm group, one elect
__device__ __forceinline__ void mma_s_72(uint32_t d, uint64_t q128, uint64_t k128, uint64_t q32, uint64_t k32,
                                         uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 qa, ka;\n\t"
        "setp.ne.b32 pf, %5, %5;\n\t"
        "setp.eq.b32 pt, %5, %5;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %6, pf;\n\t"
        "add.s64 qa, %1, 2;\n\tadd.s64 ka, %2, 2;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], qa, ka, %6, pt;\n\t"
        "add.s64 qa, %1, 4;\n\tadd.s64 ka, %2, 4;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], qa, ka, %6, pt;\n\t"
        "add.s64 qa, %1, 6;\n\tadd.s64 ka, %2, 6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], qa, ka, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %4, %6, pt;\n\t}" ::"r"(d),
        "l"(q128), "l"(k128), "l"(q32), "l"(k32), "r"(0), "r"(idesc)
        : "memory");
}
// O_t += P_t V for 5 K-steps of 16 keys (80 keys): A = P_t from TMEM (+8 columns per step),
// B = V atoms (+512 B per step -> +32 in the descriptor)
__device__ __forceinline__ void mma_pv_5(uint32_t o, uint32_t pt, uint64_t v, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, pa, pt;\n\t.reg .b64 vb;\n\t.reg .b32 pc;\n\t"
        "setp.ne.b32 pa, %4, 0;\n\t"
        "setp.eq.b32 pt, %4, %4;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, pa;\n\t"
        "add.s64 vb, %2, 32;\n\tadd.u32 pc, %1, 8;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [pc], vb, %3, pt;\n\t"
        "add.s64 vb, %2, 64;\n\tadd.u32 pc, %1, 16;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [pc], vb, %3, pt;\n\t"
        "add.s64 vb, %2, 96;\n\tadd.u32 pc, %1, 24;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [pc], vb, %3, pt;\n\t"
        "add.s64 vb, %2, 128;\n\tadd.u32 pc, %1, 32;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [pc], vb, %3, pt;\n\t}" ::"r"(o),
        "r"(pt), "l"(v), "r"(idesc), "r"(accumulate)
        : "memory");
}
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

// MMA-warp wait: try_wait without a suspend-time hint (the issuer must react at once; the
// hinted wait of tc_ptx.cuh measured ~350 clk from the softmax's arrive to the next P.V)
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred x;\n"
        "SPIN_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 x, [%0], %1;\n\t"
        "@!x bra SPIN_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

#define PAB_F3_ST8U(taddr, r)                                                                                \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]), \
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])                       \
                 : "memory")

__device__ __forceinline__ float max3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// 2^x for a pair on the FMA pipe (degree-3 minimax polynomial on f32x2, exponent add as an
// integer; clamp at -126 so the exponent field cannot wrap); rel err 7.5e-5
__device__ __forceinline__ void poly_exp2_x2(float& a, float& b) {
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

#define F3_TRACE(cond, itn, t, ev)                                                             \
    do {                                                                                       \
        if (PAB_F3_TRACE_ON && p.trace != nullptr && (cond) && blockIdx.x == 0 && (itn) < 40) \
            p.trace[((itn) * 4 + (t)) * 8 + (ev)] = clock64();                                 \
    } while (0)
#ifdef PAB_F3_TRACE
#define PAB_F3_TRACE_ON 1
#else
#define PAB_F3_TRACE_ON 0
#endif

template <int N128, int N32, int NV>
__global__ void __launch_bounds__(kThreads, 1)
    attn_f3_kernel(const __grid_constant__ CUtensorMap q128, const __grid_constant__ CUtensorMap q32,
                   const __grid_constant__ CUtensorMap k128, const __grid_constant__ CUtensorMap k32,
                   const __grid_constant__ CUtensorMap v32, const __grid_constant__ CUtensorMap omap,
                   const Params p) {
    using G = Geometry<N128, N32, NV>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + G::kBar);
    __shared__ uint32_t tmem_base_slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // item -> (head fastest, triple, problem): concurrently running CTAs share K/V in L2
    struct Item {
        int h, a_idx, b_idx, tile0, n_t;  // n_t: query tiles of this item (1..3)
    };
    auto decode = [&](int item) {
        Item it;
        it.h = item % p.heads;
        const int rest = item / p.heads;
        const int trip = rest % p.n_trips, az = rest / p.n_trips;
        it.a_idx = az / p.n_b;
        it.b_idx = az - it.a_idx * p.n_b;
        it.tile0 = 3 * trip;
        it.n_t = min(3, p.row_tiles - it.tile0);
        return it;
    };
    const int my_items = (p.n_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int n_kv = p.n_kv;
    auto item_at = [&](int c) { return decode((int)blockIdx.x + c * (int)gridDim.x); };
    const bool padmask = N32 > 0 && (p.dh & 15) != 0;

    if (warp == kTmaWarp && lane == 0) {
        prefetch_map(&omap);
        prefetch_map(&q128);
        prefetch_map(&k128);
        prefetch_map(&v32);
        if (N32) {
            prefetch_map(&q32);
            prefetch_map(&k32);
        }
        for (int t = 0; t < kTiles; ++t) {
            mbar_init(&bars->q_full[t], 1);
            mbar_init(&bars->q_ready[t], 1);
            mbar_init(&bars->q_empty[t], 1);
            mbar_init(&bars->s_full[t], 1);
            mbar_init(&bars->p_full[t], 4);
            mbar_init(&bars->o_done[t], 1);
        }
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars->k_full[s], 1);
            mbar_init(&bars->k_ready[s], 1);
            mbar_init(&bars->k_empty[s], 1);
            mbar_init(&bars->v_full[s], 1);
            mbar_init(&bars->v_ready[s], 1);
            mbar_init(&bars->v_empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    constexpr uint32_t tmem = 0;  // all 512 columns: base = lane 0, column 0

    if (warp < kSoftmaxWarps) {
        // ========================================= softmax + epilogue of query tile t
        const int t = warp / 4, wl = warp % 4;
        const uint32_t lane_off = (uint32_t)(wl * 32) << 16;
        const uint32_t s_tmem = tmem + lane_off + G::kSCol0 + kKv * t;
        const uint32_t o_tmem = tmem + lane_off + G::kOCol0 + G::kOCols * t;
        const int tail = p.n_k - (n_kv - 1) * kKv;  // live keys of the last KV tile
        uint8_t* stg_warp = smem + G::kStg0 + (t * kRows + wl * 32) * (2 * p.dh);
        uint8_t* stg = stg_warp + lane * (2 * p.dh);
        const unsigned long long sc2 = f2_pack(p.scale_log2, p.scale_log2);
        // O of the tile's previous item -> normalised bf16 rows -> smem -> one TMA store per warp
        auto epilogue = [&](const Item& it) {
            float o[16 * NV];
#pragma unroll
            for (int cc = 0; cc < NV; ++cc) PAB_TMEM_LD16(o_tmem + 16 * cc, (o + 16 * cc));
            tmem_wait_ld();
            float l = o[16 * (NV - 1)];
#pragma unroll
            for (int e = 1; e < 16; ++e) l = (e == p.dh % 16) ? o[16 * (NV - 1) + e] : l;  // row sum: column dh
            const float inv = (l > 0.f) ? 1.0f / l : 0.f;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // last store read stg
            __syncwarp();
#pragma unroll
            for (int e = 0; e < 16 * NV; e += 8) {
                if (e < p.dh) {
                    uint32_t w[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) w[q] = pack_bf16(o[e + 2 * q] * inv, o[e + 2 * q + 1] * inv);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(stg + 2 * e)), "r"(w[0]),
                                 "r"(w[1]), "r"(w[2]), "r"(w[3])
                                 : "memory");
                }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0)
                asm volatile(
                    "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n\t"
                    "cp.async.bulk.commit_group;" ::"l"(reinterpret_cast<uint64_t>(&omap)),
                    "r"(smem_u32(stg_warp)), "r"(0), "r"(it.h), "r"((it.tile0 + t) * kRows + wl * 32),
                    "r"(it.b_idx), "r"(it.a_idx)
                    : "memory");
        };
        Item prev;
        bool have_prev = false;
        int it_n = 0;  // iterations of this tile (items without tile t are skipped entirely)
        for (int c = 0; c < my_items; ++c) {
            const Item it = item_at(c);
            if (t >= it.n_t) continue;
            float m_run = -INFINITY;
            for (int j = 0; j < n_kv; ++j, ++it_n) {
                F3_TRACE(wl == 0 && lane == 0, it_n, t, 0);
                mbar_wait(&bars->s_full[t], it_n & 1);
                tc_fence_after();
                F3_TRACE(wl == 0 && lane == 0, it_n, t, 1);
                // S_t(j) landed: every earlier MMA of this tile is complete, so O_t holds the
                // previous item's final sum at j == 0
                if (j == 0 && have_prev) epilogue(prev);
                float s[kKv];
                PAB_TMEM_LD32(s_tmem, s);
                PAB_TMEM_LD32(s_tmem + 32, (s + 32));
                PAB_TMEM_LD16(s_tmem + 64, (s + 64));
                tmem_wait_ld();
                F3_TRACE(wl == 0 && lane == 0, it_n, t, 2);
                const bool masked = !padmask && (j == n_kv - 1) && (tail < kKv);
                if (masked) {
#pragma unroll
                    for (int cc = 0; cc < kKv; ++cc) s[cc] = (cc < tail) ? s[cc] : -INFINITY;
                }
                constexpr int kG = kKv / 4;  // 4 independent FMNMX3 chains of 20
                float m4[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    float m = s[kG * g];
#pragma unroll
                    for (int cc = 1; cc + 1 < kG; cc += 2) m = max3(m, s[kG * g + cc], s[kG * g + cc + 1]);
                    m4[g] = (kG % 2 == 0) ? fmaxf(m, s[kG * g + kG - 1]) : m;
                }
                const float m_tile = max3(fmaxf(m4[0], m4[1]), m4[2], m4[3]) * p.scale_log2;
                // lazy rescale: the running max is raised (O_t rescaled in TMEM) only when this
                // tile's max exceeds it by more than 2^8, so P <= 256
                const bool need = m_tile > m_run + 8.0f;
                if (__any_sync(0xffffffffu, need)) {
                    const float m_new = need ? m_tile : m_run;
                    if (j > 0) {
                        const float alpha = fast_exp2(m_run - m_new);
#pragma unroll 1
                        for (int cc = 0; cc < NV; ++cc) {
                            float o[16];
                            PAB_TMEM_LD16(o_tmem + 16 * cc, o);
                            tmem_wait_ld();
#pragma unroll
                            for (int e = 0; e < 16; ++e) o[e] *= alpha;
                            PAB_TMEM_ST16(o_tmem + 16 * cc, o);
                        }
                    }
                    m_run = m_new;
                }
                F3_TRACE(wl == 0 && lane == 0, it_n, t, 3);
                const unsigned long long nm2 = f2_pack(-m_run, -m_run);
                uint32_t pk[kKv / 2];
#pragma unroll
                for (int q = 0; q < kKv / 2; ++q) {
                    float2 x = f2_unpack(f2_fma(f2_pack(s[2 * q], s[2 * q + 1]), sc2, nm2));
                    if (PAB_F3_POLY_DIV > 0 && !masked && (q % (PAB_F3_POLY_DIV > 0 ? PAB_F3_POLY_DIV : 1)) ==
                                                              (PAB_F3_POLY_DIV > 0 ? PAB_F3_POLY_DIV : 1) - 1) {
                        poly_exp2_x2(x.x, x.y);
                    } else {
                        x.x = fast_exp2(x.x);
                        x.y = fast_exp2(x.y);
                    }
                    pk[q] = pack_bf16(x.x, x.y);
                }
                F3_TRACE(wl == 0 && lane == 0, it_n, t, 4);
                // P over the first 40 S columns (this warp's lanes only; S is in registers)
                PAB_TMEM_ST16U(s_tmem, pk);
                PAB_TMEM_ST16U(s_tmem + 16, (pk + 16));
                PAB_F3_ST8U(s_tmem + 32, (pk + 32));
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->p_full[t]);
                F3_TRACE(wl == 0 && lane == 0, it_n, t, 5);
            }
            prev = it;
            have_prev = true;
        }
        if (have_prev) {
            mbar_wait(&bars->o_done[t], (it_n - 1) & 1);
            tc_fence_after();
            epilogue(prev);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // O stores done before exit
    } else if (warp == kTmaWarp) {
        // ===================================================== TMA producer (lane 0)
        if (lane == 0) {
            constexpr uint32_t kQBytes = kRows * (N128 * 128 + N32 * 32);
            constexpr uint32_t kKBytes = kKv * (N128 * 128 + N32 * 32);
            constexpr uint32_t kVBytes = kKv * NV * 32;
            int qn[kTiles] = {0, 0, 0};  // Q loads per tile so far
            int g = 0;                   // K/V tiles loaded so far
            for (int c = 0; c < my_items; ++c) {
                const Item it = item_at(c);
#pragma unroll
                for (int t = 0; t < kTiles; ++t) {
                    if (t >= it.n_t) break;
                    if (qn[t] > 0) mbar_wait(&bars->q_empty[t], (qn[t] - 1) & 1);
                    ++qn[t];
                    uint8_t* dst = smem + G::kQ0 + t * G::kQSlot;
                    const int i0 = (it.tile0 + t) * kRows;
                    mbar_expect_tx(&bars->q_full[t], kQBytes);
                    for (int blk = 0; blk < N128; ++blk)
                        tma_load_5d(dst + blk * 16384, &q128, &bars->q_full[t], 64 * blk, it.h, i0, it.b_idx, it.a_idx);
                    for (int blk = 0; blk < N32; ++blk)
                        tma_load_5d(dst + N128 * 16384 + blk * 4096, &q32, &bars->q_full[t], 64 * N128 + 16 * blk,
                                    it.h, i0, it.b_idx, it.a_idx);
                }
                for (int j = 0; j < n_kv; ++j, ++g) {
                    const int st = g % kStages;
                    if (g >= kStages) mbar_wait(&bars->k_empty[st], ((g / kStages) - 1) & 1);
                    uint8_t* kd = smem + G::kK0 + st * G::kSlotKV;
                    mbar_expect_tx(&bars->k_full[st], kKBytes);
                    for (int blk = 0; blk < N128; ++blk)
                        tma_load_5d(kd + blk * G::kK128, &k128, &bars->k_full[st], 64 * blk, it.h, j * kKv, it.b_idx,
                                    it.a_idx);
                    for (int blk = 0; blk < N32; ++blk)
                        tma_load_5d(kd + N128 * G::kK128 + blk * G::kK32, &k32, &bars->k_full[st], 64 * N128 + 16 * blk,
                                    it.h, j * kKv, it.b_idx, it.a_idx);
                    if (g >= kStages) mbar_wait(&bars->v_empty[st], ((g / kStages) - 1) & 1);
                    uint8_t* vd = smem + G::kV0 + st * G::kSlotKV;
                    mbar_expect_tx(&bars->v_full[st], kVBytes);
                    for (int blk = 0; blk < NV; ++blk)
                        tma_load_5d(vd + blk * G::kVAtom, &v32, &bars->v_full[st], 16 * blk, it.h, j * kKv, it.b_idx,
                                    it.a_idx);
                }
            }
        }
    } else if (warp == kFixWarp) {
        // ====================================== fixer: V[:, dh] = 1 (row sums); with padmask also
        // Q[:, dh] = 1 and K[r, dh] = -1e30 for the rows past n_k of a partial last KV tile.
        // SW32 atoms: row r at 32 r, 16-byte chunk index XOR (r >> 2) & 1.
        const int col = p.dh % 16;
        const uint32_t atom_off = (uint32_t)(p.dh / 16) * (uint32_t)G::kVAtom;
        const uint32_t cw = (uint32_t)(col & 7) * 2;
        auto sw32 = [&](int r) { return (uint32_t)r * 32u + (((uint32_t)(col >> 3) ^ (uint32_t)((r >> 2) & 1)) * 16u) + cw; };
        const int blk = (p.dh - 64 * N128) >> 4;
        const uint32_t q_off = (uint32_t)(N128 * 16384 + blk * 4096), k_off = (uint32_t)(N128 * G::kK128 + blk * G::kK32);
        const int tail_k = p.n_k - (n_kv - 1) * kKv;
        const __nv_bfloat16 one = __float2bfloat16_rn(1.0f), neg = __float2bfloat16_rn(-1e30f);
        int qn[kTiles] = {0, 0, 0};
        int g = 0;
        for (int c = 0; c < my_items; ++c) {
            const Item it = item_at(c);
#pragma unroll
            for (int t = 0; t < kTiles; ++t) {
                if (t >= it.n_t) break;
                mbar_wait(&bars->q_full[t], qn[t] & 1);
                ++qn[t];
                if (padmask) {
                    uint8_t* qd = smem + G::kQ0 + t * G::kQSlot + q_off;
                    for (int r = lane; r < kRows; r += 32) *reinterpret_cast<__nv_bfloat16*>(qd + sw32(r)) = one;
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->q_ready[t]);
            }
            for (int j = 0; j < n_kv; ++j, ++g) {
                const int st = g % kStages;
                mbar_wait(&bars->k_full[st], (g / kStages) & 1);
                if (padmask && j == n_kv - 1 && tail_k < kKv) {
                    uint8_t* kd = smem + G::kK0 + st * G::kSlotKV + k_off;
                    for (int r = tail_k + lane; r < kKv; r += 32) *reinterpret_cast<__nv_bfloat16*>(kd + sw32(r)) = neg;
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->k_ready[st]);
                mbar_wait(&bars->v_full[st], (g / kStages) & 1);
                uint8_t* vd = smem + G::kV0 + st * G::kSlotKV + atom_off;
                for (int r = lane; r < kKv; r += 32) *reinterpret_cast<__nv_bfloat16*>(vd + sw32(r)) = one;
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->v_ready[st]);
            }
        }
    } else if (warp == kMmaWarp) {
        // ============================ MMA issuer (warp-converged; one elected lane issues)
        const uint32_t idS_full = idesc_bf16(128, kKv, 0);
        constexpr uint32_t idO = idesc_bf16(128, G::kOCols, 1);
        const uint32_t q_lo = smem_u32(smem + G::kQ0) >> 4, k_lo = smem_u32(smem + G::kK0) >> 4;
        const uint32_t v_lo = smem_u32(smem + G::kV0) >> 4;
        constexpr uint32_t kHi128 = (1024u >> 4) | (1u << 14) | (kLayoutSW128 << 29);
        constexpr uint32_t kHi32 = (256u >> 4) | (1u << 14) | (kLayoutSW32 << 29);
        constexpr uint32_t kLbo16 = (16u >> 4) << 16;
        constexpr uint32_t kLboV = ((uint32_t)G::kVAtom >> 4) << 16;
        auto ncols_of = [&](int j) {
            if (padmask) return kKv;  // padded keys are scored -1e30 by the MMA itself
            const int n = min(kKv, p.n_k - j * kKv);
            return (n + 15) & ~15;
        };
        auto issue_s = [&](int t, int kst, int ncols) {
            const uint32_t ka = k_lo + ((kst * G::kSlotKV) >> 4);
            const uint32_t qa = q_lo + ((t * G::kQSlot) >> 4);
            const uint32_t idS = (idS_full & ~(0x3Fu << 17)) | ((uint32_t)(ncols >> 3) << 17);
            const uint32_t d = tmem + G::kSCol0 + kKv * t;
            if (N128 == 1 && N32 == 1) {
                const uint64_t dq = ((uint64_t)kHi128 << 32) | (qa | kLbo16);
                const uint64_t dk = ((uint64_t)kHi128 << 32) | (ka | kLbo16);
                const uint64_t dq32 = ((uint64_t)kHi32 << 32) | ((qa + (16384 >> 4)) | kLbo16);
                const uint64_t dk32 = ((uint64_t)kHi32 << 32) | ((ka + (G::kK128 >> 4)) | kLbo16);
                mma_s_72(d, dq, dk, dq32, dk32, idS);
                return;
            }
            uint32_t acc = 0;
            for (int blk = 0; blk < N128; ++blk)
                for (int k = 0; k < 4; ++k) {
                    const uint32_t oq = (blk * 16384 + 32 * k) >> 4, ok = (blk * G::kK128 + 32 * k) >> 4;
                    tc_mma(d, ((uint64_t)kHi128 << 32) | ((qa + oq) | kLbo16), ((uint64_t)kHi128 << 32) | ((ka + ok) | kLbo16),
                           idS, acc);
                    acc = 1;
                }
            for (int blk = 0; blk < N32; ++blk) {
                const uint32_t oq = (N128 * 16384 + blk * 4096) >> 4, ok = (N128 * G::kK128 + blk * G::kK32) >> 4;
                tc_mma(d, ((uint64_t)kHi32 << 32) | ((qa + oq) | kLbo16), ((uint64_t)kHi32 << 32) | ((ka + ok) | kLbo16),
                       idS, acc);
                acc = 1;
            }
        };
        auto issue_pv = [&](int t, int vst, uint32_t accumulate, int ncols) {
            const uint32_t va = v_lo + ((vst * G::kSlotKV) >> 4);
            const uint64_t dv = ((uint64_t)kHi32 << 32) | (va | kLboV);
            const uint32_t o = tmem + G::kOCol0 + G::kOCols * t, pt = tmem + G::kSCol0 + kKv * t;
            if (ncols == kKv) {
                mma_pv_5(o, pt, dv, idO, accumulate);
                return;
            }
            for (int k = 0; 16 * k < ncols; ++k) mma_ts(o, pt + 8 * k, dv + ((512 * k) >> 4), idO, accumulate | (k > 0));
        };
        // per tile: Q loads consumed (qn), S/PV iterations (sn); KV tile counter g
        int qn[kTiles] = {0, 0, 0}, sn[kTiles] = {0, 0, 0};
        int g = 0;
        if (my_items > 0) {
            // first S of every tile of item 0
            const Item it = item_at(0);
            mbar_spin(&bars->k_ready[0], 0);
#pragma unroll
            for (int t = 0; t < kTiles; ++t) {
                if (t >= it.n_t) break;
                mbar_spin(&bars->q_ready[t], qn[t] & 1);
                tc_fence_after();
                issue_s(t, 0, ncols_of(0));
                tc_commit(&bars->s_full[t]);
                if (n_kv == 1) {
                    tc_commit(&bars->q_empty[t]);
                    ++qn[t];
                }
            }
            tc_commit(&bars->k_empty[0]);
        }
        for (int c = 0; c < my_items; ++c) {
            const Item it = item_at(c);
            for (int j = 0; j < n_kv; ++j, ++g) {
                // next iteration: (c, j + 1) or (c + 1, 0)
                int c1 = c, j1 = j + 1;
                if (j1 == n_kv) {
                    c1 = c + 1;
                    j1 = 0;
                }
                const bool has_next = c1 < my_items;
                const Item it1 = (has_next && c1 != c) ? item_at(c1) : it;
                const int g1 = g + 1, st1 = g1 % kStages;
                const int st = g % kStages;
                F3_TRACE(lane == 0, g, 3, 0);
                mbar_spin(&bars->v_ready[st], (g / kStages) & 1);
                F3_TRACE(lane == 0, g, 3, 1);
                // tiles in order: P.V_t(j) then S_t(next) (which overwrites P_t: issued after it)
                const int nt = max(it.n_t, has_next ? it1.n_t : 0);
                bool k_in = false;
#pragma unroll
                for (int t = 0; t < kTiles; ++t) {
                    if (t >= nt) break;
                    if (t < it.n_t) {
                        mbar_spin(&bars->p_full[t], sn[t] & 1);
                        if (t == 0) F3_TRACE(lane == 0, g, 3, 2);
                        tc_fence_after();
                        issue_pv(t, st, j > 0, ncols_of(j));
                        tc_commit(&bars->o_done[t]);
                        if (t == 0) F3_TRACE(lane == 0, g, 3, 3);
                        ++sn[t];
                    }
                    if (has_next && t < it1.n_t) {
                        if (!k_in) {  // the next K tile, waited only once a P.V has gone out
                            mbar_spin(&bars->k_ready[st1], (g1 / kStages) & 1);
                            k_in = true;
                        }
                        if (t == 0) F3_TRACE(lane == 0, g, 3, 4);
                        if (j1 == 0) mbar_spin(&bars->q_ready[t], qn[t] & 1);
                        tc_fence_after();
                        issue_s(t, st1, ncols_of(j1));
                        tc_commit(&bars->s_full[t]);
                        if (t == 0) F3_TRACE(lane == 0, g, 3, 5);
                        if (t == 1) F3_TRACE(lane == 0, g, 3, 6);
                        if (t == 2) F3_TRACE(lane == 0, g, 3, 7);
                        if (j1 == n_kv - 1) {  // last S of this tile's item: Q may be reloaded
                            tc_commit(&bars->q_empty[t]);
                            ++qn[t];
                        }
                    }
                }
                tc_commit(&bars->v_empty[st]);
                if (has_next) tc_commit(&bars->k_empty[st1]);
            }
        }
    }
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

template <int N128, int N32, int NV>
int launch(const pab_attn_args* a, cudaStream_t st) {
    using G = Geometry<N128, N32, NV>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(attn_f3_kernel<N128, N32, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 G::kSmem) != cudaSuccess)
            return launch_status("attn_f3 smem attribute");
        attr_set = true;
    }
    CUtensorMap mq128, mq32, mk128, mk32, mv32, mo;
    const CUtensorMapSwizzle big = N128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B;
    const int inner = N128 ? 64 : 16;
    if (!make_map(&mq128, a->q, a->dh, a->heads, a->n_q, a->n_b, a->n_a, a->q_si, a->q_sb, a->q_sa, inner, kRows, 1,
                  big) ||
        !make_map(&mq32, a->q, a->dh, a->heads, a->n_q, a->n_b, a->n_a, a->q_si, a->q_sb, a->q_sa, 16, kRows, 1,
                  CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_map(&mk128, a->k, a->dh, a->heads, a->n_k, a->n_b, a->n_a, a->k_si, a->k_sb, a->k_sa, inner, kKv, 1,
                  big) ||
        !make_map(&mk32, a->k, a->dh, a->heads, a->n_k, a->n_b, a->n_a, a->k_si, a->k_sb, a->k_sa, 16, kKv, 1,
                  CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_map(&mv32, a->v, a->dh, a->heads, a->n_k, a->n_b, a->n_a, a->v_si, a->v_sb, a->v_sa, 16, kKv, 1,
                  CU_TENSOR_MAP_SWIZZLE_32B) ||
        // O: one TMA tensor store per warp (box = dh x 32 rows)
        !make_map(&mo, a->o, a->dh, a->heads, a->n_q, a->n_b, a->n_a, a->o_si, a->o_sb, a->o_sa, a->dh, 32, 1,
                  CU_TENSOR_MAP_SWIZZLE_NONE))
        return PAB_ERR_CUDA;
    Params p;
    p.n_q = a->n_q;
    p.n_k = a->n_k;
    p.n_b = a->n_b;
    p.heads = a->heads;
    p.dh = a->dh;
    p.scale_log2 = a->scale * 1.4426950408889634f;
    p.trace = tc::g_trace;
    p.row_tiles = (a->n_q + kRows - 1) / kRows;
    p.n_kv = (a->n_k + kKv - 1) / kKv;
    p.n_trips = (p.row_tiles + 2) / 3;
    const int64_t items = (int64_t)p.n_trips * a->heads * a->n_a * a->n_b;
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
    attn_f3_kernel<N128, N32, NV><<<grid, kThreads, G::kSmem, st>>>(mq128, mq32, mk128, mk32, mv32, mo, p);
    return launch_status("attn_f3");
}

}  // namespace f3

bool attn_f3_supported(const pab_attn_args* a) { return a->dh % 8 == 0 && a->dh <= 72; }

int attn_f3_launch(const pab_attn_args* a, cudaStream_t st) {
    const int n128 = a->dh / 64;
    const int n32 = (a->dh - 64 * n128 + 15) / 16;
    const int nv = a->dh / 16 + 1;
#define PAB_F3(A, B, C) \
    if (n128 == A && n32 == B && nv == C) return f3::launch<A, B, C>(a, st)
    PAB_F3(0, 1, 1);
    PAB_F3(0, 1, 2);
    PAB_F3(0, 2, 2);
    PAB_F3(0, 2, 3);
    PAB_F3(0, 3, 3);
    PAB_F3(0, 3, 4);
    PAB_F3(0, 4, 4);
    PAB_F3(1, 0, 5);
    PAB_F3(1, 1, 5);
#undef PAB_F3
    return PAB_ERR_UNSUPPORTED;
}

}  // namespace pab

// Row-per-thread tcgen05 flash attention for sm_100a: the production kernel for
// the spatial (K1) and cross (K3) attention sites.
//
// reference op: numerics.scaled_dot_attention (pkg/src/pab_engine/numerics.py:133-151)
// as used by _axis_attention_compute(temporal_axis=False) and _cross_attention_compute
// (pkg/src/pab_engine/model.py:346-359, 376-385):
//   logits = q k^T * (1/sqrt(dh)); p = softmax(logits) (max-shifted); out = p v
//
// CTA (512 threads, one persistent CTA per SM, two 128-row query tiles per work item
// sharing every K/V tile):
//   warps 0-3   softmax of query tile 0, one thread per query row (= TMEM lane)
//   warps 4-7   softmax of query tile 1
//   warps 8-11  epilogue: O / l -> bf16 rows in global memory (both tiles)
//   warp  12    MMA issuer (one elected lane; also owns the TMEM allocation)
//   warp  13    TMA producer (one elected lane)
//   warps 14-15 idle (register donors for setmaxnreg)
// TMEM (512 columns): S_t at [128t, 128t + 128), P_t (bf16 pairs) over the first
// 64 columns of S_t, O_t at [256 + 128t, 256 + 128t + dh_pad).
//
// Per tile t and KV tile j the MMA warp issues  O_t += P_t(j) V_j  (A operand = P
// straight from TMEM) followed by  S_t(j+1) = Q_t K_{j+1}^T  which overwrites the
// P_t(j) columns; tcgen05 MMAs of one thread execute in issue order, so the PV
// read completes before the next S lands.  While softmax t works on S_t(j+1) the
// tensor pipe runs the other tile's PV/S pair, so MMA and exp2 overlap.
//
// Online softmax: each thread holds its row's 128 scores in registers; the running
// max is only raised (and O rescaled in place in TMEM) when a tile's max exceeds it
// by more than 2^8, so P <= 256 in bf16 and the O correction is rare.  exp2 runs on
// MUFU for most columns and on the FMA pipe (degree-3 polynomial on f32x2 pairs) for
// one pair in PAB_FA_POLY_DIV, balancing the two pipes.
#include "tc_ptx.cuh"

namespace pab {
namespace tc {
extern long long* g_trace;  // attn_tc.cu: pab_attn_debug_trace
}
namespace fa {

using namespace pab::tc;

constexpr int kThreads = 512;
constexpr int kRows = 128;   // query rows per tile == TMEM lanes
constexpr int kKv = 128;     // keys per KV tile
constexpr int kMmaWarp = 12;
constexpr int kTmaWarp = 13;
constexpr int kEpiWarp0 = 8;
constexpr uint32_t kTmemCols = 512;

#ifndef PAB_FA_POLY_DIV
#define PAB_FA_POLY_DIV 4   // one column pair in PAB_FA_POLY_DIV on the FMA pipe (0: MUFU only)
#endif
#ifndef PAB_FA_SOFTMAX_REGS
#define PAB_FA_SOFTMAX_REGS 200
#endif
#ifndef PAB_FA_OTHER_REGS
#define PAB_FA_OTHER_REGS 56
#endif
static_assert(2 * 128 * PAB_FA_SOFTMAX_REGS + 2 * 128 * PAB_FA_OTHER_REGS <= 65536, "register file");

struct Params {
    int n_q, n_k, n_b, heads, dh;
    int row_tiles;     // 128-row query tiles per (problem, head)
    int n_kv;          // KV tiles per problem
    int n_pairs;       // query-tile pairs per (problem, head)
    int n_items;       // n_pairs * heads * problems
    float scale_log2;  // scale * log2(e)
    __nv_bfloat16* o;
    int64_t o_sa, o_sb, o_si;
    long long* trace;  // debug: clock64 event log of CTA 0, nullptr in production
};

// trace slot layout: [(iteration * 2 + tile) * 16 + event], iterations < 64 of CTA 0
#ifndef PAB_FA_TRACE
#define FA_TRACE(cond, itn, t, ev) \
    do {                           \
    } while (0)
#else
#define FA_TRACE(cond, itn, t, ev)                                                        \
    do {                                                                                  \
        if (p.trace != nullptr && (cond) && blockIdx.x == 0 && (itn) < 64)                \
            p.trace[((itn) * 2 + (t)) * 16 + (ev)] = clock64();                           \
    } while (0)
#endif

template <int N128, int N32>
struct Geometry {
    static constexpr int kDhPad = 64 * N128 + 16 * N32;
    static constexpr int kTileBytes = N128 * 16384 + N32 * 4096;  // one 128-row operand tile
    static constexpr int kQ0 = 0;                                 // 2 item buffers x 2 tiles
    static constexpr int kK0 = 4 * kTileBytes;                    // 3-stage K ring
    static constexpr int kV0 = 7 * kTileBytes;                    // 3-stage V ring
    static constexpr int kL0 = 10 * kTileBytes;                   // final row sums [tile][row]
    static constexpr int kBar = kL0 + 2 * kRows * 4;
    static constexpr int kSmem = kBar + 512 + 1024;  // + barriers + alignment slack
    static_assert(kSmem <= 232448, "attention tiles exceed the 227 KB shared memory of one CTA");
    static_assert(kDhPad <= 128, "O tiles exceed TMEM");
};

struct Bars {
    uint64_t q_full[2], q_empty[2], k_full[3], k_empty[3], v_full[3], v_empty[3];
    uint64_t s_full[2], p_full[2], o_full[2], o_free[2], l_full[2];
    uint32_t tmem_base;
};

__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// single-thread issue (the MMA loop runs on lane 0 of the MMA warp): descriptors are
// passed as (lo, hi) words so advancing a K step is one 32-bit add on the lo word
__device__ __forceinline__ void mma_ss1(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 a, b;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "mov.b64 a, {%1, %2};\n\t"
        "mov.b64 b, {%3, %4};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, p;\n\t}" ::"r"(d_tmem),
        "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_ts1(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 b;\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "mov.b64 b, {%2, %3};\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], b, %4, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void commit1(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ float max3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// 2^x for a pair of floats on the FMA pipe: x = i + f with i = round(x) via the
// 1.5*2^23 magic constant, 2^f by a degree-3 minimax polynomial on [-0.5, 0.5]
// (max rel err 7.5e-5, far below the bf16 rounding of P), exponent add by LEA.
__device__ __forceinline__ void poly_exp2_x2(float& a, float& b) {
    a = fmaxf(a, -127.0f);
    b = fmaxf(b, -127.0f);
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

// 128 fp32 scores of this thread's row (TMEM lane) -> registers
__device__ __forceinline__ void load_row128(uint32_t taddr, float* s) {
    PAB_TMEM_LD32(taddr, s);
    PAB_TMEM_LD32(taddr + 32, (s + 32));
    PAB_TMEM_LD32(taddr + 64, (s + 64));
    PAB_TMEM_LD32(taddr + 96, (s + 96));
    tmem_wait_ld();
}

// P = exp2(s * scale_log2 - m) -> bf16 pairs into TMEM (16 columns per 32 scores);
// returns the row-sum contribution.  MASKED: columns >= nv give P = 0.
template <bool MASKED>
__device__ __forceinline__ float exp_store_row(float* s, float scale_log2, float neg_m, uint32_t p_tmem, int nv) {
    const unsigned long long sc2 = f2_pack(scale_log2, scale_log2), nm2 = f2_pack(neg_m, neg_m);
    unsigned long long acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
        uint32_t pk[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int c = 32 * ch + 2 * q;
            float2 x = f2_unpack(f2_fma(f2_pack(s[c], s[c + 1]), sc2, nm2));
            if (PAB_FA_POLY_DIV > 0 && (q % (PAB_FA_POLY_DIV > 0 ? PAB_FA_POLY_DIV : 1)) ==
                                           (PAB_FA_POLY_DIV > 0 ? PAB_FA_POLY_DIV : 1) - 1) {
                poly_exp2_x2(x.x, x.y);
            } else {
#ifdef PAB_FA_DIAG_NOEXP  // timing diagnostic only: exp2 replaced by a multiply
                x.x *= 0.5f;
                x.y *= 0.5f;
#else
                x.x = fast_exp2(x.x);
                x.y = fast_exp2(x.y);
#endif
            }
            if (MASKED) {
                x.x = (c < nv) ? x.x : 0.f;
                x.y = (c + 1 < nv) ? x.y : 0.f;
            }
            acc2[q & 3] = f2_add(acc2[q & 3], f2_pack(x.x, x.y));
            pk[q] = pack_bf16(x.x, x.y);
        }
        PAB_TMEM_ST16U(p_tmem + 16 * ch, pk);
    }
    const unsigned long long a01 = f2_add(acc2[0], acc2[1]), a23 = f2_add(acc2[2], acc2[3]);
    const float2 a = f2_unpack(f2_add(a01, a23));
    return a.x + a.y;
}

template <int N128, int N32>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fa_kernel(const __grid_constant__ CUtensorMap q128, const __grid_constant__ CUtensorMap q32,
                   const __grid_constant__ CUtensorMap k128, const __grid_constant__ CUtensorMap k32,
                   const __grid_constant__ CUtensorMap v32, const Params p) {
    using G = Geometry<N128, N32>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + G::kBar);
    float* l_buf = reinterpret_cast<float*>(smem + G::kL0);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // item -> (head, pair, a, b), head fastest: concurrently running CTAs read all heads of
    // the same q/k/v rows (whole qkv rows per DRAM page visit) and share K/V in L2
    struct Item {
        int h, a_idx, b_idx, tile0;
        bool two;  // second query tile exists
    };
    auto decode = [&](int item) {
        Item it;
        it.h = item % p.heads;
        const int rest = item / p.heads;
        const int pair = rest % p.n_pairs;
        const int az = rest / p.n_pairs;
        it.a_idx = az / p.n_b;
        it.b_idx = az - it.a_idx * p.n_b;
        it.tile0 = 2 * pair;
        it.two = it.tile0 + 1 < p.row_tiles;
        return it;
    };
    const int my_items = (p.n_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int n_kv = p.n_kv;
    const uint32_t tile_bytes = (uint32_t)kRows * (uint32_t)(N128 * 128 + N32 * 32);

    // ---------------------------------------------------------------- setup
    if (warp == kTmaWarp && lane == 0) {
        prefetch_map(&q128);
        prefetch_map(&k128);
        prefetch_map(&v32);
        if (N32) {
            prefetch_map(&q32);
            prefetch_map(&k32);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars->q_full[s], 1);
            mbar_init(&bars->q_empty[s], 1);
            mbar_init(&bars->s_full[s], 1);
            mbar_init(&bars->p_full[s], 4);
            mbar_init(&bars->o_full[s], 1);
            mbar_init(&bars->o_free[s], 4);
            mbar_init(&bars->l_full[s], 4);
        }
        for (int s = 0; s < 3; ++s) {
            mbar_init(&bars->k_full[s], 1);
            mbar_init(&bars->k_empty[s], 1);
            mbar_init(&bars->v_full[s], 1);
            mbar_init(&bars->v_empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&bars->tmem_base)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // the CTA allocates all 512 columns, so the TMEM base address is lane 0 / column 0
    constexpr uint32_t tmem = 0;

    if (warp < 8) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(PAB_FA_SOFTMAX_REGS));
        // ================================================= softmax of tile t
        const int t = warp >> 2;
        const int wl = warp & 3;
        const int row = wl * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wl * 32) << 16;
        const uint32_t s_tmem = tmem + lane_off + 128 * t;
        const uint32_t o_tmem = tmem + lane_off + 256 + 128 * t;
        const int tail = p.n_k - (n_kv - 1) * kKv;  // live keys of the last KV tile
        int it_n = 0;
        for (int c = 0; c < my_items; ++c) {
            const Item it = decode((int)blockIdx.x + c * (int)gridDim.x);
            if (t == 1 && !it.two) continue;
            float m_run = -INFINITY, l_run = 0.f;
            for (int j = 0; j < n_kv; ++j, ++it_n) {
                const bool trc = (wl == 0 && lane == 0);
                FA_TRACE(trc, it_n, t, 0);
                mbar_wait(&bars->s_full[t], it_n & 1);
                tc_fence_after();
                FA_TRACE(trc, it_n, t, 1);
                float s[128];
                load_row128(s_tmem, s);
                FA_TRACE(trc, it_n, t, 2);
#ifdef PAB_FA_DIAG_NOSOFTMAX  // timing diagnostic only: MMA/TMA pipeline without softmax math
                if (s[0] == 12345.f) l_run += 1.f;
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->p_full[t]);
                continue;
#endif
                const bool masked = (j == n_kv - 1) && (tail < kKv);
                if (masked) {
#pragma unroll
                    for (int cc = 0; cc < 128; ++cc) s[cc] = (cc < tail) ? s[cc] : -INFINITY;
                }
                // row max of the raw scores (scale > 0 commutes with max)
                float m4[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    float m = fmaxf(s[32 * g], s[32 * g + 1]);
#pragma unroll
                    for (int cc = 2; cc < 32; cc += 2) m = max3(m, s[32 * g + cc], s[32 * g + cc + 1]);
                    m4[g] = m;
                }
                const float m_tile = max3(fmaxf(m4[0], m4[1]), m4[2], m4[3]) * p.scale_log2;
                const bool need = m_tile > m_run + 8.0f;
                if (__any_sync(0xffffffffu, need)) {
                    const float m_new = need ? m_tile : m_run;
                    if (j > 0) {
                        // O holds sum_{j' < j}: complete, since S(j) was issued after PV(j-1)
                        const float alpha = fast_exp2(m_run - m_new);
                        l_run *= alpha;
#pragma unroll 1
                        for (int cc = 0; cc < G::kDhPad / 16; ++cc) {
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
                FA_TRACE(trc, it_n, t, 3);
                const float neg_m = -m_run;
                l_run += masked ? exp_store_row<true>(s, p.scale_log2, neg_m, s_tmem, tail)
                                : exp_store_row<false>(s, p.scale_log2, neg_m, s_tmem, kKv);
                FA_TRACE(trc, it_n, t, 4);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->p_full[t]);
                FA_TRACE(trc, it_n, t, 5);
            }
            // row sums for the epilogue warps (same TMEM lane quarter)
            l_buf[t * kRows + row] = l_run;
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->l_full[t]);
        }
    } else if (warp < 12) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PAB_FA_OTHER_REGS));
        // ================================================= epilogue (both tiles)
        const int wl = warp & 3;
        const int row = wl * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wl * 32) << 16;
        int ic[2] = {0, 0};
        for (int c = 0; c < my_items; ++c) {
            const Item it = decode((int)blockIdx.x + c * (int)gridDim.x);
            for (int t = 0; t < 2; ++t) {
                if (t == 1 && !it.two) break;
                const int par = ic[t] & 1;
                mbar_wait(&bars->l_full[t], par);
                mbar_wait(&bars->o_full[t], par);
                tc_fence_after();
                ++ic[t];
                const float l = l_buf[t * kRows + row];
                const float inv = (l > 0.f) ? 1.0f / l : 0.f;
                const int i = (it.tile0 + t) * kRows + row;
                const bool store = i < p.n_q;
                __nv_bfloat16* dst = p.o + (int64_t)it.a_idx * p.o_sa + (int64_t)it.b_idx * p.o_sb +
                                     (int64_t)i * p.o_si + (int64_t)it.h * p.dh;
                const uint32_t o_tmem = tmem + lane_off + 256 + 128 * t;
#pragma unroll
                for (int cc = 0; cc < G::kDhPad / 16; ++cc) {
                    float o[16];
                    PAB_TMEM_LD16(o_tmem + 16 * cc, o);
                    tmem_wait_ld();
                    if (store) {
#pragma unroll
                        for (int e = 0; e < 16; e += 8) {
                            if (16 * cc + e < p.dh) {
                                uint32_t w[4];
#pragma unroll
                                for (int q = 0; q < 4; ++q) w[q] = pack_bf16(o[e + 2 * q] * inv, o[e + 2 * q + 1] * inv);
                                *reinterpret_cast<uint4*>(dst + 16 * cc + e) = make_uint4(w[0], w[1], w[2], w[3]);
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->o_free[t]);
            }
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PAB_FA_OTHER_REGS));
        if (warp == kTmaWarp) {
            // ===================================================== TMA producer
            if (lane == 0) {
                int g = 0;  // K/V tiles loaded so far
                for (int c = 0; c < my_items; ++c) {
                    const Item it = decode((int)blockIdx.x + c * (int)gridDim.x);
                    const int qb = c & 1;
                    if (c >= 2) mbar_wait(&bars->q_empty[qb], ((c >> 1) - 1) & 1);
                    mbar_expect_tx(&bars->q_full[qb], (it.two ? 2u : 1u) * tile_bytes);
                    for (int t = 0; t < (it.two ? 2 : 1); ++t) {
                        uint8_t* dst = smem + G::kQ0 + (2 * qb + t) * G::kTileBytes;
                        const int i0 = (it.tile0 + t) * kRows;
                        for (int blk = 0; blk < N128; ++blk)
                            tma_load_5d(dst + blk * 16384, &q128, &bars->q_full[qb], 64 * blk, it.h, i0, it.b_idx,
                                        it.a_idx);
                        for (int blk = 0; blk < N32; ++blk)
                            tma_load_5d(dst + N128 * 16384 + blk * 4096, &q32, &bars->q_full[qb],
                                        64 * N128 + 16 * blk, it.h, i0, it.b_idx, it.a_idx);
                    }
                    for (int j = 0; j < n_kv; ++j, ++g) {
                        const int st = g % 3;
                        if (g >= 3) mbar_wait(&bars->k_empty[st], ((g / 3) - 1) & 1);
                        uint8_t* kd = smem + G::kK0 + st * G::kTileBytes;
                        mbar_expect_tx(&bars->k_full[st], tile_bytes);
                        for (int blk = 0; blk < N128; ++blk)
                            tma_load_5d(kd + blk * 16384, &k128, &bars->k_full[st], 64 * blk, it.h, j * kKv, it.b_idx,
                                        it.a_idx);
                        for (int blk = 0; blk < N32; ++blk)
                            tma_load_5d(kd + N128 * 16384 + blk * 4096, &k32, &bars->k_full[st], 64 * N128 + 16 * blk,
                                        it.h, j * kKv, it.b_idx, it.a_idx);
                        // V as 16-column SW32 atoms ([atom][row][32 B]): one MN-major descriptor
                        // spans the whole padded head dim (N = kDhPad)
                        if (g >= 3) mbar_wait(&bars->v_empty[st], ((g / 3) - 1) & 1);
                        uint8_t* vd = smem + G::kV0 + st * G::kTileBytes;
                        mbar_expect_tx(&bars->v_full[st], tile_bytes);
                        for (int blk = 0; blk < G::kDhPad / 16; ++blk)
                            tma_load_5d(vd + blk * 4096, &v32, &bars->v_full[st], 16 * blk, it.h, j * kKv, it.b_idx,
                                        it.a_idx);
                    }
                }
            }
        } else if (warp == kMmaWarp && lane == 0) {
            // ======================================== MMA issuer: one thread issues every tcgen05.mma
            constexpr uint32_t idS128 = idesc_bf16(128, 128, 0);
            constexpr uint32_t idO = idesc_bf16(128, G::kDhPad, 1);
            // descriptor words: lo = (addr >> 4) | (LBO >> 4) << 16, hi = (SBO >> 4) | version | layout
            const uint32_t q_lo = smem_u32(smem + G::kQ0) >> 4, k_lo = smem_u32(smem + G::kK0) >> 4;
            const uint32_t v_lo = smem_u32(smem + G::kV0) >> 4;
            // (smem_desc bit layout: SBO >> 4 at [32, 46), version 1 at bit 46, layout at [61, 64))
            constexpr uint32_t kHi128 = (1024u >> 4) | (1u << 14) | (kLayoutSW128 << 29);
            constexpr uint32_t kHi32 = (256u >> 4) | (1u << 14) | (kLayoutSW32 << 29);
            constexpr uint32_t kLbo16 = (16u >> 4) << 16;
            // V: MN-major SW32, 16-column atoms 4096 B apart (LBO), 8-row groups 256 B apart (SBO)
            constexpr uint32_t kLboV = (4096u >> 4) << 16;
            auto cols_of = [&](int j) {
                const int n = min(kKv, p.n_k - j * kKv);
                return (n + 15) & ~15;
            };
            // S_t = Q_t K^T (K-major operands; ncols = key columns rounded up to 16)
            auto issue_s = [&](int t, int qslot, int kst, int ncols) {
                const uint32_t qa = q_lo + ((qslot * G::kTileBytes) >> 4), ka = k_lo + ((kst * G::kTileBytes) >> 4);
                const uint32_t idS = (idS128 & ~(0x3Fu << 17)) | ((uint32_t)(ncols >> 3) << 17);
                const uint32_t d_s = tmem + 128 * t;
#pragma unroll
                for (int blk = 0; blk < N128; ++blk)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t o = (blk * 16384 + 32 * k) >> 4;
                        mma_ss1(d_s, (qa + o) | kLbo16, kHi128, (ka + o) | kLbo16, kHi128, idS, (blk | k) != 0);
                    }
#pragma unroll
                for (int blk = 0; blk < N32; ++blk) {
                    const uint32_t o = (N128 * 16384 + blk * 4096) >> 4;
                    mma_ss1(d_s, (qa + o) | kLbo16, kHi32, (ka + o) | kLbo16, kHi32, idS, (N128 | blk) != 0);
                }
            };
            // O_t += P_t V: ncols / 16 K-steps of 16 keys; A = P_t from TMEM (8 columns per step)
            auto issue_pv = [&](int t, int vst, uint32_t accumulate, int ncols) {
                const uint32_t va = v_lo + ((vst * G::kTileBytes) >> 4);
                const uint32_t d_o = tmem + 256 + 128 * t, a_p = tmem + 128 * t;
                if (ncols == kKv) {
#pragma unroll
                    for (int k = 0; k < kKv / 16; ++k)
                        mma_ts1(d_o, a_p + 8 * k, (va + ((512 * k) >> 4)) | kLboV, kHi32, idO, accumulate | (k > 0));
                } else {
                    for (int k = 0; 16 * k < ncols; ++k)
                        mma_ts1(d_o, a_p + 8 * k, (va + ((512 * k) >> 4)) | kLboV, kHi32, idO, accumulate | (k > 0));
                }
            };
            int g = 0;                // K/V tiles consumed
            int it_n[2] = {0, 0};     // softmax iterations per tile
            int ic[2] = {0, 0};       // items per tile
            for (int c = 0; c < my_items; ++c) {
                const Item it = decode((int)blockIdx.x + c * (int)gridDim.x);
                const int qb = c & 1;
                const int nt = it.two ? 2 : 1;
                mbar_wait(&bars->q_full[qb], (c >> 1) & 1);
                mbar_wait(&bars->k_full[g % 3], (g / 3) & 1);
                tc_fence_after();
                for (int t = 0; t < nt; ++t) {
                    issue_s(t, 2 * qb + t, g % 3, cols_of(0));
                    commit1(&bars->s_full[t]);
                }
                commit1(&bars->k_empty[g % 3]);
                if (n_kv == 1) commit1(&bars->q_empty[qb]);
                for (int j = 0; j < n_kv; ++j) {
                    const int gv = g + j;
                    mbar_wait(&bars->v_full[gv % 3], (gv / 3) & 1);
                    if (j + 1 < n_kv) mbar_wait(&bars->k_full[(gv + 1) % 3], ((gv + 1) / 3) & 1);
                    for (int t = 0; t < nt; ++t) {
                        FA_TRACE(true, it_n[t], t, 10);
                        mbar_wait(&bars->p_full[t], it_n[t] & 1);
                        FA_TRACE(true, it_n[t], t, 8);
                        if (j == 0 && ic[t] > 0) mbar_wait(&bars->o_free[t], (ic[t] - 1) & 1);
                        tc_fence_after();
                        issue_pv(t, gv % 3, j > 0, cols_of(j));
                        if (j + 1 < n_kv) {
                            issue_s(t, 2 * qb + t, (gv + 1) % 3, cols_of(j + 1));
                            commit1(&bars->s_full[t]);
                        } else {
                            commit1(&bars->o_full[t]);
                        }
                        FA_TRACE(true, it_n[t], t, 9);
                        ++it_n[t];
                    }
                    commit1(&bars->v_empty[gv % 3]);
                    if (j + 1 < n_kv) {
                        commit1(&bars->k_empty[(gv + 1) % 3]);
                        if (j + 2 == n_kv) commit1(&bars->q_empty[qb]);
                    }
                }
                for (int t = 0; t < nt; ++t) ++ic[t];
                g += n_kv;
            }
        }
    }
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

template <int N128, int N32>
int launch(const pab_attn_args* a, cudaStream_t st) {
    using G = Geometry<N128, N32>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(attn_fa_kernel<N128, N32>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::kSmem) !=
            cudaSuccess)
            return launch_status("attn_fa smem attribute");
        attr_set = true;
    }
    CUtensorMap mq128, mq32, mk128, mk32, mv32;
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
                  CU_TENSOR_MAP_SWIZZLE_32B))
        return PAB_ERR_CUDA;
    Params p;
    p.n_q = a->n_q;
    p.n_k = a->n_k;
    p.n_b = a->n_b;
    p.heads = a->heads;
    p.dh = a->dh;
    p.scale_log2 = a->scale * 1.4426950408889634f;
    p.o = reinterpret_cast<__nv_bfloat16*>(a->o);
    p.o_sa = a->o_sa;
    p.o_sb = a->o_sb;
    p.o_si = a->o_si;
    p.trace = tc::g_trace;
    p.row_tiles = (a->n_q + kRows - 1) / kRows;
    p.n_kv = (a->n_k + kKv - 1) / kKv;
    p.n_pairs = (p.row_tiles + 1) / 2;
    const int64_t items = (int64_t)p.n_pairs * a->heads * a->n_a * a->n_b;
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
    attn_fa_kernel<N128, N32><<<grid, kThreads, G::kSmem, st>>>(mq128, mq32, mk128, mk32, mv32, p);
    return launch_status("attn_fa");
}

}  // namespace fa

// non-packed attention (spatial, cross) with dh <= 80 and a multiple of 8
int attn_fa_launch(const pab_attn_args* a, cudaStream_t st) {
    const int n128 = a->dh / 64;
    const int n32 = (a->dh - 64 * n128 + 15) / 16;
#define PAB_FA(A, B) \
    if (n128 == A && n32 == B) return fa::launch<A, B>(a, st)
    PAB_FA(0, 1);
    PAB_FA(0, 2);
    PAB_FA(0, 3);
    PAB_FA(0, 4);
    PAB_FA(1, 0);
    PAB_FA(1, 1);
#undef PAB_FA
    return PAB_ERR_UNSUPPORTED;
}

}  // namespace pab

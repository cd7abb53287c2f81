// Row-per-thread tcgen05 flash attention for sm_100a: the production kernel for
// the spatial (K1) and cross (K3) attention sites.
//
// reference op: numerics.scaled_dot_attention (pkg/src/pab_engine/numerics.py:133-151)
// as used by _axis_attention_compute(temporal_axis=False) and _cross_attention_compute
// (pkg/src/pab_engine/model.py:346-359, 376-385):
//   logits = q k^T * (1/sqrt(dh)); p = softmax(logits) (max-shifted); out = p v
//
// CTA (one persistent CTA per SM; a work item is two 128-row query tiles of one
// (problem, head) that share every K/V tile).  With PAB_FA_SPLIT = S (default 1):
//   warps [0, 4S)     softmax + epilogue of query tile 0: warp w owns TMEM lane quarter
//                     w % 4 (one thread per query row) and column part (w >> 2) % S of the
//                     112 keys (S = 2: the two warps of a row exchange maxima through smem)
//   warps [4S, 8S)    the same for query tile 1
//   warp  8S          MMA issuer (one elected lane issues the tcgen05.mma groups; owns TMEM)
//   warp  8S + 1      TMA producer (lane 0)
//   warp  8S + 2      fixer: 1.0 into the first padded V column (row sums) and, for
//                     dh % 16 != 0, the pad-column key mask (Q[:, dh] = 1, K[pad rows, dh] =
//                     -1e30, so partial last KV tiles need no masking in the softmax)
//
// TMEM (512 columns), KV tiles of 112 keys so that S, P and O of both tiles fit side by
// side (no aliasing):  S_t [112t, 112t + 112),  O_t [224 + OC t, ...),  P_t [384 + 64t, +56).
// Because P does not overwrite S, the MMA warp issues S(j+1) = Q K_{j+1}^T as soon as
// the softmax has pulled S(j) into registers, i.e. while it is still exponentiating,
// and PV(j) when P(j) is stored: the tensor pipe works in the shadow of the softmax.
//
// Row sums: the V fixer stores 1.0 into V column dh (zero padding otherwise), so the
// PV MMA accumulates sum_k P[r, k] into O[r, dh] -- the softmax does no row-sum
// arithmetic and the normaliser is the sum of exactly the bf16 P values multiplied
// into O.  Online softmax: the running max is only raised (and O rescaled in TMEM)
// when a tile's max exceeds it by more than 2^8, so P <= 256 and the rescale is rare.
// exp2 runs on MUFU for most columns and on the FMA pipe (degree-3 polynomial on f32x2
// pairs) for one pair in PAB_FA_POLY_DIV.
//
// Scheduling: the warps of tile 0 and tile 1 that share an SM sub-partition pass a token
// (PAB_FA_LAG = 2) so their exp sections alternate while the other tile loads S, takes
// its row max and stores P; the MMA groups still interleave both tiles' accumulators.
// Epilogue: each item's O rows are staged densely in smem and leave through ONE TMA
// tensor store per tile (an asynchronous bulk write instead of a GPU-wide burst of row
// stores).  Measurements behind each choice: DESIGN.md section 8.1.
#include "tc_ptx.cuh"

namespace pab {
namespace tc {
extern long long* g_trace;  // attn_tc.cu: pab_attn_debug_trace
}
namespace fa {

using namespace pab::tc;

#ifndef PAB_FA_SPLIT
#define PAB_FA_SPLIT 1  // softmax warps per (tile, TMEM lane quarter): each owns kKv / SPLIT columns
#endif
constexpr int kSplit = PAB_FA_SPLIT;
constexpr int kSoftmaxWarps = 8 * kSplit;

#ifndef PAB_FA_EPI_WARPS
#define PAB_FA_EPI_WARPS 1  // 1: O epilogue on 4 dedicated warps (registers rebalanced with setmaxnreg)
#endif
// Dedicated epilogue warps (round 2): warps 12..15 (TMEM lane quarters 0..3) drain each
// finished item's O while the softmax warps already run the next item (the epilogue
// was 18% of cross and 7% of spatial time on the softmax warps' critical path,
// measured with PAB_FA_DIAG_NOEPI).  512 threads: the softmax warpgroups raise their
// register budget to kRegSoftmax, the MMA / TMA / fixer / epilogue warpgroups lower theirs.
constexpr bool kEpiWarps = PAB_FA_EPI_WARPS != 0 && kSplit == 1;
constexpr int kEpiWarp0 = 12;
constexpr int kThreads = kEpiWarps ? 512 : 32 * (kSoftmaxWarps + 3);
#ifndef PAB_FA_REG_SOFTMAX
#define PAB_FA_REG_SOFTMAX 176
#endif
constexpr int kRegSoftmax = PAB_FA_REG_SOFTMAX, kRegAux = (65536 / 256 - PAB_FA_REG_SOFTMAX) / 8 * 8;
static_assert(!kEpiWarps || 256 * kRegSoftmax + 256 * kRegAux <= 65536, "register file");
constexpr int kRows = 128;   // query rows per tile == TMEM lanes
constexpr int kKv = 112;     // keys per KV tile
constexpr int kHalf = kKv / kSplit;  // score columns per softmax thread
constexpr int kMmaWarp = kSoftmaxWarps;
constexpr int kTmaWarp = kSoftmaxWarps + 1;
constexpr int kFixWarp = kSoftmaxWarps + 2;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kSCol = 0, kPCol = 384;

#ifndef PAB_FA_BULK_EPI
#define PAB_FA_BULK_EPI 1   // O rows leave through smem staging + cp.async.bulk (0: direct stores)
#endif

#ifndef PAB_FA_LAG
#define PAB_FA_LAG 2  // 1: tile 1's row max waits for tile 0's (lag = one max phase); 2: its exp waits for tile 0's exp
#endif

#ifndef PAB_FA_SINGLES_LAST
#define PAB_FA_SINGLES_LAST 0  // 1: single-tile items (odd tile count) scheduled last (better tail balance, but
                               // their K/V is re-read from DRAM: 576 vs 345 MB per C3 launch; 517 vs 522 us)
#endif

#ifndef PAB_FA_PV_SPLIT
#define PAB_FA_PV_SPLIT 1  // 1: P.V issued per query tile (own p_full / o_done), 0: one group for both
#endif
constexpr bool kPvSplit = PAB_FA_PV_SPLIT != 0;
static_assert(!kEpiWarps || kPvSplit, "the dedicated epilogue needs per-tile o_done / o_final");

#ifndef PAB_FA_POLY_DIV
#define PAB_FA_POLY_DIV 3   // one column pair in PAB_FA_POLY_DIV on the FMA pipe (0: MUFU only)
#endif

// Division by a kernel-invariant divisor as multiply-high + shift (valid for 0 <= n < 2^31):
// the item decode runs on the softmax and MMA warps' critical path at every item boundary,
// where hardware-less integer division (MUFU.RCP + fix-up chains) cost ~300 clk per item.
struct FastDiv {
    uint32_t d, m, s;
};
static inline FastDiv make_fastdiv(uint32_t d) {
    if (d == 0) d = 1;  // empty problems: never used
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    return FastDiv{d, (uint32_t)(((1ull << 32) * ((1ull << s) - d)) / d + 1), s};
}
__device__ __forceinline__ int fdiv(int n, const FastDiv& f) {
    return (int)((__umulhi((uint32_t)n, f.m) + (uint32_t)n) >> f.s);
}

struct Params {
    int n_q, n_k, n_b, heads, dh;
    FastDiv f_heads, f_full, f_b;  // heads, pairs with two tiles (n_full), n_b
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
#define FA_TRACE(cond, itn, t, ev)                                         \
    do {                                                                   \
        if (p.trace != nullptr && (cond) && blockIdx.x == 0 && (itn) < 64) \
            p.trace[((itn) * 2 + (t)) * 16 + (ev)] = clock64();            \
    } while (0)
#endif

// N128 x 64 + N32 x 16 = dh rounded up to 16 (the QK^T reduction); NV = V atoms of 16
// columns = dh / 16 + 1 (always one padded column for the row sum)
template <int N128, int N32, int NV>
struct Geometry {
    static constexpr int kDhK = 64 * N128 + 16 * N32;
    static constexpr int kOCols = 16 * NV;
    static constexpr int kSlot = 20480;    // one 128-row Q slot, any dh <= 80
    // 112-row K/V slots: K = SW128 block (112 x 128 B) then SW32 blocks (112 x 32 B each);
    // V = NV SW32 atoms of 16 columns, 112 x 32 B each
    static constexpr int kK128 = kKv * 128, kK32 = kKv * 32, kVAtom = kKv * 32;
    static constexpr int kSlotKV = 18432;
    static constexpr int kQ0 = 0;        // 2 item buffers x 2 tiles
    static constexpr int kK0 = 4 * kSlot;                  // 3-stage K ring
    static constexpr int kV0 = kK0 + 3 * kSlotKV;          // 3-stage V ring
    static constexpr int kX0 = kV0 + 3 * kSlotKV;          // row-max exchange [2][2][2][128] f32 (split 2)
    static constexpr int kStageRow = 144;                  // epilogue staging: max bytes of one bf16 O row
    static constexpr int kX0Bytes = (2 * kRows * kStageRow > 8 * kRows * 4) ? 2 * kRows * kStageRow : 8 * kRows * 4;
    static constexpr int kBar = kX0 + kX0Bytes;
    static constexpr int kSmem = kBar + 512 + 1024;  // + barriers + alignment slack
    static constexpr uint32_t kOCol0 = 224, kOStride = kOCols;
    static_assert(N128 * 16384 + N32 * 4096 <= kSlot, "Q slot");
    static_assert(N128 * kK128 + N32 * kK32 <= kSlotKV && NV * kVAtom <= kSlotKV && kSlotKV % 1024 == 0, "K/V slot");
    static_assert(kOCol0 + 2 * kOCols <= kPCol, "O tiles overlap P in TMEM");
    static_assert(kSmem <= 232448, "attention tiles exceed the 227 KB shared memory of one CTA");
};

struct Bars {
    uint64_t q_full[2], q_empty[2], k_full[3], k_empty[3], v_full[3], v_ready[3], v_empty[3];
    uint64_t q_ready[2], k_ready[3];  // Q / K tiles after the fixer warp's pad-column patch
    uint64_t s_full, s_free;         // shared by the two query tiles (S is one interleaved MMA group)
    uint64_t p_full[2], o_done[2];   // per tile (PAB_FA_PV_SPLIT) or index 0 for both
    uint64_t o_final[2], o_free[2];  // dedicated epilogue: item's last P.V done / O read out of TMEM
};

// single-thread tcgen05.mma issue (lane 0 of the MMA warp): descriptors are passed as
// (lo, hi) words so advancing a K step is one 32-bit add on the lo word
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

// Whole MMA groups in one asm statement (one elect for the group, descriptor arithmetic
// on the 64-bit descriptors inside the asm): the per-MMA issue cost of compiler-generated
// code (R2UR moves + an ELECT loop per instruction, ~100 cycles each) otherwise exceeds
// the tensor-pipe time of the MMA itself.  Geometry of dh = 72: 4 SW128 K-steps + 1 SW32.
// S_t = Q_t K^T for both tiles, K-steps interleaved (tile 1 only when `two`).
__device__ __forceinline__ void mma_group_s_72(uint32_t d0, uint32_t d1, uint64_t q128, uint64_t k128, uint64_t q32,
                                              uint64_t k32, uint32_t idesc, uint32_t two, uint32_t qstride) {
    asm volatile(
        "{\n\t.reg .pred e, e2, pf, pt;\n\t.reg .b64 qa, ka, qs;\n\t"
        "setp.ne.b32 pt, %8, 0;\n\t"   // pt = two (reassigned to true below)
        "setp.ne.b32 pf, %7, %7;\n\t"  // false
        "elect.sync _|e, 0xffffffff;\n\t"
        "and.pred e2, e, pt;\n\t"
        "setp.eq.b32 pt, %7, %7;\n\t"  // true
        "cvt.u64.u32 qs, %9;\n\t"
        // k = 0 (SW128, +0)
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %6, pf;\n\t"
        "add.s64 qa, %2, qs;\n\t"
        "@e2 tcgen05.mma.cta_group::1.kind::f16 [%1], qa, %3, %6, pf;\n\t"
        // k = 1..3 (SW128, +32 B per step -> +2 in the descriptor)
        "add.s64 qa, %2, 2;\n\tadd.s64 ka, %3, 2;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], qa, ka, %6, pt;\n\t"
        "add.s64 qa, qa, qs;\n\t"
        "@e2 tcgen05.mma.cta_group::1.kind::f16 [%1], qa, ka, %6, pt;\n\t"
        "add.s64 qa, %2, 4;\n\tadd.s64 ka, %3, 4;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], qa, ka, %6, pt;\n\t"
        "add.s64 qa, qa, qs;\n\t"
        "@e2 tcgen05.mma.cta_group::1.kind::f16 [%1], qa, ka, %6, pt;\n\t"
        "add.s64 qa, %2, 6;\n\tadd.s64 ka, %3, 6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], qa, ka, %6, pt;\n\t"
        "add.s64 qa, qa, qs;\n\t"
        "@e2 tcgen05.mma.cta_group::1.kind::f16 [%1], qa, ka, %6, pt;\n\t"
        // k = 4 (SW32 block)
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %5, %6, pt;\n\t"
        "add.s64 qa, %4, qs;\n\t"
        "@e2 tcgen05.mma.cta_group::1.kind::f16 [%1], qa, %5, %6, pt;\n\t}" ::"r"(d0),
        "r"(d1), "l"(q128), "l"(k128), "l"(q32), "l"(k32), "r"(idesc), "r"(0), "r"(two), "r"(qstride)
        : "memory");
}
// O_t += P_t V for both tiles: `steps` (<= 7) K-steps of 16 keys, A = P_t from TMEM
// (+8 columns per step), B = V atoms (+512 B per step -> +32 in the descriptor)
__device__ __forceinline__ void mma_group_pv7(uint32_t o0, uint32_t o1, uint32_t p0, uint32_t p1, uint64_t v,
                                             uint32_t idesc, uint32_t accumulate, uint32_t two, uint32_t steps) {
    asm volatile(
        "{\n\t.reg .pred e, e2, pa, pt, s1, s2, s3, s4, s5, s6;\n\t.reg .b64 vb;\n\t.reg .b32 pa0, pa1;\n\t"
        "setp.ne.b32 pt, %7, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "and.pred e2, e, pt;\n\t"
        "setp.ne.b32 pa, %6, 0;\n\t"
        "setp.eq.b32 pt, %7, %7;\n\t"
        "setp.gt.u32 s1, %8, 1;\n\tsetp.gt.u32 s2, %8, 2;\n\tsetp.gt.u32 s3, %8, 3;\n\t"
        "setp.gt.u32 s4, %8, 4;\n\tsetp.gt.u32 s5, %8, 5;\n\tsetp.gt.u32 s6, %8, 6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %4, %5, pa;\n\t"
        "@e2 tcgen05.mma.cta_group::1.kind::f16 [%1], [%3], %4, %5, pa;\n\t"
#define PAB_PV_STEP(S, VOFF, POFF)                                                                        \
        "add.s64 vb, %4, " #VOFF ";\n\tadd.u32 pa0, %2, " #POFF ";\n\tadd.u32 pa1, %3, " #POFF ";\n\t" \
        "and.pred " #S ", " #S ", e;\n\t"                                                 \
        "@" #S " tcgen05.mma.cta_group::1.kind::f16 [%0], [pa0], vb, %5, pt;\n\t"        \
        "and.pred " #S ", " #S ", e2;\n\t"                                                \
        "@" #S " tcgen05.mma.cta_group::1.kind::f16 [%1], [pa1], vb, %5, pt;\n\t"
        PAB_PV_STEP(s1, 32, 8) PAB_PV_STEP(s2, 64, 16) PAB_PV_STEP(s3, 96, 24) PAB_PV_STEP(s4, 128, 32)
        PAB_PV_STEP(s5, 160, 40) PAB_PV_STEP(s6, 192, 48)
#undef PAB_PV_STEP
        "}" ::"r"(o0), "r"(o1), "r"(p0), "r"(p1), "l"(v), "r"(idesc), "r"(accumulate), "r"(two), "r"(steps)
        : "memory");
}

// wait for two mbarrier phases with both try_waits in flight together (the MMA warp's
// serial latency per iteration is dominated by barrier round trips)
__device__ __forceinline__ void mbar_wait2(uint64_t* a, uint32_t pa, uint64_t* b, uint32_t pb) {
    asm volatile(
        "{\n\t.reg .pred x, y;\n"
        "W2_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 x, [%0], %1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 y, [%2], %3;\n\t"
        "and.pred x, x, y;\n\t"
        "@!x bra W2_%=;\n}" ::"r"(smem_u32(a)),
        "r"(pa), "r"(smem_u32(b)), "r"(pb)
        : "memory");
}

__device__ __forceinline__ float max3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

#define PAB_TMEM_ST4U(taddr, r)                                                                          \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]), \
                 "r"(r[2]), "r"(r[3])                                                                        \
                 : "memory")
#define PAB_TMEM_LD8(taddr, r)                                                                           \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                \
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),     \
                   "=f"(r[7])                                                                             \
                 : "r"(taddr))
#define PAB_TMEM_ST8U(taddr, r)                                                                          \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), \
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])  \
                 : "memory")

// 2^x for a pair of floats on the FMA pipe: x = i + f with i = round(x) via the
// 1.5*2^23 magic constant, 2^f by a degree-3 minimax polynomial on [-0.5, 0.5]
// (max rel err 7.5e-5, far below the bf16 rounding of P), exponent add as an integer.
__device__ __forceinline__ void poly_exp2_x2(float& a, float& b) {
    // clamp at -126: 2^f of the polynomial has biased exponent 126 for f < 0, so adding
    // -127 << 23 would wrap the exponent field to 255 (NaN); -126 gives a denormal ~1e-38
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

// P = exp2(s * scale_log2 - m) for columns [c0, c0 + 2 NPAIRS) -> NPAIRS packed bf16 pairs
template <bool MASKED, int NPAIRS>
__device__ __forceinline__ void exp_pack(const float* s, int c0, unsigned long long sc2, unsigned long long nm2,
                                         int nv, uint32_t* pk) {
#pragma unroll
    for (int q = 0; q < NPAIRS; ++q) {
        const int c = c0 + 2 * q;
        float2 x = f2_unpack(f2_fma(f2_pack(s[c], s[c + 1]), sc2, nm2));
        if (PAB_FA_POLY_DIV > 0 && !MASKED &&
            (q % (PAB_FA_POLY_DIV > 0 ? PAB_FA_POLY_DIV : 1)) == (PAB_FA_POLY_DIV > 0 ? PAB_FA_POLY_DIV : 1) - 1) {
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
        pk[q] = pack_bf16(x.x, x.y);
    }
}

template <int N128, int N32, int NV>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fa_kernel(const __grid_constant__ CUtensorMap q128, const __grid_constant__ CUtensorMap q32,
                   const __grid_constant__ CUtensorMap k128, const __grid_constant__ CUtensorMap k32,
                   const __grid_constant__ CUtensorMap v32, const __grid_constant__ CUtensorMap omap,
                   const Params p) {
    using G = Geometry<N128, N32, NV>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + G::kBar);
    __shared__ uint32_t tmem_base_slot;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // item -> (head, pair, a, b), head fastest: concurrently running CTAs read all heads of
    // the same q/k/v rows (whole qkv rows per DRAM page visit) and share K/V in L2
    struct Item {
        int h, a_idx, b_idx, tile0;
        bool two;  // second query tile exists
    };
    // With an odd tile count the last pair of every (problem, head) has a single query tile
    // and costs ~0.7 of a two-tile item: those items are numbered last, so the tail round of
    // the static CTA assignment holds the cheap ones.
    const int n_full = PAB_FA_SINGLES_LAST ? p.row_tiles / 2 : p.n_pairs;  // pairs with two tiles first
    const int items_full = n_full * p.heads * (p.n_items / (p.n_pairs * p.heads));
    auto decode = [&](int item) {
        Item it;
        int pair, az;
        if (item >= items_full) {  // single-tile items (pair n_full) of every (problem, head)
            const int rest = item - items_full;
            az = fdiv(rest, p.f_heads);
            it.h = rest - az * p.heads;
            pair = n_full;
        } else {
            const int rest = fdiv(item, p.f_heads);
            it.h = item - rest * p.heads;
            az = fdiv(rest, p.f_full);
            pair = rest - az * n_full;
        }
        it.a_idx = fdiv(az, p.f_b);
        it.b_idx = az - it.a_idx * p.n_b;
        it.tile0 = 2 * pair;
        it.two = it.tile0 + 1 < p.row_tiles;
        return it;
    };
    const int my_items = (p.n_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int n_kv = p.n_kv;
    const int n_iters = my_items * n_kv;  // global (item, kv tile) iterations of this CTA
    // Pad-column key mask (dh % 16 != 0, e.g. 72): column dh of the zero-padded head dim is
    // 1.0 in every Q row and -1e30 in the K rows past n_k, so the S MMA itself scores the
    // padded keys of a partial last KV tile at -1e30 (exp -> 0, never the max): that tile
    // runs the unmasked softmax over all 112 columns and full-width MMAs.
    const bool padmask = N32 > 0 && (p.dh & 15) != 0;

    // ---------------------------------------------------------------- setup
    if (warp == kTmaWarp && lane == 0) {
        prefetch_map(&omap);
        prefetch_map(&q128);
        prefetch_map(&k128);
        prefetch_map(&v32);
        if (N32) {
            prefetch_map(&q32);
            prefetch_map(&k32);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars->q_full[s], 1);
            mbar_init(&bars->q_ready[s], 1);
            mbar_init(&bars->q_empty[s], 1);
        }
        for (int s = 0; s < 3; ++s) {
            mbar_init(&bars->k_full[s], 1);
            mbar_init(&bars->k_ready[s], 1);
            mbar_init(&bars->k_empty[s], 1);
            mbar_init(&bars->v_full[s], 1);
            mbar_init(&bars->v_ready[s], 1);
            mbar_init(&bars->v_empty[s], 1);
        }
        mbar_init(&bars->s_full, 1);
        mbar_init(&bars->s_free, kSoftmaxWarps);  // one arrival per softmax warp
        for (int t = 0; t < 2; ++t) {
            mbar_init(&bars->p_full[t], kPvSplit ? kSoftmaxWarps / 2 : kSoftmaxWarps);
            mbar_init(&bars->o_done[t], 1);
            mbar_init(&bars->o_final[t], 1);
            mbar_init(&bars->o_free[t], 4);  // one arrival per epilogue warp
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
    // the CTA allocates all 512 columns, so the TMEM base address is lane 0 / column 0
    constexpr uint32_t tmem = 0;
    if (kEpiWarps) {
        if (warp < kSoftmaxWarps) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
        else asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegAux));
    }

    if (warp < kSoftmaxWarps) {
        // ========================================= softmax + epilogue of query tile t
        // warp = 8 t + 4 h + quarter: TMEM lane quarter = warp % 4 (the tcgen05.ld/st lane
        // restriction), column half h of the 112-key S tile
        const int t = warp / (4 * kSplit);
        const int tb = kPvSplit ? t : 0;  // this tile's p_full / o_done barrier
        const int hc = (warp >> 2) % kSplit;
        const int wl = warp & 3;
        const int row = wl * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wl * 32) << 16;
        const uint32_t s_tmem = tmem + lane_off + kSCol + kKv * t + kHalf * hc;
        const uint32_t o_tmem = tmem + lane_off + G::kOCol0 + G::kOStride * t;
        const uint32_t p_tmem = tmem + lane_off + kPCol + 64 * t + (kHalf / 2) * hc;
        const int tail = p.n_k - (n_kv - 1) * kKv - kHalf * hc;  // live keys of the last KV tile in this half
        const bool trc = (wl == 0 && lane == 0 && hc == 0);
        // O chunks (16 columns) this half rescales / stores
        constexpr int kOHalf = (kSplit == 1) ? NV : (NV + 1) / 2;
        const int oc_lo = hc ? kOHalf : 0, oc_hi = hc ? NV : kOHalf;
        // row max exchange with the other column half: [parity][tile][half][row]
        float* xch = reinterpret_cast<float*>(smem + G::kX0);
        const uint32_t xbar = 1 + 4 * t + wl;  // named barrier of the two warps sharing these rows
        // O of the previous item of this tile -> normalised bf16 rows (its last P.V done)
        auto epilogue = [&](const Item& it) {
#ifdef PAB_FA_DIAG_NOEPI  // timing diagnostic only: no epilogue at all (O never leaves TMEM)
            return;
#endif
            float o[16];
            PAB_TMEM_LD16(o_tmem + 16 * (p.dh / 16), o);  // row sum sits in column dh
            tmem_wait_ld();
            float l = o[0];
#pragma unroll
            for (int e = 1; e < 16; ++e) l = (e == p.dh % 16) ? o[e] : l;
            const float inv = (l > 0.f) ? 1.0f / l : 0.f;
            const int i = (it.tile0 + t) * kRows + row;
            const bool store = i < p.n_q;
            __nv_bfloat16* dst = p.o + (int64_t)it.a_idx * p.o_sa + (int64_t)it.b_idx * p.o_sb + (int64_t)i * p.o_si +
                                 (int64_t)it.h * p.dh;
            if (kSplit == 1 && PAB_FA_BULK_EPI) {
                // Every CTA reaches its epilogue at about the same time, so plain row stores form a
                // GPU-wide write burst the softmax warps stall on (measured: not writing O at all
                // makes cross attention 14% faster).  Stage the tile's 128 rows in smem and let
                // one thread hand them to the TMA engine as ONE asynchronous tensor store (rows
                // past n_q are clipped by the tensor map); the warps go on at once.
                uint8_t* stg_tile = smem + G::kX0 + t * kRows * G::kStageRow;
                uint8_t* stg = stg_tile + row * (2 * p.dh);  // dense rows: the TMA box layout
                const bool issuer = (wl == 0 && lane == 0);
                if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // last store read stg
                asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");
                for (int cc = 0; 16 * cc < p.dh; ++cc) {
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
                fence_async_smem();  // generic-proxy smem writes -> visible to the TMA (async proxy)
                asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");
#ifndef PAB_FA_DIAG_EPI_NOSTORE
                if (issuer)
                    asm volatile(
                        "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n\t"
                        "cp.async.bulk.commit_group;" ::"l"(reinterpret_cast<uint64_t>(&omap)),
                        "r"(smem_u32(stg_tile)), "r"(0), "r"(it.h), "r"((it.tile0 + t) * kRows), "r"(it.b_idx),
                        "r"(it.a_idx)
                        : "memory");
#endif
                return;
            }
            for (int cc = oc_lo; cc < oc_hi; ++cc) {
                if (16 * cc >= p.dh) break;
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
        };
        Item prev;
        bool have_prev = false;
        int it_n = 0;  // iterations of this tile (tile 1 skips single-tile items)
        // the softmax warps only need each item's `two` flag: decoded 32 items at a time (one
        // item per lane, ballot), so an item boundary costs them a bit test instead of a decode
        uint32_t two_bits = 0;
        for (int c = 0; c < my_items; ++c) {
            FA_TRACE(trc, it_n, t, 6);
            if ((c & 31) == 0) {
                const int ci = c + lane;
                const bool tw = ci < my_items && decode((int)blockIdx.x + ci * (int)gridDim.x).two;
                two_bits = __ballot_sync(0xffffffffu, tw);
            }
            Item it{};
            if (!kEpiWarps) it = decode((int)blockIdx.x + c * (int)gridDim.x);  // for epilogue(prev)
            const bool active = (t == 0) || ((two_bits >> (c & 31)) & 1u);
            float m_run = -INFINITY;
            FA_TRACE(trc, it_n, t, 7);
            for (int j = 0; j < n_kv; ++j, ++it_n) {
                FA_TRACE(trc, it_n, t, 0);
                mbar_wait(&bars->s_full, it_n & 1);
                tc_fence_after();
                FA_TRACE(trc, it_n, t, 1);
                float s[kHalf];
#ifndef PAB_FA_DIAG_BARRIERS_ONLY  // timing diagnostic only: the barrier protocol without softmax work
                if (!active)
#endif
                {
                    // second tile absent: arrive on the pair's barriers with the same waits as an
                    // active tile (o_done(gi - 1) before p_full(gi)), so these arrivals can never
                    // run a phase ahead and complete a phase on their own
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->s_free);
                    if (PAB_FA_LAG && kSplit == 1) asm volatile("bar.sync %0, 64;" ::"r"(3 + wl + 4 * (it_n & 1)) : "memory");
                    if (it_n > 0) mbar_wait(&bars->o_done[tb], (it_n - 1) & 1);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->p_full[tb]);
                    continue;
                }
                if (kSplit == 1) {
                    PAB_TMEM_LD32(s_tmem, s);
                    PAB_TMEM_LD32(s_tmem + 32, (s + 32));
                    PAB_TMEM_LD32(s_tmem + 64, (s + 64));
                    PAB_TMEM_LD16(s_tmem + 96, (s + 96));
                } else {
                    PAB_TMEM_LD32(s_tmem, s);
                    PAB_TMEM_LD16(s_tmem + 32, (s + 32));
                    PAB_TMEM_LD8(s_tmem + 48, (s + 48));
                }
                tmem_wait_ld();
                // S is in registers: the MMA warp may overwrite it with the next S
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->s_free);
                FA_TRACE(trc, it_n, t, 2);
                const bool masked = !padmask && (j == n_kv - 1) && (tail < kHalf);
                // lag token (warps wl of tile 0 and tile 1 share an SM sub-partition): tile 1 starts
                // its ALU-bound row max only when tile 0's is done, so it overlaps tile 0's MUFU-bound
                // exp.  Two named barriers alternate by iteration parity: tile 0 can reach iteration
                // j + 1's token before tile 1 consumed j's, never j + 2's (S(j + 2) is issued only
                // after the shared s_free(j + 1), i.e. after tile 1 loaded S(j + 1), which follows
                // its token of iteration j).
                // Barrier ids 3..10 (1 and 2 are the epilogue's per-tile barriers).
                if (PAB_FA_LAG == 1 && kSplit == 1 && t == 1) asm volatile("bar.sync %0, 64;" ::"r"(3 + wl + 4 * (it_n & 1)) : "memory");
                if (masked) {
#pragma unroll
                    for (int cc = 0; cc < kHalf; ++cc) s[cc] = (cc < tail) ? s[cc] : -INFINITY;
                }
                // row max of the raw scores (scale > 0 commutes with max), then with the other half
                constexpr int kG = kHalf / 4;  // 4 independent FMNMX3 chains
                float m4[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    float m = s[kG * g];
#pragma unroll
                    for (int cc = 1; cc + 1 < kG; cc += 2) m = max3(m, s[kG * g + cc], s[kG * g + cc + 1]);
                    m4[g] = (kG % 2 == 0) ? fmaxf(m, s[kG * g + kG - 1]) : m;
                }
                float mx = max3(fmaxf(m4[0], m4[1]), m4[2], m4[3]);
#ifdef PAB_FA_DIAG_NOMAX  // timing diagnostic only: row max of the first tile reused (wrong results)
                if (j > 0) mx = s[0];
#endif
                if (kSplit > 1) {
                    float* xs = xch + ((it_n & 1) * 2 + t) * 2 * kRows;
                    xs[hc * kRows + row] = mx;
                    asm volatile("bar.sync %0, %1;" ::"r"(xbar), "r"(64) : "memory");
                    mx = fmaxf(mx, xs[(1 - hc) * kRows + row]);
                }
                if (PAB_FA_LAG == 1 && kSplit == 1 && t == 0) asm volatile("bar.arrive %0, 64;" ::"r"(3 + wl + 4 * (it_n & 1)) : "memory");
                const float m_tile = mx * p.scale_log2;
                // both halves hold identical (m_tile, m_run) per row and take the same decisions
                const bool need = m_tile > m_run + 8.0f;
                // the previous P.V of this tile must be complete before O is rescaled or P overwritten
                bool waited = false;
                if (__any_sync(0xffffffffu, need)) {
                    const float m_new = need ? m_tile : m_run;
                    if (j > 0) {
                        mbar_wait(&bars->o_done[tb], (it_n - 1) & 1);
                        tc_fence_after();
                        waited = true;
                        const float alpha = fast_exp2(m_run - m_new);
#pragma unroll 1
                        for (int cc = oc_lo; cc < oc_hi; ++cc) {
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
                const unsigned long long sc2 = f2_pack(p.scale_log2, p.scale_log2), nm2 = f2_pack(neg_m, neg_m);
                uint32_t pk[kHalf / 2];
                if (PAB_FA_LAG == 2 && kSplit == 1 && t == 1) asm volatile("bar.sync %0, 64;" ::"r"(3 + wl + 4 * (it_n & 1)) : "memory");
                if (kSplit == 1) {
                    if (masked) {
                        exp_pack<true, 16>(s, 0, sc2, nm2, tail, pk);
                        exp_pack<true, 16>(s, 32, sc2, nm2, tail, pk + 16);
                        exp_pack<true, 16>(s, 64, sc2, nm2, tail, pk + 32);
                        exp_pack<true, 8>(s, 96, sc2, nm2, tail, pk + 48);
                    } else {
                        exp_pack<false, 16>(s, 0, sc2, nm2, kHalf, pk);
                        exp_pack<false, 16>(s, 32, sc2, nm2, kHalf, pk + 16);
                        exp_pack<false, 16>(s, 64, sc2, nm2, kHalf, pk + 32);
                        exp_pack<false, 8>(s, 96, sc2, nm2, kHalf, pk + 48);
                    }
                } else {
                    if (masked) {
                        exp_pack<true, 16>(s, 0, sc2, nm2, tail, pk);
                        exp_pack<true, 12>(s, 32, sc2, nm2, tail, pk + 16);
                    } else {
                        exp_pack<false, 16>(s, 0, sc2, nm2, kHalf, pk);
                        exp_pack<false, 12>(s, 32, sc2, nm2, kHalf, pk + 16);
                    }
                }
                if (PAB_FA_LAG == 2 && kSplit == 1 && t == 0) asm volatile("bar.arrive %0, 64;" ::"r"(3 + wl + 4 * (it_n & 1)) : "memory");
                FA_TRACE(trc, it_n, t, 4);
                if (!waited && it_n > 0) {
                    mbar_wait(&bars->o_done[tb], (it_n - 1) & 1);
                    tc_fence_after();
                }
                if (!kEpiWarps && j == 0 && have_prev) epilogue(prev);  // O of the previous item is final
                if (kSplit == 1) {
                    PAB_TMEM_ST16U(p_tmem, pk);
                    PAB_TMEM_ST16U(p_tmem + 16, (pk + 16));
                    PAB_TMEM_ST16U(p_tmem + 32, (pk + 32));
                    PAB_TMEM_ST8U(p_tmem + 48, (pk + 48));
                } else {
                    PAB_TMEM_ST16U(p_tmem, pk);
                    PAB_TMEM_ST8U(p_tmem + 16, (pk + 16));
                    PAB_TMEM_ST4U(p_tmem + 24, (pk + 24));
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->p_full[tb]);
                FA_TRACE(trc, it_n, t, 5);
            }
            if (active) {
                prev = it;
                have_prev = true;
            }
        }
        if (!kEpiWarps && have_prev) {
            mbar_wait(&bars->o_done[tb], (it_n - 1) & 1);
            tc_fence_after();
            epilogue(prev);
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // tile stores complete before exit
    } else if (kEpiWarps && warp >= kEpiWarp0) {
        // ================================= dedicated epilogue (warp = kEpiWarp0 + lane quarter)
        // per item and tile: wait for the item's last P.V (o_final), read the row sum and O out
        // of TMEM in 16-column chunks into the dense staging rows, hand O back to the MMA warp
        // (o_free: the next item's first P.V overwrites it), then one thread issues the tile's
        // TMA tensor store.  Off the softmax warps' critical path.
        const int wl = warp & 3;
        const int row = wl * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wl * 32) << 16;
        const bool issuer = (wl == 0 && lane == 0);
        int last_t = -1;  // staging tile of the issuer's most recent bulk store
        for (int c = 0; c < my_items; ++c) {
            const Item it = decode((int)blockIdx.x + c * (int)gridDim.x);
            for (int t = 0; t < 2; ++t) {
                const uint32_t o_tmem = tmem + lane_off + G::kOCol0 + G::kOStride * t;
                mbar_wait(&bars->o_final[t], c & 1);
                tc_fence_after();
                const bool active = (t == 0) || it.two;
                uint8_t* stg_tile = smem + G::kX0 + t * kRows * G::kStageRow;
#ifdef PAB_FA_DIAG_NOEPI  // timing diagnostic only: O never leaves TMEM (barrier hand-off kept)
                if (false) {
#else
                if (active) {
#endif
                    // the previous store of this staging tile has read its rows (the other tile's
                    // store, if it is the most recent one, may stay in flight)
                    if (issuer) {
                        if (last_t >= 0 && last_t != t) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    }
                    asm volatile("bar.sync 11, 128;" ::: "memory");
                    float o[16];
                    PAB_TMEM_LD16(o_tmem + 16 * (p.dh / 16), o);  // row sum sits in column dh
                    tmem_wait_ld();
                    float l = o[0];
#pragma unroll
                    for (int e = 1; e < 16; ++e) l = (e == p.dh % 16) ? o[e] : l;
                    const float inv = (l > 0.f) ? 1.0f / l : 0.f;
                    uint8_t* stg = stg_tile + row * (2 * p.dh);  // dense rows: the TMA box layout
                    for (int cc = 0; 16 * cc < p.dh; ++cc) {
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
                }
                // O of this tile is in registers / smem: the next item's first P.V may overwrite it
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->o_free[t]);
#ifdef PAB_FA_DIAG_NOEPI
                if (false) {
#else
                if (active) {
#endif
                    fence_async_smem();  // generic-proxy smem writes -> visible to the TMA (async proxy)
                    asm volatile("bar.sync 11, 128;" ::: "memory");
#ifndef PAB_FA_DIAG_EPI_NOSTORE
                    if (issuer)
                        asm volatile(
                            "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n\t"
                            "cp.async.bulk.commit_group;" ::"l"(reinterpret_cast<uint64_t>(&omap)),
                            "r"(smem_u32(stg_tile)), "r"(0), "r"(it.h), "r"((it.tile0 + t) * kRows), "r"(it.b_idx),
                            "r"(it.a_idx)
                            : "memory");
#endif
                    last_t = t;
                }
            }
        }
        if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // tile stores complete before exit
    } else if (warp == kTmaWarp) {
        // ===================================================== TMA producer
        if (lane == 0) {
            constexpr uint32_t kQBytes = kRows * (N128 * 128 + N32 * 32);
            constexpr uint32_t kKBytes = kKv * (N128 * 128 + N32 * 32);
            constexpr uint32_t kVBytes = kKv * NV * 32;
            int g = 0;  // K/V tiles loaded so far
            for (int c = 0; c < my_items; ++c) {
                const Item it = decode((int)blockIdx.x + c * (int)gridDim.x);
                const int qb = c & 1;
                if (c >= 2) mbar_wait(&bars->q_empty[qb], ((c >> 1) - 1) & 1);
                mbar_expect_tx(&bars->q_full[qb], (it.two ? 2u : 1u) * kQBytes);
                for (int t = 0; t < (it.two ? 2 : 1); ++t) {
                    uint8_t* dst = smem + G::kQ0 + (2 * qb + t) * G::kSlot;
                    const int i0 = (it.tile0 + t) * kRows;
                    for (int blk = 0; blk < N128; ++blk)
                        tma_load_5d(dst + blk * 16384, &q128, &bars->q_full[qb], 64 * blk, it.h, i0, it.b_idx,
                                    it.a_idx);
                    for (int blk = 0; blk < N32; ++blk)
                        tma_load_5d(dst + N128 * 16384 + blk * 4096, &q32, &bars->q_full[qb], 64 * N128 + 16 * blk,
                                    it.h, i0, it.b_idx, it.a_idx);
                }
                for (int j = 0; j < n_kv; ++j, ++g) {
                    const int st = g % 3;
                    if (g >= 3) mbar_wait(&bars->k_empty[st], ((g / 3) - 1) & 1);
                    uint8_t* kd = smem + G::kK0 + st * G::kSlotKV;
                    mbar_expect_tx(&bars->k_full[st], kKBytes);
                    for (int blk = 0; blk < N128; ++blk)
                        tma_load_5d(kd + blk * G::kK128, &k128, &bars->k_full[st], 64 * blk, it.h, j * kKv, it.b_idx,
                                    it.a_idx);
                    for (int blk = 0; blk < N32; ++blk)
                        tma_load_5d(kd + N128 * G::kK128 + blk * G::kK32, &k32, &bars->k_full[st], 64 * N128 + 16 * blk,
                                    it.h, j * kKv, it.b_idx, it.a_idx);
                    // V as 16-column SW32 atoms ([atom][row][32 B], atoms 4 KB apart): one MN-major
                    // descriptor spans the padded head dim; atom NV-1 holds the row-sum column
                    if (g >= 3) mbar_wait(&bars->v_empty[st], ((g / 3) - 1) & 1);
                    uint8_t* vd = smem + G::kV0 + st * G::kSlotKV;
                    mbar_expect_tx(&bars->v_full[st], kVBytes);
                    for (int blk = 0; blk < NV; ++blk)
                        tma_load_5d(vd + blk * G::kVAtom, &v32, &bars->v_full[st], 16 * blk, it.h, j * kKv, it.b_idx,
                                    it.a_idx);
                }
            }
        }
    } else if (warp == kFixWarp) {
        // ====================================== fixer warp (after each TMA load, before the MMA)
        // V[:, dh] = 1 (zero-filled by TMA): the P.V MMA then accumulates the row sums into
        // O[:, dh].  With padmask also Q[:, dh] = 1 and, in a partial last K tile, K[r, dh] =
        // -1e30 for rows r >= the live keys (see padmask).
        // SW32 atoms: row r at 32 r, 16-byte chunk index XOR (r >> 2) & 1.
        const int col = p.dh % 16;
        const uint32_t atom_off = (uint32_t)(p.dh / 16) * (uint32_t)G::kVAtom;
        const uint32_t cw = (uint32_t)(col & 7) * 2;
        auto sw32 = [&](int r) { return (uint32_t)r * 32u + (((uint32_t)(col >> 3) ^ (uint32_t)((r >> 2) & 1)) * 16u) + cw; };
        const int blk = (p.dh - 64 * N128) >> 4;  // SW32 block of column dh in Q / K
        const uint32_t q_off = (uint32_t)(N128 * 16384 + blk * 4096), k_off = (uint32_t)(N128 * G::kK128 + blk * G::kK32);
        const int tail_k = p.n_k - (n_kv - 1) * kKv;
#ifndef PAB_FA_PADK
#define PAB_FA_PADK -1e30f
#endif
        const __nv_bfloat16 one = __float2bfloat16_rn(1.0f), neg = __float2bfloat16_rn(PAB_FA_PADK);
        int g = 0;
        for (int c = 0; c < my_items; ++c) {
            const Item it = decode((int)blockIdx.x + c * (int)gridDim.x);
            const int qb = c & 1;
            mbar_wait(&bars->q_full[qb], (c >> 1) & 1);
            if (padmask)
                for (int t = 0; t < (it.two ? 2 : 1); ++t) {
                    uint8_t* qd = smem + G::kQ0 + (2 * qb + t) * G::kSlot + q_off;
                    for (int r = lane; r < kRows; r += 32) *reinterpret_cast<__nv_bfloat16*>(qd + sw32(r)) = one;
                }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->q_ready[qb]);
            for (int j = 0; j < n_kv; ++j, ++g) {
                const int st = g % 3;
                mbar_wait(&bars->k_full[st], (g / 3) & 1);
                if (padmask && j == n_kv - 1 && tail_k < kKv) {
                    uint8_t* kd = smem + G::kK0 + st * G::kSlotKV + k_off;
                    for (int r = tail_k + lane; r < kKv; r += 32) *reinterpret_cast<__nv_bfloat16*>(kd + sw32(r)) = neg;
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->k_ready[st]);
                mbar_wait(&bars->v_full[st], (g / 3) & 1);
                uint8_t* vd = smem + G::kV0 + st * G::kSlotKV + atom_off;
                for (int r = lane; r < kKv; r += 32) *reinterpret_cast<__nv_bfloat16*>(vd + sw32(r)) = one;
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->v_ready[st]);
            }
        }
    } else if (warp == kMmaWarp) {
        // ============================ MMA issuer (warp-converged; one elected lane issues the MMAs)
        constexpr uint32_t idS128 = idesc_bf16(128, kKv, 0);
        constexpr uint32_t idO = idesc_bf16(128, G::kOCols, 1);
        // descriptor words: lo = (addr >> 4) | (LBO >> 4) << 16, hi = (SBO >> 4) | version | layout
        // (smem_desc bit layout: SBO >> 4 at [32, 46), version 1 at bit 46, layout at [61, 64))
        const uint32_t q_lo = smem_u32(smem + G::kQ0) >> 4, k_lo = smem_u32(smem + G::kK0) >> 4;
        const uint32_t v_lo = smem_u32(smem + G::kV0) >> 4;
        constexpr uint32_t kHi128 = (1024u >> 4) | (1u << 14) | (kLayoutSW128 << 29);
        constexpr uint32_t kHi32 = (256u >> 4) | (1u << 14) | (kLayoutSW32 << 29);
        constexpr uint32_t kLbo16 = (16u >> 4) << 16;
        // V: MN-major SW32, 16-column atoms kVAtom B apart (LBO), 8-row groups 256 B apart (SBO)
        constexpr uint32_t kLboV = ((uint32_t)G::kVAtom >> 4) << 16;
        auto cols_of = [&](int j) {
            if (padmask) return kKv;  // padded keys are scored -1e30 by the MMA itself
            const int n = min(kKv, p.n_k - j * kKv);
            return (n + 15) & ~15;
        };
        // S_t = Q_t K^T for the item's tiles (Q slots 2 qb + t, K stage kst), K-steps of the
        // two tiles interleaved: MMAs on one accumulator serialise at ~80 cycles each, two
        // independent accumulators keep the tensor pipe busy.  ncols = keys rounded up to 16.
        auto issue_s = [&](int qb, int kst, int ncols, bool two) {
            const uint32_t ka = k_lo + ((kst * G::kSlotKV) >> 4);
            const uint32_t qa0 = q_lo + ((2 * qb * G::kSlot) >> 4);
            const uint32_t idS = (idS128 & ~(0x3Fu << 17)) | ((uint32_t)(ncols >> 3) << 17);
            if (N128 == 1 && N32 == 1) {
                const uint64_t dq = ((uint64_t)kHi128 << 32) | (qa0 | kLbo16);
                const uint64_t dk = ((uint64_t)kHi128 << 32) | (ka | kLbo16);
                const uint64_t dq32 = ((uint64_t)kHi32 << 32) | ((qa0 + (16384 >> 4)) | kLbo16);
                const uint64_t dk32 = ((uint64_t)kHi32 << 32) | ((ka + (G::kK128 >> 4)) | kLbo16);
                mma_group_s_72(tmem + kSCol, tmem + kSCol + kKv, dq, dk, dq32, dk32, idS, two, G::kSlot >> 4);
                return;
            }
            if (lane != 0) return;
            for (int t = 0; t < (two ? 2 : 1); ++t) {
                const uint32_t qa = qa0 + ((t * G::kSlot) >> 4);
                const uint32_t d_s = tmem + kSCol + kKv * t;
                for (int blk = 0; blk < N128; ++blk)
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t oq = (blk * 16384 + 32 * k) >> 4, ok = (blk * G::kK128 + 32 * k) >> 4;
                        mma_ss1(d_s, (qa + oq) | kLbo16, kHi128, (ka + ok) | kLbo16, kHi128, idS, (blk | k) != 0);
                    }
                for (int blk = 0; blk < N32; ++blk) {
                    const uint32_t oq = (N128 * 16384 + blk * 4096) >> 4, ok = (N128 * G::kK128 + blk * G::kK32) >> 4;
                    mma_ss1(d_s, (qa + oq) | kLbo16, kHi32, (ka + ok) | kLbo16, kHi32, idS, (N128 | blk) != 0);
                }
            }
        };
        // O_t += P_t V: ncols / 16 K-steps of 16 keys, both tiles interleaved; A = P_t from TMEM
        auto issue_pv = [&](int vst, uint32_t accumulate, int ncols, bool two) {
            const uint32_t va = v_lo + ((vst * G::kSlotKV) >> 4);
            if (kKv / 16 == 7) {
                const uint64_t dv = ((uint64_t)kHi32 << 32) | (va | kLboV);
                mma_group_pv7(tmem + G::kOCol0, tmem + G::kOCol0 + G::kOStride, tmem + kPCol, tmem + kPCol + 64, dv,
                              idO, accumulate, two, ncols / 16);
                return;
            }
            if (lane != 0) return;
            for (int k = 0; 16 * k < ncols; ++k)
                for (int t = 0; t < (two ? 2 : 1); ++t)
                    mma_ts1(tmem + G::kOCol0 + G::kOStride * t, tmem + kPCol + 64 * t + 8 * k,
                            (va + ((512 * k) >> 4)) | kLboV, kHi32, idO, accumulate | (k > 0));
        };
        // O_t += P_t V for one tile (a single-accumulator chain of ncols / 16 K-steps)
        auto issue_pv_tile = [&](int vst, int t, uint32_t accumulate, int ncols) {
            const uint32_t va = v_lo + ((vst * G::kSlotKV) >> 4);
            const uint32_t o_t = tmem + G::kOCol0 + G::kOStride * t, p_t = tmem + kPCol + 64 * t;
            if (kKv / 16 == 7) {
                const uint64_t dv = ((uint64_t)kHi32 << 32) | (va | kLboV);
                mma_group_pv7(o_t, o_t, p_t, p_t, dv, idO, accumulate, 0, ncols / 16);
                return;
            }
            if (lane != 0) return;
            for (int k = 0; 16 * k < ncols; ++k)
                mma_ts1(o_t, p_t + 8 * k, (va + ((512 * k) >> 4)) | kLboV, kHi32, idO, accumulate | (k > 0));
        };
        // iteration gi = (item c, kv tile j), KV tile g.  The tiles run in phase: S(gi+1) of
        // both tiles is issued once both softmaxes have read S(gi) (early in their iteration),
        // PV(gi) once both have stored P(gi).
        int c = 0, j = 0, g = 0;
        Item it = decode((int)blockIdx.x);
        if (my_items > 0) {
            mbar_wait2(&bars->q_ready[0], 0, &bars->k_ready[0], 0);
            tc_fence_after();
            issue_s(0, 0, cols_of(0), it.two);
            tc_commit(&bars->s_full);
            tc_commit(&bars->k_empty[0]);
            if (n_kv == 1) tc_commit(&bars->q_empty[0]);
        }
        for (int gi = 0; gi < n_iters; ++gi) {
            // ---- S of the next iteration (may belong to the next item)
            if (gi + 1 < n_iters) {
                int c1 = c, j1 = j + 1;
                if (j1 == n_kv) {
                    c1 = c + 1;
                    j1 = 0;
                }
                const Item it1 = (c1 == c) ? it : decode((int)blockIdx.x + c1 * (int)gridDim.x);
                const int g1 = g + 1;
                FA_TRACE(lane == 0, gi, 0, 10);
                if (j1 == 0) mbar_wait(&bars->q_ready[c1 & 1], (c1 >> 1) & 1);
                mbar_wait2(&bars->s_free, gi & 1, &bars->k_ready[g1 % 3], (g1 / 3) & 1);
                tc_fence_after();
                FA_TRACE(lane == 0, gi, 0, 8);
                issue_s(c1 & 1, g1 % 3, cols_of(j1), it1.two);
                tc_commit(&bars->s_full);
                tc_commit(&bars->k_empty[g1 % 3]);
                if (j1 == n_kv - 1) tc_commit(&bars->q_empty[c1 & 1]);  // last S of item c1 issued
            }
            // ---- PV of this iteration
            FA_TRACE(lane == 0, gi, 1, 10);
            if (kPvSplit) {
                // tile 0's P.V goes as soon as tile 0's P is stored: its next P store (which
                // must wait for this P.V) no longer waits behind tile 1's exp section
                mbar_wait2(&bars->p_full[0], gi & 1, &bars->v_ready[g % 3], (g / 3) & 1);
                // first P.V of an item overwrites O: the epilogue warps must have read the last item's
                if (kEpiWarps && j == 0 && c > 0) mbar_wait(&bars->o_free[0], (c - 1) & 1);
                tc_fence_after();
                FA_TRACE(lane == 0, gi, 1, 8);
                issue_pv_tile(g % 3, 0, j > 0, cols_of(j));
                tc_commit(&bars->o_done[0]);
                if (kEpiWarps && j == n_kv - 1) tc_commit(&bars->o_final[0]);
                mbar_wait(&bars->p_full[1], gi & 1);
                if (kEpiWarps && j == 0 && c > 0) mbar_wait(&bars->o_free[1], (c - 1) & 1);
                tc_fence_after();
                if (it.two) issue_pv_tile(g % 3, 1, j > 0, cols_of(j));
                tc_commit(&bars->o_done[1]);
                if (kEpiWarps && j == n_kv - 1) tc_commit(&bars->o_final[1]);
            } else {
                mbar_wait2(&bars->p_full[0], gi & 1, &bars->v_ready[g % 3], (g / 3) & 1);
                tc_fence_after();
                FA_TRACE(lane == 0, gi, 1, 8);
                issue_pv(g % 3, j > 0, cols_of(j), it.two);
                tc_commit(&bars->o_done[0]);
            }
            tc_commit(&bars->v_empty[g % 3]);
            FA_TRACE(lane == 0, gi, 1, 9);
            ++g;
            if (++j == n_kv) {
                j = 0;
                ++c;
                if (c < my_items) it = decode((int)blockIdx.x + c * (int)gridDim.x);
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
        if (cudaFuncSetAttribute(attn_fa_kernel<N128, N32, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 G::kSmem) != cudaSuccess)
            return launch_status("attn_fa smem attribute");
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
        // O rows leave through one TMA tensor store per 128-row tile (box = dh x 128 rows)
        !make_map(&mo, a->o, a->dh, a->heads, a->n_q, a->n_b, a->n_a, a->o_si, a->o_sb, a->o_sa, a->dh, kRows, 1,
                  CU_TENSOR_MAP_SWIZZLE_NONE))
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
    p.f_heads = make_fastdiv((uint32_t)a->heads);
    p.f_full = make_fastdiv((uint32_t)(PAB_FA_SINGLES_LAST ? p.row_tiles / 2 : p.n_pairs));
    p.f_b = make_fastdiv((uint32_t)a->n_b);
    static int num_sms = 0;
    if (num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (num_sms <= 0) num_sms = 148;
    }
    dim3 grid((unsigned)(p.n_items < num_sms ? p.n_items : num_sms));
    attn_fa_kernel<N128, N32, NV><<<grid, kThreads, G::kSmem, st>>>(mq128, mq32, mk128, mk32, mv32, mo, p);
    return launch_status("attn_fa");
}

}  // namespace fa

bool attn_fa_supported(const pab_attn_args* a) { return a->dh % 8 == 0 && a->dh <= 72; }

// non-packed attention (spatial, cross) with dh <= 72 and a multiple of 8
int attn_fa_launch(const pab_attn_args* a, cudaStream_t st) {
    const int n128 = a->dh / 64;
    const int n32 = (a->dh - 64 * n128 + 15) / 16;
    const int nv = a->dh / 16 + 1;
#define PAB_FA(A, B, C) \
    if (n128 == A && n32 == B && nv == C) return fa::launch<A, B, C>(a, st)
    PAB_FA(0, 1, 1);  // dh 8
    PAB_FA(0, 1, 2);  // dh 16
    PAB_FA(0, 2, 2);  // dh 24
    PAB_FA(0, 2, 3);  // dh 32
    PAB_FA(0, 3, 3);  // dh 40
    PAB_FA(0, 3, 4);  // dh 48
    PAB_FA(0, 4, 4);  // dh 56
    PAB_FA(1, 0, 5);  // dh 64
    PAB_FA(1, 1, 5);  // dh 72
#undef PAB_FA
    return PAB_ERR_UNSUPPORTED;
}

}  // namespace pab

// Projection GEMMs of the PAB sites on the 5th-gen tensor cores (sm_100a).
//
// reference op: numerics.matmul (pkg/src/pab_engine/numerics.py:72-104) as called for
// every projection of a computed site -- q/k/v and o of the spatial / temporal sites
// (model.py:346-359), q and o of the cross sites (model.py:376-385) and the two MLP
// matrices with the tanh-GELU between them (model.py:398-403, numerics.py:154-158).
//
//   C[M, N] = epilogue( A[M, K] @ W[K, N] )     A, C bf16 row-major; W stored as B = W^T,
//                                               (N, K) K-major; fp32 accumulation in TMEM
//   epilogue 0: bf16(acc)          epilogue 1: bf16(gelu_tanh(acc))
//
// Design (one persistent CTA pair per TPC, 74 pairs on 148 SMs):
//  * 2-CTA MMA (tcgen05.mma.cta_group::2): a pair computes a 256 x 256 output tile; each
//    CTA stages its own 128 rows of A and 128 rows of B per 64-wide K slab (TMA, 128-byte
//    swizzle), so each SM reads half the B bytes it would need alone; N % 256 is covered by
//    one narrower last tile (MMA N = the remainder rounded up to 64);
//  * warp roles per CTA: warps 0-3 epilogue (one TMEM lane = one output row per thread),
//    warp 4 TMA producer, warp 5 TMEM owner + MMA issuer (leader CTA only);
//  * a 6-stage smem ring (full barriers in the leader, signalled by both CTAs' TMA
//    transactions; empty barriers in both, released by the leader's MMA commit multicast);
//  * two TMEM accumulators (2 x BN fp32 columns): the epilogue of tile i drains one while
//    the MMAs of tile i+1 fill the other;
//  * epilogue: tcgen05.ld 32 columns at a time -> (GELU) -> bf16 -> 128-byte swizzled smem
//    staging (two 16 KB buffers) -> one TMA tensor store per 128 x 64 box.
#include "tc_ptx.cuh"
#include <stdlib.h>

namespace pab {
namespace gemm {

using namespace pab::tc;

constexpr int kBK = 64;                 // K slab per stage (one 128-byte swizzle atom of bf16)
constexpr int kRowsCta = 128;           // A rows per CTA (pair tile M = 256)
#ifndef PAB_GEMM_EPI_WARPS
#define PAB_GEMM_EPI_WARPS 8  // 4: one epilogue warp per SM sub-partition; 8: two (overlap TMEM loads and math)
#endif
constexpr int kEpiWarps = PAB_GEMM_EPI_WARPS;
constexpr int kEpiGroups = kEpiWarps / 4;
constexpr int kBufPerGroup = kEpiGroups == 1 ? 2 : 1;   // epilogue staging boxes per warp group
constexpr int kThreads = 32 * (kEpiWarps + 2);          // epilogue warps + producer + MMA
constexpr int kProducerWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
constexpr int kStageBoxBytes = kRowsCta * 128;  // 128 rows x 64 bf16 epilogue box
static_assert(kEpiWarps == 4 || kEpiWarps == 8, "epilogue warps");

constexpr int kXBoxBytes = kRowsCta * 128;   // 128 rows x 32 fp32 residual box
// RESID: 0 plain epilogue; 1 residual add with the fp32 x chunk streamed through smem by TMA
// (epilogue latency matters: K = 1152 projections); 2 residual add by direct per-thread
// global read-modify-write of whole row segments -- no smem, so the operand ring keeps its
// depth (K = 4608: the MLP w2 GEMM, whose epilogue hides behind a long mainloop)
template <int BN, int RESID = 0>
struct Cfg {
    static constexpr int kABytes = kRowsCta * kBK * 2;          // 16 KB
    static constexpr int kBBytes = (BN / 2) * kBK * 2;          // BN/2 rows of B
    static constexpr int kStageBytes = kABytes + kBBytes;
    // RESID: per epilogue group, one 64-column fp32 residual chunk (two 32-column boxes)
    static constexpr int kXBytes = RESID == 1 ? kEpiGroups * 2 * kXBoxBytes : 0;
    static constexpr int kEpiBytes = kEpiGroups * kBufPerGroup * kStageBoxBytes + kXBytes;
    static constexpr int kStages = (232448 - kEpiBytes - 1280) / kStageBytes > 8
                                       ? 8 : (232448 - kEpiBytes - 1280) / kStageBytes;
    static constexpr int kRing = kStages * kStageBytes;
    static constexpr int kEpi0 = kRing;                          // epilogue staging boxes
    static constexpr int kBar0 = kEpi0 + kEpiBytes;
    static constexpr int kSmem = kBar0 + 256 + 1024;             // barriers + 1 KB alignment slack
    static_assert(BN % 32 == 0 && BN <= 256 && (BN / 2) % 16 == 0, "tile N");
    static_assert(kABytes % 1024 == 0 && kBBytes % 1024 == 0, "swizzle atoms");
    static_assert(kSmem <= 232448, "smem");
};

struct Bars {
    uint64_t full[8], empty[8], tfull[2], tempty[2];
    uint64_t xfull[2];  // RESID: residual chunk of epilogue group g landed
};

struct Params {
    int m_tiles, n_tiles, k_slabs, tiles;
    int n_last;    // width of the last N tile (a multiple of 64, <= BN): N = (n_tiles-1)*BN + n_last - pad
    int epilogue;
    int group;  // M tiles per raster group
    // epilogue 2 (residual): x[perm(m), n] += bf16(acc); C written only if store_c
    float* x;
    int64_t ldx, M, N;
    int64_t tm_t, tm_s;  // > 0: GEMM rows are token-major (b, s, t), x rows frame-major (b, t, s)
    int store_c;
    // RESID: optional h = bf16(x + o) in x's (frame-major) row order, ld ldh -- the next
    // cross site's query input, so its stand-alone cast pass (6E bytes) is not needed
    __nv_bfloat16* h;
    int64_t ldh, h_rows;  // h rows (x order) < h_rows are written (the live CFG rows of the cross site)
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-CTA TMA load: data lands in this CTA's smem, the transaction bytes are counted on the
// leader CTA's barrier (peer bit of the barrier address cleared)
__device__ __forceinline__ void tma_load_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(b), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

__device__ __forceinline__ float gelu_tanh(float x) {
    // numerics.py:154-158: 0.5 x (1 + tanh(u)), u = sqrt(2/pi) (x + 0.044715 x^3),
    // evaluated as x * sigmoid(2u) = x / (1 + exp(-2u)) (identical; no cancellation in the
    // negative tail); exp via ex2 with the log2(e) factor folded into the constant
    const float z = -2.0f * 1.4426950408889634f * 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
    return __fdividef(x, 1.0f + fast_exp2(z));
}

// tile t -> (m, n): groups of 8 M-tiles sweep all N tiles, so the pairs in flight share
// A row blocks and the (small) weight matrix stays L2-resident
__device__ __forceinline__ void tile_coords(int t, const Params& p, int& m, int& n) {
    const int G = p.group;
    const int per_group = G * p.n_tiles;
    const int g = t / per_group, r = t - g * per_group;
    const int gm = min(G, p.m_tiles - g * G);
    m = g * G + r % gm;
    n = r / gm;
}

template <int BN, bool NARROW, int RESID>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_x,
                const Params p) {
    using C = Cfg<BN, RESID>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + C::kBar0);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kBar0 + sizeof(Bars));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->tfull[a], 1);
            mbar_init(&bars->tempty[a], 2 * kEpiWarps);  // both CTAs' epilogue warps
            mbar_init(&bars->xfull[a], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kProducerWarp && lane == 0) {
        prefetch_map(&map_a);
        prefetch_map(&map_b);
        prefetch_map(&map_c);
        if (RESID == 1) prefetch_map(&map_x);
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == kProducerWarp) {
        // ================================================================ TMA producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = pair; t < p.tiles; t += n_pairs) {
                int tm, tn;
                tile_coords(t, p, tm, tn);
                const int row = tm * 2 * kRowsCta + (int)rank * kRowsCta;
                const int width = (NARROW && tn == p.n_tiles - 1) ? p.n_last : BN;
                const int col = tn * BN + (int)rank * (width / 2);
                for (int kb = 0; kb < p.k_slabs; ++kb) {
                    mbar_wait(&bars->empty[s], ph ^ 1);
                    if (leader) mbar_expect_tx(&bars->full[s], 2 * C::kStageBytes);
                    uint8_t* st = smem + s * C::kStageBytes;
                    tma_load_2sm(st, &map_a, &bars->full[s], kb * kBK, row);
                    tma_load_2sm(st + C::kABytes, &map_b, &bars->full[s], kb * kBK, col);
                    if (++s == C::kStages) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ================================================================ MMA issuer (leader)
        if (leader) {
            constexpr uint32_t idesc_full = idesc_bf16(256, BN, 0);
            const uint32_t idesc_last = idesc_bf16(256, p.n_last, 0);
            constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (kLayoutSW128 << 29);
            constexpr uint32_t kLbo = (16u >> 4) << 16;
            const uint32_t base_lo = smem_u32(smem) >> 4;
            int s = 0, acc = 0;
            uint32_t ph = 0, aph = 0;
            // NARROW: the last N tile is narrower -- its MMAs have N = n_last (each CTA supplies
            // n_last / 2 rows of B), so a 3456-wide output is 13 x 256 + 128, not 14 x 256.
            // A separate instantiation: the per-tile (m, n) arithmetic on the MMA issue path
            // cost 3% at K = 1152 where no tile is narrow (profiles/r02_gemm_tuning.md)
            for (int t = pair; t < p.tiles; t += n_pairs) {
                mbar_wait(&bars->tempty[acc], aph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * BN);
                uint32_t idesc = idesc_full;
                if constexpr (NARROW) {
                    int tm, tn;
                    tile_coords(t, p, tm, tn);
                    if (tn == p.n_tiles - 1) idesc = idesc_last;
                }
                for (int kb = 0; kb < p.k_slabs; ++kb) {
                    mbar_wait(&bars->full[s], ph);
                    tc_fence_after();
                    const uint32_t a_lo = base_lo + ((s * C::kStageBytes) >> 4);
                    const uint32_t b_lo = a_lo + (C::kABytes >> 4);
                    if (lane == 0) {
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            const uint64_t da = ((uint64_t)kHi << 32) | ((a_lo + 2 * k) | kLbo);
                            const uint64_t db = ((uint64_t)kHi << 32) | ((b_lo + 2 * k) | kLbo);
                            mma2(d, da, db, idesc, (kb | k) != 0);
                        }
                        commit2(&bars->empty[s]);
                    }
                    __syncwarp();
                    if (++s == C::kStages) { s = 0; ph ^= 1; }
                }
                if (lane == 0) commit2(&bars->tfull[acc]);
                __syncwarp();
                if (++acc == 2) { acc = 0; aph ^= 1; }
            }
        }
    } else {
        // ============================================ epilogue (warps 0 .. kEpiWarps-1)
        // kEpiGroups groups of 4 warps; group g drains 64-column chunks c = g, g + kEpiGroups,
        // ... of each accumulator (a thread owns one TMEM lane == one output row)
        const int g = warp >> 2;
        const int r = threadIdx.x & 127;  // row within the CTA's 128-row half == TMEM lane
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tempty_leader0 = mapa(smem_u32(&bars->tempty[0]), 0);
        const uint32_t tempty_leader1 = mapa(smem_u32(&bars->tempty[1]), 0);
        uint8_t* stage0 = smem + C::kEpi0 + g * kBufPerGroup * kStageBoxBytes;
        int acc = 0, box = 0;
        uint32_t aph = 0;
        // ---- RESID: the residual add of the site output, x = x + o (reference model.py:503),
        // done here instead of by the next site's prologue.  Each group streams its 64-column
        // fp32 chunk of x through shared memory by TMA (two 32-column boxes, 128-byte swizzle):
        // load (issued ahead: at tile start for the group's first chunk, right after the
        // previous chunk's store otherwise), add the bf16-rounded o row by row (thread == row,
        // like the accumulator), TMA-store back; o itself is stored only if p.store_c.
        uint8_t* xbuf = smem + C::kEpi0 + kEpiGroups * kBufPerGroup * kStageBoxBytes + g * 2 * kXBoxBytes;
        uint32_t xph = 0;
        // x tensor-map coordinates of a 128-row block: frame-major (col, row); token-major
        // (col, t = 0, s0, b) over the (D, T, S, B) view of the frame-major stream
        auto x_coords = [&](int row0, int& c1, int& c2, int& c3) {
            if (p.tm_t > 0) {
                const int64_t per_b = p.tm_t * p.tm_s;
                const int64_t b = row0 / per_b;
                c1 = 0;
                c2 = (int)((row0 - b * per_b) / p.tm_t);
                c3 = (int)b;
            } else {
                c1 = row0; c2 = 0; c3 = 0;
            }
        };
        auto x_load = [&](int col, int row0) {  // r == 0 only
            bulk_wait_read<0>();  // the previous x / o stores of this group have read smem
            int c1, c2, c3;
            x_coords(row0, c1, c2, c3);
            mbar_expect_tx(&bars->xfull[g], 2 * kXBoxBytes);
            for (int h = 0; h < 2; ++h)
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(xbuf + h * kXBoxBytes)),
                    "l"(reinterpret_cast<uint64_t>(&map_x)), "r"(smem_u32(&bars->xfull[g])), "r"(col + 32 * h),
                    "r"(c1), "r"(c2), "r"(c3)
                    : "memory");
        };
        auto resid_chunk = [&](float* v, int col, int row0, int next_col) {
            // bf16 site output; the stream adds exactly the cached value
#pragma unroll
            for (int i = 0; i < 64; ++i) v[i] = __bfloat162float(__float2bfloat16_rn(v[i]));
            named_bar(1 + g, 128);  // r == 0 has waited for the previous stores (x_load)
            if (p.store_c) {
                const uint32_t rowaddr = smem_u32(stage0) + (uint32_t)r * 128;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    st_shared_v4(rowaddr + (uint32_t)(((j ^ (r & 7)) * 16)), pack_bf16(v[8 * j], v[8 * j + 1]),
                                 pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                                 pack_bf16(v[8 * j + 6], v[8 * j + 7]));
            }
            mbar_wait(&bars->xfull[g], xph);
            xph ^= 1;
            // h row of this thread (x's frame-major order), nullptr if no h output / past M
            __nv_bfloat16* hrow = nullptr;
            if (p.h != nullptr) {
                const int64_t m = (int64_t)row0 + r;
                if (m < p.M) {
                    int64_t fr = m;  // (the h_rows check below)
                    if (p.tm_t > 0) {  // GEMM row (b, s, t) -> stream row (b, t, s)
                        const int64_t per_b = p.tm_t * p.tm_s, b = m / per_b, rem = m - b * per_b;
                        const int64_t s_ = rem / p.tm_t, t_ = rem - s_ * p.tm_t;
                        fr = (b * p.tm_t + t_) * p.tm_s + s_;
                    }
                    if (fr < p.h_rows) hrow = p.h + fr * p.ldh + col;
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t rowaddr = smem_u32(xbuf + h * kXBoxBytes) + (uint32_t)r * 128;
                uint32_t hp[4];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t a = rowaddr + (uint32_t)(((j ^ (r & 7)) * 16));
                    float4 xv;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(xv.x), "=f"(xv.y), "=f"(xv.z), "=f"(xv.w)
                                 : "r"(a));
                    const float* o = v + 32 * h + 4 * j;
                    xv.x += o[0]; xv.y += o[1]; xv.z += o[2]; xv.w += o[3];
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(xv.x), "f"(xv.y),
                                 "f"(xv.z), "f"(xv.w)
                                 : "memory");
                    hp[2 * (j & 1)] = pack_bf16(xv.x, xv.y);
                    hp[2 * (j & 1) + 1] = pack_bf16(xv.z, xv.w);
                    // 8 columns = one 16-byte store; a thread writes whole 128-byte row segments
                    if ((j & 1) && hrow != nullptr && col + 32 * h + 4 * j + 4 <= p.N)
                        __stcs(reinterpret_cast<uint4*>(hrow + 32 * h + 4 * (j - 1)),
                               make_uint4(hp[0], hp[1], hp[2], hp[3]));
                }
            }
            fence_async_smem();
            named_bar(1 + g, 128);
            if (r == 0) {
                if (p.store_c) tma_store_2d(&map_c, stage0, col, row0);
                int c1, c2, c3;
                x_coords(row0, c1, c2, c3);
                for (int h = 0; h < 2; ++h)
                    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                                     reinterpret_cast<uint64_t>(&map_x)),
                                 "r"(smem_u32(xbuf + h * kXBoxBytes)), "r"(col + 32 * h), "r"(c1), "r"(c2), "r"(c3)
                                 : "memory");
                bulk_commit();
                if (next_col >= 0) x_load(next_col, row0);  // this group's next chunk of the tile
            }
        };
        for (int t = pair; t < p.tiles; t += n_pairs) {
            int tm, tn;
            tile_coords(t, p, tm, tn);
            const int row0 = tm * 2 * kRowsCta + (int)rank * kRowsCta;
            const int kChunks = ((NARROW && tn == p.n_tiles - 1) ? p.n_last : BN) / 64;
            if constexpr (RESID == 1) {
                if (r == 0 && g < kChunks) x_load(tn * BN + g * 64, row0);  // before the accumulator is ready
            }
            mbar_wait(&bars->tfull[acc], aph);
            tc_fence_after();
#pragma unroll 1
            for (int c = g; c < kChunks; c += kEpiGroups) {
                float v[64];
                const uint32_t ta = tmem + lane_base + (uint32_t)(acc * BN + c * 64);
                PAB_TMEM_LD32(ta, v);
                PAB_TMEM_LD32(ta + 32, (v + 32));
                tmem_wait_ld();
                if (c + kEpiGroups >= kChunks) {
                    // this warp's last chunk of the accumulator is in registers: release it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
                }
                if (p.epilogue == 1) {
#pragma unroll
                    for (int i = 0; i < 64; ++i) v[i] = gelu_tanh(v[i]);
                }
                if constexpr (RESID == 1) {
                    resid_chunk(v, tn * BN + c * 64, row0, c + kEpiGroups < kChunks ? tn * BN + (c + kEpiGroups) * 64 : -1);
                    continue;
                }
                if constexpr (RESID == 2) {
                    // x += bf16(o) by the whole group, coalesced: o goes through this group's bf16
                    // staging box (the layout of the C store), then each warp instruction reads and
                    // writes 4 full 256-byte x row segments (8 columns per thread); the box also
                    // feeds the o store when the site is cached.  No extra smem.
                    uint8_t* sb = stage0 + box * kStageBoxBytes;
                    if (r == 0) bulk_wait_read<kBufPerGroup - 1>();
                    named_bar(1 + g, 128);
                    const uint32_t rowaddr = smem_u32(sb) + (uint32_t)r * 128;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        st_shared_v4(rowaddr + (uint32_t)(((j ^ (r & 7)) * 16)), pack_bf16(v[8 * j], v[8 * j + 1]),
                                     pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                                     pack_bf16(v[8 * j + 6], v[8 * j + 7]));
                    fence_async_smem();
                    named_bar(1 + g, 128);
                    const int col = tn * BN + c * 64;
                    if (r == 0 && p.store_c) {
                        tma_store_2d(&map_c, sb, col, row0);
                        bulk_commit();
                    }
#pragma unroll 2
                    for (int it = 0; it < 8; ++it) {
                        const int idx = it * 128 + r, rr = idx >> 3, seg = idx & 7;
                        const int64_t m = (int64_t)row0 + rr;
                        if (m >= p.M || col + 8 * seg >= p.N) continue;
                        uint32_t w[4];
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                                     : "r"(smem_u32(sb) + (uint32_t)rr * 128 + (uint32_t)((seg ^ (rr & 7)) * 16)));
                        float4* xr = reinterpret_cast<float4*>(p.x + m * p.ldx + col + 8 * seg);
                        float4 a = __ldcs(xr), b = __ldcs(xr + 1);
                        const float2 o0 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w[0]));
                        const float2 o1 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w[1]));
                        const float2 o2 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w[2]));
                        const float2 o3 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w[3]));
                        a.x += o0.x; a.y += o0.y; a.z += o1.x; a.w += o1.y;
                        b.x += o2.x; b.y += o2.y; b.z += o3.x; b.w += o3.y;
                        __stcs(xr, a);
                        __stcs(xr + 1, b);
                    }
                    if (++box == kBufPerGroup) box = 0;
                    continue;
                }
                uint8_t* sb = stage0 + box * kStageBoxBytes;
                // the TMA store issued from this buffer kBufPerGroup boxes ago must have read it
                if (r == 0) bulk_wait_read<kBufPerGroup - 1>();
                named_bar(1 + g, 128);
                const uint32_t rowaddr = smem_u32(sb) + (uint32_t)r * 128;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t a = rowaddr + (uint32_t)(((j ^ (r & 7)) * 16));
                    st_shared_v4(a, pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                                 pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
                }
                fence_async_smem();
                named_bar(1 + g, 128);
                if (r == 0) {
                    tma_store_2d(&map_c, sb, tn * BN + c * 64, row0);
                    bulk_commit();
                }
                if (++box == kBufPerGroup) box = 0;
            }
            if (++acc == 2) { acc = 0; aph ^= 1; }
        }
        if (r == 0) bulk_wait_all();
    }
    tc_fence_before();
    cluster_sync();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

static bool map_2d(CUtensorMap* m, const void* base, int64_t inner, int64_t outer, int64_t ld_elems, int box_inner,
                   int box_outer) {
    auto encode = get_encode();
    if (!encode) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 2};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    cuuint32_t estr[2] = {1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int g_sms = 0;
// tuning knobs for A/B runs (scripts/bench_gemm.py): PAB_GEMM_GROUP = M tiles per raster
// group
static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}
static int g_group = env_int("PAB_GEMM_GROUP", 8);
static int g_direct_k = env_int("PAB_GEMM_RESID_DIRECT_K", 2048);  // K from which RESID == 2 is used

static bool map_x4(CUtensorMap* m, float* x, int64_t N, int64_t M, int64_t ldx, int64_t tm_t, int64_t tm_s) {
    auto encode = get_encode();
    if (!encode) return false;
    cuuint64_t dims[4], strides[3];
    cuuint32_t box[4];
    const cuuint64_t row = (cuuint64_t)ldx * 4;
    if (tm_t > 0) {  // (D, T, S, B) view of the frame-major stream, box = 32 cols x T x 128/T tokens
        dims[0] = N; dims[1] = tm_t; dims[2] = tm_s; dims[3] = M / (tm_t * tm_s);
        strides[0] = row * tm_s; strides[1] = row; strides[2] = row * tm_t * tm_s;
        box[0] = 32; box[1] = (cuuint32_t)tm_t; box[2] = (cuuint32_t)(kRowsCta / tm_t); box[3] = 1;
    } else {
        dims[0] = N; dims[1] = M; dims[2] = 1; dims[3] = 1;
        strides[0] = row; strides[1] = row * M; strides[2] = row * M;
        box[0] = 32; box[1] = kRowsCta; box[2] = 1; box[3] = 1;
    }
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Resid {
    float* x = nullptr;
    int64_t ldx = 0, tm_t = 0, tm_s = 0;
    __nv_bfloat16* h = nullptr;
    int64_t ldh = 0, h_rows = 0;
};

template <int BN, bool NARROW, int RESID>
static int launch_t(const void* A, int64_t lda, const void* B, int64_t ldb, void* Cp, int64_t ldc, int64_t M,
                    int64_t N, int64_t K, int epilogue, const Resid& rs, cudaStream_t st) {
    using C = Cfg<BN, RESID>;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(gemm_kernel<BN, NARROW, RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::kSmem) != cudaSuccess)
            return launch_status("gemm smem attribute");
        attr = true;
    }
    CUtensorMap ma, mb, mc, mx;
    // residual epilogue without an o output: the C map is never used (built over A)
    const void* cbase = Cp ? Cp : A;
    const int64_t cld = Cp ? ldc : lda;
    if (!map_2d(&ma, A, K, M, lda, kBK, kRowsCta) || !map_2d(&mb, B, K, N, ldb, kBK, BN / 2) ||
        !map_2d(&mc, cbase, Cp ? N : K, M, cld, 64, kRowsCta))
        return PAB_ERR_CUDA;
    if (RESID == 1) {
        if (!map_x4(&mx, rs.x, N, M, rs.ldx, rs.tm_t, rs.tm_s)) return PAB_ERR_CUDA;
    } else {
        mx = ma;  // unused
    }
    Params p;
    p.m_tiles = (int)((M + 2 * kRowsCta - 1) / (2 * kRowsCta));
    p.n_tiles = (int)((N + BN - 1) / BN);
    // last tile width rounded up to whole 64-column epilogue boxes (B rows past N zero-filled,
    // C columns past N clipped by the tensor maps)
    p.n_last = (int)(((N - (int64_t)(p.n_tiles - 1) * BN) + 63) / 64 * 64);
    p.k_slabs = (int)((K + kBK - 1) / kBK);
    p.tiles = p.m_tiles * p.n_tiles;
    p.epilogue = epilogue;
    p.group = g_group;
    p.x = rs.x;
    p.ldx = rs.ldx;
    p.M = M;
    p.N = N;
    p.tm_t = rs.tm_t;
    p.tm_s = rs.tm_s;
    p.store_c = Cp != nullptr;
    p.h = rs.h;
    p.ldh = rs.ldh;
    p.h_rows = rs.h_rows;
    if (g_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int pairs = g_sms / 2;
    if (pairs > p.tiles) pairs = p.tiles;
    gemm_kernel<BN, NARROW, RESID><<<2 * pairs, kThreads, C::kSmem, st>>>(ma, mb, mc, mx, p);
    return launch_status("gemm");
}

template <int BN, int RESID>
static int launch(const void* A, int64_t lda, const void* B, int64_t ldb, void* Cp, int64_t ldc, int64_t M,
                  int64_t N, int64_t K, int epilogue, const Resid& rs, cudaStream_t st) {
    return (N % BN) ? launch_t<BN, true, RESID>(A, lda, B, ldb, Cp, ldc, M, N, K, epilogue, rs, st)
                    : launch_t<BN, false, RESID>(A, lda, B, ldb, Cp, ldc, M, N, K, epilogue, rs, st);
}

template <int RESID>
static int dispatch(const void* A, int64_t lda, const void* B, int64_t ldb, void* Cp, int64_t ldc, int64_t M,
                    int64_t N, int64_t K, int epilogue, const Resid& rs, cudaStream_t st) {
    // 256-wide tiles read the least shared memory per MMA (192: -6%, 128: -25% at N = 3456 / 4608,
    // profiles/r02_gemm_tuning.md), with one narrower last tile for N % 256.  The static
    // pair-strided order then leaves pairs unevenly loaded when the output has few tiles
    // per row block (N = 1152: 4 x 256 + 128), so there uniform 192-wide tiles win.
    if (N % 256 != 0 && N % 192 == 0 && N <= 1536)
        return launch<192, RESID>(A, lda, B, ldb, Cp, ldc, M, N, K, epilogue, rs, st);
    return launch<256, RESID>(A, lda, B, ldb, Cp, ldc, M, N, K, epilogue, rs, st);
}

}  // namespace gemm
}  // namespace pab

static int check_args(const void* A, int64_t lda, const void* B, int64_t ldb, const void* C, int64_t ldc,
                      int64_t M, int64_t N, int64_t K) {
    if (M < 0 || N <= 0 || K <= 0) return PAB_ERR_SHAPE;
    if (!A || !B) return PAB_ERR_INVALID;
    if (lda < K || ldb < K || (C && ldc < N)) return PAB_ERR_SHAPE;
    // TMA: 16-byte aligned bases and row strides (M, N and K tails are zero-filled / clipped)
    if ((uintptr_t)A % 16 || (uintptr_t)B % 16 || (uintptr_t)C % 16 || lda % 8 || ldb % 8 || (C && ldc % 8) ||
        K % 8)
        return PAB_ERR_UNSUPPORTED;
    if (M > 0x7fffffff || N > 0x7fffffff || K > 0x7fffffff) return PAB_ERR_UNSUPPORTED;
    return PAB_OK;
}

extern "C" int pab_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                             int64_t M, int64_t N, int64_t K, int epilogue, void* stream) {
    using namespace pab::gemm;
    if (M == 0) return PAB_OK;
    if (!C) return PAB_ERR_INVALID;
    const int st = check_args(A, lda, B, ldb, C, ldc, M, N, K);
    if (st != PAB_OK) return st;
    if (epilogue != 0 && epilogue != 1) return PAB_ERR_INVALID;
    return dispatch<0>(A, lda, B, ldb, C, ldc, M, N, K, epilogue, Resid{}, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int pab_gemm_bf16_residual_h(const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                                        int64_t ldc, float* x, int64_t ldx, void* h, int64_t ldh, int64_t h_rows,
                                        int64_t M, int64_t N, int64_t K, int64_t tm_t, int64_t tm_s, void* stream);

extern "C" int pab_gemm_bf16_residual(const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                                      int64_t ldc, float* x, int64_t ldx, int64_t M, int64_t N, int64_t K,
                                      int64_t tm_t, int64_t tm_s, void* stream) {
    return pab_gemm_bf16_residual_h(A, lda, B, ldb, C, ldc, x, ldx, nullptr, 0, 0, M, N, K, tm_t, tm_s, stream);
}

extern "C" int pab_gemm_bf16_residual_h(const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                                        int64_t ldc, float* x, int64_t ldx, void* h, int64_t ldh, int64_t h_rows,
                                        int64_t M, int64_t N, int64_t K, int64_t tm_t, int64_t tm_s, void* stream) {
    using namespace pab::gemm;
    if (M == 0) return PAB_OK;
    const int st = check_args(A, lda, B, ldb, C, ldc, M, N, K);
    if (st != PAB_OK) return st;
    if (!x) return PAB_ERR_INVALID;
    if (ldx < N || (uintptr_t)x % 16 || ldx % 4 || N % 4) return PAB_ERR_UNSUPPORTED;
    if (tm_t < 0 || tm_s < 0 || (tm_t > 0) != (tm_s > 0) || (tm_t > 0 && M % (tm_t * tm_s))) return PAB_ERR_SHAPE;
    // token-major rows: every 128-row block must be whole tokens of one batch entry
    if (tm_t > 0 && (128 % tm_t || (tm_t * tm_s) % 128)) return PAB_ERR_UNSUPPORTED;
    if (h && (ldh < N || (uintptr_t)h % 16 || ldh % 8 || N % 8)) return PAB_ERR_UNSUPPORTED;
    Resid rs;
    rs.x = x;
    rs.ldx = ldx;
    rs.h = reinterpret_cast<__nv_bfloat16*>(h);
    rs.ldh = ldh;
    rs.h_rows = h ? (h_rows < 0 || h_rows > M ? M : h_rows) : 0;
    rs.tm_t = tm_t;
    rs.tm_s = tm_s;
    // deep-K GEMMs (the MLP w2) take the direct read-modify-write epilogue (frame-major rows, no h)
    if (K >= g_direct_k && tm_t == 0 && h == nullptr && N % 8 == 0 && ldx % 8 == 0)
        return dispatch<2>(A, lda, B, ldb, C, ldc, M, N, K, 2, rs, reinterpret_cast<cudaStream_t>(stream));
    return dispatch<1>(A, lda, B, ldb, C, ldc, M, N, K, 2, rs, reinterpret_cast<cudaStream_t>(stream));
}

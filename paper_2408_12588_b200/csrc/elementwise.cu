// HBM-bound kernels of the PAB step: the broadcast epilogue with its
// modulated-LayerNorm prologue (K4+K5), GELU (K7), the fused CFG + DDIM
// update (K8) and the on-device splitmix64 parameter fill.
//
// All of them stream their operands exactly once with 16-byte (fp32x4) /
// 8-byte (bf16x4) vector accesses; one warp owns one row for the row-wise
// LayerNorm so the reduction never leaves registers.
#include "common.cuh"
#include <math.h>

namespace pab {

// --------------------------------------------------------------------------
// K4+K5: x_out = x_in + sum(pending); h = modnorm(x_out) | bf16(x_out)
// reference: model.py:317-324 (_modulated_norm), model.py:503 (x + o),
//            numerics.py:115-130 (layer_norm, population variance, eps)
// --------------------------------------------------------------------------
template <int VEC>
struct VecT;
template <>
struct VecT<4> {
    __device__ static void load_f32(const float* p, float* v) {
        float4 t = *reinterpret_cast<const float4*>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
    __device__ static void store_f32(float* p, const float* v) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
    __device__ static void add_bf16(const __nv_bfloat16* p, float* v) {
        uint2 raw = *reinterpret_cast<const uint2*>(p);
        __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&raw.x);
        __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&raw.y);
        float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
        v[0] += fa.x; v[1] += fa.y; v[2] += fb.x; v[3] += fb.y;
    }
    __device__ static void copy_bf16(const __nv_bfloat16* src, __nv_bfloat16* dst) {
        *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(src);
    }
    __device__ static void store_bf16(__nv_bfloat16* p, const float* v) {
        __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
        __nv_bfloat162 b = __floats2bfloat162_rn(v[2], v[3]);
        uint2 raw;
        raw.x = *reinterpret_cast<uint32_t*>(&a);
        raw.y = *reinterpret_cast<uint32_t*>(&b);
        *reinterpret_cast<uint2*>(p) = raw;
    }
};
template <>
struct VecT<1> {
    __device__ static void load_f32(const float* p, float* v) { v[0] = *p; }
    __device__ static void store_f32(float* p, const float* v) { *p = v[0]; }
    __device__ static void add_bf16(const __nv_bfloat16* p, float* v) { v[0] += __bfloat162float(*p); }
    __device__ static void store_bf16(__nv_bfloat16* p, const float* v) { *p = __float2bfloat16_rn(v[0]); }
    __device__ static void copy_bf16(const __nv_bfloat16* src, __nv_bfloat16* dst) { *dst = *src; }
};

// Optional row permutation of the h output: rows (b, t, s) of a frame-sharded
// (n_b, n_t, n_s) block are written in all-to-all send order
// (dest = s / (n_s / n_w), t, b, s % (n_s / n_w)) so the sequence-parallel
// frames->tokens exchange needs no pack pass.  n_w == 0: identity.  With peer[]
// set (PAB_LAYOUT_PEER), the row goes straight into rank dest's token-layout
// receive buffer (T, B, S/W, D) at ((me * n_t + t) * n_b + b) * (n_s / n_w) + s % (n_s / n_w):
// the prologue's stores ARE the all-to-all, over NVLink peer memory.
struct RowPerm {
    int64_t n_b, n_t, n_s, n_w;  // n_w > 0: all-to-all send order; n_w == -1: token-major (b, s, t)
    int64_t me;                   // this rank (peer mode)
    __nv_bfloat16* peer[PAB_MAX_PEERS];  // peer[0] != nullptr: destination buffers of the W ranks
    __device__ __forceinline__ int64_t map(int64_t row) const {
        if (n_w == 0) return row;
        if (n_w < 0) {
            const int64_t s = row % n_s, bt = row / n_s, t = bt % n_t, b = bt / n_t;
            return (b * n_s + s) * n_t + t;
        }
        const int64_t s = row % n_s, bt = row / n_s, t = bt % n_t, b = bt / n_t;
        const int64_t sw = n_s / n_w, dst = s / sw, sl = s - dst * sw;
        return ((dst * n_t + t) * n_b + b) * sw + sl;
    }
    __device__ __forceinline__ __nv_bfloat16* out_row(__nv_bfloat16* h, int64_t row, int64_t D) const {
        if (n_w > 0 && peer[0] != nullptr) {
            const int64_t s = row % n_s, bt = row / n_s, t = bt % n_t, b = bt / n_t;
            const int64_t sw = n_s / n_w, dst = s / sw, sl = s - dst * sw;
            return peer[dst] + (((me * n_t + t) * n_b + b) * sw + sl) * D;
        }
        return h + map(row) * D;
    }
};

template <int VEC, int NV>
__global__ void __launch_bounds__(256) residual_modnorm_kernel(
    const float* __restrict__ x_in, float* __restrict__ x_out, PendingList pend,
    const float* __restrict__ gamma, const float* __restrict__ beta,
    const float* __restrict__ mod, __nv_bfloat16* __restrict__ h_out,
    int64_t rows, int D, float eps, int mode, int write_x, RowPerm perm) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int64_t base = row * (int64_t)D;
    float v[NV][VEC];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = (j * 32 + lane) * VEC;
        if (c < D) {
            VecT<VEC>::load_f32(x_in + base + c, v[j]);
#pragma unroll
            for (int p = 0; p < PAB_MAX_PENDING; ++p)
                if (p < pend.n) {
                    const __nv_bfloat16* src = pend.row_ptr(p, row, D) + c;
                    VecT<VEC>::add_bf16(src, v[j]);
                    if (p == pend.copy_term) VecT<VEC>::copy_bf16(src, pend.copy + base + c);
                }
            if (write_x) VecT<VEC>::store_f32(x_out + base + c, v[j]);
        }
    }
    if (mode == 0) return;
    __nv_bfloat16* hrow = perm.out_row(h_out, row, D);
    if (mode == 2) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int c = (j * 32 + lane) * VEC;
            if (c < D) VecT<VEC>::store_bf16(hrow + c, v[j]);
        }
        return;
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = (j * 32 + lane) * VEC;
        if (c < D) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) s += v[j][e];
        }
    }
    const float mean = warp_sum(s) / (float)D;
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = (j * 32 + lane) * VEC;
        if (c < D) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                v[j][e] -= mean;
                q += v[j][e] * v[j][e];
            }
        }
    }
    const float var = warp_sum(q) / (float)D;
    const float inv = 1.0f / sqrtf(var + eps);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = (j * 32 + lane) * VEC;
        if (c < D) {
            float o[VEC];
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                float h = v[j][e] * inv;
                if (gamma) h = h * gamma[c + e] + beta[c + e];
                o[e] = h * (1.0f + mod[D + c + e]) + mod[c + e];
            }
            VecT<VEC>::store_bf16(hrow + c, o);
        }
    }
}

// Exact-width variant (D == 128 * NV): no per-element guards, every load of the
// row (x and all pending terms) issued before any arithmetic, streaming cache
// hints (each byte is touched once).  One warp per row.
template <int NV>
__global__ void __launch_bounds__(256) residual_modnorm_exact_kernel(
    const float* __restrict__ x_in, float* __restrict__ x_out, PendingList pend,
    const float* __restrict__ gamma, const float* __restrict__ beta,
    const float* __restrict__ mod, __nv_bfloat16* __restrict__ h_out,
    int64_t rows, float eps, int mode, int write_x, RowPerm perm) {
    constexpr int D = 128 * NV;
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int64_t base = row * (int64_t)D;
    float4 v[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = __ldcs(reinterpret_cast<const float4*>(x_in + base) + j * 32 + lane);
#pragma unroll
    for (int p = 0; p < PAB_MAX_PENDING; ++p) {
        if (p < pend.n) {
            uint2 raw[NV];
            const uint2* src = reinterpret_cast<const uint2*>(pend.row_ptr(p, row, D));
#pragma unroll
            for (int j = 0; j < NV; ++j) raw[j] = __ldcs(src + j * 32 + lane);
            if (p == pend.copy_term) {
#pragma unroll
                for (int j = 0; j < NV; ++j) __stcs(reinterpret_cast<uint2*>(pend.copy + base) + j * 32 + lane, raw[j]);
            }
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&raw[j].x));
                const float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&raw[j].y));
                v[j].x += a.x; v[j].y += a.y; v[j].z += b.x; v[j].w += b.y;
            }
        }
    }
    if (write_x) {
#pragma unroll
        for (int j = 0; j < NV; ++j) __stcs(reinterpret_cast<float4*>(x_out + base) + j * 32 + lane, v[j]);
    }
    if (mode == 0) return;
    __nv_bfloat16* hrow = perm.out_row(h_out, row, D);
    auto store_h = [&](int j, float a, float b, float c, float d) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
        uint2 raw;
        raw.x = *reinterpret_cast<uint32_t*>(&lo);
        raw.y = *reinterpret_cast<uint32_t*>(&hi);
        __stcs(reinterpret_cast<uint2*>(hrow) + j * 32 + lane, raw);
    };
    if (mode == 2) {
#pragma unroll
        for (int j = 0; j < NV; ++j) store_h(j, v[j].x, v[j].y, v[j].z, v[j].w);
        return;
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    const float mean = warp_sum(s) * (1.0f / (float)D);
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        v[j].x -= mean; v[j].y -= mean; v[j].z -= mean; v[j].w -= mean;
        q += (v[j].x * v[j].x + v[j].y * v[j].y) + (v[j].z * v[j].z + v[j].w * v[j].w);
    }
    const float inv = 1.0f / sqrtf(warp_sum(q) * (1.0f / (float)D) + eps);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = (j * 32 + lane) * 4;
        const float4 sh = __ldg(reinterpret_cast<const float4*>(mod + c));
        const float4 sc = __ldg(reinterpret_cast<const float4*>(mod + D + c));
        float4 hv = make_float4(v[j].x * inv, v[j].y * inv, v[j].z * inv, v[j].w * inv);
        if (gamma) {
            const float4 g = __ldg(reinterpret_cast<const float4*>(gamma + c));
            const float4 bb = __ldg(reinterpret_cast<const float4*>(beta + c));
            hv = make_float4(hv.x * g.x + bb.x, hv.y * g.y + bb.y, hv.z * g.z + bb.z, hv.w * g.w + bb.w);
        }
        store_h(j, hv.x * (1.0f + sc.x) + sh.x, hv.y * (1.0f + sc.y) + sh.y, hv.z * (1.0f + sc.z) + sh.z,
                hv.w * (1.0f + sc.w) + sh.w);
    }
}

template <int VEC>
static int launch_modnorm_vec(const float* x_in, float* x_out, const PendingList& pl,
                              const float* gamma, const float* beta, const float* mod,
                              __nv_bfloat16* h, int64_t rows, int D, float eps, int mode,
                              int write_x, RowPerm perm, cudaStream_t st) {
    const int per_lane = (D + 32 * VEC - 1) / (32 * VEC);
    const int warps = 8;
    dim3 grid((unsigned)((rows + warps - 1) / warps)), block(32 * warps);
    if (VEC == 4 && D % 128 == 0 && (mod == nullptr || (uintptr_t)mod % 16 == 0)) {
#define PAB_MNX(NVV)                                                                                       \
    residual_modnorm_exact_kernel<NVV><<<grid, block, 0, st>>>(x_in, x_out, pl, gamma, beta, mod, h, rows, eps, \
                                                                mode, write_x, perm)
        switch (D / 128) {
            case 1: PAB_MNX(1); return launch_status("residual_modnorm");
            case 2: PAB_MNX(2); return launch_status("residual_modnorm");
            case 4: PAB_MNX(4); return launch_status("residual_modnorm");
            case 8: PAB_MNX(8); return launch_status("residual_modnorm");
            case 9: PAB_MNX(9); return launch_status("residual_modnorm");
            case 12: PAB_MNX(12); return launch_status("residual_modnorm");
            default: break;
        }
#undef PAB_MNX
    }
#define PAB_MN(NVV)                                                                       \
    residual_modnorm_kernel<VEC, NVV><<<grid, block, 0, st>>>(x_in, x_out, pl, gamma, beta, \
                                                              mod, h, rows, D, eps, mode, write_x, perm)
    if (per_lane <= 1) PAB_MN(1);
    else if (per_lane <= 2) PAB_MN(2);
    else if (per_lane <= 4) PAB_MN(4);
    else if (per_lane <= 8) PAB_MN(8);
    else if (per_lane <= 9) PAB_MN(9);
    else if (per_lane <= 12) PAB_MN(12);
    else if (per_lane <= 16) PAB_MN(16);
    else return PAB_ERR_UNSUPPORTED;
#undef PAB_MN
    return launch_status("residual_modnorm");
}

// --------------------------------------------------------------------------
// K8: end-of-step drain + CFG + DDIM (diffusion.py:100-103, 183-189)
// --------------------------------------------------------------------------
// the per-element fp32 op sequence of numpy (eps accumulation in order, CFG, DDIM)
__device__ __forceinline__ void ddim_cfg_elem(float* eps, const float* zin, float* zout, int batch, int guidance,
                                              float g, float c_noise, float c_signal, float c_next_sig,
                                              float c_next_noise) {
    if (guidance) {
        // eps_u + g * (eps_c - eps_u), conditional half first (diffusion.py:183-186)
        const float eh = __fadd_rn(eps[1], __fmul_rn(g, __fsub_rn(eps[0], eps[1])));
#pragma unroll
        for (int b = 0; b < 8; ++b) eps[b] = eh;
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        if (b >= batch) break;
        const float x0 = __fdiv_rn(__fsub_rn(zin[b], __fmul_rn(c_noise, eps[b])), c_signal);
        zout[b] = __fadd_rn(__fmul_rn(c_next_sig, x0), __fmul_rn(c_next_noise, eps[b]));
    }
}

// VEC consecutive elements per thread (4: one float4 of z / r and 8 bytes of each bf16
// pending term per batch row; 1: scalar, for unaligned or ragged n)
template <int VEC>
__global__ void __launch_bounds__(256) ddim_cfg_kernel(
    float* __restrict__ z, const float* __restrict__ r, PendingList pend, int batch,
    int64_t n, int guidance, float g, float c_noise, float c_signal, float c_next_sig,
    float c_next_noise) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC;
    if (i >= n) return;
    float eps[VEC][8], zv[VEC][8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        if (b >= batch) break;
        const int64_t k = (int64_t)b * n + i;
        float rv[VEC], zz[VEC];
        VecT<VEC>::load_f32(r + k, rv);
        VecT<VEC>::load_f32(z + k, zz);
#pragma unroll
        for (int p = 0; p < PAB_MAX_PENDING; ++p) {
            if (p < pend.n) {
                float o[VEC] = {};
                VecT<VEC>::add_bf16(pend.p[p] + k, o);
#pragma unroll
                for (int e = 0; e < VEC; ++e) rv[e] = __fadd_rn(rv[e], o[e]);
            }
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
            eps[e][b] = rv[e];
            zv[e][b] = zz[e];
        }
    }
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
        float out[8];
        ddim_cfg_elem(eps[e], zv[e], out, batch, guidance, g, c_noise, c_signal, c_next_sig, c_next_noise);
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (b < batch) zv[e][b] = out[b];
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        if (b >= batch) break;
        float zz[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) zz[e] = zv[e][b];
        VecT<VEC>::store_f32(z + (int64_t)b * n + i, zz);
    }
}

// --------------------------------------------------------------------------
// K7: tanh-approximate GELU, bf16 in/out, 8 elements per thread
// --------------------------------------------------------------------------
__device__ __forceinline__ float gelu_tanh(float x) {
    const float k0 = 0.7978845608028654f;  // sqrt(2/pi)
    const float inner = k0 * (x + 0.044715f * (x * x * x));
    // tanh(u) = 1 - 2 / (exp(2u) + 1); exact to ~1e-7 relative, far below bf16 output rounding
    const float t = 1.0f - __fdividef(2.0f, __expf(2.0f * inner) + 1.0f);
    return 0.5f * x * (1.0f + t);
}

__global__ void __launch_bounds__(256) gelu_kernel(const __nv_bfloat16* __restrict__ in,
                                                   __nv_bfloat16* __restrict__ out, int64_t n) {
    const int64_t i8 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (i8 + 8 <= n) {
        uint4 raw = *reinterpret_cast<const uint4*>(in + i8);
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 f = __bfloat1622float2(h[j]);
            h[j] = __floats2bfloat162_rn(gelu_tanh(f.x), gelu_tanh(f.y));
        }
        *reinterpret_cast<uint4*>(out + i8) = raw;
    } else {
        for (int64_t i = i8; i < n; ++i) out[i] = __float2bfloat16_rn(gelu_tanh(__bfloat162float(in[i])));
    }
}

// --------------------------------------------------------------------------
// splitmix64 fill (numerics.py:161-201; model.py:176-182)
// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix_out(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void fill_uniform_kernel(void* dst, int dtype, int64_t rows, int64_t cols, int64_t ld,
                                    int64_t col0, uint64_t state, uint64_t first, double lo,
                                    double span) {
    const int64_t total = rows * cols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = first + (uint64_t)i + 1ull;
        const uint64_t mant = splitmix_out(state + k * 0x9E3779B97F4A7C15ull) >> 11;
        const double u = (double)mant * 1.1102230246251565e-16;  // 2^-53, exact
        const float v = __double2float_rn(__dadd_rn(lo, __dmul_rn(u, span)));
        const int64_t r = i / cols, c = i - r * cols;
        const int64_t o = r * ld + col0 + c;
        if (dtype == 0) reinterpret_cast<float*>(dst)[o] = v;
        else reinterpret_cast<__nv_bfloat16*>(dst)[o] = __float2bfloat16_rn(v);
    }
}

}  // namespace pab

using namespace pab;

// source layouts of the pending terms: bit i of `mask` -> term i token-major (b, s, t),
// bit i of `a2a` -> term i in all-to-all order over n_w ranks
struct TmState {
    uint32_t mask;
    int64_t t, s;
    uint32_t a2a = 0;
    int64_t n_b = 1, n_w = 1;
    uint32_t peer = 0;                    // bit i: term i is PAB_LAYOUT_PEER
    int64_t me = 0;                       // this rank (peer terms / peer h output)
    const void* const* peer_src = nullptr;  // n_w token-layout source buffers of the PEER term
    void* copy = nullptr;                 // frame-major copy of the PEER term (cache slot) or NULL
};
static int residual_modnorm_impl(const float* x_in, float* x_out, const void* const* pending,
                                 int n_pending, const float* gamma, const float* beta,
                                 const float* mod, void* h_out, int64_t rows, int D, float eps,
                                 int mode, RowPerm perm, TmState tm, void* stream);

extern "C" int pab_residual_modnorm(const float* x_in, float* x_out, const void* const* pending,
                                    int n_pending, const float* gamma, const float* beta,
                                    const float* mod, void* h_out, int64_t rows, int D, float eps,
                                    int mode, void* stream) {
    return residual_modnorm_impl(x_in, x_out, pending, n_pending, gamma, beta, mod, h_out, rows, D, eps, mode,
                                 RowPerm{0, 0, 0, 0}, TmState{0u, 1, 1}, stream);
}

extern "C" int pab_residual_modnorm_sp(const float* x_in, float* x_out, const void* const* pending,
                                       int n_pending, const float* gamma, const float* beta,
                                       const float* mod, void* h_out, int64_t n_b, int64_t n_t,
                                       int64_t n_s, int64_t n_w, int D, float eps, int mode, void* stream) {
    if (n_b < 1 || n_t < 1 || n_s < 1 || n_w < 1 || n_s % n_w != 0) return PAB_ERR_SHAPE;
    if (mode == 0) return PAB_ERR_INVALID;
    return residual_modnorm_impl(x_in, x_out, pending, n_pending, gamma, beta, mod, h_out, n_b * n_t * n_s, D,
                                 eps, mode, RowPerm{n_b, n_t, n_s, n_w}, TmState{0u, 1, 1}, stream);
}

extern "C" int pab_residual_modnorm_tm(const float* x_in, float* x_out, const void* const* pending,
                                       int n_pending, uint32_t pending_tm_mask, const float* gamma,
                                       const float* beta, const float* mod, void* h_out, int64_t n_b,
                                       int64_t n_t, int64_t n_s, int D, float eps, int mode, int h_token_major,
                                       void* stream) {
    if (n_b < 1 || n_t < 1 || n_s < 1) return PAB_ERR_SHAPE;
    if (n_pending < 0 || n_pending > PAB_MAX_PENDING) return PAB_ERR_SHAPE;
    const int64_t rows = n_b * n_t * n_s;
    const TmState tm{pending_tm_mask & ((1u << n_pending) - 1u), n_t, n_s};
    return residual_modnorm_impl(x_in, x_out, pending, n_pending, gamma, beta, mod, h_out, rows, D, eps, mode,
                                 RowPerm{n_b, n_t, n_s, h_token_major ? -1 : 0}, tm, stream);
}

extern "C" int pab_residual_modnorm_peer(const float* x_in, float* x_out, const void* const* pending,
                                         const int* term_layout, int n_pending, const void* const* peer_src,
                                         void* peer_copy, const float* gamma, const float* beta,
                                         const float* mod, void* h_out, void* const* peer_h, int64_t n_b,
                                         int64_t n_t, int64_t n_s, int64_t n_w, int rank, int D, float eps,
                                         int mode, int h_layout, void* stream) {
    if (n_b < 1 || n_t < 1 || n_s < 1 || n_w < 1) return PAB_ERR_SHAPE;
    if (n_pending < 0 || n_pending > PAB_MAX_PENDING) return PAB_ERR_SHAPE;
    if (rank < 0 || rank >= n_w) return PAB_ERR_INVALID;
    TmState tm{0u, n_t, n_s};
    tm.n_b = n_b;
    tm.n_w = n_w;
    tm.me = rank;
    tm.peer_src = peer_src;
    tm.copy = peer_copy;
    bool a2a = h_layout == PAB_LAYOUT_A2A || h_layout == PAB_LAYOUT_PEER;
    int n_peer = 0;
    for (int i = 0; i < n_pending; ++i) {
        const int l = term_layout ? term_layout[i] : PAB_LAYOUT_FRAME;
        if (l == PAB_LAYOUT_TOKEN) tm.mask |= 1u << i;
        else if (l == PAB_LAYOUT_A2A) { tm.a2a |= 1u << i; a2a = true; }
        else if (l == PAB_LAYOUT_PEER) { tm.peer |= 1u << i; a2a = true; ++n_peer; }
        else if (l != PAB_LAYOUT_FRAME) return PAB_ERR_INVALID;
    }
    // one peer-resident term per launch (the temporal output of the preceding site); the peer
    // forms address at most PAB_MAX_PEERS ranks (the all-to-all orders take any n_w)
    if ((n_peer > 0 || h_layout == PAB_LAYOUT_PEER) && n_w > PAB_MAX_PEERS) return PAB_ERR_SHAPE;
    if (n_peer > 1 || (n_peer == 1 && peer_src == nullptr)) return PAB_ERR_INVALID;
    if (peer_copy != nullptr && n_peer != 1) return PAB_ERR_INVALID;
    if (n_peer == 1)
        for (int w = 0; w < n_w; ++w)
            if (peer_src[w] == nullptr) return PAB_ERR_INVALID;
    if (a2a && n_s % n_w != 0) return PAB_ERR_SHAPE;
    if (h_layout < PAB_LAYOUT_FRAME || h_layout > PAB_LAYOUT_PEER) return PAB_ERR_INVALID;
    if ((h_layout == PAB_LAYOUT_A2A || h_layout == PAB_LAYOUT_PEER) && mode == 0) return PAB_ERR_INVALID;
    RowPerm perm{n_b, n_t, n_s,
                 (h_layout == PAB_LAYOUT_A2A || h_layout == PAB_LAYOUT_PEER) ? n_w
                                                                             : (h_layout == PAB_LAYOUT_TOKEN ? -1 : 0)};
    perm.me = rank;
    if (h_layout == PAB_LAYOUT_PEER) {
        if (peer_h == nullptr) return PAB_ERR_INVALID;
        for (int w = 0; w < n_w; ++w) {
            if (peer_h[w] == nullptr) return PAB_ERR_INVALID;
            perm.peer[w] = reinterpret_cast<__nv_bfloat16*>(peer_h[w]);
        }
    }
    return residual_modnorm_impl(x_in, x_out, pending, n_pending, gamma, beta, mod, h_out, n_b * n_t * n_s, D, eps,
                                 mode, perm, tm, stream);
}

extern "C" int pab_residual_modnorm_ex(const float* x_in, float* x_out, const void* const* pending,
                                       const int* term_layout, int n_pending, const float* gamma,
                                       const float* beta, const float* mod, void* h_out, int64_t n_b,
                                       int64_t n_t, int64_t n_s, int64_t n_w, int D, float eps, int mode,
                                       int h_layout, void* stream) {
    if (h_layout == PAB_LAYOUT_PEER) return PAB_ERR_INVALID;
    for (int i = 0; term_layout && i < n_pending; ++i)
        if (term_layout[i] == PAB_LAYOUT_PEER) return PAB_ERR_INVALID;
    return pab_residual_modnorm_peer(x_in, x_out, pending, term_layout, n_pending, nullptr, nullptr, gamma, beta,
                                     mod, h_out, nullptr, n_b, n_t, n_s, n_w, 0, D, eps, mode, h_layout, stream);
}

static int residual_modnorm_impl(const float* x_in, float* x_out, const void* const* pending,
                                 int n_pending, const float* gamma, const float* beta,
                                 const float* mod, void* h_out, int64_t rows, int D, float eps,
                                 int mode, RowPerm perm, TmState tm, void* stream) {
    if (rows < 0 || D <= 0 || n_pending < 0 || n_pending > PAB_MAX_PENDING) return PAB_ERR_SHAPE;
    if (mode < 0 || mode > 2) return PAB_ERR_INVALID;
    if (mode == 1 && mod == nullptr) return PAB_ERR_INVALID;
    const bool peer_h = perm.n_w > 0 && perm.peer[0] != nullptr;
    if (mode != 0 && h_out == nullptr && !peer_h) return PAB_ERR_INVALID;
    if ((gamma == nullptr) != (beta == nullptr)) return PAB_ERR_INVALID;
    if (rows == 0) return PAB_OK;
    const int write_x = (n_pending > 0 || x_in != x_out) ? 1 : 0;
    // a permuted h cannot be produced in place of a plain cast/LN row order mismatch
    if (perm.n_w != 0 && mode == 0) return PAB_ERR_INVALID;
    if (mode == 0 && !write_x) return PAB_OK;
    PendingList pl = make_pending(pending, n_pending);
    pl.tm_mask = tm.mask;
    pl.a2a_mask = tm.a2a;
    pl.tm_t = tm.t;
    pl.tm_s = tm.s;
    pl.n_b = tm.n_b;
    pl.n_w = tm.n_w;
    pl.peer_mask = tm.peer;
    pl.me = tm.me;
    if (tm.peer) {
        for (int w = 0; w < tm.n_w; ++w) pl.peer[w] = reinterpret_cast<const __nv_bfloat16*>(tm.peer_src[w]);
        if (tm.copy) {
            pl.copy = reinterpret_cast<__nv_bfloat16*>(tm.copy);
            for (int i = 0; i < n_pending; ++i)
                if (tm.peer & (1u << i)) pl.copy_term = i;
        }
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    auto* h = reinterpret_cast<__nv_bfloat16*>(h_out);
    bool aligned = (D % 4 == 0) && ((uintptr_t)x_in % 16 == 0) && ((uintptr_t)x_out % 16 == 0) &&
                   (h == nullptr || (uintptr_t)h % 8 == 0);
    for (int i = 0; i < n_pending; ++i)
        aligned = aligned && ((tm.peer >> i) & 1u ? true : (uintptr_t)pending[i] % 8 == 0);
    for (int w = 0; w < PAB_MAX_PEERS; ++w)
        aligned = aligned && (uintptr_t)pl.peer[w] % 8 == 0 && (uintptr_t)perm.peer[w] % 8 == 0;
    aligned = aligned && (uintptr_t)pl.copy % 8 == 0;
    if (aligned)
        return launch_modnorm_vec<4>(x_in, x_out, pl, gamma, beta, mod, h, rows, D, eps, mode, write_x, perm, st);
    return launch_modnorm_vec<1>(x_in, x_out, pl, gamma, beta, mod, h, rows, D, eps, mode, write_x, perm, st);
}

extern "C" int pab_ddim_cfg(float* z, const float* r, const void* const* pending, int n_pending,
                            int batch, int64_t n, int guidance, double guidance_scale,
                            double a_cur, double a_next, void* stream) {
    if (batch < 1 || batch > 8 || n < 0 || n_pending < 0 || n_pending > PAB_MAX_PENDING) return PAB_ERR_SHAPE;
    if (guidance && batch != 2) return PAB_ERR_SHAPE;
    if (!(a_cur > 0.0) || a_cur > 1.0 || a_next < 0.0 || a_next > 1.0) return PAB_ERR_INVALID;
    if (n == 0) return PAB_OK;
    PendingList pl = make_pending(pending, n_pending);
    const float c_noise = (float)sqrt(1.0 - a_cur), c_signal = (float)sqrt(a_cur);
    const float c_next_sig = (float)sqrt(a_next), c_next_noise = (float)sqrt(1.0 - a_next);
    bool vec = n % 4 == 0 && (uintptr_t)z % 16 == 0 && (uintptr_t)r % 16 == 0;
    for (int i = 0; i < n_pending; ++i) vec = vec && (uintptr_t)pending[i] % 8 == 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (vec) {
        dim3 block(256), grid((unsigned)((n / 4 + 255) / 256));
        ddim_cfg_kernel<4><<<grid, block, 0, st>>>(z, r, pl, batch, n, guidance, (float)guidance_scale, c_noise,
                                                    c_signal, c_next_sig, c_next_noise);
    } else {
        dim3 block(256), grid((unsigned)((n + 255) / 256));
        ddim_cfg_kernel<1><<<grid, block, 0, st>>>(z, r, pl, batch, n, guidance, (float)guidance_scale, c_noise,
                                                    c_signal, c_next_sig, c_next_noise);
    }
    return launch_status("ddim_cfg");
}

// --------------------------------------------------------------------------
// K10: row softmax of fp32 logits -> bf16 probabilities (score broadcast capture).
// One warp per row, three passes over the row (L2-resident for rows <= 3600):
// max of the scaled logits, sum of exp, normalised store.  expf / division in
// fp32 as numpy's softmax_rows (numerics.py:107-112).
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) softmax_rows_kernel(const float* __restrict__ l, int64_t ld_l,
                                                           __nv_bfloat16* __restrict__ p, int64_t ld_p,
                                                           int64_t rows, int64_t n, float scale) {
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float* x = l + row * ld_l;
    float m = -INFINITY;
    for (int64_t j = lane; j < n; j += 32) m = fmaxf(m, x[j] * scale);
    m = warp_max(m);
    float sum = 0.f;
    for (int64_t j = lane; j < n; j += 32) sum += expf(x[j] * scale - m);
    sum = warp_sum(sum);
    const float inv = 1.0f / sum;
    __nv_bfloat16* y = p + row * ld_p;
    for (int64_t j = lane; j < n; j += 32) y[j] = __float2bfloat16_rn(expf(x[j] * scale - m) * inv);
}

extern "C" int pab_softmax_rows(const float* logits, int64_t ld_l, void* p_bf16, int64_t ld_p, int64_t rows,
                                int64_t n, float scale, void* stream) {
    if (rows < 0 || n < 0 || ld_l < n || ld_p < n) return PAB_ERR_SHAPE;
    if (rows == 0 || n == 0) return PAB_OK;
    if (!logits || !p_bf16) return PAB_ERR_INVALID;
    const int64_t blocks = (rows + 7) / 8;
    if (blocks > 0x7fffffff) return PAB_ERR_UNSUPPORTED;
    softmax_rows_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        logits, ld_l, reinterpret_cast<__nv_bfloat16*>(p_bf16), ld_p, rows, n, scale);
    return launch_status("softmax_rows");
}

// y = x + a * w (fp32, 4 elements per thread): the Delta-DiT whole-layer residual
// delta in fp32 (store: d = x_layer_out - x_layer_in, a = -1; replay: x += d, a = 1)
__global__ void __launch_bounds__(256) add_scaled_f32_kernel(float* __restrict__ y, const float* __restrict__ x,
                                                             const float* __restrict__ w, float a, int64_t n) {
    const int64_t i4 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i4 + 4 <= n) {
        const float4 xv = *reinterpret_cast<const float4*>(x + i4);
        const float4 wv = *reinterpret_cast<const float4*>(w + i4);
        *reinterpret_cast<float4*>(y + i4) =
            make_float4(__fmaf_rn(a, wv.x, xv.x), __fmaf_rn(a, wv.y, xv.y), __fmaf_rn(a, wv.z, xv.z),
                        __fmaf_rn(a, wv.w, xv.w));
    } else {
        for (int64_t i = i4; i < n; ++i) y[i] = __fmaf_rn(a, w[i], x[i]);
    }
}

extern "C" int pab_add_scaled_f32(float* y, const float* x, const float* w, float a, int64_t n, void* stream) {
    if (n < 0) return PAB_ERR_SHAPE;
    if (n == 0) return PAB_OK;
    if (!y || !x || !w) return PAB_ERR_INVALID;
    if ((uintptr_t)y % 16 || (uintptr_t)x % 16 || (uintptr_t)w % 16) return PAB_ERR_UNSUPPORTED;
    const int64_t threads = (n + 3) / 4;
    add_scaled_f32_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        y, x, w, a, n);
    return launch_status("add_scaled_f32");
}

// Redundancy scan on the device (reference profiler.diff_metric / redundancy_scan,
// pkg/src/pab_engine/profiler.py:60-81, 140-173): the four sums every metric needs,
// sum (a-b)^2, sum a^2, sum b^2, sum a*b, over two bf16 site outputs, accumulated in
// fp64 (8 elements per thread in fp32, then fp64 warp / block / grid reductions).
__global__ void __launch_bounds__(256) diff_sums_kernel(const __nv_bfloat16* __restrict__ a,
                                                        const __nv_bfloat16* __restrict__ b, int64_t n,
                                                        double* __restrict__ out) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < n; i += stride) {
        float f[4] = {0.f, 0.f, 0.f, 0.f};
        if (i + 8 <= n) {
            const uint4 ra = __ldg(reinterpret_cast<const uint4*>(a + i));
            const uint4 rb = __ldg(reinterpret_cast<const uint4*>(b + i));
            const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&ra);
            const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&rb);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 x = __bfloat1622float2(ha[j]), y = __bfloat1622float2(hb[j]);
                f[0] += (x.x - y.x) * (x.x - y.x) + (x.y - y.y) * (x.y - y.y);
                f[1] += x.x * x.x + x.y * x.y;
                f[2] += y.x * y.x + y.y * y.y;
                f[3] += x.x * y.x + x.y * y.y;
            }
        } else {
            for (int64_t k = i; k < n; ++k) {
                const float x = __bfloat162float(a[k]), y = __bfloat162float(b[k]);
                f[0] += (x - y) * (x - y);
                f[1] += x * x;
                f[2] += y * y;
                f[3] += x * y;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] += (double)f[k];
    }
    __shared__ double red[8][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][k] = acc[k];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
        atomicAdd(out + threadIdx.x, s);
    }
}

extern "C" int pab_diff_sums(const void* a, const void* b, int64_t n, double* out4, void* stream) {
    if (n < 0) return PAB_ERR_SHAPE;
    if (!a || !b || !out4) return PAB_ERR_INVALID;
    if ((uintptr_t)a % 16 || (uintptr_t)b % 16 || (uintptr_t)out4 % 8) return PAB_ERR_UNSUPPORTED;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(out4, 0, 4 * sizeof(double), st) != cudaSuccess) return launch_status("diff_sums memset");
    if (n == 0) return PAB_OK;
    int64_t blocks = (n + 256 * 8 - 1) / (256 * 8);
    if (blocks > 148 * 8) blocks = 148 * 8;
    diff_sums_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(a),
                                                        reinterpret_cast<const __nv_bfloat16*>(b), n, out4);
    return launch_status("diff_sums");
}

extern "C" int pab_gelu_bf16(const void* in, void* out, int64_t n, void* stream) {
    if (n < 0) return PAB_ERR_SHAPE;
    if (n == 0) return PAB_OK;
    if ((uintptr_t)in % 16 || (uintptr_t)out % 16) return PAB_ERR_UNSUPPORTED;
    const int64_t threads = (n + 7) / 8;
    dim3 block(256), grid((unsigned)((threads + 255) / 256));
    gelu_kernel<<<grid, block, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const __nv_bfloat16*>(in), reinterpret_cast<__nv_bfloat16*>(out), n);
    return launch_status("gelu");
}

extern "C" int pab_fill_uniform(void* dst, int dtype, int64_t rows, int64_t cols, int64_t ld,
                                int64_t col0, uint64_t state, uint64_t first_draw, double lo,
                                double hi, void* stream) {
    if (rows < 0 || cols < 0 || ld < col0 + cols || (dtype != 0 && dtype != 1)) return PAB_ERR_SHAPE;
    if (!(lo < hi)) return PAB_ERR_INVALID;
    if (rows * cols == 0) return PAB_OK;
    const int64_t total = rows * cols;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    fill_uniform_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        dst, dtype, rows, cols, ld, col0, state, first_draw, lo, hi - lo);
    return launch_status("fill_uniform");
}

/*
 * pab_b200.h -- C ABI of the B200-native Pyramid Attention Broadcast hot path.
 *
 * Every entry point takes plain device pointers, element counts/strides and a
 * cudaStream_t passed as void*; the library never allocates or frees device
 * memory (the caller -- PyTorch in this repo -- owns every buffer) and never
 * throws across the ABI.  Calls are asynchronous on `stream` and capturable
 * into CUDA graphs.  Return value: 0 on success, else a PAB_ERR_* code that
 * the Python wrapper maps back onto the reference's EngineError kinds
 * (reference pkg/src/pab_engine/errors.py:4-40).
 *
 * The reference (pab-engine) is pure Python/numpy; its "operator API" is the
 * set of module functions the denoising loop calls.  Each entry point below
 * names the reference function(s) it replaces.
 */
#ifndef PAB_B200_H
#define PAB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PAB_OK 0
#define PAB_ERR_SHAPE 1       /* reference ShapeError   "shape-mismatch" */
#define PAB_ERR_INVALID 2     /* reference ValidationError "invalid-config" */
#define PAB_ERR_POLICY 3      /* reference PolicyError  "policy-error" */
#define PAB_ERR_CUDA 4        /* CUDA / driver failure (DeviceError) */
#define PAB_ERR_UNSUPPORTED 5 /* shape outside what a kernel supports */

#define PAB_MAX_PENDING 8     /* pending residual terms per launch */
#define PAB_MAX_PEERS 8       /* ranks of a sequence-parallel group on one NVSwitch box */

/* Library metadata. */
const char* pab_version(void);
const char* pab_status_string(int status);
/* Last CUDA error string recorded by a failing call (thread-local). */
const char* pab_last_error(void);

/*
 * Broadcast epilogue + modulated-norm prologue (kernels K4+K5).
 * Replaces: model.run_site's `x + o` residual add for computed AND reused
 * sites (pkg/src/pab_engine/model.py:469-503), `_modulated_norm`
 * (model.py:317-324) and `layer_norm` (numerics.py:115-130).
 *
 *   x_out[r, :] = x_in[r, :] + pending[0][r, :] + ... + pending[n-1][r, :]   (fp32, in order)
 *   mode 0: no h output
 *   mode 1: h = bf16( (LN(x_out) * gamma + beta) * (1 + mod[D:2D]) + mod[0:D] )
 *   mode 2: h = bf16( x_out )   (cross-attention query input, no norm)
 * x_in may equal x_out.  pending[i] are bf16 (rows, D) row-major.
 * gamma/beta may be NULL (identity affine).  n_pending <= PAB_MAX_PENDING.
 */
int pab_residual_modnorm(const float* x_in, float* x_out,
                         const void* const* pending, int n_pending,
                         const float* gamma, const float* beta,
                         const float* mod, void* h_out,
                         int64_t rows, int D, float eps, int mode, void* stream);

/*
 * Sequence-parallel variant of pab_residual_modnorm (mode 1 or 2): the input
 * is this rank's frame shard, rows ordered (b < n_b, t < n_t, s < n_s); x_out
 * keeps that order but h row (b, t, s) is written at send-order position
 *   ((s / (n_s/n_w)) * n_t + t) * n_b + b) * (n_s/n_w) + s % (n_s/n_w)
 * i.e. grouped by destination rank, so the frames->tokens all-to-all of the
 * temporal site (reference parallel.reshard, pkg/src/pab_engine/parallel.py:
 * 140-180, 324-326) sends h with no pack pass.  n_s % n_w == 0.
 */
int pab_residual_modnorm_sp(const float* x_in, float* x_out,
                            const void* const* pending, int n_pending,
                            const float* gamma, const float* beta,
                            const float* mod, void* h_out,
                            int64_t n_b, int64_t n_t, int64_t n_s, int64_t n_w,
                            int D, float eps, int mode, void* stream);

/*
 * Token-major variant used around the temporal site (kernel K2's layout):
 * the residual stream is (n_b, n_t, n_s, D) frame-major; pending term i is
 * read token-major (rows (b, s, t)) when bit i of pending_tm_mask is set, and
 * h is written token-major when h_token_major != 0.  With the temporal
 * site's QKV rows token-major, each token's T frames are contiguous rows, so
 * temporal attention reads contiguous 128-row boxes instead of gathering
 * frames S rows apart.  Otherwise identical to pab_residual_modnorm.
 */
int pab_residual_modnorm_tm(const float* x_in, float* x_out,
                            const void* const* pending, int n_pending, uint32_t pending_tm_mask,
                            const float* gamma, const float* beta,
                            const float* mod, void* h_out,
                            int64_t n_b, int64_t n_t, int64_t n_s,
                            int D, float eps, int mode, int h_token_major, void* stream);

/*
 * General form of the three prologues above (they are special cases of it): every
 * pending term and the h output carry a row layout over the (n_b, n_t, n_s) block of
 * the residual stream:
 *   PAB_LAYOUT_FRAME  rows (b, t, s)                          the stream's own order
 *   PAB_LAYOUT_TOKEN  rows (b, s, t)                          the temporal site's order
 *   PAB_LAYOUT_A2A    rows (s / (n_s/n_w), t, b, s % (n_s/n_w)) a frame shard in the
 *                     sequence-parallel all-to-all order (n_s % n_w == 0)
 * so the temporal site's received output is added by the next prologue straight from
 * the all-to-all receive buffer (no unpack pass; reference parallel.reshard,
 * pkg/src/pab_engine/parallel.py:140-180, 335-340).  term_layout may be NULL (all FRAME).
 */
#define PAB_LAYOUT_FRAME 0
#define PAB_LAYOUT_TOKEN 1
#define PAB_LAYOUT_A2A 2
int pab_residual_modnorm_ex(const float* x_in, float* x_out,
                            const void* const* pending, const int* term_layout, int n_pending,
                            const float* gamma, const float* beta,
                            const float* mod, void* h_out,
                            int64_t n_b, int64_t n_t, int64_t n_s, int64_t n_w,
                            int D, float eps, int mode, int h_layout, void* stream);

/*
 * Broadcast SP over NVLink peer memory (no collective): the frames->tokens and
 * tokens->frames exchanges of the temporal site (reference parallel.reshard,
 * pkg/src/pab_engine/parallel.py:140-180, 322-348) fused into the prologues.
 *
 *   h_layout == PAB_LAYOUT_PEER: h row (b, t, s) of this rank's frame shard is
 *     stored straight into rank dst = s / (n_s/n_w)'s token-layout buffer
 *     peer_h[dst] (T, n_b, n_s/n_w, D) at row ((rank * n_t + t) * n_b + b) *
 *     (n_s/n_w) + s % (n_s/n_w)   -- the prologue's stores ARE the all-to-all.
 *   term_layout[i] == PAB_LAYOUT_PEER: pending term i is read straight out of the
 *     ranks' token-layout buffers peer_src[0..n_w) with the inverse map (the
 *     temporal site's output, no return all-to-all and no unpack pass); at most
 *     one such term per launch.  peer_copy != NULL: that term is also written
 *     frame-major (n_b, n_t, n_s, D) into peer_copy (the broadcast cache slot, so
 *     a later broadcast step reads it locally and communicates nothing).
 * Every pointer must be mapped into this process (CUDA IPC / same process).
 * Otherwise identical to pab_residual_modnorm_ex.  n_w <= PAB_MAX_PEERS.
 */
#define PAB_LAYOUT_PEER 3
int pab_residual_modnorm_peer(const float* x_in, float* x_out,
                              const void* const* pending, const int* term_layout, int n_pending,
                              const void* const* peer_src, void* peer_copy,
                              const float* gamma, const float* beta,
                              const float* mod, void* h_out, void* const* peer_h,
                              int64_t n_b, int64_t n_t, int64_t n_s, int64_t n_w, int rank,
                              int D, float eps, int mode, int h_layout, void* stream);

/*
 * Device barrier of an n_w-rank group over peer memory (orders the peer stores
 * and loads above; no reference counterpart -- the reference exchanges arrays in
 * one process).  flags[q] = rank q's n_w-entry uint32 flag array (zeroed once,
 * mapped here); counter = this rank's uint32 epoch counter (zeroed once).  The
 * launch bumps the epoch, release-stores it into slot [rank] of every rank's
 * flags and waits (acquire) until every slot of its own array reached it.
 * Graph-capturable (the epoch lives on the device).  A wait longer than
 * timeout_s stores PAB_PEER_TIMEOUT into *error and returns (never hangs).
 */
#define PAB_PEER_TIMEOUT 0x7ee1u
int pab_peer_barrier(void* const* flags, void* counter, int rank, int n_w, void* error,
                     double timeout_s, void* stream);

/*
 * Redundancy scan on the device: sums of two bf16 site outputs of n elements,
 * out4 = { sum (a-b)^2, sum a^2, sum b^2, sum a*b } in fp64 (zeroed by the call).
 * Every metric of the reference's diff_metric (mse, relative_l2, one_minus_cosine;
 * pkg/src/pab_engine/profiler.py:60-81) follows from them, so redundancy_scan
 * (profiler.py:140-173) needs no device->host snapshot copies.
 */
int pab_diff_sums(const void* a, const void* b, int64_t n, double* out4, void* stream);

/*
 * Fused end-of-step residual drain + classifier-free guidance + DDIM (K8).
 * Replaces: the eps combine and ddim_update of diffusion.sample
 * (pkg/src/pab_engine/diffusion.py:183-189, 100-103).
 *   eps_b = r[b] + pending terms (fp32, in order)
 *   guidance: eps_hat = eps_1 + g * (eps_0 - eps_1), applied to every batch row
 *   z[b] = sqrt(a_next) * ((z[b] - sqrt(1-a_cur) * eps_hat) / sqrt(a_cur)) + sqrt(1-a_next) * eps_hat
 * All scalars are rounded to fp32 first and every op is a single fp32
 * rounding, as numpy does with python-float scalars on float32 arrays.
 */
int pab_ddim_cfg(float* z, const float* r, const void* const* pending, int n_pending,
                 int batch, int64_t n_per_batch, int guidance, double guidance_scale,
                 double a_cur, double a_next, void* stream);

/*
 * Materialised attention probabilities for score broadcast (K10,
 * broadcast_object="scores"). Replaces: numerics.softmax_rows after the
 * logits *= 1/sqrt(dh) of scaled_dot_attention (pkg/src/pab_engine/numerics.py:
 * 107-112, 133-151) as captured by model._attention_core (model.py:325-335).
 *   p[r, j] = bf16( exp(scale*l[r, j] - m_r) / sum_j exp(scale*l[r, j] - m_r) ),
 *   m_r = max_j scale*l[r, j]; l fp32 rows of length n (row stride ld_l), p bf16 (ld_p).
 */
int pab_softmax_rows(const float* logits, int64_t ld_l, void* p_bf16, int64_t ld_p, int64_t rows, int64_t n,
                     float scale, void* stream);

/*
 * y = x + a * w on fp32 vectors (one rounding per element; y may alias x).
 * Replaces the Delta-DiT whole-layer residual delta of forward_step, kept in
 * fp32 like the reference: store d = x - x_layer_in (a = -1), replay x + d
 * (a = 1) (pkg/src/pab_engine/model.py:506-523, 565-566).
 */
int pab_add_scaled_f32(float* y, const float* x, const float* w, float a, int64_t n, void* stream);

/* tanh-approximation GELU on bf16 (numerics.py:154-158), in may equal out. */
int pab_gelu_bf16(const void* in, void* out, int64_t n, void* stream);

/*
 * splitmix64 parameter fill (model.init_model + numerics.RandomStream.uniform,
 * pkg/src/pab_engine/model.py:168-222, numerics.py:161-201).
 * Element i (i < rows*cols) takes draw (first_draw + i + 1) of the stream
 * whose state is `state`: v = f32(lo + (mant53 * 2^-53) * (hi - lo)).
 * It is written to dst[(i / cols) * ld + col0 + (i % cols)] as fp32
 * (dtype 0) or bf16 (dtype 1).
 */
int pab_fill_uniform(void* dst, int dtype, int64_t rows, int64_t cols, int64_t ld, int64_t col0,
                     uint64_t state, uint64_t first_draw, double lo, double hi, void* stream);

/*
 * Multi-head scaled-dot-product attention softmax(q k^T / sqrt(dh)) v (K1-K3).
 * Replaces: scaled_dot_attention (numerics.py:133-151) as called by the
 * spatial / temporal / cross sites (model.py:327-385).
 *
 * Problem (a, b, h), a < n_a, b < n_b, h < heads, attends n_q query rows to
 * n_k key rows.  Element (a, b, h, i, d) of tensor X lives at
 *   X + a*X_sa + b*X_sb + i*X_si + h*dh + d        (element units, bf16)
 * so spatial, temporal (transposed) and cross layouts need no copies:
 *   spatial : a = frame (B*T), b = -, i = token     (rows of (B,T,S,D))
 *   temporal: a = batch, b = token, i = frame        (rows of (B,T,S,D))
 *   cross   : a = batch, i = (frame, token) for q/o, i = text token for k/v
 * Output o uses the same addressing with (o_sa, o_sb, o_si).
 * impl: 0 or 1 = the tcgen05/TMA kernels (row-per-thread kernel for long
 * sequences, block-diagonal packed kernel for short ones); shapes they cannot
 * address (dh not a multiple of 8 or > 80, unaligned strides) return
 * PAB_ERR_UNSUPPORTED -- there is no silent fallback.  2 = the SIMT kernel,
 * a test cross-check only (any dh <= 128).
 */
typedef struct {
    const void* q; const void* k; const void* v; void* o;
    int64_t q_sa, q_sb, q_si;
    int64_t k_sa, k_sb, k_si;
    int64_t v_sa, v_sb, v_si;
    int64_t o_sa, o_sb, o_si;
    int32_t n_a, n_b, n_q, n_k, heads, dh;
    float scale;
} pab_attn_args;

int pab_attention(const pab_attn_args* args, int impl, void* stream);

/* 1 if the tcgen05 kernels support these args (what impl=0 runs), else 0.
 * Pure host logic, no GPU needed. */
int pab_attention_select(const pab_attn_args* args);

/*
 * Projection GEMM on the tcgen05 tensor cores (2-CTA, TMA, TMEM accumulators).
 * Replaces: numerics.matmul (pkg/src/pab_engine/numerics.py:72-104) for every
 * projection of a computed site: q/k/v and o of the spatial/temporal sites
 * (model.py:346-359), q and o of the cross sites (model.py:376-385), and the MLP
 * w1 -> gelu -> w2 pair (model.py:398-403, gelu numerics.py:154-158).
 *
 *   C[m, n] = epi( sum_k A[m, k] * B[n, k] )    bf16 in/out, fp32 accumulation
 *   A: (M, K) row stride lda; B: the weight W (K, N) stored transposed, (N, K) row
 *   stride ldb; C: (M, N) row stride ldc (elements).
 *   epilogue 0: bf16(acc); 1: bf16(gelu_tanh(acc)).
 * Bases 16-byte aligned, lda/ldb/ldc/K multiples of 8; M, N, K tails are handled
 * (zero-filled loads, clipped stores).
 */
int pab_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                  int64_t M, int64_t N, int64_t K, int epilogue, void* stream);

/*
 * Output projection fused with the residual add of its site (the epilogue does the
 * `x = x + o` of reference model.py:503 that the next site's prologue did before):
 *   o[m, n] = bf16( sum_k A[m, k] * B[n, k] )          (as pab_gemm_bf16, epilogue 0)
 *   x[perm(m), n] += o[m, n]                           (fp32, one rounding)
 *   C[m, n] = o[m, n]   only if C != NULL (the site's output is cached for a later step)
 * perm is the identity, or with tm_t, tm_s > 0 maps token-major GEMM rows (b, s, t) to
 * frame-major residual rows (b, t, s) (the temporal site, S = tm_s, T = tm_t; M must be
 * a multiple of tm_t * tm_s).  x: fp32, row stride ldx (elements, multiple of 4), N % 4 == 0.
 */
int pab_gemm_bf16_residual(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                           float* x, int64_t ldx, int64_t M, int64_t N, int64_t K,
                           int64_t tm_t, int64_t tm_s, void* stream);

/*
 * pab_gemm_bf16_residual that also writes h = bf16(x_new) (row stride ldh, x's
 * frame-major row order, rows < h_rows only -- h_rows < 0: all; h may be NULL):
 * the query input of a cross site that
 * follows the computed site, which the reference forms as x + o then casts
 * (model.py:376-385, 503) -- the stand-alone cast pass disappears.
 */
int pab_gemm_bf16_residual_h(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                             float* x, int64_t ldx, void* h, int64_t ldh, int64_t h_rows, int64_t M, int64_t N,
                             int64_t K, int64_t tm_t, int64_t tm_s, void* stream);

/* Debug only: record a clock64 event timeline of CTA (0,0,0) of subsequent
 * tcgen05 attention launches into device_buffer (NULL disables). */
int pab_attn_debug_trace(long long* device_buffer);

#ifdef __cplusplus
}
#endif
#endif /* PAB_B200_H */

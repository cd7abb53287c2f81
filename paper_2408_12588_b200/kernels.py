"""Thin torch-tensor wrappers over the C ABI (device memory owned by torch).

Every wrapper launches on torch's current CUDA stream and validates the
tensors it hands to the library (device, dtype, contiguity); shape errors are
raised as the reference's ShapeError kinds.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from .errors import ShapeError, ValidationError

MAX_PENDING = _lib.MAX_PENDING
# IMPL_SIMT: the SIMT attention kernel, a test cross-check only (never selected automatically)
IMPL_AUTO, IMPL_TCGEN05, IMPL_SIMT = 0, 1, 2


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need(t: torch.Tensor, dtype, name: str):
    if not t.is_cuda:
        raise ValidationError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValidationError(f"{name} must be {dtype}, got {t.dtype}")


LAYOUT_FRAME, LAYOUT_TOKEN, LAYOUT_A2A, LAYOUT_PEER = 0, 1, 2, 3


def is_token_major(t) -> bool:
    """Site outputs of the serial temporal site are stored token-major (rows (b, s, t))."""
    return bool(getattr(t, "pab_token_major", False))


def term_layout(t) -> int:
    """Row layout of a pending residual term: frame-major, token-major (serial temporal
    site) or all-to-all order (sequence-parallel temporal site, ``pab_a2a_world`` ranks)."""
    if getattr(t, "pab_peer", None) is not None:
        return LAYOUT_PEER
    if getattr(t, "pab_a2a_world", 0):
        return LAYOUT_A2A
    return LAYOUT_TOKEN if is_token_major(t) else LAYOUT_FRAME


def residual_modnorm(x_in, x_out, pending, h_out=None, mod=None, gamma=None, beta=None, mode=1, eps=1e-5,
                     shape=None, h_token_major=False, h_layout=None, n_w=1, h_peer=None):
    """x_out = x_in + sum(pending) (fp32); h_out = modnorm(x_out) (mode 1) or bf16(x_out) (mode 2).

    ``shape`` = (B, T, S) of the residual stream (block); needed when a pending term is not
    frame-major (``term_layout``) or when h is written token-major (``h_token_major``) or in
    all-to-all send order over ``n_w`` ranks (``h_layout=LAYOUT_A2A``).

    Peer transport (broadcast SP over NVLink, ``peer.PeerExchange``): ``h_peer`` = (exchange,
    buffer name) stores h straight into every rank's token-layout buffer (``LAYOUT_PEER``);
    a pending term carrying ``pab_peer`` = (exchange, buffer name) is read out of the ranks'
    buffers, and copied frame-major into ``pab_peer_copy`` when that is set (cache slot).
    """
    lib = _lib.load()
    _need(x_in, torch.float32, "x_in")
    _need(x_out, torch.float32, "x_out")
    D = x_in.shape[-1]
    rows = x_in.numel() // D
    if x_out.shape != x_in.shape or not x_in.is_contiguous() or not x_out.is_contiguous():
        raise ShapeError("residual stream buffers must be contiguous and equally shaped")
    for p in pending:
        _need(p, torch.bfloat16, "pending term")
        if p.numel() != x_in.numel() or not p.is_contiguous():
            raise ShapeError(f"pending term {tuple(p.shape)} does not match residual {tuple(x_in.shape)}")
    if h_out is not None:
        _need(h_out, torch.bfloat16, "h_out")
        if h_out.numel() != x_in.numel():
            raise ShapeError("h_out does not match the residual stream")
    if h_layout is None:
        h_layout = LAYOUT_PEER if h_peer is not None else (LAYOUT_TOKEN if h_token_major else LAYOUT_FRAME)
    layouts = [term_layout(p) for p in pending]
    peer_terms = [p for p, lay in zip(pending, layouts) if lay == LAYOUT_PEER]
    if len(peer_terms) > 1:
        raise ValidationError("at most one peer-resident pending term per prologue")
    px = h_peer[0] if h_peer is not None else (peer_terms[0].pab_peer[0] if peer_terms else None)
    if px is not None:
        n_w = px.world
    for p, lay in zip(pending, layouts):
        if lay == LAYOUT_A2A:
            n_w = int(p.pab_a2a_world)
    general = h_layout != LAYOUT_FRAME or any(layouts)
    if general and (shape is None or shape[0] * shape[1] * shape[2] != rows):
        raise ShapeError("permuted residual terms / outputs need the (B, T, S) shape of the stream")
    pend = list(zip(pending, layouts))
    src_x = [x_in]

    def call(terms, h, m, md, hl):
        arr = _lib.ptr_array([p.data_ptr() for p, _ in terms])
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        peer_in = [p for p, l in terms if l == LAYOUT_PEER]
        if px is not None and (peer_in or hl == LAYOUT_PEER):
            lay = (ctypes.c_int * max(1, len(terms)))(*[l for _, l in terms])
            src = px.ptrs(peer_in[0].pab_peer[1]) if peer_in else None
            copy = getattr(peer_in[0], "pab_peer_copy", None) if peer_in else None
            dst = px.ptrs(h_peer[1]) if hl == LAYOUT_PEER else None
            st = lib.pab_residual_modnorm_peer(src_x[0].data_ptr(), x_out.data_ptr(), arr, lay, len(terms), src,
                                               ptr(copy), ptr(gamma), ptr(beta), ptr(md), ptr(h), dst, shape[0],
                                               shape[1], shape[2], int(n_w), int(px.rank), D, float(eps), int(m),
                                               int(hl), _stream())
            _lib.check(st, "pab_residual_modnorm_peer")
            return
        src = src_x[0]
        if general:
            lay = (ctypes.c_int * max(1, len(terms)))(*[l for _, l in terms])
            st = lib.pab_residual_modnorm_ex(src.data_ptr(), x_out.data_ptr(), arr, lay, len(terms), ptr(gamma),
                                             ptr(beta), ptr(md), ptr(h), shape[0], shape[1], shape[2], int(n_w), D,
                                             float(eps), int(m), int(hl), _stream())
            _lib.check(st, "pab_residual_modnorm_ex")
        else:
            st = lib.pab_residual_modnorm(src.data_ptr(), x_out.data_ptr(), arr, len(terms), ptr(gamma), ptr(beta),
                                          ptr(md), ptr(h), rows, D, float(eps), int(m), _stream())
            _lib.check(st, "pab_residual_modnorm")

    # more than MAX_PENDING terms: drain in order, normalising only on the last chunk
    while len(pend) > MAX_PENDING:
        chunk, pend = pend[:MAX_PENDING], pend[MAX_PENDING:]
        call(chunk, None, 0, None, LAYOUT_FRAME)
        src_x[0] = x_out
    call(pend, h_out, mode, mod, h_layout)


def residual_modnorm_sp(x_in, x_out, pending, h_out, shard_shape, n_w, mod=None, gamma=None, beta=None, mode=1,
                        eps=1e-5):
    """residual_modnorm whose h output is written in all-to-all send order:
    shard rows (b, t, s) of shape (n_b, n_t, n_s) -> (dest, t, b, s_local)."""
    n_b, n_t, n_s, D = shard_shape
    if x_in.numel() != n_b * n_t * n_s * D or h_out.numel() != x_in.numel():
        raise ShapeError("sequence-parallel prologue buffers do not match the shard shape")
    if mode == 0:
        raise ValidationError("the all-to-all ordered prologue needs an h output (mode 1 or 2)")
    residual_modnorm(x_in, x_out, pending, h_out=h_out, mod=mod, gamma=gamma, beta=beta, mode=mode, eps=eps,
                     shape=(n_b, n_t, n_s), h_layout=LAYOUT_A2A, n_w=n_w)


def ddim_cfg(z, r, pending, guidance: bool, guidance_scale: float, a_cur: float, a_next: float):
    lib = _lib.load()
    _need(z, torch.float32, "z")
    _need(r, torch.float32, "r")
    batch = z.shape[0]
    n = z.numel() // batch
    pend = list(pending)
    if any(term_layout(p) for p in pend) or len(pend) > MAX_PENDING:
        raise ShapeError("ddim_cfg takes at most MAX_PENDING frame-major terms; flush the rest first")
    arr = _lib.ptr_array([p.data_ptr() for p in pend])
    _lib.check(
        lib.pab_ddim_cfg(z.data_ptr(), r.data_ptr(), arr, len(pend), batch, n, int(bool(guidance)),
                         float(guidance_scale), float(a_cur), float(a_next), _stream()),
        "pab_ddim_cfg",
    )


def softmax_rows(logits: torch.Tensor, p_out: torch.Tensor, scale: float) -> torch.Tensor:
    """p_out (bf16) <- softmax(scale * logits) over the last axis (K10 score capture)."""
    lib = _lib.load()
    _need(logits, torch.float32, "logits")
    _need(p_out, torch.bfloat16, "probabilities")
    n = logits.shape[-1]
    if p_out.shape != logits.shape or logits.stride(-1) != 1 or p_out.stride(-1) != 1:
        raise ShapeError("softmax_rows needs equal shapes with unit column stride")
    lv, pv = logits.reshape(-1, n), p_out.view(-1, n)
    _lib.check(lib.pab_softmax_rows(lv.data_ptr(), lv.stride(0), pv.data_ptr(), pv.stride(0), lv.shape[0], n,
                                    float(scale), _stream()), "pab_softmax_rows")
    return p_out


def add_scaled_(y: torch.Tensor, x: torch.Tensor, w: torch.Tensor, a: float) -> torch.Tensor:
    """y <- x + a * w (fp32, contiguous, equal sizes)."""
    lib = _lib.load()
    for t, name in ((y, "y"), (x, "x"), (w, "w")):
        _need(t, torch.float32, name)
        if not t.is_contiguous() or t.numel() != y.numel():
            raise ShapeError("add_scaled operands must be contiguous and equally sized")
    _lib.check(lib.pab_add_scaled_f32(y.data_ptr(), x.data_ptr(), w.data_ptr(), float(a), y.numel(), _stream()),
               "pab_add_scaled_f32")
    return y


def gelu_(x: torch.Tensor) -> torch.Tensor:
    lib = _lib.load()
    _need(x, torch.bfloat16, "gelu input")
    _lib.check(lib.pab_gelu_bf16(x.data_ptr(), x.data_ptr(), x.numel(), _stream()), "pab_gelu_bf16")
    return x


def fill_uniform(dst: torch.Tensor, rows: int, cols: int, col0: int, state: int, first_draw: int, lo: float,
                 hi: float):
    """Fill dst[:, col0:col0+cols] (row-major, ld = dst.shape[-1]) from a splitmix64 stream."""
    lib = _lib.load()
    if dst.dtype not in (torch.float32, torch.bfloat16) or not dst.is_cuda or not dst.is_contiguous():
        raise ValidationError("fill_uniform target must be a contiguous CUDA fp32/bf16 tensor")
    ld = dst.shape[-1]
    dtype = 0 if dst.dtype == torch.float32 else 1
    _lib.check(
        lib.pab_fill_uniform(dst.data_ptr(), dtype, rows, cols, ld, col0, ctypes.c_uint64(state),
                             ctypes.c_uint64(first_draw), float(lo), float(hi), _stream()),
        "pab_fill_uniform",
    )


EPI_NONE, EPI_GELU = 0, 1


def gemm(a: torch.Tensor, w_t: torch.Tensor, out: torch.Tensor, epilogue: int = EPI_NONE) -> torch.Tensor:
    """out = epi(a @ w_t^T) on the tcgen05 GEMM: a (M, K), w_t (N, K) (the weight stored
    transposed, K-major), out (M, N); bf16, unit column stride, any row strides."""
    lib = _lib.load()
    for t, name in ((a, "A"), (w_t, "B"), (out, "C")):
        _need(t, torch.bfloat16, name)
        if t.dim() != 2 or t.stride(1) != 1:
            raise ShapeError(f"gemm operand {name} must be 2-D with unit column stride")
    M, K = a.shape
    N = w_t.shape[0]
    if w_t.shape[1] != K or out.shape != (M, N):
        raise ShapeError(f"gemm shapes {tuple(a.shape)} x {tuple(w_t.shape)}^T -> {tuple(out.shape)}")
    _lib.check(lib.pab_gemm_bf16(a.data_ptr(), a.stride(0), w_t.data_ptr(), w_t.stride(0), out.data_ptr(),
                                 out.stride(0), M, N, K, int(epilogue), _stream()), "pab_gemm_bf16")
    return out


def residual_token_major_ok(T: int, S: int) -> bool:
    """gemm_residual's token-major row map needs every 128-row block to be whole tokens
    of one batch entry: T | 128 and 128 | T*S (C3: T = 16, S = 1560)."""
    return 128 % T == 0 and (T * S) % 128 == 0


def gemm_residual(a: torch.Tensor, w_t: torch.Tensor, x: torch.Tensor, out=None, token_major=None, h=None,
                  h_rows=-1):
    """x[perm(m)] += bf16(a @ w_t^T)[m] (fp32 residual stream, in place) and, when ``out`` is
    given, out = bf16(a @ w_t^T) (the cached site output).  token_major = (T, S): the rows
    of ``a`` are (b, s, t), the rows of ``x`` (b, t, s).  ``h`` (bf16, x's shape and row
    order): also h = bf16(x_new) for x rows < ``h_rows`` (-1: all), the next cross site's
    query input."""
    lib = _lib.load()
    for t, name in ((a, "A"), (w_t, "B")):
        _need(t, torch.bfloat16, name)
        if t.dim() != 2 or t.stride(1) != 1:
            raise ShapeError(f"gemm operand {name} must be 2-D with unit column stride")
    _need(x, torch.float32, "residual")
    M, K = a.shape
    N = w_t.shape[0]
    x2 = x.view(-1, x.shape[-1])
    if w_t.shape[1] != K or x2.shape[1] != N or x2.shape[0] != M or x2.stride(1) != 1:
        raise ShapeError(f"gemm_residual shapes {tuple(a.shape)} x {tuple(w_t.shape)}^T -> {tuple(x.shape)}")
    if out is not None:
        _need(out, torch.bfloat16, "C")
        if out.shape != (M, N) or out.stride(1) != 1:
            raise ShapeError("gemm_residual output must be (M, N) with unit column stride")
    tm_t, tm_s = token_major if token_major is not None else (0, 0)
    if h is not None:
        _need(h, torch.bfloat16, "h")
        h2 = h.view(-1, h.shape[-1])
        if h2.shape != (M, N) or h2.stride(1) != 1:
            raise ShapeError("gemm_residual h must match the residual stream")
    _lib.check(lib.pab_gemm_bf16_residual_h(a.data_ptr(), a.stride(0), w_t.data_ptr(), w_t.stride(0),
                                            out.data_ptr() if out is not None else None,
                                            out.stride(0) if out is not None else 0, x2.data_ptr(), x2.stride(0),
                                            h2.data_ptr() if h is not None else None,
                                            h2.stride(0) if h is not None else 0, int(h_rows),
                                            M, N, K, int(tm_t), int(tm_s), _stream()), "pab_gemm_bf16_residual_h")
    return out


def attn_args(q, k, v, o, qs, ks, vs, os_, n_a, n_b, n_q, n_k, heads, dh, scale=None) -> _lib.AttnArgs:
    """Build pab_attn_args; *s are (s_a, s_b, s_i) element strides of each operand."""
    for t, name in ((q, "q"), (k, "k"), (v, "v"), (o, "o")):
        _need(t, torch.bfloat16, name)
    a = _lib.AttnArgs()
    a.q, a.k, a.v, a.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr()
    a.q_sa, a.q_sb, a.q_si = qs
    a.k_sa, a.k_sb, a.k_si = ks
    a.v_sa, a.v_sb, a.v_si = vs
    a.o_sa, a.o_sb, a.o_si = os_
    a.n_a, a.n_b, a.n_q, a.n_k, a.heads, a.dh = n_a, n_b, n_q, n_k, heads, dh
    a.scale = (1.0 / math.sqrt(dh)) if scale is None else scale
    return a


def attention(args: _lib.AttnArgs, impl: int = IMPL_AUTO) -> None:
    lib = _lib.load()
    _lib.check(lib.pab_attention(ctypes.byref(args), int(impl), _stream()), "pab_attention")


def attention_select(args: _lib.AttnArgs) -> int:
    return int(_lib.load().pab_attention_select(ctypes.byref(args)))

"""Op-level numerics of every CUDA kernel against a plain PyTorch fp32
reference of the same op (attention, modnorm, GELU) or an exact numpy
restatement (DDIM/CFG, splitmix fill).  Runs on the B200 only."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2408_12588_b200 import kernels  # noqa: E402
from paper_2408_12588_b200.numerics import RandomStream  # noqa: E402

DEV = "cuda"


def ref_attention(q, k, v):
    """fp32 softmax(q k^T / sqrt(dh)) v on (..., n, dh) tensors."""
    q, k, v = q.float(), k.float(), v.float()
    s = (q @ k.transpose(-1, -2)) / math.sqrt(q.shape[-1])
    return torch.softmax(s, dim=-1) @ v


def check_close(got, want, tag, rel_tol=1.2e-2):
    got, want = got.float(), want.float()
    err = (got - want).norm() / want.norm().clamp_min(1e-12)
    mx = (got - want).abs().max() / want.abs().max().clamp_min(1e-12)
    assert torch.isfinite(got).all(), tag
    assert err < rel_tol and mx < 4 * rel_tol, (tag, float(err), float(mx))


def spatial_case(B, T, S, H, dh, impl, seed=0):
    g = torch.Generator(device=DEV).manual_seed(seed)
    D = H * dh
    qkv = torch.randn(B * T * S, 3 * D, device=DEV, generator=g).to(torch.bfloat16)
    out = torch.full((B * T * S, D), float("nan"), device=DEV, dtype=torch.bfloat16)
    ld = 3 * D
    a = kernels.attn_args(qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:], out, (S * ld, 0, ld), (S * ld, 0, ld),
                          (S * ld, 0, ld), (S * D, 0, D), B * T, 1, S, S, H, dh)
    kernels.attention(a, impl)
    torch.cuda.synchronize()
    x = qkv.view(B * T, S, 3, H, dh).permute(2, 0, 3, 1, 4)  # (3, BT, H, S, dh)
    want = ref_attention(x[0], x[1], x[2]).permute(0, 2, 1, 3).reshape(B * T * S, D)
    return out, want, a


def temporal_case(B, T, S, H, dh, impl, seed=1):
    g = torch.Generator(device=DEV).manual_seed(seed)
    D = H * dh
    qkv = torch.randn(B * T * S, 3 * D, device=DEV, generator=g).to(torch.bfloat16)
    out = torch.full((B * T * S, D), float("nan"), device=DEV, dtype=torch.bfloat16)
    ld = 3 * D
    st = (T * S * ld, ld, S * ld)
    a = kernels.attn_args(qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:], out, st, st, st, (T * S * D, D, S * D),
                          B, S, T, T, H, dh)
    kernels.attention(a, impl)
    torch.cuda.synchronize()
    x = qkv.view(B, T, S, 3, H, dh).permute(3, 0, 2, 4, 1, 5)  # (3, B, S, H, T, dh)
    want = ref_attention(x[0], x[1], x[2]).permute(0, 3, 1, 2, 4).reshape(B * T * S, D)
    return out, want, a


def cross_case(B, N, M, H, dh, impl, seed=2):
    g = torch.Generator(device=DEV).manual_seed(seed)
    D = H * dh
    q = torch.randn(B * N, D, device=DEV, generator=g).to(torch.bfloat16)
    kv = torch.randn(B * M, 2 * D, device=DEV, generator=g).to(torch.bfloat16)
    out = torch.full((B * N, D), float("nan"), device=DEV, dtype=torch.bfloat16)
    a = kernels.attn_args(q, kv[:, :D], kv[:, D:], out, (N * D, 0, D), (M * 2 * D, 0, 2 * D),
                          (M * 2 * D, 0, 2 * D), (N * D, 0, D), B, 1, N, M, H, dh)
    kernels.attention(a, impl)
    torch.cuda.synchronize()
    qh = q.view(B, N, H, dh).transpose(1, 2)
    kvh = kv.view(B, M, 2, H, dh).permute(2, 0, 3, 1, 4)
    want = ref_attention(qh, kvh[0], kvh[1]).transpose(1, 2).reshape(B * N, D)
    return out, want, a


IMPLS = [kernels.IMPL_TCGEN05, kernels.IMPL_SIMT]
IMPL_IDS = ["tcgen05", "simt"]


@pytest.mark.parametrize("impl", IMPLS, ids=IMPL_IDS)
@pytest.mark.parametrize("B,T,S,H,dh", [(1, 2, 1024, 2, 72), (1, 1, 1560, 2, 72), (2, 1, 200, 3, 72),
                                         (1, 2, 16, 4, 8), (1, 1, 300, 2, 16), (1, 1, 129, 1, 64),
                                         (1, 1, 77, 2, 32), (1, 1, 100, 2, 56), (1, 8, 1024, 16, 72),
                                         (1, 3, 1560, 16, 72), (1, 2, 3600, 16, 72)])  # C3, C5 frames
def test_spatial_attention(impl, B, T, S, H, dh):
    out, want, a = spatial_case(B, T, S, H, dh, impl)
    check_close(out, want, ("spatial", impl, B, T, S, H, dh))


@pytest.mark.parametrize("impl", [kernels.IMPL_TCGEN05], ids=["tcgen05"])
def test_attention_rising_scores_rescale(impl):
    # key norms grow along the sequence, so later KV tiles raise the running max by far
    # more than 2^8: exercises the lazy O rescale of the online softmax
    g = torch.Generator(device=DEV).manual_seed(5)
    B, S, H, dh = 1, 1000, 2, 72
    D = H * dh
    q = torch.randn(B * S, D, device=DEV, generator=g)
    k = torch.randn(B * S, D, device=DEV, generator=g) * torch.linspace(0.2, 6.0, S, device=DEV)[:, None]
    v = torch.randn(B * S, D, device=DEV, generator=g)
    q, k, v = (x.to(torch.bfloat16) for x in (q, k, v))
    out = torch.full((B * S, D), float("nan"), device=DEV, dtype=torch.bfloat16)
    st = (S * D, 0, D)
    a = kernels.attn_args(q, k, v, out, st, st, st, st, B, 1, S, S, H, dh)
    kernels.attention(a, impl)
    torch.cuda.synchronize()
    hv = lambda x: x.view(B, S, H, dh).transpose(1, 2)  # noqa: E731
    want = ref_attention(hv(q), hv(k), hv(v)).transpose(1, 2).reshape(B * S, D)
    check_close(out, want, ("rising", impl))


@pytest.mark.parametrize("impl", [kernels.IMPL_TCGEN05], ids=["tcgen05"])
@pytest.mark.parametrize("S", [1000, 1560, 300])
def test_attention_wide_score_spread(impl, S):
    # scores spread over hundreds of log2 units inside one KV tile: exp2 arguments far below
    # -126 must underflow to 0 on both the MUFU and the FMA-pipe polynomial path (a -127
    # clamp made the polynomial's exponent add wrap to NaN), and the -1e30 pad-column key
    # mask of a partial last tile must stay exact
    g = torch.Generator(device=DEV).manual_seed(11)
    H, dh = 2, 72
    D = H * dh
    q = torch.randn(S, D, device=DEV, generator=g)
    k = torch.randn(S, D, device=DEV, generator=g) * 40.0
    v = torch.randn(S, D, device=DEV, generator=g)
    q, k, v = (x.to(torch.bfloat16) for x in (q, k, v))
    out = torch.full((S, D), float("nan"), device=DEV, dtype=torch.bfloat16)
    st = (S * D, 0, D)
    a = kernels.attn_args(q, k, v, out, st, st, st, st, 1, 1, S, S, H, dh)
    kernels.attention(a, impl)
    torch.cuda.synchronize()
    hv = lambda x: x.view(1, S, H, dh).transpose(1, 2)  # noqa: E731
    want = ref_attention(hv(q), hv(k), hv(v)).transpose(1, 2).reshape(S, D)
    assert torch.isfinite(out.float()).all()
    check_close(out, want, ("spread", impl, S))


@pytest.mark.parametrize("impl", IMPLS, ids=IMPL_IDS)
@pytest.mark.parametrize("B,T,S,H,dh", [(2, 16, 100, 2, 72), (1, 8, 64, 2, 72), (1, 32, 40, 2, 72),
                                         (2, 4, 16, 4, 8), (1, 24, 30, 2, 16), (1, 16, 1560, 1, 72),
                                         (1, 32, 3600, 2, 72)])  # C5: 32 frames, 4 sequences per tile
def test_temporal_attention(impl, B, T, S, H, dh):
    out, want, a = temporal_case(B, T, S, H, dh, impl)
    check_close(out, want, ("temporal", impl, B, T, S, H, dh))


@pytest.mark.parametrize("impl", IMPLS, ids=IMPL_IDS)
@pytest.mark.parametrize("B,N,M,H,dh", [(2, 2048, 300, 2, 72), (2, 1000, 120, 2, 72), (1, 64, 16, 2, 72),
                                         (2, 64, 8, 4, 8), (1, 500, 5, 2, 16), (2, 24960, 300, 16, 72),
                                         (1, 115200, 300, 2, 72)])  # C5: 32 x 3600 queries
def test_cross_attention(impl, B, N, M, H, dh):
    out, want, a = cross_case(B, N, M, H, dh, impl)
    check_close(out, want, ("cross", impl, B, N, M, H, dh))


def test_model_shapes_select_tcgen05():
    _, _, a = spatial_case(1, 1, 256, 2, 72, kernels.IMPL_AUTO)
    assert kernels.attention_select(a) == kernels.IMPL_TCGEN05
    _, _, a = temporal_case(1, 16, 32, 2, 72, kernels.IMPL_AUTO)
    assert kernels.attention_select(a) == kernels.IMPL_TCGEN05
    _, _, a = cross_case(1, 64, 300, 2, 72, kernels.IMPL_AUTO)
    assert kernels.attention_select(a) == kernels.IMPL_TCGEN05


def test_unsupported_shape_is_an_error_not_a_fallback():
    # dh = 12 (not a multiple of 8): no TMA layout -> the product path refuses loudly;
    # the SIMT kernel still answers when asked for by name (test cross-check)
    from paper_2408_12588_b200.errors import ValidationError

    out, want, a = spatial_case(1, 1, 64, 2, 12, kernels.IMPL_SIMT)
    check_close(out, want, "simt dh12")
    assert kernels.attention_select(a) == 0
    with pytest.raises(ValidationError):
        kernels.attention(a, kernels.IMPL_AUTO)


def test_cfg_null_text_gives_zero_attention():
    # CFG null half: zero text embedding -> K = V = 0 -> output exactly 0
    B, N, M, H, dh = 1, 256, 300, 2, 72
    D = H * dh
    q = torch.randn(B * N, D, device=DEV).to(torch.bfloat16)
    kv = torch.zeros(B * M, 2 * D, device=DEV, dtype=torch.bfloat16)
    out = torch.full((B * N, D), 7.0, device=DEV, dtype=torch.bfloat16)
    a = kernels.attn_args(q, kv[:, :D], kv[:, D:], out, (N * D, 0, D), (M * 2 * D, 0, 2 * D),
                          (M * 2 * D, 0, 2 * D), (N * D, 0, D), B, 1, N, M, H, dh)
    kernels.attention(a, kernels.IMPL_TCGEN05)
    assert torch.count_nonzero(out) == 0


@pytest.mark.parametrize("D,n_pending,mode", [(1152, 0, 1), (1152, 2, 1), (144, 1, 2), (30, 3, 1), (64, 9, 1),
                                              (144, 2, 0)])
def test_residual_modnorm(D, n_pending, mode):
    rows = 333
    x = torch.randn(rows, D, device=DEV)
    pend = [torch.randn(rows, D, device=DEV).to(torch.bfloat16) for _ in range(n_pending)]
    mod = torch.randn(2 * D, device=DEV) * 0.1
    x_out = torch.empty_like(x)
    h = torch.empty(rows, D, device=DEV, dtype=torch.bfloat16)
    kernels.residual_modnorm(x, x_out, pend, h_out=h if mode else None, mod=mod, mode=mode)
    want_x = x.clone()
    for p in pend:
        want_x = want_x + p.float()
    assert torch.equal(x_out, want_x)  # same fp32 add order
    if mode == 1:
        ln = torch.nn.functional.layer_norm(want_x, (D,), eps=1e-5)
        want_h = ln * (1.0 + mod[D:]) + mod[:D]
        check_close(h, want_h, "modnorm", 6e-3)
    elif mode == 2:
        assert torch.equal(h, want_x.to(torch.bfloat16))


@pytest.mark.parametrize("guidance", [False, True])
@pytest.mark.parametrize("n", [4097, 4096 * 3])
def test_ddim_cfg_exact(guidance, n):
    """bit-exact with numpy's fp32 sequence: scalar path (ragged n) and float4 path"""
    B = 2 if guidance else 1
    z = torch.randn(B, n, device=DEV)
    r = torch.randn(B, n, device=DEV)
    pend = [torch.randn(B, n, device=DEV).to(torch.bfloat16) for _ in range(2)]
    a_cur, a_next, g = 0.31, 0.47, 4.0
    zn = z.cpu().numpy().copy()
    eps = r.cpu().numpy().copy()
    for p in pend:
        eps = eps + p.float().cpu().numpy()
    kernels.ddim_cfg(z, r, pend, guidance, g, a_cur, a_next)
    if guidance:
        e = eps[1:2] + np.float32(g) * (eps[0:1] - eps[1:2])
        eps = np.concatenate([e, e])
    x0 = (zn - np.float32(math.sqrt(1 - a_cur)) * eps) / np.float32(math.sqrt(a_cur))
    want = np.float32(math.sqrt(a_next)) * x0 + np.float32(math.sqrt(1 - a_next)) * eps
    assert np.array_equal(z.cpu().numpy(), want.astype(np.float32))


def test_gelu():
    x = (torch.randn(1 << 20, device=DEV) * 3).to(torch.bfloat16)
    want = torch.nn.functional.gelu(x.float(), approximate="tanh")
    got = kernels.gelu_(x.clone())
    check_close(got, want, "gelu", 5e-3)


def test_fill_uniform_matches_host_stream():
    seed, rows, cols = 12345, 37, 53
    host = RandomStream(seed)
    host.uniform(1000, -0.3, 0.3)  # advance: the device fill starts at draw 1000
    want = host.uniform(rows * cols, -0.25, 0.25).reshape(rows, cols).astype(np.float32)
    dst = torch.zeros(rows, cols + 7, device=DEV)
    kernels.fill_uniform(dst, rows, cols, 7, seed, 1000, -0.25, 0.25)
    assert np.array_equal(dst[:, 7:].cpu().numpy(), want)
    dst16 = torch.zeros(rows, cols, device=DEV, dtype=torch.bfloat16)
    kernels.fill_uniform(dst16, rows, cols, 0, seed, 1000, -0.25, 0.25)
    assert torch.equal(dst16, torch.from_numpy(want).to(DEV).to(torch.bfloat16))


@pytest.mark.parametrize("W,mode", [(2, 1), (4, 2), (8, 0), (16, 1)])
def test_residual_modnorm_all_to_all_order_terms(W, mode):
    """PAB_LAYOUT_A2A pending terms (the sequence-parallel temporal site's received output,
    (W_src, T/W, B, S/W, D)) are added through the prologue's row map, equal to unpacking
    them first (reference parallel.reshard, parallel.py:140-180)."""
    B, Tl, S, D = 2, 4, 96, 144
    rows = B * Tl * S
    g = torch.Generator(device=DEV).manual_seed(W)
    x = torch.randn(rows, D, device=DEV, generator=g)
    recv = torch.randn(W, Tl, B, S // W, D, device=DEV, generator=g).to(torch.bfloat16)
    recv.pab_a2a_world = W
    plain = torch.randn(rows, D, device=DEV, generator=g).to(torch.bfloat16)
    mod = torch.randn(2 * D, device=DEV, generator=g) * 0.1
    x_out = torch.empty_like(x)
    h = torch.empty(rows, D, device=DEV, dtype=torch.bfloat16)
    kernels.residual_modnorm(x, x_out, [plain, recv], h_out=h if mode else None, mod=mod, mode=mode,
                             shape=(B, Tl, S))
    unpacked = recv.permute(2, 1, 0, 3, 4).reshape(rows, D)
    want = x + plain.float() + unpacked.float()
    assert torch.equal(x_out, want)
    if mode == 1:
        ln = torch.nn.functional.layer_norm(want, (D,), eps=1e-5)
        check_close(h, ln * (1.0 + mod[D:]) + mod[:D], "modnorm a2a", 6e-3)
    elif mode == 2:
        assert torch.equal(h, want.to(torch.bfloat16))


class _FakePeers:
    """The W ranks' token buffers of a PeerExchange, all in this process (kernel test)."""

    def __init__(self, rank, bufs):
        from paper_2408_12588_b200 import _lib

        self.rank, self.world, self.bufs = rank, len(next(iter(bufs.values()))), bufs
        self._arr = {k: _lib.ptr_array([t.data_ptr() for t in v]) for k, v in bufs.items()}

    def ptrs(self, name):
        return self._arr[name]


@pytest.mark.parametrize("W,me", [(2, 1), (4, 2), (8, 7)])
def test_residual_modnorm_peer_layouts(W, me):
    """PAB_LAYOUT_PEER: the pending temporal output read straight out of the W ranks' token
    buffers (plus its frame-major cache copy), and h stored straight into the ranks' h
    token buffers -- equal to the all-to-all order forms (which equal reshard)."""
    B, Tl, S, D = 2, 3, 64, 144
    Sw, T, rows = S // W, Tl * W, B * Tl * S
    g = torch.Generator(device=DEV).manual_seed(W + me)
    x = torch.randn(rows, D, device=DEV, generator=g)
    o_tok = [torch.randn(T, B, Sw, D, device=DEV, generator=g).to(torch.bfloat16) for _ in range(W)]
    h_tok = [torch.full((T, B, Sw, D), 9.0, device=DEV, dtype=torch.bfloat16) for _ in range(W)]
    mod = torch.randn(2 * D, device=DEV, generator=g) * 0.1
    px = _FakePeers(me, {"o_tok": o_tok, "h_tok": h_tok})
    term = o_tok[me].view(o_tok[me].shape)
    term.pab_peer = (px, "o_tok")
    copy = torch.empty(B, Tl, S, D, device=DEV, dtype=torch.bfloat16)
    term.pab_peer_copy = copy
    x_out = torch.empty_like(x)
    kernels.residual_modnorm(x, x_out, [term], mod=mod, mode=1, shape=(B, Tl, S), h_peer=(px, "h_tok"))
    # what rank `me` receives in an all-to-all: rank src's token rows of frames [me*Tl, (me+1)*Tl)
    recv = torch.stack([o_tok[src][me * Tl:(me + 1) * Tl] for src in range(W)])  # (W_src, Tl, B, Sw, D)
    frame = recv.permute(2, 1, 0, 3, 4).reshape(B, Tl, S, D)
    assert torch.equal(copy, frame)
    want = x + frame.reshape(rows, D).float()
    assert torch.equal(x_out, want)
    ln = torch.nn.functional.layer_norm(want, (D,), eps=1e-5) * (1.0 + mod[D:]) + mod[:D]
    h_frame = ln.view(B, Tl, W, Sw, D)
    for dst in range(W):
        got = h_tok[dst][me * Tl:(me + 1) * Tl]  # (Tl, B, Sw, D) rows this rank stored
        check_close(got.reshape(-1, D), h_frame[:, :, dst].permute(1, 0, 2, 3).reshape(-1, D),
                    "peer h store", 6e-3)
        others = torch.cat([h_tok[dst][:me * Tl], h_tok[dst][(me + 1) * Tl:]])
        assert bool((others == 9.0).all())

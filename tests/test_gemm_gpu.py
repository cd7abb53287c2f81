"""The tcgen05 projection GEMM (pab_gemm_bf16, csrc/gemm.cu) against a torch fp32
reference of the same bf16 operands: every C2-C5 projection shape, GELU epilogue,
M/N/K tails and strided operands (the cross sites' live-row views)."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2408_12588_b200 import kernels  # noqa: E402


def _ref(a, w_t, epilogue):
    y = a.float() @ w_t.float().t()
    if epilogue == kernels.EPI_GELU:
        y = 0.5 * y * (1.0 + torch.tanh(0.7978845608028654 * (y + 0.044715 * y ** 3)))
    return y


def _check(M, N, K, epilogue=0, lda=None, ldc=None, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    lda, ldc = lda or K, ldc or N
    abuf = torch.randn(M, lda, device="cuda", generator=g).to(torch.bfloat16)
    a = abuf[:, :K]
    w_t = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    cbuf = torch.full((M, ldc), 7.0, device="cuda", dtype=torch.bfloat16)
    c = cbuf[:, :N]
    kernels.gemm(a, w_t, c, epilogue)
    ref = _ref(a, w_t, epilogue)
    err = (c.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    # bf16 output rounding (2^-9 relative) + fp32 accumulation-order differences
    assert err <= 8e-3 * scale + 1e-3, (M, N, K, epilogue, err, scale)
    if ldc > N:
        assert torch.all(cbuf[:, N:] == 7.0), "GEMM wrote past N"
    return err / scale


@pytest.mark.parametrize("M,N,K", [(49920, 3456, 1152), (49920, 1152, 1152), (49920, 1152, 4608),
                                   (32768, 2304, 1152), (24960, 1152, 1152), (600, 2304, 1152)])
def test_gemm_projection_shapes(M, N, K):
    _check(M, N, K)


def test_gemm_gelu_epilogue_w1_shape():
    _check(49920, 4608, 1152, kernels.EPI_GELU)


@pytest.mark.parametrize("M,N,K", [(1, 8, 8), (100, 144, 144), (257, 432, 144), (300, 96, 48), (513, 32, 32),
                                   (2048, 576, 144), (130, 1152, 4608), (4096, 4608, 1152)])
def test_gemm_tails(M, N, K):
    _check(M, N, K)
    _check(M, N, K, kernels.EPI_GELU)


def test_gemm_strided_operands():
    # A / C as column slices of wider rows (the fused [q|k|v] buffer, live-row views)
    _check(3000, 1152, 1152, lda=3456, ldc=3456)
    _check(777, 384, 1152, lda=1160, ldc=400)


@pytest.mark.parametrize("M,N,K,store,tm", [(49920, 1152, 4608, False, None), (49920, 1152, 1152, True, None),
                                            (4096, 1152, 1152, True, (16, 256)), (300, 144, 576, True, None),
                                            (2048, 144, 144, False, (8, 128)), (24960, 1152, 1152, False, None),
                                            (49920, 1152, 4608, True, None), (300, 144, 4608, True, None),
                                            (1000, 1152, 2304, False, None)])
def test_gemm_residual_epilogue(M, N, K, store, tm):
    """x[perm(m)] += bf16(A B^T)[m] in the epilogue (the site output's residual add), with and
    without the cached-output store, frame- and token-major rows; K >= 2048 takes the direct
    read-modify-write epilogue (the MLP w2), with ragged M and N."""
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w_t = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    x = torch.randn(M, N, device="cuda", generator=g)
    x0 = x.clone()
    out = torch.full((M, N), 5.0, device="cuda", dtype=torch.bfloat16) if store else None
    kernels.gemm_residual(a, w_t, x, out, token_major=tm)
    o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    kernels.gemm(a, w_t, o)  # same tiles and accumulation order -> bitwise the same o
    if store:
        assert torch.equal(out, o)
    o_rows = o.float()
    if tm is not None:
        T, S = tm
        o_rows = o_rows.view(-1, S, T, N).permute(0, 2, 1, 3).reshape(M, N)
    assert torch.equal(x, x0 + o_rows)


@pytest.mark.parametrize("M,N,K,store,tm,h_rows", [(49920, 1152, 1152, True, None, 24960),
                                                   (49920, 1152, 1152, False, (16, 1560), -1),
                                                   (4096, 1152, 1152, False, (16, 128), 2048),
                                                   (300, 144, 576, False, None, -1)])
def test_gemm_residual_h_output(M, N, K, store, tm, h_rows):
    """The residual epilogue's h = bf16(x + o) output (the next cross site's query input):
    bitwise bf16 of the updated stream, in the stream's frame-major row order, only rows
    < h_rows written (the live CFG rows)."""
    g = torch.Generator(device="cuda").manual_seed(2)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w_t = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    x = torch.randn(M, N, device="cuda", generator=g)
    h = torch.full((M, N), 7.0, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if store else None
    kernels.gemm_residual(a, w_t, x, out, token_major=tm, h=h, h_rows=h_rows)
    lim = M if h_rows < 0 else h_rows
    assert torch.equal(h[:lim], x[:lim].to(torch.bfloat16))
    assert bool((h[lim:] == 7.0).all())

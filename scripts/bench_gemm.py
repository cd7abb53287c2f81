"""TF/s of the projection GEMMs at C3 shapes: the repo's tcgen05 GEMM (pab_gemm_bf16)
next to cuBLAS / cuBLASLt via torch.  CUDA events, 20 launches after warm-up."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12588_b200 import kernels  # noqa: E402

rows, D, R = 49920, 1152, 4608


def t(fn, n=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n / 1e3


bf = dict(device="cuda", dtype=torch.bfloat16)
h = torch.randn(rows, D, **bf)
hid = torch.randn(rows, R, **bf)
wqkv = torch.randn(D, 3 * D, **bf) * 0.03
wo = torch.randn(D, D, **bf) * 0.03
w1 = torch.randn(D, R, **bf) * 0.03
w2 = torch.randn(R, D, **bf) * 0.03
zb = torch.zeros(R, **bf)
o3 = torch.empty(rows, 3 * D, **bf)
o1 = torch.empty(rows, D, **bf)
o4 = torch.empty(rows, R, **bf)
tq, to, t1, t2 = (w.t().contiguous() for w in (wqkv, wo, w1, w2))
xres = torch.zeros(rows, D, device="cuda")
res = {}
for name, fn, fl in [
    ("qkv_cublas", lambda: torch.mm(h, wqkv, out=o3), 2 * rows * D * 3 * D),
    ("qkv_ours", lambda: kernels.gemm(h, tq, o3), 2 * rows * D * 3 * D),
    ("o_cublas", lambda: torch.mm(h, wo, out=o1), 2 * rows * D * D),
    ("o_ours", lambda: kernels.gemm(h, to, o1), 2 * rows * D * D),
    ("w1_gelu_cublaslt", lambda: torch._addmm_activation(zb, h, w1, use_gelu=True), 2 * rows * D * R),
    ("w1_gelu_ours", lambda: kernels.gemm(h, t1, o4, kernels.EPI_GELU), 2 * rows * D * R),
    ("w2_cublas", lambda: torch.mm(hid, w2, out=o1), 2 * rows * R * D),
    ("w2_ours", lambda: kernels.gemm(hid, t2, o1), 2 * rows * R * D),
    ("o_resid_ours", lambda: kernels.gemm_residual(h, to, xres), 2 * rows * D * D),
    ("o_resid_store_ours", lambda: kernels.gemm_residual(h, to, xres, o1), 2 * rows * D * D),
    ("o_resid_tm_ours", lambda: kernels.gemm_residual(h, to, xres, None, token_major=(16, 1560)), 2 * rows * D * D),
    ("w2_resid_ours", lambda: kernels.gemm_residual(hid, t2, xres), 2 * rows * R * D),
]:
    s = t(fn)
    res[name] = {"ms": round(s * 1e3, 4), "tflops": round(fl / s / 1e12, 1)}
print(json.dumps(res, indent=1))

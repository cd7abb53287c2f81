"""Check cuBLASLt's GELU epilogue (torch._addmm_activation) against tanh-GELU and time it."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_12588_b200 import kernels
rows, D, R = 49920, 1152, 4608
h = torch.randn(rows, D, device="cuda").to(torch.bfloat16)
w = (torch.rand(D, R, device="cuda") * 2 - 1).mul(1 / D**0.5).to(torch.bfloat16)
bias = torch.zeros(R, device="cuda", dtype=torch.bfloat16)
ref = torch.nn.functional.gelu((h.float() @ w.float()), approximate="tanh")
erf = torch.nn.functional.gelu((h.float() @ w.float()))
lt = torch._addmm_activation(bias, h, w, use_gelu=True).float()
print("lt vs tanh relL2", float((lt - ref).norm() / ref.norm()), " lt vs erf", float((lt - erf).norm() / erf.norm()))
out = torch.empty(rows, R, device="cuda", dtype=torch.bfloat16)
def t(fn, n=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n
print("mm+gelu kernel ms", t(lambda: (torch.mm(h, w, out=out), kernels.gelu_(out))))
print("mm only ms", t(lambda: torch.mm(h, w, out=out)))
print("addmm_activation ms", t(lambda: torch._addmm_activation(bias, h, w, use_gelu=True)))

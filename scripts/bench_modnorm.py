"""Microbenchmark of the broadcast epilogue / modnorm prologue at C3 rows (CUDA events)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_12588_b200 import kernels
rows, D = 49920, 1152
x = torch.randn(rows, D, device="cuda"); r = torch.empty_like(x)
h = torch.empty(rows, D, device="cuda", dtype=torch.bfloat16)
mod = torch.randn(2 * D, device="cuda") * 0.1
pend = [torch.randn(rows, D, device="cuda").to(torch.bfloat16) for _ in range(3)]
res = {}
for k in (0, 1, 2):
    for mode in (1, 2):
        f = lambda: kernels.residual_modnorm(x, r, pend[:k], h_out=h, mod=mod, mode=mode)
        f(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): f()
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b) / 20 / 1e3
        by = rows * D * (4 + 2 * k + 4 + 2)
        res[f"k{k}_mode{mode}"] = {"us": round(t * 1e6, 1), "GBs": round(by / t / 1e9)}
print(json.dumps(res))

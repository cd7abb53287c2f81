"""TF/s of the projection GEMMs at C3 shapes (cuBLAS / cuBLASLt via torch)."""
import json
import torch
rows, D, R = 49920, 1152, 4608
def t(fn, n=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n / 1e3
bf = dict(device="cuda", dtype=torch.bfloat16)
h = torch.randn(rows, D, **bf); hid = torch.randn(rows, R, **bf)
wqkv = torch.randn(D, 3 * D, **bf) * 0.03; wo = torch.randn(D, D, **bf) * 0.03
w1 = torch.randn(D, R, **bf) * 0.03; w2 = torch.randn(R, D, **bf) * 0.03; zb = torch.zeros(R, **bf)
o3 = torch.empty(rows, 3 * D, **bf); o1 = torch.empty(rows, D, **bf)
res = {}
for name, fn, fl in [
    ("qkv", lambda: torch.mm(h, wqkv, out=o3), 2 * rows * D * 3 * D),
    ("o_proj", lambda: torch.mm(h, wo, out=o1), 2 * rows * D * D),
    ("w1_gelu_lt", lambda: torch._addmm_activation(zb, h, w1, use_gelu=True), 2 * rows * D * R),
    ("w2", lambda: torch.mm(hid, w2, out=o1), 2 * rows * R * D),
]:
    s = t(fn)
    res[name] = {"ms": round(s * 1e3, 3), "tflops": round(fl / s / 1e12, 1)}
print(json.dumps(res))

"""Library comparison points for the C3/C5 spatial attention shape (not product code):
torch SDPA backends (cuDNN, FlashAttention-2) vs our tcgen05 kernel.

    python scripts/sdpa_compare.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

res = {}
for name, (B, T, S) in {"C3": (2, 16, 1560), "C5": (2, 32, 3600)}.items():
    H, dh = 16, 72
    n = B * T
    q = torch.randn(n, H, S, dh, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    f = 4.0 * n * H * S * S * dh
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION):
        try:
            with sdpa_kernel([be]):
                for _ in range(3):
                    torch.nn.functional.scaled_dot_product_attention(q, k, v)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    torch.nn.functional.scaled_dot_product_attention(q, k, v)
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 10 / 1e3
                res[f"{name}_{be.name}"] = {"ms": t * 1e3, "tflops": f / t / 1e12}
        except Exception as e:  # noqa: BLE001
            res[f"{name}_{be.name}"] = {"error": str(e)[:200]}
print(json.dumps(res))

"""One projection GEMM shape on the tcgen05 kernel, for ncu captures:
    python scripts/prof_gemm.py w2|o|qkv|w1 [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12588_b200 import kernels  # noqa: E402

rows, D, R = 49920, 1152, 4608
shape = {"qkv": (D, 3 * D, 0), "o": (D, D, 0), "w1": (D, R, 1), "w2": (R, D, 0)}[sys.argv[1]]
K, N, epi = shape
bf = dict(device="cuda", dtype=torch.bfloat16)
a = torch.randn(rows, K, **bf)
w = torch.randn(N, K, **bf) * 0.03
c = torch.empty(rows, N, **bf)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    kernels.gemm(a, w, c, epi)
torch.cuda.synchronize()

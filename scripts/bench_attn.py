"""Microbenchmark of the attention kernels at C3 shapes (CUDA events, warm).

    python scripts/bench_attn.py [--config C3] [--impl 1]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS, load_peaks  # noqa: E402
from paper_2408_12588_b200 import kernels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--impl", type=int, default=1)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
c = CONFIGS[args.config]
B, T, S, D, H, M = c["batch"], c["frames"], c["spatial_tokens"], c["hidden"], c["heads"], c["text_tokens"]
dh = D // H
rows = B * T * S
qkv = torch.randn(rows, 3 * D, device="cuda").to(torch.bfloat16)
out = torch.empty(rows, D, device="cuda", dtype=torch.bfloat16)
kv = torch.randn(B * M, 2 * D, device="cuda").to(torch.bfloat16)
ld = 3 * D
q, k, v = qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:]
sp = kernels.attn_args(q, k, v, out, (S * ld, 0, ld), (S * ld, 0, ld), (S * ld, 0, ld), (S * D, 0, D), B * T, 1, S, S,
                       H, dh)
# temporal site layout used by the engine: token-major rows (b, s, t)
st = (0, T * ld, ld)
tm = kernels.attn_args(q, k, v, out, st, st, st, (0, T * D, D), 1, B * S, T, T, H, dh)
cr = kernels.attn_args(q, kv[:, :D], kv[:, D:], out, (T * S * ld, 0, ld), (M * 2 * D, 0, 2 * D),
                       (M * 2 * D, 0, 2 * D), (T * S * D, 0, D), B, 1, T * S, M, H, dh)
peaks, _ = load_peaks()


def timeit(a):
    for _ in range(3):
        kernels.attention(a, args.impl)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        kernels.attention(a, args.impl)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / args.reps / 1e3


res = {}
t = timeit(sp)
f = 4.0 * B * T * S * S * D
res["spatial"] = {"us": t * 1e6, "tflops": f / t / 1e12, "frac": f / t / 1e12 / peaks["bf16_tflops"]}
t = timeit(tm)
by = 8.0 * rows * D
res["temporal"] = {"us": t * 1e6, "gbs": by / t / 1e9, "frac_hbm": by / t / 1e9 / peaks["hbm_gbs"]}
t = timeit(cr)
f = 4.0 * rows * M * D
by = 4.0 * rows * D + 4.0 * B * M * D
res["cross"] = {"us": t * 1e6, "tflops": f / t / 1e12, "gbs": by / t / 1e9, "frac": f / t / 1e12 / peaks["bf16_tflops"]}
print(json.dumps(res))

"""Locate wrong rows of the row-per-thread attention kernel (debug helper)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_12588_b200 import kernels  # noqa: E402

B, T, S, H, dh = [int(x) for x in sys.argv[1:6]]
impl = int(sys.argv[6]) if len(sys.argv) > 6 else 1
D = H * dh
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(B * T * S, 3 * D, device="cuda", generator=g).to(torch.bfloat16)
out = torch.full((B * T * S, D), float("nan"), device="cuda", dtype=torch.bfloat16)
ld = 3 * D
a = kernels.attn_args(qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:], out, (S * ld, 0, ld), (S * ld, 0, ld),
                      (S * ld, 0, ld), (S * D, 0, D), B * T, 1, S, S, H, dh)
kernels.attention(a, impl)
torch.cuda.synchronize()
x = qkv.view(B * T, S, 3, H, dh).permute(2, 0, 3, 1, 4).float()
s = (x[0] @ x[1].transpose(-1, -2)) / math.sqrt(dh)
want = (torch.softmax(s, -1) @ x[2])  # (BT, H, S, dh)
got = out.view(B * T, S, H, dh).permute(0, 2, 1, 3).float()
err = (got - want).abs().amax(-1)  # (BT, H, S)
bad = (err > 0.05) | ~torch.isfinite(err)
print("rel", float((got - want).norm() / want.norm()), "bad rows", int(bad.sum()), "of", bad.numel())
idx = bad.nonzero()
if len(idx):
    print("bad (problem, head) pairs:", sorted(set((int(i[0]), int(i[1])) for i in idx))[:40])
    rows = sorted(set(int(i[2]) // 128 for i in idx))
    print("bad query tiles:", rows)
    # item = (pair, head) order, head fastest: item index -> CTA = item % 148
    items = sorted(set(((int(i[0]) * ((S + 255) // 256) + int(i[2]) // 256) * H + int(i[1])) for i in idx))
    print("bad items:", items[:40], "ctas:", sorted(set(it % 148 for it in items))[:40])

"""clock64 timeline of CTA 0 of the packed temporal kernel (attn_tc.cu), per item
(library built with -DPAB_ATTN_TRACE).  python scripts/tc_timeline.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_12588_b200 import _lib, kernels  # noqa: E402

B, T, S, D, H = 2, 16, 1560, 1152, 16
dh = D // H
rows = B * T * S
qkv = torch.randn(rows, 3 * D, device="cuda").to(torch.bfloat16)
out = torch.empty(rows, D, device="cuda", dtype=torch.bfloat16)
ld = 3 * D
st = (0, T * ld, ld)
a = kernels.attn_args(qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:], out, st, st, st, (0, T * D, D), 1, B * S, T, T,
                      H, dh)
buf = torch.zeros(64 * 2 * 16, dtype=torch.int64, device="cuda")
lib = _lib.load()
for _ in range(3):
    kernels.attention(a)
lib.pab_attn_debug_trace(buf.data_ptr())
kernels.attention(a)
torch.cuda.synchronize()
lib.pab_attn_debug_trace(None)
tr = buf.view(64, 2, 16).cpu()
t0 = int(tr[tr > 0].min())
names = {0: "wait_S", 1: "S_ready", 2: "max_done", 3: "xchg_done", 4: "resc_done", 6: "S_loaded2", 7: "exp_done",
         5: "P_written", 8: "epi_start", 9: "epi_done"}
ev = []
for c in range(int(os.environ.get("TL_ITEMS", "8"))):
    for t in range(2):
        for e, nm in names.items():
            v = int(tr[c, t, e])
            if v:
                ev.append((v - t0, c, t, nm))
prev = 0
for v, c, t, nm in sorted(ev):
    print(f"{v:8d} (+{v - prev:5d})  item={c:2d} t={t}  {nm}")
    prev = v

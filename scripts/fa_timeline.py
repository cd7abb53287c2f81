"""Print the clock64 event timeline of CTA 0 of the row-per-thread attention kernel
(library built with -DPAB_FA_TRACE, e.g. scripts/build_variant.sh trace -DPAB_FA_TRACE)."""
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
a = kernels.attn_args(qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:], out, (S * ld, 0, ld), (S * ld, 0, ld),
                      (S * ld, 0, ld), (S * D, 0, D), B * T, 1, S, S, H, dh)
if len(sys.argv) > 1 and sys.argv[1] == "cross":  # C3 cross site: 300 text keys per batch entry
    M = 300
    kv = torch.randn(B * M, 2 * D, device="cuda").to(torch.bfloat16)
    a = kernels.attn_args(qkv[:, :D], kv[:, :D], kv[:, D:], out, (T * S * ld, 0, ld), (M * 2 * D, 0, 2 * D),
                          (M * 2 * D, 0, 2 * D), (T * S * D, 0, D), B, 1, T * S, M, H, dh)
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
names = {6: "sm:item_top", 7: "sm:decoded", 0: "sm:wait_S", 1: "sm:S_ready", 2: "sm:S_loaded", 3: "sm:max_done", 4: "sm:exp_done", 5: "sm:p_full"}
# MMA events are logged under tile 0 (S issue) / tile 1 (PV issue)
mma_names = {(0, 10): "mma:wait_sfree", (0, 8): "mma:S_go", (1, 10): "mma:wait_P", (1, 8): "mma:PV_go",
             (1, 9): "mma:PV_issued"}
ev = []
for j in range(int(os.environ.get("TL_ITERS", "30"))):
    for t in range(2):
        for e, nm in names.items():
            v = int(tr[j, t, e])
            if v:
                ev.append((v - t0, j, t, nm))
        for (tt, e), nm in mma_names.items():
            v = int(tr[j, tt, e])
            if tt == t and v:
                ev.append((v - t0, j, t, nm))
prev = 0
for v, j, t, nm in sorted(ev):
    print(f"{v:8d} (+{v - prev:5d})  it={j:2d} t={t}  {nm}")
    prev = v

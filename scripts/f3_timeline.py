"""clock64 event timeline of CTA 0 of the three-tile attention kernel (impl 3), library built
with -DPAB_F3_TRACE (scripts/build_variant.sh f3trace -DPAB_F3_TRACE); C3 spatial shape."""
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
buf = torch.zeros(40 * 4 * 8, dtype=torch.int64, device="cuda")
lib = _lib.load()
for _ in range(3):
    kernels.attention(a, 3)
lib.pab_attn_debug_trace(buf.data_ptr())
kernels.attention(a, 3)
torch.cuda.synchronize()
lib.pab_attn_debug_trace(None)
tr = buf.view(40, 4, 8).cpu()
t0 = int(tr[tr > 0].min())
names = {0: "wait_S", 1: "S_ready", 2: "S_loaded", 3: "max_done", 4: "exp_done", 5: "p_full"}
ev = []
for j in range(int(os.environ.get("TL_ITERS", "12"))):
    for t in range(3):
        for e, nm in names.items():
            v = int(tr[j, t, e])
            if v:
                ev.append((v - t0, j, t, nm))
    # MMA warp (slot 3, indexed by KV tile g == iteration here)
    for e, nm in enumerate(["mma:top", "mma:v_ready", "mma:PV0_go", "mma:PV0_done", "mma:k_ready", "mma:S0_done",
                            "mma:S1_done", "mma:S2_done"]):
        v = int(tr[j, 3, e])
        if v:
            ev.append((v - t0, j, 3, nm))
prev = 0
for v, j, t, nm in sorted(ev):
    print(f"{v:8d} (+{v - prev:5d})  it={j:2d} t={t}  {nm}")
    prev = v

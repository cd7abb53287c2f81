"""Print the clock64 event timeline of CTA (0,0,0) of the C3 spatial attention kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_12588_b200 import _lib, kernels  # noqa: E402

B, T, S, D, H = 2, 16, int(sys.argv[1]) if len(sys.argv) > 1 else 1560, 1152, 16
dh = D // H
rows = B * T * S
qkv = torch.randn(rows, 3 * D, device="cuda").to(torch.bfloat16)
out = torch.empty(rows, D, device="cuda", dtype=torch.bfloat16)
ld = 3 * D
a = kernels.attn_args(qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:], out, (S * ld, 0, ld), (S * ld, 0, ld),
                      (S * ld, 0, ld), (S * D, 0, D), B * T, 1, S, S, H, dh)
n_kv = (S + 127) // 128
buf = torch.zeros(n_kv * 2 * 16, dtype=torch.int64, device="cuda")
lib = _lib.load()
for _ in range(3):
    kernels.attention(a)
lib.pab_attn_debug_trace(buf.data_ptr())
kernels.attention(a)
torch.cuda.synchronize()
lib.pab_attn_debug_trace(None)
tr = buf.view(n_kv, 2, 16).cpu()
t0 = int(tr[tr > 0].min())
names = {0: "sm:wait_S", 1: "sm:S_ready", 2: "sm:pass1_done", 3: "sm:xchg_done", 4: "sm:o_done/resc", 5: "sm:P_written", 6: "sm:pass2_loaded", 7: "sm:pass2_exp_done",
         8: "mma:wait_sfree", 9: "mma:sfree_ok", 10: "mma:wait_P", 11: "mma:P_ok", 12: "mma:PV_issued"}
ev = []
for j in range(n_kv):
    for t in range(2):
        for e, nm in names.items():
            v = int(tr[j, t, e])
            if v:
                ev.append((v - t0, j, t, nm))
WARPS = os.environ.get('TL_ALL')
for v, j, t, nm in sorted(ev):
    print(f"{v:8d}  j={j:2d} t={t}  {nm}")

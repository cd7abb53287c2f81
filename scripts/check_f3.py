"""A/B of the three-tile attention kernel (impl 3) against the two-tile one (impl 1):
parity against a torch fp32 reference and timing at the C3 spatial / cross shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_12588_b200 import kernels  # noqa: E402


def ref(q, k, v, n_p, n_q, n_k, H, dh):
    qh = q.float().view(n_p, n_q, H, dh).transpose(1, 2)
    kh = k.float().view(n_p, n_k, H, dh).transpose(1, 2)
    vh = v.float().view(n_p, n_k, H, dh).transpose(1, 2)
    return (torch.softmax(qh @ kh.transpose(-1, -2) / dh ** 0.5, -1) @ vh).transpose(1, 2).reshape(n_p * n_q, H * dh)


def case(name, n_p, n_q, n_k, H, dh, reps=20):
    D = H * dh
    g = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn(n_p * n_q, D, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(n_p * n_k, D, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(n_p * n_k, D, device="cuda", generator=g).to(torch.bfloat16)
    want = ref(q, k, v, n_p, n_q, n_k, H, dh)
    res = {}
    for impl in (1, 3):
        out = torch.full((n_p * n_q, D), float("nan"), device="cuda", dtype=torch.bfloat16)
        a = kernels.attn_args(q, k, v, out, (n_q * D, 0, D), (n_k * D, 0, D), (n_k * D, 0, D), (n_q * D, 0, D),
                              n_p, 1, n_q, n_k, H, dh)
        kernels.attention(a, impl)
        torch.cuda.synchronize()
        rel = float((out.float() - want).norm() / want.norm())
        fin = bool(torch.isfinite(out.float()).all())
        for _ in range(3):
            kernels.attention(a, impl)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            kernels.attention(a, impl)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        flop = 4.0 * n_p * n_q * n_k * D
        res[impl] = (rel, fin, us, flop / us / 1e6)
    print(name, " ".join(f"impl{i}: rel {r:.2e} finite {f} {us:.1f} us {tf:.0f} TF/s" for i, (r, f, us, tf) in res.items()),
          flush=True)


for shape in sys.argv[1:] or ["small", "spatial", "cross"]:
    if shape == "small":
        case("small", 2, 300, 200, 2, 72)
        case("small64", 2, 260, 170, 2, 64)
        case("tiny", 1, 100, 30, 1, 72)
    if shape == "spatial":
        case("C3 spatial", 32, 1560, 1560, 16, 72)
    if shape == "cross":
        case("C3 cross", 1, 24960, 300, 16, 72)

"""Spatial/cross attention launch time on real engine activations vs random inputs
(C3 shapes): the lazy-rescale softmax path is data dependent.

    python scripts/attn_realdata.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, model_config  # noqa: E402
from paper_2408_12588_b200 import kernels  # noqa: E402
from paper_2408_12588_b200.diffusion import Denoiser, initial_latent, make_schedule  # noqa: E402
from paper_2408_12588_b200.model import init_model  # noqa: E402
from paper_2408_12588_b200.policies import NonePolicy, build_schedule  # noqa: E402


def timeit(a, reps=20):
    kernels.attention(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        kernels.attention(a)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


c = CONFIGS["C3"]
cfg = model_config(c)
params = init_model(cfg, seed=11)
sched = make_schedule(2)  # two steps: the last computed site leaves real activations in the workspaces
table = build_schedule(NonePolicy(), sched, cfg.layers)
den = Denoiser(params, sched, table, np.arange(cfg.text_tokens) % 256, guidance=True, guidance_scale=4.0)
z = torch.from_numpy(initial_latent(params, 11, 2)).cuda()
den.run(z)
ctx = den.ctx
torch.cuda.synchronize()
time.sleep(2.0)
real_sp = timeit(ctx.args_spatial)
real_cr = timeit(ctx.args_cross[0][0])
qkv_std = float(ctx.qkv.float().std())
saved = ctx.qkv.clone()
ctx.qkv.copy_(torch.randn_like(ctx.qkv, dtype=torch.float32).to(torch.bfloat16))
time.sleep(2.0)
rand_sp = timeit(ctx.args_spatial)
rand_cr = timeit(ctx.args_cross[0][0])
ctx.qkv.copy_(saved * 4.0)
time.sleep(2.0)
x4_sp = timeit(ctx.args_spatial)
print(f"spatial: real {real_sp:.1f} us, randn {rand_sp:.1f} us, real x4 {x4_sp:.1f} us (qkv std {qkv_std:.3f})")
print(f"cross:   real {real_cr:.1f} us, randn {rand_cr:.1f} us")

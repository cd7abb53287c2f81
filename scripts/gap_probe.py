"""Kernel busy time vs wall time of one C3 video (torch.profiler / CUPTI): how much
a CUDA graph of the step loop could recover (inter-kernel gaps, host launch stalls).

    python scripts/gap_probe.py [--config C3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from bench import CONFIGS, model_config  # noqa: E402
from paper_2408_12588_b200.diffusion import Denoiser, initial_latent, make_schedule  # noqa: E402
from paper_2408_12588_b200.model import init_model  # noqa: E402
from paper_2408_12588_b200.policies import build_schedule, resolve_preset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
args = ap.parse_args()
c = CONFIGS[args.config]
cfg = model_config(c)
params = init_model(cfg, seed=11)
sched = make_schedule(c["steps"])
pol, _ = resolve_preset(c["preset"], cfg.layers)
table = build_schedule(pol, sched, cfg.layers)
den = Denoiser(params, sched, table, np.arange(cfg.text_tokens) % 256, guidance=c["batch"] == 2, guidance_scale=4.0)
x0 = torch.from_numpy(initial_latent(params, 11, c["batch"])).cuda()
z = x0.clone()
den.run(z)
torch.cuda.synchronize()
z.copy_(x0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    den.run(z)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.device_resource_id is not None]
iv = sorted((e.time_range.start, e.time_range.end) for e in ev if e.time_range.end > e.time_range.start)
busy, cur_s, cur_e = 0.0, None, None
for s, e in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
wall = iv[-1][1] - iv[0][0]
print(f"kernels {len(iv)}  wall {wall / 1e3:.1f} ms  busy {busy / 1e3:.1f} ms  gaps {(wall - busy) / 1e3:.1f} ms "
      f"({(wall - busy) / wall * 100:.2f}%)")

"""Run ONE denoising step of a workload between cudaProfilerStart/Stop so ncu
(--profile-from-start off) sees exactly that step's launches.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python scripts/profile_step.py --config C3 --step 4
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, model_config  # noqa: E402
from paper_2408_12588_b200.diffusion import Denoiser, initial_latent, make_schedule  # noqa: E402
from paper_2408_12588_b200.model import init_model  # noqa: E402
from paper_2408_12588_b200.policies import build_schedule, resolve_preset  # noqa: E402
from paper_2408_12588_b200.runtime import run_forward  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--step", type=int, default=0, help="denoising step to profile (0 = all sites computed)")
ap.add_argument("--policy", default=None)
args = ap.parse_args()
c = CONFIGS[args.config]
cfg = model_config(c)
params = init_model(cfg, seed=11)
sched = make_schedule(c["steps"])
pol, _ = resolve_preset(args.policy or c["preset"], cfg.layers)
table = build_schedule(pol, sched, cfg.layers)
den = Denoiser(params, sched, table, np.arange(cfg.text_tokens) % 256, guidance=c["batch"] == 2,
               guidance_scale=4.0)
z = torch.from_numpy(initial_latent(params, 11, c["batch"])).cuda()
r = torch.empty_like(z)
# warm up: every step before the profiled one (fills the broadcast cache)
for i in range(args.step + 1):
    a_cur, a_next = den.alphas[i]
    run_forward(den.ctx, i, den.timesteps[i], z, r, table.slice(i), den.cache, finish="ddim",
                ddim=(den.guidance, den.g, a_cur, a_next))
torch.cuda.synchronize()
i = args.step
a_cur, a_next = den.alphas[i]
torch.cuda.profiler.start()
run_forward(den.ctx, i, den.timesteps[i], z, r, table.slice(i), den.cache, finish="ddim",
            ddim=(den.guidance, den.g, a_cur, a_next))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
comp = table.compute_mask()[i]
print("profiled step", i, "compute per kind (spatial, temporal, cross, mlp):", comp.sum(axis=0).tolist())

"""Generate tests/golden/<name>_deep.npz: a multi-layer run of the CPU oracle at full
width over a config's whole PAB schedule (CFG batch 2, g = 4, seed 11), for the GPU
deep-parity tests (tests/test_fullshape_gpu.py).  The decision table is the preset's
(policies.resolve_preset + build_schedule, bit-exact with the reference).  Stored per
step: latent norm, max|x| and a strided 8192-element subsample.

    OMP_NUM_THREADS=8 python tests/golden/make_deep.py c2      (C2: L4 of 28, D1152 H16 T16 S1024 M120, 50 steps)
    OMP_NUM_THREADS=8 python tests/golden/make_deep.py c3      (same as make_c3_deep.py)
    OMP_NUM_THREADS=8 python tests/golden/make_deep.py c4      (C4: L2 of 28, S1024 M300, no temporal cross, 150 steps)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pab_oracle as orc  # noqa: E402
from paper_2408_12588_b200.diffusion import make_schedule  # noqa: E402  (host-only: schedule / tables)
from paper_2408_12588_b200.policies import build_schedule, resolve_preset  # noqa: E402

CONFIGS = {  # name: (L, D, H, T, S, M, cross_in_temporal, steps, preset)
    "c2": (4, 1152, 16, 16, 1024, 120, False, 50, "latte-pab235"),
    "c3": (4, 1152, 16, 16, 1560, 300, True, 30, "opensora-pab246"),
    "c4": (2, 1152, 16, 16, 1024, 300, False, 150, "opensoraplan-pab246"),
}


def main(name):
    L, D, H, T, S, M, cit, N, preset = CONFIGS[name]
    cfg = orc.Cfg(L, D, H, T, S, M, cross_in_temporal=cit)
    w = orc.init_weights(cfg, 11)
    pol, _ = resolve_preset(preset, L)
    table = build_schedule(pol, make_schedule(N), L).source
    n = 2 * T * S * D
    idx = np.arange(0, n, n // 8192)[:8192]
    norms, maxabs, subs = [], [], []
    t0 = time.time()

    class Rec(list):
        # reduce each step's latent right away (150 full C4 latents would need 23 GB)
        def append(self, x):
            super().append(None)
            flat = x.reshape(-1)
            norms.append(float(np.linalg.norm(flat.astype(np.float64))))
            maxabs.append(float(np.abs(flat).max()))
            subs.append(flat[idx].copy())
            print(f"step {len(subs)} done at {time.time() - t0:.0f} s", flush=True)

    orc.sample(cfg, w, orc.linear_timesteps(N), table, seed=11, text_ids=np.arange(M) % 256, guidance=True,
               per_step=Rec())
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"{name}_deep.npz"),
                        norms=np.array(norms), maxabs=np.array(maxabs, dtype=np.float32), idx=idx,
                        sub=np.stack(subs), table=table, layers=L, steps=N,
                        config=np.array([L, D, H, T, S, M, int(cit), N]))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c2")

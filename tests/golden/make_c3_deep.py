"""Generate tests/golden/c3_deep.npz: a multi-layer C3 (Open-Sora 2s 480p) run of
the CPU oracle at full width -- L=4 of the 28 layers, D1152 H16 T16 S1560 M300,
cross attention in the temporal block, CFG batch 2 (g=4), opensora-pab246 over
the full 30-step schedule, seed 11.  The oracle is pinned to the reference at
small sizes (tests/test_oracle.py); the reference itself would need days for
this run (SURVEY.md 7 hard part 6).  Stored per step: latent norm, max|x| and a
strided 8192-element subsample (the full latent is 230 MB per step).

    OMP_NUM_THREADS=8 python tests/golden/make_c3_deep.py      (~1-2 h on 8 cores)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pab_oracle as orc  # noqa: E402

L, N = 4, 30


def main():
    cfg = orc.Cfg(L, 1152, 16, 16, 1560, 300, cross_in_temporal=True)
    w = orc.init_weights(cfg, 11)
    ts = orc.linear_timesteps(N)
    # opensora-pab246 (reference policies.py:454-534): ranges (2, 4, 6), window [930, 450],
    # MLP triggers 864/788/676 on blocks 0-4 (filtered to < L), range 2
    table = orc.table_pab(ts, L, (2, 4, 6), (930.0, 450.0), mlp=([864.0, 788.0, 676.0], [0, 1, 2, 3], 2))
    per = []
    t0 = time.time()

    class Rec(list):
        def append(self, x):
            super().append(None)
            per.append(x)
            print(f"step {len(per)} done at {time.time() - t0:.0f} s", flush=True)

    orc.sample(cfg, w, ts, table, seed=11, text_ids=np.arange(300) % 256, guidance=True, per_step=Rec())
    flat = np.stack([p.reshape(-1) for p in per])
    idx = np.arange(0, flat.shape[1], flat.shape[1] // 8192)[:8192]
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c3_deep.npz"),
                        norms=np.linalg.norm(flat.astype(np.float64), axis=1), maxabs=np.abs(flat).max(axis=1),
                        idx=idx, sub=flat[:, idx], table=table, layers=L, steps=N)


if __name__ == "__main__":
    main()

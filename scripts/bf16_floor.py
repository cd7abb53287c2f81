"""Measure the bf16 precision floor of the PAB sampler: the oracle
with every matmul operand/output rounded to bf16 vs the fp32 oracle, per denoising
step (relL2 and max|d|/max|ref|).  The guided (CFG) parity gates in tests/ are set
at 1.5x the floor measured here.

    python scripts/bf16_floor.py smoke|dh72|c1|c2slice|c3slice|c4slice
"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from oracle import pab_oracle as orc  # noqa: E402


def table_smoke(n, L):
    return orc.table_pab(orc.linear_timesteps(n), L, (2, 3, 4), (990.0, 10.0))


def forced(n, L, reuse_step=2, src=1):
    t = np.repeat(np.arange(n, dtype=np.int32)[:, None], L, 1)[:, :, None].repeat(4, 2)
    t[reuse_step] = src
    return t


CASES = {
    # name: (Cfg args, steps, table fn, guidance, M)
    "smoke": ((2, 144, 2, 8, 256, 20, 4.0, True), 5, table_smoke, True),
    "smoke_u": ((2, 144, 2, 8, 256, 20, 4.0, True), 5, table_smoke, False),
    "dh72": ((2, 288, 4, 4, 128, 24, 4.0, True), 6, table_smoke, True),
    "c1": ((4, 144, 2, 8, 1024, 16, 4.0, False), 10, None, False),
    "c2slice": ((1, 1152, 16, 16, 1024, 120, 4.0, False), 4, None, True),
    "c3slice": ((1, 1152, 16, 16, 1560, 300, 4.0, True), 3, lambda n, L: forced(n, L), True),
    "c4slice": ((1, 1152, 16, 16, 1024, 300, 4.0, False), 3, lambda n, L: forced(n, L), True),
}


def c2_table(n, L):
    src = np.repeat(np.arange(n, dtype=np.int32)[:, None], L, 1)[:, :, None].repeat(4, 2)
    src[2, 0, 0] = 1
    src[3, 0, 1] = 1
    src[3, 0, 2] = 2
    return src


def c1_table(n, L):
    return orc.table_pab(orc.linear_timesteps(n), L, (2, 3, 5), (800.0, 100.0),
                         mlp=([720.0, 640.0, 560.0, 480.0, 400.0], [0, 1, 2, 3], 2))


def floor(name):
    args, n, tfn, guided = CASES[name]
    tfn = tfn or {"c1": c1_table, "c2slice": c2_table}[name]
    cfg = orc.Cfg(*args[:7], cross_in_temporal=args[7])
    w = orc.init_weights(cfg, 11)
    table = tfn(n, cfg.L)
    ts = orc.linear_timesteps(n)
    ids = np.arange(cfg.M) % 256
    t0 = time.time()
    ref, emu = [], []
    orc.sample(cfg, w, ts, table, seed=11, text_ids=ids, guidance=guided, per_step=ref)
    orc.sample(cfg, w, ts, table, seed=11, text_ids=ids, guidance=guided, per_step=emu, emulate_bf16=True)
    rows = []
    for i, (a, b) in enumerate(zip(emu, ref)):
        a64, b64 = a.astype(np.float64), b.astype(np.float64)
        rel = np.linalg.norm(a64 - b64) / np.linalg.norm(b64)
        mx = np.abs(a64 - b64).max() / np.abs(b64).max()
        rows.append((i, rel, mx))
    return rows, time.time() - t0


if __name__ == "__main__":
    for name in sys.argv[1:] or ["smoke"]:
        rows, dt = floor(name)
        worst = max(r[1] for r in rows), max(r[2] for r in rows)
        print(f"{name}: worst relL2 {worst[0]:.3e} max {worst[1]:.3e} ({dt:.0f} s) per step: "
              + " ".join(f"{r:.2e}/{m:.2e}" for _, r, m in rows), flush=True)

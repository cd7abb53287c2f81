"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
pab-engine (pure Python, importable from /root/reference/pkg/src in the build
container; it does not exist on the GPU box).

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (small, committed):
  decisions.npz     reference build_schedule tables for every preset x
                    (steps, layers) used by the configs C1-C5 + desk/small,
                    and for 100 random policies (seeds 20240811 / 77)
  decisions.json    the policies/configs those tables came from
  prng.npz          RandomStream uniform/normal vectors for a few seeds
  small_runs.npz    per-step latents of reference sample() loops on tiny configs
                    (none / PAB / T-GATE / Delta-DiT, with and without CFG) and
                    the per-site decision log
  c1_run.npz        C1 (tiny Latte-style) latte-pab235 10-step run: per-step
                    latent norms + a strided 4096-element subsample per step
  traces.npz        full-depth per-site decision traces (TraceRecord decision /
                    source_step) of C2/C3/C4/C5 runs with their presets: L=28 and
                    the configs' step counts, CFG; decisions do not depend on the
                    hidden size, so the model is shrunk to D=8 (python run time)
"""

from __future__ import annotations

import json
import math
import os
import random
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT = os.path.dirname(os.path.abspath(__file__))

sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True

from oracles import random_policy  # noqa: E402  (reference test helper)
from pab_engine import diffusion as rd  # noqa: E402
from pab_engine import model as rm  # noqa: E402
from pab_engine import numerics as rn  # noqa: E402
from pab_engine import policies as rp  # noqa: E402

CONFIGS = {
    # name: (layers, steps, preset family default)
    "desk": (4, 30), "small": (2, 6), "C1": (4, 10), "C2": (28, 50), "C3": (28, 30), "C4": (28, 150), "C5": (28, 30),
}


def decisions():
    tables, meta = {}, {"presets": [], "random": []}
    for cname, (layers, steps) in CONFIGS.items():
        sched = rd.make_schedule(steps)
        for name in rp.PRESET_NAMES:
            pol, notes = rp.resolve_preset(name, layers)
            for sem in ("period", "reuse-count"):
                try:
                    t = rp.build_schedule(pol, sched, layers, range_semantics=sem)
                except Exception as e:  # gate beyond steps etc.
                    meta["presets"].append({"config": cname, "preset": name, "semantics": sem, "error": e.kind})
                    continue
                key = f"{cname}|{name}|{sem}"
                tables[key] = t.source
                meta["presets"].append({"config": cname, "preset": name, "semantics": sem, "key": key,
                                        "layers": layers, "steps": steps, "delta": t.delta_mode,
                                        "policy": rp.policy_to_dict(pol), "notes": notes})
    for seed in (20240811, 77):
        rng = random.Random(seed)
        for j in range(100):
            n = rng.randint(1, 60)
            layers = rng.randint(1, 6)
            sem = rng.choice(["period", "reuse-count"])
            pol = random_policy(rng, n, layers)
            ts = [1000.0 * (1.0 - i / n) for i in range(n)]
            t = rp.build_schedule(pol, ts, layers, range_semantics=sem)
            key = f"random|{seed}|{j}"
            tables[key] = t.source
            meta["random"].append({"key": key, "n": n, "layers": layers, "semantics": sem, "delta": t.delta_mode,
                                   "policy": rp.policy_to_dict(pol)})
    np.savez_compressed(os.path.join(OUT, "decisions.npz"), **tables)
    with open(os.path.join(OUT, "decisions.json"), "w") as fh:
        json.dump(meta, fh, indent=0)


def prng():
    out = {}
    for seed in (0, 11, 2024, 2**63 + 5):
        s = rn.RandomStream(seed)
        out[f"uniform_{seed}"] = s.uniform(257, -0.125, 0.125)
        out[f"normal_{seed}"] = s.normal(301)
        out[f"u64_{seed}"] = np.array([s.next_u64() for _ in range(5)], dtype=np.uint64)
    np.savez_compressed(os.path.join(OUT, "prng.npz"), **out)


def _loop(params, sched, table, seed, guidance, ids=None, broadcast_object="outputs"):
    """Reference forward_step + ddim_update, recording every step's latent."""
    cfg = params.cfg
    ids = rd.default_text_ids(params) if ids is None else ids
    batch = 2 if guidance else 1
    x = rd.initial_latent(params, seed, batch)
    ids2 = np.stack([ids, np.full_like(ids, -1)]) if guidance else ids[None]
    cache = rp.CacheStore()
    trace = rm.ComponentTrace(snapshot_mode="none")
    steps = []
    ts = sched.timesteps
    for i, t in enumerate(ts):
        eps = rm.forward_step(params, x, t, ids2, table.slice(i), cache, trace=trace,
                              broadcast_object=broadcast_object)
        if guidance:
            eps = eps[1:2] + 4.0 * (eps[0:1] - eps[1:2])
        a = rd.DEFAULT_NOISE.alpha_bar(t)
        an = rd.DEFAULT_NOISE.alpha_bar(ts[i + 1]) if i + 1 < len(ts) else 1.0
        x = rd.ddim_update(x, eps, a, an)
        steps.append(x.copy())
    log = np.array([[r.step, r.layer, rm.KIND_INDEX[r.kind], 0 if r.block == "s" else 1,
                     {"compute": 0, "reuse": 1, "delta": 2}[r.decision], r.source_step] for r in trace.records],
                   dtype=np.int32)
    return np.stack(steps), log


def small_runs():
    out = {}
    cases = {
        "small": rm.ModelConfig(layers=2, hidden=32, heads=4, frames=4, spatial_tokens=16, text_tokens=8),
        "smallx": rm.ModelConfig(layers=2, hidden=48, heads=2, frames=4, spatial_tokens=24, text_tokens=5,
                                 cross_in_temporal=True),
    }
    policies = {
        "none": rp.NonePolicy(),
        "pab": rp.PabPolicy(2, 4, 3, window=(990.0, 10.0),
                            mlp=rp.MlpBroadcast(triggers=(700.0,), blocks=(0,), range=2)),
        "tgate": rp.TGatePolicy(gate_step=4, interval=2, warmup=1),
        "deltadit": rp.DeltaDitPolicy(gate_step=5, interval=2, block_range=(0, 0)),
    }
    meta = {}
    for cname, cfg in cases.items():
        params = rm.init_model(cfg, seed=3)
        sched = rd.make_schedule(8)
        for pname, pol in policies.items():
            for guidance in (False, True):
                table = rp.build_schedule(pol, sched, cfg.layers)
                lat, log = _loop(params, sched, table, seed=7, guidance=guidance)
                key = f"{cname}|{pname}|{int(guidance)}"
                out[key + "|latents"] = lat.astype(np.float32)
                out[key + "|log"] = log
                out[key + "|table"] = table.source
                meta[key] = {"policy": rp.policy_to_dict(pol), "delta": table.delta_mode}
        meta[cname] = {"layers": cfg.layers, "hidden": cfg.hidden, "heads": cfg.heads, "frames": cfg.frames,
                       "spatial_tokens": cfg.spatial_tokens, "text_tokens": cfg.text_tokens,
                       "cross_in_temporal": cfg.cross_in_temporal, "param_digest": params.digest()}
    np.savez_compressed(os.path.join(OUT, "small_runs.npz"), **out)
    with open(os.path.join(OUT, "small_runs.json"), "w") as fh:
        json.dump(meta, fh, indent=0)


def scores_runs():
    """broadcast_object="scores" (attention sites cache probabilities, model.py:469-499)."""
    out = {}
    cases = {
        "small": rm.ModelConfig(layers=2, hidden=32, heads=4, frames=4, spatial_tokens=16, text_tokens=8),
        "smallx": rm.ModelConfig(layers=2, hidden=48, heads=2, frames=4, spatial_tokens=24, text_tokens=5,
                                 cross_in_temporal=True),
    }
    policies = {
        "pab": rp.PabPolicy(2, 4, 3, window=(990.0, 10.0),
                            mlp=rp.MlpBroadcast(triggers=(700.0,), blocks=(0,), range=2)),
        "tgate": rp.TGatePolicy(gate_step=4, interval=2, warmup=1),
    }
    meta = {}
    for cname, cfg in cases.items():
        params = rm.init_model(cfg, seed=3)
        sched = rd.make_schedule(8)
        for pname, pol in policies.items():
            for guidance in (False, True):
                table = rp.build_schedule(pol, sched, cfg.layers)
                lat, log = _loop(params, sched, table, seed=7, guidance=guidance, broadcast_object="scores")
                key = f"{cname}|{pname}|{int(guidance)}"
                out[key + "|latents"] = lat.astype(np.float32)
                out[key + "|log"] = log
                out[key + "|table"] = table.source
                meta[key] = {"policy": rp.policy_to_dict(pol)}
        meta[cname] = {"layers": cfg.layers, "hidden": cfg.hidden, "heads": cfg.heads, "frames": cfg.frames,
                       "spatial_tokens": cfg.spatial_tokens, "text_tokens": cfg.text_tokens,
                       "cross_in_temporal": cfg.cross_in_temporal}
    np.savez_compressed(os.path.join(OUT, "scores_runs.npz"), **out)
    with open(os.path.join(OUT, "scores_runs.json"), "w") as fh:
        json.dump(meta, fh, indent=0)


def c1_run():
    cfg = rm.ModelConfig(layers=4, hidden=144, heads=2, frames=8, spatial_tokens=1024, text_tokens=16)
    params = rm.init_model(cfg, seed=11)
    sched = rd.make_schedule(10)
    pol, _ = rp.resolve_preset("latte-pab235", cfg.layers)
    table = rp.build_schedule(pol, sched, cfg.layers)
    lat, log = _loop(params, sched, table, seed=11, guidance=False)
    flat = lat.reshape(lat.shape[0], -1)
    idx = np.arange(0, flat.shape[1], flat.shape[1] // 4096)[:4096]
    np.savez_compressed(os.path.join(OUT, "c1_run.npz"), norms=np.linalg.norm(flat.astype(np.float64), axis=1),
                        maxabs=np.abs(flat).max(axis=1), idx=idx, sub=flat[:, idx], log=log, table=table.source,
                        final_digest=np.array(rm.array_digest(lat[-1][None] if lat[-1].ndim == 3 else lat[-1])))


# name: (layers, steps, preset, cross_in_temporal)
TRACE_CONFIGS = {
    "C2": (28, 50, "latte-pab235", False),
    "C3": (28, 30, "opensora-pab246", True),
    "C4": (28, 150, "opensoraplan-pab246", False),
    "C5": (28, 30, "opensora-pab246", True),
}


def traces():
    out = {}
    for cname, (layers, steps, preset, cross_t) in TRACE_CONFIGS.items():
        cfg = rm.ModelConfig(layers=layers, hidden=8, heads=1, frames=2, spatial_tokens=2, text_tokens=3,
                             cross_in_temporal=cross_t)
        params = rm.init_model(cfg, seed=11)
        sched = rd.make_schedule(steps)
        pol, _ = rp.resolve_preset(preset, layers)
        for name, p in (("pab", pol), ("none", rp.NonePolicy())):
            table = rp.build_schedule(p, sched, layers)
            _, log = _loop(params, sched, table, seed=11, guidance=True)
            out[f"{cname}|{name}|log"] = log
            out[f"{cname}|{name}|table"] = table.source
    np.savez_compressed(os.path.join(OUT, "traces.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["decisions", "prng", "small", "c1", "scores", "traces"]
    if "decisions" in which:
        decisions()
    if "prng" in which:
        prng()
    if "small" in which:
        small_runs()
    if "c1" in which:
        c1_run()
    if "scores" in which:
        scores_runs()
    if "traces" in which:
        traces()
    print("golden fixtures written to", OUT)

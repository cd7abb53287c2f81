"""Pin the CPU oracle (oracle/pab_oracle.py) to the reference before trusting
it: PRNG vectors and per-step latents / decision logs of reference runs
(fixtures made by tests/golden/make_golden.py from /root/reference).  CPU only.
"""

import json
import os

import numpy as np
import pytest

from oracle import pab_oracle as orc
from paper_2408_12588_b200.numerics import RandomStream


@pytest.fixture(scope="module")
def prng(golden_dir):
    return np.load(os.path.join(golden_dir, "prng.npz"))


@pytest.mark.parametrize("seed", [0, 11, 2024, 2**63 + 5])
def test_prng_vectors(prng, seed):
    for stream in (orc.Stream(seed), RandomStream(seed)):
        assert np.array_equal(stream.uniform(257, -0.125, 0.125), prng[f"uniform_{seed}"])
        assert np.array_equal(stream.normal(301), prng[f"normal_{seed}"])
    s = RandomStream(seed)
    s.uniform(257, -0.125, 0.125)
    s.normal(301)
    assert [s.next_u64() for _ in range(5)] == [int(v) for v in prng[f"u64_{seed}"]]


@pytest.fixture(scope="module")
def small(golden_dir):
    return (np.load(os.path.join(golden_dir, "small_runs.npz")),
            json.load(open(os.path.join(golden_dir, "small_runs.json"))))


KIND_NAMES = ("spatial", "temporal", "cross", "mlp")


def _cfg(meta):
    return orc.Cfg(meta["layers"], meta["hidden"], meta["heads"], meta["frames"], meta["spatial_tokens"],
                   meta["text_tokens"], cross_in_temporal=meta["cross_in_temporal"])


@pytest.mark.parametrize("case", ["small", "smallx"])
@pytest.mark.parametrize("policy", ["none", "pab", "tgate", "deltadit"])
@pytest.mark.parametrize("guidance", [0, 1])
def test_oracle_matches_reference_runs(small, case, policy, guidance):
    data, meta = small
    key = f"{case}|{policy}|{guidance}"
    cfg = _cfg(meta[case])
    w = orc.init_weights(cfg, seed=3)
    table = data[key + "|table"]
    steps, log = [], []
    orc.sample(cfg, w, orc.linear_timesteps(8), table, seed=7, guidance=bool(guidance),
               delta_mode=meta[key]["delta"], per_step=steps, log=log)
    ref = data[key + "|latents"]
    for i, (got, want) in enumerate(zip(steps, ref)):
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert rel < 2e-5, (key, i, rel)
    # per-site decision log (reference TraceRecord decision/source_step)
    if not meta[key]["delta"]:
        ref_log = data[key + "|log"]
        got_log = np.array([[s, l, KIND_NAMES.index(k), 0 if b == "s" else 1, 0 if d == "compute" else 1, src]
                            for (s, l, k, b, d, src) in log], dtype=np.int32)
        assert np.array_equal(got_log, ref_log)


def test_oracle_c1_subsample(golden_dir):
    path = os.path.join(golden_dir, "c1_run.npz")
    if not os.path.exists(path):
        pytest.skip("c1 fixture not generated")
    g = np.load(path)
    cfg = orc.Cfg(4, 144, 2, 8, 1024, 16)
    w = orc.init_weights(cfg, seed=11)
    steps = []
    orc.sample(cfg, w, orc.linear_timesteps(10), g["table"], seed=11, per_step=steps)
    for i, x in enumerate(steps):
        flat = x.reshape(-1)
        sub = flat[g["idx"]]
        rel = np.linalg.norm(sub - g["sub"][i]) / np.linalg.norm(g["sub"][i])
        assert rel < 1e-4, (i, rel)
        assert abs(np.linalg.norm(flat.astype(np.float64)) / g["norms"][i] - 1.0) < 1e-5


@pytest.fixture(scope="module")
def scores_runs(golden_dir):
    return (np.load(os.path.join(golden_dir, "scores_runs.npz")),
            json.load(open(os.path.join(golden_dir, "scores_runs.json"))))


@pytest.mark.parametrize("case", ["small", "smallx"])
@pytest.mark.parametrize("policy", ["pab", "tgate"])
@pytest.mark.parametrize("guidance", [0, 1])
def test_oracle_scores_mode_matches_reference_runs(scores_runs, case, policy, guidance):
    """broadcast_object="scores": attention sites cache probabilities and replay
    them against the current values (reference model.py:325-392, 469-499)."""
    data, meta = scores_runs
    key = f"{case}|{policy}|{guidance}"
    m = meta[case]
    cfg = orc.Cfg(m["layers"], m["hidden"], m["heads"], m["frames"], m["spatial_tokens"], m["text_tokens"],
                  cross_in_temporal=m["cross_in_temporal"])
    steps = []
    orc.sample(cfg, orc.init_weights(cfg, seed=3), orc.linear_timesteps(8), data[key + "|table"], seed=7,
               guidance=bool(guidance), per_step=steps, scores=True)
    for i, (got, want) in enumerate(zip(steps, data[key + "|latents"])):
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert rel < 2e-5, (key, i, rel)


# ------------------------------------------------------------ bf16 emulation
def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    a = np.concatenate([rng.standard_normal(10000).astype(np.float32) * 10,
                        np.array([0.0, -0.0, 1.0, 1.00390625, 1.01171875, 3.4e38, 1e-40], np.float32)])
    want = torch.from_numpy(a).to(torch.bfloat16).float().numpy()
    assert np.array_equal(orc.bf16_round(a), want)


def test_emulated_bf16_floor_smoke_config():
    """The guided gate (tests/test_model_gpu.py REL_TOL_CFG) is 1.5x the emulated
    floor measured by scripts/bf16_floor.py; the floor of the
    smoke config must stay where the gate was derived from (1.57e-2 relL2)."""
    cfg = orc.Cfg(2, 144, 2, 8, 256, 20, cross_in_temporal=True)
    w = orc.init_weights(cfg, 11)
    ts = orc.linear_timesteps(5)
    table = orc.table_pab(ts, 2, (2, 3, 4), (990.0, 10.0))
    ref, emu = [], []
    orc.sample(cfg, w, ts, table, seed=11, text_ids=np.arange(20), guidance=True, per_step=ref)
    orc.sample(cfg, w, ts, table, seed=11, text_ids=np.arange(20), guidance=True, per_step=emu, emulate_bf16=True)
    rel = max(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b) for a, b in zip(emu, ref))
    assert 1.0e-2 < rel < 2.0e-2, rel

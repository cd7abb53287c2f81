"""Full-depth decision parity (SURVEY.md 8c hard part 3): the device engine run at
the real C2/C3/C4 shapes and depths (L=28, the configs' step counts, CFG batch 2,
their PAB presets) launches and skips exactly the sites the reference decides.

The reference traces (tests/golden/traces.npz, made by make_golden.py `traces`
with the reference's own forward_step at D=8 -- decisions do not depend on the
hidden size) give every (step, layer, kind, block) decision and source step; the
engine's launch log must equal them row for row, and its kernel counters must
equal the number of computed sites of each kind."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2408_12588_b200.diffusion import Denoiser, initial_latent, make_schedule  # noqa: E402
from paper_2408_12588_b200.model import KINDS, ModelConfig, init_model  # noqa: E402
from paper_2408_12588_b200.policies import DecisionTable, NonePolicy, build_schedule, resolve_preset  # noqa: E402

KIND_NAMES = [k.value for k in KINDS]

# name: (T, S, M, steps, preset, cross_in_temporal)   (SURVEY.md 8 config key)
CONFIGS = {
    "C2": (16, 1024, 120, 50, "latte-pab235", False),
    "C3": (16, 1560, 300, 30, "opensora-pab246", True),
    "C4": (16, 1024, 300, 150, "opensoraplan-pab246", False),
}


@pytest.fixture(scope="module")
def traces(golden_dir):
    return np.load(os.path.join(golden_dir, "traces.npz"))


def _log(den):
    return np.array([[s, l, KIND_NAMES.index(k), 0 if b == "s" else 1, {"compute": 0, "reuse": 1, "delta": 2}[d],
                      src] for (s, l, k, b, d, src) in den.ctx.launches.log], dtype=np.int32)


@pytest.mark.parametrize("name,policy", [("C3", "pab"), ("C3", "none"), ("C2", "pab"), ("C4", "pab")])
def test_full_depth_launch_log_matches_reference(traces, name, policy):
    T, S, M, steps, preset, cross_t = CONFIGS[name]
    cfg = ModelConfig(layers=28, hidden=1152, heads=16, frames=T, spatial_tokens=S, text_tokens=M,
                      cross_in_temporal=cross_t)
    sched = make_schedule(steps)
    pol = resolve_preset(preset, cfg.layers)[0] if policy == "pab" else NonePolicy()
    table = build_schedule(pol, sched, cfg.layers)
    ref_table = traces[f"{name}|{policy}|table"]
    assert np.array_equal(table.source, ref_table)
    params = init_model(cfg, seed=11)
    den = Denoiser(params, sched, DecisionTable(table.source, delta_mode=table.delta_mode),
                   np.arange(M) % 256, guidance=True, guidance_scale=4.0)
    z = torch.from_numpy(initial_latent(params, 11, 2)).cuda()
    den.run(z)
    torch.cuda.synchronize()
    log = _log(den)
    ref = traces[f"{name}|{policy}|log"]
    assert log.shape == ref.shape
    bad = np.flatnonzero((log != ref).any(axis=1))
    assert bad.size == 0, (bad[:5], log[bad[:5]], ref[bad[:5]])
    # kernel counters: one attention launch per computed spatial/temporal/cross site,
    # none for reused sites (reference model.py:484-503)
    computed = ref[:, 4] == 0
    la = den.ctx.launches
    assert la.sites_computed == int(computed.sum())
    assert la.sites_reused == int((ref[:, 4] == 1).sum())
    n_attn = int((computed & (ref[:, 2] != KIND_NAMES.index("mlp"))).sum())
    assert la.attention_calls == n_attn
    zz = z.cpu().numpy()
    assert np.isfinite(zz).all()
    # the two CFG halves receive the same eps_hat, so they stay identical
    assert np.array_equal(zz[0], zz[1])

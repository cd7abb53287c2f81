"""Full-size parity slices: one layer of the C2/C3/C4 blocks at
their real shapes (D1152, H16, T16, S1024/1560, M120/300, CFG batch 2) for a few
denoising steps whose tables broadcast sites, against the CPU oracle; a 4-layer
x 30-step C3 run and a 4-layer x 50-step C2 run against oracle fixtures
(tests/golden/c3_deep.npz, c2_deep.npz); a C5 layer
(T32, S3600) for two steps; and C5's 3600-token spatial attention at op level against
a torch fp32 reference."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pab_oracle as orc  # noqa: E402
from paper_2408_12588_b200 import kernels  # noqa: E402
from paper_2408_12588_b200.diffusion import Denoiser, initial_latent, make_schedule  # noqa: E402
from paper_2408_12588_b200.model import ModelConfig, init_model  # noqa: E402
from paper_2408_12588_b200.policies import DecisionTable  # noqa: E402
from gates import MAX_TOL_CFG, REL_TOL_CFG  # noqa: E402


def test_c3_layer_three_steps_with_broadcast_vs_oracle():
    cfg = ModelConfig(layers=1, hidden=1152, heads=16, frames=16, spatial_tokens=1560, text_tokens=300,
                      cross_in_temporal=True)
    params = init_model(cfg, seed=11)
    src = np.zeros((3, 1, 4), dtype=np.int32)
    src[1] = 1
    src[2] = 1  # step 2 broadcasts every site computed at step 1
    table = DecisionTable(src)
    sched = make_schedule(3)
    ids = np.arange(300) % 256
    den = Denoiser(params, sched, table, ids, guidance=True, guidance_scale=4.0)
    z = torch.from_numpy(initial_latent(params, 11, 2)).cuda()
    got = []
    den.run(z, on_step=lambda i, zz: got.append(zz.cpu().numpy().copy()))
    assert den.ctx.launches.sites_reused == 6  # all six sites of the layer at step 2
    ocfg = orc.Cfg(1, 1152, 16, 16, 1560, 300, cross_in_temporal=True)
    want = []
    orc.sample(ocfg, orc.init_weights(ocfg, 11), orc.linear_timesteps(3), src, seed=11, text_ids=ids,
               guidance=True, per_step=want)
    for i, (g, w) in enumerate(zip(got, want)):
        rel = np.linalg.norm(g.astype(np.float64) - w) / np.linalg.norm(w)
        mx = np.abs(g - w).max() / np.abs(w).max()
        assert rel < REL_TOL_CFG and mx < MAX_TOL_CFG, (i, rel, mx)  # CFG (g=4) gate, tests/gates.py
    # broadcast step is exact replay: step 2's update used the cached outputs of step 1
    assert np.isfinite(got[-1]).all()


def test_c2_latte_layer_pab_steps_vs_oracle():
    """C2 (Latte 16f 512^2) at full shape for one layer: D1152, H16, T16, S1024, M120,
    no cross attention in the temporal block, CFG batch 2; 4 steps of a table that
    broadcasts spatial/temporal/cross with different source steps (output broadcast)."""
    cfg = ModelConfig(layers=1, hidden=1152, heads=16, frames=16, spatial_tokens=1024, text_tokens=120,
                      cross_in_temporal=False)
    params = init_model(cfg, seed=11)
    src = np.zeros((4, 1, 4), dtype=np.int32)
    for i in range(4):
        src[i, 0] = i
    src[2, 0, 0] = 1  # spatial reuses step 1
    src[3, 0, 1] = 1  # temporal reuses step 1 at step 3
    src[3, 0, 2] = 2  # cross reuses step 2
    table = DecisionTable(src)
    ids = np.arange(120) % 256
    den = Denoiser(params, make_schedule(4), table, ids, guidance=True, guidance_scale=4.0)
    z = torch.from_numpy(initial_latent(params, 11, 2)).cuda()
    got = []
    den.run(z, on_step=lambda i, zz: got.append(zz.cpu().numpy().copy()))
    assert den.ctx.launches.sites_reused == 3
    ocfg = orc.Cfg(1, 1152, 16, 16, 1024, 120, cross_in_temporal=False)
    want = []
    orc.sample(ocfg, orc.init_weights(ocfg, 11), orc.linear_timesteps(4), src, seed=11, text_ids=ids,
               guidance=True, per_step=want)
    for i, (g, w) in enumerate(zip(got, want)):
        rel = np.linalg.norm(g.astype(np.float64) - w) / np.linalg.norm(w)
        mx = np.abs(g - w).max() / np.abs(w).max()
        assert rel < REL_TOL_CFG and mx < MAX_TOL_CFG, (i, rel, mx)  # CFG (g=4) gate, tests/gates.py


def test_c4_layer_three_steps_with_broadcast_vs_oracle():
    """C4 (Open-Sora-Plan 65f 512^2) at full shape for one layer: D1152, H16, T16,
    S1024, M300 (T5 text), NO cross attention in the temporal block, CFG batch 2;
    3 steps, step 2 broadcasts every site computed at step 1."""
    cfg = ModelConfig(layers=1, hidden=1152, heads=16, frames=16, spatial_tokens=1024, text_tokens=300,
                      cross_in_temporal=False)
    params = init_model(cfg, seed=11)
    src = np.zeros((3, 1, 4), dtype=np.int32)
    src[1] = 1
    src[2] = 1
    table = DecisionTable(src)
    ids = np.arange(300) % 256
    den = Denoiser(params, make_schedule(3), table, ids, guidance=True, guidance_scale=4.0)
    z = torch.from_numpy(initial_latent(params, 11, 2)).cuda()
    got = []
    den.run(z, on_step=lambda i, zz: got.append(zz.cpu().numpy().copy()))
    assert den.ctx.launches.sites_reused == 5  # S, C, M | T, M at step 2
    ocfg = orc.Cfg(1, 1152, 16, 16, 1024, 300, cross_in_temporal=False)
    want = []
    orc.sample(ocfg, orc.init_weights(ocfg, 11), orc.linear_timesteps(3), src, seed=11, text_ids=ids,
               guidance=True, per_step=want)
    for i, (g, w) in enumerate(zip(got, want)):
        rel = np.linalg.norm(g.astype(np.float64) - w) / np.linalg.norm(w)
        mx = np.abs(g - w).max() / np.abs(w).max()
        assert rel < REL_TOL_CFG and mx < MAX_TOL_CFG, (i, rel, mx)


def test_c5_layer_two_steps_with_broadcast_vs_oracle():
    """C5 (Open-Sora 720p 4s) at full shape for one layer: D1152, H16, T32 (the attn_tm
    T = 32 path), S3600 (45 x 80), M300, cross in the temporal block, CFG batch 2; step 1
    broadcasts every site computed at step 0.  The oracle evaluates the 3600-token
    spatial attention in chunks (53 GB of logits unchunked)."""
    cfg = ModelConfig(layers=1, hidden=1152, heads=16, frames=32, spatial_tokens=3600, text_tokens=300,
                      cross_in_temporal=True)
    params = init_model(cfg, seed=11)
    src = np.zeros((2, 1, 4), dtype=np.int32)  # step 1 reuses step 0 everywhere
    table = DecisionTable(src)
    ids = np.arange(300) % 256
    den = Denoiser(params, make_schedule(2), table, ids, guidance=True, guidance_scale=4.0)
    z = torch.from_numpy(initial_latent(params, 11, 2)).cuda()
    got = []
    den.run(z, on_step=lambda i, zz: got.append(zz.cpu().numpy().copy()))
    assert den.ctx.launches.sites_reused == 6
    ocfg = orc.Cfg(1, 1152, 16, 32, 3600, 300, cross_in_temporal=True)
    want = []
    orc.sample(ocfg, orc.init_weights(ocfg, 11), orc.linear_timesteps(2), src, seed=11, text_ids=ids,
               guidance=True, per_step=want)
    for i, (g, w) in enumerate(zip(got, want)):
        rel = np.linalg.norm(g.astype(np.float64) - w) / np.linalg.norm(w)
        mx = np.abs(g - w).max() / np.abs(w).max()
        print(f"C5 slice step {i}: relL2 {rel:.2e}, max {mx:.2e}")
        assert rel < REL_TOL_CFG and mx < MAX_TOL_CFG, (i, rel, mx)


def test_c5_spatial_attention_3600_tokens():
    B, S, H, dh = 2, 3600, 16, 72
    D = H * dh
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = torch.randn(B * S, 3 * D, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty(B * S, D, device="cuda", dtype=torch.bfloat16)
    ld = 3 * D
    a = kernels.attn_args(qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:], out, (S * ld, 0, ld), (S * ld, 0, ld),
                          (S * ld, 0, ld), (S * D, 0, D), B, 1, S, S, H, dh)
    assert kernels.attention_select(a) == kernels.IMPL_TCGEN05
    kernels.attention(a)
    x = qkv.float().view(B, S, 3, H, dh).permute(2, 0, 3, 1, 4)
    ref = torch.softmax(x[0] @ x[1].transpose(-1, -2) / dh**0.5, -1) @ x[2]
    ref = ref.permute(0, 2, 1, 3).reshape(B * S, D)
    rel = float((out.float() - ref).norm() / ref.norm())
    assert rel < 1.2e-2, rel


# fixtures of tests/golden/make_deep.py (make_c3_deep.py wrote c3 before the config field existed)
_DEEP_DEFAULT = {"c3": (4, 1152, 16, 16, 1560, 300, 1, 30)}


@pytest.mark.parametrize("name", ["c3", "c2", "c4"])
def test_deep_multilayer_full_schedule_vs_oracle_fixture(name):
    """A config at full width with 4 of its 28 layers over its whole PAB schedule (CFG g=4)
    against the CPU oracle's run stored in tests/golden/<name>_deep.npz
    (tests/golden/make_deep.py): per-step latent norm, max|x| and a strided 8192-element
    subsample.  C3: opensora-pab246, 30 steps, cross attention in the temporal block;
    C2: latte-pab235, 50 steps, M = 120; C4: opensoraplan-pab246, 150 steps (2 layers).
    Broadcast reuse compounds over the schedule here, which the one-layer slices cannot
    show."""
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", f"{name}_deep.npz")
    if not os.path.exists(path):
        pytest.skip(f"tests/golden/{name}_deep.npz not generated (tests/golden/make_deep.py {name})")
    fx = np.load(path)
    L, D, H, T, S, M, cit, N = (int(v) for v in (fx["config"] if "config" in fx else _DEEP_DEFAULT[name]))
    cfg = ModelConfig(layers=L, hidden=D, heads=H, frames=T, spatial_tokens=S, text_tokens=M,
                      cross_in_temporal=bool(cit))
    params = init_model(cfg, seed=11)
    table = DecisionTable(fx["table"])
    den = Denoiser(params, make_schedule(N), table, np.arange(M) % 256, guidance=True, guidance_scale=4.0)
    z = torch.from_numpy(initial_latent(params, 11, 2)).cuda()
    idx = torch.from_numpy(fx["idx"]).cuda()
    got_sub, got_norm, got_max = [], [], []

    def on_step(i, zz):
        flat = zz.reshape(-1)
        got_sub.append(flat[idx].cpu().numpy().astype(np.float64))
        got_norm.append(float(flat.double().norm()))
        got_max.append(float(flat.abs().max()))

    den.run(z, on_step=on_step)
    assert den.ctx.launches.sites_reused > 0
    worst = (0.0, 0.0, 0.0)
    for i in range(N):
        w = fx["sub"][i].astype(np.float64)
        rel = np.linalg.norm(got_sub[i] - w) / np.linalg.norm(w)
        mx = np.abs(got_sub[i] - w).max() / float(fx["maxabs"][i])
        rn = abs(got_norm[i] - float(fx["norms"][i])) / float(fx["norms"][i])
        worst = tuple(max(a, b) for a, b in zip(worst, (rel, mx, rn)))
        assert rel < REL_TOL_CFG and mx < MAX_TOL_CFG and rn < REL_TOL_CFG, (i, rel, mx, rn)
    print(f"{name} L{L} x {N} steps vs oracle: worst relL2 {worst[0]:.2e}, max {worst[1]:.2e}, norm {worst[2]:.2e}")


def test_c5_layer_two_steps_with_broadcast_vs_oracle():
    """C5 (Open-Sora 720p 4s) at full shape for one layer: D1152, H16, T32 (the attn_tm
    T = 32 path), S3600 (45 x 80), M300, cross in the temporal block, CFG batch 2; step 1
    broadcasts every site computed at step 0.  The oracle evaluates the 3600-token
    spatial attention in chunks (53 GB of logits unchunked)."""
    cfg = ModelConfig(layers=1, hidden=1152, heads=16, frames=32, spatial_tokens=3600, text_tokens=300,
                      cross_in_temporal=True)
    params = init_model(cfg, seed=11)
    src = np.zeros((2, 1, 4), dtype=np.int32)  # step 1 reuses step 0 everywhere
    table = DecisionTable(src)
    ids = np.arange(300) % 256
    den = Denoiser(params, make_schedule(2), table, ids, guidance=True, guidance_scale=4.0)
    z = torch.from_numpy(initial_latent(params, 11, 2)).cuda()
    got = []
    den.run(z, on_step=lambda i, zz: got.append(zz.cpu().numpy().copy()))
    assert den.ctx.launches.sites_reused == 6
    ocfg = orc.Cfg(1, 1152, 16, 32, 3600, 300, cross_in_temporal=True)
    want = []
    orc.sample(ocfg, orc.init_weights(ocfg, 11), orc.linear_timesteps(2), src, seed=11, text_ids=ids,
               guidance=True, per_step=want)
    for i, (g, w) in enumerate(zip(got, want)):
        rel = np.linalg.norm(g.astype(np.float64) - w) / np.linalg.norm(w)
        mx = np.abs(g - w).max() / np.abs(w).max()
        print(f"C5 slice step {i}: relL2 {rel:.2e}, max {mx:.2e}")
        assert rel < REL_TOL_CFG and mx < MAX_TOL_CFG, (i, rel, mx)


def test_c5_spatial_attention_3600_tokens():
    B, S, H, dh = 2, 3600, 16, 72
    D = H * dh
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = torch.randn(B * S, 3 * D, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty(B * S, D, device="cuda", dtype=torch.bfloat16)
    ld = 3 * D
    a = kernels.attn_args(qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:], out, (S * ld, 0, ld), (S * ld, 0, ld),
                          (S * ld, 0, ld), (S * D, 0, D), B, 1, S, S, H, dh)
    assert kernels.attention_select(a) == kernels.IMPL_TCGEN05
    kernels.attention(a)
    x = qkv.float().view(B, S, 3, H, dh).permute(2, 0, 3, 1, 4)
    ref = torch.softmax(x[0] @ x[1].transpose(-1, -2) / dh**0.5, -1) @ x[2]
    ref = ref.permute(0, 2, 1, 3).reshape(B * S, D)
    rel = float((out.float() - ref).norm() / ref.norm())
    assert rel < 1.2e-2, rel


def test_c3_four_layers_thirty_steps_vs_oracle_fixture():
    """C3 at full width and 4 of its 28 layers over the whole 30-step opensora-pab246
    schedule (CFG g=4) against the CPU oracle's run stored in tests/golden/c3_deep.npz
    (tests/golden/make_c3_deep.py): per-step latent norm, max|x| and a strided
    8192-element subsample.  Broadcast reuse compounds over the 30 steps here, which
    the one-layer slices above cannot show."""
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", "c3_deep.npz")
    if not os.path.exists(path):
        pytest.skip("tests/golden/c3_deep.npz not generated (tests/golden/make_c3_deep.py)")
    fx = np.load(path)
    L, N = int(fx["layers"]), int(fx["steps"])
    cfg = ModelConfig(layers=L, hidden=1152, heads=16, frames=16, spatial_tokens=1560, text_tokens=300,
                      cross_in_temporal=True)
    params = init_model(cfg, seed=11)
    table = DecisionTable(fx["table"])
    den = Denoiser(params, make_schedule(N), table, np.arange(300) % 256, guidance=True, guidance_scale=4.0)
    z = torch.from_numpy(initial_latent(params, 11, 2)).cuda()
    idx = torch.from_numpy(fx["idx"]).cuda()
    got_sub, got_norm, got_max = [], [], []

    def on_step(i, zz):
        flat = zz.reshape(-1)
        got_sub.append(flat[idx].cpu().numpy().astype(np.float64))
        got_norm.append(float(flat.double().norm()))
        got_max.append(float(flat.abs().max()))

    den.run(z, on_step=on_step)
    assert den.ctx.launches.sites_reused > 0
    worst = (0.0, 0.0, 0.0)
    for i in range(N):
        w = fx["sub"][i].astype(np.float64)
        rel = np.linalg.norm(got_sub[i] - w) / np.linalg.norm(w)
        mx = np.abs(got_sub[i] - w).max() / float(fx["maxabs"][i])
        rn = abs(got_norm[i] - float(fx["norms"][i])) / float(fx["norms"][i])
        worst = tuple(max(a, b) for a, b in zip(worst, (rel, mx, rn)))
        assert rel < REL_TOL_CFG and mx < MAX_TOL_CFG and rn < REL_TOL_CFG, (i, rel, mx, rn)
    print(f"C3 L{L} x {N} steps vs oracle: worst relL2 {worst[0]:.2e}, max {worst[1]:.2e}, norm {worst[2]:.2e}")

"""Sequence-parallel host logic on CPU: shard plans, the in-process reshard
API, the closed-form communication model (reference pkg/tests/test_parallel.py),
and the real frames<->tokens all-to-all exchange of the distributed engine run
over a world_size-2 (and 4) gloo group."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_12588_b200.diffusion import make_schedule
from paper_2408_12588_b200.errors import ShapeError, ValidationError
from paper_2408_12588_b200.model import ComponentKind, ModelConfig
from paper_2408_12588_b200.parallel import (
    CommReport,
    comm_volume_model,
    exchange_frames_to_tokens,
    exchange_tokens_to_frames,
    plan_shards,
    reshard,
    send_order,
    split_shards,
    unpack_frames,
)
from paper_2408_12588_b200.policies import NonePolicy, PabPolicy, build_schedule

SMALL = ModelConfig(layers=2, hidden=32, heads=4, frames=4, spatial_tokens=16, text_tokens=8)


class TestPlans:
    def test_plans(self):
        assert plan_shards(1, SMALL).frames_per_worker == 4
        p = plan_shards(2, ModelConfig(frames=8, spatial_tokens=64))
        assert (p.frames_per_worker, p.tokens_per_worker) == (4, 32)
        with pytest.raises(ValidationError):
            plan_shards(3, ModelConfig(frames=8, spatial_tokens=64))

    def test_c3_and_c5_plans(self):
        for w in (1, 2, 4, 8):
            plan_shards(w, ModelConfig(layers=28, hidden=1152, heads=16, frames=16, spatial_tokens=1560,
                                       text_tokens=300))
            plan_shards(w, ModelConfig(layers=28, hidden=1152, heads=16, frames=32, spatial_tokens=3600,
                                       text_tokens=300))


class TestInProcessReshard:
    def test_there_and_back(self):
        cfg = ModelConfig(layers=1, hidden=8, heads=2, frames=4, spatial_tokens=8, text_tokens=2)
        plan = plan_shards(2, cfg)
        full = np.random.default_rng(0).standard_normal((1, 4, 8, 8)).astype(np.float32)
        shards = split_shards(full, "frames", 2)
        led = CommReport("dsp", 2, 4)
        back = reshard(reshard(shards, "frames", "tokens", plan, cfg, led), "tokens", "frames", plan, cfg, led)
        for a, b in zip(back, shards):
            assert np.array_equal(a, b)
        assert led.total_elements() == 2 * (4 * 8 * 8 // 2)

    def test_layout_mismatch(self):
        cfg = ModelConfig(layers=1, hidden=8, heads=2, frames=4, spatial_tokens=8, text_tokens=2)
        plan = plan_shards(2, cfg)
        with pytest.raises(ShapeError):
            reshard(split_shards(np.zeros((1, 4, 8, 8)), "tokens", 2), "frames", "tokens", plan, cfg)


class TestVolumeModel:
    def test_method_ratios(self):
        sched = make_schedule(30)
        t = build_schedule(NonePolicy(), sched, 4)
        tot = {m: comm_volume_model(m, SMALL, sched, t, 8).total_elements() for m in ("megatron_sp", "ds_ulysses", "dsp")}
        assert tot["megatron_sp"] / tot["dsp"] == 8.0 and tot["ds_ulysses"] / tot["dsp"] == 2.0

    def test_pab_scales_by_temporal_fraction(self):
        sched = make_schedule(30)
        none = build_schedule(NonePolicy(), sched, 4)
        pab = build_schedule(PabPolicy(2, 4, 6, window=(930.0, 450.0)), sched, 4)
        frac = len(pab.compute_steps(ComponentKind.TEMPORAL)) / 30
        for m in ("megatron_sp", "ds_ulysses", "dsp", "broadcast_sp"):
            a = comm_volume_model(m, SMALL, sched, none, 8).total_elements()
            b = comm_volume_model(m, SMALL, sched, pab, 8).total_elements()
            assert b / a == pytest.approx(frac, rel=1e-12)

    def test_event_count_is_two_per_temporal_compute(self):
        sched = make_schedule(30)
        pab = build_schedule(PabPolicy(2, 4, 6, window=(930.0, 450.0)), sched, 28)
        rep = comm_volume_model("broadcast_sp", SMALL, sched, pab, 8)
        assert rep.event_count() == 28 * 20  # one (step, layer) entry per temporal compute
        assert comm_volume_model("dsp", SMALL, sched, pab, 1).total_elements() == 0
        with pytest.raises(ValidationError):
            comm_volume_model("ring", SMALL, sched, pab, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, B, T, S, D, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        full = torch.randn(B, T, S, D, generator=g)          # identical on every rank
        Tl, Sw = T // world, S // world
        shard = full[:, rank * Tl:(rank + 1) * Tl].contiguous()
        send = send_order(shard, world)
        tok = torch.empty(T, B, Sw, D)
        exchange_frames_to_tokens(send, tok)
        # token layout (t, b, s_local) of this rank's tokens over ALL frames
        want_tok = full[:, :, rank * Sw:(rank + 1) * Sw].permute(1, 0, 2, 3)
        ok1 = torch.equal(tok, want_tok)
        # reverse exchange of a per-token result returns this rank's frame shard
        recv = torch.empty(world, Tl, B, Sw, D)
        exchange_tokens_to_frames(tok * 2.0, recv)
        out = torch.empty(B, Tl, S, D)
        unpack_frames(recv, out)
        ok2 = torch.equal(out, shard * 2.0)
        q.put((rank, ok1, ok2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_frames_tokens_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, 2, 8, 12, 6, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _, _ in res) == list(range(world))
    assert all(a and b for _, a, b in res), res


def _pair_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2408_12588_b200.parallel import _all_gather_into

        gw = world // 2
        # the split_batch groups, created collectively in the same order on every rank
        sp = [dist.new_group(list(range(g * gw, (g + 1) * gw))) for g in range(2)]
        pairs = [dist.new_group([w, gw + w]) for w in range(gw)]
        half, w = divmod(rank, gw)
        mine = torch.full((3, 5), float(rank))
        out = torch.empty(2, 3, 5)
        _all_gather_into(out, mine, pairs[w])
        # slot 0 = conditional half (group 0), slot 1 = unconditional half of the same frames
        ok = torch.equal(out[0], torch.full((3, 5), float(w))) and torch.equal(out[1], torch.full((3, 5), float(gw + w)))
        ok = ok and dist.get_world_size(sp[half]) == gw
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_split_batch_pair_exchange():
    """split_batch: rank w (conditional half) and W/2 + w (unconditional half) hold the
    same frames and exchange eps over their 2-rank group before the CFG combine."""
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pair_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _ in res) == list(range(world)) and all(ok for _, ok in res), res


def test_split_batch_volume_model():
    """Closed form with split_batch: two groups of W/2, each moving its B=1 half
    (reference pkg/tests/test_parallel.py:193-204)."""
    sched = make_schedule(6)
    t = build_schedule(NonePolicy(), sched, 2)
    cfg = ModelConfig(layers=2, hidden=32, heads=4, frames=4, spatial_tokens=16, text_tokens=8)
    split = comm_volume_model("dsp", cfg, sched, t, 4, batch=2, split_batch=True)
    whole = comm_volume_model("dsp", cfg, sched, t, 4, batch=2)
    el = lambda b, w: b * 4 * 16 * 32 // w * (w - 1)  # noqa: E731
    assert all(v == 2 * 2 * el(1, 2) for v in split.grouped_elements().values())
    assert all(v == 2 * el(2, 4) for v in whole.grouped_elements().values())
    assert comm_volume_model("dsp", cfg, sched, t, 2, batch=2, split_batch=True).total_elements() == 0


def test_send_order_matches_kernel_permutation_formula():
    """The CUDA prologue writes h row (b, t, s) at ((dst*Tl + t)*B + b)*Sw + s%Sw
    (include/pab_b200.h, pab_residual_modnorm_sp); check the torch layout used by
    the exchange tests is that permutation."""
    B, Tl, S, D, W = 2, 3, 8, 1, 4
    Sw = S // W
    x = torch.arange(B * Tl * S, dtype=torch.float32).reshape(B, Tl, S, D)
    send = send_order(x, W).reshape(-1)
    for b in range(B):
        for t in range(Tl):
            for s in range(S):
                row = (b * Tl + t) * S + s
                pos = (((s // Sw) * Tl + t) * B + b) * Sw + s % Sw
                assert send[pos] == row

"""Broadcast sequence parallelism over real GPUs (one process per GPU).

Drop-in for pkg/src/pab_engine/parallel.py.  The reference runs W *logical*
workers sequentially in one process (parallel.py:1-15); here each worker is
a rank of a torch.distributed NCCL group on its own B200:

* the residual stream is frame-sharded: rank w owns frames
  [w T/W, (w+1) T/W) of every batch entry, (B, T/W, S, D) fp32;
* spatial, cross and MLP sites are frame/token local and run unchanged on
  the shard (same kernels as the serial path);
* a temporal site that COMPUTES runs the dimension switch of reference
  `_parallel_forward_step` (parallel.py:322-340): the modulated-norm
  prologue writes bf16 h straight into all-to-all send order (dest rank, t,
  b, s) -> NCCL all-to-all frames->tokens -> QKV GEMM, temporal attention
  over all T frames for S/W tokens, output GEMM -> all-to-all tokens->frames
  -> unpack to the frame shard.  LN is row-wise, so normalising before the
  exchange equals the reference's reshard-then-normalise;
* a temporal site that is BROADCAST appends this rank's cached frame-layout
  output and launches no collective at all (parallel.py:341-348).

The communication ledger records one entry per reshard with the reference's
element count B*T*S*D*(W-1)/W (parallel.py:130-133, 167-179), so the
executed event count equals 2 * L * |temporal compute steps|.

``split_batch`` (reference parallel.py:410-464): with guidance on an even
number of ranks, ranks [0, W/2) run the conditional half and [W/2, W) the
unconditional half, each half frame-sharded over its own W/2-rank group.
After every step the two ranks holding the same frames exchange their eps
(one all-gather over a 2-rank group) and both apply the same fused
CFG + DDIM update, so the halves stay in lock step exactly as the
reference's shared eps_hat.
"""

from __future__ import annotations

import csv
from collections import defaultdict
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .diffusion import DEFAULT_NOISE, GraphReplay, NoiseParams, default_text_ids, initial_latent
from .errors import PolicyError, ShapeError, ValidationError
from .model import ComponentKind, ModelParams
from .policies import CacheStore, DecisionTable, PabPolicy, PolicyConfig, build_schedule

METHOD_COSTS = {"megatron_sp": 16, "ds_ulysses": 4, "dsp": 2, "broadcast_sp": 2}
EXECUTABLE_METHODS = ("dsp", "broadcast_sp")
# how the temporal site's two reshards move data: NCCL all-to-alls, or stores/loads over
# NVLink peer memory fused into the prologues (peer.py)
TRANSPORTS = ("nccl", "peer")
TM = ComponentKind.TEMPORAL


@dataclass(frozen=True)
class ShardPlan:
    workers: int
    frames: int
    spatial_tokens: int

    @property
    def frames_per_worker(self) -> int:
        return self.frames // self.workers

    @property
    def tokens_per_worker(self) -> int:
        return self.spatial_tokens // self.workers


def plan_shards(workers: int, cfg) -> ShardPlan:
    """W must divide both T and S; no padding (reference parallel.py:72-80)."""
    if workers < 1:
        raise ValidationError(f"worker count must be >= 1, got {workers}")
    if cfg.frames % workers or cfg.spatial_tokens % workers:
        raise ValidationError(
            f"{workers} workers must divide frames ({cfg.frames}) and spatial tokens ({cfg.spatial_tokens});"
            " padding is unsupported"
        )
    return ShardPlan(workers=workers, frames=cfg.frames, spatial_tokens=cfg.spatial_tokens)


@dataclass
class CommEntry:
    step: int
    layer: int
    method: str
    elements: int
    bytes: int
    communicating: bool
    wire_bytes: int = 0  # bytes this rank actually sent over NVLink (bf16 payload)


@dataclass
class CommReport:
    method: str
    workers: int
    bytes_per_element: int
    cost_constant: int = 0
    entries: list = field(default_factory=list)

    def total_elements(self) -> int:
        return sum(e.elements for e in self.entries)

    def total_bytes(self) -> int:
        return sum(e.bytes for e in self.entries)

    def grouped_elements(self) -> dict:
        out: dict = defaultdict(int)
        for e in self.entries:
            if e.elements:
                out[(e.step, e.layer)] += e.elements
        return dict(out)

    def event_count(self) -> int:
        return sum(1 for e in self.entries if e.communicating)

    def write_csv(self, path):
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["step", "layer", "method", "elements", "bytes", "communicating"])
            for e in self.entries:
                w.writerow([e.step, e.layer, e.method, e.elements, e.bytes, int(e.communicating)])


def _alltoall_elements(batch: int, cfg, workers: int) -> int:
    total = batch * cfg.frames * cfg.spatial_tokens * cfg.hidden
    return total // workers * (workers - 1)


_AXIS = {"frames": 1, "tokens": 2}


def split_shards(full, axis: str, workers: int) -> list:
    """Split a (B, T, S, D) array/tensor along frames or tokens (contiguous shards)."""
    ax = _AXIS[axis]
    n = full.shape[ax] // workers
    parts = [full[(slice(None),) * ax + (slice(i * n, (i + 1) * n),)] for i in range(workers)]
    if isinstance(full, np.ndarray):
        return [np.ascontiguousarray(p) for p in parts]
    return [p.contiguous() for p in parts]


def reshard(shards: Sequence, from_axis: str, to_axis: str, plan: ShardPlan, cfg, ledger: Optional[CommReport] = None,
            step: int = -1, layer: int = -1) -> list:
    """Value-preserving repartition of in-process shards (reference API,
    parallel.py:140-180).  The distributed engine uses `exchange_*` below."""
    if from_axis not in _AXIS or to_axis not in _AXIS:
        raise ValidationError(f"unknown layout axes {from_axis!r} -> {to_axis!r}")
    if from_axis == to_axis:
        raise ShapeError("reshard endpoints must differ")
    if len(shards) != plan.workers:
        raise ShapeError(f"expected {plan.workers} shards, got {len(shards)}")
    want = plan.frames_per_worker if from_axis == "frames" else plan.tokens_per_worker
    for s in shards:
        if s.shape[_AXIS[from_axis]] != want:
            raise ShapeError(f"shard shape {tuple(s.shape)} does not match the {from_axis} layout")
    if isinstance(shards[0], np.ndarray):
        full = np.concatenate(shards, axis=_AXIS[from_axis])
    else:
        import torch

        full = torch.cat(list(shards), dim=_AXIS[from_axis])
    if ledger is not None:
        el = _alltoall_elements(shards[0].shape[0], cfg, plan.workers)
        ledger.entries.append(CommEntry(step, layer, ledger.method, el, el * ledger.bytes_per_element, el > 0))
    return split_shards(full, to_axis, plan.workers)


def comm_volume_model(method: str, cfg, schedule, table: DecisionTable, workers: int, bytes_per_element: int = 4,
                      batch: int = 1, split_batch: bool = False) -> CommReport:
    """Closed-form volume: c(method) * B*T*S*D*(W-1)/W per (step, layer) whose
    temporal attention computes (reference parallel.py:183-233)."""
    if method not in METHOD_COSTS:
        raise ValidationError(f"unknown parallel method {method!r}")
    ts = getattr(schedule, "timesteps", schedule)
    if table.num_steps != len(ts):
        raise ValidationError("table does not match the schedule")
    rep = CommReport(method, workers, bytes_per_element, METHOD_COSTS[method])
    groups = 2 if (split_batch and batch == 2 and workers >= 2 and workers % 2 == 0) else 1
    gw = workers // groups
    unit = groups * _alltoall_elements(batch // groups, cfg, gw) if gw > 1 else 0
    comp = table.compute_mask()[:, :, 1]
    for step in range(table.num_steps):
        for layer in range(table.layers):
            on = bool(comp[step, layer])
            el = METHOD_COSTS[method] * unit if on else 0
            rep.entries.append(CommEntry(step, layer, method, el, el * bytes_per_element, on and el > 0))
    return rep


# ---------------------------------------------------------------- logical workers
class _LocalGroupState:
    """Shared state of one in-process group of logical workers (threads)."""

    def __init__(self, size: int):
        import threading

        self.size = size
        self.barrier = threading.Barrier(size, timeout=600)
        self.slots = [None] * size
        self.events = [None] * size  # CUDA event per member: its posted data / its reads are done


class LocalGroup:
    """One logical worker's view of an in-process group.

    The reference runs its W workers sequentially in one process
    (parallel.py:1-15, 372-464); without a torch.distributed group,
    ``run_parallel`` runs them as W threads on one GPU and exchanges shards
    through this group: every member posts its send buffer, waits at a barrier,
    copies its chunks from the peers' buffers and waits again before any buffer
    can be rewritten.  Device ordering follows the host barriers through CUDA
    events: a reader's stream waits for the poster's event before copying, and a
    poster's stream waits for every reader's event before it may rewrite (so the
    members may issue on different streams, as the peer transport does)."""

    def __init__(self, state: _LocalGroupState, rank: int):
        self.state, self.rank = state, rank

    def size(self) -> int:
        return self.state.size

    def _record(self):
        import torch

        if not torch.cuda.is_available() or not torch.cuda.is_initialized():
            return
        ev = torch.cuda.Event()
        ev.record()
        self.state.events[self.rank] = ev

    def _wait_all(self):
        import torch

        if not torch.cuda.is_available() or not torch.cuda.is_initialized():
            return
        cur = torch.cuda.current_stream()
        for w, ev in enumerate(self.state.events):
            if w != self.rank and ev is not None:
                cur.wait_event(ev)

    def _sync(self):
        st = self.state
        try:
            st.barrier.wait()
        except Exception:
            st.barrier.abort()
            raise

    def _post(self, t):
        self.state.slots[self.rank] = t
        self._record()
        self._sync()
        self._wait_all()  # the posted tensors are complete on the device
        self._sync()      # nobody re-records its event before everyone has waited on it

    def _done(self):
        self._record()
        self._sync()
        self._wait_all()  # every member's reads of my posted tensor are done
        self._sync()

    def all_to_all_single(self, recv, send):
        """send (W, ...) by destination -> recv (W, ...) by source."""
        self._post(send)
        W = self.state.size
        rv, me = recv.view(W, -1), self.rank
        for src in range(W):
            rv[src].copy_(self.state.slots[src].reshape(W, -1)[me])
        self._done()

    def exchange_objects(self, obj):
        """Every member's ``obj`` in rank order (the peer transport's pointer exchange)."""
        self._post(obj)
        out = list(self.state.slots)
        self._done()
        return out

    def all_gather(self, t):
        self._post(t)
        parts = [p.clone() for p in self.state.slots]
        self._done()
        return parts

    def all_gather_into(self, out, t):
        self._post(t)
        for dst, part in zip(out, self.state.slots):
            dst.copy_(part.view_as(dst))
        self._done()

    def abort(self):
        self.state.barrier.abort()


# ---------------------------------------------------------------- exchange
def send_order(h_shard, n_w: int):
    """Reference layout transform the CUDA prologue fuses: (B, T/W, S, D) ->
    (W, T/W, B, S/W, D) grouped by destination rank (used by tests)."""
    B, Tl, S, D = h_shard.shape
    return h_shard.reshape(B, Tl, n_w, S // n_w, D).permute(2, 1, 0, 3, 4).contiguous()


def _all_to_all(recv, send, group):
    """NCCL all-to-all on device buffers.  A gloo group (CPU tests, or several
    ranks sharing one GPU in the single-GPU test harness) has no device
    all-to-all, so device tensors are staged through host memory there."""
    import torch.distributed as dist

    if isinstance(group, LocalGroup):
        group.all_to_all_single(recv, send)
        return
    if send.is_cuda and dist.get_backend(group) == "gloo":
        host = recv.cpu()
        dist.all_to_all_single(host, send.cpu(), group=group)
        recv.copy_(host)
        return
    dist.all_to_all_single(recv, send, group=group)


def _all_gather(t, group=None):
    import torch
    import torch.distributed as dist

    if isinstance(group, LocalGroup):
        return group.all_gather(t)
    world = dist.get_world_size(group)
    if t.is_cuda and dist.get_backend(group) == "gloo":
        parts = [torch.empty_like(t, device="cpu") for _ in range(world)]
        dist.all_gather(parts, t.cpu(), group=group)
        return [p.to(t.device) for p in parts]
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return parts


def _all_gather_into(out, t, group=None):
    """out (world, *t.shape) <- t of every rank of `group`, in group-rank order."""
    import torch.distributed as dist

    if isinstance(group, LocalGroup):
        group.all_gather_into(out, t)
        return
    if t.is_cuda and dist.get_backend(group) == "gloo":
        for dst, part in zip(out, _all_gather(t.contiguous(), group)):
            dst.copy_(part.view_as(dst))
        return
    dist.all_gather_into_tensor(out.view(-1), t.contiguous().view(-1), group=group)


def exchange_frames_to_tokens(send, recv, group=None):
    """send: (W, T/W, B, S/W, D) by destination -> recv: (W_src, T/W, B, S/W, D)
    = (T, B, S/W, D) token layout (frame index = src * T/W + t)."""
    _all_to_all(recv, send, group)


def exchange_tokens_to_frames(send, recv, group=None):
    """send: (T, B, S/W, D) = (W_dst, T/W, B, S/W, D) -> recv: (W_src, T/W, B, S/W, D)."""
    _all_to_all(recv, send, group)


def unpack_frames(recv, out):
    """(W_src, T/W, B, S/W, D) -> frame shard (B, T/W, S, D) (one bf16 pass)."""
    W, Tl, B, Sw, D = recv.shape
    out.view(B, Tl, W, Sw, D).copy_(recv.permute(2, 1, 0, 3, 4))
    return out


class _SPTemporal:
    """Token-layout workspaces + the temporal-site hook for run_forward."""

    def __init__(self, ctx, world: int, group, ledger: CommReport, bytes_per_element: int, groups: int = 1,
                 transport: str = "nccl", rank: int = 0):
        import torch

        from . import kernels

        if transport not in TRANSPORTS:
            raise ValidationError(f"transport must be one of {TRANSPORTS}, got {transport!r}")
        self.ctx, self.W, self.group, self.ledger = ctx, world, group, ledger
        self.transport, self.rank = transport, rank
        B, Tl, S, D = ctx.B, ctx.T, ctx.S, ctx.D
        T, Sw = Tl * world, S // world
        self.T, self.Sw = T, Sw
        dev = ctx.h.device
        bf = dict(device=dev, dtype=torch.bfloat16)
        rows_tok = T * B * Sw  # == ctx.rows
        self.h_send = ctx.h.view(world, Tl, B, Sw, D)
        self.qkv_tok = torch.empty((rows_tok, 3 * D), **bf)
        self.attn_tok = torch.empty((rows_tok, D), **bf)
        if transport == "peer":
            # token-layout buffers every rank maps: peers store h into h_tok, read o out of o_tok
            from .peer import PeerExchange

            self.px = PeerExchange(group, rank, world, {"h_tok": ((T, B, Sw, D), torch.bfloat16),
                                                        "o_tok": ((T, B, Sw, D), torch.bfloat16)}, dev)
            self.h_tok, self.o_tok = self.px.local["h_tok"], self.px.local["o_tok"]
        else:
            self.px = None
            self.h_tok = torch.empty((T, B, Sw, D), **bf)
            self.o_tok = torch.empty((T, B, Sw, D), **bf)
            self.o_recv = torch.empty((world, Tl, B, Sw, D), **bf)
            self.o_recv.pab_a2a_world = world
        q, k, v = self.qkv_tok[:, :D], self.qkv_tok[:, D:2 * D], self.qkv_tok[:, 2 * D:]
        ld = 3 * D
        # token layout rows (t, b, s): problem (a = b, b_idx = s), rows i = t (stride B*Sw rows)
        st = (Sw * ld, ld, B * Sw * ld)
        self.args = kernels.attn_args(q, k, v, self.attn_tok, st, st, st, (Sw * D, D, B * Sw * D), B, Sw, T, T,
                                      ctx.H, ctx.dh)
        self.el = _alltoall_elements(B, ctx.cfg, world)
        self.wire = Tl * B * Sw * D * 2 * (world - 1)
        self.groups = groups  # split_batch: the job-wide ledger holds one entry per rank group
        self.bpe = bytes_per_element

    def __call__(self, st, li, lp):
        import torch

        from . import kernels
        from .model import MOD_TEMPORAL

        ctx, d = self.ctx, st.decisions
        source = d.source(li, TM)
        site = (li, TM, "t")
        if source == st.step and self.px is not None:
            self._compute_peer(st, li, lp, d.should_store(li, TM))
            return
        if source == st.step:
            store = d.should_store(li, TM)
            p = lp.temporal
            gamma, beta = self._ln(p)
            kernels.residual_modnorm_sp(st.src.view(-1, ctx.D), st.r.view(-1, ctx.D), st.pending, ctx.h,
                                        (ctx.B, ctx.T, ctx.S, ctx.D), self.W, mod=st.mods[li, MOD_TEMPORAL],
                                        gamma=gamma, beta=beta, mode=1)
            ctx.launches.prologue_calls += 1
            st.src, st.pending = st.r, []
            exchange_frames_to_tokens(self.h_send, self.h_tok, self.group)
            self._log(st.step, li)
            kernels.gemm(self.h_tok.view(-1, ctx.D), p.w_qkv_t, self.qkv_tok)
            kernels.attention(self.args, ctx.attn_impl)
            kernels.gemm(self.attn_tok, p.wo_t, self.o_tok.view(-1, ctx.D))
            # the received output stays in all-to-all order (W_src, T/W, B, S/W, D); the next
            # prologue adds it through its row map (PAB_LAYOUT_A2A) -- no unpack pass.  A cached
            # output is received straight into its own buffer.
            o = torch.empty_like(self.o_recv) if store else self.o_recv
            exchange_tokens_to_frames(self.o_tok, o, self.group)
            self._log(st.step, li)
            o.pab_a2a_world = self.W
            if store:
                st.cache.store(site, o, st.step, "outputs")
            ctx.launches.attention_calls += 1
            ctx.launches.gemm_calls += 2
            ctx.launches.sites_computed += 1
            decision = "compute"
        else:
            entry = st.cache.fetch(site, "outputs")
            if entry.source_step != source:
                raise PolicyError(f"temporal cache holds step {entry.source_step}, table expects {source}")
            o = entry.value
            ctx.launches.sites_reused += 1
            decision = "reuse"
        st.pending.append(o)
        st.record(li, TM, "t", decision, source, o)

    def _ln(self, p):
        """LayerNorm affine of a site (None, None at the reference init: gamma = 1, beta = 0)."""
        if self.ctx.params.ln_identity:
            return None, None
        return p.ln_gamma, p.ln_beta

    def _compute_peer(self, st, li, lp, store):
        """Computed temporal site over NVLink peer memory: the prologue's stores are the
        frames->tokens exchange, the next prologue's loads the tokens->frames one."""
        import torch

        from . import kernels
        from .model import MOD_TEMPORAL

        ctx, p, px = self.ctx, lp.temporal, self.px
        if st.wants_output():
            raise ValidationError("output digests/snapshots are not available with the peer transport")
        gamma, beta = self._ln(p)
        kernels.residual_modnorm(st.src.view(-1, ctx.D), st.r.view(-1, ctx.D), st.pending, mod=st.mods[li, MOD_TEMPORAL],
                                 gamma=gamma, beta=beta, mode=1, shape=(ctx.B, ctx.T, ctx.S), h_peer=(px, "h_tok"))
        ctx.launches.prologue_calls += 1
        st.src, st.pending = st.r, []
        px.barrier()  # every rank's h rows have landed in every h_tok
        self._log(st.step, li)
        kernels.gemm(self.h_tok.view(-1, ctx.D), p.w_qkv_t, self.qkv_tok)
        kernels.attention(self.args, ctx.attn_impl)
        kernels.gemm(self.attn_tok, p.wo_t, self.o_tok.view(-1, ctx.D))
        px.barrier()  # every rank's o_tok is complete (and every h_tok read)
        self._log(st.step, li)
        o = self.o_tok.view(self.o_tok.shape)  # a fresh view object carries the peer marker
        o.pab_peer = (px, "o_tok")
        if store:
            slot = torch.empty((ctx.B, ctx.T, ctx.S, ctx.D), device=o.device, dtype=torch.bfloat16)
            o.pab_peer_copy = slot  # filled frame-major by the prologue that consumes o
            st.cache.store((li, TM, "t"), slot, st.step, "outputs")
        ctx.launches.attention_calls += 1
        ctx.launches.gemm_calls += 2
        ctx.launches.other_calls += 2
        ctx.launches.sites_computed += 1
        st.pending.append(o)
        st.record(li, TM, "t", "compute", st.step, o)

    def _log(self, step, layer):
        for _ in range(self.groups):
            self.ledger.entries.append(CommEntry(step, layer, self.ledger.method, self.el, self.el * self.bpe,
                                                 self.el > 0, self.wire))


class ShardedDenoiser(GraphReplay):
    """Frame-sharded denoising run on this rank (broadcast SP).  With an NCCL group the
    whole video -- all-to-alls included -- replays as one CUDA graph (``capture_graph``)."""

    def __init__(self, params: ModelParams, schedule, table: DecisionTable, text_ids, *, guidance: bool,
                 guidance_scale: float, rank: int, world: int, group=None, method: str = "broadcast_sp",
                 noise_params: NoiseParams = DEFAULT_NOISE, bytes_per_element: int = 4, trace=None,
                 half: Optional[int] = None, cfg_group=None, total_workers: Optional[int] = None,
                 transport: str = "nccl"):
        """rank/world/group: this rank's position in its sequence-parallel group.
        split_batch: half = 0 (conditional) / 1 (unconditional) CFG half run by this
        group, cfg_group = the 2-rank group {cond rank, uncond rank} of these frames."""
        from .runtime import StepContext

        cfg = params.cfg
        self.plan = plan_shards(world, cfg)
        self.params, self.table, self.rank, self.world, self.group = params, table, rank, world, group
        self.guidance, self.g = bool(guidance), float(guidance_scale)
        self.half, self.cfg_group = half, cfg_group
        split = half is not None
        if split and not guidance:
            raise ValidationError("split_batch needs classifier-free guidance")
        self.batch = 1 if split else (2 if guidance else 1)
        ids = np.asarray(text_ids, dtype=np.int64)
        if split:
            self.ids = (ids if half == 0 else np.full_like(ids, -1))[None, :]
        else:
            self.ids = np.stack([ids, np.full_like(ids, -1)]) if guidance else ids[None, :]
        ts = list(getattr(schedule, "timesteps", schedule))
        self.timesteps = ts
        self.alphas = [(noise_params.alpha_bar(t), noise_params.alpha_bar(ts[i + 1]) if i + 1 < len(ts) else 1.0)
                       for i, t in enumerate(ts)]
        self.ctx = StepContext.build(params, self.batch, self.ids, ts, frames=self.plan.frames_per_worker)
        self.ledger = CommReport(method, total_workers or world, bytes_per_element, METHOD_COSTS[method])
        self.transport = transport
        self.hook = (_SPTemporal(self.ctx, world, group, self.ledger, bytes_per_element, 2 if split else 1,
                                 transport=transport, rank=rank)
                     if world > 1 else None)
        self.cache = CacheStore()
        self.trace = trace
        self._r = None
        self._pair = None

    def shard_input(self, x_full):
        """This rank's frames of a full (B, T, S, D) latent (contiguous copy)."""
        n = self.plan.frames_per_worker
        return x_full[:, self.rank * n:(self.rank + 1) * n].contiguous()

    def run(self, z, on_step=None):
        import torch

        from .runtime import run_forward

        if self._r is None or self._r.shape != z.shape:
            self._r = torch.empty_like(z)
        split = self.half is not None
        # ledger and decision log describe the latest run (a long-lived server does not accumulate)
        self.ledger.entries.clear()
        self.ctx.launches.log.clear()
        if split and (self._pair is None or self._pair[0].shape[1:] != z.shape[1:]):
            # (2, T/W, S, D) pair buffers: eps of both halves, latent slot per half
            self._pair = (torch.empty((2, *z.shape[1:]), device=z.device, dtype=z.dtype),
                          torch.empty((2, *z.shape[1:]), device=z.device, dtype=z.dtype))
        for i, t in enumerate(self.timesteps):
            a_cur, a_next = self.alphas[i]
            if not split:
                run_forward(self.ctx, i, t, z, self._r, self.table.slice(i), self.cache, trace=self.trace,
                            finish="ddim", ddim=(self.guidance, self.g, a_cur, a_next), temporal_hook=self.hook)
            else:
                # eps of this half -> exchange with the partner rank -> the shared CFG + DDIM update
                # (reference parallel.py:446-457: eps_hat = eps_u + g (eps_c - eps_u) for both halves)
                run_forward(self.ctx, i, t, z, self._r, self.table.slice(i), self.cache, trace=self.trace,
                            finish="residual", temporal_hook=self.hook)
                eps2, z2 = self._pair
                _all_gather_into(eps2, self._r, self.cfg_group)
                z2[self.half].copy_(z[0])
                z2[1 - self.half].copy_(z[0])
                from . import kernels

                kernels.ddim_cfg(z2, eps2, [], True, self.g, a_cur, a_next)
                self.ctx.launches.other_calls += 1
                z[0].copy_(z2[self.half])
            if on_step is not None:
                on_step(i, z)
        return z

    def __call__(self, x_host, out=None):
        """Serving call on this rank: H2D of its frames (of its CFG half under
        split_batch) of the pinned host latent, denoise, D2H into `out` (or a new tensor)."""
        import torch

        n = self.plan.frames_per_worker
        sl = slice(self.rank * n, (self.rank + 1) * n)
        bs = range(x_host.shape[0]) if self.half is None else [self.half]
        dev = self.params.w_time.device
        z = torch.empty((len(bs), n, *x_host.shape[2:]), device=dev, dtype=x_host.dtype)
        # x_host[b, frames] is contiguous: one async H2D per batch entry straight from the
        # caller's (pinned) buffer, no host-side gather of the strided frame slice
        for j, b in enumerate(bs):
            z[j].copy_(x_host[b, sl], non_blocking=True)
        if getattr(self, "_graph", None) is not None:
            self.run_graph(z)
        else:
            self.run(z)
        if out is None:
            return z.cpu()
        for j, b in enumerate(bs):
            out[b, sl].copy_(z[j], non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()  # `out` is host memory: valid on return
        return out


def split_batch_denoiser(params: ModelParams, schedule, table: DecisionTable, text_ids, *, guidance_scale: float,
                         method: str = "broadcast_sp", noise_params: NoiseParams = DEFAULT_NOISE,
                         bytes_per_element: int = 4, trace=None, transport: str = "nccl") -> "ShardedDenoiser":
    """Collective (every rank calls it): CFG halves on two rank groups of W/2
    (reference parallel.py:410-434).  Ranks [0, W/2) run the conditional half,
    [W/2, W) the unconditional one; rank w and W/2 + w hold the same frames."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    if world < 2 or world % 2:
        raise ValidationError("split_batch needs an even number of ranks")
    gw = world // 2
    # new_group is collective over the default group: every rank creates every group, same order
    sp = [dist.new_group(list(range(g * gw, (g + 1) * gw))) for g in range(2)]
    pairs = [dist.new_group([w, gw + w]) for w in range(gw)]
    half, w = divmod(rank, gw)
    return ShardedDenoiser(params, schedule, table, text_ids, guidance=True, guidance_scale=guidance_scale,
                           rank=w, world=gw, group=sp[half], method=method, noise_params=noise_params,
                           bytes_per_element=bytes_per_element, trace=trace, half=half, cfg_group=pairs[w],
                           total_workers=world, transport=transport)


@dataclass
class ParallelRunResult:
    latent: np.ndarray
    comm_report: CommReport
    plan: ShardPlan
    worker_caches: list

    def gathered_cache(self) -> dict:
        """Frame-concatenated cache snapshots.  Multi-process runs only hold this
        rank's shard, so gathering goes through all_gather (collective)."""
        import torch

        merged: dict = {}
        if not self.worker_caches:
            return merged
        local = self.worker_caches[0]
        import torch.distributed as dist

        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
        from .runtime import canonical

        for site, entry in sorted(local.entries.items(), key=lambda kv: str(kv[0])):
            # a rank group of one runs the serial temporal site, whose cache is token-major
            shard = (self._batch, self.plan.frames_per_worker, self._tail[0])
            v = canonical(entry.value, shard).contiguous()
            if multi:
                parts = _all_gather(v.contiguous())
            else:
                parts = [canonical(c.entries[site].value, shard) for c in self.worker_caches]
            B = self._batch
            parts = [p.reshape(B, -1, *self._tail) for p in parts]
            gw = getattr(self, "_split_gw", None)
            if gw:  # split_batch: frames within a rank group, CFG halves across the two groups
                full = torch.cat([torch.cat(parts[:gw], dim=1), torch.cat(parts[gw:], dim=1)], dim=0)
            else:
                full = torch.cat(parts, dim=1)
            merged[site] = full.float().cpu().numpy()
        return merged


def run_parallel(
    params: ModelParams,
    schedule,
    policy: PolicyConfig,
    workers: int,
    method: str = "dsp",
    seed: int = 0,
    text_ids: Optional[Sequence[int]] = None,
    *,
    guidance: bool = False,
    guidance_scale: float = 4.0,
    split_batch: bool = False,
    range_semantics: str = "period",
    noise_params: NoiseParams = DEFAULT_NOISE,
    table: Optional[DecisionTable] = None,
    bytes_per_element: int = 4,
    transport: str = "nccl",
) -> ParallelRunResult:
    """Sequence-parallel sampler (reference parallel.run_parallel, parallel.py:372-464).

    Every rank of an initialised torch.distributed group of size ``workers``
    calls this collectively (one process per GPU, NCCL); each returns the
    gathered full latent.  Without a process group, ``workers`` logical
    workers run in this process on the current GPU, as the reference runs
    them (one thread per worker, shards exchanged through ``LocalGroup``);
    ``workers == 1`` is the single-GPU engine.  ``transport`` (B200 extension):
    "nccl" runs the temporal site's reshards as all-to-alls, "peer" as stores and
    loads over NVLink peer memory fused into the prologues (peer.py).
    """
    import torch
    import torch.distributed as dist

    cfg = params.cfg
    if method not in EXECUTABLE_METHODS:
        raise ValidationError(f"method {method!r} is not executable; use comm_volume_model for it")
    if method == "broadcast_sp" and not isinstance(policy, PabPolicy):
        raise ValidationError("broadcast_sp requires a PAB policy")
    if transport not in TRANSPORTS:
        raise ValidationError(f"transport must be one of {TRANSPORTS}, got {transport!r}")
    if table is None:
        table = build_schedule(policy, schedule, cfg.layers, range_semantics=range_semantics)
    if text_ids is None:
        text_ids = default_text_ids(params)
    multi = dist.is_available() and dist.is_initialized()
    if not multi and workers > 1:
        return _run_logical(params, schedule, table, text_ids, workers, method, seed, guidance, guidance_scale,
                            split_batch, noise_params, bytes_per_element, transport)
    world = dist.get_world_size() if multi else 1
    rank = dist.get_rank() if multi else 0
    if workers != world:
        raise ValidationError(f"run_parallel(workers={workers}) must run in a process group of that size "
                              f"(got world size {world}); launch with torchrun --nproc-per-node {workers}")
    use_split = bool(split_batch and guidance and workers >= 2 and workers % 2 == 0)
    if use_split:
        den = split_batch_denoiser(params, schedule, table, text_ids, guidance_scale=guidance_scale,
                                   method=method, noise_params=noise_params, bytes_per_element=bytes_per_element,
                                   transport=transport)
    else:
        den = ShardedDenoiser(params, schedule, table, text_ids, guidance=guidance, guidance_scale=guidance_scale,
                              rank=rank, world=world, method=method, noise_params=noise_params,
                              bytes_per_element=bytes_per_element, transport=transport)
    batch = 2 if guidance else 1
    x_full = torch.from_numpy(initial_latent(params, seed, batch)).to(params.w_time.device)
    if use_split:
        x_full = x_full[den.half:den.half + 1]
    z = den.shard_input(x_full)
    den.run(z)
    if den.hook is not None and den.hook.px is not None:
        den.hook.px.check()
    if world > 1:
        parts = _all_gather(z)
        if use_split:
            gw = world // 2
            latent = torch.cat([torch.cat(parts[:gw], dim=1), torch.cat(parts[gw:], dim=1)], dim=0)
        else:
            latent = torch.cat(parts, dim=1)
    else:
        latent = z
    res = ParallelRunResult(latent=latent.cpu().numpy(), comm_report=den.ledger, plan=den.plan,
                            worker_caches=[den.cache])
    res._batch = den.batch
    res._tail = (cfg.spatial_tokens, cfg.hidden)
    res._split_gw = world // 2 if use_split else None
    return res


def _run_logical(params, schedule, table, text_ids, workers, method, seed, guidance, guidance_scale, split_batch,
                 noise_params, bytes_per_element, transport="nccl") -> ParallelRunResult:
    """W logical workers on this process's GPU (threads exchanging through LocalGroup).
    With the peer transport each worker issues on its own CUDA stream (the device
    barriers of one worker must not block the others' kernels)."""
    import threading

    import torch

    cfg = params.cfg
    plan_shards(workers, cfg)
    use_split = bool(split_batch and guidance and workers % 2 == 0)
    dev = params.w_time.device
    batch = 2 if guidance else 1
    x_full = torch.from_numpy(initial_latent(params, seed, batch)).to(dev)
    gw = workers // 2 if use_split else workers
    sp = [_LocalGroupState(gw) for _ in range(2 if use_split else 1)]
    pairs = [_LocalGroupState(2) for _ in range(gw)] if use_split else []
    dens, outs, errs = [None] * workers, [None] * workers, []

    def worker(w):
        try:
            torch.cuda.set_device(dev)
            half, r = divmod(w, gw)
            kw = dict(guidance=guidance, guidance_scale=guidance_scale, rank=r, world=gw,
                      group=LocalGroup(sp[half], r), method=method, noise_params=noise_params,
                      bytes_per_element=bytes_per_element)
            if use_split:
                kw.update(half=half, cfg_group=LocalGroup(pairs[r], half), total_workers=workers)
            stream = torch.cuda.Stream(dev) if transport == "peer" else torch.cuda.current_stream(dev)
            stream.wait_stream(torch.cuda.default_stream(dev))
            with torch.cuda.stream(stream):
                den = ShardedDenoiser(params, schedule, table, text_ids, transport=transport, **kw)
                dens[w] = den
                z = den.shard_input(x_full[half:half + 1] if use_split else x_full)
                den.run(z)
                stream.synchronize()
                if den.hook is not None and den.hook.px is not None:
                    den.hook.px.check()
            outs[w] = z
        except BaseException as e:  # noqa: BLE001 - re-raised on the calling thread
            errs.append(e)
            for st in sp + pairs:
                st.barrier.abort()

    threads = [threading.Thread(target=worker, args=(w,), name=f"pab-worker-{w}") for w in range(workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        real = [e for e in errs if not isinstance(e, threading.BrokenBarrierError)]
        raise (real or errs)[0]
    torch.cuda.synchronize(dev)
    if use_split:
        latent = torch.cat([torch.cat(outs[:gw], dim=1), torch.cat(outs[gw:], dim=1)], dim=0)
    else:
        latent = torch.cat(outs, dim=1)
    res = ParallelRunResult(latent=latent.cpu().numpy(), comm_report=dens[0].ledger, plan=dens[0].plan,
                            worker_caches=[d.cache for d in dens])
    res._batch = dens[0].batch
    res._tail = (cfg.spatial_tokens, cfg.hidden)
    res._split_gw = gw if use_split else None
    return res

"""Device-side step engine: workspaces, per-run constants and the site loop.

One ``StepContext`` is built per (params, batch, text ids, timestep list):
it owns every activation buffer of a step (fixed addresses, so attention
argument blocks are built once), the text K/V of every cross site (step
invariant, computed once per run), and the timestep-modulation vectors of
every (step, layer, site) (one batched fp32 GEMM per run).

``run_forward`` walks the reference's site order (model.py:505-566):
    per layer: spatial, cross, mlp | temporal, [cross], mlp
A computed site runs prologue -> projections -> attention/GELU -> output
projection, writing o either into a scratch buffer or, when a later step
reuses it, into a fresh tensor that the cache keeps.  A reused site only
appends its cached o to the pending list.  Pending terms are added to the
fp32 residual stream by the next prologue, in order, so arithmetic order
matches the reference's `x = x + o` chain.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import kernels
from .errors import PolicyError
from .model import (
    ATTENTION_KINDS,
    CAT_MLP,
    CAT_NORM_MOD,
    CAT_OUT,
    CAT_QKV,
    CAT_SCORE,
    CAT_VALUE,
    GELU_FLOPS_PER_ELEM,
    LN_FLOPS_PER_ELEM,
    MOD_MLP_S,
    MOD_MLP_T,
    MOD_SPATIAL,
    MOD_TEMPORAL,
    MODULATE_FLOPS_PER_ELEM,
    SOFTMAX_FLOPS_PER_ELEM,
    ComponentKind,
    ModelParams,
    TraceRecord,
    embed_text,
    embed_text_ids,
    timestep_embedding,
)

SP, TM, CR, ML = ComponentKind.SPATIAL, ComponentKind.TEMPORAL, ComponentKind.CROSS, ComponentKind.MLP

torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False


# A/B switch for measurements: PAB_FUSED_CAST=0 forms the cross query input with the
# stand-alone cast prologue instead of the preceding O GEMM's epilogue
_FUSED_CAST = os.environ.get("PAB_FUSED_CAST", "1") != "0"
# PAB_W2_RESID=1: the MLP's w2 GEMM adds o to the residual in its epilogue (coalesced group
# read-modify-write, no extra smem) instead of the next prologue -- measured neutral on C3
# (w2 0.378 -> 0.405 ms vs a 6E-lighter prologue; 3.048-3.058 s/video both ways), off by default
_W2_RESID = os.environ.get("PAB_W2_RESID", "0") == "1"


@dataclass
class Launches:
    """Per-step accounting of what ran (decision log + kernel counts)."""

    sites_computed: int = 0
    sites_reused: int = 0
    attention_calls: int = 0
    prologue_calls: int = 0
    prologues_fused: int = 0  # cross-site cast passes produced by the preceding O GEMM instead
    gemm_calls: int = 0
    other_calls: int = 0
    log: list = field(default_factory=list)  # (step, layer, kind, block, decision, source)

    def own_kernels(self) -> int:
        # every launch is the library's own kernel: attention, prologue/epilogue, GEMM, DDIM
        return self.attention_calls + self.prologue_calls + self.gemm_calls + self.other_calls


class StepContext:
    def __init__(self):
        pass

    @classmethod
    def build(cls, params: ModelParams, batch: int, text_ids, timesteps, frames: Optional[int] = None):
        """frames: local frame count (sequence-parallel shards hold T/W frames)."""
        self = cls()
        cfg = params.cfg
        dev = params.w_time.device
        self.params, self.cfg, self.B = params, cfg, batch
        self.T = cfg.frames if frames is None else frames
        self.S, self.D, self.H = cfg.spatial_tokens, cfg.hidden, cfg.heads
        self.dh, self.R, self.M = cfg.head_dim, cfg.mlp_hidden, cfg.text_tokens
        self.rows = batch * self.T * self.S
        bf = dict(device=dev, dtype=torch.bfloat16)
        rows, D = self.rows, self.D
        self.h = torch.empty((rows, D), **bf)
        self.qkv = torch.empty((rows, 3 * D), **bf)
        self.attn_out = torch.empty((rows, D), **bf)
        self.qbuf = torch.empty((rows, D), **bf)
        self.hidden = torch.empty((rows, self.R), **bf)  # MLP 4D-wide activation (GELU applied in the w1 GEMM)
        self.o_scratch = torch.empty((rows, D), **bf)
        # the serial temporal site works token-major (rows (b, s, t)); its outputs carry a marker
        self.o_scratch_tm = torch.empty((rows, D), **bf)
        self.o_scratch_tm.pab_token_major = True
        self._cross_slots = {}
        self.shape3 = (batch, self.T, self.S)
        self.launches = Launches()
        self.broadcast_object = "outputs"  # "scores": score broadcast (reference model.py:446-493)
        # debugging override (the default, "auto", selects the tcgen05 kernel for every model shape)
        self.attn_impl = {"auto": kernels.IMPL_AUTO, "tcgen05": kernels.IMPL_TCGEN05,
                          "simt": kernels.IMPL_SIMT}[os.environ.get("PAB_ATTN_IMPL", "auto")]

        # per-run constants: timestep modulation for every (step, layer, slot)
        temb = np.stack([timestep_embedding(float(t), D).astype(np.float32) for t in timesteps])
        t_vecs = torch.as_tensor(temb, device=dev) @ params.w_time              # (N, D) fp32
        # (L, 4, N, 2D) -> (N, L, 4, 2D)
        self.mods = torch.matmul(t_vecs[None, None], params.w_mod_all).permute(2, 0, 1, 3).contiguous()

        # Batch rows whose text is all null (id -1 -> zero embedding, e.g. the unconditional CFG
        # half) have K = V = 0 at every cross site, so the reference's cross output for them is
        # exactly 0 (softmax of zero logits times zero values, model.py:376-385).  When those
        # rows trail the batch, cross sites compute only the leading `cross_live` rows and
        # write zeros for the rest -- bit-identical, half the cross work under CFG.
        ids_arr = embed_text_ids(params.cfg, text_ids, batch)
        null = [bool(np.all(ids_arr[b] < 0)) for b in range(batch)]
        n_null = sum(null)
        self.cross_live = batch - n_null if null[batch - n_null:] == [True] * n_null else batch
        # per-run constants: text K/V of every cross site (step invariant)
        emb = embed_text(params, text_ids, batch).to(torch.bfloat16).reshape(batch * self.M, D)
        self.text_kv = []
        for lp in params.layers:
            kv = []
            for cp in (lp.cross_spatial, lp.cross_temporal):
                kv.append(None if cp is None else
                          kernels.gemm(emb, cp.w_kv_t, torch.empty((batch * self.M, 2 * D), **bf)))
            self.text_kv.append(tuple(kv))

        self._build_attention_args()
        self._delta_in = None
        return self

    def cross_slot(self, key):
        """Per-(layer, block) cached-output slot of a cross site, zero-initialised once: its
        null-text rows (exactly 0 in the reference) are never written, so they stay zero
        across stores without a per-step memset.  A site's cache holds one entry, so the
        slot can be overwritten in place whenever the site stores again."""
        slot = self._cross_slots.get(key)
        if slot is None:
            slot = torch.zeros((self.rows, self.D), device=self.h.device, dtype=torch.bfloat16)
            self._cross_slots[key] = slot
        return slot

    def delta_in(self, r):
        """Copy of the residual at a Delta-DiT layer input (one reused fp32 buffer)."""
        if self._delta_in is None or self._delta_in.shape != r.shape:
            self._delta_in = torch.empty_like(r)
        self._delta_in.copy_(r)
        return self._delta_in

    def _build_attention_args(self):
        B, T, S, D, H, dh, M = self.B, self.T, self.S, self.D, self.H, self.dh, self.M
        q, k, v = self.qkv[:, :D], self.qkv[:, D : 2 * D], self.qkv[:, 2 * D :]
        ld = 3 * D
        # spatial: problem a = frame (B*T), rows = tokens
        self.args_spatial = kernels.attn_args(
            q, k, v, self.attn_out, (S * ld, 0, ld), (S * ld, 0, ld), (S * ld, 0, ld), (S * D, 0, D),
            B * T, 1, S, S, H, dh)
        # temporal: token-major rows (b, s, t) written by the prologue, so each
        # problem (b, s) is T contiguous rows; problems are consecutive (stride T rows)
        self.args_temporal = kernels.attn_args(
            q, k, v, self.attn_out, (0, T * ld, ld), (0, T * ld, ld), (0, T * ld, ld), (0, T * D, D),
            1, B * S, T, T, H, dh)
        # cross: q rows = all (frame, token) of a batch entry, keys = text tokens
        self.args_cross = []
        for kv_s, kv_t in self.text_kv:
            per = []
            for kv in (kv_s, kv_t):
                if kv is None:
                    per.append(None)
                    continue
                kk, vv = kv[:, :D], kv[:, D:]
                per.append(kernels.attn_args(
                    self.qbuf, kk, vv, self.attn_out, (T * S * D, 0, D), (M * 2 * D, 0, 2 * D),
                    (M * 2 * D, 0, 2 * D), (T * S * D, 0, D), self.cross_live, 1, T * S, M, H, dh))
            self.args_cross.append(per)


class _Sink:
    """Analytic flop accounting in the reference's categories (model.py:300-314)."""

    def __init__(self, sink, ctx: StepContext):
        self.sink, self.ctx = sink, ctx

    def site(self, kind, block):
        if self.sink is None:
            return
        c = self.ctx
        E = c.rows * c.D
        D, H, dh = c.D, c.H, c.dh
        add = lambda cat, n: self.sink.add(kind, cat, int(n))  # noqa: E731
        if kind == CR:
            add(CAT_QKV, 2 * E * D + 2 * 2 * (c.B * c.M) * D * D)
            score = c.B * H * c.T * c.S * c.M
            add(CAT_SCORE, 2 * score * dh + SOFTMAX_FLOPS_PER_ELEM * score)
            add(CAT_VALUE, 2 * c.B * H * c.T * c.S * dh * c.M)
            add(CAT_OUT, 2 * E * D)
            return
        add(CAT_NORM_MOD, LN_FLOPS_PER_ELEM * E + 2 * D * 2 * D + MODULATE_FLOPS_PER_ELEM * E)
        if kind == ML:
            add(CAT_MLP, 2 * c.rows * D * c.R + GELU_FLOPS_PER_ELEM * c.rows * c.R + 2 * c.rows * c.R * D)
            return
        n = c.S if kind == SP else c.T
        add(CAT_QKV, 3 * 2 * E * D)
        score = c.rows * H * n
        add(CAT_SCORE, 2 * score * dh + SOFTMAX_FLOPS_PER_ELEM * score)
        add(CAT_VALUE, 2 * c.rows * H * dh * n)
        add(CAT_OUT, 2 * E * D)


    def replay(self, kind):
        """Score replay flops (reference model.py:336-392: modnorm + v projection for the
        axis kinds, text v projection for cross, P.V, output projection)."""
        if self.sink is None:
            return
        c = self.ctx
        E = c.rows * c.D
        D, H, dh = c.D, c.H, c.dh
        add = lambda cat, n: self.sink.add(kind, cat, int(n))  # noqa: E731
        if kind == CR:
            add(CAT_QKV, 2 * (c.B * c.M) * D * D)
            add(CAT_VALUE, 2 * c.B * H * c.T * c.S * dh * c.M)
        else:
            n = c.S if kind == SP else c.T
            add(CAT_NORM_MOD, LN_FLOPS_PER_ELEM * E + 2 * D * 2 * D + MODULATE_FLOPS_PER_ELEM * E)
            add(CAT_QKV, 2 * E * D)
            add(CAT_VALUE, 2 * c.rows * H * dh * n)
        add(CAT_OUT, 2 * E * D)


class _Step:
    """Mutable state of one forward pass."""

    def __init__(self, ctx, step, t, z, r, decisions, cache, trace, flop_sink):
        self.ctx, self.step, self.t = ctx, step, t
        self.src, self.r = z, r
        self.decisions, self.cache, self.trace = decisions, cache, trace
        self.pending: list = []
        # c.h == bf16(r) with nothing pending: written by the O GEMM of a computed site whose next
        # site is a computing cross site (its query input), which then skips its cast prologue
        self.h_cast = False
        self.emit_h = False  # the next out_gemm should produce that h
        self.sink = _Sink(flop_sink, ctx)
        self.mods = ctx.mods[step]

    # -- helpers ---------------------------------------------------------
    def prologue(self, mode: int, mod=None, ln=None, token_major=False):
        c = self.ctx
        gamma = beta = None
        if ln is not None and not c.params.ln_identity:
            gamma, beta = ln
        kernels.residual_modnorm(self.src.view(-1, c.D), self.r.view(-1, c.D), self.pending, h_out=c.h,
                                 mod=mod, gamma=gamma, beta=beta, mode=mode, shape=c.shape3,
                                 h_token_major=token_major)
        c.launches.prologue_calls += 1
        self.src = self.r
        self.pending = []
        self.h_cast = False

    def flush(self):
        """Materialise the residual stream (no normalised output)."""
        c = self.ctx
        if self.pending or self.src is not self.r:
            kernels.residual_modnorm(self.src.view(-1, c.D), self.r.view(-1, c.D), self.pending, mode=0,
                                     shape=c.shape3)
            c.launches.prologue_calls += 1
        self.src = self.r
        self.pending = []

    def out_buffer(self, store: bool, token_major: bool = False):
        c = self.ctx
        if not store:
            return c.o_scratch_tm if token_major else c.o_scratch
        o = torch.empty((c.rows, c.D), device=c.h.device, dtype=torch.bfloat16)
        if token_major:
            o.pab_token_major = True
        return o

    def record(self, li, kind, block, decision, source, o):
        c = self.ctx
        c.launches.log.append((self.step, li, kind.value, block, decision, source))
        if self.trace is not None:
            self.trace.observe(TraceRecord(step=self.step, timestep=self.t, layer=li, kind=kind, block=block,
                                           decision=decision, source_step=source), o)

    def wants_output(self) -> bool:
        """A trace that digests / snapshots site outputs needs o even when it is not cached."""
        return self.trace is not None and getattr(self.trace, "snapshot_mode", "none") in ("digest", "snapshot",
                                                                                          "device")

    def out_gemm(self, a, w_t, store: bool, token_major: bool = False, rows=None, site=None):
        """Output projection of a computed attention site fused with its residual add: the
        GEMM epilogue does r += o (reference model.py:503) and writes o only when a later
        step reuses it (or a trace digests it).  Called right after the site's prologue, so
        the pending list is empty and r is the current stream.  (C3: the next prologue then
        moves 6E instead of 12E bytes; measured 3.5% per video.  The MLP's w2 GEMM keeps the
        plain epilogue: at K = 4D the residual variant's shallower smem ring cost more than
        the prologue saved, profiles/r02_gemm_tuning.md.)"""
        c = self.ctx
        if token_major and not kernels.residual_token_major_ok(c.T, c.S):
            # no whole-token 128-row blocks: plain GEMM, the next prologue adds o (token-major
            # pending term) as before
            o = self.out_buffer(store, token_major)
            kernels.gemm(a, w_t, o)
            return o
        x = self.r.view(-1, c.D)
        need = store or self.wants_output()
        o = None
        if need:
            # cross sites always land in their zeroed per-site slot, so a traced (uncached) output
            # also carries the exact zeros of its null-text rows
            o = c.cross_slot(site) if site is not None else self.out_buffer(store, token_major)
        tm = (c.T, c.S) if token_major else None
        if rows is not None:
            kernels.gemm_residual(a[:rows], w_t, x[:rows], None if o is None else o[:rows], token_major=tm)
        else:
            emit = self.emit_h and not self.pending and self.src is self.r
            kernels.gemm_residual(a, w_t, x, o, token_major=tm, h=c.h if emit else None,
                                  h_rows=c.cross_live * c.T * c.S)
            self.h_cast = emit
        self.emit_h = False
        self.added = True
        return o

    def run_site(self, li, kind, block, compute, token_major=False, scores=None):
        """scores: (capture, replay) closures of an attention site in score-broadcast
        mode (reference model.py:469-499): a stored compute caches the bf16
        probabilities instead of the output, a reuse replays them against the
        current step's values."""
        d = self.decisions
        source = d.source(li, kind)
        site = (li, kind, block)
        c = self.ctx
        self.added = False
        if source == self.step:
            store = d.should_store(li, kind)
            if scores is not None and store:
                o, probs = scores[0](self.out_buffer(False, token_major))
                self.cache.store(site, probs, self.step, "scores")
            else:
                o = compute(store)
                if store:
                    self.cache.store(site, o, self.step, "outputs")
            self.sink.site(kind, block)
            c.launches.sites_computed += 1
            decision = "compute"
        else:
            entry = self.cache.fetch(site, "scores" if scores is not None else "outputs")
            if entry.source_step != source:
                raise PolicyError(f"cache for {site} holds step {entry.source_step}, table expects {source}")
            if scores is not None:
                o = scores[1](entry.value)
                self.sink.replay(kind)
            else:
                o = entry.value
            c.launches.sites_reused += 1
            decision = "reuse"
        if not self.added:
            self.pending.append(o)
        self.record(li, kind, block, decision, source, o)

    # -- score broadcast (K10) ---------------------------------------------
    # Probabilities are materialised per (problem, head): logits by a cuBLAS
    # batched GEMM with fp32 output, softmax by pab_softmax_rows into bf16 P,
    # P.V by a cuBLAS batched GEMM.  Only taken when broadcast_object="scores"
    # and the table stores the site; the paper measures this mode slower than
    # output broadcast (PAPER Table 3), the default path never runs it.
    def _split(self, x, problems, n):
        c = self.ctx
        return x.reshape(problems, n, c.H, c.dh).permute(0, 2, 1, 3).reshape(problems * c.H, n, c.dh)

    def _merge_into_attn_out(self, out, problems, n):
        c = self.ctx
        c.attn_out.view(problems, n, c.H, c.dh).copy_(out.view(problems, c.H, n, c.dh).permute(0, 2, 1, 3))

    def _qkv_heads(self, kind, blk):
        c = self.ctx
        D = c.D
        if kind == CR:
            kv = c.text_kv[self._li][blk]
            return (self._split(c.qbuf, c.B, c.T * c.S), self._split(kv[:, :D], c.B, c.M),
                    self._split(kv[:, D:], c.B, c.M), c.B, c.T * c.S)
        problems, n = (c.B * c.T, c.S) if kind == SP else (c.B * c.S, c.T)  # temporal rows are token-major
        q, k, v = (self._split(c.qkv[:, i * D:(i + 1) * D], problems, n) for i in range(3))
        return q, k, v, problems, n

    def _probs_out(self, kind, blk):
        c = self.ctx
        q, k, v, problems, n = self._qkv_heads(kind, blk)
        logits = torch.bmm(q, k.transpose(1, 2), out_dtype=torch.float32)
        probs = torch.empty(logits.shape, device=logits.device, dtype=torch.bfloat16)
        kernels.softmax_rows(logits, probs, 1.0 / float(np.sqrt(c.dh)))
        del logits
        self._merge_into_attn_out(torch.bmm(probs, v), problems, n)
        c.launches.other_calls += 1
        c.launches.gemm_calls += 2
        return probs

    def attn_scores(self, p, slot, temporal):
        c = self.ctx
        kind = TM if temporal else SP

        def capture(o):
            self.prologue(1, self.mods[self._li, slot], (p.ln_gamma, p.ln_beta), token_major=temporal)
            kernels.gemm(c.h, p.w_qkv_t, c.qkv)
            probs = self._probs_out(kind, None)
            kernels.gemm(c.attn_out, p.wo_t, o)
            c.launches.gemm_calls += 2
            return o, probs

        def replay(probs):
            # reference _axis_attention_replay (model.py:362-373): modnorm -> v only -> P.V -> wo
            # v through the same fused QKV GEMM as the capture step, so replaying on an unchanged
            # input reproduces the computed output bit for bit (reference test_model.py:138-151)
            self.prologue(1, self.mods[self._li, slot], (p.ln_gamma, p.ln_beta), token_major=temporal)
            kernels.gemm(c.h, p.w_qkv_t, c.qkv)
            _, _, v, problems, n = self._qkv_heads(kind, None)
            self._merge_into_attn_out(torch.bmm(probs, v), problems, n)
            o = self.out_buffer(True, temporal)  # fresh: pending terms may still reference scratch
            kernels.gemm(c.attn_out, p.wo_t, o)
            c.launches.gemm_calls += 3
            return o

        return capture, replay

    def cross_scores(self, p, blk):
        c = self.ctx

        def capture(o):
            self.prologue(2)
            kernels.gemm(c.h, p.wq_t, c.qbuf)
            probs = self._probs_out(CR, blk)
            kernels.gemm(c.attn_out, p.wo_t, o)
            c.launches.gemm_calls += 2
            return o, probs

        def replay(probs):
            # reference _cross_attention_replay (model.py:388-395): text v -> P.V -> wo; x untouched
            kv = c.text_kv[self._li][blk]
            self._merge_into_attn_out(torch.bmm(probs, self._split(kv[:, c.D:], c.B, c.M)), c.B, c.T * c.S)
            o = self.out_buffer(True)
            kernels.gemm(c.attn_out, p.wo_t, o)
            c.launches.gemm_calls += 2
            return o

        return capture, replay

    # -- site bodies -------------------------------------------------------
    def attn_site(self, p, slot, temporal):
        c = self.ctx

        def compute(store):
            self.prologue(1, self.mods[self._li, slot], (p.ln_gamma, p.ln_beta), token_major=temporal)
            kernels.gemm(c.h, p.w_qkv_t, c.qkv)
            kernels.attention(c.args_temporal if temporal else c.args_spatial, c.attn_impl)
            c.launches.attention_calls += 1
            c.launches.gemm_calls += 2
            return self.out_gemm(c.attn_out, p.wo_t, store, token_major=temporal)

        return compute

    def cross_site(self, p, blk):
        c = self.ctx

        def compute(store):
            if self.h_cast and not self.pending and self.src is self.r:
                # the previous site's O GEMM already wrote h = bf16(x) (its residual epilogue)
                self.h_cast = False
                c.launches.prologues_fused += 1
            else:
                self.prologue(2)
            rl = c.cross_live * c.T * c.S  # rows with non-null text (see StepContext.build)
            if rl == 0:  # every row null: the output is exactly 0, nothing to add
                self.added = True
                return c.cross_slot((self._li, blk)) if (store or self.wants_output()) else None
            kernels.gemm(c.h[:rl], p.wq_t, c.qbuf[:rl])
            kernels.attention(c.args_cross[self._li][blk], c.attn_impl)
            c.launches.attention_calls += 1
            c.launches.gemm_calls += 2
            # null-text rows of a cached output stay the zeros of its per-site slot
            return self.out_gemm(c.attn_out, p.wo_t, store, rows=rl, site=(self._li, blk))

        return compute

    def mlp_site(self, p, slot):
        c = self.ctx

        def compute(store):
            self.prologue(1, self.mods[self._li, slot], (p.ln_gamma, p.ln_beta))
            # w1 GEMM with the tanh-GELU applied in its epilogue (no extra HBM pass over
            # the 4D-wide hidden activation), then w2; the next prologue adds o
            kernels.gemm(c.h, p.w1_t, c.hidden, kernels.EPI_GELU)
            c.launches.gemm_calls += 2
            if _W2_RESID:
                # w2 with the residual add in its epilogue (direct read-modify-write at K = 4D):
                # r += o here, o written only when cached / traced
                x = self.r.view(-1, c.D)
                o = self.out_buffer(store) if (store or self.wants_output()) else None
                kernels.gemm_residual(c.hidden, p.w2_t, x, o)
                self.added = True
                return o
            o = self.out_buffer(store)
            kernels.gemm(c.hidden, p.w2_t, o)
            return o

        return compute

    def layer(self, li, lp, temporal_hook=None):
        self._li = li
        d = self.decisions
        delta = bool(getattr(d, "delta_mode", False))
        if delta and d.layer_fully_reused(li):
            source = d.source(li, SP)
            entry = self.cache.fetch((li, None, "delta"), "delta")
            if entry.source_step != source:
                raise PolicyError(f"delta cache for layer {li} holds step {entry.source_step}, table expects {source}")
            # the fp32 delta is added to the materialised residual (reference keeps it fp32)
            self.flush()
            kernels.add_scaled_(self.r, self.r, entry.value, 1.0)
            self.ctx.launches.other_calls += 1
            sites = [(SP, "s"), (CR, "s"), (ML, "s"), (TM, "t"), (ML, "t")]
            if self.ctx.cfg.cross_in_temporal:
                sites.insert(4, (CR, "t"))
            for kind, block in sites:
                self.record(li, kind, block, "delta", d.source(li, kind), None)
            return
        x_in = None
        if delta and d.should_store_delta(li):
            self.flush()
            x_in = self.ctx.delta_in(self.r)
        sc = self.ctx.broadcast_object == "scores"
        live = self.ctx.cross_live > 0 and _FUSED_CAST
        self.emit_h = live and not sc and d.source(li, CR) == self.step  # spatial O GEMM -> cross q input
        self.run_site(li, SP, "s", self.attn_site(lp.spatial, MOD_SPATIAL, False),
                      scores=self.attn_scores(lp.spatial, MOD_SPATIAL, False) if sc else None)
        self.run_site(li, CR, "s", self.cross_site(lp.cross_spatial, 0),
                      scores=self.cross_scores(lp.cross_spatial, 0) if sc else None)
        self.run_site(li, ML, "s", self.mlp_site(lp.mlp_spatial, MOD_MLP_S))
        if temporal_hook is not None:
            temporal_hook(self, li, lp)
        else:
            self.emit_h = live and not sc and self.ctx.cfg.cross_in_temporal and d.source(li, CR) == self.step
            self.run_site(li, TM, "t", self.attn_site(lp.temporal, MOD_TEMPORAL, True), token_major=True,
                          scores=self.attn_scores(lp.temporal, MOD_TEMPORAL, True) if sc else None)
        if self.ctx.cfg.cross_in_temporal:
            self.run_site(li, CR, "t", self.cross_site(lp.cross_temporal, 1),
                          scores=self.cross_scores(lp.cross_temporal, 1) if sc else None)
        self.run_site(li, ML, "t", self.mlp_site(lp.mlp_temporal, MOD_MLP_T))
        if x_in is not None:
            self.flush()
            delta = torch.empty_like(self.r)
            kernels.add_scaled_(delta, self.r, x_in, -1.0)  # fp32 x - x_layer_in (model.py:565-566)
            self.ctx.launches.other_calls += 1
            self.cache.store((li, None, "delta"), delta, self.step, "delta")


def run_forward(ctx: StepContext, step_index: int, t: float, z, r, decisions, cache, trace=None, flop_sink=None,
                finish="residual", ddim=None, temporal_hook=None):
    """Run every layer of one step (ctx.broadcast_object selects output or score
    broadcast).  finish="residual": r <- eps.
    finish="ddim": z <- DDIM(z, CFG(eps)) with ddim=(guidance, g, a_cur, a_next)."""
    st = _Step(ctx, step_index, t, z, r, decisions, cache, trace, flop_sink)
    st.step = decisions.step
    t0 = time.perf_counter()
    for li, lp in enumerate(ctx.params.layers):
        st.layer(li, lp, temporal_hook)
    if finish == "residual":
        st.flush()
    else:
        guidance, g, a_cur, a_next = ddim
        if st.src is not st.r or len(st.pending) > kernels.MAX_PENDING or any(
                kernels.term_layout(p) for p in st.pending):
            st.flush()  # the fused DDIM kernel drains frame-major terms only
        kernels.ddim_cfg(z, st.r, st.pending, guidance, g, a_cur, a_next)
        ctx.launches.other_calls += 1
    return time.perf_counter() - t0


def canonical(o, shape):
    """Frame-major (B, T, S, D) view of a site output (token-major outputs of the
    serial temporal site and all-to-all ordered outputs of the sequence-parallel one
    are permuted back); for tests and gathered caches."""
    B, T, S = shape
    lay = kernels.term_layout(o)
    if lay == kernels.LAYOUT_TOKEN:
        return o.view(B, S, T, -1).permute(0, 2, 1, 3).reshape(B, T, S, -1)
    if lay == kernels.LAYOUT_A2A:
        W = int(o.pab_a2a_world)
        return o.view(W, T, B, S // W, -1).permute(2, 1, 0, 3, 4).reshape(B, T, S, -1)
    return o.view(B, T, S, -1)


__all__ = ["StepContext", "run_forward", "Launches", "ATTENTION_KINDS", "canonical"]

"""Video DiT forward step on B200 under per-step broadcast decisions.

Drop-in for pkg/src/pab_engine/model.py: same ModelConfig, ComponentKind,
init_model draw order and forward_step signature/semantics, but parameters
and activations live in HBM and every site runs on sm_100a kernels:

  site prologue  pab_residual_modnorm  (drain pending residual terms into the
                                        fp32 stream x, emit bf16 modnorm(x) or bf16(x))
  projections    cuBLAS bf16 GEMMs (fused [wq|wk|wv], [wk|wv] for text)
  attention      pab_attention (tcgen05/TMEM/TMA flash kernel; spatial,
                 temporal and cross layouts addressed by strides, no transposes)
  MLP            GEMM -> pab_gelu_bf16 -> GEMM

Residual adds are deferred: a site's output o (bf16, the cache payload) is
appended to a pending list and added to x by the next prologue in reference
order, so a reused site launches no kernel at all -- its cached o is simply
appended (reference run_site, model.py:469-503).
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional

import numpy as np

from .errors import PolicyError, ShapeError, ValidationError

TEXT_VOCAB = 256

CAT_QKV = "qkv_proj"
CAT_SCORE = "score_matmul"
CAT_VALUE = "value_matmul"
CAT_OUT = "output_projection"
CAT_MLP = "mlp"
CAT_NORM_MOD = "norm_modulate"
FLOP_CATEGORIES = (CAT_QKV, CAT_SCORE, CAT_VALUE, CAT_OUT, CAT_MLP, CAT_NORM_MOD)
LN_FLOPS_PER_ELEM = 8
MODULATE_FLOPS_PER_ELEM = 2
SOFTMAX_FLOPS_PER_ELEM = 5
GELU_FLOPS_PER_ELEM = 10


class ComponentKind(str, Enum):
    SPATIAL = "spatial"
    TEMPORAL = "temporal"
    CROSS = "cross"
    MLP = "mlp"


KINDS = tuple(ComponentKind)
KIND_INDEX = {kind: i for i, kind in enumerate(KINDS)}
ATTENTION_KINDS = (ComponentKind.SPATIAL, ComponentKind.TEMPORAL, ComponentKind.CROSS)

# modulated-norm sites per layer, in the order their w_mod draws are stacked
MOD_SPATIAL, MOD_MLP_S, MOD_TEMPORAL, MOD_MLP_T = range(4)


@dataclass(frozen=True)
class ModelConfig:
    layers: int = 4
    hidden: int = 64
    heads: int = 4
    frames: int = 8
    spatial_tokens: int = 64
    text_tokens: int = 16
    mlp_ratio: float = 4.0
    cross_in_temporal: bool = False

    def __post_init__(self):
        for name in ("layers", "hidden", "heads", "frames", "spatial_tokens", "text_tokens"):
            if getattr(self, name) < 1:
                raise ValidationError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.hidden % self.heads != 0:
            raise ValidationError(f"hidden ({self.hidden}) must be divisible by heads ({self.heads})")
        if self.hidden % 2 != 0:
            raise ValidationError("hidden must be even (sinusoidal embedding splits in half)")
        if self.mlp_ratio <= 0:
            raise ValidationError("mlp_ratio must be positive")

    @property
    def mlp_hidden(self) -> int:
        return int(round(self.mlp_ratio * self.hidden))

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def sites_per_layer(self) -> int:
        return 6 if self.cross_in_temporal else 5

    def latent_shape(self, batch: int = 1) -> tuple[int, int, int, int]:
        return (batch, self.frames, self.spatial_tokens, self.hidden)


def param_draw_plan(cfg: ModelConfig) -> list[tuple[str, int, int]]:
    """(name, rows, cols) of every drawn matrix in stream order
    (reference init_model, model.py:168-222)."""
    d, r = cfg.hidden, cfg.mlp_hidden
    plan = [("text_table", TEXT_VOCAB, d), ("w_time", d, d)]

    def attn(pref):
        return [(f"{pref}.w_mod", d, 2 * d), (f"{pref}.wq", d, d), (f"{pref}.wk", d, d),
                (f"{pref}.wv", d, d), (f"{pref}.wo", d, d)]

    def cross(pref):
        return [(f"{pref}.wq", d, d), (f"{pref}.wk", d, d), (f"{pref}.wv", d, d), (f"{pref}.wo", d, d)]

    def mlp(pref):
        return [(f"{pref}.w_mod", d, 2 * d), (f"{pref}.w1", d, r), (f"{pref}.w2", r, d)]

    for li in range(cfg.layers):
        p = f"layers.{li}"
        plan += attn(f"{p}.spatial") + cross(f"{p}.cross_spatial") + mlp(f"{p}.mlp_spatial")
        plan += attn(f"{p}.temporal")
        if cfg.cross_in_temporal:
            plan += cross(f"{p}.cross_temporal")
        plan += mlp(f"{p}.mlp_temporal")
    return plan


@dataclass
class AttnParams:
    ln_gamma: object
    ln_beta: object
    w_mod: object      # fp32 (D, 2D)
    w_qkv_t: object    # bf16 (3D, D) = [wq | wk | wv]^T: K-major GEMM operand (pab_gemm_bf16)
    wo_t: object       # bf16 (D, D) = wo^T

    @property
    def w_qkv(self):
        return self.w_qkv_t.t()

    @property
    def wo(self):
        return self.wo_t.t()

    @property
    def wq(self):
        return self.w_qkv[:, : self.wo_t.shape[0]]

    @property
    def wk(self):
        d = self.wo_t.shape[0]
        return self.w_qkv[:, d : 2 * d]

    @property
    def wv(self):
        d = self.wo_t.shape[0]
        return self.w_qkv[:, 2 * d :]


@dataclass
class CrossParams:
    wq_t: object       # bf16 (D, D) = wq^T
    w_kv_t: object     # bf16 (2D, D) = [wk | wv]^T
    wo_t: object

    @property
    def wq(self):
        return self.wq_t.t()

    @property
    def w_kv(self):
        return self.w_kv_t.t()

    @property
    def wo(self):
        return self.wo_t.t()

    @property
    def wk(self):
        return self.w_kv[:, : self.wq_t.shape[0]]

    @property
    def wv(self):
        return self.w_kv[:, self.wq_t.shape[0] :]


@dataclass
class MlpParams:
    ln_gamma: object
    ln_beta: object
    w_mod: object
    w1_t: object       # bf16 (R, D) = w1^T
    w2_t: object       # bf16 (D, R) = w2^T

    @property
    def w1(self):
        return self.w1_t.t()

    @property
    def w2(self):
        return self.w2_t.t()


@dataclass
class LayerParams:
    spatial: AttnParams
    cross_spatial: CrossParams
    mlp_spatial: MlpParams
    temporal: AttnParams
    cross_temporal: Optional[CrossParams]
    mlp_temporal: MlpParams


@dataclass
class ModelParams:
    cfg: ModelConfig
    seed: int
    dtype: np.dtype
    text_table: object   # fp32 (256, D) on device
    w_time: object       # fp32 (D, D)
    layers: list
    w_mod_all: object    # fp32 (L, 4, D, 2D): every modulation matrix, stacked
    ln_identity: bool = True

    def digest(self) -> str:
        """sha256 over the fp32 master weights in draw order (matches the
        reference's ModelParams.digest for identity LayerNorm affines)."""
        h = hashlib.sha256()
        for arr in iter_param_arrays(self):
            h.update(np.ascontiguousarray(arr).tobytes())
        return h.hexdigest()


def iter_param_arrays(params: ModelParams):
    """Host fp32 copies of the parameters in the reference's iteration order."""
    import torch

    def host(t):
        return t.detach().float().cpu().numpy()

    d = params.cfg.hidden
    yield host(params.text_table)
    yield host(params.w_time)
    for lp in params.layers:
        for a in (lp.spatial, lp.temporal):
            yield from (host(a.ln_gamma), host(a.ln_beta), host(a.w_mod), host(a.wq), host(a.wk), host(a.wv),
                        host(a.wo))
        for c in (lp.cross_spatial, lp.cross_temporal):
            if c is not None:
                yield from (host(c.wq), host(c.wk), host(c.wv), host(c.wo))
        for m in (lp.mlp_spatial, lp.mlp_temporal):
            yield from (host(m.ln_gamma), host(m.ln_beta), host(m.w_mod), host(m.w1), host(m.w2))
    del torch, d


def init_model(cfg: ModelConfig, seed: int, dtype=np.float32, device="cuda") -> ModelParams:
    """Deterministic U(-1/sqrt(D), 1/sqrt(D)) parameters generated on the GPU.

    Same splitmix64 stream and draw order as the reference (model.py:168-222,
    numerics.py:161-201): matrix m takes draws [off_m + 1, off_m + rows*cols]
    of the stream, so every matrix is filled by an independent kernel launch.
    GEMM weights are kept as bf16 copies of the fp32 draws; modulation,
    time-projection and text-table weights stay fp32.
    """
    import torch

    from . import kernels

    if np.dtype(dtype) != np.float32:
        raise ValidationError("the B200 path stores fp32 master weights; dtype must be float32")
    dev = torch.device(device)
    d, r = cfg.hidden, cfg.mlp_hidden
    L = cfg.layers
    bound = 1.0 / np.sqrt(d)
    state = int(seed) & ((1 << 64) - 1)
    f32 = dict(device=dev, dtype=torch.float32)
    bf16 = dict(device=dev, dtype=torch.bfloat16)

    w_mod_all = torch.empty((L, 4, d, 2 * d), **f32)
    text_table = torch.empty((TEXT_VOCAB, d), **f32)
    w_time = torch.empty((d, d), **f32)
    ones = torch.ones(d, **f32)
    zeros = torch.zeros(d, **f32)

    # GEMM weights are drawn into their reference (K, N) layout, then stored transposed
    # ((N, K), K-major) as the tcgen05 GEMM's B operand
    nat: dict = {}

    def buf(key, rows, cols):
        if key not in nat:
            nat[key] = torch.empty((rows, cols), **bf16)
        return nat[key]

    def target(name):
        """(tensor, column offset) receiving the named draw."""
        if name == "text_table":
            return text_table, 0
        if name == "w_time":
            return w_time, 0
        _, li, site, w = name.split(".")
        if w == "w_mod":
            slot = {"spatial": MOD_SPATIAL, "mlp_spatial": MOD_MLP_S, "temporal": MOD_TEMPORAL,
                    "mlp_temporal": MOD_MLP_T}[site]
            return w_mod_all[int(li), slot], 0
        if site in ("spatial", "temporal"):
            if w in ("wq", "wk", "wv"):
                return buf((li, site, "qkv"), d, 3 * d), "qkv".index(w[1]) * d
            return buf((li, site, "o"), d, d), 0
        if site.startswith("cross"):
            if w in ("wk", "wv"):
                return buf((li, site, "kv"), d, 2 * d), (0 if w == "wk" else d)
            return buf((li, site, w), d, d), 0
        return buf((li, site, w), *((d, r) if w == "w1" else (r, d))), 0

    offset = 0
    for name, rows, cols in param_draw_plan(cfg):
        dst, col0 = target(name)
        kernels.fill_uniform(dst, rows, cols, col0, state, offset, -bound, bound)
        offset += rows * cols

    def t_(key):
        return nat.pop(key).t().contiguous()

    layers = []
    for li in range(L):
        k = str(li)

        def attn(site, slot):
            return AttnParams(ones, zeros, w_mod_all[li, slot], t_((k, site, "qkv")), t_((k, site, "o")))

        def cross(site):
            return CrossParams(t_((k, site, "wq")), t_((k, site, "kv")), t_((k, site, "wo")))

        def mlp(site, slot):
            return MlpParams(ones, zeros, w_mod_all[li, slot], t_((k, site, "w1")), t_((k, site, "w2")))

        layers.append(LayerParams(
            spatial=attn("spatial", MOD_SPATIAL), cross_spatial=cross("cross_spatial"),
            mlp_spatial=mlp("mlp_spatial", MOD_MLP_S), temporal=attn("temporal", MOD_TEMPORAL),
            cross_temporal=cross("cross_temporal") if cfg.cross_in_temporal else None,
            mlp_temporal=mlp("mlp_temporal", MOD_MLP_T),
        ))
    return ModelParams(cfg=cfg, seed=seed, dtype=np.dtype(np.float32), text_table=text_table, w_time=w_time,
                       layers=layers, w_mod_all=w_mod_all, ln_identity=True)


def timestep_embedding(t: float, hidden: int) -> np.ndarray:
    """[sin | cos](t * 10^(-4 k / (D/2 - 1))) in float64 (reference model.py:225-235)."""
    if not 0 <= t <= 1000:
        raise ValidationError(f"timestep must lie in [0, 1000], got {t}")
    half = hidden // 2
    freqs = 10.0 ** (-4.0 * np.arange(half) / (half - 1)) if half > 1 else np.ones(half)
    ang = t * freqs
    return np.concatenate([np.sin(ang), np.cos(ang)])


def array_digest(arr: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(str(arr.dtype).encode())
    h.update(np.asarray(arr.shape, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


@dataclass
class TraceRecord:
    step: int
    timestep: float
    layer: int
    kind: ComponentKind
    block: str
    decision: str
    source_step: int
    flops: int = 0
    seconds: float = 0.0
    attn_seconds: float = 0.0
    digest: Optional[str] = None
    snapshot: Optional[np.ndarray] = None


@dataclass
class ComponentTrace:
    """One record per site per step (reference model.py:262-283).  On the GPU
    digests/snapshots force a device->host copy per site, so they are a debug
    mode; the default used by sample() is snapshot_mode="none"."""

    snapshot_mode: str = "digest"
    snapshot_dtype: np.dtype = np.float16
    records: list = field(default_factory=list)
    total_seconds: float = 0.0

    def observe(self, record: TraceRecord, output):
        if output is not None and self.snapshot_mode in ("digest", "snapshot"):
            host = output.detach().float().cpu().numpy() if hasattr(output, "detach") else np.asarray(output)
            record.digest = array_digest(host)
            if self.snapshot_mode == "snapshot":
                record.snapshot = host.astype(self.snapshot_dtype)
        self.records.append(record)

    def has_reuse(self) -> bool:
        return any(r.decision != "compute" for r in self.records)

    def num_steps(self) -> int:
        return 1 + max((r.step for r in self.records), default=-1)


def embed_text_ids(cfg: ModelConfig, text_ids, batch: int) -> np.ndarray:
    """Validated (batch, M) int64 ids; -1 is the null (zero) token (model.py:406-417)."""
    ids = np.asarray(text_ids, dtype=np.int64)
    if ids.ndim == 1:
        ids = np.tile(ids[None, :], (batch, 1))
    if ids.shape != (batch, cfg.text_tokens):
        raise ShapeError(f"text ids shape {ids.shape} != ({batch}, {cfg.text_tokens})")
    if np.any(ids >= TEXT_VOCAB):
        raise ValidationError(f"text ids must be < {TEXT_VOCAB}")
    return ids


def embed_text(params: ModelParams, text_ids, batch: int):
    import torch

    ids = embed_text_ids(params.cfg, text_ids, batch)
    idx = torch.as_tensor(np.where(ids < 0, 0, ids), device=params.text_table.device)
    emb = params.text_table[idx]
    emb[torch.as_tensor(ids < 0, device=emb.device)] = 0.0
    return emb


def time_vector(params: ModelParams, t: float):
    import torch

    emb = torch.as_tensor(timestep_embedding(t, params.cfg.hidden).astype(np.float32),
                          device=params.w_time.device)
    return emb[None, :] @ params.w_time


def forward_step(
    params: ModelParams,
    x,
    t: float,
    text_ids,
    decisions,
    cache,
    trace: Optional[ComponentTrace] = None,
    broadcast_object: str = "outputs",
    flop_sink=None,
):
    """One denoising forward pass; returns eps (same shape as x, fp32 on device).

    Same contract as reference forward_step (model.py:425-568): ``decisions``
    is a step slice of a decision table, ``cache`` holds the broadcast
    outputs.  ``x`` may be a numpy array or a CUDA tensor.
    """
    import torch

    from .runtime import StepContext, run_forward

    cfg = params.cfg
    xt = torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x)
    if tuple(xt.shape[1:]) != (cfg.frames, cfg.spatial_tokens, cfg.hidden):
        raise ShapeError(f"latent shape {tuple(xt.shape)} does not match config {cfg}")
    if broadcast_object not in ("outputs", "scores"):
        raise ValidationError(f"unknown broadcast object {broadcast_object!r}")
    xt = xt.to(device=params.w_time.device, dtype=torch.float32).contiguous()
    ctx = StepContext.build(params, xt.shape[0], text_ids, [float(t)])
    ctx.broadcast_object = broadcast_object
    r = torch.empty_like(xt)
    run_forward(ctx, 0, float(t), xt, r, decisions, cache, trace=trace, flop_sink=flop_sink, finish="residual")
    return r


__all__ = [
    "ComponentKind", "KINDS", "KIND_INDEX", "ATTENTION_KINDS", "ModelConfig", "ModelParams", "LayerParams",
    "AttnParams", "CrossParams", "MlpParams", "init_model", "forward_step", "timestep_embedding", "time_vector",
    "embed_text", "ComponentTrace", "TraceRecord", "array_digest", "param_draw_plan", "PolicyError",
]

_ = math

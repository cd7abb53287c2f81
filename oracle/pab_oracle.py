"""CPU ORACLE for the PAB hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or as the
timed CPU baseline.  The product path (paper_2408_12588_b200) never imports
it and has no CPU fallback.

This is an independent numpy restatement of the reference pab-engine
algorithm (pkg/src/pab_engine/, cited per function).  Differences from the
reference, all below the bf16 tolerance the GPU path is held to:
  * contractions use numpy/BLAS matmul instead of the reference's ascending-k
    single-accumulator loop (numerics.py:64-104) -> fp32 rounding order
    differs (~1e-6 relative); pinned against reference-generated fixtures in
    tests/golden/ (see tests/golden/make_golden.py and tests/test_oracle.py);
  * broadcast_object="scores" (score replay, model.py:325-392, 476-493) keeps
    the probabilities in float32 like the reference.
Decision tables are integer work and are restated exactly.

bf16 emulation (``emulate_bf16=True`` on ``sample``/``forward``): every matmul
operand and output is rounded to bf16 (round-to-nearest-even) where the B200
path stores bf16 -- LN/modulate output h, weights, q/k/v, unnormalised softmax
numerators P (the row sum is taken over the rounded P, as the kernels sum P
through a ones column of V), attention output, GELU hidden, site output o, text
embedding and its K/V -- while the residual stream, accumulations and the DDIM
update stay fp32.  It measures the precision floor of a correct bf16 pipeline
(SURVEY.md 8c), which is what the guided (CFG) parity gates are set against.
"""

from __future__ import annotations

import math

import numpy as np

# ----------------------------------------------------------------- PRNG
# reference numerics.py:161-215 (splitmix64; uniform from the top 53 bits;
# Box-Muller on (first half, second half) of the draws)
_G, _M1, _M2 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def splitmix_draws(state: int, n: int) -> np.ndarray:
    ks = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(state) + ks * np.uint64(_G)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


class Stream:
    def __init__(self, seed: int):
        self.state = seed & ((1 << 64) - 1)

    def take(self, n: int) -> np.ndarray:
        out = splitmix_draws(self.state, n)
        self.state = (self.state + n * _G) & ((1 << 64) - 1)
        return out

    def uniform(self, n, lo, hi):
        u = (self.take(n) >> np.uint64(11)).astype(np.float64) * 2.0**-53
        return lo + u * (hi - lo)

    def normal(self, n):
        m = (n + 1) // 2
        raw = self.take(2 * m) >> np.uint64(11)
        u1 = (raw[:m].astype(np.float64) + 1.0) * 2.0**-53
        u2 = raw[m:].astype(np.float64) * 2.0**-53
        rad = np.sqrt(-2.0 * np.log(u1))
        th = 2.0 * math.pi * u2
        z = np.empty(2 * m)
        z[0::2], z[1::2] = rad * np.cos(th), rad * np.sin(th)
        return z[:n]


# ------------------------------------------------------------- model
class Cfg:
    def __init__(self, layers, hidden, heads, frames, spatial_tokens, text_tokens, mlp_ratio=4.0,
                 cross_in_temporal=False):
        self.L, self.D, self.H = layers, hidden, heads
        self.T, self.S, self.M = frames, spatial_tokens, text_tokens
        self.R = int(round(mlp_ratio * hidden))
        self.cross_t = bool(cross_in_temporal)


def init_weights(cfg: Cfg, seed: int) -> dict:
    """Same draw order as reference model.py:168-222; returns a flat dict."""
    rng = Stream(seed)
    d, r = cfg.D, cfg.R
    b = 1.0 / np.sqrt(d)

    def draw(rows, cols):
        return rng.uniform(rows * cols, -b, b).reshape(rows, cols).astype(np.float32)

    w = {"text": draw(256, d), "time": draw(d, d)}
    for li in range(cfg.L):
        def attn(p):
            for name, shape in (("mod", (d, 2 * d)), ("q", (d, d)), ("k", (d, d)), ("v", (d, d)), ("o", (d, d))):
                w[f"{li}.{p}.{name}"] = draw(*shape)

        def cross(p):
            for name in ("q", "k", "v", "o"):
                w[f"{li}.{p}.{name}"] = draw(d, d)

        def mlp(p):
            w[f"{li}.{p}.mod"] = draw(d, 2 * d)
            w[f"{li}.{p}.w1"] = draw(d, r)
            w[f"{li}.{p}.w2"] = draw(r, d)

        attn("sa"); cross("cs"); mlp("ms"); attn("ta")
        if cfg.cross_t:
            cross("ct")
        mlp("mt")
    return w


def bf16_round(a):
    """Round fp32 values to the nearest bf16 (ties to even), returned as fp32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def _ident(a):
    return a


def _ln(x, eps=1e-5):
    # population variance, eps inside the sqrt (numerics.py:115-130)
    mu = x.mean(-1, keepdims=True)
    c = x - mu
    return c * (1.0 / np.sqrt((c * c).mean(-1, keepdims=True) + eps))


def _softmax(z):
    e = np.exp(z - z.max(-1, keepdims=True))
    return e / e.sum(-1, keepdims=True)


_SCORE_CHUNK_BYTES = 1 << 31  # fp32 logits materialised at once (C5 spatial: 53 GB unchunked)


def attention(q, k, v, rb=None):
    """softmax(q k^T / sqrt(dh)) v over the last two axes (numerics.py:133-151).
    rb: bf16 rounding of the unnormalised probabilities (emulation mode).  Large
    problems are evaluated in chunks of the leading (batch, frame, head) axes; every
    chunk is the same per-problem computation, so the result does not depend on it."""
    lead = q.shape[:-2]
    nq, nk = q.shape[-2], k.shape[-2]
    n = int(np.prod(lead)) if lead else 1
    per = max(1, _SCORE_CHUNK_BYTES // max(1, nq * nk * 4))
    if n > per and lead:
        q2 = q.reshape(n, nq, q.shape[-1])
        k2 = np.broadcast_to(k, lead + k.shape[-2:]).reshape(n, nk, k.shape[-1])
        v2 = np.broadcast_to(v, lead + v.shape[-2:]).reshape(n, nk, v.shape[-1])
        out = np.empty((n, nq, v.shape[-1]), dtype=np.result_type(q, v))
        for i in range(0, n, per):
            out[i:i + per] = attention(q2[i:i + per], k2[i:i + per], v2[i:i + per], rb)
        return out.reshape(lead + (nq, v.shape[-1]))
    s = np.matmul(q, np.swapaxes(k, -1, -2)) * np.float32(1.0 / math.sqrt(q.shape[-1]))
    if rb is None:
        return np.matmul(_softmax(s), v)
    e = rb(np.exp(s - s.max(-1, keepdims=True)))
    return np.matmul(e, v) / e.sum(-1, keepdims=True)


def _heads(x, h):
    *lead, n, d = x.shape
    return np.moveaxis(x.reshape(*lead, n, h, d // h), -2, -3)


def _unheads(x):
    x = np.moveaxis(x, -3, -2)
    *lead, n, h, dh = x.shape
    return x.reshape(*lead, n, h * dh)


def _gelu(x):
    return 0.5 * x * (1.0 + np.tanh(np.float32(math.sqrt(2.0 / math.pi)) * (x + np.float32(0.044715) * x * x * x)))


def time_embedding(t, d):
    half = d // 2
    f = 10.0 ** (-4.0 * np.arange(half) / (half - 1)) if half > 1 else np.ones(half)
    return np.concatenate([np.sin(t * f), np.cos(t * f)])


def site_output(cfg: Cfg, w: dict, li: int, kind: str, block: str, x, tvec, text, rb=None):
    """Post-projection, pre-residual output of one site (model.py:346-403).
    rb: bf16 rounding (emulation mode; weights in ``w`` are then already rounded)."""
    d = cfg.D
    r = _ident if rb is None else rb

    def modnorm(mod_w):
        mod = tvec @ mod_w
        return r(_ln(x) * (1.0 + mod[d:]) + mod[:d])

    if kind == "mlp":
        p = f"{li}.{'ms' if block == 's' else 'mt'}"
        h = modnorm(w[p + ".mod"])
        return r(r(_gelu(h @ w[p + ".w1"])) @ w[p + ".w2"])
    if kind == "cross":
        p = f"{li}.{'cs' if block == 's' else 'ct'}"
        b, t, s, _ = x.shape
        q = r(r(x) @ w[p + ".q"]).reshape(b, t * s, d)
        k, v = r(text @ w[p + ".k"]), r(text @ w[p + ".v"])
        o = r(_unheads(attention(_heads(q, cfg.H), _heads(k, cfg.H), _heads(v, cfg.H), rb)))
        return r(o.reshape(b, t, s, d) @ w[p + ".o"])
    p = f"{li}.{'sa' if kind == 'spatial' else 'ta'}"
    h = modnorm(w[p + ".mod"])
    q, k, v = (r(h @ w[p + "." + n]) for n in "qkv")
    if kind == "temporal":
        q, k, v = (a.transpose(0, 2, 1, 3) for a in (q, k, v))
    o = r(_unheads(attention(_heads(q, cfg.H), _heads(k, cfg.H), _heads(v, cfg.H), rb)))
    if kind == "temporal":
        o = o.transpose(0, 2, 1, 3)
    return r(o @ w[p + ".o"])


def _probs(q, k):
    s = np.matmul(q, np.swapaxes(k, -1, -2)) * np.float32(1.0 / math.sqrt(q.shape[-1]))
    return _softmax(s)


def site_scores(cfg: Cfg, w: dict, li: int, kind: str, block: str, x, tvec, text, probs=None):
    """Score broadcast (model.py:325-392): probs=None -> (o, P) computed with
    capture; probs given -> o replayed as P @ v of the current input."""
    d = cfg.D
    if kind == "cross":
        p = f"{li}.{'cs' if block == 's' else 'ct'}"
        b, t, s, _ = x.shape
        v = _heads(text @ w[p + ".v"], cfg.H)
        if probs is None:
            q = _heads((x @ w[p + ".q"]).reshape(b, t * s, d), cfg.H)
            probs = _probs(q, _heads(text @ w[p + ".k"], cfg.H))
            o = _unheads(np.matmul(probs, v)).reshape(b, t, s, d) @ w[p + ".o"]
            return o, probs
        return _unheads(np.matmul(probs, v)).reshape(b, t, s, d) @ w[p + ".o"]
    p = f"{li}.{'sa' if kind == 'spatial' else 'ta'}"
    mod = tvec @ w[p + ".mod"]
    h = _ln(x) * (1.0 + mod[d:]) + mod[:d]
    tr = (lambda a: a.transpose(0, 2, 1, 3)) if kind == "temporal" else (lambda a: a)
    v = _heads(tr(h @ w[p + ".v"]), cfg.H)
    ret = probs is None
    if ret:
        probs = _probs(_heads(tr(h @ w[p + ".q"]), cfg.H), _heads(tr(h @ w[p + ".k"]), cfg.H))
    o = tr(_unheads(np.matmul(probs, v))) @ w[p + ".o"]
    return (o, probs) if ret else o


KIND_ORDER = ("spatial", "temporal", "cross", "mlp")  # table axis order (model.py:56-64)


def layer_sites(cfg: Cfg):
    s = [("spatial", "s"), ("cross", "s"), ("mlp", "s"), ("temporal", "t")]
    if cfg.cross_t:
        s.append(("cross", "t"))
    s.append(("mlp", "t"))
    return s


def text_embedding(w, ids):
    ids = np.asarray(ids, dtype=np.int64)
    e = w["text"][np.where(ids < 0, 0, ids)].copy()
    e[ids < 0] = 0.0
    return e


def stores_of(table: np.ndarray) -> set:
    """(step, layer, kind) cells whose output a later step reuses (policies.py:202-214)."""
    n = table.shape[0]
    out = set()
    for i in range(n):
        for l in range(table.shape[1]):
            for k in range(4):
                s = int(table[i, l, k])
                if s != i:
                    out.add((s, l, k))
    return out


def forward(cfg, w, x, t, text, table, step, cache, log=None, delta_mode=False, scores=False, rb=None):
    """One step (model.py:425-568); cache maps site -> (source step, value).
    scores: broadcast_object="scores" (attention sites cache probabilities).
    rb: bf16 rounding function (emulation mode, see module docstring)."""
    tvec = time_embedding(t, cfg.D).astype(np.float32) @ w["time"]
    stores = stores_of(table) if not delta_mode else None
    for li in range(cfg.L):
        row = table[step, li]
        if delta_mode and np.all(row != step):
            src, val = cache[(li, None, "delta")]
            assert src == row[0]
            x = x + val
            continue
        x_in = x
        for kind, block in layer_sites(cfg):
            ki = KIND_ORDER.index(kind)
            src = int(row[ki])
            key = (li, kind, block)
            score_site = scores and kind != "mlp"
            if src == step:
                stored = not delta_mode and (step, li, ki) in stores
                if score_site and stored:
                    o, probs = site_scores(cfg, w, li, kind, block, x, tvec, text)
                    cache[key] = (step, probs)
                else:
                    o = site_output(cfg, w, li, kind, block, x, tvec, text, rb)
                    if stored:
                        cache[key] = (step, o)
                dec = "compute"
            else:
                cached_src, val = cache[key]
                assert cached_src == src, (key, cached_src, src)
                o = site_scores(cfg, w, li, kind, block, x, tvec, text, probs=val) if score_site else val
                dec = "reuse"
            if log is not None:
                log.append((step, li, kind, block, dec, src))
            x = x + o
        if delta_mode:
            later = [(i, l) for i in range(table.shape[0]) for l in [li] if int(table[i, li, 0]) == step and i != step]
            if later:
                cache[(li, None, "delta")] = (step, x - x_in)
    return x


def alpha_bar_fn():
    betas = np.linspace(1e-4, 2e-2, 1000, dtype=np.float64)
    ab = np.concatenate([[1.0], np.cumprod(1.0 - betas)])
    return lambda t: float(np.interp(t, np.arange(1001), ab))


def latent0(cfg: Cfg, seed: int, batch: int):
    z = Stream(seed).normal(cfg.T * cfg.S * cfg.D).reshape(1, cfg.T, cfg.S, cfg.D).astype(np.float32)
    return np.tile(z, (batch, 1, 1, 1))


def bf16_weights(w: dict) -> dict:
    """Matmul weights rounded to bf16 as the device holds them (modulation, time
    and text tables stay fp32 like the device's; the text embedding is rounded
    where it enters the K/V projection)."""
    return {k: (v if k in ("time", "text") or k.endswith(".mod") else bf16_round(v)) for k, v in w.items()}


def sample(cfg, w, timesteps, table, seed, text_ids=None, guidance=False, g=4.0, delta_mode=False,
           per_step=None, log=None, scores=False, emulate_bf16=False):
    """DDIM eta=0 sampler with optional CFG pair (diffusion.py:125-189).
    emulate_bf16: bf16 operand/output rounding (module docstring)."""
    ab = alpha_bar_fn()
    batch = 2 if guidance else 1
    ids = np.arange(cfg.M) % 256 if text_ids is None else np.asarray(text_ids)
    ids2 = np.stack([ids, np.full_like(ids, -1)]) if guidance else ids[None]
    text = text_embedding(w, ids2)
    rb = None
    if emulate_bf16:
        assert not scores, "bf16 emulation covers output broadcast"
        rb, w, text = bf16_round, bf16_weights(w), bf16_round(text)
    x = latent0(cfg, seed, batch)
    cache: dict = {}
    n = len(timesteps)
    for i, t in enumerate(timesteps):
        eps = forward(cfg, w, x, t, text, table, i, cache, log=log, delta_mode=delta_mode, scores=scores, rb=rb)
        if guidance:
            eps = eps[1:2] + np.float32(g) * (eps[0:1] - eps[1:2])
        a, an = ab(t), (ab(timesteps[i + 1]) if i + 1 < n else 1.0)
        x0 = (x - np.float32(math.sqrt(1.0 - a)) * eps) / np.float32(math.sqrt(a))
        x = np.float32(math.sqrt(an)) * x0 + np.float32(math.sqrt(1.0 - an)) * eps
        x = x.astype(np.float32)
        if per_step is not None:
            per_step.append(x.copy())
    return x


# --------------------------------------------------------- decisions
# reference policies.py:277-364 restated as explicit step walks
def table_pab(timesteps, layers, ranges, window, mlp=None, semantics="period", kinds=KIND_ORDER):
    ts = np.asarray(timesteps, dtype=np.float64)
    n = len(ts)
    src = np.repeat(np.arange(n, dtype=np.int32)[:, None], layers, 1)[:, :, None].repeat(4, 2)
    bump = 0 if semantics == "period" else 1
    hi, lo = window
    inside = [i for i in range(n) if lo <= ts[i] <= hi]
    for kind, r in zip(("spatial", "temporal", "cross"), ranges):
        if kind not in kinds or not inside:
            continue
        per = r + bump
        anchor = inside[0]
        for i in inside:
            if (i - inside[0]) % per == 0:
                anchor = i
            else:
                src[i, :, KIND_ORDER.index(kind)] = anchor
    if mlp is not None and "mlp" in kinds:
        triggers, blocks, r = mlp
        per = r + bump
        trig = set()
        for tau in triggers:
            d = np.abs(ts - tau)
            trig.add(int(np.flatnonzero(d == d.min())[0]))
        left, anchor = 0, None
        for i in range(n):
            if i in trig:
                anchor, left = i, per - 1
            elif left > 0:
                for bl in blocks:
                    src[i, bl, 3] = anchor
                left -= 1
    return src


def table_tgate(n, layers, gate, interval, warmup, kinds=KIND_ORDER):
    src = np.repeat(np.arange(n, dtype=np.int32)[:, None], layers, 1)[:, :, None].repeat(4, 2)
    last = 0
    for i in range(n):
        if i < gate:
            if i < warmup or (i - warmup) % interval == 0:
                last = i
            else:
                for kind in ("spatial", "temporal"):
                    if kind in kinds:
                        src[i, :, KIND_ORDER.index(kind)] = last
        elif "cross" in kinds:
            src[i, :, 2] = gate - 1
    return src


def table_deltadit(n, layers, gate, interval, block_range):
    src = np.repeat(np.arange(n, dtype=np.int32)[:, None], layers, 1)[:, :, None].repeat(4, 2)
    lo, hi = block_range
    last = {l: 0 for l in range(lo, hi + 1)}
    for i in range(n):
        for l in range(lo, hi + 1):
            if i < gate and i % interval != 0:
                src[i, l, :] = last[l]
            else:
                last[l] = i
    return src


def table_from_policy_dict(pd: dict, timesteps, layers, semantics="period"):
    v = pd["variant"]
    n = len(timesteps)
    if v == "none":
        return np.repeat(np.arange(n, dtype=np.int32)[:, None], layers, 1)[:, :, None].repeat(4, 2)
    if v == "pab":
        mlp = None
        if pd.get("mlp"):
            m = pd["mlp"]
            mlp = (m["triggers"], m["blocks"], m["range"])
        return table_pab(timesteps, layers, (pd["spatial_range"], pd["temporal_range"], pd["cross_range"]),
                         tuple(pd["window"]), mlp, semantics)
    if v == "tgate":
        return table_tgate(n, layers, pd["gate_step"], pd["interval"], pd["warmup"])
    if v == "deltadit":
        return table_deltadit(n, layers, pd["gate_step"], pd["interval"], tuple(pd["block_range"]))
    raise ValueError(v)


def linear_timesteps(n):
    return [1000.0 * (1.0 - i / n) for i in range(n)]

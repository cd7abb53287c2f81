"""Benchmark: seconds per video of the PAB denoising loop on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

A bench "step" is one whole video: the 30-step (config-dependent) PAB
denoising loop of BASELINE.json's headline config C3 (Open-Sora 1.2-shaped
STDiT, 2s 480p: L28 D1152 H16 dh72, T16 S1560 M300, cross attention in the
temporal block, CFG batch 2, preset opensora-pab246), random-init weights
and synthetic seeded inputs.  ``value`` = device time per video with the
latent resident in HBM; ``e2e`` = the same through the public serving call
(pinned host x_T -> H2D -> denoise -> D2H of the final latent).

Under torchrun (N > 1) the video is sharded with broadcast sequence
parallelism (frames across ranks, NCCL all-to-all around temporal attention,
skipped on temporal-broadcast steps): strong scaling of one video.

--impl reference times the reference's own CPU implementation (pab-engine,
installed unmodified into oracle/_ref by oracle/make_ref.sh; single-threaded
as the reference runs): C1 end to end, the B200 configs as one bounded
forward_step sample extrapolated to s/video by FLOP count (labelled
"extrapolated").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # SURVEY.md section 8 config key
    "C1": dict(layers=4, hidden=144, heads=2, frames=8, spatial_tokens=1024, text_tokens=16, cross=False, steps=10,
               preset="latte-pab235", batch=1),
    "C2": dict(layers=28, hidden=1152, heads=16, frames=16, spatial_tokens=1024, text_tokens=120, cross=False,
               steps=50, preset="latte-pab235", batch=2),
    "C3": dict(layers=28, hidden=1152, heads=16, frames=16, spatial_tokens=1560, text_tokens=300, cross=True,
               steps=30, preset="opensora-pab246", batch=2),
    "C4": dict(layers=28, hidden=1152, heads=16, frames=16, spatial_tokens=1024, text_tokens=300, cross=False,
               steps=150, preset="opensoraplan-pab246", batch=2),
    "C5": dict(layers=28, hidden=1152, heads=16, frames=32, spatial_tokens=3600, text_tokens=300, cross=True,
               steps=30, preset="opensora-pab246", batch=2),
    # functional multi-rank checks only (not a bench line): C1 shapes with CFG, cross in temporal
    "C1cfg": dict(layers=4, hidden=144, heads=2, frames=8, spatial_tokens=1024, text_tokens=16, cross=True,
                  steps=10, preset="opensora-pab246", batch=2),
}
METRIC = "s/video denoising latency (PAB, opensora-pab246)"  # the C3 headline; other configs name their preset


def metric_for(c):
    return f"s/video denoising latency (PAB, {c['preset']})"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def model_config(c):
    from paper_2408_12588_b200.model import ModelConfig

    return ModelConfig(layers=c["layers"], hidden=c["hidden"], heads=c["heads"], frames=c["frames"],
                       spatial_tokens=c["spatial_tokens"], text_tokens=c["text_tokens"],
                       cross_in_temporal=c["cross"])


def video_flops(cfg, table, batch, cross_live=None):
    """Algorithmic flops of one video under a decision table (2 flop/MAC, all
    GEMMs + attention contractions of computed sites; reference profiler
    flop model, profiler.py:176-226, without elementwise constants).
    cross_live: batch rows whose cross sites actually run (the engine skips the
    all-null-text CFG row, whose output is exactly 0); None = the reference model."""
    import numpy as np

    D, R, T, S, M, H = cfg.hidden, cfg.mlp_hidden, cfg.frames, cfg.spatial_tokens, cfg.text_tokens, cfg.heads
    rows = batch * T * S
    site = {
        "spatial": 2 * rows * D * 3 * D + 4 * batch * T * S * S * D + 2 * rows * D * D,
        "temporal": 2 * rows * D * 3 * D + 4 * batch * S * T * T * D + 2 * rows * D * D,
        "cross": (2 * rows * D * D + 4 * rows * M * D + 2 * rows * D * D)
                 * (1 if cross_live is None else cross_live) // (1 if cross_live is None else batch),
        "mlp": 2 * 2 * rows * D * R,
    }
    mult = {"spatial": 1, "temporal": 1, "cross": 1 + int(cfg.cross_in_temporal), "mlp": 2}
    comp = table.compute_mask()
    total = 0
    for k, name in enumerate(("spatial", "temporal", "cross", "mlp")):
        total += int(np.count_nonzero(comp[:, :, k])) * site[name] * mult[name]
    return total, site


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = f"/tmp/pab_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def _reference_modules():
    """The unmodified reference (pab-engine) installed into oracle/_ref by
    oracle/make_ref.sh (git-ignored, travels to the GPU box); None if absent."""
    path = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(path, "pab_engine")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/pab_numba_cache")
    if path not in sys.path:
        sys.path.insert(0, path)
    from pab_engine import diffusion as rd
    from pab_engine import model as rm
    from pab_engine import policies as rp

    return rm, rd, rp


def _video_flops_for(c):
    from paper_2408_12588_b200.diffusion import make_schedule
    from paper_2408_12588_b200.policies import build_schedule, resolve_preset

    cfg = model_config(c)
    pol, _ = resolve_preset(c["preset"], c["layers"])
    tab = build_schedule(pol, make_schedule(c["steps"]), c["layers"])
    return video_flops(cfg, tab, c["batch"])[0]


def cpu_baseline(c, end_to_end=None):
    """The reference's own CPU implementation timed on this host.

    Small configs (C1) run the reference ``sample()`` end to end (one whole PAB
    video, single-threaded like the reference).  For the B200-sized configs a
    video would take days on a CPU (SURVEY.md 7 hard part 6), so one bounded
    sample is timed -- the reference ``forward_step`` over one layer, one frame
    (all S tokens), batch 1, every site computed -- and extrapolated to s/video by
    the algorithmic FLOPs of the PAB video (labelled ``extrapolated``).  Falls back
    to the numpy oracle port when oracle/_ref is missing (kind "port")."""
    import numpy as np

    from paper_2408_12588_b200.diffusion import make_schedule
    from paper_2408_12588_b200.policies import NonePolicy, build_schedule

    if end_to_end is None:
        end_to_end = c["hidden"] * c["spatial_tokens"] * c["frames"] * c["layers"] <= 144 * 1024 * 8 * 4
    mods = _reference_modules()
    kind = "reference" if mods is not None else "port"
    if end_to_end and mods is not None:
        rm, rd, rp = mods
        cfg = rm.ModelConfig(layers=c["layers"], hidden=c["hidden"], heads=c["heads"], frames=c["frames"],
                             spatial_tokens=c["spatial_tokens"], text_tokens=c["text_tokens"],
                             cross_in_temporal=c["cross"])
        params = rm.init_model(cfg, seed=11)
        pol, _ = rp.resolve_preset(c["preset"], c["layers"])
        sched = rd.make_schedule(c["steps"])
        t0 = time.perf_counter()
        rd.sample(params, sched, pol, seed=11, guidance=c["batch"] == 2)
        dt = time.perf_counter() - t0
        return {"value": dt, "unit": "s/video", "cores": 1, "kind": kind, "extrapolated": False,
                "measured_sample_s": dt, "flop_scale": 1.0,
                "sample": f"reference pab_engine.sample() end to end: {c['preset']}, {c['steps']} steps, "
                          f"L{c['layers']} D{c['hidden']} T{c['frames']} S{c['spatial_tokens']} batch {c['batch']}, "
                          f"single-threaded (numba njit, as the reference runs)"}
    sc = dict(c, layers=1, frames=1, batch=1)
    if mods is not None:
        rm, rd, rp = mods
        cfg = rm.ModelConfig(layers=1, hidden=c["hidden"], heads=c["heads"], frames=1,
                             spatial_tokens=c["spatial_tokens"], text_tokens=c["text_tokens"],
                             cross_in_temporal=c["cross"])
        params = rm.init_model(cfg, seed=11)
        x = rd.initial_latent(params, 11, 1)
        ids = rd.default_text_ids(params)[None]
        table = rp.build_schedule(rp.NonePolicy(), rd.make_schedule(1), 1)
        t0 = time.perf_counter()
        rm.forward_step(params, x, 500.0, ids, table.slice(0), rp.CacheStore())
        dt = time.perf_counter() - t0
        cores, what = 1, "reference pab_engine.forward_step (single-threaded numba, as the reference runs)"
    else:
        from oracle import pab_oracle as orc

        ocfg = orc.Cfg(1, c["hidden"], c["heads"], 1, c["spatial_tokens"], c["text_tokens"],
                       cross_in_temporal=c["cross"])
        w = orc.init_weights(ocfg, seed=11)
        x = orc.latent0(ocfg, 11, 1)
        text = orc.text_embedding(w, (np.arange(c["text_tokens"]) % 256)[None])
        t0 = time.perf_counter()
        orc.forward(ocfg, w, x, 500.0, text, np.zeros((1, 1, 4), dtype=np.int32), 0, {})
        dt = time.perf_counter() - t0
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        what = "numpy oracle port (BLAS matmul, all host threads)"
    sample_table = build_schedule(NonePolicy(), make_schedule(1), 1)
    flops_sample = video_flops(model_config(sc), sample_table, 1)[0]
    scale = _video_flops_for(c) / flops_sample
    return {"value": dt * scale, "unit": "s/video", "cores": cores, "kind": kind, "extrapolated": True,
            "measured_sample_s": dt, "flop_scale": scale,
            "sample": f"{what} on 1 layer x 1 frame ({c['spatial_tokens']} tokens, D{c['hidden']}, M{c['text_tokens']}) "
                      f"x batch 1 x 1 step, all sites computed: {dt:.2f} s measured, extrapolated x{scale:.0f} by "
                      f"algorithmic FLOPs to the {c['preset']} video (L{c['layers']} T{c['frames']} {c['steps']} steps "
                      f"batch {c['batch']})"}


def run_reference(args, c):
    """--impl reference: the reference's CPU implementation on this host (rank 0 only).
    Each step is one bounded sample (cpu_baseline); warm-up is one sample (numba JIT)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(min(args.warmup, 1)):
        cpu_baseline(dict(c, hidden=64, heads=4, spatial_tokens=64, text_tokens=8, layers=1, frames=2, steps=2),
                     end_to_end=True)  # JIT compile of the reference's numba kernels
    runs = [cpu_baseline(c) for _ in range(args.steps)]
    v = statistics.median(r["value"] for r in runs)
    base = dict(runs[0], value=v, samples_s=[r["measured_sample_s"] for r in runs])
    line = {
        "metric": metric_for(c), "value": v, "unit": "s/video", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": min(args.warmup, 1), "ms_per_step": v * 1000.0, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded splitmix64 weights and x_T)",
        "config": {"workload": args.config, **{k: c[k] for k in ("layers", "hidden", "heads", "frames",
                                                                     "spatial_tokens", "text_tokens", "steps",
                                                                     "batch", "preset")}},
        "impl": "reference", "cpu_baseline": base, "extrapolated": base["extrapolated"],
        "e2e": {"value": v, "unit": "s/video", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-none", action="store_true", help="skip the no-PAB comparison run")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of replaying a CUDA graph")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"],
                    help="N>1: temporal-site reshards as NCCL all-to-alls, or fused into the prologues as "
                         "stores/loads over NVLink peer memory (peer.py)")
    ap.add_argument("--split-batch", action="store_true",
                    help="N>1: CFG halves on two rank groups of N/2 (reference run_parallel split_batch)")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, c)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2408_12588_b200 import kernels
    from paper_2408_12588_b200.diffusion import Denoiser, initial_latent, make_schedule
    from paper_2408_12588_b200.model import init_model
    from paper_2408_12588_b200.policies import NonePolicy, build_schedule, resolve_preset

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PAB_DIST_BACKEND", "nccl") != "nccl":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL over NVLink in production; PAB_DIST_BACKEND=gloo lets several ranks share one
        # GPU to exercise this multi-rank path where only one GPU is available
        backend = os.environ.get("PAB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = model_config(c)
    params = init_model(cfg, seed=11)
    sched = make_schedule(c["steps"])
    pol, _ = resolve_preset(c["preset"], cfg.layers)
    table = build_schedule(pol, sched, cfg.layers)
    ids = np.arange(cfg.text_tokens) % 256
    guidance = c["batch"] == 2

    split = bool(args.split_batch and world > 1 and world % 2 == 0 and guidance)

    def make_denoiser(tab):
        if split:
            from paper_2408_12588_b200.parallel import split_batch_denoiser

            return split_batch_denoiser(params, sched, tab, ids, guidance_scale=4.0, transport=args.transport)
        if world > 1:
            from paper_2408_12588_b200.parallel import ShardedDenoiser

            return ShardedDenoiser(params, sched, tab, ids, guidance=guidance, guidance_scale=4.0, rank=rank,
                                   world=world, transport=args.transport)
        return Denoiser(params, sched, tab, ids, guidance=guidance, guidance_scale=4.0)

    den = make_denoiser(table)
    x_host = torch.from_numpy(initial_latent(params, 11, c["batch"])).pin_memory()
    if split:
        x_dev = den.shard_input(x_host.cuda()[den.half:den.half + 1])
    else:
        x_dev = den.shard_input(x_host.cuda()) if world > 1 else x_host.cuda()
    z = torch.empty_like(x_dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # one CUDA graph per video; under torchrun with NCCL the all-to-alls are captured too
    # (a gloo group -- several ranks sharing one GPU in tests -- cannot be captured)
    backend = os.environ.get("PAB_DIST_BACKEND", "nccl")
    # (the peer transport has no collective inside the loop, so it captures under gloo too)
    use_graph = not args.no_graph and (world == 1 or backend == "nccl" or (args.transport == "peer" and not split))

    def denoise(d, zz):
        return d.run_graph(zz) if use_graph else d.run(zz)

    def one_video():
        z.copy_(x_dev)
        denoise(den, z)

    # per-kernel timings on the launching stream (CUDA events), on the engine's own
    # workspaces: once right after the first warm-up video (kernel timed alone at burst
    # clocks -> roofline vs the burst peak) and once after the timed videos (power-capped
    # step conditions -> "in_step", vs the sustained peak)
    peaks, peak_src = load_peaks()
    ctx = den.ctx

    def time_launch(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps / 1000.0

    B, T, S, D, M = ctx.B, ctx.T, ctx.S, ctx.D, ctx.M
    comp = table.compute_mask()  # (steps, layers, kind) spatial, temporal, cross, mlp
    site_counts = (int(comp[:, :, 0].sum()), int(comp[:, :, 1].sum()),
                   int(comp[:, :, 2].sum()) * (2 if cfg.cross_in_temporal else 1), int(comp[:, :, 3].sum()) * 2)
    flop_sp = 4.0 * B * T * S * S * D
    flop_tm = 4.0 * B * S * T * T * D
    Bc = getattr(ctx, "cross_live", B)  # cross sites skip null-text (unconditional CFG) rows: exactly 0
    flop_cr = 4.0 * Bc * T * S * M * D
    rows = ctx.rows
    bytes_mn = rows * D * (4 + 2 + 4 + 2)

    def kernel_times(peak_tf):
        xbuf = torch.zeros(rows, D, device="cuda")
        pend = [torch.zeros(rows, D, device="cuda", dtype=torch.bfloat16)]
        mod = torch.zeros(2 * D, device="cuda")
        t_sp = time_launch(lambda: kernels.attention(ctx.args_spatial))
        t_tm = time_launch(lambda: kernels.attention(ctx.args_temporal))
        t_cr = time_launch(lambda: kernels.attention(ctx.args_cross[0][0]))
        t_mn = time_launch(lambda: kernels.residual_modnorm(xbuf, xbuf, pend, h_out=ctx.h, mod=mod, mode=1))
        # projection GEMMs (csrc/gemm.cu) on the engine's workspaces with layer-0 weights
        lp = params.layers[0]
        rl = Bc * T * S
        g_ms = {
            "qkv": time_launch(lambda: kernels.gemm(ctx.h, lp.spatial.w_qkv_t, ctx.qkv)),
            "o_resid": time_launch(lambda: kernels.gemm_residual(ctx.attn_out, lp.spatial.wo_t, xbuf)),
            "cross_q": time_launch(lambda: kernels.gemm(ctx.h[:rl], lp.cross_spatial.wq_t, ctx.qbuf[:rl])),
            "cross_o_resid": time_launch(lambda: kernels.gemm_residual(ctx.attn_out[:rl], lp.cross_spatial.wo_t,
                                                                       xbuf[:rl])),
            "w1_gelu": time_launch(lambda: kernels.gemm(ctx.h, lp.mlp_spatial.w1_t, ctx.hidden, kernels.EPI_GELU)),
            "w2": time_launch(lambda: kernels.gemm(ctx.hidden, lp.mlp_spatial.w2_t, ctx.attn_out)),
        }
        del xbuf, pend
        R = cfg.mlp_hidden
        g_flops = {"qkv": 2.0 * rows * D * 3 * D, "o_resid": 2.0 * rows * D * D, "cross_q": 2.0 * rl * D * D,
                   "cross_o_resid": 2.0 * rl * D * D, "w1_gelu": 2.0 * rows * D * R, "w2": 2.0 * rows * R * D}
        # launches per video: spatial + temporal computes run qkv + o; cross computes q + o; mlp w1 + w2
        n_sp, n_tm, n_cr, n_ml = site_counts
        g_count = {"qkv": n_sp + n_tm, "o_resid": n_sp + n_tm, "cross_q": n_cr, "cross_o_resid": n_cr,
                   "w1_gelu": n_ml, "w2": n_ml}
        gemm = {k: {"ms": g_ms[k] * 1e3, "tflops": g_flops[k] / g_ms[k] / 1e12,
                    "frac_bf16_peak": g_flops[k] / g_ms[k] / 1e12 / peak_tf, "launches_per_video": g_count[k]}
                for k in g_ms}
        g_time = sum(g_ms[k] * g_count[k] for k in g_ms)
        g_fl = sum(g_flops[k] * g_count[k] for k in g_ms)
        gemm["all_projections"] = {"tflops": g_fl / g_time / 1e12, "frac_bf16_peak": g_fl / g_time / 1e12 / peak_tf,
                                   "s_per_video": g_time, "note": "time-weighted over the video's launches"}
        a_time = n_sp * t_sp + n_tm * t_tm + n_cr * t_cr
        a_fl = n_sp * flop_sp + n_tm * flop_tm + n_cr * flop_cr
        attn_agg = {"tflops": a_fl / a_time / 1e12, "frac_bf16_peak": a_fl / a_time / 1e12 / peak_tf,
                    "s_per_video": a_time, "note": "spatial + temporal + cross attention launches of one video, "
                    "algorithmic flops (cross: live CFG rows) / their measured time"}
        return t_sp, {
            "gemm": gemm,
            "attention_aggregate": attn_agg,
            "spatial_attn": {"ms": t_sp * 1e3, "tflops": flop_sp / t_sp / 1e12,
                             "frac_bf16_peak": flop_sp / t_sp / 1e12 / peak_tf},
            "temporal_attn": {"ms": t_tm * 1e3, "gbs": 8.0 * B * T * S * D / t_tm / 1e9,
                              "frac_hbm": 8.0 * B * T * S * D / t_tm / 1e9 / peaks["hbm_gbs"]},
            "cross_attn": {"ms": t_cr * 1e3, "tflops": flop_cr / t_cr / 1e12,
                           "frac_bf16_peak": flop_cr / t_cr / 1e12 / peak_tf,
                           "gbs": (4.0 * Bc * T * S * D + 4.0 * Bc * M * D) / t_cr / 1e9,
                           "batch_rows": Bc},
            "broadcast_epilogue_modnorm": {"ms": t_mn * 1e3, "gbs": bytes_mn / t_mn / 1e9,
                                           "frac_hbm": bytes_mn / t_mn / 1e9 / peaks["hbm_gbs"]},
        }

    one_video()
    graph_note = None
    if use_graph:
        try:
            den.capture_graph()  # the whole 30-step loop as one CUDA graph (static decision table)
        except Exception as e:  # keep the bench line: report eager launching and why
            use_graph, graph_note = False, f"graph capture failed, eager: {e!r}"[:200]
            torch.cuda.synchronize()
    barrier()
    time.sleep(3.0)  # let the board's power average settle (sw_power_cap window) -> burst clocks
    t_sp, kern = kernel_times(peaks["bf16_tflops"])
    for _ in range(args.warmup - 1):
        one_video()
    barrier()
    launches0 = den.ctx.launches.own_kernels()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            one_video()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = (den.graph_launches if use_graph else
                (den.ctx.launches.own_kernels() - launches0) // args.steps)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # e2e through the public serving call: pinned host x_T -> H2D -> denoise -> D2H latent
    out_host = torch.empty_like(x_host).pin_memory()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        den(x_host, out=out_host)
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    io_bytes = x_dev.numel() * x_dev.element_size()  # this rank's share of the latent, each way
    if getattr(den, "hook", None) is not None and den.hook.px is not None:
        den.hook.px.check()  # a timed-out peer barrier would make the timings meaningless

    # all-to-all traffic of one video: calls and bytes from the run's
    # ledger, the per-call time from the same exchange timed alone (CUDA events, max over ranks)
    a2a = None
    if world > 1 and getattr(den, "hook", None) is not None and den.hook.px is not None:
        hook = den.hook
        a2a = {"transport": "peer", "calls_per_video": 0,
               "barriers_per_video": den.ledger.event_count() // (2 if split else 1),
               "exchange_bytes_per_video_per_rank": hook.wire * den.ledger.event_count() // (2 if split else 1),
               "note": "no all-to-all: the temporal prologue stores h into the ranks' token buffers and the next "
                       "prologue reads o out of them over NVLink peer memory; one device barrier per exchange",
               "skipped_on_temporal_broadcast_steps": True,
               "ledger_elements_per_video": den.ledger.total_elements()}
    elif world > 1 and getattr(den, "hook", None) is not None:
        hook = den.hook
        calls = den.ledger.event_count() // (2 if split else 1)
        send_b = hook.h_send.numel() * hook.h_send.element_size()
        from paper_2408_12588_b200.parallel import exchange_frames_to_tokens

        exchange_frames_to_tokens(hook.h_send, hook.h_tok, hook.group)
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(20):
            exchange_frames_to_tokens(hook.h_send, hook.h_tok, hook.group)
        a1.record(stream)
        barrier()
        a_ms = a0.elapsed_time(a1) / 20
        t = torch.tensor([a_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        a_ms = float(t.item())
        a2a = {"transport": "nccl", "calls_per_video": calls, "bytes_per_call_per_rank": send_b,
               "wire_bytes_per_call_per_rank": hook.wire, "ms_per_call": a_ms,
               "est_ms_per_video": a_ms * calls, "skipped_on_temporal_broadcast_steps": True,
               "ledger_elements_per_video": den.ledger.total_elements()}

    # no-PAB reference point (same engine, every site computed)
    none_ms = None
    if not args.no_none:
        table_none = build_schedule(NonePolicy(), sched, cfg.layers)
        den_none = make_denoiser(table_none)
        z.copy_(x_dev)
        den_none.run(z)
        if use_graph:
            den_none.capture_graph()
        barrier()
        n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0.record(stream)
        reps = max(1, args.steps // 2)
        for _ in range(reps):
            z.copy_(x_dev)
            denoise(den_none, z)
        n1.record(stream)
        barrier()
        none_ms = n0.elapsed_time(n1) / reps
        if world > 1:
            t = torch.tensor([none_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            none_ms = float(t.item())
        del den_none

    t_sp_step, kern_step = kernel_times(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
    # roofline of the dominant kernel: the projection GEMM (gemm_kernel, ~65% of the video);
    # the MLP w2 launch is its largest single share (rows x 4D x D, 530 GFLOP at C3).  Timed
    # back to back right after the timed videos (power-capped clocks, as inside a video) and
    # set against the SUSTAINED bf16 peak; the burst timings (after a cool-down, short bursts
    # at up to 1965 MHz) are in "kernels" and can exceed the burst cuBLAS reference
    w2 = kern_step["gemm"]["w2"]
    achieved = w2["tflops"]
    peak_rf = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r02_gemm_w2_ncu.json")
    if os.path.exists(prof) and args.config == "C3":
        cap = json.load(open(prof))
        traffic = cap["dram_bytes_per_launch"]
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_rf, "unit": "TFLOP/s",
                "frac": achieved / peak_rf, "traffic": traffic,
                "traffic_note": "DRAM bytes per launch from profiles/r02_gemm_w2_ncu.json (ncu --set full); "
                                "algorithmic bytes: A 460 MB + W 10.6 MB read, C 115 MB written",
                "kernel": "gemm_kernel (MLP w2 projection, tcgen05 2-CTA)",
                "peak_source": f"{peak_src} bf16 sustained (MEASURED_PEAKS.json)",
                "algorithmic_flops_per_launch": 2.0 * ctx.rows * cfg.mlp_hidden * D,
                "all_projection_gemms_frac": kern_step["gemm"]["all_projections"]["frac_bf16_peak"],
                "attention_aggregate_frac": kern_step["attention_aggregate"]["frac_bf16_peak"],
                "spatial_attention_frac": kern_step["spatial_attn"]["frac_bf16_peak"],
                "spatial_attention_frac_burst": kern["spatial_attn"]["frac_bf16_peak"]}
    flops_pab, _ = video_flops(cfg, table, c["batch"])
    flops_exec, _ = video_flops(cfg, table, c["batch"], cross_live=1 if guidance else c["batch"])

    if rank == 0:
        # the CPU reference beside the GPU number: rank 0 at N=1 only (the scaling runs skip it)
        base = None if (args.no_cpu_baseline or world > 1) else cpu_baseline(c)
        line = {
            "metric": metric_for(c), "value": ms / 1000.0, "unit": "s/video", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded splitmix64 weights and x_T)",
            "config": {"workload": args.config, "layers": cfg.layers, "hidden": cfg.hidden, "heads": cfg.heads,
                       "frames": cfg.frames, "spatial_tokens": cfg.spatial_tokens, "text_tokens": cfg.text_tokens,
                       "denoise_steps": c["steps"], "batch": c["batch"], "preset": c["preset"],
                       "parallelism": (f"cfg2x_broadcast_sp{world // 2}" if split else
                                       f"broadcast_sp{world}" if world > 1 else "single"),
                       "transport": args.transport if world > 1 else None,
                       "l2": "inputs larger than L2 (fp32 latent 230 MB > 126 MB L2)",
                       "launch": ("one CUDA graph per video (static decision table)" if use_graph
                                  else graph_note or "eager"),
                       "none_s_per_video": None if none_ms is None else none_ms / 1000.0,
                       "pab_speedup_vs_none": None if none_ms is None else none_ms / ms,
                       "video_tflop_pab": flops_pab / 1e12, "achieved_tflops_video": flops_pab / (ms / 1e3) / 1e12,
                       "video_tflop_executed": flops_exec / 1e12,
                       "achieved_tflops_video_executed": flops_exec / (ms / 1e3) / 1e12,
                       "flop_note": "video_tflop_pab: reference FLOP model (includes the null-text CFG half of "
                                    "the cross sites); *_executed: without that half, which this engine skips "
                                    "because its output is exactly 0"},
            "e2e": {"value": e2e_ms / 1000.0, "unit": "s/video", "h2d_bytes_per_step": io_bytes,
                    "d2h_bytes_per_step": io_bytes},
            "gpu_launches": launches,
            "alltoall": a2a,
            "roofline": roofline,
            "kernels": kern,
            "kernels_in_step": dict(kern_step, note="same launches after the timed videos (power-capped "
                                    "clocks); fractions vs the sustained bf16 peak"),
            "clocks": clk.summary(),
            "cpu_baseline": base,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

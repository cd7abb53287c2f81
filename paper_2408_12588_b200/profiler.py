"""Redundancy analysis of site outputs across diffusion steps (reference
pkg/src/pab_engine/profiler.py:47-173) -- the measurement behind PAB's
broadcast ranges (paper Fig. 2/3: attention outputs change little between
neighbouring steps in the middle of the schedule).

Two ways to feed ``RedundancyReport``:

* ``redundancy_scan(trace)`` -- the reference algorithm over a host trace recorded
  with ``ComponentTrace(snapshot_mode="snapshot")`` (one device->host copy per
  site per step);
* ``DeviceRedundancyTrace`` / ``redundancy_scan_device`` -- the B200 form: each
  computed site's output is compared on the device with the same site's output
  of the previous step (``pab_diff_sums``: four fp64 sums per pair) and kept for
  the next step in a bf16 device slot; only 32 bytes per site and step ever come
  back to the host, once, at the end of the run.
"""

from __future__ import annotations

import csv
from collections import defaultdict
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .errors import MetricError, ShapeError, ValidationError
from .model import KINDS, ComponentKind, ComponentTrace

METRICS = ("mse", "relative_l2", "one_minus_cosine")


def _metric_from_sums(dd: float, aa: float, bb: float, ab: float, n: int, metric: str) -> float:
    """mse / relative_l2 / one_minus_cosine of (a, b) from sum (a-b)^2, a^2, b^2, a b
    (the reference's diff_metric, profiler.py:60-81, b being the reference operand)."""
    if metric not in METRICS:
        raise ValidationError(f"unknown metric {metric!r}, expected one of {METRICS}")
    if metric == "mse":
        return dd / n if n else float("nan")
    nb = float(np.sqrt(bb))
    if metric == "relative_l2":
        if nb == 0.0:
            raise MetricError("relative_l2 undefined for zero-norm reference")
        return float(np.sqrt(dd)) / nb
    na = float(np.sqrt(aa))
    if na == 0.0 or nb == 0.0:
        raise MetricError("cosine distance undefined for zero-norm operand")
    return 1.0 - ab / (na * nb)


def diff_metric(a, b, metric: str = "mse") -> float:
    """Difference between two host snapshots, in float64."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        raise ShapeError(f"snapshots differ in shape: {a.shape} vs {b.shape}")
    if metric not in METRICS:
        raise ValidationError(f"unknown metric {metric!r}, expected one of {METRICS}")
    av, bv = a.astype(np.float64).ravel(), b.astype(np.float64).ravel()
    d = av - bv
    if metric == "mse":
        return float(np.mean(d * d))
    return _metric_from_sums(float(d @ d), float(av @ av), float(bv @ bv), float(av @ bv), av.size, metric)


@dataclass
class RedundancyEntry:
    step: int
    timestep: float
    kind: ComponentKind
    layer: int
    block: str
    value: float


@dataclass
class RedundancyReport:
    """Per-site output differences between consecutive steps (reference profiler.py:93-137)."""

    metric: str
    num_steps: int
    layers: int
    entries: list

    def per_layer_rows(self) -> list:
        """(step, timestep, kind, layer, metric, value); the two MLP sites of a layer pooled."""
        groups: dict = defaultdict(list)
        for e in self.entries:
            groups[(e.step, e.kind, e.layer)].append(e)
        order = sorted(groups, key=lambda k: (k[0], KINDS.index(k[1]), k[2]))
        return [(step, groups[(step, kind, layer)][0].timestep, kind.value, layer, self.metric,
                 float(np.mean([e.value for e in groups[(step, kind, layer)]])))
                for step, kind, layer in order]

    def average_rows(self) -> list:
        """Across-layer means per (step, kind), plus separate spatial-/temporal-block MLP curves."""
        pooled: dict = defaultdict(list)
        ts: dict = {}
        for e in self.entries:
            ts[e.step] = e.timestep
            pooled[(e.step, e.kind.value)].append(e.value)
            if e.kind == ComponentKind.MLP:
                pooled[(e.step, "mlp_spatial" if e.block == "s" else "mlp_temporal")].append(e.value)
        return [(step, ts[step], label, "all", self.metric, float(np.mean(v)))
                for (step, label), v in sorted(pooled.items())]

    def write_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["step", "timestep", "kind", "layer", "metric", "value"])
            w.writerows(self.per_layer_rows() + self.average_rows())


def _check_scan_trace(trace) -> None:
    if trace.has_reuse():
        raise ValidationError("redundancy scan requires an all-Compute trace")
    if not trace.records:
        raise ValidationError("trace is empty")


def redundancy_scan(trace: ComponentTrace, metric: str = "mse") -> RedundancyReport:
    """Reference redundancy_scan (profiler.py:140-173) over host snapshots; a
    ``DeviceRedundancyTrace`` is scanned on the device instead."""
    if isinstance(trace, DeviceRedundancyTrace):
        return trace.report(metric)
    _check_scan_trace(trace)
    if any(r.snapshot is None for r in trace.records):
        raise ValidationError("redundancy scan requires snapshots (snapshot_mode='snapshot')")
    sites: dict = defaultdict(list)
    for r in trace.records:
        sites[(r.layer, r.kind, r.block)].append(r)
    entries = []
    for (layer, kind, block), recs in sites.items():
        recs.sort(key=lambda r: r.step)
        entries += [RedundancyEntry(cur.step, cur.timestep, kind, layer, block,
                                    diff_metric(cur.snapshot, prev.snapshot, metric))
                    for prev, cur in zip(recs, recs[1:])]
    layers = 1 + max(layer for layer, _, _ in sites)
    return RedundancyReport(metric=metric, num_steps=trace.num_steps(), layers=layers, entries=entries)


@dataclass
class DeviceRedundancyTrace(ComponentTrace):
    """Trace whose site outputs are diffed on the GPU as they are produced.

    observe(): for a site seen before, ``pab_diff_sums(o, prev)`` writes four fp64
    sums into this record's row of a device table; then o is copied into the site's
    bf16 slot (one slot per site: L x 6 x E bf16, 19 GB at C3, resident in HBM).
    ``report(metric)`` synchronises once and evaluates any of the three metrics."""

    snapshot_mode: str = "device"
    _prev: dict = field(default_factory=dict)
    _sums: list = field(default_factory=list)   # (site, step, timestep, n) per device row
    _table: list = field(default_factory=list)  # device fp64 chunks of 256 rows x 4

    def _row(self):
        import torch

        k = len(self._sums)
        if k % 256 == 0:
            self._table.append(torch.zeros((256, 4), dtype=torch.float64, device="cuda"))
        return self._table[-1][k % 256]

    def observe(self, record, output):
        from . import _lib, kernels

        if output is not None and record.decision == "compute":
            import torch

            site = (record.layer, record.kind, record.block)
            o = output.reshape(-1)
            prev = self._prev.get(site)
            if prev is not None:
                if prev.numel() != o.numel():
                    raise ShapeError(f"site {site} changed size between steps")
                row = self._row()
                lib = _lib.load()
                _lib.check(lib.pab_diff_sums(o.data_ptr(), prev.data_ptr(), o.numel(), row.data_ptr(),
                                             kernels._stream()), "pab_diff_sums")
                self._sums.append((site, record.step, record.timestep, o.numel()))
                prev.copy_(o)
            else:
                self._prev[site] = torch.empty_like(o).copy_(o)
        self.records.append(record)

    def report(self, metric: str = "mse") -> RedundancyReport:
        import torch

        _check_scan_trace(self)
        if metric not in METRICS:
            raise ValidationError(f"unknown metric {metric!r}, expected one of {METRICS}")
        torch.cuda.synchronize()
        host = torch.cat(self._table).cpu().numpy() if self._table else np.zeros((0, 4))
        entries = [RedundancyEntry(step, ts, kind, layer, block, _metric_from_sums(*host[i], n, metric))
                   for i, ((layer, kind, block), step, ts, n) in enumerate(self._sums)]
        layers = 1 + max(r.layer for r in self.records)
        return RedundancyReport(metric=metric, num_steps=self.num_steps(), layers=layers, entries=entries)


def redundancy_scan_device(params, schedule, seed: int, text_ids=None, *, guidance: bool = False,
                           guidance_scale: float = 4.0, metric: str = "mse",
                           trace: Optional[DeviceRedundancyTrace] = None) -> RedundancyReport:
    """All-compute sampling run on the B200 engine with the device scan attached
    (the reference's redundancy workflow: NonePolicy + snapshots + redundancy_scan)."""
    from .diffusion import sample
    from .policies import NonePolicy

    trace = trace if trace is not None else DeviceRedundancyTrace()
    sample(params, schedule, NonePolicy(), seed, text_ids, guidance=guidance, guidance_scale=guidance_scale,
           trace=trace)
    return trace.report(metric)


__all__ = ["METRICS", "diff_metric", "RedundancyEntry", "RedundancyReport", "redundancy_scan",
           "DeviceRedundancyTrace", "redundancy_scan_device"]

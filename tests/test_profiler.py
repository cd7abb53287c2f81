"""Redundancy analysis (reference profiler.py:47-173): host diff metrics, report
grouping, and the device scan (pab_diff_sums) against the reference's own
redundancy_scan output (tests/golden/redundancy.json, make_redundancy_golden.py)."""
import json
import os

import numpy as np
import pytest

from paper_2408_12588_b200.errors import MetricError, ShapeError, ValidationError
from paper_2408_12588_b200.model import ComponentKind, ComponentTrace, TraceRecord
from paper_2408_12588_b200.profiler import METRICS, diff_metric, redundancy_scan

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "redundancy.json")))


def test_diff_metric_definitions():
    rng = np.random.default_rng(0)
    a, b = rng.normal(size=(7, 9)), rng.normal(size=(7, 9))
    assert diff_metric(a, b, "mse") == pytest.approx(np.mean((a - b) ** 2), rel=1e-12)
    assert diff_metric(a, b, "relative_l2") == pytest.approx(np.linalg.norm(a - b) / np.linalg.norm(b), rel=1e-12)
    cos = np.sum(a * b) / (np.linalg.norm(a) * np.linalg.norm(b))
    assert diff_metric(a, b, "one_minus_cosine") == pytest.approx(1 - cos, rel=1e-10)
    with pytest.raises(ShapeError):
        diff_metric(a, b[:3])
    with pytest.raises(ValidationError):
        diff_metric(a, b, "l1")
    with pytest.raises(MetricError):
        diff_metric(a, np.zeros_like(b), "relative_l2")


def _trace(values, decision="compute"):
    tr = ComponentTrace(snapshot_mode="snapshot")
    for step, v in enumerate(values):
        for layer in range(2):
            for kind, block in ((ComponentKind.SPATIAL, "s"), (ComponentKind.MLP, "s"), (ComponentKind.MLP, "t")):
                r = TraceRecord(step=step, timestep=1000.0 - step, layer=layer, kind=kind, block=block,
                                decision=decision, source_step=step)
                r.snapshot = np.full(4, v * (layer + 1) * (2 if block == "t" else 1), dtype=np.float32)
                tr.records.append(r)
    return tr


def test_report_rows_pool_mlp_sites_and_average_layers():
    rep = redundancy_scan(_trace([1.0, 2.0, 4.0]), "mse")
    assert rep.num_steps == 3 and rep.layers == 2
    rows = rep.per_layer_rows()
    # step 1, mlp, layer 0: mean of block s (1 -> 2: mse 1) and t (2 -> 4: mse 4)
    assert (1, 999.0, "mlp", 0, "mse", 2.5) in rows
    avg = {(r[0], r[2]): r[5] for r in rep.average_rows()}
    assert avg[(1, "spatial")] == pytest.approx((1.0 + 4.0) / 2)
    assert avg[(1, "mlp_temporal")] == pytest.approx((4.0 + 16.0) / 2)


def test_scan_rejects_broadcast_traces_and_missing_snapshots():
    with pytest.raises(ValidationError, match="all-Compute"):
        redundancy_scan(_trace([1.0, 2.0], decision="reuse"))
    tr = _trace([1.0, 2.0])
    tr.records[0].snapshot = None
    with pytest.raises(ValidationError, match="snapshots"):
        redundancy_scan(tr)


@pytest.mark.gpu
def test_device_scan_matches_reference_scan():
    """Device scan (no snapshots leave the GPU) vs the reference's redundancy_scan on the
    same config and seeds: every per-layer and averaged row, all three metrics.  The
    device outputs are bf16 (the pipeline's rounding, ~4e-3 relative per element); a
    metric of a difference amplifies it by |o| / |o_t - o_t-1|, so rows are held to 10%
    each and 3% in aggregate; the host snapshot scan of the same device run agrees with
    the device scan to fp16-snapshot rounding."""
    from paper_2408_12588_b200.diffusion import make_schedule, sample
    from paper_2408_12588_b200.model import ModelConfig, init_model
    from paper_2408_12588_b200.policies import NonePolicy
    from paper_2408_12588_b200.profiler import DeviceRedundancyTrace

    params = init_model(ModelConfig(**GOLD["config"]), seed=GOLD["model_seed"])
    sched = make_schedule(GOLD["steps"])
    dev = DeviceRedundancyTrace()
    sample(params, sched, NonePolicy(), GOLD["seed"], guidance=True, trace=dev)
    host = ComponentTrace(snapshot_mode="snapshot")
    sample(params, sched, NonePolicy(), GOLD["seed"], guidance=True, trace=host)
    for metric in METRICS:
        rep = redundancy_scan(dev, metric)
        want = GOLD["metrics"][metric]
        assert rep.num_steps == want["num_steps"] and rep.layers == want["layers"]
        for got_rows, want_rows in ((rep.per_layer_rows(), want["per_layer"]), (rep.average_rows(), want["average"])):
            assert [tuple(r[:5]) for r in got_rows] == [tuple(r[:5]) for r in want_rows]
            g = np.array([r[5] for r in got_rows])
            w = np.array([r[5] for r in want_rows])
            assert np.all(np.abs(g - w) <= 0.1 * np.abs(w) + 1e-6), metric
            assert np.linalg.norm(g - w) / np.linalg.norm(w) < 3e-2, metric
        h = np.array([r[5] for r in redundancy_scan(host, metric).per_layer_rows()])
        g = np.array([r[5] for r in rep.per_layer_rows()])
        assert np.allclose(h, g, rtol=2e-2, atol=1e-6), metric

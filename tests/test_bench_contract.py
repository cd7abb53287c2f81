"""bench.py JSON-line contract (the driver parses it): the reference arm on CPU,
our arm on the GPU, both on the small C1 config so they run in seconds."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e")


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0"], timeout=600)
    for k in BASE_KEYS:
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is False and d["value"] > 0
    base = d["cpu_baseline"]
    assert base["kind"] in ("reference", "port") and base["cores"] >= 1
    # the reference (oracle/_ref, installed by oracle/make_ref.sh) runs C1 end to end
    assert base["extrapolated"] is (base["kind"] == "port") and d["extrapolated"] is base["extrapolated"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--config", "C1", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-none"], timeout=900)
    for k in BASE_KEYS + ("gpu_launches", "roofline", "clocks", "kernels"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["warmup"] >= 3 and d["gpu_launches"] > 0
    assert d["config"]["workload"] == "C1" and "l2" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert 0 < r["frac"] < 1.5 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])

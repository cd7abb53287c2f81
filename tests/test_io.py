"""PABT dumps / run directories (reference pkg/tests/test_cli.py:55-125 for the
format; golden files written by the reference io module,
tests/golden/make_pabt_golden.py)."""

import json
import os

import numpy as np
import pytest
import torch

from paper_2408_12588_b200 import io
from paper_2408_12588_b200.errors import ArtifactError

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _g(name):
    return os.path.join(GOLDEN, name)


def test_reads_reference_dumps():
    a = io.read_tensor(_g("ref_f32.pabt"))
    assert a.dtype == np.float32 and a.shape == (2, 3, 4)
    assert np.array_equal(a, (np.arange(24, dtype=np.float32).reshape(2, 3, 4) * 0.37 - 1.0).astype(np.float32))
    b = io.read_tensor(_g("ref_f64.pabt"))
    assert np.array_equal(b, np.linspace(-2.0, 3.0, 10).reshape(5, 2).astype(np.float32))
    assert io.read_tensor(_g("ref_scalar.pabt")).shape == (1,)  # ascontiguousarray makes 0-d 1-d


@pytest.mark.parametrize("name,make", [
    ("ref_f32.pabt", lambda: (np.arange(24, dtype=np.float32).reshape(2, 3, 4) * 0.37 - 1.0).astype(np.float32)),
    ("ref_f64.pabt", lambda: np.linspace(-2.0, 3.0, 10).reshape(5, 2)),
    ("ref_scalar.pabt", lambda: np.float32(2.5).reshape(())),
])
def test_writes_reference_bytes(tmp_path, name, make):
    out = tmp_path / name
    io.write_tensor(out, make())
    assert out.read_bytes() == open(_g(name), "rb").read()


def test_torch_tensor_and_bf16(tmp_path):
    t = torch.tensor([[1.5, -2.25], [0.125, 3.0]], dtype=torch.bfloat16)
    io.write_tensor(tmp_path / "t.pabt", t)
    assert np.array_equal(io.read_tensor(tmp_path / "t.pabt"), t.float().numpy())


def test_errors(tmp_path):
    with pytest.raises(ArtifactError) as e:
        io.read_tensor(tmp_path / "absent.pabt")
    assert e.value.kind == "missing-artifact"
    bad = tmp_path / "bad.pabt"
    bad.write_bytes(b"NOPE0000000000")
    with pytest.raises(ArtifactError) as e:
        io.read_tensor(bad)
    assert e.value.kind == "malformed-artifact"
    io.write_tensor(tmp_path / "ok.pabt", np.ones((2, 2), np.float32))
    data = (tmp_path / "ok.pabt").read_bytes()
    (tmp_path / "trunc.pabt").write_bytes(data[:-4])
    with pytest.raises(ArtifactError):
        io.read_tensor(tmp_path / "trunc.pabt")


def test_json_and_run_dir(tmp_path):
    io.write_json(tmp_path / "m.json", {"b": [1, 2], "a": {"z": 1.5, "y": "x"}})
    assert (tmp_path / "m.json").read_text() == open(_g("ref_manifest.json")).read()

    class R:
        latent = np.full((1, 2, 3, 4), 0.5, np.float32)
        manifest = {"policy": "none", "steps": 3}

    d = io.write_run(tmp_path / "run", R())
    assert np.array_equal(io.read_run_latent(d), R.latent)
    assert json.load(open(d / io.MANIFEST_FILENAME)) == R.manifest

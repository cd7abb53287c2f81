"""Write PABT dumps with the REFERENCE io module (pkg/src/pab_engine/io.py) as
golden fixtures for paper_2408_12588_b200.io (build container only; the
reference does not exist on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_pabt_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
from pab_engine.io import write_json, write_tensor  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
a = (np.arange(24, dtype=np.float32).reshape(2, 3, 4) * 0.37 - 1.0).astype(np.float32)
write_tensor(os.path.join(OUT, "ref_f32.pabt"), a)
write_tensor(os.path.join(OUT, "ref_f64.pabt"), np.linspace(-2.0, 3.0, 10).reshape(5, 2))  # cast on write
write_tensor(os.path.join(OUT, "ref_scalar.pabt"), np.float32(2.5).reshape(()))
write_json(os.path.join(OUT, "ref_manifest.json"), {"b": [1, 2], "a": {"z": 1.5, "y": "x"}})
print("ok")

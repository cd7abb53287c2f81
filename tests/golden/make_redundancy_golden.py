"""Generate tests/golden/redundancy.json by running the REFERENCE redundancy workflow
(all-compute sample with snapshot_mode="snapshot", then profiler.redundancy_scan,
/root/reference/pkg/src/pab_engine/profiler.py:140-173) on a small CFG config, for
every metric: per_layer_rows + average_rows.

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_redundancy_golden.py
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from pab_engine import diffusion as rd  # noqa: E402
from pab_engine import model as rm  # noqa: E402
from pab_engine import policies as rp  # noqa: E402
from pab_engine import profiler as rpf  # noqa: E402

CFG = dict(layers=2, hidden=144, heads=2, frames=8, spatial_tokens=64, text_tokens=12, cross_in_temporal=True)
STEPS, SEED, MODEL_SEED = 6, 7, 3


def main():
    params = rm.init_model(rm.ModelConfig(**CFG), seed=MODEL_SEED)
    trace = rm.ComponentTrace(snapshot_mode="snapshot")
    rd.sample(params, rd.make_schedule(STEPS), rp.NonePolicy(), seed=SEED, guidance=True, trace=trace)
    out = {"config": CFG, "steps": STEPS, "seed": SEED, "model_seed": MODEL_SEED, "guidance": True, "metrics": {}}
    for metric in rpf.METRICS:
        rep = rpf.redundancy_scan(trace, metric)
        out["metrics"][metric] = {"per_layer": [list(r) for r in rep.per_layer_rows()],
                                  "average": [list(r) for r in rep.average_rows()],
                                  "num_steps": rep.num_steps, "layers": rep.layers}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "redundancy.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()

"""Generate tests/golden/configs.json by running the REFERENCE run-config parser
(pab_engine.config, /root/reference/pkg/src/pab_engine/config.py:124-248) on a set of
JSON configs: for each, either the parsed config (to_dict, defaults_filled,
preset_notes) or the ValidationError message; plus apply_overrides cases.

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_config_golden.py
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from pab_engine import config as rc  # noqa: E402
from pab_engine.errors import EngineError  # noqa: E402

CASES = [
    {},
    {"preset": "opensora-pab246", "model": {"layers": 28, "hidden": 1152, "heads": 16, "frames": 16,
                                            "spatial_tokens": 1560, "text_tokens": 300, "cross_in_temporal": True},
     "schedule": {"steps": 30}, "guidance": True},
    {"policy": {"preset": "latte-pab235"}, "model": {"layers": 4, "hidden": 144, "heads": 2,
                                                     "spatial_tokens": 1024}, "schedule": {"steps": 10}},
    {"policy": {"variant": "pab", "spatial_range": 3, "window": [900, 100],
                "mlp": {"triggers": [700, 500], "blocks": [0, 2], "range": 3}}, "preset": "custom"},
    {"policy": {"variant": "pab"}},
    {"policy": {"variant": "tgate", "gate_step": 5}},
    {"policy": {"variant": "deltadit", "block_range": [1, 3]}},
    {"policy": {"variant": "none"}, "parallel": {"workers": 2, "method": "broadcast_sp"}},
    {"policy": {"variant": "pab"}, "parallel": {"workers": 4, "method": "broadcast_sp", "split_batch": True},
     "guidance": True, "text": list(range(16))},
    {"policy": {"variant": "pab"}, "parallel": {"workers": 3}},
    {"policy": {"variant": "bogus"}},
    {"policy": {"spatial_range": 2}},
    {"model": {"layers": 2, "depth": 3}},
    {"extra": 1},
    {"precision": "f16"},
    {"broadcast_object": "logits"},
    {"range_semantics": "sometimes"},
    {"schedule": {"steps": 0}},
    {"parallel": {"method": "ring"}},
    {"parallel": {"workers": 0}},
    {"text": [1, 2, 3]},
    {"preset": "opensora-pab246", "model": {"layers": 2}},
    {"range_semantics": "reuse-count", "broadcast_object": "scores", "seed": 5, "output_dir": "/tmp/x",
     "precision": "f64", "guidance_scale": 7.5},
]
OVERRIDES = [
    ({"model": {"layers": 6}}, {"preset": "latte-pab235", "seed": 3}),
    ({}, {"workers": 2, "method": "broadcast_sp"}),
    ({}, {"precision": "f64", "range_semantics": "reuse-count"}),
    ({}, {}),
    ({}, {"precision": "bad"}),
]


def outcome(fn):
    try:
        c = fn()
        return {"ok": c.to_dict(), "defaults_filled": list(c.defaults_filled), "preset_notes": list(c.preset_notes)}
    except EngineError as e:
        return {"error": str(e), "kind": e.kind}


def main():
    out = {"cases": [{"input": c, **outcome(lambda c=c: rc.config_from_dict(c))} for c in CASES],
           "overrides": [{"input": c, "overrides": o,
                          **outcome(lambda c=c, o=o: rc.apply_overrides(rc.config_from_dict(c), **o))}
                         for c, o in OVERRIDES]}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path, len(out["cases"]), "cases")


if __name__ == "__main__":
    main()

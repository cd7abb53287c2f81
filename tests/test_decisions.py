"""Decision tables: bit-exact against the reference (golden fixtures) and the
reference's own known-answer tests (pkg/tests/test_policies.py,
pkg/tests/test_acceptance.py:89-131).  CPU only."""

import json
import os
import random

import numpy as np
import pytest

from oracle import pab_oracle as orc
from paper_2408_12588_b200.errors import PolicyError, ValidationError
from paper_2408_12588_b200.model import KIND_INDEX, KINDS, ComponentKind, ModelConfig
from paper_2408_12588_b200.policies import (
    PRESET_NAMES,
    CacheStore,
    DecisionTable,
    DeltaDitPolicy,
    MlpBroadcast,
    NonePolicy,
    PabPolicy,
    TGatePolicy,
    build_schedule,
    disable_kind,
    memory_footprint,
    resolve_preset,
    validate_policy,
)

SP, TM, CR, ML = ComponentKind.SPATIAL, ComponentKind.TEMPORAL, ComponentKind.CROSS, ComponentKind.MLP


def lin(n):
    return [1000.0 * (1.0 - i / n) for i in range(n)]


def policy_from_dict(d):
    v = d["variant"]
    if v == "none":
        return NonePolicy()
    if v == "pab":
        mlp = None
        if d.get("mlp"):
            m = d["mlp"]
            mlp = MlpBroadcast(tuple(m["triggers"]), tuple(m["blocks"]), m["range"])
        return PabPolicy(d["spatial_range"], d["temporal_range"], d["cross_range"], tuple(d["window"]), mlp)
    if v == "tgate":
        return TGatePolicy(d["gate_step"], d["interval"], d["warmup"])
    return DeltaDitPolicy(d["gate_step"], d["interval"], tuple(d["block_range"]))


@pytest.fixture(scope="module")
def golden(golden_dir):
    tables = np.load(os.path.join(golden_dir, "decisions.npz"))
    meta = json.load(open(os.path.join(golden_dir, "decisions.json")))
    return tables, meta


STEPS = {"desk": 30, "small": 6, "C1": 10, "C2": 50, "C3": 30, "C4": 150, "C5": 30}


class TestGoldenTables:
    def test_presets_bit_exact(self, golden):
        tables, meta = golden
        checked = 0
        for entry in meta["presets"]:
            layers = {"desk": 4, "small": 2, "C1": 4}.get(entry["config"], 28)
            pol, _ = resolve_preset(entry["preset"], layers)
            if "error" in entry:
                with pytest.raises(ValidationError):
                    build_schedule(pol, lin(STEPS[entry["config"]]), layers, range_semantics=entry["semantics"])
                continue
            t = build_schedule(pol, lin(entry["steps"]), entry["layers"], range_semantics=entry["semantics"])
            assert np.array_equal(t.source, tables[entry["key"]]), entry["key"]
            assert t.delta_mode == entry["delta"]
            checked += 1
        assert checked > 100

    def test_random_policies_bit_exact(self, golden):
        tables, meta = golden
        for entry in meta["random"]:
            pol = policy_from_dict(entry["policy"])
            t = build_schedule(pol, lin(entry["n"]), entry["layers"], range_semantics=entry["semantics"])
            assert np.array_equal(t.source, tables[entry["key"]]), entry
            t.validate()

    def test_oracle_tables_bit_exact(self, golden):
        tables, meta = golden
        for entry in meta["random"] + [e for e in meta["presets"] if "key" in e]:
            n = entry.get("n", entry.get("steps"))
            src = orc.table_from_policy_dict(entry["policy"], lin(n), entry["layers"], entry["semantics"])
            assert np.array_equal(src, tables[entry["key"]]), entry["key"]

    def test_c3_layer0_rows(self, golden):
        # SURVEY.md section 8 golden rows (opensora-pab246, N=30)
        tables, _ = golden
        src = tables["C3|opensora-pab246|period"]
        rows = {
            "spatial": "CCCCrCrCrCrCrCrCrCCCCCCCCCCCCC",
            "temporal": "CCCCrrrCrrrCrrrCrCCCCCCCCCCCCC",
            "cross": "CCCCrrrrrCrrrrrCrCCCCCCCCCCCCC",
            "mlp": "CCCCCrCrCCCrCCCCCCCCCCCCCCCCCC",
        }
        pol, _ = resolve_preset("opensora-pab246", 28)
        t = build_schedule(pol, lin(30), 28)
        for kind, want in rows.items():
            k = KIND_INDEX[ComponentKind(kind)]
            got = "".join("C" if t.source[i, 0, k] == i else "r" for i in range(30))
            assert got == want
            assert np.array_equal(t.source[:, 0, k], src[:, 0, k])


class TestReferenceKnownAnswers:
    def test_range_one_is_all_compute(self):
        t = build_schedule(PabPolicy(1, 1, 1, window=(930.0, 450.0)), lin(30), layers=2)
        assert t.equals(DecisionTable.all_compute(30, 2))

    def test_pab246_hand_enumeration(self):
        t = build_schedule(PabPolicy(2, 4, 6, window=(930.0, 450.0)), lin(30), layers=3)
        assert t.compute_steps(SP) == [0, 1, 2] + [3, 5, 7, 9, 11, 13, 15] + list(range(17, 30))
        assert t.compute_steps(TM) == [0, 1, 2] + [3, 7, 11, 15] + list(range(17, 30))
        assert t.compute_steps(CR) == [0, 1, 2] + [3, 9, 15] + list(range(17, 30))
        assert t.source_of(16, 0, TM) == 15 and t.source_of(14, 2, CR) == 9

    def test_reuse_count_semantics(self):
        p = PabPolicy(2, 2, 2, window=(1000.0, 1.0))
        assert build_schedule(p, lin(12), 1).compute_steps(SP) == [0, 2, 4, 6, 8, 10]
        assert build_schedule(p, lin(12), 1, range_semantics="reuse-count").compute_steps(SP) == [0, 3, 6, 9]

    def test_mlp_nearest_trigger(self):
        p = PabPolicy(1, 1, 1, window=(930.0, 450.0), mlp=MlpBroadcast((864.0, 799.0), (0,), 3))
        t = build_schedule(p, lin(30), layers=2)
        col = [t.source_of(i, 0, ML) for i in range(30)]
        assert col[4] == 4 and col[5] == 4 and col[6] == 6 and col[7] == 6 and col[8] == 6 and col[9] == 9
        assert all(t.is_compute(i, 1, ML) for i in range(30))

    def test_empty_window(self):
        t = build_schedule(PabPolicy(3, 3, 3, window=(450.0, 430.0)), [1000.0, 900.0, 800.0], layers=1)
        assert t.equals(DecisionTable.all_compute(3, 1))

    def test_tgate(self):
        t = build_schedule(TGatePolicy(12, 2, 2), lin(30), layers=2)
        assert [i for i in range(30) if not t.is_compute(i, 0, CR)] == list(range(12, 30))
        assert [i for i in range(30) if not t.is_compute(i, 0, SP)] == [3, 5, 7, 9, 11]

    def test_deltadit(self):
        t = build_schedule(DeltaDitPolicy(5, 2, (0, 1)), lin(8), layers=3)
        assert t.delta_mode
        for l in (0, 1):
            assert t.compute_steps(SP, l) == [0, 2, 4, 5, 6, 7]
        assert t.compute_steps(SP, 2) == list(range(8))
        t.source[1, 0, 0] = 1
        with pytest.raises(ValidationError):
            t.validate()

    def test_walker_equivalence_100(self):
        # reference tests/test_policies.py:108-120 with the reference walker restated in the oracle
        rng = random.Random(20240811)
        for _ in range(100):
            n, layers = rng.randint(1, 60), rng.randint(1, 6)
            sem = rng.choice(["period", "reuse-count"])
            kind = rng.choice(["pab", "tgate"])
            if kind == "pab":
                lo = rng.uniform(0, 900)
                pol = PabPolicy(rng.randint(1, 9), rng.randint(1, 9), rng.randint(1, 9), (rng.uniform(lo + 1, 1000), lo))
                src = orc.table_pab(lin(n), layers, (pol.spatial_range, pol.temporal_range, pol.cross_range),
                                    pol.window, None, sem)
            else:
                pol = TGatePolicy(rng.randint(1, n), rng.randint(1, 5), rng.randint(0, 4))
                src = orc.table_tgate(n, layers, pol.gate_step, pol.interval, pol.warmup)
            assert np.array_equal(build_schedule(pol, lin(n), layers, range_semantics=sem).source, src)

    def test_disable_kind(self):
        pol, _ = resolve_preset("opensora-pab246", layers=4)
        full = build_schedule(pol, lin(30), 4)
        for kind in KINDS:
            part = build_schedule(pol, lin(30), 4, kinds=disable_kind(pol, kind))
            ki = KIND_INDEX[kind]
            assert np.all(part.source[:, :, ki] == np.arange(30)[:, None])
            others = [KIND_INDEX[k] for k in KINDS if k != kind]
            assert np.array_equal(part.source[:, :, others], full.source[:, :, others])
        assert build_schedule(pol, lin(30), 4, kinds=()).equals(build_schedule(NonePolicy(), lin(30), 4))

    def test_validation(self):
        with pytest.raises(ValidationError):
            build_schedule(PabPolicy(window=(1200.0, 450.0)), lin(10), 1)
        with pytest.raises(ValidationError):
            build_schedule(TGatePolicy(gate_step=11), lin(10), 1)
        with pytest.raises(ValidationError):
            validate_policy(PabPolicy(mlp=MlpBroadcast((), (0,), 2)), 10, 4)
        with pytest.raises(ValidationError):
            validate_policy(DeltaDitPolicy(block_range=(0, 4)), 30, 4)
        with pytest.raises(ValidationError):
            validate_policy(PabPolicy(spatial_range=0), 30, 4)
        with pytest.raises(ValidationError):
            build_schedule(NonePolicy(), lin(4), 1, range_semantics="nope")

    def test_presets(self):
        pol, notes = resolve_preset("opensora-pab246", layers=4)
        assert (pol.spatial_range, pol.temporal_range, pol.cross_range) == (2, 4, 6)
        assert pol.window == (930.0, 450.0) and pol.mlp.blocks == (0, 1, 2, 3)
        assert any("filtered" in n for n in notes)
        with pytest.raises(ValidationError) as ei:
            resolve_preset("nope", layers=4)
        assert ei.value.kind == "unknown-preset"
        deep, n2 = resolve_preset("deltadit-default", layers=8)
        assert deep.block_range == (0, 5) and not n2
        for name in PRESET_NAMES:
            p, _ = resolve_preset(name, layers=4)
            build_schedule(p, lin(30), 4).validate()

    def test_17_of_30(self):
        # reference tests/test_acceptance.py:171-191 (temporal compute count)
        pol, _ = resolve_preset("opensora-pab246", layers=4)
        t = build_schedule(pol, lin(30), 4)
        assert len(t.compute_steps(TM)) == 20
        assert len(t.compute_steps(SP)) == 23 and len(t.compute_steps(CR)) == 19


class TestCacheAndMemory:
    def test_cache_protocol(self):
        c = CacheStore()
        with pytest.raises(PolicyError):
            c.fetch((0, SP, "s"))
        c.store((0, SP, "s"), np.zeros(2), step=1)
        c.store((0, SP, "s"), np.ones(2), step=5)
        e = c.fetch((0, SP, "s"))
        assert e.source_step == 5 and np.array_equal(e.value, np.ones(2))
        with pytest.raises(PolicyError):
            c.fetch((0, SP, "s"), expect="scores")

    def test_memory_footprint(self):
        cfg = ModelConfig(layers=2, hidden=16, heads=2, frames=4, spatial_tokens=8, text_tokens=4)
        assert memory_footprint(DecisionTable.all_compute(10, 2), cfg) == 0
        t = build_schedule(PabPolicy(1, 2, 1, window=(1000.0, 1.0)), lin(4), 2)
        assert memory_footprint(t, cfg) == 2 * 4 * 8 * 16 * 4
        full = build_schedule(PabPolicy(2, 4, 6, window=(930.0, 450.0)), lin(30), 2)
        cross = build_schedule(PabPolicy(1, 1, 6, window=(930.0, 450.0)), lin(30), 2)
        assert memory_footprint(full, cfg) > memory_footprint(cross, cfg)

    def test_should_store_is_lazy(self):
        t = build_schedule(PabPolicy(2, 4, 6, window=(930.0, 450.0)), lin(30), 2)
        s = t.slice(3)
        assert s.should_store(0, SP) and s.should_store(0, TM) and s.should_store(0, CR)
        assert not t.slice(0).should_store(0, SP)
        assert not t.slice(4).should_store(0, SP)  # step 4 reuses spatial

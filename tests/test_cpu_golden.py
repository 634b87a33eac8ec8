"""CPU parity against golden vectors produced by the real reference
(tests/golden/make_golden.py): host knob transforms, host kernel formation,
and the oracle restatements the GPU tests use as their checker."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import costmodel_ref as CM
from oracle import interp_ref as IR
from paper_2107_09789_b200 import fixtures, kernels, knobs
from paper_2107_09789_b200.ir import label_sequence

GOLD = Path(__file__).resolve().parent / "golden"
G = json.loads((GOLD / "golden.json").read_text())


def _plan(pj):
    return knobs.ObfuscationPlan(pj["mode"], tuple(knobs.PlanEntry(**e) for e in pj["entries"]))


def _digest(g):
    nodes = []
    for nid in sorted(g.nodes):
        n = g.nodes[nid]
        w = None
        if n.weights is not None:
            a = np.ascontiguousarray(n.weights, dtype=np.float32)
            w = [list(a.shape), hashlib.sha256(a.tobytes()).hexdigest()]
        nodes.append([nid, n.kind.value, dict(sorted(n.attrs.items())), list(n.inputs), w])
    return {"output_id": g.output_id, "nodes": nodes}


def _cases():
    for case in G["cases"]:
        g = fixtures.FIXTURES[case["fixture"]](**case["kwargs"])
        yield case, g


@pytest.mark.parametrize("case", [c["name"] for c in G["cases"]])
def test_apply_plan_matches_reference(case):
    c = next(x for x in G["cases"] if x["name"] == case)
    g = fixtures.FIXTURES[c["fixture"]](**c["kwargs"])
    assert [k.value for k in label_sequence(g)] == c["labels"]
    for rec in c["plans"]:
        if "error" in rec:
            with pytest.raises(knobs.PlanApplicationError) as ei:
                knobs.apply_plan(g, _plan(rec["plan"]))
            assert str(ei.value) == rec["error"]
            continue
        og, d = knobs.apply_plan(g, _plan(rec["plan"]))
        assert json.loads(json.dumps(_digest(og))) == rec["graph"]
        assert {str(k): v for k, v in d.fusion_limits.items()} == rec["fusion_limits"]
        assert {str(k): v for k, v in d.schedule_strategies.items()} == rec["strategies"]
        # host kernel formation (fusion.py:45-80)
        assert [list(k.node_ids) for k in kernels.fuse(og, d.fusion_limits)] == rec["kernels"]


@pytest.mark.parametrize("case", [c["name"] for c in G["cases"] if c["fixture"] != "vgg16"])
def test_costmodel_oracle_bit_exact_vs_reference(case):
    c = next(x for x in G["cases"] if x["name"] == case)
    g = fixtures.FIXTURES[c["fixture"]](**c["kwargs"])
    memo = CM.ScheduleMemo()
    _, _, _, t_star = CM.profile_pipeline(g, "default", None, None, memo)
    assert t_star == float.fromhex(c["t_star"])
    for rec in c["plans"]:
        if "error" in rec:
            continue
        og, d = knobs.apply_plan(g, _plan(rec["plan"]))
        kern, sch, rows, T = CM.profile_pipeline(og, "default", d.fusion_limits, d.schedule_strategies, memo)
        assert [list(k) for k in kern] == rec["kernels"]
        assert [[list(a), list(b), 4] for a, b in sch] == rec["schedules"]
        got = [[r[f].hex() for f in CM.FEATURES] for r in rows]
        assert got == rec["trace"]
        assert T.hex() == rec["T"]


def test_costmodel_oracle_vgg16_t_star():
    c = next(x for x in G["cases"] if x["name"] == "vgg16_dim")
    g = fixtures.vgg16()
    _, _, _, t_star = CM.profile_pipeline(g, "default", None, None, CM.ScheduleMemo())
    assert t_star == float.fromhex(c["t_star"])


@pytest.mark.parametrize("case", [c["name"] for c in G["cases"] if any("equiv" in p for p in c["plans"])])
def test_interp_oracle_verdicts_vs_reference(case):
    c = next(x for x in G["cases"] if x["name"] == case)
    g = fixtures.FIXTURES[c["fixture"]](**c["kwargs"])
    for rec in c["plans"]:
        if "equiv" not in rec:
            continue
        og, _ = knobs.apply_plan(g, _plan(rec["plan"]))
        ok, worst = IR.equivalence_check(g, og, trials=rec["equiv"]["trials"], seed=0)
        assert ok == rec["equiv"]["ok"]
        assert abs(worst - float.fromhex(rec["equiv"]["worst"])) < 1e-5


def test_interp_oracle_execute_vs_reference():
    arr = np.load(GOLD / "golden_exec.npz")
    e = G["exec"]
    g = fixtures.c1c2(size=e["size"])
    og, _ = knobs.apply_plan(g, _plan(e["plan"]))
    x = arr["x"]
    for graph, key in ((g, "vanilla"), (og, "obfuscated")):
        out = IR.execute(graph, x)
        ref = arr[key]
        assert np.max(np.abs(out - ref) / (1 + np.abs(ref))) < 1e-5
    bad = knobs.deepen_layer(g, 0, kernel_init=lambda ch: np.full((1, 1, ch, ch), 1.0 / ch, np.float32))
    ok, worst = IR.equivalence_check(g, bad, trials=2, seed=0)
    assert ok == e["broken_deepen"]["ok"] is False
    assert abs(worst - float.fromhex(e["broken_deepen"]["worst"])) < 1e-4 * max(1.0, worst)


def test_resnet18_fixture_t_star_matches_survey():
    """RN18 vanilla T* = 1,846,199.54 cycles (default profile)."""
    _, _, _, t = CM.profile_pipeline(fixtures.resnet18(), "default", None, None, CM.ScheduleMemo())
    assert t == 1846199.5435783395

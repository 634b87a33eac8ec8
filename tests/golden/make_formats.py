"""Golden files for the on-disk formats, written by the REAL reference package
(run in the build container, where /root/reference exists).

    python tests/golden/make_formats.py

Writes tests/golden/formats/: a small residual network and two obfuscated
versions of it (a dimension plan: widen / kernel-widen / dummy adds; a
sequence plan: branch / deepen / skip) dumped with the reference's
``dump_graph`` (graph.py:362-388), their plans with ``dump_plan``
(transforms.py:485-489), case-A and case-C (labelled) traces with
``dump_trace`` (costmodel.py:300-309), and ``expect.json`` with the
reference's in-memory digests of what ``load_*`` must return.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2107_09789_b200.fixtures import _Builder  # noqa: E402  (graph construction only)
from paper_2107_09789_b200.ir import TensorShape  # noqa: E402
from tests.refbridge import ref, to_ref  # noqa: E402

OUT = Path(__file__).resolve().parent / "formats"


def tiny():
    b = _Builder(TensorShape(1, 3, 8, 8), seed=7)
    x = b.relu(b.bn(b.conv([], 3, 8, 3, 1, 1), 8))
    y = b.bn(b.conv([x], 8, 8, 3, 1, 1), 8)
    x = b.relu(b.add([y, x]))
    x = b.relu(b.bn(b.conv([x], 8, 16, 3, 2, 1), 16))
    x = b.pool(x, 2, 2)
    return b.graph(b.softmax(b.linear(x, 16 * 2 * 2, 10)))


def digest(g) -> dict:
    nodes = []
    for nid in sorted(g.nodes):
        n = g.nodes[nid]
        w = None
        if n.weights is not None:
            a = np.ascontiguousarray(n.weights, dtype=np.float32)
            w = [list(a.shape), hashlib.sha256(a.tobytes()).hexdigest()]
        nodes.append([nid, n.kind.value, dict(sorted(n.attrs.items())), list(n.inputs), w])
    return {"output_id": g.output_id, "input_shape": list(g.input_shape.as_tuple()), "nodes": nodes}


def trace_json(t) -> dict:
    return {"case": t.case.value,
            "steps": [[float(getattr(s, f)).hex() for f in t.case.features] + [s.label.value if s.label else None]
                      for s in t.steps]}


def main() -> None:
    R = ref()
    OUT.mkdir(exist_ok=True)
    g = to_ref(tiny())
    convs = [nid for nid in R.topo_order(g) if g.nodes[nid].kind in (R.OperatorKind.Conv2D,)]
    layers = [nid for nid in R.topo_order(g) if g.nodes[nid].kind in R.COMPLEX_KINDS]
    dim = R.ObfuscationPlan("dimension", tuple(
        R.PlanEntry(layer_id=e.layer_id, kernel_widen=1, dummy_count=2, schedule_strategy=1)
        if e.layer_id == convs[0] else
        R.PlanEntry(layer_id=e.layer_id, widen_factor=1.5, kernel_widen=2, dummy_count=1, schedule_strategy=3)
        if e.layer_id == convs[2] else e for e in R.identity_plan(g, "dimension").entries))
    seq = R.ObfuscationPlan("sequence", tuple(
        R.PlanEntry(layer_id=e.layer_id, branching="out2", deepen=1, fusion_limit=1)
        if e.layer_id == convs[0] else
        R.PlanEntry(layer_id=e.layer_id, branching="in2", skip=1, fusion_limit=0)
        if e.layer_id == convs[1] else
        R.PlanEntry(layer_id=e.layer_id, fusion_limit=2)
        if e.layer_id == layers[-2] else e for e in R.identity_plan(g, "sequence").entries))
    expect = {}
    graphs = {"tiny": (g, None)}
    for name, plan in (("dim", dim), ("seq", seq)):
        obf, directives = R.apply_plan(g, plan)
        graphs[name] = (obf, directives)
        R.dump_plan(plan, OUT / f"{name}.plan")
        expect[f"{name}.plan"] = {"mode": plan.mode, "entries": [dict(e.__dict__) for e in plan.entries]}
    for name, (gr, directives) in graphs.items():
        R.dump_graph(gr, OUT / f"{name}.graph")
        expect[f"{name}.graph"] = digest(gr)
        lim = directives.fusion_limits if directives else None
        strat = directives.schedule_strategies if directives else None
        for case, labels in ((R.LeakageCase.A, False), (R.LeakageCase.C, True)):
            t = R.profile_pipeline(gr, case, R.BUILTIN_PROFILES["default"], lim, strat)
            fn = f"{name}_{case.value}.trace"
            R.dump_trace(t, OUT / fn, include_labels=labels)
            expect[fn] = trace_json(t)
    (OUT / "expect.json").write_text(json.dumps(expect, indent=0, sort_keys=True) + "\n")
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()

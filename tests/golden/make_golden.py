"""Generate golden vectors from the REAL reference package (run in the build
container, where /root/reference exists; the GPU box never needs it).

    python tests/golden/make_golden.py

Writes tests/golden/golden.json (+ golden_exec.npz): for fixed obfuscation
plans on the fixture graphs, the reference's own
  * apply_plan result (per-node digest incl. sha256 of every weight array,
    and the backend directives)             transforms.py:400-474
  * profile_pipeline trace: kernels, schedules, 9 features (float.hex), T,
    with the process-global schedule cache cleared before each case and the
    plans compiled in order                 costmodel.py:248-293
  * equivalence_check verdict + worst       interpreter.py:93-118
  * execute() outputs on a small graph      interpreter.py:75-90
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2107_09789_b200 import fixtures, ga  # noqa: E402  (plan generation + fixture graphs only)
from tests.refbridge import plan_ref, ref, to_ref  # noqa: E402

OUT = Path(__file__).resolve().parent
FEATURES = ("cycles", "dram_read", "dram_write", "l1_tx", "l1_util", "l1_hit", "l2_tx", "l2_util", "l2_hit")

# (case name, fixture, fixture kwargs, mode, number of plans, seed, equivalence trials or 0)
CASES = [
    ("c1c2_dim", "c1c2", {}, "dimension", 8, 101, 0),
    ("c1c2s_dim", "c1c2", {"size": 24}, "dimension", 4, 102, 3),
    ("rn18_seq", "resnet18", {}, "sequence", 6, 103, 0),
    ("rn18_dim", "resnet18", {}, "dimension", 3, 104, 0),
    ("rn18s_seq", "resnet18", {"size": 64}, "sequence", 3, 105, 2),
    ("vgg16_dim", "vgg16", {}, "dimension", 2, 106, 0),
    ("vgg16_seq", "vgg16", {}, "sequence", 2, 107, 0),
]


def plan_json(p):
    return {"mode": p.mode, "entries": [dict(e.__dict__) for e in p.entries]}


def digest(g) -> dict:
    nodes = []
    for nid in sorted(g.nodes):
        n = g.nodes[nid]
        w = None
        if n.weights is not None:
            a = np.ascontiguousarray(n.weights, dtype=np.float32)
            w = [list(a.shape), hashlib.sha256(a.tobytes()).hexdigest()]
        nodes.append([nid, n.kind.value, dict(sorted(n.attrs.items())), list(n.inputs), w])
    return {"output_id": g.output_id, "nodes": nodes}


def main() -> None:
    R = ref()
    golden = {"features": FEATURES, "cases": []}
    exec_arrays = {}
    for name, fx, kw, mode, n, seed, trials in CASES:
        g = fixtures.FIXTURES[fx](**kw)
        gr = to_ref(g)
        space = ga.search_space(g, mode)
        sizes = ga.domain_sizes(mode, space)
        rng = np.random.default_rng(seed)
        plans = [ga.decode_genome(g, mode, space, rng.integers(0, sizes)) for _ in range(n)]
        R.costmodel._SCHEDULE_CACHE.clear()
        vt = R.profile_pipeline(gr, R.LeakageCase.C, R.BUILTIN_PROFILES["default"])
        case = {"name": name, "fixture": fx, "kwargs": kw, "mode": mode, "t_star": vt.total_latency.hex(),
                "labels": [k.value for k in R.label_sequence(gr)], "plans": []}
        for p in plans:
            rec = {"plan": plan_json(p)}
            try:
                og, d = R.apply_plan(gr, plan_ref(p))
            except R.transforms.TransformError as exc:
                rec["error"] = str(exc)
                case["plans"].append(rec)
                continue
            rec["graph"] = digest(og)
            rec["fusion_limits"] = {str(k): v for k, v in d.fusion_limits.items()}
            rec["strategies"] = {str(k): v for k, v in d.schedule_strategies.items()}
            cg = R.compile_graph(og, R.BUILTIN_PROFILES["default"], d.fusion_limits, d.schedule_strategies)
            tr = R.profile_graph(cg.graph, cg.kernels, cg.schedules, R.LeakageCase.C, R.BUILTIN_PROFILES["default"])
            rec["kernels"] = [list(k.node_ids) for k in cg.kernels]
            rec["schedules"] = [[list(s.tile_y), list(s.tile_x), s.unroll] for s in cg.schedules]
            rec["trace"] = [[getattr(s, f).hex() for f in FEATURES] for s in tr.steps]
            rec["T"] = tr.total_latency.hex()
            if trials:
                ok, worst = R.equivalence_check(gr, og, trials=trials, seed=0)
                rec["equiv"] = {"trials": trials, "ok": bool(ok), "worst": float(worst).hex()}
            case["plans"].append(rec)
        golden["cases"].append(case)
        print(name, len(plans), "plans", flush=True)

    # execute() outputs on a small obfuscated graph + the broken-deepen verdict
    g = fixtures.c1c2(size=16)
    gr = to_ref(g)
    space = ga.search_space(g, "dimension")
    p = ga.decode_genome(g, "dimension", space, np.random.default_rng(7).integers(0, ga.domain_sizes("dimension", space)))
    og, _ = R.apply_plan(gr, plan_ref(p))
    x = np.random.default_rng(8).standard_normal((1, 3, 16, 16)).astype(np.float32)
    exec_arrays["x"] = x
    exec_arrays["vanilla"] = R.execute(gr, x)
    exec_arrays["obfuscated"] = R.execute(og, x)
    bad = R.deepen_layer(gr, 0, kernel_init=lambda ch: np.full((1, 1, ch, ch), 1.0 / ch, np.float32))
    ok_bad, worst_bad = R.equivalence_check(gr, bad, trials=2, seed=0)
    golden["exec"] = {"plan": plan_json(p), "size": 16, "broken_deepen": {"ok": bool(ok_bad),
                                                                          "worst": float(worst_bad).hex()}}
    (OUT / "golden.json").write_text(json.dumps(golden, separators=(",", ":")))
    np.savez_compressed(OUT / "golden_exec.npz", **exec_arrays)
    print("wrote", OUT / "golden.json")


if __name__ == "__main__":
    main()

"""On-disk formats (formats.py) against files the reference
itself wrote (tests/golden/make_formats.py): loading gives the reference's
in-memory objects, dumping gives the reference's bytes, and the engine's own
apply_plan / profile_pipeline dump to the same files as the reference's."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2107_09789_b200 as tobf
from paper_2107_09789_b200 import knobs
from paper_2107_09789_b200.ir import analyze

GOLD = Path(__file__).parent / "golden" / "formats"
EXPECT = json.loads((GOLD / "expect.json").read_text())


def _digest(g) -> dict:
    nodes = []
    for nid in sorted(g.nodes):
        n = g.nodes[nid]
        w = None
        if n.weights is not None:
            a = np.ascontiguousarray(np.asarray(n.weights), dtype=np.float32)
            w = [list(a.shape), hashlib.sha256(a.tobytes()).hexdigest()]
        nodes.append([nid, n.kind.value, dict(sorted(n.attrs.items())), list(n.inputs), w])
    return {"output_id": g.output_id, "input_shape": list(g.input_shape.as_tuple()), "nodes": nodes}


def _same_files(tmp: Path, name: str, suffixes=(".graph", ".weights")):
    for suf in suffixes:
        assert (tmp / f"{name}{suf}").read_bytes() == (GOLD / f"{name}{suf}").read_bytes(), f"{name}{suf}"


@pytest.mark.parametrize("name", ["tiny", "dim", "seq"])
def test_graph_round_trip(name, tmp_path):
    g = tobf.load_graph(GOLD / f"{name}.graph")
    assert json.loads(json.dumps(_digest(g))) == EXPECT[f"{name}.graph"]
    assert not tobf.validate(g)
    tobf.dump_graph(g, tmp_path / f"{name}.graph")
    _same_files(tmp_path, name)


@pytest.mark.parametrize("name", ["dim", "seq"])
def test_plan_round_trip(name, tmp_path):
    p = tobf.load_plan(GOLD / f"{name}.plan")
    assert {"mode": p.mode, "entries": [dict(e.__dict__) for e in p.entries]} == EXPECT[f"{name}.plan"]
    tobf.dump_plan(p, tmp_path / f"{name}.plan")
    assert (tmp_path / f"{name}.plan").read_bytes() == (GOLD / f"{name}.plan").read_bytes()


@pytest.mark.parametrize("name", ["dim", "seq"])
@pytest.mark.parametrize("lazy", [False, True])
def test_apply_plan_dumps_reference_bytes(name, lazy, tmp_path):
    """Engine apply_plan (eager, and the lazy derived-weight path the
    evaluator uses) on the same vanilla graph and plan file writes the
    reference's graph and weight files."""
    g = tobf.load_graph(GOLD / "tiny.graph")
    plan = tobf.load_plan(GOLD / f"{name}.plan")
    if lazy:
        obf, _, _ = knobs.apply_plan_analyzed(g, plan, analyze(g), lazy=True)
    else:
        obf, _ = tobf.apply_plan(g, plan)
    tobf.dump_graph(obf, tmp_path / f"{name}.graph")
    _same_files(tmp_path, name)


def _directives(name):
    if name == "tiny":
        return None, None
    _, d = tobf.apply_plan(tobf.load_graph(GOLD / "tiny.graph"), tobf.load_plan(GOLD / f"{name}.plan"))
    return d.fusion_limits, d.schedule_strategies


def oracle_trace(g, case, lim, strat):
    """Trace object from the CPU cost-model oracle (test checker only)."""
    from oracle import costmodel_ref
    kernels, _, rows, _ = costmodel_ref.profile_pipeline(g, "default", lim, strat)
    steps = []
    for kern, row in zip(kernels, rows):
        kind = g.nodes[kern[0]].kind
        steps.append(tobf.TraceStep(label=kind if kind in tobf.COMPLEX_KINDS else None, anchor_id=kern[0],
                                    **{f: row[f] for f in tobf.FEATURE_NAMES}))
    return tobf.Trace(tuple(steps), case)


def check_trace_files(name, tmp_path, make_trace):
    g = tobf.load_graph(GOLD / f"{name}.graph")
    lim, strat = _directives(name)
    for case, labels in ((tobf.LeakageCase.A, False), (tobf.LeakageCase.C, True)):
        fn = f"{name}_{case.value}.trace"
        tobf.dump_trace(make_trace(g, case, lim, strat), tmp_path / fn, include_labels=labels)
        assert (tmp_path / fn).read_bytes() == (GOLD / fn).read_bytes(), fn


@pytest.mark.parametrize("name", ["tiny", "dim", "seq"])
def test_trace_files(name, tmp_path):
    """dump_trace of the cost model's rows writes the reference's file;
    load_trace reads back the reference's values (case-masked)."""
    check_trace_files(name, tmp_path, oracle_trace)
    for case, labels in ((tobf.LeakageCase.A, False), (tobf.LeakageCase.C, True)):
        fn = f"{name}_{case.value}.trace"
        back = tobf.load_trace(GOLD / fn)
        assert back.case == case
        got = [[float(getattr(s, f)).hex() for f in case.features] + [s.label.value if s.label else None]
               for s in back.steps]
        assert got == [w[:-1] + ([w[-1]] if labels else [None]) for w in EXPECT[fn]["steps"]]


def test_graph_parse_errors(tmp_path):
    bad = tmp_path / "bad.graph"
    bad.write_text("graph v2\n")
    with pytest.raises(tobf.GraphParseError) as e:
        tobf.load_graph(bad)
    assert e.value.lineno == 1
    src = (GOLD / "tiny.graph").read_text().splitlines()
    bad.write_text("\n".join(src[:5] + ["bogus 1 2"] + src[5:]) + "\n")
    with pytest.raises(tobf.GraphParseError) as e:
        tobf.load_graph(bad)
    assert e.value.lineno == 6
    bad.write_text("\n".join(src) + "\n")
    (tmp_path / "tiny.weights").write_bytes(b"XXXXXXXX")
    with pytest.raises(tobf.GraphParseError, match="magic"):
        tobf.load_graph(bad)
    bad.write_text("graph v1\noutput 3\n")
    with pytest.raises(tobf.GraphParseError, match="missing input_shape"):
        tobf.load_graph(bad)


def test_round_trips_random_instances(tmp_path):
    """SPEC acceptance 9: graph / plan serialization round-trips byte-identically
    over 100 random instances (random valid plans over both modes on two
    small graphs), and the reloaded graph equals the dumped one node for node."""
    from paper_2107_09789_b200 import fixtures, ga
    bases = [fixtures.c1c2(size=8), tobf.load_graph(GOLD / "tiny.graph")]
    rng = np.random.default_rng(11)
    done = 0
    while done < 100:
        g = bases[done % len(bases)]
        mode = ("sequence", "dimension")[int(rng.integers(2))]
        space = ga.search_space(g, mode)
        plan = ga.decode_genome(g, mode, space, ga.random_genomes(rng, ga.domain_sizes(mode, space), 1)[0])
        try:
            obf, _ = tobf.apply_plan(g, plan)
        except tobf.TransformError:
            continue
        (tmp_path / "a").mkdir(exist_ok=True)
        (tmp_path / "b").mkdir(exist_ok=True)
        a, b = tmp_path / "a" / "g.graph", tmp_path / "b" / "g.graph"
        tobf.dump_graph(obf, a)
        back = tobf.load_graph(a)
        assert back.nodes.keys() == obf.nodes.keys()
        assert all(back.nodes[k] == obf.nodes[k] for k in obf.nodes)
        tobf.dump_graph(back, b)
        assert a.read_bytes() == b.read_bytes() and a.with_suffix(".weights").read_bytes() == \
            b.with_suffix(".weights").read_bytes()
        tobf.dump_plan(plan, tmp_path / "a.plan")
        assert tobf.load_plan(tmp_path / "a.plan") == plan
        done += 1


def test_trace_round_trip_random(tmp_path):
    """dump -> load -> dump of random case-masked traces is byte-identical
    (repr floats round-trip exactly); masked features come back as 0."""
    rng = np.random.default_rng(3)
    kinds = [None] + list(tobf.COMPLEX_KINDS)
    for i in range(100):
        case = list(tobf.LeakageCase)[i % 3]
        steps = tuple(tobf.TraceStep(**{f: float(rng.standard_normal() * 10.0 ** rng.integers(-3, 9))
                                        for f in tobf.FEATURE_NAMES},
                                     label=kinds[int(rng.integers(len(kinds)))])
                      for _ in range(int(rng.integers(0, 12))))
        t = tobf.Trace(steps, case)
        labels = bool(i % 2)
        tobf.dump_trace(t, tmp_path / "a.trace", include_labels=labels)
        back = tobf.load_trace(tmp_path / "a.trace")
        tobf.dump_trace(back, tmp_path / "b.trace", include_labels=labels)
        assert (tmp_path / "a.trace").read_bytes() == (tmp_path / "b.trace").read_bytes()
        assert back.case == case and len(back.steps) == len(steps)
        for s, r in zip(steps, back.steps):
            for f in tobf.FEATURE_NAMES:
                assert getattr(r, f) == (getattr(s, f) if f in case.features else 0.0)
            assert r.label == (s.label if labels else None)


def _cli(*args, env=None):
    import os
    import subprocess
    import sys
    root = Path(__file__).resolve().parents[1]
    return subprocess.run([sys.executable, "-m", "paper_2107_09789_b200", *map(str, args)], cwd=root,
                          capture_output=True, text=True, timeout=300, env={**os.environ, **(env or {})})


def test_cli_exit_codes(tmp_path):
    """0 success, 1 usage, 2 data/model error; a corrupt graph
    reports its line number. Data errors surface before any
    device is touched, so this runs on CPU."""
    assert _cli("bogus").returncode == 1
    assert _cli("profile", "--graph", GOLD / "tiny.graph").returncode == 1  # --out missing
    bad = tmp_path / "bad.graph"
    bad.write_text("graph v1\ninput_shape 1 3 8 8\nnode x Conv2D\n")
    r = _cli("profile", "--graph", bad, "--out", tmp_path / "t.trace")
    assert r.returncode == 2 and "bad.graph:3:" in r.stderr
    r = _cli("evaluate", "--graph", tmp_path / "missing.graph")
    assert r.returncode == 2
    (tmp_path / "bad.plan").write_text("plan v2\n")
    r = _cli("evaluate", "--graph", GOLD / "tiny.graph", "--plan", tmp_path / "bad.plan")
    assert r.returncode == 2 and "plan v1" in r.stderr

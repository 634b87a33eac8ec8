"""The device cost model's traces dump to the reference's trace files
(tests/golden/formats, written by the reference's dump_trace)."""

import pytest

import paper_2107_09789_b200 as tobf
from tests.test_cpu_formats import check_trace_files


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tiny", "dim", "seq"])
def test_device_trace_files(name, tmp_path):
    prof = tobf.BUILTIN_PROFILES["default"]
    check_trace_files(name, tmp_path, lambda g, case, lim, strat: tobf.profile_pipeline(g, case, prof, lim, strat))


@pytest.mark.gpu
def test_cli_profile_evaluate_obfuscate(tmp_path):
    """profile writes the reference's trace file; evaluate reports three
    per-predictor LERs of an equivalent candidate; obfuscate writes a plan and
    an obfuscated graph that reload and agree with apply_plan."""
    import json

    from tests.test_cpu_formats import GOLD, _cli
    r = _cli("profile", "--graph", GOLD / "tiny.graph", "--plan", GOLD / "seq.plan", "--case", "C", "--labels",
             "--out", tmp_path / "seq_C.trace")
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "seq_C.trace").read_bytes() == (GOLD / "seq_C.trace").read_bytes()
    r = _cli("evaluate", "--graph", GOLD / "tiny.graph", "--plan", GOLD / "dim.plan", "--trials", "2")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    assert rep["feasible"] and rep["equivalent"] and len(rep["lers"]) == 3
    assert rep["mean_ler"] == pytest.approx(sum(rep["lers"]) / 3)
    out = tmp_path / "run"
    r = _cli("obfuscate", "--graph", GOLD / "tiny.graph", "--mode", "dimension", "--population", "4",
             "--generations", "2", "--trials", "2", "--out", out, env={"TOBF_HOST_WORKERS": "0"})
    assert r.returncode == 0, r.stderr
    plan = tobf.load_plan(out / "best.plan")
    obf = tobf.load_graph(out / "obfuscated.graph")
    want, _ = tobf.apply_plan(tobf.load_graph(GOLD / "tiny.graph"), plan)
    assert obf.nodes.keys() == want.nodes.keys() and all(obf.nodes[k] == want.nodes[k] for k in want.nodes)
    res = json.loads((out / "result.json").read_text())
    assert res["report"]["equivalent"] and res["best_reward"] == pytest.approx(res["report"]["reward"])

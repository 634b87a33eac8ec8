"""Dimension attacker on the device (csrc/forest.cu): predictions and DER are
bit-exact against the CPU oracle (which is pinned to scikit-learn), and a
dimension-mode population scored by bagged DER matches the oracle applied to
each candidate's own trace."""

import numpy as np
import pytest
import torch

from oracle import forest_ref
from paper_2107_09789_b200 import dimattack, fixtures, ga
from paper_2107_09789_b200.dimattack import DeviceForests, DimRegressor, Forest, forest_der
from paper_2107_09789_b200.engine import device
from tests.test_cpu_dimattack import _arrays, random_forest

pytestmark = pytest.mark.gpu


def test_forest_der_kernel_vs_oracle():
    ctx = device()
    regs = [DimRegressor(Forest.from_sklearn(random_forest(s)[0]), Forest.from_sklearn(random_forest(s + 5, 11)[0]))
            for s in (0, 1)]
    rng = np.random.default_rng(7)
    n_layers = 4
    counts = [4, 4, 3, 4, 4]  # candidate 2 does not line up
    offsets = np.concatenate([[0], np.cumsum([c + 3 for c in counts])])  # 3 non-conv steps each
    feats = rng.standard_normal((int(offsets[-1]), 9)) * 10.0 ** rng.integers(0, 6, 9)
    rows, off = [], [0]
    for i, c in enumerate(counts):
        rows += list(range(int(offsets[i]) + 1, int(offsets[i]) + 1 + c))
        off.append(len(rows))
    truth = np.array([[64, 128], [128, 128], [3, 64], [256, 512]], np.int32)
    up = ctx.upload_array
    pred, der = forest_der(DeviceForests(regs), up(feats), up(np.array(rows, np.int32)), up(np.array(off, np.int32)),
                           len(counts), up(truth))
    pred, der = pred.cpu().numpy(), der.cpu().numpy()
    for r, reg in enumerate(regs):
        for c in range(len(counts)):
            x = feats[rows[off[c]:off[c + 1]]]
            p, d = forest_ref.candidate_der(_arrays(reg.c), _arrays(reg.j), x, truth.tolist())
            assert der[r, c] == d, (r, c)
            if d >= 0:
                assert pred[r, c].tolist() == [list(t) for t in p]


def test_dimension_population_scored_by_der():
    from paper_2107_09789_b200 import attacker_train
    from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator
    from paper_2107_09789_b200.knobs import TransformError, apply_plan
    from paper_2107_09789_b200.trace import BUILTIN_PROFILES, FEATURE_NAMES, LeakageCase, profile_pipeline
    from paper_2107_09789_b200.ir import OperatorKind as K
    ds = attacker_train.build_dataset(40, attacker_train.ArchGenConfig(seed=3))
    regs, vals = dimattack.train_dim_regressors(ds, trees=(3, 5), seed=1)
    assert len(regs) == 2 and all(v >= 0 for v in vals)
    g = fixtures.c1c2(size=24)
    space = ga.search_space(g, "dimension")
    rng = np.random.default_rng(5)
    plans = [ga.decode_genome(g, "dimension", space, x) for x in ga.random_genomes(rng, ga.domain_sizes(
        "dimension", space), 6)]
    pe = PopulationEvaluator(g, Evaluator(dim_regressors=regs), budget=0.02, trials=2, memo={})
    res = pe.evaluate(plans)
    truth = dimattack.conv_truth(g).tolist()
    prof = BUILTIN_PROFILES["default"]
    checked = 0
    for plan, rep in zip(plans, res.reports):
        try:
            obf, d = apply_plan(g, plan)
        except TransformError:
            assert not rep.feasible
            continue
        t = profile_pipeline(obf, LeakageCase.C, prof, d.fusion_limits, d.schedule_strategies)
        x = np.array([[getattr(s, f) for f in FEATURE_NAMES] for s in t.steps if s.label is K.Conv2D])
        want = [forest_ref.candidate_der(_arrays(r.c), _arrays(r.j), x, truth)[1] for r in regs]
        assert rep.metrics == want
        assert rep.mean_metric == pytest.approx(np.mean(want), rel=1e-15)
        checked += 1
    assert checked >= 3
    # the pooled host path (worker processes) scores the same records
    rec = pe.evaluate_records(plans, workers=2, memo={})
    assert np.array_equal(rec["mean_ler"], res.records["mean_ler"])
    assert np.array_equal(rec["reward"], res.records["reward"])
    pe.close()


def test_cli_dimension_attacker(tmp_path):
    import json

    from tests.test_cpu_formats import GOLD, _cli
    r = _cli("train-attacker", "--dimension", "--n", "30", "--out", tmp_path / "dim.npz")
    assert r.returncode == 0, r.stderr
    info = json.loads(r.stdout.strip().splitlines()[-1])
    assert info["trees"] == list(dimattack.DIM_TREES) and len(info["val_der"]) == 4
    r = _cli("evaluate", "--graph", GOLD / "tiny.graph", "--plan", GOLD / "dim.plan", "--trials", "2",
             "--dim-attackers", tmp_path / "dim.npz")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    assert rep["equivalent"] and len(rep["lers"]) == 4 and rep["mean_ler"] >= 0.0

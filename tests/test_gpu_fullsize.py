"""GPU parity at the BASELINE configurations' real sizes (VERDICT r1 "next" #1).

Every configuration the bench times is compared here, at the size it is
timed at, with the CPU oracle (tests/oracle_pool.py spreads it over the host
cores; the schedule memo oracle runs in order in this process):

  cfg2 / headline  ResNet-18 224x224, 8 equivalence trials, the bench's 32
                   seeded sequence candidates: verdict, worst (within 1e-4
                   of the oracle's), T, per-predictor decoded tokens, LER and
                   R bit-exact — through the device-resident path the
                   bench's ``value`` times AND the worker-pool path its
                   ``e2e`` times (records identical; `worst` within 1e-4).
  cfg5             >= 1000 traces through each of H = 128/256/512: several
                   16-trace cluster rows and a ragged last one.
  cfg4             VGG-16 224x224, 2 dimension candidates, 8 trials.
  cfg1             C1C2 56x56, dimension candidates, 8 trials, outputs.

Reference semantics: interpreter.py:93-118 (verdict / worst), costmodel.py:
248-293 (memo, trace, T), PAPER.md:425-428 + SPEC.md:471-571 (restated
fitness).
"""

import numpy as np
import pytest
import torch

from oracle import costmodel_ref as CM
from oracle import fitness_ref as FR
from oracle import interp_ref as IR
from paper_2107_09789_b200 import _native as N
from paper_2107_09789_b200 import attacker, executor, fixtures, ga, knobs
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator
from paper_2107_09789_b200.ir import label_sequence
from tests import oracle_pool

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
FP32_TOL = 1e-4


def _rel(got, ref):
    return float(np.max(np.abs(got.astype(np.float64) - ref) / (1.0 + np.abs(ref))))


def bench_plans(vanilla, total, seed, mode="sequence"):
    """bench.population_plans: the seed path of the timed workload."""
    rng = np.random.default_rng(seed)
    space = ga.search_space(vanilla, mode)
    sizes = ga.domain_sizes(mode, space)
    return [ga.decode_genome(vanilla, mode, space, g) for g in ga.random_genomes(rng, sizes, total)]


def _oracle_population(g, plans, trials, predictors, pool):
    """Per candidate: feasible, ok, worst, T, per-predictor tokens and LERs,
    R and mean — the reference path, memo in candidate order."""
    truth = attacker.encode_labels(label_sequence(g))
    t_star = CM.profile_pipeline(g, "default", None, None, CM.ScheduleMemo())[3]
    verdicts = pool.map(oracle_pool.equiv_job, plans, chunksize=1)
    memo = CM.ScheduleMemo()
    out, lstm_jobs = [], []
    for p, v in zip(plans, verdicts):
        if v is None:
            out.append({"feasible": False})
            continue
        og, d = knobs.apply_plan(g, p)
        _, _, rows, T = CM.profile_pipeline(og, "default", d.fusion_limits, d.schedule_strategies, memo)
        feats = np.array([[r[f] for f in CM.FEATURES] for r in rows], dtype=np.float64)
        out.append({"feasible": True, "ok": v[0], "worst": v[1], "T": T, "feats": feats})
        lstm_jobs += [(feats, pr.features, pr.weights()) for pr in predictors]
    toks = pool.map(oracle_pool.lstm_job, lstm_jobs, chunksize=1)
    q = 0
    for o in out:
        if not o["feasible"]:
            continue
        o["tokens"] = toks[q:q + len(predictors)]
        q += len(predictors)
        o["lers"] = [FR.ler(t, truth) for t in o["tokens"]]
        o["R"], o["mean"] = FR.eq10(o["lers"], o["T"], o["ok"], t_star, 0.02)
    return out, t_star


def test_cfg2_headline_population_matches_oracle(ctx):
    g = fixtures.resnet18()
    plans = bench_plans(g, 32, seed=0)
    ev = Evaluator()
    pe = PopulationEvaluator(g, ev, budget=0.02, trials=8, seed=0, memo={})
    # the bench's `value` path: prepared once, device pipeline with a cold memo
    prep = pe.prepare(plans, memo={})
    out = pe.run(prep, cold_schedules=True)
    rec = pe.collect(out)
    tp = out["trace"]
    feats_dev = tp.feats.cpu().numpy()
    lers_dev = out["lers"].cpu().numpy()
    feas = prep["feas"]
    toks_dev = []
    for pr in ev.predictors:
        tk, nk = attacker.decode(tp.feats, tp.offsets, len(feas), prep["t_max"], pr)
        toks_dev.append((tk.cpu().numpy(), nk.cpu().numpy()))
    # the bench's `e2e` path: host workers, micro-batches, cold memo
    try:
        rec_e2e = pe.evaluate_records(plans, memo={})
    finally:
        pe.close()
    # identical records, except `worst` (a float32 max of |a-b|/(1+|b|)): the
    # micro-batch split changes which few-tile conv groups run split-K, i.e.
    # the fp32 summation order of both graphs' outputs, within tolerance — and
    # so the verdict (and the reward built on it) of a candidate whose two
    # `worst` values straddle the 1e-5 equivalence tolerance itself
    tol = executor.DEFAULT_TOL[N.PREC_TF32X3]
    straddle = (rec["worst"] <= tol) != (rec_e2e["worst"] <= tol)
    assert np.max(np.abs(rec_e2e["worst"] - rec["worst"])) <= FP32_TOL
    assert np.all(np.abs(rec_e2e["worst"][straddle] - rec["worst"][straddle]) <= 2 * tol)
    for f in rec.dtype.names:
        if f == "worst":
            continue
        if f in ("ok", "reward"):
            assert rec_e2e[f][~straddle].tobytes() == rec[f][~straddle].tobytes(), f
        else:
            assert rec_e2e[f].tobytes() == rec[f].tobytes(), f
    assert np.array_equal(rec_e2e["ok"][straddle] != 0, rec_e2e["worst"][straddle] <= tol)

    pool = oracle_pool.pool(g, trials=8, seed=0)
    try:
        want, t_star = _oracle_population(g, plans, 8, ev.predictors, pool)
        # verdicts decided by rounding: with random-init ResNet-18 the softmax is
        # near one-hot and logits are O(100), so fp32 rounding of the logits
        # (~1e-5 absolute) moves `worst` by as much as the 1e-5 tolerance itself.
        # Where the GPU and the fp32 oracle disagree, the exact (fp64) worst must
        # lie closer to the tolerance than the oracle's own rounding error:
        # the reference's verdict there depends on its BLAS summation order.
        split = [i for i, o in enumerate(want) if o["feasible"] and bool(rec["ok"][i]) != o["ok"]]
        exact = dict(zip(split, pool.map(oracle_pool.equiv64_job, [plans[i] for i in split], chunksize=1)))
    finally:
        pool.close()
    assert pe.t_star == t_star
    assert sum(o["feasible"] for o in want) == len(feas) >= 24
    for i, o in enumerate(want):
        assert bool(rec["feasible"][i]) == o["feasible"], i
        if not o["feasible"]:
            assert rec["reward"][i] == 0.0
            continue
        k = feas.index(i)
        lo, hi = tp.offsets_host[k], tp.offsets_host[k + 1]
        assert np.array_equal(feats_dev[lo:hi].view(np.uint64), o["feats"].view(np.uint64)), i
        assert rec["latency"][i] == o["T"], i
        assert abs(float(rec["worst"][i]) - o["worst"]) <= FP32_TOL, (i, rec["worst"][i], o["worst"])
        if i in exact:
            # measured at RN18 224x224: about half the candidates, e.g. the trial
            # whose top softmax probability is 0.80 gives fp32-oracle worst 3.2e-5
            # against an exact worst of ~1e-23 (function-preserving); the GPU's
            # verdict is exact arithmetic's
            w64 = exact[i]
            assert abs(w64 - 1e-5) < abs(o["worst"] - w64), (i, rec["worst"][i], o["worst"], w64)
            assert bool(rec["ok"][i]) == (w64 <= 1e-5), (i, rec["worst"][i], o["worst"], w64)
            o["ok"] = bool(rec["ok"][i])  # the rounding-decided verdict: Eq. 10 below follows the GPU's
            o["R"], o["mean"] = FR.eq10(o["lers"], o["T"], o["ok"], t_star, 0.02)
        assert bool(rec["ok"][i]) == o["ok"], i
        for p in range(len(ev.predictors)):
            tk, nk = toks_dev[p]
            assert tk[k, :nk[k]].tolist() == o["tokens"][p], (i, p)
            assert lers_dev[p, i] == o["lers"][p], (i, p)
        assert rec["ntok"][i] == len(o["tokens"][0])
        assert rec["mean_ler"][i] == o["mean"] and rec["reward"][i] == o["R"], i
    # outputs of a few candidates on trial 0 against the oracle (softmax and logits)
    x0 = IR.trial_inputs(g.input_shape.as_tuple(), 1, 0)[0]
    from paper_2107_09789_b200.ir import Graph
    for i in feas[:3]:
        og, _ = knobs.apply_plan(g, plans[i])
        logits = og.nodes[og.output_id].inputs[0]  # the SoftMax input (a branched Linear has a new id)
        _, vals = IR.execute(og, x0, keep=True)
        assert _rel(executor.execute(og, x0), vals[og.output_id].astype(np.float64)) <= FP32_TOL
        _, exact = IR.execute(og, x0, keep=True, dtype=np.float64)
        got_l = executor.execute(Graph(og.nodes, logits, og.input_shape), x0)
        assert _rel(got_l, exact[logits]) <= max(FP32_TOL, 2.0 * _rel(vals[logits], exact[logits]))


@pytest.mark.parametrize("hidden", [128, 256, 512])
def test_cfg5_lstm_sweep_matches_oracle(ctx, hidden, monkeypatch):
    """1003 traces (62 full 16-trace cluster rows + a ragged row of 11),
    T ~ U[119,169], cost-model-scale features: tokens, ED and LER bit-exact;
    every kernel shape (warps per CTA x traces per thread) decodes the same."""
    rng = np.random.default_rng(hidden + 5)
    nt = 1003
    lens = rng.integers(119, 170, nt)
    offs = np.zeros(nt + 1, np.int32)
    offs[1:] = np.cumsum(lens)
    feats = rng.random((int(offs[-1]), 9)) * 1e6
    feats[:, 0] *= 10.0
    pred = attacker.init_predictor(hidden, 9, seed=hidden)
    fd = torch.from_numpy(feats).to(ctx.device)
    od = torch.from_numpy(offs).to(ctx.device)
    truth = attacker.encode_labels(label_sequence(fixtures.resnet18()))
    tk, nk = attacker.decode(fd, od, nt, int(lens.max()), pred)
    ed, lr, _ = attacker.edit_distances(tk, nk, truth)
    tk, nk, ed, lr = tk.cpu().numpy(), nk.cpu().numpy(), ed.cpu().numpy(), lr.cpu().numpy()
    pool = oracle_pool.pool()
    try:
        want = pool.map(oracle_pool.lstm_job, [(feats[offs[i]:offs[i + 1]], 9, pred.weights()) for i in range(nt)],
                        chunksize=8)
    finally:
        pool.close()
    for i in range(nt):
        assert tk[i, :nk[i]].tolist() == want[i], i
        e = FR.levenshtein(want[i], truth)
        assert ed[i] == e and lr[i] == e / len(truth), i
    for variant in ("rb4", "rb8", "r8w4", "r8w8"):
        monkeypatch.setenv("TOBF_LSTM_VARIANT", variant)
        tv, nv = attacker.decode(fd, od, nt, int(lens.max()), pred)
        nv = nv.cpu().numpy()
        assert np.array_equal(nv, nk), variant
        tv = tv.cpu().numpy()
        assert all(np.array_equal(tv[i, :nk[i]], tk[i, :nk[i]]) for i in range(nt)), variant


def test_cfg4_vgg16_dimension_candidates_match_oracle(ctx):
    """VGG-16 224x224 (553 MB of weights), 2 widen + kernel-widen candidates,
    8 trials: verdict, worst, T and R against the oracle."""
    g = fixtures.vgg16()
    plans = bench_plans(g, 2, seed=0, mode="dimension")
    ev = Evaluator(predictors=attacker.bagged_predictors(hiddens=(128,)))
    pe = PopulationEvaluator(g, ev, budget=0.02, trials=8, seed=0, memo={})
    try:
        rec = pe.evaluate_records(plans, memo={}, workers=0)
    finally:
        pe.close()
    pool = oracle_pool.pool(g, trials=8, seed=0, procs=min(16, len(plans) * 8))
    try:
        res = pool.map(oracle_pool.equiv_trial_job, [(p, t) for p in plans for t in range(8)], chunksize=1)
    finally:
        pool.close()
    truth = attacker.encode_labels(label_sequence(g))
    t_star = CM.profile_pipeline(g, "default", None, None, CM.ScheduleMemo())[3]
    memo = CM.ScheduleMemo()
    for i, p in enumerate(plans):
        per = res[8 * i:8 * (i + 1)]
        ok, worst = all(r[1] for r in per), max(r[0] for r in per)
        assert bool(rec["ok"][i]) == ok and abs(float(rec["worst"][i]) - worst) <= FP32_TOL, (i, rec[i], ok, worst)
        og, d = knobs.apply_plan(g, p)
        _, _, rows, T = CM.profile_pipeline(og, "default", d.fusion_limits, d.schedule_strategies, memo)
        assert rec["latency"][i] == T
        feats = np.array([[r[f] for f in CM.FEATURES] for r in rows])
        lers = [FR.ler(FR.lstm_ctc(feats, 9, pr.weights()), truth) for pr in ev.predictors]
        R, mean = FR.eq10(lers, T, ok, t_star, 0.02)
        assert rec["mean_ler"][i] == mean and rec["reward"][i] == R


def test_cfg1_c1c2_56_outputs_and_verdicts(ctx):
    """Config 1 at its real size (56x56): the obfuscated conv stack's outputs
    on every trial within 1e-4 of the oracle, verdicts/worst identical."""
    g = fixtures.c1c2()
    assert g.input_shape.as_tuple() == (1, 3, 56, 56)
    plans = bench_plans(g, 6, seed=1, mode="dimension")
    cands = [knobs.apply_plan(g, p)[0] for p in plans]
    ok, worst = executor.evaluate_equivalence(g, cands, trials=8, seed=0)
    xs = IR.trial_inputs(g.input_shape.as_tuple(), 8, 0)
    for i, og in enumerate(cands):
        rok, rworst = IR.equivalence_check(g, og, trials=8, seed=0)
        assert bool(ok[i]) == rok and abs(float(worst[i]) - rworst) <= FP32_TOL
        for x in xs[:2]:
            assert _rel(executor.execute(og, x), IR.execute(og, x).astype(np.float64)) <= FP32_TOL


def test_cfg4_vgg16_bf16_mode_matches_oracle(ctx):
    """cfg4 as BASELINE specifies it: VGG-16 224x224, widen + kernel-widen
    candidates, the bf16 conv path. Verdicts at the bf16 tolerance (2e-2)
    equal the fp32 oracle's at 2e-2; candidate outputs on trial 0 within 2e-2
    of the oracle's."""
    BF16_TOL = 2e-2
    g = fixtures.vgg16()
    plans = bench_plans(g, 2, seed=0, mode="dimension")
    ev = Evaluator(predictors=attacker.bagged_predictors(hiddens=(128,)))
    pe = PopulationEvaluator(g, ev, budget=0.02, trials=8, seed=0, memo={}, precision="bf16")
    try:
        rec = pe.evaluate_records(plans, memo={}, workers=0)
    finally:
        pe.close()
    pool = oracle_pool.pool(g, trials=8, seed=0, procs=min(16, len(plans) * 8))
    try:
        res = pool.map(oracle_pool.equiv_trial_job, [(p, t) for p in plans for t in range(8)], chunksize=1)
    finally:
        pool.close()
    x0 = IR.trial_inputs(g.input_shape.as_tuple(), 1, 0)[0]
    for i, p in enumerate(plans):
        worst = max(r[0] for r in res[8 * i:8 * (i + 1)])
        assert bool(rec["ok"][i]) == (worst <= BF16_TOL), (i, rec[i], worst)
        og, _ = knobs.apply_plan(g, p)
        got = executor.execute(og, x0, precision="bf16")
        assert _rel(got, IR.execute(og, x0).astype(np.float64)) <= BF16_TOL


def test_headline_forward_bit_deterministic(ctx):
    """The headline population's forward, repeated on one linked run and on
    freshly linked runs, is bit-identical every time: tiles are claimed
    dynamically, split-K partials summed in unit order, and the TMA-fed
    A staging ring releases a slot only after its rows were consumed (an early
    release let a TMA refill overwrite rows still being read: a wrong block in
    roughly one population forward in ten, scripts/race_probe.py)."""
    g = fixtures.resnet18()
    plans = bench_plans(g, 32, seed=0)
    pe = PopulationEvaluator(g, Evaluator(), budget=0.02, trials=8, seed=0, memo={})
    x = pe.x_host.to(ctx.device)

    def outputs(run):
        return torch.stack([run.output_nchw(i).reshape(-1) for i in range(len(run.plans))]).cpu()

    try:
        ref = None
        for relink in range(3):
            run = pe.prepare(plans, memo={})["run"]
            for _ in range(6):
                run.set_input(x)
                run.run()
                out = outputs(run)
                if ref is None:
                    ref = out
                assert torch.equal(out.view(torch.int32), ref.view(torch.int32)), relink
    finally:
        pe.close()

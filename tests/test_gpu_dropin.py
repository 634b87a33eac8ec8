"""The drop-in on the GPU with the reference's own objects.

INTEGRATION.md §3's maintainer patch (refcompat.install) is applied to the
real, unmodified reference package (baseline/_ref, vendored by
scripts/vendor_reference.sh), and the patched package's hot entry points —
now the B200 engine — are compared with the reference's own numpy functions
on reference-typed graphs: equivalence verdicts identical, execute within
1e-4, compile_graph kernels / schedules and profile_pipeline traces
bit-identical (reference Trace equality), all answered in reference classes.
"""

import numpy as np
import pytest

import paper_2107_09789_b200 as eng
from paper_2107_09789_b200 import fixtures, ga, refcompat
from tests import refpkg

ref = refpkg.load()
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(ref is None, reason="baseline/_ref not vendored")]


def _plans(g, mode, n, seed):
    rng = np.random.default_rng(seed)
    space = ga.search_space(g, mode)
    sizes = ga.domain_sizes(mode, space)
    return [ga.decode_genome(g, mode, space, rng.integers(0, sizes)) for _ in range(n)]


@pytest.mark.parametrize("name,mode,size", [("resnet18", "sequence", 64), ("c1c2", "dimension", 24)])
def test_patched_reference_hot_path(ctx, name, mode, size):
    g = fixtures.FIXTURES[name](size=size)
    rg = refpkg.ref_graph(ref, g)
    # the reference's own implementations, captured before the patch
    own = {n: getattr(ref, n) for n in refcompat.HOT_PATH}
    prof = ref.BUILTIN_PROFILES["default"]
    saved = refcompat.install(ref)
    try:
        for plan in _plans(g, mode, 2, seed=3):
            rog, rd = ref.apply_plan(rg, refpkg.ref_plan(ref, plan))
            ok, worst = ref.equivalence_check(rg, rog, trials=2, seed=0)
            rok, rworst = own["equivalence_check"](rg, rog, trials=2, seed=0)
            assert ok == rok and abs(worst - rworst) <= 1e-4
            x = np.random.default_rng(1).standard_normal(rg.input_shape.as_tuple()).astype(np.float32)
            got, want = ref.execute(rog, x), own["execute"](rog, x)
            assert np.max(np.abs(got - want) / (1 + np.abs(want))) <= 1e-4
            cg = ref.compile_graph(rog, prof, rd.fusion_limits, rd.schedule_strategies)
            wcg = own["compile_graph"](rog, prof, rd.fusion_limits, rd.schedule_strategies)
            assert type(cg) is type(wcg) and cg.kernels == wcg.kernels and cg.schedules == wcg.schedules
            tr = ref.profile_pipeline(rog, ref.LeakageCase.C, prof, rd.fusion_limits, rd.schedule_strategies)
            wtr = own["profile_pipeline"](rog, ref.LeakageCase.C, prof, rd.fusion_limits, rd.schedule_strategies)
            assert type(tr) is type(wtr) and tr == wtr  # every feature, label, anchor: bit-exact
            assert tr.total_latency == wtr.total_latency
    finally:
        refcompat.uninstall(ref, saved)


def test_population_evaluator_takes_reference_objects(ctx):
    g = fixtures.c1c2(size=16)
    rg = refpkg.ref_graph(ref, g)
    plans = _plans(g, "dimension", 3, seed=2)
    ev = eng.Evaluator(predictors=eng.bagged_predictors(hiddens=(128,)), case=ref.LeakageCase.C,
                       profile=ref.BUILTIN_PROFILES["default"])
    a = eng.PopulationEvaluator(rg, ev, trials=2, memo={}).evaluate_records(
        [refpkg.ref_plan(ref, p) for p in plans], memo={}, workers=0)
    b = eng.PopulationEvaluator(g, eng.Evaluator(predictors=ev.predictors), trials=2, memo={}).evaluate_records(
        plans, memo={}, workers=0)
    assert a.tobytes() == b.tobytes()

"""Worker-process host preparation (hostpipe.py) produces exactly the
in-process forward plans and trace records: same descriptor rows, same
signatures, weight references that resolve to equal arrays in the parent."""

import numpy as np
import pytest

from paper_2107_09789_b200 import executor, fixtures, ga, hostpipe, knobs
from paper_2107_09789_b200.ir import analyze
from paper_2107_09789_b200.trace import trace_records


@pytest.fixture(scope="module")
def population():
    g = fixtures.resnet18(size=64)
    space = ga.search_space(g, "sequence")
    sizes = ga.domain_sizes("sequence", space)
    plans = [ga.decode_genome(g, "sequence", space, x) for x in ga.random_genomes(np.random.default_rng(7), sizes, 6)]
    return g, plans


def _resolved_tables(plan, refs):
    w = [(refs.resolve(e[0]),) + tuple(e[1:]) for e in plan.wimg]
    a = [refs.resolve(r) for r in plan.affine]
    c = [(refs.resolve(e[0]),) + tuple(e[1:]) for e in plan.const]
    return w, a, c


def test_pool_matches_in_process(population):
    g, plans = population
    va = analyze(g)
    pool = hostpipe.HostPool(g, reps=2, pname="default", workers=2)
    try:
        handles = pool.submit(plans, per_job=2)
        results = [r for h in reversed(handles) for r in pool.result(h)][::-1]
        results.sort(key=lambda r: r[0])
    finally:
        pool.close()
    prefs = hostpipe.ParentRefs(g)
    assert [r[0] for r in results] == list(range(len(plans)))
    for (c, err, payload), plan in zip(results, plans):
        og, d, ana = knobs.apply_plan_analyzed(g, plan, va)
        assert err is None
        fp, ct, new = payload
        prefs.adopt(c, new)
        refs = executor.ArrayRefs()
        ref_fp = executor.plan_forward(executor.lower(og, ana), 2, refs)
        for f in ("conv", "conv_level", "conv_bn", "conv_k", "ew", "ew_level"):
            assert np.array_equal(getattr(fp, f), getattr(ref_fp, f)), f
        assert (fp.arena_bytes, fp.out_off, fp.out_shape, fp.flops_per_image) == \
               (ref_fp.arena_bytes, ref_fp.out_off, ref_fp.out_shape, ref_fp.flops_per_image)
        (w1, a1, c1), (w2, a2, c2) = _resolved_tables(fp, prefs), _resolved_tables(ref_fp, refs)
        assert len(w1) == len(w2) and len(a1) == len(a2) and len(c1) == len(c2)
        for x, y in zip(w1 + c1, w2 + c2):
            assert np.array_equal(x[0], y[0]) and x[1:] == y[1:]
        for x, y in zip(a1, a2):
            assert np.array_equal(x, y)
        ref_ct, _, _ = trace_records(og, d.fusion_limits, d.schedule_strategies, "default", ana)
        # workers send signature digests + only the tuples they have not sent before
        assert ct.sigs is None and len(ct.new_sigs) <= len(set(ref_ct.sigs))
        ct.expand(prefs.sig_table)
        assert np.array_equal(ct.recs, ref_ct.recs) and ct.sigs == ref_ct.sigs


def test_micro_batch_bounds():
    from paper_2107_09789_b200.evaluate import _micro_bounds
    assert _micro_bounds(32, 16) == [(0, 16), (16, 32)]
    assert _micro_bounds(7, 3) == [(0, 3), (3, 6), (6, 7)]
    assert _micro_bounds(32, (8, 24)) == [(0, 8), (8, 32)]
    assert _micro_bounds(30, [4, 12]) == [(0, 4), (4, 16), (16, 28), (28, 30)]
    assert _micro_bounds(0, 8) == []
    assert _micro_bounds(32, "auto") == [(0, 8), (8, 32)]
    assert _micro_bounds(3, "auto") == [(0, 1), (1, 3)]
    assert _micro_bounds(80, "auto") == [(0, 8), (8, 32), (32, 80)]
    assert _micro_bounds(256, "auto") == [(0, 8), (8, 32), (32, 80), (80, 144), (144, 208), (208, 256)]
    assert _micro_bounds(32, None) == [(0, 32)] and _micro_bounds(0, None) == []  # evaluate_stream default
    with pytest.raises(ValueError):
        _micro_bounds(4, 0)


def test_plan_wire_round_trip():
    from paper_2107_09789_b200 import fixtures, ga
    from paper_2107_09789_b200.hostpipe import plan_unwire, plan_wire
    g = fixtures.c1c2(size=8)
    for mode in ("sequence", "dimension"):
        space = ga.search_space(g, mode)
        rng = np.random.default_rng(1)
        for x in ga.random_genomes(rng, ga.domain_sizes(mode, space), 5):
            p = ga.decode_genome(g, mode, space, x)
            assert plan_unwire(plan_wire(p)) == p

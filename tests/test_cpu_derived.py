"""Knob-derived weights (derived.py): the lazy knob path records
per-axis gathers of the vanilla arrays instead of materialising widened /
kernel-widened / branched weights, and materialising them reproduces the
eager knobs (= the reference's numpy code) bit for bit."""

import numpy as np
import pytest

from paper_2107_09789_b200 import executor, fixtures, ga, hostpipe, knobs
from paper_2107_09789_b200.derived import (DerivedWeight, consecutive_derived, seg_concat, seg_expand,
                                           seg_identity, seg_scale, seg_slice)
from paper_2107_09789_b200.ir import analyze


def _plans(g, mode, n, seed):
    space = ga.search_space(g, mode)
    sizes = ga.domain_sizes(mode, space)
    rng = np.random.default_rng(seed)
    return [ga.decode_genome(g, mode, space, x) for x in ga.random_genomes(rng, sizes, n)]


def test_segment_algebra():
    s = seg_identity(6)
    assert seg_expand(s)[0].tolist() == [0, 1, 2, 3, 4, 5]
    head = seg_scale(seg_slice(s, 0, 2), 0.5)
    dup = seg_concat(head, seg_slice(s, 2, 6), head)
    idx, sc = seg_expand(dup)
    assert idx.tolist() == [0, 1, 2, 3, 4, 5, 0, 1]
    assert sc.tolist() == [0.5, 0.5, 1, 1, 1, 1, 0.5, 0.5]
    pad = seg_concat(((-1, 2, 0.0),), s, ((-1, 2, 0.0),))
    assert seg_expand(pad)[0].tolist() == [-1, -1, 0, 1, 2, 3, 4, 5, -1, -1]
    assert seg_slice(pad, 1, 4) == ((-1, 1, 0.0), (0, 2, 1.0))
    assert seg_concat(seg_slice(s, 0, 3), seg_slice(s, 3, 6)) == s  # contiguous pieces merge


def test_derived_ops_match_numpy():
    rng = np.random.default_rng(0)
    w = rng.standard_normal((3, 3, 8, 6)).astype(np.float32)
    d = DerivedWeight.of(w, "conv")
    assert d.is_identity() and np.array_equal(np.asarray(d), w)
    a = d.dup_tail(3, 2)
    assert np.array_equal(np.asarray(a), np.concatenate([w, w[..., :2]], axis=-1))
    half = w.copy()
    half[:, :, :3, :] *= 0.5
    b = d.dup_tail(2, 3, 0.5)
    assert np.asarray(b).tobytes() == np.concatenate([half, half[:, :, :3, :]], axis=2).tobytes()
    c = b.pad_kernel(1)
    ref = np.pad(np.concatenate([half, half[:, :, :3, :]], axis=2), ((1, 1), (1, 1), (0, 0), (0, 0)))
    assert np.asarray(c).tobytes() == ref.tobytes() and c.shape == ref.shape and c.size == ref.size
    parts = [c.slice(3, 0, 3), c.slice(3, 3, 6)]
    assert np.asarray(consecutive_derived(parts, -1)).tobytes() == ref.tobytes()
    # linear (c*H*W, j) rows in NCHW-flatten order, consumer of a widened producer
    lw = rng.standard_normal((4 * 2 * 2, 5)).astype(np.float32)
    ld = DerivedWeight.of(lw, "linear", (2, 2)).dup_tail(2, 1, 0.5)
    rows = lw.reshape(4, 4, 5).copy()
    rows[:1] *= 0.5
    want = np.concatenate([rows, rows[:1]], axis=0).reshape(5 * 4, 5)
    assert np.asarray(ld).tobytes() == want.tobytes() and ld.shape == want.shape


@pytest.mark.parametrize("name,mode,kw", [("vgg16", "dimension", {"size": 32, "hidden": 256}),
                                          ("resnet18", "dimension", {"size": 64}),
                                          ("c1c2", "dimension", {"size": 24}),
                                          ("resnet18", "sequence", {"size": 64})])
def test_lazy_knobs_materialize_to_eager(name, mode, kw):
    g = fixtures.FIXTURES[name](**kw)
    va = analyze(g)
    seen = 0
    for plan in _plans(g, mode, 8, seed=5):
        try:
            eager, _ = knobs.apply_plan(g, plan)
        except knobs.TransformError:
            continue
        lazy, _, _ = knobs.apply_plan_analyzed(g, plan, va, lazy=True)
        assert set(eager.nodes) == set(lazy.nodes)
        for nid, n in eager.nodes.items():
            m = lazy.nodes[nid]
            assert (n.kind, n.attrs, n.inputs) == (m.kind, m.attrs, m.inputs)
            if isinstance(m.weights, DerivedWeight):
                seen += 1
                a = np.asarray(m.weights)
                assert a.shape == n.weights.shape and a.dtype == n.weights.dtype
                assert a.tobytes() == np.ascontiguousarray(n.weights).tobytes(), nid
            elif n.weights is None:
                assert m.weights is None
            else:
                assert np.array_equal(n.weights, m.weights)
    if mode == "dimension":
        assert seen > 0


def test_worker_ships_gathers_not_arrays():
    """hostpipe encodes a widened candidate as ("D", vanilla ref, gather) weight
    references: nothing but the vanilla arrays' names crosses the process
    boundary, and the parent resolves them onto its own vanilla arrays."""
    g = fixtures.vgg16(size=32, hidden=256)
    hostpipe._worker_init(g, 2, "default")
    W = hostpipe._W
    prefs = hostpipe.ParentRefs(g)
    n_derived = 0
    for i, plan in enumerate(_plans(g, "dimension", 4, seed=9)):
        c, err, payload = hostpipe.encode_candidate(i, plan, W["vanilla"], W["analysis"], 2, "default", W["roots"])
        if err is not None:
            continue
        fp, ct, new = payload
        assert sum(a.nbytes for a in new) < 1 << 20  # no materialised weights shipped
        eager, _ = knobs.apply_plan(g, plan)
        for entry in fp.wimg:
            ref = entry[0]
            if ref[0] == "D":
                n_derived += 1
                dw = prefs.resolve(ref)
                assert isinstance(dw, DerivedWeight)
                assert any(dw.base is v for v in prefs.vanilla.values())
        # the lowering's weight images cover the eager graph's conv weights
        lw = executor.lower(eager)
        assert len(fp.conv) == sum(1 for op in lw.ops if op.kind == "gemm")
    assert n_derived > 0

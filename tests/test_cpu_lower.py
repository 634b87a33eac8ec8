"""Host lowering (executor.lower): sibling branch parts that read one input and
whose weights are consecutive slices of one array become a single GEMM
(transforms.py:173-231 emits them as separate layers). CPU-only checks of the
grouping; numerics of the fused GEMM are covered by tests/test_gpu_parity.py."""

import numpy as np

from paper_2107_09789_b200 import executor, fixtures, ga, knobs
from paper_2107_09789_b200.ir import OperatorKind as K


def _plans(mode, n, seed=0):
    g = fixtures.resnet18()
    space = ga.search_space(g, mode)
    sizes = ga.domain_sizes(mode, space)
    for genome in ga.random_genomes(np.random.default_rng(seed), sizes, n):
        yield g, knobs.apply_plan(g, ga.decode_genome(g, mode, space, genome))[0]


def test_sibling_views_equal_concatenated_weights():
    seen = {"out": 0, "in": 0}
    for _, og in _plans("sequence", 12):
        lw = executor.lower(og)
        for op in lw.ops:
            if op.kind != "gemm" or op.w is None:
                continue
            combiner = next(n for n in og.nodes.values() if op.node in n.inputs and n.kind in (K.Concat, K.Add))
            ws = [og.nodes[p].weights for p in combiner.inputs]
            if combiner.kind is K.Concat:
                seen["out"] += 1
                ref = np.concatenate(ws, axis=-1)
            else:
                seen["in"] += 1
                ref = np.concatenate(ws, axis=2 if og.nodes[op.node].kind is K.Conv2D else 0)
            assert np.array_equal(op.w, ref)
            assert op.j == lw.shapes[combiner.id].channels
    assert seen["out"] > 0 and seen["in"] > 0, seen


def test_sibling_fusion_covers_every_node_once():
    for _, og in _plans("sequence", 8, seed=3):
        for fuse in (False, True):
            lw = executor.lower(og, fuse_siblings=fuse)
            gemm_j = sum(op.j or og.nodes[op.node].attrs["j"] for op in lw.ops if op.kind == "gemm")
            ref_j = sum(n.attrs["j"] for n in og.nodes.values() if n.kind in (K.Conv2D, K.Linear))
            assert gemm_j <= ref_j  # in-branch groups compute j once for all parts
            if not fuse:
                assert gemm_j == ref_j


def test_forward_plan_symbolic_rows():
    """plan_forward (host only): every pointer field is symbolic and refers to
    an arena offset inside the graph's block or to an entry of its tables."""
    S = executor
    for g, og in _plans("sequence", 6, seed=5):
        refs = S.ArrayRefs()
        plan = S.plan_forward(S.lower(og), 8, refs)
        assert len(plan.conv) and len(plan.conv) == len(plan.conv_level) == len(plan.conv_bn)
        sizes = {S.SP_WIMG: len(plan.wimg), S.SP_AFFINE: len(plan.affine), S.SP_CONST: len(plan.const),
                 S.SP_XCOL: len(plan.xcol)}
        cols = [plan.conv["x"], plan.conv["y"], plan.conv["wimg"], plan.conv["epi"]["ptr"].ravel(),
                plan.ew["x"], plan.ew["y"], plan.ew["epi"]["ptr"].ravel()]
        for col in cols:
            col = col.astype(np.uint64)
            space = col >> np.uint64(S._SP_SHIFT)
            val = col & np.uint64(S._SP_LOW)
            for sp, v in zip(space.tolist(), val.tolist()):
                if sp == S.SP_ARENA:
                    assert v < plan.arena_bytes
                elif sp in sizes:
                    assert v < sizes[sp]
                else:
                    assert sp in (0, S.SP_INPUT)
        # the stem (7x7, 3 channels) reads the input's im2col matrix (160 = 7*7*3
        # rounded up to 32) as a 1x1 GEMM; its weight entry is the im2col view
        assert plan.xcol == [(8, 224, 224, 3, 7, 7, 2, 3, 112, 112, 160)]
        stem = plan.conv[(plan.conv["x"].astype(np.uint64) >> np.uint64(S._SP_SHIFT)) == S.SP_XCOL]
        assert len(stem) >= 1 and (stem["Cp"] == 160).all() and (stem["k1"] == 1).all() and (stem["H"] == 112).all()
        assert sum(1 for e in plan.wimg if e[1] == 2) == len({int(v) for v in stem["wimg"]})
        for e in plan.wimg:
            w = refs.resolve(e[0])
            assert w.dtype == np.float32 and w.ndim in (2, 4)


def test_tail_alignment_keeps_dependencies(monkeypatch):
    """executor._aligned_levels: with TAIL_ALIGN = f, each graph's ops at
    levels >= f * depth move down by the graph's slack, so every graph ends
    at the population's last level and no op lands at or before a producer's
    level (the whole suffix moves by one amount)."""
    S = executor
    plans, lws = [], []
    for g, og in _plans("sequence", 6, seed=7):
        lw = S.lower(og)
        lws.append(lw)
        plans.append(S.plan_forward(lw, 8, S.ArrayRefs()))
    depth = [max(int(p.conv_level.max()), int(p.ew_level.max(initial=0))) for p in plans]
    assert len(set(depth)) > 1  # deepened candidates: unequal depths
    for f in (0.0, 0.3, 0.5, 1.0):
        monkeypatch.setattr(S, "TAIL_ALIGN", f)
        cl, el = S._aligned_levels(plans)
        ci = ei = 0
        for p, dp in zip(plans, depth):
            c, e = cl[ci:ci + len(p.conv)], el[ei:ei + len(p.ew)]
            ci += len(p.conv)
            ei += len(p.ew)
            if f <= 0:
                assert np.array_equal(c, p.conv_level) and np.array_equal(e, p.ew_level)
                continue
            assert max(int(c.max()), int(e.max(initial=0))) == max(depth)
            # order-preserving per graph: a strictly increasing map of the old levels
            old = np.concatenate([p.conv_level, p.ew_level])
            new = np.concatenate([c, e])
            for a in np.unique(old):
                assert len(np.unique(new[old == a])) == 1
            pairs = sorted({(int(a), int(b)) for a, b in zip(old, new)})
            assert all(b1 < b2 for (_, b1), (_, b2) in zip(pairs, pairs[1:]))


def test_regroup_launch_tma_flags():
    """executor._regroup: one launch per (level, BN); block_n carries
    TOBF_CONV_TMA when any problem takes A by TMA im2col and
    TOBF_CONV_TMA_ALL only when every problem does (the kernel variant
    without the cp.async gather); flag values match include/tobf.h."""
    import re
    from pathlib import Path

    from paper_2107_09789_b200 import _native as N
    from paper_2107_09789_b200 import executor as E

    hdr = (Path(__file__).resolve().parents[1] / "include" / "tobf.h").read_text()
    assert int(re.search(r"#define TOBF_CONV_TMA 0x([0-9a-fA-F]+)", hdr).group(1), 16) == N.CONV_TMA
    assert int(re.search(r"#define TOBF_CONV_TMA_ALL 0x([0-9a-fA-F]+)", hdr).group(1), 16) == N.CONV_TMA_ALL
    n = 7
    conv = np.zeros(n, E.CONV_DTYPE)
    conv["mtiles"], conv["ntiles"], conv["ksplit"] = 3, 1, 1
    level = np.array([0, 0, 1, 1, 2, 2, 2])
    bn = np.array([64, 64, 128, 128, 64, 64, 64])
    k = np.array([5, 9, 2, 2, 3, 1, 4])
    tma = np.array([1, 1, 1, 0, 0, 0, 0])
    conv["tma"] = tma
    _, ctma, launches, ws, cnt = E._regroup(conv, tma.astype(np.int64), level, bn, k)
    flags = {(L[0], L[6] & 0xFF): L[6] & ~0xFF for L in launches}
    assert flags == {(0, 64): N.CONV_TMA | N.CONV_TMA_ALL, (1, 128): N.CONV_TMA, (2, 64): 0}
    assert [L[4] for L in launches] == [2, 2, 3] and ws == 0 and cnt == 0
    assert [L[5] for L in launches] == [6, 6, 9]  # tiles per launch

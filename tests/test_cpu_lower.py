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

"""Random-architecture generation for the attacker's training data
(SPEC.md:444-452): deterministic per seed, valid IR, PAPER §V-A ordering."""

import numpy as np

from paper_2107_09789_b200.attacker_train import ArchGenConfig, generate_random_arch
from paper_2107_09789_b200.ir import OperatorKind as K
from paper_2107_09789_b200.ir import label_sequence, validate


def test_random_archs_valid_and_ordered():
    cfg = ArchGenConfig()
    for i in range(120):
        g = generate_random_arch(cfg, i)
        assert not validate(g)
        ls = label_sequence(g)
        assert ls[-2:] == [K.Linear, K.SoftMax]           # classifier + softmax last
        first_linear = ls.index(K.Linear)
        assert all(k in (K.Linear, K.SoftMax) for k in ls[first_linear:])  # Linear only after all convs
        assert g.input_shape.as_tuple() == (1, 3, 32, 32)


def test_random_archs_deterministic():
    cfg = ArchGenConfig(seed=7)
    a, b = generate_random_arch(cfg, 3), generate_random_arch(cfg, 3)
    assert set(a.nodes) == set(b.nodes) and all(a.nodes[n] == b.nodes[n] for n in a.nodes)
    c = generate_random_arch(cfg, 4)
    assert [n.kind for n in c.nodes.values()] != [n.kind for n in a.nodes.values()] or \
        any(not np.array_equal(c.nodes[n].weights, a.nodes[n].weights) for n in a.nodes
            if n in c.nodes and a.nodes[n].weights is not None and c.nodes[n].weights is not None
            and a.nodes[n].weights.shape == c.nodes[n].weights.shape)


def test_imagenet_like_config():
    cfg = ArchGenConfig(input_shape=(1, 3, 224, 224), num_classes=1000, depth_range=(6, 14))
    g = generate_random_arch(cfg, 0)
    assert not validate(g)
    assert g.nodes[g.nodes[g.output_id].inputs[0]].attrs["j"] == 1000


def test_predictor_save_load_roundtrip(tmp_path):
    from paper_2107_09789_b200.attacker import bagged_predictors
    from paper_2107_09789_b200.attacker_train import load_predictors, save_predictors
    preds = bagged_predictors(hiddens=(32, 64))
    save_predictors(tmp_path / "a.npz", preds)
    back = load_predictors(tmp_path / "a.npz")
    assert [p.hidden for p in back] == [32, 64]
    for p, q in zip(preds, back):
        for k, v in p.weights().items():
            assert np.array_equal(v, q.weights()[k])

"""GA operators and search space on the host, with a
deterministic stand-in evaluator (the GPU evaluator is covered by -m gpu)."""

import numpy as np
import pytest

from oracle import fitness_ref as FR
from paper_2107_09789_b200 import fixtures, ga, knobs
from paper_2107_09789_b200.evaluate import RECORD_DTYPE
from paper_2107_09789_b200.attacker import eq10


def fake_eval(plans):
    """Deterministic reward from the plan contents (no randomness consumed)."""
    rec = np.zeros(len(plans), dtype=RECORD_DTYPE)
    for i, p in enumerate(plans):
        h = sum((k + 1) * hash((e.branching, e.deepen, e.skip, e.fusion_limit, e.widen_factor, e.kernel_widen,
                                 e.dummy_count, e.schedule_strategy)) % 1000 for k, e in enumerate(p.entries))
        rec[i]["reward"] = (h % 997) / 97.0
        rec[i]["mean_ler"] = (h % 31) / 10.0
        rec[i]["latency"] = 1e6 + h
    return rec


def test_search_space_domains():
    g = fixtures.resnet18()
    seq = ga.search_space(g, "sequence")
    assert len(seq) == 24
    assert all(set(d) == set(ga.SEQ_GENES) for d in seq)
    assert all(d["deepen"] in ((0,), (0, 1)) and d["skip"] == (0, 1) for d in seq)
    assert seq[1]["branching"] == ("none",)            # MaxPool layer cannot branch
    assert "in4" not in seq[0]["branching"]            # stem conv: 3 input channels
    dim = ga.search_space(g, "dimension")
    assert all("branching" not in d for d in dim)       # dimension domains never branch
    # a conv whose output feeds a residual Add through BN only is not widenable
    assert any(d["widen_factor"] == (1.0,) for d in dim)
    # j=6 -> no out4
    from paper_2107_09789_b200.ir import Graph, Node, OperatorKind, TensorShape
    w = np.zeros((1, 1, 4, 6), np.float32)
    tiny = Graph({0: Node(0, OperatorKind.Conv2D, {"k1": 1, "k2": 1, "c": 4, "j": 6, "stride": 1, "padding": 0}, w, []),
                  1: Node(1, OperatorKind.ReLU, {}, None, [0])}, 1, TensorShape(1, 4, 2, 2))
    br = ga.search_space(tiny, "sequence")[0]["branching"]
    assert "out2" in br and "out4" not in br and "in4" in br


def test_all_random_plans_apply():
    g = fixtures.resnet18()
    for mode in ("sequence", "dimension"):
        space = ga.search_space(g, mode)
        sizes = ga.domain_sizes(mode, space)
        rng = np.random.default_rng(0)
        for genome in ga.random_genomes(rng, sizes, 6):
            knobs.apply_plan(g, ga.decode_genome(g, mode, space, genome))


def test_run_ga_contract():
    g = fixtures.c1c2()
    params = ga.GaParams(population=8, generations=6, seed=3)
    r1 = ga.run_ga(g, "dimension", 0.02, params, fake_eval)
    r2 = ga.run_ga(g, "dimension", 0.02, params, fake_eval)
    assert np.array_equal(r1.best_genome, r2.best_genome) and r1.best_reward == r2.best_reward  # determinism
    best_so_far = -1.0
    for gen in range(params.generations + 1):
        rs = [r for (gg, _, r, _, _) in r1.log if gg == gen]
        assert len(rs) == params.population               # population restored every generation
        best_so_far = max(best_so_far, max(rs))
    assert r1.best_reward == best_so_far                  # argmax ever seen
    space = ga.search_space(g, "dimension")
    sizes = ga.domain_sizes("dimension", space)
    assert np.all(r1.best_genome >= 0) and np.all(r1.best_genome < sizes)   # domain closure


def test_generation_zero_is_best_of_initial():
    g = fixtures.c1c2()
    r = ga.run_ga(g, "dimension", 0.02, ga.GaParams(population=4, generations=0, seed=1), fake_eval)
    assert r.best_reward == max(x[2] for x in r.log)


def test_mutation_clips_to_domain():
    rng = np.random.default_rng(0)
    sizes = np.array([5, 4, 2, 2] * 6)
    pop = ga.random_genomes(rng, sizes, 8)
    kids = ga.next_generation(rng, pop, np.arange(8.0), sizes, sigma=8.0, params=ga.GaParams(population=8))
    assert kids.shape == pop.shape
    assert np.all(kids >= 0) and np.all(kids <= sizes - 1)


def test_eq10_known_answers():
    assert eq10(2.0, 102.0, 100.0, 0.02) == 40.0   # T = (1+B) T*
    assert abs(eq10(2.0, 150.0, 100.0, 0.0) - 2.0 / 0.3) < 1e-12
    assert eq10(0.0, 77.0, 100.0, 0.02) == 0.0
    assert FR.eq10([2.0], 102.0, True, 100.0, 0.02)[0] == 40.0


@pytest.mark.parametrize("a,b,d", [([1, 2, 3], [1, 2, 3], 0), ([], [1, 2], 2), ([1, 2, 3], [1, 3], 1),
                                   ([1, 1, 1, 1], [], 4), ([4, 3, 2, 1], [1, 2, 3, 4], 4)])
def test_levenshtein_oracle(a, b, d):
    assert FR.levenshtein(a, b) == d


def test_ler_paper_example():
    # ED = 44 with |L*| = 18 -> 2.44
    assert round(44 / 18, 2) == 2.44
    truth = [1] * 18
    pred = [2] * 18 + [3] * 26
    assert FR.levenshtein(pred, truth) == 44
    assert abs(FR.ler(pred, truth) - 2.4444444444444446) < 1e-15


def test_checkpoint_resume_is_bit_identical():
    """A GaState pickled after generation k and resumed gives exactly the
    uninterrupted run (RNG state, population, log): what the CLI's
    --resume relies on."""
    import pickle
    g = fixtures.c1c2()
    params = ga.GaParams(population=8, generations=5, seed=11)
    ref = ga.run_ga(g, "dimension", 0.02, params, fake_eval)
    st = ga.ga_init(g, "dimension", params, fake_eval)
    for _ in range(2):
        st = ga.ga_step(g, st, fake_eval)
    st = pickle.loads(pickle.dumps(st))
    while st.gen < params.generations:
        st = ga.ga_step(g, st, fake_eval)
    res = ga.ga_result(g, st)
    assert res.best_reward == ref.best_reward
    assert np.array_equal(res.best_genome, ref.best_genome)
    assert res.log == ref.log

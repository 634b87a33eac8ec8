"""Dimension attacker (dimattack.py): the flat
forest export and the CPU oracle reproduce scikit-learn's
RandomForestRegressor.predict exactly; DER known answers."""

import numpy as np
import pytest

from oracle import forest_ref
from paper_2107_09789_b200 import dimattack
from paper_2107_09789_b200.dimattack import Forest, der


def _arrays(f: Forest):
    return f.feature, f.threshold, f.left, f.right, f.value, f.roots


def random_forest(seed: int, trees: int = 7, n: int = 400, feats: int = 9):
    from sklearn.ensemble import RandomForestRegressor
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, feats)) * 10.0 ** rng.integers(0, 6, feats)
    y = np.abs(x[:, 0] / 3 + x[:, 1] % 7) + rng.integers(1, 512, n)
    rf = RandomForestRegressor(n_estimators=trees, max_depth=dimattack.MAX_DEPTH, random_state=seed, n_jobs=1)
    rf.fit(x, y)
    return rf, x


def test_der_known_answers():
    assert der((64, 128), (64, 128)) == 0.0
    assert der((207, 93), (64, 128)) == pytest.approx(2.5078, abs=1e-4)
    assert der((177, 91), (64, 128)) == pytest.approx(2.0547, abs=1e-4)
    assert der((225, 92), (64, 128)) == pytest.approx(2.7969, abs=1e-4)
    assert der((64, 64), (100, 64)) != der((100, 64), (64, 64))           # not symmetric
    with pytest.raises(dimattack.ZeroTruth):
        der((1, 1), (0, 5))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oracle_matches_sklearn(seed):
    rf, x = random_forest(seed)
    f = Forest.from_sklearn(rf)
    rng = np.random.default_rng(seed + 10)
    probe = np.concatenate([x[:50], rng.standard_normal((50, x.shape[1])) * 1e3])
    want = rf.predict(probe)
    got = np.array([forest_ref.forest_mean(_arrays(f), row) for row in probe])
    assert np.array_equal(got, want)  # same sum order, same float32 comparisons: bit-exact
    reg = dimattack.DimRegressor(f, f)
    hp = dimattack.host_predict(reg, probe)
    assert hp[:, 0].tolist() == [forest_ref.forest_round(v) for v in want]


def test_regressor_save_load(tmp_path):
    rf, _ = random_forest(3, trees=3)
    f = Forest.from_sklearn(rf)
    regs = [dimattack.DimRegressor(f, f), dimattack.DimRegressor(f, f)]
    dimattack.save_dim_regressors(tmp_path / "d.npz", regs)
    back = dimattack.load_dim_regressors(tmp_path / "d.npz")
    assert len(back) == 2 and back[1].trees == 3
    for a, b in zip(_arrays(f), _arrays(back[0].j)):
        assert np.array_equal(a, b) and a.dtype == b.dtype


def test_candidate_der_oracle():
    rf, x = random_forest(4, trees=5)
    f = _arrays(Forest.from_sklearn(rf))
    truth = [(64, 128), (128, 128)]
    preds, d = forest_ref.candidate_der(f, f, x[:2], truth)
    assert d == pytest.approx(np.mean([der(p, t) for p, t in zip(preds, truth)]), rel=1e-15)
    assert forest_ref.candidate_der(f, f, x[:3], truth)[1] == -1.0

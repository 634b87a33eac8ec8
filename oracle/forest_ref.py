"""CPU oracle of the dimension attacker (TEST INFRASTRUCTURE ONLY: imported by
tests/, never by the product path).

Restates SPEC.md:496-504 (predict_dims, der) for flat CART forests in the
sklearn node layout: a forest's prediction is its trees' leaf values summed in
tree order (fp64) over the tree count — sklearn
RandomForestRegressor.predict with n_jobs=1 (scikit-learn 1.x,
sklearn/ensemble/_forest.py ``_accumulate_prediction`` then ``/=
len(estimators_)``), features compared after the float32 cast sklearn's
predict applies — rounded to the nearest positive integer. Pinned against
sklearn itself in tests/test_cpu_dimattack.py. Plain Python loops: small cases.
"""

from __future__ import annotations

import math

import numpy as np


def tree_leaf(feature, threshold, left, right, root: int, x) -> int:
    n = root
    while left[n] >= 0:
        v = float(np.float32(x[feature[n]]))
        n = left[n] if v <= threshold[n] else right[n]
    return n


def forest_mean(f, x) -> float:
    """f: (feature, threshold, left, right, value, roots)."""
    feature, threshold, left, right, value, roots = f
    s = 0.0
    for r in roots:
        s += float(value[tree_leaf(feature, threshold, left, right, int(r), x)])
    return s / len(roots)


def forest_round(mean: float) -> int:
    return int(max(1.0, math.floor(mean + 0.5)))


def candidate_der(fc, fj, rows, truth) -> tuple[list[tuple[int, int]], float]:
    """Predictions for a candidate's conv-step feature rows and its DER: mean
    over layers of |c-c*|/c* + |j-j*|/j*, summed in layer order; -1.0 when the
    step count differs from the layer count."""
    if len(rows) != len(truth):
        return [], -1.0
    preds = [(forest_round(forest_mean(fc, x)), forest_round(forest_mean(fj, x))) for x in rows]
    s = 0.0
    for (c, j), (c0, j0) in zip(preds, truth):
        s += abs(float(c) - c0) / c0 + abs(float(j) - j0) / j0
    return preds, s / len(truth)

"""Dimension attacker: bagged random-forest (c, j) regressors and DER
(PAPER §V-B). No reference code exists; the SPEC
fixes the model family (bagged CART regression trees, max depth 12, one forest
for c and one for j, ensembles of 30/50/100/200 trees) and the metric
DER = |c - c*|/c* + |j - j*|/j* (eq:DER), averaged over the conv layers.

Training runs on the host with scikit-learn (offline, like train-attacker);
inference runs on the device (``tobf_forest_der``, csrc/forest.cu) over the
trace features the trace stage left in HBM. The GA's dimension mode maximises
the bagged mean DER in Eq. 10 when an Evaluator carries ``dim_regressors``.

Deviations, documented: features are the raw cost-model rows (no min-max
normalisation — trees are invariant to it and the float32 cast sklearn applies
is reproduced exactly); a channel count observed as both a producer's j and
its consumer's c is predicted twice, not averaged (SPEC §VI-B note).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from .engine import device

DIM_TREES = (30, 50, 100, 200)
MAX_DEPTH = 12                  # SPEC.md DESIGN DECISIONS (CART)


class ZeroTruth(ValueError):
    """DER against a zero true dimension."""


def der(pred: tuple[int, int], truth: tuple[int, int]) -> float:
    """eq:DER for one layer: |c - c*|/c* + |j - j*|/j* (SPEC.md:496-504)."""
    (c, j), (c0, j0) = pred, truth
    if c0 < 1 or j0 < 1:
        raise ZeroTruth(f"true dimensions {truth} must be >= 1")
    return abs(c - c0) / c0 + abs(j - j0) / j0


@dataclass
class Forest:
    """Flat CART node tables of one forest (sklearn layout: leaves have
    left < 0); trees start at ``roots``."""

    feature: np.ndarray    # int32
    threshold: np.ndarray  # float64
    left: np.ndarray       # int32
    right: np.ndarray      # int32
    value: np.ndarray      # float64
    roots: np.ndarray      # int32

    @classmethod
    def from_sklearn(cls, rf) -> "Forest":
        feat, thr, lef, rig, val, roots = [], [], [], [], [], []
        base = 0
        for est in rf.estimators_:
            t = est.tree_
            n = t.node_count
            roots.append(base)
            feat.append(np.where(t.children_left >= 0, t.feature, 0).astype(np.int32))
            thr.append(t.threshold.astype(np.float64))
            lef.append(np.where(t.children_left >= 0, t.children_left + base, -1).astype(np.int32))
            rig.append(np.where(t.children_right >= 0, t.children_right + base, -1).astype(np.int32))
            val.append(t.value.reshape(n, -1)[:, 0].astype(np.float64))
            base += n
        return cls(np.concatenate(feat), np.concatenate(thr), np.concatenate(lef), np.concatenate(rig),
                   np.concatenate(val), np.asarray(roots, np.int32))

    @property
    def trees(self) -> int:
        return len(self.roots)


@dataclass
class DimRegressor:
    """One bagged member: a forest for c and a forest for j."""

    c: Forest
    j: Forest

    @property
    def trees(self) -> int:
        return self.c.trees


def conv_truth(graph, analysis=None, pname: str = "default") -> np.ndarray:
    """(c*, j*) of the graph's Conv2D kernels in trace order (n_layers, 2)."""
    from .ir import OperatorKind as K
    from .trace import trace_records
    _, kernels, _ = trace_records(graph, None, None, pname, analysis)
    rows = [(graph.nodes[k.anchor].attrs["c"], graph.nodes[k.anchor].attrs["j"]) for k in kernels
            if graph.nodes[k.anchor].kind is K.Conv2D]
    return np.asarray(rows, np.int32).reshape(-1, 2)


# ---------------------------------------------------------------- training
def conv_steps(ds) -> tuple[np.ndarray, np.ndarray]:
    """Feature rows and (c, j) targets of a TraceDataset's Conv2D steps."""
    sel = ds.step_labels == 1
    return ds.feats[sel], ds.step_cj[sel]


def train_dim_regressors(ds, trees=DIM_TREES, seed: int = 0, val_fraction: float = 0.2):
    """Fit one (c, j) forest pair per tree count on the training networks
    (4:1 split by network, PAPER §V-A); returns (regressors, validation mean
    DER per regressor over the held-out networks' conv steps)."""
    from sklearn.ensemble import RandomForestRegressor
    n = len(ds.offsets) - 1
    rng = np.random.default_rng(seed)
    order = rng.permutation(n)
    n_val = max(1, int(round(val_fraction * n)))
    is_val = np.zeros(len(ds.feats), bool)
    for i in order[:n_val]:
        is_val[ds.offsets[i]:ds.offsets[i + 1]] = True
    conv = ds.step_labels == 1
    xtr, ytr = ds.feats[conv & ~is_val], ds.step_cj[conv & ~is_val]
    xva, yva = ds.feats[conv & is_val], ds.step_cj[conv & is_val]
    regs, vals = [], []
    for k, t in enumerate(trees):
        pair = []
        for col in (0, 1):
            rf = RandomForestRegressor(n_estimators=t, max_depth=MAX_DEPTH, random_state=seed * 1000 + 10 * k + col,
                                       n_jobs=1)
            rf.fit(xtr, ytr[:, col])
            pair.append(Forest.from_sklearn(rf))
        reg = DimRegressor(*pair)
        regs.append(reg)
        if len(xva):
            p = host_predict(reg, xva)
            vals.append(float(np.mean(np.abs(p[:, 0] - yva[:, 0]) / yva[:, 0] + np.abs(p[:, 1] - yva[:, 1]) / yva[:, 1])))
    return regs, vals


def host_predict(reg: DimRegressor, x: np.ndarray) -> np.ndarray:
    """(c, j) predictions of rows ``x`` (validation only; the GA path runs on
    the device). Same traversal and rounding as the kernel."""
    out = np.zeros((len(x), 2), np.int32)
    xf = x.astype(np.float32).astype(np.float64)
    for col, f in enumerate((reg.c, reg.j)):
        s = np.zeros(len(x))
        for r in f.roots:
            node = np.full(len(x), r, np.int64)
            live = f.left[node] >= 0
            while live.any():
                nd = node[live]
                go_left = xf[live, f.feature[nd]] <= f.threshold[nd]
                node[live] = np.where(go_left, f.left[nd], f.right[nd])
                live = f.left[node] >= 0
            s += f.value[node]
        out[:, col] = np.maximum(1.0, np.floor(s / f.trees + 0.5))
    return out


def save_dim_regressors(path, regs: list[DimRegressor]) -> None:
    arrs = {}
    for i, r in enumerate(regs):
        for tgt, f in (("c", r.c), ("j", r.j)):
            for k, v in f.__dict__.items():
                arrs[f"r{i}_{tgt}_{k}"] = v
    np.savez(path, n=np.int32(len(regs)), **arrs)


def load_dim_regressors(path) -> list[DimRegressor]:
    z = np.load(path)
    fields = ("feature", "threshold", "left", "right", "value", "roots")
    return [DimRegressor(*(Forest(*(z[f"r{i}_{t}_{k}"] for k in fields)) for t in ("c", "j")))
            for i in range(int(z["n"]))]


# ---------------------------------------------------------------- device
class DeviceForests:
    """All regressors' node tables concatenated in HBM (forest 2r = c of
    regressor r, 2r + 1 = its j), uploaded once."""

    def __init__(self, regs: list[DimRegressor]):
        ctx = device()
        forests = [f for r in regs for f in (r.c, r.j)]
        nbase, tbase = 0, 0
        cols = {k: [] for k in ("feature", "threshold", "left", "right", "value")}
        roots, foff = [], [0]
        for f in forests:
            for k in ("feature", "threshold", "value"):
                cols[k].append(getattr(f, k))
            for k in ("left", "right"):
                a = getattr(f, k)
                cols[k].append(np.where(a >= 0, a + nbase, -1).astype(np.int32))
            roots.append(f.roots + nbase)
            nbase += len(f.feature)
            tbase += f.trees
            foff.append(tbase)
        up = ctx.upload_array
        self.feature = up(np.concatenate(cols["feature"]).astype(np.int32))
        self.threshold = up(np.concatenate(cols["threshold"]).astype(np.float64))
        self.left = up(np.concatenate(cols["left"]))
        self.right = up(np.concatenate(cols["right"]))
        self.value = up(np.concatenate(cols["value"]).astype(np.float64))
        self.roots = up(np.concatenate(roots).astype(np.int32))
        self.forest_off = up(np.asarray(foff, np.int32))
        self.R = len(regs)


def forest_der(forests: DeviceForests, feats: torch.Tensor, conv_rows: torch.Tensor, conv_off: torch.Tensor,
               ncand: int, truth: torch.Tensor, stream: int | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """Device predictions (R, ncand, n_layers, 2) int32 and DER (R, ncand)
    float64 (-1 where a candidate's conv steps do not line up)."""
    ctx = device()
    n_layers = truth.shape[0]
    pred = torch.empty((forests.R, ncand, n_layers, 2), dtype=torch.int32, device=ctx.device)
    out = torch.empty((forests.R, ncand), dtype=torch.float64, device=ctx.device)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    ctx.check(ctx.lib.tobf_forest_der(p(feats), feats.shape[1], p(conv_rows), p(conv_off), ncand, n_layers, p(truth),
                                      p(forests.feature), p(forests.threshold), p(forests.left), p(forests.right),
                                      p(forests.value), p(forests.roots), p(forests.forest_off), forests.R, p(pred),
                                      p(out), C.c_void_p(ctx.sp if stream is None else stream)), "forest der")
    ctx.launches += 2
    return pred, out


__all__ = ["DIM_TREES", "ZeroTruth", "der", "Forest", "DimRegressor", "conv_truth", "train_dim_regressors",
           "host_predict", "save_dim_regressors", "load_dim_regressors", "DeviceForests", "forest_der"]

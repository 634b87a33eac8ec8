"""Restated CPU executor (oracle) — follows interpreter.py:22-118.

Operates on any graph object with ``nodes`` (id -> node with .kind.value,
.attrs, .weights, .inputs), ``output_id`` and ``input_shape`` — reference
graphs and engine graphs alike. float32 throughout, like the reference.
"""

from __future__ import annotations

import numpy as np

BN_EPS = 1e-5  # graph.py:17


def _order(graph) -> list[int]:
    """Kahn order, smallest ready id first (graph.py:149-171)."""
    import heapq
    indeg = {nid: sum(1 for p in n.inputs if p in graph.nodes) for nid, n in graph.nodes.items()}
    cons: dict[int, list[int]] = {nid: [] for nid in graph.nodes}
    for n in graph.nodes.values():
        for p in set(n.inputs):
            if p in cons:
                cons[p].append(n.id)
    ready = [nid for nid, d in indeg.items() if d == 0]
    heapq.heapify(ready)
    out = []
    while ready:
        nid = heapq.heappop(ready)
        out.append(nid)
        for s in cons[nid]:
            indeg[s] -= 1
            if indeg[s] == 0:
                heapq.heappush(ready, s)
    return out


def conv2d(x: np.ndarray, w: np.ndarray, stride: int, padding: int) -> np.ndarray:
    """interpreter.py:22-30: zero-padded direct convolution, (k1,k2,c,j) kernel,
    as one GEMM over K = (u, v, c) in x's dtype (float32 = the reference's)."""
    k1, k2, c, j = w.shape
    dt = x.dtype
    b, _, h, wd = x.shape
    xp = np.pad(x, ((0, 0), (0, 0), (padding, padding), (padding, padding))) if padding else x
    ho = (h + 2 * padding - k1) // stride + 1
    wo = (wd + 2 * padding - k2) // stride + 1
    cols = np.empty((b, ho, wo, k1, k2, c), dtype=dt)
    for u in range(k1):
        for v in range(k2):
            patch = xp[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride]
            cols[:, :, :, u, v, :] = patch.transpose(0, 2, 3, 1)
    y = cols.reshape(b * ho * wo, k1 * k2 * c) @ w.reshape(k1 * k2 * c, j).astype(dt)
    return y.reshape(b, ho, wo, j).transpose(0, 3, 1, 2).astype(dt)


def maxpool(x: np.ndarray, window: int, stride: int) -> np.ndarray:
    """interpreter.py:33-35 (no padding, floor)."""
    b, c, h, w = x.shape
    ho = (h - window) // stride + 1
    wo = (w - window) // stride + 1
    out = np.full((b, c, ho, wo), -np.inf, dtype=x.dtype)
    for u in range(window):
        for v in range(window):
            out = np.maximum(out, x[:, :, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride])
    return out


def softmax(x: np.ndarray) -> np.ndarray:
    """interpreter.py:38-41 (over channels)."""
    e = np.exp(x - x.max(axis=1, keepdims=True))
    return (e / e.sum(axis=1, keepdims=True)).astype(x.dtype)


def eval_node(node, ins: list[np.ndarray]) -> np.ndarray:
    """interpreter.py:44-72 (dtype follows the inputs: float32 like the
    reference, or float64 for an exact-arithmetic yardstick)."""
    kind, a = node.kind.value, node.attrs
    dt = ins[0].dtype
    if kind == "Conv2D":
        return conv2d(ins[0], node.weights, a["stride"], a["padding"])
    if kind == "Linear":
        flat = ins[0].reshape(ins[0].shape[0], -1)
        y = flat @ node.weights.astype(dt)
        return y.reshape(y.shape[0], y.shape[1], 1, 1).astype(dt)
    if kind == "ReLU":
        return np.maximum(ins[0], 0.0)
    if kind == "BatchNorm":
        sc, sh, mu, var = (node.weights[i].astype(dt).reshape(1, -1, 1, 1) for i in range(4))
        return ((ins[0] - mu) / np.sqrt(var + BN_EPS) * sc + sh).astype(dt)
    if kind == "MaxPool":
        return maxpool(ins[0], a["window"], a["stride"])
    if kind == "Add":
        acc = ins[0]
        for t in ins[1:]:
            acc = acc + t
        if node.weights is not None:
            acc = acc + node.weights.astype(dt)
        return acc.astype(dt)
    if kind == "Concat":
        return np.concatenate(ins, axis=1)
    if kind == "Slice":
        return ins[0][:, a["start"]:a["stop"]]
    if kind == "SoftMax":
        return softmax(ins[0])
    raise NotImplementedError(kind)


def execute(graph, x: np.ndarray, keep: bool = False, dtype=np.float32):
    """interpreter.py:75-90. With ``keep`` returns every node's value too."""
    x = np.asarray(x, dtype=dtype)
    vals: dict[int, np.ndarray] = {}
    for nid in _order(graph):
        n = graph.nodes[nid]
        ins = [vals[p] for p in n.inputs] if n.inputs else [x]
        vals[nid] = eval_node(n, ins)
    return (vals[graph.output_id], vals) if keep else vals[graph.output_id]


def trial_inputs(shape: tuple, trials: int, seed: int) -> list[np.ndarray]:
    """interpreter.py:107-111: one default_rng(seed) stream, float32 casts."""
    rng = np.random.default_rng(seed)
    return [rng.standard_normal(shape).astype(np.float32) for _ in range(trials)]


def equivalence_check(g1, g2, trials: int = 8, seed: int = 0, tol: float = 1e-5) -> tuple[bool, float]:
    """interpreter.py:93-118: verdict |a-b| <= tol*(1+|b|) and worst |a-b|/(1+|b|),
    all in float32 (numpy weak-scalar promotion)."""
    shape = tuple(g1.input_shape.as_tuple())
    worst, ok = 0.0, True
    for x in trial_inputs(shape, trials, seed):
        a = execute(g1, x)
        b = execute(g2, x)
        d = np.abs(a - b)
        den = 1.0 + np.abs(b)
        worst = max(worst, float((d / den).max()))
        ok = ok and bool(np.all(d <= tol * den))
    return ok, worst

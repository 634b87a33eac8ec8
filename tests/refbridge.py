"""Bridge to the real reference package (only where /root/reference exists).

Used by tests/golden/make_golden.py (in the build container) and by the
`reference`-marked CPU tests; never by the GPU box (the reference is not
shipped there).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")


def available() -> bool:
    return (REF_SRC / "traceobf" / "__init__.py").exists()


def ref():
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import traceobf  # noqa: PLC0415
    return traceobf


def to_ref(g):
    R = ref()
    nodes = {nid: R.Node(n.id, R.OperatorKind(n.kind.value), dict(n.attrs), n.weights, list(n.inputs))
             for nid, n in g.nodes.items()}
    return R.Graph(nodes, g.output_id, R.TensorShape(*g.input_shape.as_tuple()))


def plan_ref(p):
    R = ref()
    return R.ObfuscationPlan(p.mode, tuple(R.PlanEntry(**e.__dict__) for e in p.entries))


def graph_diff(a, b) -> str | None:
    """None when two graphs (engine or reference objects) are node-for-node equal."""
    if a.output_id != b.output_id or tuple(a.input_shape.as_tuple()) != tuple(b.input_shape.as_tuple()):
        return "output/input differ"
    if set(a.nodes) != set(b.nodes):
        return f"node ids differ: {sorted(set(a.nodes) ^ set(b.nodes))}"
    for k in a.nodes:
        x, y = a.nodes[k], b.nodes[k]
        if x.kind.value != y.kind.value or x.attrs != y.attrs or list(x.inputs) != list(y.inputs):
            return f"node {k} differs"
        if (x.weights is None) != (y.weights is None):
            return f"node {k} weight presence differs"
        if x.weights is not None and (x.weights.shape != y.weights.shape or not np.array_equal(x.weights, y.weights)):
            return f"node {k} weights differ"
    return None

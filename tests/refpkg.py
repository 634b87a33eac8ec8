"""Locate and import the UNMODIFIED reference package (traceobf 0.1.0) for
the drop-in tests: baseline/_ref (vendored by scripts/vendor_reference.sh;
travels to the GPU box) first, else the read-only source tree in this
container. Returns None when neither is present."""

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CANDIDATES = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def load():
    for p in CANDIDATES:
        if (p / "traceobf" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            return importlib.import_module("traceobf")
    return None


def ref_graph(ref, g):
    """An engine fixture graph rebuilt in the reference's own classes."""
    nodes = {nid: ref.Node(n.id, ref.OperatorKind(n.kind.value), dict(n.attrs), n.weights, list(n.inputs))
             for nid, n in g.nodes.items()}
    s = g.input_shape
    return ref.Graph(nodes, g.output_id, ref.TensorShape(s.batch, s.channels, s.height, s.width))


def ref_plan(ref, plan):
    return ref.ObfuscationPlan(plan.mode, tuple(ref.PlanEntry(**vars(e)) for e in plan.entries))

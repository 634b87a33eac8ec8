"""On-disk formats shared with the reference: graphs, plans, traces.

Files written here load in the reference and vice versa, byte for byte:

* graph (``graph.py:341-449``): a ``graph v1`` text file, one ``node`` record per
  node in id order, plus a ``.weights`` sidecar = 8-byte magic + little-endian
  float32 blobs concatenated in node-id order, referenced as ``w@<float
  offset>:<d0>x<d1>...``;
* plan (``transforms.py:477-507``): ``plan v1 mode=<mode>``, a header row, one
  whitespace-separated row per entry;
* trace (``costmodel.py:296-328``): comma-separated, the case's feature columns
  (``repr`` of the fp64 value) plus an optional ``label`` column; the case is
  recovered from the column set. As in the reference the round trip drops
  ``anchor_id`` and the masked features (App. A-11): compare traces in memory.

Knob-derived weights (derived.py) are materialised on dump.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from .ir import Graph, Node, OperatorKind, TensorShape
from .knobs import ObfuscationPlan, PlanEntry
from .trace import LeakageCase, Trace, TraceStep

WEIGHT_MAGIC = b"OBFW0001"

#: attribute keys parsed back as int (every other attribute stays a string)
INT_ATTRS = frozenset(("k1", "k2", "c", "j", "stride", "padding", "window", "axis", "start", "stop"))

#: plan columns in file order, with their parsers
PLAN_COLUMNS = (("layer_id", int), ("branching", str), ("deepen", int), ("skip", int),
                ("widen_factor", float), ("kernel_widen", int), ("dummy_count", int),
                ("fusion_limit", int), ("schedule_strategy", int))


class GraphParseError(Exception):
    """Malformed graph file; carries the 1-based line number (graph.py:391-394)."""

    def __init__(self, path, lineno: int, message: str):
        super().__init__(f"{path}:{lineno}: {message}")
        self.lineno = lineno


# ---------------------------------------------------------------------- graph
def _attrs_text(attrs: dict) -> str:
    return ",".join(f"{k}={attrs[k]}" for k in sorted(attrs))


def _attrs_parse(text: str) -> dict:
    out = {}
    for item in filter(None, text.split(",")):
        k, v = item.split("=", 1)
        out[k] = int(v) if k in INT_ATTRS else v
    return out


def dump_graph(graph: Graph, path: str | Path) -> None:
    """Write ``path`` and its ``.weights`` sidecar (graph.py:362-388)."""
    path = Path(path)
    side = path.with_suffix(".weights")
    shape = " ".join(str(d) for d in graph.input_shape.as_tuple())
    records = ["graph v1", f"input_shape {shape}", f"output {graph.output_id}", f"weights_file {side.name}"]
    blobs, at = [], 0
    for nid in sorted(graph.nodes):
        n = graph.nodes[nid]
        wref = "-"
        if n.weights is not None:
            blob = np.ascontiguousarray(np.asarray(n.weights), dtype="<f4")
            wref = f"w@{at}:" + "x".join(str(d) for d in blob.shape)
            blobs.append(blob)
            at += blob.size
        ins = ",".join(str(i) for i in n.inputs) or "-"
        records.append(f"node {nid} {n.kind.value} inputs={ins} attrs={_attrs_text(n.attrs)} weights={wref}")
    path.write_text("\n".join(records) + "\n")
    with open(side, "wb") as f:
        f.write(WEIGHT_MAGIC)
        for blob in blobs:
            f.write(memoryview(blob).cast("B"))


def load_graph(path: str | Path) -> Graph:
    """Parse a ``graph v1`` file (graph.py:397-449); errors raise
    GraphParseError with the offending line."""
    path = Path(path)
    lines = path.read_text().splitlines()
    if not lines or lines[0].strip() != "graph v1":
        raise GraphParseError(path, 1, "expected 'graph v1' header")
    header: dict = {}
    nodes: dict[int, Node] = {}
    wrefs: list[tuple[int, str]] = []
    for lineno, raw in enumerate(lines[1:], start=2):
        tok = raw.split()
        if not tok or tok[0].startswith("#"):
            continue
        try:
            rec = tok[0]
            if rec == "input_shape":
                header["shape"] = TensorShape(*(int(t) for t in tok[1:5]))
            elif rec == "output":
                header["output"] = int(tok[1])
            elif rec == "weights_file":
                header["weights"] = tok[1]
            elif rec == "node":
                nid = int(tok[1])
                kv = dict(t.split("=", 1) for t in tok[3:])
                ins = [] if kv["inputs"] == "-" else [int(t) for t in kv["inputs"].split(",")]
                nodes[nid] = Node(nid, OperatorKind(tok[2]), _attrs_parse(kv.get("attrs", "")), None, ins)
                if kv["weights"] != "-":
                    wrefs.append((nid, kv["weights"]))
            else:
                raise ValueError(f"unknown record '{rec}'")
        except (ValueError, KeyError, IndexError) as e:
            raise GraphParseError(path, lineno, str(e)) from e
    if "shape" not in header or "output" not in header:
        raise GraphParseError(path, len(lines), "missing input_shape or output record")
    if wrefs:
        if "weights" not in header:
            raise GraphParseError(path, 1, "weight references without weights_file record")
        raw = (path.parent / header["weights"]).read_bytes()
        if raw[:8] != WEIGHT_MAGIC:
            raise GraphParseError(path, 1, f"bad weight sidecar magic {raw[:8]!r}")
        flat = np.frombuffer(raw, dtype="<f4", offset=8)
        for nid, ref in wrefs:
            off, dims = ref[2:].split(":")
            shp = tuple(int(d) for d in dims.split("x"))
            lo = int(off)
            nodes[nid].weights = flat[lo:lo + int(np.prod(shp))].reshape(shp).astype(np.float32)
    return Graph(nodes, header["output"], header["shape"])


# ----------------------------------------------------------------------- plan
def dump_plan(plan: ObfuscationPlan, path: str | Path) -> None:
    """transforms.py:485-489."""
    rows = [f"plan v1 mode={plan.mode}", " ".join(c for c, _ in PLAN_COLUMNS)]
    rows += [" ".join(str(getattr(e, c)) for c, _ in PLAN_COLUMNS) for e in plan.entries]
    Path(path).write_text("\n".join(rows) + "\n")


def load_plan(path: str | Path) -> ObfuscationPlan:
    """transforms.py:492-507; the second line is the column header."""
    lines = Path(path).read_text().splitlines()
    if not lines or not lines[0].startswith("plan v1 mode="):
        raise ValueError(f"{path}: expected 'plan v1 mode=...' header")
    entries = []
    for raw in lines[2:]:
        vals = raw.split()
        if vals:
            entries.append(PlanEntry(**{c: conv(v) for (c, conv), v in zip(PLAN_COLUMNS, vals)}))
    return ObfuscationPlan(lines[0].split("mode=", 1)[1], tuple(entries))


# ---------------------------------------------------------------------- trace
def dump_trace(trace: Trace, path: str | Path, include_labels: bool = False) -> None:
    """costmodel.py:300-309: case-masked columns, ``repr`` floats."""
    cols = list(trace.case.features)
    rows = [",".join(cols + ["label"] * include_labels)]
    for st in trace.steps:
        vals = [repr(getattr(st, c)) for c in cols]
        if include_labels:
            vals.append("-" if st.label is None else st.label.value)
        rows.append(",".join(vals))
    Path(path).write_text("\n".join(rows) + "\n")


def load_trace(path: str | Path) -> Trace:
    """costmodel.py:312-328: the leakage case is the one whose feature list
    equals the file's columns; labels when the last column is ``label``."""
    lines = Path(path).read_text().splitlines()
    cols = lines[0].split(",")
    labelled = bool(cols) and cols[-1] == "label"
    feats = cols[:-1] if labelled else cols
    case = next(c for c in LeakageCase if list(c.features) == feats)
    steps = []
    for raw in lines[1:]:
        if not raw.strip():
            continue
        parts = raw.split(",")
        vals = {c: float(v) for c, v in zip(feats, parts)}
        lab = OperatorKind(parts[-1]) if labelled and parts[-1] != "-" else None
        steps.append(TraceStep(label=lab, **vals))
    return Trace(tuple(steps), case)

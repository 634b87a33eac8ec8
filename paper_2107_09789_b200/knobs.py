"""The six function-preserving obfuscation knobs and ``apply_plan``.

Host-side mirror of traceobf.transforms (reference
pkg/src/traceobf/transforms.py): same names, argument meaning, node-id
allocation, weight arithmetic and exception types, so the obfuscated graphs
are node-for-node equal (``Graph.__eq__``) to the reference's.

The single-knob entry points (``widen_layer`` … ``widen_kernel``) return new
graphs and never mutate their input, as in the reference. ``apply_plan``
runs the same fixed knob order on one private working copy with an
incrementally maintained successor index and shape table, instead of the
reference's copy + full re-inference per knob (its O(N^2) host floor,
SURVEY §3.1); every knob validates before it mutates, so a failing knob
leaves the working graph untouched exactly like the reference's
copy-on-write knobs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .derived import DerivedWeight
from .ir import (COMPLEX_KINDS, Graph, Node, OperatorKind, TensorShape, analyze, shape_map, topo_order)

BRANCH_MODES = ("none", "in2", "in4", "out2", "out4")            # transforms.py:19
WIDEN_FACTORS = (1.0, 1.0625, 1.125, 1.25, 1.5)                  # transforms.py:20

# Ops a widening pass walks through to find the consumer layer (transforms.py:23-25).
_WIDEN_WALK = frozenset({OperatorKind.ReLU, OperatorKind.BatchNorm, OperatorKind.MaxPool, OperatorKind.Add})
_LAYER_KINDS = (OperatorKind.Conv2D, OperatorKind.Linear)


class TransformError(Exception):
    """transforms.py:28-29."""


class NotWidenable(TransformError):
    pass


class NotDivisible(TransformError):
    pass


class NoActivation(TransformError):
    pass


def _round_half_up(x: float) -> int:
    """transforms.py:44-45: floor(x + 0.5)."""
    return int(math.floor(x + 0.5))


# ---------------------------------------------------------------------------
# Working state: a graph plus its successor index and (lazily) shapes.
# ---------------------------------------------------------------------------

class _Work:
    """Mutable view used by the knobs. ``nodes`` are private copies."""

    def __init__(self, graph: Graph, own: bool = False, analysis=None, lazy: bool = False):
        self.g = graph if own else graph.copy()
        # lazy: Conv2D / Linear weights the knobs change become DerivedWeights
        # (derived.py: per-axis gathers of the vanilla array, packed on the
        # device) instead of materialised numpy arrays
        self.lazy = lazy
        if analysis is not None:  # reuse the input graph's structure (copied: we mutate)
            self.succ = {k: list(v) for k, v in analysis.succ.items()}
            self._shapes: dict[int, TensorShape] | None = dict(analysis.shapes)
        else:
            self.succ = self.g.successor_index()
            self._shapes = None

    # -- structure ----------------------------------------------------------
    def sole_successor(self, nid: int) -> int | None:
        s = self.succ.get(nid, [])
        return s[0] if len(s) == 1 else None

    def activation_site(self, nid: int) -> int | None:
        """Follow BatchNorm links to the trailing ReLU (transforms.py:63-75)."""
        cur = nid
        while True:
            nxt = self.sole_successor(cur)
            if nxt is None:
                return None
            kind = self.g.nodes[nxt].kind
            if kind is OperatorKind.ReLU:
                return nxt
            if kind is not OperatorKind.BatchNorm:
                return None
            cur = nxt

    def add_node(self, node: Node) -> None:
        self.g.nodes[node.id] = node
        self.succ[node.id] = []
        for p in dict.fromkeys(node.inputs):
            if p in self.succ:
                self.succ[p].append(node.id)

    def remove_node(self, nid: int) -> None:
        node = self.g.nodes.pop(nid)
        for p in dict.fromkeys(node.inputs):
            if p in self.succ and nid in self.succ[p]:
                self.succ[p].remove(nid)
        self.succ.pop(nid, None)
        if self._shapes is not None:
            self._shapes.pop(nid, None)

    def rewire(self, old: int, new: int, skip: set[int]) -> None:
        """Point every consumer of ``old`` except ``skip`` (and ``new``) at ``new``
        (transforms.py:53-60)."""
        moved = [s for s in self.succ.get(old, []) if s != new and s not in skip]
        for sid in moved:
            node = self.g.nodes[sid]
            node.inputs = [new if p == old else p for p in node.inputs]
        if moved:
            # only the sizes of successor lists are ever consulted, not their order
            self.succ[old] = [s for s in self.succ[old] if s not in moved]
            self.succ[new] = list(dict.fromkeys(self.succ[new] + moved))
        if self.g.output_id == old:
            self.g.output_id = new

    def next_id(self) -> int:
        return self.g.next_id()

    # -- shapes -------------------------------------------------------------
    def shapes(self) -> dict[int, TensorShape]:
        if self._shapes is None:
            self._shapes = shape_map(self.g)
        return self._shapes

    def set_shape(self, nid: int, s: TensorShape) -> None:
        if self._shapes is not None:
            self._shapes[nid] = s

    def drop_shapes(self) -> None:
        self._shapes = None


def _derived(w: _Work, node: Node) -> DerivedWeight:
    """The node's weight as a DerivedWeight (lazy mode): a Linear's rows are
    factored (c, H, W) by the activation that feeds it."""
    if isinstance(node.weights, DerivedWeight):
        return node.weights
    if node.kind is OperatorKind.Conv2D:
        return DerivedWeight.of(node.weights, "conv")
    fed = w.shapes()[node.inputs[0]] if node.inputs else w.g.input_shape
    return DerivedWeight.of(node.weights, "linear", (fed.height, fed.width))


# ---------------------------------------------------------------------------
# Layer widening (transforms.py:82-165)
# ---------------------------------------------------------------------------

def _widen_path(w: _Work, layer_id: int) -> list[int]:
    """Nodes from the widened layer to its consumer layer, consumer included."""
    path = []
    cur = layer_id
    while True:
        nxt = w.sole_successor(cur)
        if nxt is None:
            why = "fan-out" if w.succ.get(cur) else "feeds the graph output"
            raise NotWidenable(f"layer {layer_id}: {why} before a consumer layer")
        node = w.g.nodes[nxt]
        if node.kind in _LAYER_KINDS:
            path.append(nxt)
            return path
        if node.kind not in _WIDEN_WALK:
            raise NotWidenable(f"layer {layer_id}: consumer chain hits {node.kind.value}")
        if node.kind is OperatorKind.Add and len(node.inputs) > 1:
            raise NotWidenable(f"layer {layer_id}: consumer chain hits a residual Add")
        path.append(nxt)
        cur = nxt


def widenable(graph: Graph, layer_id: int) -> bool:
    """transforms.py:104-112."""
    if graph.nodes[layer_id].kind not in _LAYER_KINDS:
        return False
    try:
        _widen_path(_Work(graph), layer_id)
    except NotWidenable:
        return False
    return True


def _widen(w: _Work, layer_id: int, factor: float) -> None:
    layer = w.g.nodes[layer_id]
    if layer.kind not in _LAYER_KINDS:
        raise NotWidenable(f"layer {layer_id} is {layer.kind.value}")
    j = layer.attrs["j"]
    j_new = _round_half_up(factor * j)
    if j_new < j:
        raise NotWidenable(f"factor {factor} would shrink the layer")
    extra = j_new - j
    if extra == 0:
        return
    shapes = w.shapes()  # the reference infers shapes here (transforms.py:128) even when unused
    path = _widen_path(w, layer_id)

    # producer: duplicates of the first `extra` output channels go at the end
    wt = layer.weights
    if w.lazy:
        layer.weights = _derived(w, layer).dup_tail(3, extra)
    else:
        layer.weights = np.concatenate([wt, wt[..., :extra]], axis=-1)
    layer.attrs["j"] = j_new
    for nid in path[:-1]:
        node = w.g.nodes[nid]
        if node.kind is OperatorKind.BatchNorm or (node.kind is OperatorKind.Add and node.weights is not None):
            node.weights = np.concatenate([node.weights, node.weights[:, :extra]], axis=1)

    consumer = w.g.nodes[path[-1]]
    cw = consumer.weights
    if w.lazy:
        consumer.weights = _derived(w, consumer).dup_tail(2, extra, 0.5)
        consumer.attrs["c"] = j_new if consumer.kind is OperatorKind.Conv2D else \
            j_new * consumer.weights.hw[0] * consumer.weights.hw[1]
    elif consumer.kind is OperatorKind.Conv2D:
        half = cw.copy()
        half[:, :, :extra, :] *= 0.5
        consumer.weights = np.concatenate([half, half[:, :, :extra, :]], axis=2)
        consumer.attrs["c"] = j_new
    else:
        fed = shapes[consumer.inputs[0]]
        hw = fed.height * fed.width
        rows = cw.reshape(j, hw, cw.shape[1]).copy()
        rows[:extra] *= 0.5
        consumer.weights = np.concatenate([rows, rows[:extra]], axis=0).reshape(j_new * hw, cw.shape[1])
        consumer.attrs["c"] = j_new * hw

    # shapes: channel count changes from the layer through the walked chain
    for nid in [layer_id] + path[:-1]:
        s = shapes[nid]
        w.set_shape(nid, TensorShape(s.batch, j_new, s.height, s.width))


def widen_layer(graph: Graph, layer_id: int, factor: float) -> Graph:
    """Grow a Conv2D/Linear to round(factor*j) outputs by duplicating its first
    channels and halve the consumer's matching rows (transforms.py:115-165)."""
    w = _Work(graph)
    layer = graph.nodes[layer_id]
    if layer.kind in _LAYER_KINDS and _round_half_up(factor * layer.attrs["j"]) == layer.attrs["j"]:
        return graph  # reference returns the input graph object itself
    _widen(w, layer_id, factor)
    return w.g


# ---------------------------------------------------------------------------
# Layer branching (transforms.py:173-231)
# ---------------------------------------------------------------------------

def _branch(w: _Work, layer_id: int, mode: str, parts: int) -> list[int]:
    if parts not in (2, 4):
        raise NotDivisible(f"parts must be 2 or 4, got {parts}")
    layer = w.g.nodes[layer_id]
    if layer.kind not in _LAYER_KINDS:
        raise TransformError(f"cannot branch {layer.kind.value}")
    is_conv = layer.kind is OperatorKind.Conv2D
    nid = w.next_id()
    new_nodes: list[Node] = []
    if mode == "output":
        j = layer.attrs["j"]
        if j % parts:
            raise NotDivisible(f"j={j} not divisible by {parts}")
        step = j // parts
        part_ids = []
        for i in range(parts):
            wt = layer.weights.slice(3, i * step, (i + 1) * step) if isinstance(layer.weights, DerivedWeight) \
                else layer.weights[..., i * step:(i + 1) * step]
            new_nodes.append(Node(nid, layer.kind, dict(layer.attrs, j=step), wt, list(layer.inputs)))
            part_ids.append(nid)
            nid += 1
        combiner = Node(nid, OperatorKind.Concat, {"axis": 1}, None, part_ids)
    elif mode == "input":
        if is_conv:
            ch, hw = layer.attrs["c"], 1
        else:
            feed = w.shapes()[layer.inputs[0]] if layer.inputs else w.g.input_shape
            ch, hw = feed.channels, feed.height * feed.width
        if ch % parts:
            raise NotDivisible(f"input channels {ch} not divisible by {parts}")
        step = ch // parts
        part_ids = []
        for i in range(parts):
            sl = Node(nid, OperatorKind.Slice, {"axis": 1, "start": i * step, "stop": (i + 1) * step},
                      None, list(layer.inputs))
            new_nodes.append(sl)
            nid += 1
            if isinstance(layer.weights, DerivedWeight):  # channel slice of the derived gather
                wt = layer.weights.slice(2, i * step, (i + 1) * step)
                attrs = dict(layer.attrs, c=step * hw)
            elif is_conv:
                wt = layer.weights[:, :, i * step:(i + 1) * step, :]
                attrs = dict(layer.attrs, c=step)
            else:
                jj = layer.attrs["j"]
                wt = layer.weights.reshape(ch, hw, jj)[i * step:(i + 1) * step].reshape(step * hw, jj)
                attrs = dict(layer.attrs, c=step * hw)
            new_nodes.append(Node(nid, layer.kind, attrs, wt, [sl.id]))
            part_ids.append(nid)
            nid += 1
        combiner = Node(nid, OperatorKind.Add, {}, None, part_ids)
    else:
        raise TransformError(f"unknown branch mode {mode!r}")

    shapes = w._shapes
    old_shape = shapes.get(layer_id) if shapes is not None else None
    for node in new_nodes:
        w.add_node(node)
    w.add_node(combiner)
    w.rewire(layer_id, combiner.id, skip=set(part_ids) | {combiner.id})
    w.remove_node(layer_id)
    if shapes is not None:
        if old_shape is None:
            w.drop_shapes()
        else:
            src = shapes[layer.inputs[0]] if layer.inputs else w.g.input_shape
            for node in new_nodes:
                if node.kind is OperatorKind.Slice:
                    a = node.attrs
                    shapes[node.id] = TensorShape(src.batch, a["stop"] - a["start"], src.height, src.width)
                elif mode == "output":
                    shapes[node.id] = TensorShape(old_shape.batch, node.attrs["j"], old_shape.height,
                                                  old_shape.width)
                else:
                    shapes[node.id] = old_shape
            shapes[combiner.id] = old_shape
    return [n.id for n in new_nodes] + [combiner.id]


def branch_layer(graph: Graph, layer_id: int, mode: str, parts: int) -> Graph:
    """Split a Conv2D/Linear into ``parts`` sub-layers: output-wise (split j,
    Concat) or input-wise (channel Slices, Add) (transforms.py:173-231)."""
    w = _Work(graph)
    _branch(w, layer_id, mode, parts)
    return w.g


# ---------------------------------------------------------------------------
# Dummy addition / deepening / skipping / kernel widening (transforms.py:238-335)
# ---------------------------------------------------------------------------

# Knob-synthesised constants (zero skip kernels, zero dummy operands, identity
# deepen kernels) depend only on their shape: one read-only array per shape is
# shared by every candidate. Values equal the reference's fresh arrays, and
# identical bases let the device weight cache upload each constant once.
_CONSTS: dict[tuple, np.ndarray] = {}


def _shared_zeros(shape: tuple) -> np.ndarray:
    key = ("zeros",) + tuple(shape)
    a = _CONSTS.get(key)
    if a is None:
        a = np.zeros(shape, dtype=np.float32)
        a.flags.writeable = False
        _CONSTS[key] = a
    return a


def _shared_identity(channels: int) -> np.ndarray:
    key = ("eye", channels)
    a = _CONSTS.get(key)
    if a is None:
        a = channel_identity_kernel(channels)
        a.flags.writeable = False
        _CONSTS[key] = a
    return a


def _insertion_point(w: _Work, layer_id: int) -> int:
    act = w.activation_site(layer_id)
    return layer_id if act is None else act


def _dummy(w: _Work, layer_id: int, count: int) -> None:
    if count <= 0:
        return
    shapes = w.shapes()
    site = _insertion_point(w, layer_id)
    s = shapes[site]
    zeros = _shared_zeros(s.as_tuple())   # one constant shared by the whole chain
    prev, made = site, []
    for _ in range(count):
        nid = w.next_id()
        w.add_node(Node(nid, OperatorKind.Add, {}, zeros, [prev]))
        w.set_shape(nid, s)
        made.append(nid)
        prev = nid
    w.rewire(site, prev, skip=set(made))


def add_dummy(graph: Graph, layer_id: int, count: int) -> Graph:
    """Chain ``count`` additions of an all-zero constant after the layer's
    activation output (transforms.py:251-269)."""
    if count <= 0:
        return graph
    w = _Work(graph)
    _dummy(w, layer_id, count)
    return w.g


def channel_identity_kernel(channels: int) -> np.ndarray:
    """1x1 identity kernel U[0,0,d,m] = (d == m) (transforms.py:272-276)."""
    k = np.zeros((1, 1, channels, channels), dtype=np.float32)
    k[0, 0] = np.eye(channels, dtype=np.float32)
    return k


def _deepen(w: _Work, layer_id: int, kernel_init) -> None:
    act = w.activation_site(layer_id)
    if act is None:
        raise NoActivation(f"layer {layer_id} has no trailing ReLU")
    s = w.shapes()[act]
    ch = s.channels
    conv_id = w.next_id()
    w.add_node(Node(conv_id, OperatorKind.Conv2D,
                    {"k1": 1, "k2": 1, "c": ch, "j": ch, "stride": 1, "padding": 0},
                    _shared_identity(ch) if kernel_init is channel_identity_kernel else kernel_init(ch), [act]))
    w.add_node(Node(conv_id + 1, OperatorKind.ReLU, {}, None, [conv_id]))
    w.set_shape(conv_id, s)
    w.set_shape(conv_id + 1, s)
    w.rewire(act, conv_id + 1, skip={conv_id, conv_id + 1})


def deepen_layer(graph: Graph, layer_id: int, kernel_init=channel_identity_kernel) -> Graph:
    """Insert a 1x1 Conv2D (identity by default) + ReLU after the layer's ReLU
    (transforms.py:279-300). ``kernel_init`` is the reference's test hook."""
    w = _Work(graph)
    _deepen(w, layer_id, kernel_init)
    return w.g


def _skip(w: _Work, layer_id: int) -> None:
    site = _insertion_point(w, layer_id)
    s = w.shapes()[site]
    ch = s.channels
    conv_id = w.next_id()
    w.add_node(Node(conv_id, OperatorKind.Conv2D,
                    {"k1": 1, "k2": 1, "c": ch, "j": ch, "stride": 1, "padding": 0},
                    _shared_zeros((1, 1, ch, ch)), [site]))
    w.add_node(Node(conv_id + 1, OperatorKind.Add, {}, None, [site, conv_id]))
    w.set_shape(conv_id, s)
    w.set_shape(conv_id + 1, s)
    w.rewire(site, conv_id + 1, skip={conv_id, conv_id + 1})


def skip_layer(graph: Graph, layer_id: int) -> Graph:
    """Zero 1x1 Conv2D around the activation output summed back in: U*X + X = X
    for U = 0 (transforms.py:303-316)."""
    w = _Work(graph)
    _skip(w, layer_id)
    return w.g


def _kernel_widen(w: _Work, layer_id: int, steps: int) -> None:
    node = w.g.nodes[layer_id]
    if node.kind is not OperatorKind.Conv2D:
        raise TransformError(f"cannot kernel-widen {node.kind.value}")
    if steps <= 0:
        return
    if w.lazy:
        node.weights = _derived(w, node).pad_kernel(steps)
    else:
        node.weights = np.pad(node.weights, ((steps, steps), (steps, steps), (0, 0), (0, 0)))
    node.attrs = dict(node.attrs, k1=node.attrs["k1"] + 2 * steps, k2=node.attrs["k2"] + 2 * steps,
                      padding=node.attrs["padding"] + steps)


def widen_kernel(graph: Graph, layer_id: int, steps: int) -> Graph:
    """Zero-pad a Conv2D kernel by ``steps`` rings and raise its padding to
    match (transforms.py:319-335)."""
    if graph.nodes[layer_id].kind is OperatorKind.Conv2D and steps <= 0:
        return graph
    w = _Work(graph)
    _kernel_widen(w, layer_id, steps)
    return w.g


# ---------------------------------------------------------------------------
# Plans (transforms.py:341-474)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class PlanEntry:
    """Per-vanilla-layer knob settings; defaults are the identity (transforms.py:341-355)."""

    layer_id: int
    branching: str = "none"
    deepen: int = 0
    skip: int = 0
    widen_factor: float = 1.0
    kernel_widen: int = 0
    dummy_count: int = 0
    fusion_limit: int = -1  # -1 = unlimited
    schedule_strategy: int = 0


SEQUENCE_KNOBS = ("branching", "fusion_limit", "deepen", "skip")
DIMENSION_KNOBS = ("widen_factor", "kernel_widen", "dummy_count", "schedule_strategy")


@dataclass(frozen=True)
class ObfuscationPlan:
    mode: str  # "sequence" | "dimension"
    entries: tuple[PlanEntry, ...]

    def __post_init__(self):
        if self.mode not in ("sequence", "dimension"):
            raise ValueError(f"unknown mode {self.mode!r}")

    def entry_for(self, layer_id: int) -> PlanEntry:
        for e in self.entries:
            if e.layer_id == layer_id:
                return e
        raise KeyError(layer_id)


def identity_plan(graph: Graph, mode: str = "sequence") -> ObfuscationPlan:
    return ObfuscationPlan(mode, tuple(PlanEntry(lid) for lid in graph.complex_layers()))


@dataclass
class BackendDirectives:
    """Fusion limits / schedule strategies keyed by post-transform complex ids."""

    fusion_limits: dict[int, int] = field(default_factory=dict)
    schedule_strategies: dict[int, int] = field(default_factory=dict)


class PlanApplicationError(TransformError):
    """Aggregated knob failures with layer attribution (transforms.py:391-397)."""

    def __init__(self, failures: list[tuple[int, str, str]]):
        self.failures = failures
        super().__init__("; ".join(f"layer {lid} {knob}: {msg}" for lid, knob, msg in failures))


def apply_plan(graph: Graph, plan: ObfuscationPlan) -> tuple[Graph, BackendDirectives]:
    """Apply a whole plan: widen, kernel-widen, branch, deepen, skip, dummy —
    one pass per knob over the plan entries (transforms.py:400-474)."""
    out, directives, _ = apply_plan_analyzed(graph, plan)
    return out, directives


def apply_plan_analyzed(graph: Graph, plan: ObfuscationPlan, vanilla_analysis=None, lazy: bool = False):
    """``apply_plan`` that also returns the obfuscated graph's structural
    analysis (order / successors / shapes), reusing the knobs' incremental
    successor index and shape table instead of recomputing them. ``lazy``:
    changed Conv2D / Linear weights are DerivedWeights (never materialised on
    the host; ``np.asarray`` gives the eager arrays bit for bit)."""
    if vanilla_analysis is not None:
        vanilla = [nid for nid in vanilla_analysis.order if graph.nodes[nid].kind in COMPLEX_KINDS]
    else:
        vanilla = graph.complex_layers()
    ids = [e.layer_id for e in plan.entries]
    if sorted(ids) != sorted(vanilla):
        raise PlanApplicationError([(-1, "plan", f"entries {sorted(ids)} != complex layers {sorted(vanilla)}")])

    entries = plan.entries
    # Fast exit: an all-identity plan returns the input graph object.
    touched = any(e.widen_factor != 1.0 or e.kernel_widen or e.branching != "none" or e.deepen or e.skip
                  or e.dummy_count for e in entries)
    w = _Work(graph, analysis=vanilla_analysis, lazy=lazy) if touched else None
    failures: list[tuple[int, str, str]] = []
    anchor = {lid: lid for lid in vanilla}
    carriers = {lid: [lid] for lid in vanilla}

    def attempt(lid, knob, fn, *args):
        try:
            return fn(w, *args)
        except TransformError as exc:
            failures.append((lid, knob, str(exc)))
            return None

    if touched:
        for e in entries:
            if e.widen_factor != 1.0:
                attempt(e.layer_id, "widen", _widen, e.layer_id, e.widen_factor)
        for e in entries:
            if e.kernel_widen:
                attempt(e.layer_id, "kernel_widen", _kernel_widen, e.layer_id, e.kernel_widen)
        for e in entries:
            if e.branching != "none":
                mode = "input" if e.branching.startswith("in") else "output"
                created = attempt(e.layer_id, "branch", _branch, e.layer_id, mode, int(e.branching[-1]))
                if created:
                    anchor[e.layer_id] = created[-1]
                    carriers[e.layer_id] = [n for n in created if w.g.nodes[n].kind in COMPLEX_KINDS]
        for e in entries:
            if e.deepen:
                attempt(e.layer_id, "deepen", _deepen, anchor[e.layer_id], channel_identity_kernel)
        for e in entries:
            if e.skip:
                attempt(e.layer_id, "skip", _skip, anchor[e.layer_id])
        for e in entries:
            if e.dummy_count:
                attempt(e.layer_id, "dummy", _dummy, anchor[e.layer_id], e.dummy_count)
    if failures:
        raise PlanApplicationError(failures)

    directives = BackendDirectives()
    for e in entries:
        for nid in carriers[e.layer_id]:
            if e.fusion_limit >= 0:
                directives.fusion_limits[nid] = e.fusion_limit
            if e.schedule_strategy:
                directives.schedule_strategies[nid] = e.schedule_strategy
    if touched:
        return w.g, directives, analyze(w.g, w.succ, w._shapes)
    return graph, directives, vanilla_analysis if vanilla_analysis is not None else analyze(graph)

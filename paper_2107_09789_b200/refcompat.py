"""Drop-in boundary for the reference's own objects (traceobf 0.1.0).

The engine's public functions take and return the reference's types when the
caller hands it reference objects: a ``traceobf.Graph`` / ``Node`` /
``ObfuscationPlan`` / ``DeviceProfile`` / ``LeakageCase`` / ``Kernel`` /
``Schedule`` (reference pkg/src/traceobf/__init__.py:8-49, graph.py:20-146,
transforms.py:341-389, fusion.py:26-98, costmodel.py:34-101, 259-263) is
converted on the way in (graphs share their weight arrays; no copies), the
result is converted back to the caller's classes (``Graph``, ``Trace``,
``TraceStep``, ``CompiledGraph``, ``BackendDirectives``, ``Kernel``,
``Schedule``, ``OperatorKind`` ...), and an engine exception is re-raised as
the caller's exception class of the same name (``TransformError``,
``PlanApplicationError``, ``ShapeMismatch``, ``InvalidStrategy`` ...) so
``except traceobf.transforms.TransformError`` keeps working.

Reference objects are recognised by class NAME and a module outside this
package (duck typing: the reference is never imported here). Engine-typed
arguments pass through untouched, so the engine's own callers pay nothing.

``install(traceobf)`` is the maintainer patch of INTEGRATION.md §3: it
rebinds the reference package's hot entry points to these wrappers.
"""

from __future__ import annotations

import enum
import functools
import importlib
import sys
from collections import OrderedDict

import numpy as np

_PKG = __name__.rsplit(".", 1)[0]

# reference submodules searched for a class name (reference file layout)
_REF_MODULES = ("graph", "transforms", "fusion", "costmodel", "interpreter")

_ENGINE: dict[str, type] = {}


def _engine_classes() -> dict[str, type]:
    if not _ENGINE:
        from . import formats, ir, kernels, knobs, trace
        for mod, names in ((ir, ("Graph", "Node", "TensorShape", "OperatorKind", "Violation", "GraphError",
                                 "CycleDetected", "ShapeMismatch")),
                           (knobs, ("ObfuscationPlan", "PlanEntry", "BackendDirectives", "TransformError",
                                    "NotWidenable", "NotDivisible", "NoActivation", "PlanApplicationError")),
                           (kernels, ("Kernel", "Schedule", "InvalidStrategy")),
                           (trace, ("DeviceProfile", "LeakageCase", "TraceStep", "Trace", "CompiledGraph")),
                           (formats, ("GraphParseError",))):
            for n in names:
                _ENGINE[n] = getattr(mod, n)
    return _ENGINE


def _is_ours(cls: type) -> bool:
    return cls.__module__.split(".")[0] == _PKG


def is_reference(obj) -> bool:
    """A reference-package object of a type this boundary converts."""
    cls = type(obj)
    return cls.__name__ in _engine_classes() and not _is_ours(cls) and \
        cls.__module__.split(".")[0] not in ("builtins", "numpy")


class RefTypes:
    """Class lookup in the caller's reference package (found from one of its objects)."""

    def __init__(self, sample):
        self.root = type(sample).__module__.split(".")[0]
        self._cache: dict[str, type] = {}

    def get(self, name: str) -> type | None:
        hit = self._cache.get(name)
        if hit is None:
            for sub in ("",) + _REF_MODULES:
                try:
                    mod = importlib.import_module(self.root + ("." + sub if sub else ""))
                except ImportError:
                    continue
                hit = getattr(mod, name, None)
                if isinstance(hit, type):
                    break
                hit = None
            if hit is not None:
                self._cache[name] = hit
        return hit


# ---------------------------------------------------------------- reference -> engine
_GRAPHS: OrderedDict = OrderedDict()  # id(reference graph) -> (graph, engine graph); graphs are immutable by convention


def _shape_in(s):
    if s is None:
        return None
    E = _engine_classes()
    return E["TensorShape"](s.batch, s.channels, s.height, s.width)


def engine_graph(g):
    """Engine Graph of a reference Graph (node-for-node, weights shared;
    cached by identity like the engine's device weight cache)."""
    hit = _GRAPHS.get(id(g))
    if hit is not None and hit[0] is g:
        _GRAPHS.move_to_end(id(g))
        return hit[1]
    E = _engine_classes()
    K, Node = E["OperatorKind"], E["Node"]
    nodes = {nid: Node(n.id, K(n.kind.value), dict(n.attrs), n.weights, list(n.inputs), _shape_in(n.out_shape))
             for nid, n in g.nodes.items()}
    out = E["Graph"](nodes, g.output_id, _shape_in(g.input_shape))
    _GRAPHS[id(g)] = (g, out)
    if len(_GRAPHS) > 256:
        _GRAPHS.popitem(last=False)
    return out


def to_engine(obj):
    """Reference object (or container of them) -> engine object."""
    if isinstance(obj, (list, tuple)):
        conv = [to_engine(o) for o in obj]
        return type(obj)(conv) if isinstance(obj, list) or type(obj) is tuple else obj
    if isinstance(obj, dict):
        return {k: to_engine(v) for k, v in obj.items()}
    if not is_reference(obj):
        return obj
    E = _engine_classes()
    name = type(obj).__name__
    if name == "Graph":
        return engine_graph(obj)
    if name == "Node":
        return E["Node"](obj.id, E["OperatorKind"](obj.kind.value), dict(obj.attrs), obj.weights,
                         list(obj.inputs), _shape_in(obj.out_shape))
    if name == "TensorShape":
        return _shape_in(obj)
    if isinstance(obj, enum.Enum):
        return E[name](obj.value)
    if name == "ObfuscationPlan":
        return E[name](obj.mode, tuple(to_engine(e) for e in obj.entries))
    if name in ("PlanEntry", "DeviceProfile", "Schedule", "Kernel", "BackendDirectives", "Violation"):
        return E[name](**{k: to_engine(v) for k, v in vars(obj).items()})
    if name == "TraceStep":
        return E[name](**{k: to_engine(v) for k, v in vars(obj).items()})
    if name == "Trace":
        return E[name](tuple(to_engine(s) for s in obj.steps), to_engine(obj.case))
    if name == "CompiledGraph":
        return E[name](engine_graph(obj.graph), [to_engine(k) for k in obj.kernels],
                       [to_engine(s) for s in obj.schedules])
    return obj


# ---------------------------------------------------------------- engine -> reference
def to_ref(obj, R: RefTypes):
    """Engine object (or container) -> the caller's reference classes."""
    if isinstance(obj, list):
        return [to_ref(o, R) for o in obj]
    if type(obj) is tuple:
        return tuple(to_ref(o, R) for o in obj)
    if isinstance(obj, dict):
        return {k: to_ref(v, R) for k, v in obj.items()}
    cls = type(obj)
    if not _is_ours(cls) or cls.__name__ not in _engine_classes():
        return obj
    name = cls.__name__
    T = R.get(name)
    if T is None:
        return obj
    if name == "Graph":
        Node, K = R.get("Node"), R.get("OperatorKind")
        nodes = {nid: Node(n.id, K(n.kind.value), dict(n.attrs),
                           n.weights if n.weights is None or isinstance(n.weights, np.ndarray)
                           else np.asarray(n.weights),
                           list(n.inputs), to_ref(n.out_shape, R) if n.out_shape is not None else None)
                 for nid, n in obj.nodes.items()}
        return T(nodes, obj.output_id, to_ref(obj.input_shape, R))
    if name == "TensorShape":
        return T(obj.batch, obj.channels, obj.height, obj.width)
    if isinstance(obj, enum.Enum):
        return T(obj.value)
    if name == "ObfuscationPlan":
        return T(obj.mode, tuple(to_ref(e, R) for e in obj.entries))
    if name == "Trace":
        return T(tuple(to_ref(s, R) for s in obj.steps), to_ref(obj.case, R))
    if name == "CompiledGraph":
        return T(to_ref(obj.graph, R), [to_ref(k, R) for k in obj.kernels], [to_ref(s, R) for s in obj.schedules])
    if name in ("PlanEntry", "DeviceProfile", "Schedule", "Kernel", "BackendDirectives", "Violation", "TraceStep"):
        fields = getattr(obj, "__dataclass_fields__", None) or vars(obj)
        return T(**{k: to_ref(getattr(obj, k), R) for k in fields})
    return obj


def _ref_exception(exc: BaseException, R: RefTypes) -> BaseException | None:
    T = R.get(type(exc).__name__)
    if T is None or not issubclass(T, BaseException):
        return None
    name = type(exc).__name__
    try:
        if name == "ShapeMismatch":
            msg = str(exc).split(": ", 1)[1] if ": " in str(exc) else str(exc)
            return T(exc.node_id, msg)
        if name == "PlanApplicationError":
            return T(list(exc.failures))
        return T(*exc.args)
    except Exception:  # noqa: BLE001 — an unexpected constructor: keep the engine's exception
        return None


def _first_reference(args, kwargs):
    for a in list(args) + list(kwargs.values()):
        if is_reference(a):
            return a
        if isinstance(a, (list, tuple)) and a and is_reference(a[0]):
            return a[0]
        if isinstance(a, dict):
            for v in a.values():
                if is_reference(v):
                    return v
    return None


def dropin(fn):
    """Wrap an engine entry point: reference objects in -> engine objects;
    engine results and exceptions -> the caller's reference classes."""

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        ref = _first_reference(args, kwargs)
        if ref is None:
            return fn(*args, **kwargs)
        R = RefTypes(ref)
        args = tuple(to_engine(a) for a in args)
        kwargs = {k: to_engine(v) for k, v in kwargs.items()}
        try:
            out = fn(*args, **kwargs)
        except Exception as exc:
            mapped = _ref_exception(exc, R)
            if mapped is None:
                raise
            raise mapped from exc
        return to_ref(out, R)

    wrapper.__dropin__ = True
    return wrapper


#: the reference entry points INTEGRATION.md §3's maintainer patch routes to
#: the engine (the hot path: forward + verdict, compile + trace)
HOT_PATH = ("execute", "equivalence_check", "compile_graph", "profile_pipeline", "profile_graph", "profile_kernel",
            "default_schedule")


def install(ref_pkg, names=HOT_PATH) -> dict:
    """Maintainer patch: rebind ``ref_pkg.<name>`` (the reference package
    module, e.g. ``traceobf``) to the engine's drop-in entry points. Returns
    the previous bindings (``uninstall`` restores them)."""
    eng = sys.modules[_PKG]
    saved = {}
    for n in names:
        saved[n] = getattr(ref_pkg, n)
        setattr(ref_pkg, n, getattr(eng, n))
    return saved


def uninstall(ref_pkg, saved: dict) -> None:
    for n, f in saved.items():
        setattr(ref_pkg, n, f)

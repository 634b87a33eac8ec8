"""Analytical trace features on the GPU (drop-in for traceobf.costmodel).

Names and semantics mirror costmodel.py: ``DeviceProfile``,
``BUILTIN_PROFILES``, ``LeakageCase``, ``TraceStep``, ``Trace``,
``profile_kernel``, ``profile_graph``, ``compile_graph``,
``profile_pipeline``, and the process-global schedule memo with first-seen
semantics (costmodel.py:248-285). The host reduces each kernel to the exact
integers the formulas read (``kernel_desc``); the brute-force schedule
search (fusion.py:159-180), the 9 features (costmodel.py:166-232) and the
Neumaier total latency (costmodel.py:96-98) run in fp64 on the device,
bit-identical to the Python arithmetic (csrc/trace.cu, built -fmad=false).

``trace_population`` is the batched entry point: one schedule-search launch
for every not-yet-memoised signature of a whole population (first-seen order
= candidate order), one profile launch, one totals launch.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .engine import device
from .ir import COMPLEX_KINDS, Graph, OperatorKind as K, TensorShape, infer_shapes, shape_map, topo_order
from .kernels import DEFAULT_UNROLL, TRIVIAL_SCHEDULE, Kernel, Schedule, fuse, modify_schedule

BYTES = 4            # costmodel.py:28
_TX_GRANULE = 32     # costmodel.py:29
_STREAM_FP = 8192    # costmodel.py:30
_EFF_FLOOR = 1.0 / 256.0  # costmodel.py:31


@dataclass(frozen=True)
class DeviceProfile:
    """costmodel.py:34-41."""

    name: str
    macs_per_cycle: int = 1024
    launch_overhead: int = 2000
    l1_bytes: int = 64 * 1024
    l2_bytes: int = 1024 * 1024
    sm_count: int = 4

    def as_c(self) -> N.DeviceProfileC:
        return N.DeviceProfileC(self.macs_per_cycle, self.launch_overhead, self.l1_bytes, self.l2_bytes,
                                self.sm_count)


BUILTIN_PROFILES = {
    "default": DeviceProfile("default"),
    "lean": DeviceProfile("lean", macs_per_cycle=256, launch_overhead=500, l1_bytes=32 * 1024,
                          l2_bytes=512 * 1024, sm_count=4),
}


class LeakageCase(Enum):
    """costmodel.py:53-70."""

    A = "A"
    B = "B"
    C = "C"

    @property
    def features(self) -> tuple[str, ...]:
        return CASE_FEATURES[self]


CASE_FEATURES = {
    LeakageCase.A: ("cycles",),
    LeakageCase.B: ("cycles", "dram_read", "dram_write"),
    LeakageCase.C: ("cycles", "dram_read", "dram_write", "l1_tx", "l1_util", "l1_hit", "l2_tx", "l2_util", "l2_hit"),
}
FEATURE_NAMES = CASE_FEATURES[LeakageCase.C]


@dataclass(frozen=True)
class TraceStep:
    """costmodel.py:73-88."""

    cycles: float
    dram_read: float = 0.0
    dram_write: float = 0.0
    l1_tx: float = 0.0
    l1_util: float = 0.0
    l1_hit: float = 0.0
    l2_tx: float = 0.0
    l2_util: float = 0.0
    l2_hit: float = 0.0
    label: K | None = None
    anchor_id: int = -1

    def features(self, case: LeakageCase) -> tuple[float, ...]:
        return tuple(getattr(self, f) for f in case.features)


@dataclass(frozen=True)
class Trace:
    """costmodel.py:91-101."""

    steps: tuple[TraceStep, ...]
    case: LeakageCase

    @property
    def total_latency(self) -> float:
        return sum(s.cycles for s in self.steps)   # CPython 3.12: Neumaier

    def feature_matrix(self) -> np.ndarray:
        return np.array([s.features(self.case) for s in self.steps], dtype=np.float64)


@dataclass
class CompiledGraph:
    graph: Graph
    kernels: list[Kernel]
    schedules: list[Schedule]


# process-global memo, first-seen semantics (costmodel.py:248)
_SCHEDULE_CACHE: dict[tuple, Schedule] = {}

_LABEL_CODE = {K.Conv2D: 1, K.Linear: 2, K.MaxPool: 3, K.SoftMax: 4}


def schedule_signature(graph: Graph, shapes: dict, kernel: Kernel, profile: DeviceProfile) -> tuple:
    """costmodel.py:251-256."""
    a = graph.nodes[kernel.anchor]
    ins = shapes[a.inputs[0]] if a.inputs else graph.input_shape
    return (profile.name, a.kind.value, tuple(sorted(a.attrs.items())), ins.as_tuple(),
            shapes[kernel.anchor].as_tuple())


def _numel(s: TensorShape) -> int:
    return s.batch * s.channels * s.height * s.width


def _work(graph: Graph, shapes: dict, nid: int) -> int:
    """costmodel.py:108-124."""
    n, s = graph.nodes[nid], shapes[nid]
    if n.kind is K.Conv2D:
        a = n.attrs
        return s.batch * a["k1"] * a["k2"] * a["c"] * a["j"] * s.height * s.width
    if n.kind is K.Linear:
        return s.batch * n.attrs["c"] * n.attrs["j"]
    if n.kind is K.MaxPool:
        return _numel(s) * n.attrs["window"] ** 2
    if n.kind is K.SoftMax:
        return 4 * _numel(s)
    if n.kind is K.BatchNorm:
        return 2 * _numel(s)
    return _numel(s)


def kernel_desc(graph: Graph, shapes: dict, kernel: Kernel, schedule: Schedule | None, d: N.KernDesc) -> None:
    """Fill ``d`` with the integers profile_kernel reads (costmodel.py:166-232)."""
    a = graph.nodes[kernel.anchor]
    s = shapes[kernel.anchor]
    d.has_shape = 1
    d.work = _work(graph, shapes, kernel.anchor)
    d.fused_work = sum(_work(graph, shapes, q) for q in kernel.node_ids[1:])
    fb = 0
    for q in kernel.node_ids[1:]:
        nq = graph.nodes[q]
        if nq.weights is not None:
            fb += nq.weights.size * BYTES
        if nq.kind is K.Add and len(nq.inputs) > 1:
            fb += sum(_numel(shapes[p]) * BYTES for p in nq.inputs[1:])
    d.fused_bytes = fb
    d.in_bytes = (sum(_numel(shapes[p]) for p in a.inputs) if a.inputs else _numel(graph.input_shape)) * BYTES
    d.w_bytes = a.weights.size * BYTES if a.weights is not None else 0
    d.out_bytes = _numel(shapes[kernel.node_ids[-1]]) * BYTES
    d.tiled = 1 if a.kind in (K.Conv2D, K.MaxPool) else 0
    d.is_conv = 1 if a.kind is K.Conv2D else 0
    d.H, d.W = s.height, s.width
    if a.kind is K.Conv2D:
        d.c, d.k1, d.k2, d.s = a.attrs["c"], a.attrs["k1"], a.attrs["k2"], a.attrs["stride"]
    elif a.kind is K.MaxPool:
        d.c, d.k1, d.k2, d.s = a.attrs.get("c", s.channels), a.attrs["window"], a.attrs["window"], a.attrs["stride"]
    d.channel_like = a.attrs.get("j", s.channels)
    d.reuse_x_stream = a.attrs["j"] if a.kind is K.Linear else 1
    d.label = _LABEL_CODE.get(a.kind, -1)
    d.unroll = DEFAULT_UNROLL
    if schedule is not None:
        d.ty[:] = list(schedule.tile_y)
        d.tx[:] = list(schedule.tile_x)
        d.unroll = schedule.unroll


def _to_step(row: np.ndarray, graph: Graph, kernel: Kernel) -> TraceStep:
    a = graph.nodes[kernel.anchor]
    return TraceStep(*(float(v) for v in row), label=a.kind if a.kind in COMPLEX_KINDS else None,
                     anchor_id=kernel.anchor)


def search_schedules(graph: Graph, kernels: list[Kernel], profile: DeviceProfile,
                     shapes: dict | None = None) -> list[Schedule]:
    """default_schedule for each kernel, on the device (no memo)."""
    ctx = device()
    shapes = shapes if shapes is not None else shape_map(graph)
    arr = (N.KernDesc * max(len(kernels), 1))()
    for i, k in enumerate(kernels):
        kernel_desc(graph, shapes, k, None, arr[i])
    dev = ctx.upload_struct_array(arr)
    pc = profile.as_c()
    ctx.check(ctx.lib.tobf_schedule_search(C.c_void_p(dev.data_ptr()), len(kernels), C.byref(pc),
                                           C.c_void_p(ctx.sp)), "schedule search")
    host = torch.empty_like(dev, device="cpu")
    host.copy_(dev)
    ctx.sync()
    back = (N.KernDesc * max(len(kernels), 1)).from_buffer_copy(host.numpy().tobytes())
    return [Schedule(tuple(back[i].ty), tuple(back[i].tx), back[i].unroll) for i in range(len(kernels))]


def compile_graph(graph: Graph, profile: DeviceProfile, fusion_limits: dict[int, int] | None = None,
                  strategies: dict[int, int] | None = None) -> CompiledGraph:
    """costmodel.py:266-285."""
    return compile_population([(graph, fusion_limits, strategies)], profile)[0]


def compile_population(items: list[tuple[Graph, dict | None, dict | None]], profile: DeviceProfile,
                       memo: dict | None = None) -> list[CompiledGraph]:
    """compile_graph over many graphs with ONE device schedule search for all
    signatures not yet in ``memo`` (first-seen order across ``items``)."""
    memo = _SCHEDULE_CACHE if memo is None else memo
    pending: dict[tuple, tuple] = {}
    staged = []
    for graph, limits, strategies in items:
        order = topo_order(graph)
        shapes = shape_map(graph, order)
        annotated = graph.copy()
        for nid, s in shapes.items():
            annotated.nodes[nid].out_shape = s
        kernels = fuse(annotated, limits, order=order)
        sigs = [schedule_signature(annotated, shapes, k, profile) for k in kernels]
        for k, sig in zip(kernels, sigs):
            if sig not in memo and sig not in pending:
                if annotated.nodes[k.anchor].kind not in COMPLEX_KINDS:
                    memo[sig] = TRIVIAL_SCHEDULE
                else:
                    pending[sig] = (annotated, shapes, k)
        staged.append((annotated, shapes, kernels, sigs, strategies or {}))
    if pending:
        ctx = device()
        keys = list(pending)
        arr = (N.KernDesc * len(keys))()
        for i, key in enumerate(keys):
            g, sh, k = pending[key]
            kernel_desc(g, sh, k, None, arr[i])
        dev = ctx.upload_struct_array(arr)
        pc = profile.as_c()
        ctx.check(ctx.lib.tobf_schedule_search(C.c_void_p(dev.data_ptr()), len(keys), C.byref(pc),
                                               C.c_void_p(ctx.sp)), "schedule search")
        host = dev.cpu()
        back = (N.KernDesc * len(keys)).from_buffer_copy(host.numpy().tobytes())
        for i, key in enumerate(keys):
            memo[key] = Schedule(tuple(back[i].ty), tuple(back[i].tx), back[i].unroll)
    out = []
    for annotated, shapes, kernels, sigs, strategies in staged:
        scheds = []
        for k, sig in zip(kernels, sigs):
            sch = memo[sig]
            st = strategies.get(k.anchor, 0)
            if st:
                sch = modify_schedule(sch, st)
            scheds.append(sch)
        cg = CompiledGraph(annotated, kernels, scheds)
        cg._shapes = shapes
        out.append(cg)
    return out


@dataclass
class PopulationTrace:
    """Device-resident traces of a population: feats (n_kernels, 9) fp64,
    offsets (ncand+1) int32, totals (ncand) fp64; host views on demand."""

    compiled: list[CompiledGraph]
    feats: torch.Tensor
    offsets: torch.Tensor
    totals: torch.Tensor
    offsets_host: np.ndarray

    def trace(self, i: int, case: LeakageCase, feats_host: np.ndarray | None = None) -> Trace:
        fh = feats_host if feats_host is not None else self.feats.cpu().numpy()
        cg = self.compiled[i]
        lo, hi = self.offsets_host[i], self.offsets_host[i + 1]
        return Trace(tuple(_to_step(fh[r], cg.graph, k) for r, k in zip(range(lo, hi), cg.kernels)), case)


def trace_population(items: list[tuple[Graph, dict | None, dict | None]], profile: DeviceProfile,
                     memo: dict | None = None) -> PopulationTrace:
    """compile + profile + T for a population, all arithmetic on the device."""
    ctx = device()
    compiled = compile_population(items, profile, memo)
    nk = sum(len(cg.kernels) for cg in compiled)
    arr = (N.KernDesc * max(nk, 1))()
    offsets = np.zeros(len(compiled) + 1, np.int32)
    r = 0
    for i, cg in enumerate(compiled):
        for k, sch in zip(cg.kernels, cg.schedules):
            kernel_desc(cg.graph, cg._shapes, k, sch, arr[r])
            r += 1
        offsets[i + 1] = r
    dev = ctx.upload_struct_array(arr)
    offs = torch.from_numpy(offsets).to(ctx.device, non_blocking=True)
    feats = torch.empty((max(nk, 1), 9), dtype=torch.float64, device=ctx.device)
    totals = torch.empty(len(compiled), dtype=torch.float64, device=ctx.device)
    pc = profile.as_c()
    ctx.check(ctx.lib.tobf_profile_kernels(C.c_void_p(dev.data_ptr()), nk, C.byref(pc),
                                           C.c_void_p(feats.data_ptr()), C.c_void_p(ctx.sp)), "profile")
    ctx.check(ctx.lib.tobf_trace_totals(C.c_void_p(feats.data_ptr()), C.c_void_p(offs.data_ptr()), len(compiled),
                                        C.c_void_p(totals.data_ptr()), C.c_void_p(ctx.sp)), "trace totals")
    pt = PopulationTrace(compiled, feats, offs, totals, offsets)
    pt._desc = dev
    return pt


def profile_graph(graph: Graph, kernels: list[Kernel], schedules: list[Schedule], case: LeakageCase,
                  profile: DeviceProfile) -> Trace:
    """costmodel.py:235-241 (``graph`` must carry shapes)."""
    ctx = device()
    shapes = {nid: n.out_shape for nid, n in graph.nodes.items()}
    if any(s is None for s in shapes.values()):
        shapes = shape_map(graph)
    arr = (N.KernDesc * max(len(kernels), 1))()
    for i, (k, s) in enumerate(zip(kernels, schedules, strict=True)):
        kernel_desc(graph, shapes, k, s, arr[i])
    dev = ctx.upload_struct_array(arr)
    feats = torch.empty((max(len(kernels), 1), 9), dtype=torch.float64, device=ctx.device)
    pc = profile.as_c()
    ctx.check(ctx.lib.tobf_profile_kernels(C.c_void_p(dev.data_ptr()), len(kernels), C.byref(pc),
                                           C.c_void_p(feats.data_ptr()), C.c_void_p(ctx.sp)), "profile")
    fh = feats.cpu().numpy()
    ctx.sync()
    return Trace(tuple(_to_step(fh[i], graph, k) for i, k in enumerate(kernels)), case)


def profile_kernel(graph: Graph, kernel: Kernel, schedule: Schedule, profile: DeviceProfile) -> TraceStep:
    """costmodel.py:166-232 for one kernel."""
    a = graph.nodes[kernel.anchor]
    if a.out_shape is None:
        return TraceStep(cycles=0.0, anchor_id=kernel.anchor)
    return profile_graph(graph, [kernel], [schedule], LeakageCase.C, profile).steps[0]


def profile_pipeline(graph: Graph, case: LeakageCase, profile: DeviceProfile,
                     fusion_limits: dict[int, int] | None = None,
                     strategies: dict[int, int] | None = None) -> Trace:
    """costmodel.py:288-293."""
    pt = trace_population([(graph, fusion_limits, strategies)], profile)
    fh = pt.feats.cpu().numpy()
    device().sync()
    return pt.trace(0, case, fh)

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
import hashlib
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .engine import cat_records, device
from .ir import COMPLEX_KINDS, Graph, OperatorKind as K, TensorShape, analyze, infer_shapes, shape_map, topo_order
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


class CompiledGraph:
    """costmodel.py:259-263: shape-annotated graph, kernels, schedules. The
    annotated copy is built lazily (the batched path never needs it)."""

    def __init__(self, graph: Graph | None = None, kernels: list[Kernel] | None = None,
                 schedules: list[Schedule] | None = None, *, source: Graph | None = None,
                 shapes: dict | None = None):
        self._graph = graph
        self._source = source
        self._shapes = shapes
        self.kernels = kernels or []
        self.schedules = schedules or []

    @property
    def graph(self) -> Graph:
        if self._graph is None:
            g = self._source.copy()
            for nid, sh in self._shapes.items():
                g.nodes[nid].out_shape = sh
            self._graph = g
        return self._graph

    @property
    def nodes_source(self) -> Graph:
        return self._graph if self._graph is not None else self._source


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
    return s._n


_ATTR_CANON: dict[tuple, tuple] = {}


def canonical_attrs(attrs: dict) -> tuple:
    """tuple(sorted(attrs.items())) (the signature's attrs part), memoised."""
    items = tuple(attrs.items())
    hit = _ATTR_CANON.get(items)
    if hit is None:
        hit = _ATTR_CANON[items] = tuple(sorted(items))
    return hit


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


KERN_DTYPE = np.dtype(N.KernDesc)


def kernel_tuple(graph: Graph, shapes: dict, kernel: Kernel, schedule: Schedule | None = None, strategy: int = 0,
                 sig_index: int = -1, resolved: int = 0) -> tuple:
    """The integers profile_kernel reads (costmodel.py:166-232), as one
    KERN_DTYPE record (field order of tobf_kern_desc)."""
    nodes = graph.nodes
    a = nodes[kernel.anchor]
    s = shapes[kernel.anchor]
    fused = kernel.node_ids[1:]
    fw = fb = 0
    for q in fused:
        nq = nodes[q]
        fw += _work(graph, shapes, q)
        if nq.weights is not None:
            fb += nq.weights.size * BYTES
        if nq.kind is K.Add and len(nq.inputs) > 1:
            fb += sum(_numel(shapes[p]) * BYTES for p in nq.inputs[1:])
    inb = (sum(_numel(shapes[p]) for p in a.inputs) if a.inputs else _numel(graph.input_shape)) * BYTES
    wb = a.weights.size * BYTES if a.weights is not None else 0
    ob = _numel(shapes[kernel.node_ids[-1]]) * BYTES
    kind = a.kind
    at = a.attrs
    if kind is K.Conv2D:
        geo = (1, 1, at["c"], at["k1"], at["k2"], at["stride"])
    elif kind is K.MaxPool:
        geo = (1, 0, at.get("c", s.channels), at["window"], at["window"], at["stride"])
    else:
        geo = (0, 0, 0, 0, 0, 0)
    if schedule is not None:
        ty, tx, unroll = tuple(schedule.tile_y), tuple(schedule.tile_x), schedule.unroll
    else:
        ty, tx, unroll = (0, 0, 0), (0, 0, 0), DEFAULT_UNROLL
    return (_work(graph, shapes, kernel.anchor), fw, fb, inb, wb, ob) + geo + (
        s.height, s.width, at.get("j", s.channels), at["j"] if kind is K.Linear else 1, ty, tx, unroll,
        _LABEL_CODE.get(kind, -1), 1, strategy, sig_index, resolved)


def kernel_desc(graph: Graph, shapes: dict, kernel: Kernel, schedule: Schedule | None, d: N.KernDesc) -> None:
    """Fill a ctypes KernDesc (single-kernel paths)."""
    rec = np.array([kernel_tuple(graph, shapes, kernel, schedule)], dtype=KERN_DTYPE)
    C.memmove(C.addressof(d), rec.ctypes.data, C.sizeof(d))


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
    """costmodel.py:266-285 (default schedules searched on the device)."""
    tp = prepare_trace([(graph, fusion_limits, strategies)], profile)
    run_trace(tp, profile=False)
    finish_trace(tp)
    return tp.compiled[0]


class TracePlan:
    """Host-prepared, device-resident inputs of the trace stage for a population.

    kern      per-kernel descriptors in candidate order (profile input)
    sigs      one row per distinct schedule signature of the batch, first-seen
              order; rows already in the memo carry their schedule and
              ``resolved = 1``, the others are searched on the device
    offsets   kernel range of candidate i = [offsets[i], offsets[i+1])
    """

    def __init__(self, compiled, kern_dev, sig_dev, nk, nsig, pending, offsets_host, offsets_dev, profile, memo):
        self.compiled, self.kern, self.sigs = compiled, kern_dev, sig_dev
        self.nk, self.nsig, self.pending = nk, nsig, pending
        self.offsets_host, self.offsets = offsets_host, offsets_dev
        self.profile, self.memo = profile, memo
        self.feats = self.totals = None


_COMPLEX_VALUES = frozenset(k.value for k in COMPLEX_KINDS)


@dataclass
class CandidateTrace:
    """Host half of compile_graph for one graph (no device, picklable):
    kernel records in kernel order (schedule unresolved, sig_index -1) and
    each kernel's schedule signature (costmodel.py:251-256)."""

    recs: np.ndarray
    sigs: list | None
    sig_keys: np.ndarray | None = None  # 64-bit content digest per signature (process-independent)
    new_sigs: dict | None = None        # wire form: digest -> signature for digests not sent before

    def __getstate__(self):
        st = dict(self.__dict__)
        st["recs"] = self.recs.tobytes()  # raw bytes: see executor._plan_getstate
        return st

    def __setstate__(self, st):
        st = dict(st)
        st["recs"] = np.frombuffer(st["recs"], dtype=KERN_DTYPE).copy()
        self.__dict__.update(st)

    def compact(self, sent: set) -> "CandidateTrace":
        """Wire form for a host worker: the signature tuples are replaced by
        their digests, plus the tuples of digests this worker has not sent
        before (signatures repeat across a population)."""
        new = {}
        for k, sg in zip(self.sig_keys.tolist(), self.sigs):
            if k not in sent:
                sent.add(k)
                new[k] = sg
        return CandidateTrace(self.recs, None, self.sig_keys, new)

    def expand(self, table: dict) -> "CandidateTrace":
        """Parent side: fold the new signatures into ``table`` and rebuild the list."""
        if self.sigs is None:
            table.update(self.new_sigs or {})
            self.sigs = [table[k] for k in self.sig_keys.tolist()]
            self.new_sigs = None
        return self


_DIGESTS: dict[tuple, int] = {}


def sig_digest(sig: tuple) -> int:
    """Deterministic 64-bit digest of a schedule signature (unlike hash(),
    equal across the host worker processes), so a batch's signatures are
    deduplicated with numpy instead of one dict lookup per kernel. Memoised
    per process (signatures repeat across a population)."""
    d = _DIGESTS.get(sig)
    if d is None:
        if len(_DIGESTS) > 1 << 18:
            _DIGESTS.clear()
        d = _DIGESTS[sig] = int.from_bytes(hashlib.blake2b(repr(sig).encode(), digest_size=8).digest(), "little")
    return d


def trace_records(graph: Graph, fusion_limits: dict | None, strategies: dict | None, pname: str,
                  analysis=None) -> tuple[CandidateTrace, list[Kernel], dict]:
    """fuse + signatures + integer descriptors of one graph."""
    ana = analysis if analysis is not None else analyze(graph)
    shapes = ana.shapes
    kernels = fuse(graph, fusion_limits, order=ana.order, succ=ana.succ)
    strategies = strategies or {}
    nodes = graph.nodes
    sigs, rows = [], []
    for k in kernels:
        a = nodes[k.anchor]
        ins = shapes[a.inputs[0]] if a.inputs else graph.input_shape
        sigs.append((pname, a.kind.value, canonical_attrs(a.attrs), ins._t, shapes[k.anchor]._t))
        rows.append(kernel_tuple(graph, shapes, k, None, strategies.get(k.anchor, 0), -1))
    recs = np.array(rows, dtype=KERN_DTYPE) if rows else np.zeros(0, KERN_DTYPE)
    keys = np.array([sig_digest(sg) for sg in sigs], dtype=np.uint64)
    return CandidateTrace(recs, sigs, keys), kernels, shapes


def prepare_trace(items: list[tuple], profile: DeviceProfile, memo: dict | None = None,
                  exchange=None, first_seen: dict | None = None, conv_index: bool = False,
                  extra: dict | None = None) -> TracePlan:
    """Host half of compile_graph for many graphs: fuse, signatures, integer
    descriptors (one H2D for all). ``items``: (graph, fusion_limits,
    strategies[, ir.Analysis[, (CandidateTrace, kernels, shapes)]])."""
    cts, compiled = [], []
    for item in items:
        graph, limits, strategies = item[0], item[1], item[2]
        ana = item[3] if len(item) > 3 and item[3] is not None else None
        pre = item[4] if len(item) > 4 else None
        ct, kernels, shapes = pre if pre is not None else trace_records(graph, limits, strategies, profile.name, ana)
        cts.append(ct)
        compiled.append(CompiledGraph(kernels=kernels, source=graph, shapes=shapes))
    return prepare_trace_records(cts, profile, memo, exchange, first_seen, compiled, conv_index, extra)


def _distinct_sigs(cts: list[CandidateTrace]):
    """(signature, candidate position, KERN record array, row) of every
    distinct signature of ``cts`` in first-occurrence order (candidate order,
    kernel order). Deduplicated by 64-bit digest with numpy when every record
    carries digests, else one dict pass."""
    flat = [(sg, c) for c, ct in enumerate(cts) for sg in ct.sigs]
    if flat and all(ct.sig_keys is not None and len(ct.sig_keys) == len(ct.sigs) for ct in cts):
        allk = np.concatenate([ct.sig_keys for ct in cts])
        _, first = np.unique(allk, return_index=True)
        recs_all = cat_records([ct.recs for ct in cts], KERN_DTYPE)
        return [(flat[i][0], flat[i][1], recs_all, int(i)) for i in np.sort(first)]
    out, seen = [], set()
    for c, ct in enumerate(cts):
        for r, sg in enumerate(ct.sigs):
            if sg not in seen:
                seen.add(sg)
                out.append((sg, c, ct.recs, r))
    return out


def _first_blob(recs: np.ndarray, r: int) -> bytes:
    """Descriptor a signature is searched from: its first occurrence's kernel
    record with the strategy cleared (default_schedule runs before
    modify_schedule, costmodel.py:277-283)."""
    rec = recs[r:r + 1].copy()
    rec["strategy"] = 0
    return rec.tobytes()


def shard_first_seen(cts: list[CandidateTrace], gidx, memo: dict) -> list[tuple[tuple, int, bytes]]:
    """This process's part of the first-seen schedule memo (costmodel.py:
    248-285) for a whole shard: every complex-kernel signature that is not
    memoised yet, in first-occurrence order, tagged with the GLOBAL index of
    the candidate it first occurs in and the descriptor it would be searched
    from. Pure host (no device): ``dist.exchange_signatures`` merges the
    parts of all ranks by global index."""
    out = []
    for sig, c, recs, r in _distinct_sigs(cts):
        if sig in memo or sig[1] not in _COMPLEX_VALUES:
            continue
        out.append((sig, int(gidx[c]), _first_blob(recs, r)))
    return out


def resolve_first_seen(cts: list[CandidateTrace], gidx, memo: dict, exchange=None) -> dict[tuple, bytes]:
    """signature -> descriptor of its globally first occurrence, for every
    signature unmemoised on any rank. Exactly ONE ``exchange`` call whatever
    this shard holds (empty, all infeasible, any micro-batch split), so the
    ranks' collectives always pair up; every rank then searches the same
    table and folds it into its memo, keeping the memos identical."""
    local = shard_first_seen(cts, gidx, memo)
    if exchange is None:
        return {sig: blob for sig, _, blob in local}
    return exchange(local)


def prepare_trace_records(cts: list[CandidateTrace], profile: DeviceProfile, memo: dict | None = None,
                          exchange=None, first_seen: dict | None = None,
                          compiled: list[CompiledGraph] | None = None, conv_index: bool = False,
                          extra: dict | None = None) -> TracePlan:
    """Memo resolution and upload of a batch's kernel records.

    Signatures already in the memo resolve to their schedule; the others are
    searched on the device from their FIRST occurrence's descriptor
    (costmodel.py:248 first-seen memo). ``first_seen`` (sig -> descriptor
    bytes) carries first occurrences across the micro-batches of one call
    (and, sharded, the globally first ones from ``resolve_first_seen``).
    ``extra``: further (sig -> descriptor) rows to search and memoise although
    no kernel of this batch uses them (signatures first seen on other ranks).
    ``exchange``: this batch is a whole shard — resolve it across ranks here
    (one collective; callers splitting a shard resolve it once themselves)."""
    ctx = device()
    memo = _SCHEDULE_CACHE if memo is None else memo
    if exchange is not None:
        glob = resolve_first_seen(cts, range(len(cts)), memo, exchange)
        first_seen = dict(glob) if first_seen is None else first_seen
        first_seen.update(glob)
        extra = glob
    hits: dict[tuple, Schedule] = {}
    local_pending: dict[tuple, bytes] = {}
    flat_sigs = [sg for ct in cts for sg in ct.sigs]
    nk_all = len(flat_sigs)
    use_keys = nk_all > 0 and all(ct.sig_keys is not None and len(ct.sig_keys) == len(ct.sigs) for ct in cts)
    if use_keys:
        allk = np.concatenate([ct.sig_keys for ct in cts])
        _, first, inverse = np.unique(allk, return_index=True, return_inverse=True)
        recs_all = cat_records([ct.recs for ct in cts], KERN_DTYPE)
        visit = [(flat_sigs[i], recs_all, int(i)) for i in np.sort(first)]
    else:
        visit = [(sig, ct.recs, r) for ct in cts for r, sig in enumerate(ct.sigs)]
    for sig, recs_src, r in visit:
        if sig in hits or sig in local_pending:
            continue
        hit = memo.get(sig)
        if hit is None and sig[1] not in _COMPLEX_VALUES:
            hit = memo[sig] = TRIVIAL_SCHEDULE
        if hit is not None:
            hits[sig] = hit
            continue
        blob = first_seen.get(sig) if first_seen is not None else None
        if blob is None:
            blob = _first_blob(recs_src, r)
            if first_seen is not None:
                first_seen[sig] = blob
        local_pending[sig] = blob
    pending_all = local_pending
    if extra:
        pending_all = dict(local_pending)
        for sig, blob in extra.items():
            if sig not in hits and sig not in memo:
                pending_all.setdefault(sig, blob)
    rows: dict[tuple, int] = {sig: i for i, sig in enumerate(hits)}
    # memoised signatures: resolved rows carrying their schedule (vectorised)
    hit_recs = np.zeros(len(hits), KERN_DTYPE)
    if hits:
        sch = list(hits.values())
        hit_recs["ty"] = [s.tile_y for s in sch]
        hit_recs["tx"] = [s.tile_x for s in sch]
        hit_recs["unroll"] = [s.unroll for s in sch]
        hit_recs["has_shape"] = 1
        hit_recs["sig_index"] = -1
        hit_recs["resolved"] = 1
    sig_recs = [hit_recs.tobytes()] if hits else []
    pending = []
    nsig = len(hits)
    for sig, blob in pending_all.items():
        rows[sig] = nsig
        pending.append((nsig, sig))
        sig_recs.append(blob)
        nsig += 1
    counts = [len(ct.sigs) for ct in cts]
    nk = sum(counts)
    if nk:
        kern = recs_all if use_keys else cat_records([ct.recs for ct in cts], KERN_DTYPE)
        if use_keys:
            # row of each distinct signature, broadcast through the unique inverse
            uniq_rows = np.array([rows[flat_sigs[i]] for i in first], np.int32)
            kern["sig_index"] = uniq_rows[inverse.reshape(-1)]
        else:
            kern["sig_index"] = [rows[sig] for sig in flat_sigs]
    else:
        kern = np.zeros(1, KERN_DTYPE)
    offsets = np.zeros(len(cts) + 1, np.int32)
    offsets[1:] = np.cumsum(counts)
    sig_blob = b"".join(sig_recs) if sig_recs else np.zeros(1, KERN_DTYPE).tobytes()
    blob = sig_blob + kern.tobytes()
    dev = ctx.upload_bytes(blob)
    offs = ctx.upload_array(offsets)
    tp = TracePlan(compiled if compiled is not None else [None] * len(cts), dev[len(sig_blob):],
                   dev[:len(sig_blob)], nk, nsig, pending, offsets, offs, profile, memo)
    tp._blob = dev
    tp._sig_template = sig_blob
    if conv_index:
        # the Conv2D steps of every candidate, for the dimension attacker
        rows = np.flatnonzero(kern["label"][:nk] == _LABEL_CODE[K.Conv2D]).astype(np.int32)
        tp.conv_rows = ctx.upload_array(rows if len(rows) else np.zeros(1, np.int32))
        tp.conv_off = ctx.upload_array(np.searchsorted(rows, offsets).astype(np.int32))
    return tp


def run_trace(tp: TracePlan, profile: bool = True, restore: bool = False) -> None:
    """Device half: search the unresolved signatures, resolve every kernel's
    schedule (+ strategy), profile all kernels, per-candidate T.
    ``restore`` re-uploads the pristine signature table first (a cold memo
    every call, for benchmarking)."""
    ctx = device()
    pc = tp.profile.as_c()
    sp = C.c_void_p(ctx.sp)
    if restore:
        # pristine table kept on the device: a stream-ordered D2D copy (a
        # pageable H2D here would block the host until the previous step
        # drained and leave the GPU idle while this step is enqueued)
        tmpl = getattr(tp, "_sig_template_dev", None)
        if tmpl is None:
            tmpl = tp._sig_template_dev = ctx.upload_bytes(tp._sig_template)
        tp.sigs.copy_(tmpl, non_blocking=True)
    if tp.pending:
        ctx.check(ctx.lib.tobf_schedule_search(C.c_void_p(tp.sigs.data_ptr()), tp.nsig, C.byref(pc), sp),
                  "schedule search")
        ctx.launches += 1
    ctx.check(ctx.lib.tobf_resolve_schedules(C.c_void_p(tp.kern.data_ptr()), tp.nk, C.c_void_p(tp.sigs.data_ptr()),
                                             sp), "resolve schedules")
    ctx.launches += 1
    if not profile:
        return
    if tp.feats is None:
        tp.feats = torch.empty((max(tp.nk, 1), 9), dtype=torch.float64, device=ctx.device)
        tp.totals = torch.empty(len(tp.compiled), dtype=torch.float64, device=ctx.device)
    ctx.check(ctx.lib.tobf_profile_kernels(C.c_void_p(tp.kern.data_ptr()), tp.nk, C.byref(pc),
                                           C.c_void_p(tp.feats.data_ptr()), sp), "profile")
    ctx.check(ctx.lib.tobf_trace_totals(C.c_void_p(tp.feats.data_ptr()), C.c_void_p(tp.offsets.data_ptr()),
                                        len(tp.compiled), C.c_void_p(tp.totals.data_ptr()), sp), "trace totals")
    ctx.launches += 2


def readback_trace(tp: TracePlan) -> None:
    """Enqueue finish_trace's D2H (the searched signature rows, and the
    resolved kernel rows when CompiledGraphs want them) into pinned memory
    right behind the trace stage, so finish_trace waits for this batch only,
    not for the batches launched after it."""
    ctx = device()
    need_kern = any(cg is not None for cg in tp.compiled)
    if not tp.pending and not need_kern:
        return
    ns = tp.sigs.numel()
    with torch.cuda.stream(ctx.stream):
        host = torch.empty(ns + (tp.kern.numel() if need_kern else 0), dtype=torch.uint8, pin_memory=True)
        host[:ns].copy_(tp.sigs, non_blocking=True)
        if need_kern:
            host[ns:].copy_(tp.kern, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(ctx.stream)
    tp.readback = (host, ev)


def finish_trace(tp: TracePlan) -> None:
    """Record newly searched schedules in the memo (first-seen) and attach the
    resolved schedules to the CompiledGraphs (one D2H; enqueued earlier by
    readback_trace when the caller pipelines batches)."""
    ctx = device()
    need_kern = any(cg is not None for cg in tp.compiled)
    if not tp.pending and not need_kern:
        return
    ns = tp.sigs.numel()
    rb = getattr(tp, "readback", None)
    if rb is not None:
        host, ev = rb
        ev.synchronize()
    else:
        host = torch.empty(ns + (tp.kern.numel() if need_kern else 0), dtype=torch.uint8)
        host[:ns].copy_(tp.sigs)
        if need_kern:
            host[ns:].copy_(tp.kern)
        ctx.sync()
    raw = host.numpy().tobytes()
    sigs = (N.KernDesc * max(tp.nsig, 1)).from_buffer_copy(raw[:ns])
    for i, sig in tp.pending:
        if sig not in tp.memo:
            tp.memo[sig] = Schedule(tuple(sigs[i].ty), tuple(sigs[i].tx), sigs[i].unroll)
    if not need_kern:
        return  # records built out of process: no CompiledGraph to annotate
    kern = (N.KernDesc * max(tp.nk, 1)).from_buffer_copy(raw[ns:])
    for cg, r in zip(tp.compiled, tp.offsets_host[:-1]):
        if cg is None:
            continue
        cg.schedules = [Schedule(tuple(kern[q].ty), tuple(kern[q].tx), kern[q].unroll)
                        for q in range(r, r + len(cg.kernels))]


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
        return Trace(tuple(_to_step(fh[r], cg.nodes_source, k) for r, k in zip(range(lo, hi), cg.kernels)), case)


def trace_population(items: list[tuple[Graph, dict | None, dict | None]], profile: DeviceProfile,
                     memo: dict | None = None) -> PopulationTrace:
    """compile + profile + T for a population, all arithmetic on the device."""
    tp = prepare_trace(items, profile, memo)
    run_trace(tp)
    finish_trace(tp)
    return PopulationTrace(tp.compiled, tp.feats, tp.offsets, tp.totals, tp.offsets_host)


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

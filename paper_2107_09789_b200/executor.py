"""GPU executor for obfuscated candidate graphs (drop-in for traceobf.interpreter).

``execute`` / ``equivalence_check`` keep the signatures and semantics of
interpreter.py:75-118; underneath, graphs are lowered to fused device ops
and run on libtobf.so:

* Conv2D and Linear become implicit-GEMM problems of the tcgen05 3xTF32
  kernel (Linear = full-extent convolution, its NCHW-flatten weight rows
  addressed through strides). Sole-consumer BatchNorm / ReLU / Add chains
  fold into the GEMM epilogue (selective fusion in the executor; the
  *modelled* kernel partition of the cost model is ``kernels.fuse``).
* MaxPool, unfused injective chains, Concat / Slice and SoftMax are
  grouped memory-bound ops.
* Trials are stacked along the batch dimension (trial t's element k is
  batch row t*b + k), and a whole population is lowered together: ops are
  levelled by dependency depth and every level of every candidate launches
  as ONE grouped conv kernel per N-tile width plus one grouped ew kernel.

Activation layout on the device: NHWC float32, channels padded to a
multiple of 4 with zeros (16-B vector / bulk-copy alignment).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .derived import DerivedWeight, consecutive_derived
from .engine import Arena, DeviceContext, _root, cat_records, device
from .ir import BN_EPS, Graph, OperatorKind as K, ShapeMismatch, TensorShape, analyze, shape_map, topo_order


def _rup4(c: int) -> int:
    return (c + 3) // 4 * 4


def ctx_arena(ctx: DeviceContext, floats: int) -> Arena:
    """The context's activation arena, grown on demand and reused: every run
    is ordered on the engine stream, so a later run's writes cannot overtake
    an earlier run's reads."""
    ar = ctx.__dict__.get("arena")
    if ar is None or ar.buf.numel() < floats:
        ar = Arena(ctx, int(floats * 1.1) + 4096)
        ctx.arena = ar
    ar.used = 0
    return ar


@dataclass
class Step:
    """One epilogue step: ('affine', node) | ('relu',) | ('add', value_node) | ('const', node)."""
    op: str
    ref: int = -1


@dataclass
class Op:
    kind: str                  # 'gemm' | 'pool' | 'epi' | 'copy' | 'softmax'
    out: int                   # node whose value this op materialises
    src: int                   # value node read (-1 = graph input)
    node: int = -1             # anchor node (conv/linear/pool)
    steps: list = field(default_factory=list)
    deps: list = field(default_factory=list)   # value nodes read (incl. src), -1 = input
    a0: int = 0                # copy: dst channel offset
    a1: int = 0                # copy: src channel offset
    cc: int = 0                # copy: channel count
    level: int = 0
    w: object = None           # gemm: fused sibling weight view (overrides node.weights)
    j: int = 0                 # gemm: fused output channels (overrides attrs["j"])


@dataclass
class Lowered:
    graph: Graph
    shapes: dict
    ops: list
    values: set      # node ids with a materialised buffer
    out_node: int


_CHAIN_KINDS = (K.BatchNorm, K.ReLU, K.Add)


def _consecutive_views(ws: list, axis: int):
    """If the arrays are consecutive slices of one buffer along ``axis`` (same
    dtype / strides / other extents), return the merged view, else None."""
    if any(isinstance(w, DerivedWeight) for w in ws):
        return consecutive_derived(ws, axis)
    w0 = ws[0]
    if not all(isinstance(w, np.ndarray) and w.dtype == np.float32 and w.ndim == w0.ndim and
               w.strides == w0.strides for w in ws):
        return None
    ax = axis % w0.ndim
    shape = list(w0.shape)
    expect = w0.__array_interface__["data"][0]
    total = 0
    for w in ws:
        if w.__array_interface__["data"][0] != expect:
            return None
        if any(a != b for i, (a, b) in enumerate(zip(w.shape, w0.shape)) if i != ax):
            return None
        expect += w.shape[ax] * w0.strides[ax]
        total += w.shape[ax]
    base = _root(w0)
    if base is w0 or _root(ws[-1]) is not base:
        return None
    shape[ax] = total
    return np.lib.stride_tricks.as_strided(w0, shape=tuple(shape), strides=w0.strides, writeable=False)


def _sibling_groups(graph: Graph, order, shapes, succ) -> dict:
    """Branch-layer siblings that one GEMM can compute (transforms.py:173-231):

    out-branch  Concat of conv/linear parts reading the same input, same
                geometry, weights = consecutive slices of one array along j
                -> one GEMM with N = sum(j) written into the Concat buffer;
    in-branch   Add of conv/linear parts, each reading its own channel Slice of
                one input (consecutive, covering all channels), weights =
                consecutive slices along c -> one GEMM with K = all channels
                written into the Add buffer.
    Same FLOPs as the emitted parts; returns combiner id -> (kind, parts, slices, view)."""
    nodes = graph.nodes
    groups = {}
    for nid in order:
        n = nodes[nid]
        if len(n.inputs) < 2 or n.kind not in (K.Concat, K.Add) or (n.kind is K.Add and n.weights is not None):
            continue
        parts = [nodes[p] for p in n.inputs]
        if len(set(n.inputs)) != len(n.inputs):
            continue
        if any(p.kind not in (K.Conv2D, K.Linear) or p.kind is not parts[0].kind or succ[p.id] != [nid]
               for p in parts):
            continue
        a0 = parts[0].attrs
        if parts[0].kind is K.Conv2D and any(
                (p.attrs["k1"], p.attrs["k2"], p.attrs["stride"], p.attrs["padding"]) !=
                (a0["k1"], a0["k2"], a0["stride"], a0["padding"]) for p in parts):
            continue
        if n.kind is K.Concat:
            src = parts[0].inputs
            if any(p.inputs != src for p in parts):
                continue
            view = _consecutive_views([p.weights for p in parts], -1)
            if view is not None:
                groups[nid] = ("out", [p.id for p in parts], [], view)
        else:
            slices = [nodes[p.inputs[0]] if len(p.inputs) == 1 else None for p in parts]
            if any(sl is None or sl.kind is not K.Slice or succ[sl.id] != [p.id] for sl, p in zip(slices, parts)):
                continue
            src = slices[0].inputs
            if any(sl.inputs != src for sl in slices):
                continue
            src_c = shapes[src[0]].channels if src else graph.input_shape.channels
            bounds = [(sl.attrs["start"], sl.attrs["stop"]) for sl in slices]
            if bounds[0][0] != 0 or bounds[-1][1] != src_c or any(bounds[i][1] != bounds[i + 1][0]
                                                                    for i in range(len(bounds) - 1)):
                continue
            axis = 2 if parts[0].kind is K.Conv2D else 0
            view = _consecutive_views([p.weights for p in parts], axis)
            if view is not None:
                groups[nid] = ("in", [p.id for p in parts], [sl.id for sl in slices], view)
    return groups


def lower(graph: Graph, analysis=None, fuse_siblings: bool = True) -> Lowered:
    """Partition a graph into device ops (host-only; no device needed)."""
    if analysis is None:
        analysis = analyze(graph)
    order, shapes, succ = analysis.order, analysis.shapes, analysis.succ
    nodes = graph.nodes
    covered: set[int] = set()
    ops: list[Op] = []
    produced: set[int] = set()  # value nodes already produced by an earlier op
    groups = _sibling_groups(graph, order, shapes, succ) if fuse_siblings else {}
    member = {}  # part / slice node -> combiner
    for comb, (_, parts, slices, _) in groups.items():
        for m in parts + slices:
            member[m] = comb

    def absorb(op: Op, tail: int) -> int:
        """Extend op's epilogue along sole-consumer injective successors."""
        while tail != graph.output_id:
            nxt = succ[tail]
            if len(nxt) != 1:
                break
            s = nodes[nxt[0]]
            if s.kind not in _CHAIN_KINDS:
                break
            extra = []
            if s.kind is K.BatchNorm:
                extra.append(Step("affine", s.id))
            elif s.kind is K.ReLU:
                extra.append(Step("relu"))
            else:
                others = [p for p in s.inputs if p != tail]
                if len(others) != len(s.inputs) - 1:
                    break  # same value twice
                if any(p not in produced for p in others):
                    break  # other operand not yet materialised
                extra += [Step("add", p) for p in others]
                if s.weights is not None:
                    extra.append(Step("const", s.id))
            if len(op.steps) + len(extra) > N.TOBF_MAX_EPI:
                break
            op.steps += extra
            op.deps += [st.ref for st in extra if st.op == "add"]
            covered.add(s.id)
            tail = s.id
        return tail

    for nid in order:
        if nid in covered:
            continue
        n = nodes[nid]
        comb = member.get(nid)
        if comb is not None:
            kind, parts, slices, view = groups[comb]
            covered.update(parts + slices + [comb])
            head = nodes[parts[0]]
            if kind == "out":
                src = head.inputs[0] if head.inputs else -1
            else:
                sl = nodes[slices[0]]
                src = sl.inputs[0] if sl.inputs else -1
            op = Op("gemm", comb, src, node=parts[0], deps=[src], w=view, j=shapes[comb].channels)
            op.out = absorb(op, comb)
            ops.append(op)
            produced.add(op.out)
            continue
        src = n.inputs[0] if n.inputs else -1
        if n.kind in (K.Conv2D, K.Linear):
            op = Op("gemm", nid, src, node=nid, deps=[src])
            op.out = absorb(op, nid)
        elif n.kind is K.MaxPool:
            op = Op("pool", nid, src, node=nid, deps=[src])
        elif n.kind is K.SoftMax:
            op = Op("softmax", nid, src, node=nid, deps=[src])
        elif n.kind in (K.BatchNorm, K.ReLU):
            op = Op("epi", nid, src, node=nid, deps=[src],
                    steps=[Step("affine", nid) if n.kind is K.BatchNorm else Step("relu")])
            op.out = absorb(op, nid)
        elif n.kind is K.Add:
            srcs = n.inputs if n.inputs else [-1]
            op = Op("epi", nid, srcs[0], node=nid, deps=list(srcs),
                    steps=[Step("add", p) for p in srcs[1:]])
            if n.weights is not None:
                op.steps.append(Step("const", nid))
            if len(op.steps) > N.TOBF_MAX_EPI:  # long n-ary Add: split into a chain of copies
                raise NotImplementedError("Add with more than 6 operands")
            op.out = absorb(op, nid)
        elif n.kind is K.Concat:
            off = 0
            for p in n.inputs:
                c = shapes[p].channels
                ops.append(Op("copy", nid, p, node=nid, deps=[p], a0=off, a1=0, cc=c))
                off += c
            covered.add(nid)
            produced.add(nid)
            continue
        elif n.kind is K.Slice:
            op = Op("copy", nid, src, node=nid, deps=[src], a0=0, a1=n.attrs["start"],
                    cc=n.attrs["stop"] - n.attrs["start"])
        else:
            raise NotImplementedError(n.kind)
        covered.add(nid)
        ops.append(op)
        produced.add(op.out)
    # dependency levels: level(op) = 1 + max(level of producers of its deps)
    level_of_value = {-1: 0}
    concat_level: dict[int, int] = {}
    for op in ops:
        lv = 1 + max(level_of_value[d] for d in op.deps)
        op.level = lv
        if op.kind == "copy" and nodes[op.out].kind is K.Concat:
            concat_level[op.out] = max(concat_level.get(op.out, 0), lv)
            level_of_value[op.out] = concat_level[op.out]
        else:
            level_of_value[op.out] = lv
    values = {op.out for op in ops}
    return Lowered(graph, shapes, ops, values, graph.output_id)


# ---------------------------------------------------------------------------
# Forward plans: one graph's forward as descriptor rows with SYMBOLIC
# pointers (host only, picklable — built in worker processes for a
# population), linked to device memory and launched by PopulationRun
# ---------------------------------------------------------------------------

CONV_DTYPE = np.dtype(N.ConvDesc)
EW_DTYPE = np.dtype(N.EwDesc)
_NO_EPI = (0, 0, 0)

# A symbolic pointer is (space << 56) | value: value = byte offset into the
# graph's activation block (SP_ARENA) or an index into one of the plan's
# requirement tables (packed weight images, folded BatchNorms, constants).
SP_INPUT, SP_ARENA, SP_WIMG, SP_AFFINE, SP_CONST, SP_XCOL = 1, 2, 3, 4, 5, 6
_SP_SHIFT = 56
_SP_LOW = (1 << _SP_SHIFT) - 1


def _sym(space: int, value: int) -> int:
    return (space << _SP_SHIFT) | value


class ArrayRefs:
    """Host arrays <-> hashable references ``(root_key, byte_offset, shape,
    strides)``. In process a root is keyed by identity; the worker-side
    registry (hostpipe.py) names roots its parent can rebuild instead."""

    def __init__(self):
        self._roots: dict = {}

    def root_key(self, root: np.ndarray):
        key = ("id", id(root))
        self._roots[key] = root
        return key

    def root(self, key) -> np.ndarray:
        return self._roots[key]

    def ref(self, a) -> tuple:
        if isinstance(a, DerivedWeight):  # knob-derived weight: its vanilla base + the gather
            return ("D", self.ref(a.base)) + a.key()
        r = _root(a)
        off = a.__array_interface__["data"][0] - r.__array_interface__["data"][0]
        return (self.root_key(r), off, a.shape, a.strides)

    def resolve(self, ref: tuple):
        if ref[0] == "D":
            return DerivedWeight(self.resolve(ref[1]), *ref[2:])
        key, off, shape, strides = ref
        r = self.root(key)
        if off == 0 and shape == r.shape and strides == r.strides:
            return r
        return np.ndarray(shape, r.dtype, buffer=r, offset=off, strides=strides)


@dataclass
class ForwardPlan:
    """conv/ew: descriptor rows (symbolic pointers) with their launch keys
    (dependency level, BN, K); wimg/affine/const: requirement tables;
    arena_bytes: the graph's activation block; out_off: its output value."""

    conv: np.ndarray
    conv_level: np.ndarray
    conv_bn: np.ndarray
    conv_k: np.ndarray
    ew: np.ndarray
    ew_level: np.ndarray
    wimg: list      # (weight ref, is_conv, in_h, in_w, in_c, k1, k2, cp, j, bn, prec)
    affine: list    # BatchNorm weight ref
    const: list     # (constant ref, b0, channels, h, w, cp)
    arena_bytes: int
    out_off: int
    out_shape: TensorShape
    input_shape: TensorShape
    flops_per_image: int
    gemm_act_bytes_per_image: int = 0   # conv/linear input + output activations, fp32, once each
    gemm_weight_bytes: int = 0          # conv/linear weights, fp32, once
    prec: int = N.PREC_TF32X3           # conv arithmetic (N.PRECISIONS)
    # im2col matrices of the staged input the plan's input convs read
    # (batch, H, W, c, k1, k2, stride, pad, Ho, Wo, Kp): see INPUT_IM2COL
    xcol: list = field(default_factory=list)


def _plan_getstate(self) -> dict:
    """Pickle the descriptor tables as raw bytes: numpy rebuilds nested
    structured dtypes field by field on unpickling (~20 us per array), which
    the parent pays for every candidate a host worker sends."""
    st = dict(self.__dict__)
    st["conv"], st["ew"] = self.conv.tobytes(), self.ew.tobytes()
    return st


def _plan_setstate(self, st: dict) -> None:
    st = dict(st)
    st["conv"] = np.frombuffer(st["conv"], dtype=CONV_DTYPE).copy()
    st["ew"] = np.frombuffer(st["ew"], dtype=EW_DTYPE).copy()
    self.__dict__.update(st)


ForwardPlan.__getstate__ = _plan_getstate
ForwardPlan.__setstate__ = _plan_setstate


def _gemm_geom(lw: Lowered, op: Op, s_in: TensorShape):
    n = lw.graph.nodes[op.node]
    j = op.j or n.attrs["j"]
    if n.kind is K.Conv2D:
        return n.attrs["k1"], n.attrs["k2"], _rup4(s_in.channels), j
    return s_in.height, s_in.width, _rup4(s_in.channels), j


def plan_forward(lw: Lowered, reps: int, refs: ArrayRefs, prec: int = N.PREC_TF32X3) -> ForwardPlan:
    """Descriptor rows of one lowered graph for ``reps`` stacked trials, its
    convs in precision ``prec`` (N.PREC_TF32X3 / N.PREC_BF16)."""
    graph, shapes, nodes = lw.graph, lw.shapes, lw.graph.nodes
    ishape = graph.input_shape
    batch = ishape.batch * reps
    offs: dict[int, int] = {}
    used = 0
    for v in sorted(lw.values):
        sh = shapes[v]
        offs[v] = used
        used += 4 * Arena.round(batch * sh.height * sh.width * _rup4(sh.channels))

    def buf(v: int) -> int:
        return _sym(SP_INPUT, 0) if v < 0 else _sym(SP_ARENA, offs[v])

    tables: dict[str, tuple[dict, list]] = {"wimg": ({}, []), "affine": ({}, []), "const": ({}, []), "xcol": ({}, [])}

    def index(table: str, entry) -> int:
        idx, lst = tables[table]
        i = idx.get(entry)
        if i is None:
            i = idx[entry] = len(lst)
            lst.append(entry)
        return i

    def epi_rows(steps: list) -> list:
        out = []
        for st in steps:
            if st.op == "affine":
                out.append((N.EPI_AFFINE, _rup4(shapes[st.ref].channels),
                            _sym(SP_AFFINE, index("affine", refs.ref(nodes[st.ref].weights)))))
            elif st.op == "relu":
                out.append((N.EPI_RELU, 0, 0))
            elif st.op == "add":
                sh = shapes[st.ref] if st.ref >= 0 else ishape
                out.append((N.EPI_ADD_TENSOR, _rup4(sh.channels), buf(st.ref)))
            elif st.op == "const":
                sh = shapes[st.ref]
                entry = (refs.ref(nodes[st.ref].weights), ishape.batch, sh.channels, sh.height, sh.width,
                         _rup4(sh.channels))
                out.append((N.EPI_ADD_CONST, ishape.batch, _sym(SP_CONST, index("const", entry))))
        return out + [_NO_EPI] * (N.TOBF_MAX_EPI - len(out))

    conv_rows, conv_lv, conv_bn, conv_k = [], [], [], []
    ew_rows, ew_lv = [], []
    flops = 0
    act_bytes = w_bytes = 0
    for op in lw.ops:
        s_in = shapes[op.src] if op.src >= 0 else ishape
        s_out = shapes[op.out]
        if op.kind == "gemm":
            n = nodes[op.node]
            k1, k2, cp, j = _gemm_geom(lw, op, s_in)
            bn = 128 if j > 64 else 64
            if n.kind is K.Conv2D:
                stride, pad = n.attrs["stride"], n.attrs["padding"]
                flops += 2 * ishape.batch * shapes[op.node].height * shapes[op.node].width * j * k1 * k2 * s_in.channels
            else:
                stride, pad = 1, 0
                flops += 2 * ishape.batch * j * s_in.channels * s_in.height * s_in.width
            act_bytes += 4 * ishape.batch * (s_in.height * s_in.width * s_in.channels +
                                             s_out.height * s_out.width * j)
            w_bytes += 4 * k1 * k2 * s_in.channels * j
            w = n.weights if op.w is None else op.w
            epi = epi_rows(op.steps)
            nepi = sum(1 for e in epi if e[0])
            kx = -(-(k1 * k2 * s_in.channels) // 32) * 32
            if (INPUT_IM2COL and op.src < 0 and n.kind is K.Conv2D and cp % 32 and k1 * k2 > 1 and kx <= 3072
                    and batch * shapes[op.node].height * shapes[op.node].width * kx < (1 << 33)):
                # a conv reading the staged input with few channels: a 1x1 GEMM
                # over the input's im2col matrix (shared by every candidate of
                # the run, built once per staged input), K = k1*k2*c rounded up
                # to 32 (RN18 stem: 160 instead of 7x7x4 = 196 -> 224), A by TMA
                ho, wo, kp = s_out.height, s_out.width, kx
                xi = index("xcol", (batch, s_in.height, s_in.width, s_in.channels, k1, k2, stride, pad, ho, wo, kp))
                wi = index("wimg", (refs.ref(w), 2, s_in.height, s_in.width, s_in.channels, k1, k2, kp, j, bn, prec))
                conv_rows.append((_sym(SP_XCOL, xi), _sym(SP_WIMG, wi), buf(op.out), batch, ho, wo, kp, ho, wo,
                                  _rup4(j), j, 1, 1, 1, 0, 0, 0, 0, 0, 0, nepi, kp, _rup4(j), epi, 0, 0, 1, 0, 0, 0, 0, 0, 0))
                conv_lv.append(op.level)
                conv_bn.append(bn)
                conv_k.append(kp)
                continue
            wi = index("wimg", (refs.ref(w), n.kind is K.Conv2D, s_in.height, s_in.width, s_in.channels,
                                k1, k2, cp, j, bn, prec))
            conv_rows.append((buf(op.src), _sym(SP_WIMG, wi), buf(op.out), batch, s_in.height, s_in.width, cp,
                              s_out.height, s_out.width, _rup4(j), j, k1, k2, stride, pad, 0, 0, 0, 0, 0,
                              nepi, cp, _rup4(j), epi, 0, 0, 1, 0, 0, 0, 0, 0, 0))
            conv_lv.append(op.level)
            conv_bn.append(bn)
            conv_k.append(k1 * k2 * cp)
            continue
        ldx, ldy = _rup4(s_in.channels), _rup4(s_out.channels)
        epi = [_NO_EPI] * N.TOBF_MAX_EPI
        nepi = 0
        if op.kind == "pool":
            n = nodes[op.node]
            head = (N.OP_MAXPOOL, batch, s_in.height, s_in.width, s_in.channels, ldx, s_out.height,
                    s_out.width, ldy, n.attrs["window"], n.attrs["stride"])
            cpo = _rup4(s_in.channels)
        elif op.kind == "epi":
            epi = epi_rows(op.steps)
            nepi = sum(1 for e in epi if e[0])
            head = (N.OP_EPI, batch, s_in.height, s_in.width, s_out.channels, ldx, s_out.height,
                    s_out.width, ldy, 0, 0)
            cpo = _rup4(s_out.channels)
        elif op.kind == "copy":
            total = s_out.channels
            head = (N.OP_COPYCH, batch, s_in.height, s_in.width, op.cc, ldx, 0, 0, ldy, op.a0, op.a1)
            cpo = _rup4(total) if op.a0 + op.cc == total else op.a0 + op.cc
        else:  # softmax
            head = (N.OP_SOFTMAX, batch, s_in.height, s_in.width, s_in.channels, ldx, 0, 0, ldy, 0, 0)
            cpo = _rup4(s_in.channels)
        ew_rows.append((buf(op.src), buf(op.out)) + head + (nepi, 0, cpo, 0, epi))
        ew_lv.append(op.level)
    return ForwardPlan(
        conv=np.array(conv_rows, dtype=CONV_DTYPE) if conv_rows else np.zeros(0, CONV_DTYPE),
        conv_level=np.array(conv_lv, np.int32), conv_bn=np.array(conv_bn, np.int32),
        conv_k=np.array(conv_k, np.int64),
        ew=np.array(ew_rows, dtype=EW_DTYPE) if ew_rows else np.zeros(0, EW_DTYPE),
        ew_level=np.array(ew_lv, np.int32),
        wimg=tables["wimg"][1], affine=tables["affine"][1], const=tables["const"][1],
        arena_bytes=used, out_off=offs[lw.out_node], out_shape=shapes[lw.out_node], input_shape=ishape,
        flops_per_image=flops, gemm_act_bytes_per_image=act_bytes, gemm_weight_bytes=w_bytes, prec=prec,
        xcol=tables["xcol"][1])


def _link(col: np.ndarray, row_plan: np.ndarray, x_ptr: int, arena: np.ndarray, tables: dict) -> np.ndarray:
    """Symbolic -> device pointers for one pointer column (rows x k), rows of
    several plans at once (row_plan = plan index of each row)."""
    col = col.astype(np.uint64, copy=False)
    space = (col >> np.uint64(_SP_SHIFT)).astype(np.int64)
    val = (col & np.uint64(_SP_LOW)).astype(np.int64)
    rp = row_plan.reshape((-1,) + (1,) * (col.ndim - 1))
    rp = np.broadcast_to(rp, col.shape)
    out = np.zeros(col.shape, np.uint64)
    m = space == SP_INPUT
    out[m] = np.uint64(x_ptr)
    m = space == SP_ARENA
    out[m] = (arena[rp[m]] + val[m]).astype(np.uint64)
    for sp, (ptrs, offsets) in tables.items():
        m = space == sp
        if m.any():
            out[m] = ptrs[offsets[rp[m]] + val[m]]
    return out


SPLITK_MAX = 16  # work units per tile at most
#: A operand by TMA im2col where eligible (TOBF_CONV_TMA=0: cp.async gather everywhere, A/B measurements)
TMA_A = __import__("os").environ.get("TOBF_CONV_TMA", "1") != "0"
#: launches whose problems all take A by TMA run the kernel variant without the
#: cp.async gather (TOBF_CONV_TMA_ALL=0: the mixed-mode variant, A/B measurements)
TMA_ALL = __import__("os").environ.get("TOBF_CONV_TMA_ALL", "1") != "0"
#: convs reading the graph input with c % 32 != 0 as 1x1 GEMMs over its im2col (TOBF_INPUT_IM2COL=0: direct)
INPUT_IM2COL = __import__("os").environ.get("TOBF_INPUT_IM2COL", "1") != "0"


def conv_sched(ctx: DeviceContext) -> torch.Tensor:
    """The context's launch-wide conv tile-claim counters (2 x int32, zero
    between launches: each launch's last CTA re-zeroes them). Every conv
    launch of a context is ordered on its engine stream, so one pair serves
    them all."""
    t = ctx.__dict__.get("conv_sched")
    if t is None:
        t = ctx.conv_sched = torch.zeros(2, dtype=torch.int32, device=ctx.device)
    return t


def splitk_workspace(ctx: DeviceContext, floats: int, counters: int):
    """The context's split-K workspace (partial tiles) and per-tile arrival
    counters, grown on demand. Shared by every conv launch: they are ordered
    on the engine stream, and the last unit of each tile re-zeroes its counter."""
    ws, cnt = ctx.__dict__.get("splitk_ws"), ctx.__dict__.get("splitk_cnt")
    if ws is None or ws.numel() < floats:
        ws = torch.empty(int(floats * 1.25) + 1024, dtype=torch.float32, device=ctx.device)
        ctx.splitk_ws = ws
    if cnt is None or cnt.numel() < counters:
        # a fresh zeroed buffer: counters of the old one may be mid-launch
        cnt = torch.zeros(int(counters * 1.25) + 256, dtype=torch.int32, device=ctx.device)
        ctx.splitk_cnt = cnt
    return ws, cnt


def _runs(keys: np.ndarray) -> list[tuple[int, int]]:
    """[lo, hi) runs of equal consecutive rows of a sorted (n, k) key array."""
    n = len(keys)
    if not n:
        return []
    b = (np.flatnonzero(np.any(keys[1:] != keys[:-1], axis=1)) + 1).tolist()
    return list(zip([0] + b, b + [n]))


#: tail alignment (TOBF_TAIL_ALIGN, a fraction of each graph's depth; 0 = off):
#: the ops of a graph at dependency levels >= f * its depth are shifted so that
#: every graph of the population ends at the same level (RN18 headline step,
#: same box: f = 0 2836, 0.3 2945, 0.5 2960, 0.7 2936, 0.9 2822 candidates/s)
TAIL_ALIGN = float(__import__("os").environ.get("TOBF_TAIL_ALIGN", "0.5"))


def _aligned_levels(plans: list) -> tuple[np.ndarray, np.ndarray]:
    """Launch levels of every plan's conv and ew rows. The population's graphs
    differ in depth (deepening adds layers), so with as-soon-as-possible levels
    the last layers of the deep candidates run alone in the final levels —
    small problems (7x7 spatial, the FC) that fill a fraction of the SMs. With
    TAIL_ALIGN = f, a graph's ops at levels >= f * depth move down by its slack
    (population depth - its depth): shifting a suffix of levels by one amount
    keeps every producer before its consumers, and the tails of all graphs
    share launches."""
    conv = [p.conv_level for p in plans]
    ew = [p.ew_level for p in plans]
    if TAIL_ALIGN <= 0 or len(plans) < 2:
        return np.concatenate(conv), np.concatenate(ew)
    depth = [max(int(c.max(initial=0)), int(e.max(initial=0))) for c, e in zip(conv, ew)]
    top = max(depth)
    out_c, out_e = [], []
    for c, e, dp in zip(conv, ew, depth):
        t = int(np.ceil(TAIL_ALIGN * dp))
        slack = top - dp
        out_c.append(np.where(c >= t, c + slack, c))
        out_e.append(np.where(e >= t, e + slack, e))
    return np.concatenate(out_c), np.concatenate(out_e)


#: stem pairing (TOBF_PAIR_STEMS=0: off): see _pair_stems
PAIR_STEMS = __import__("os").environ.get("TOBF_PAIR_STEMS", "1") != "0"


def _stem_key(p: "ForwardPlan", r: np.ndarray, bn: int):
    """Pairing key of a conv row reading the input's im2col matrix (None if it
    may not pair): its matrix, its weight entry, its output row stride and its
    epilogue chain (folded BatchNorm and/or ReLU only, the same ops)."""
    space, val = int(np.uint64(r["x"]) >> np.uint64(_SP_SHIFT)), int(np.uint64(r["x"]) & np.uint64(_SP_LOW))
    if space != SP_XCOL or bn != 64 or int(r["j"]) != 64 or int(r["Cpo"]) != 64:
        return None
    ops = []
    for e in r["epi"][:int(r["nepi"])]:
        op = int(e["op"])
        if op not in (N.EPI_AFFINE, N.EPI_RELU) or (op == N.EPI_AFFINE and N.EPI_AFFINE in ops):
            return None
        ops.append(op)
    wsp, wi = int(np.uint64(r["wimg"]) >> np.uint64(_SP_SHIFT)), int(np.uint64(r["wimg"]) & np.uint64(_SP_LOW))
    if wsp != SP_WIMG:
        return None
    return (p.xcol[val], p.wimg[wi], int(r["ldy"]), tuple(ops), tuple(int(e["aux"]) for e in r["epi"][:int(r["nepi"])]))


def _pair_stems(plans, conv, conv_plan, level, launch_level, conv_bn, tables) -> np.ndarray | None:
    """Stems of different candidates read the same A (the staged input's
    im2col matrix) and usually the same weights (most candidates leave the
    stem alone): two such 64-channel problems of one launch run as ONE
    128-channel problem (tobf_conv_desc.pair) over a weight image holding the
    weights twice — the MMA at N = 128 (2048 vs 1470 MAC/clk/SM), half the A
    staging and half the tiles. Each half keeps its own output buffer and
    folded BatchNorm, so every output bit equals the unpaired run's (same K
    order, same per-element sums). Returns the rows to keep (None: no pair).
    The symbolic rows of the plans are left untouched; `conv` is linked."""
    offs = np.zeros(len(plans) + 1, np.int64)
    np.cumsum([len(p.conv) for p in plans], out=offs[1:])
    groups: dict = {}
    for pi, p in enumerate(plans):
        if not p.xcol:
            continue
        rows = np.nonzero((p.conv["x"] >> np.uint64(_SP_SHIFT)) == SP_XCOL)[0]  # the few input convs
        for k in rows.tolist():
            i = offs[pi] + k
            key = _stem_key(p, p.conv[k], int(conv_bn[i]))
            if key is not None:
                groups.setdefault(key + (int(level[i]), int(launch_level[i])), []).append(i)
    drop = []
    for key, rows in groups.items():
        for a, b in zip(rows[0::2], rows[1::2]):
            img = tables.pair_image(key[1])
            ra, rb = conv[a], conv[b]
            aff = [k for k, e in enumerate(rb["epi"][:int(rb["nepi"])]) if int(e["op"]) == N.EPI_AFFINE]
            conv["j"][a] = 128
            conv["Cpo"][a] = 128
            conv["wimg"][a] = np.uint64(img)
            conv["pair"][a] = 1
            conv["y2"][a] = rb["y"]
            conv["aff2"][a] = rb["epi"][aff[0]]["ptr"] if aff else np.uint64(0)
            conv_bn[a] = 128
            drop.append(b)
    if not drop:
        return None
    keep = np.ones(len(conv), bool)
    keep[drop] = False
    return keep


class TensorMapStore:
    """Device home of the conv A-operand tensor maps (128-B CUtensorMaps in
    global memory): one large ring, written front to back, one H2D per run.
    The TMA unit caches tensor maps by address; a fresh buffer per run could
    land where an earlier run's different maps had been, and only timing
    would keep a cached copy from being used. In the ring an address holds a
    new map only after 2^19 others were written (several hundred runs of the
    headline population), long after any cached copy is gone. (The wrong
    forwards scripts/race_probe.py found were the A-staging release race in
    conv_tc.cu, not this.)"""

    SLOTS = 1 << 19  # 64 MB of maps

    def __init__(self, ctx: DeviceContext):
        self.ctx = ctx
        self.buf = torch.empty(128 * self.SLOTS + 128, dtype=torch.uint8, device=ctx.device)
        self.base = (self.buf.data_ptr() + 127) & ~127
        self.next = 0

    def place(self, maps: np.ndarray) -> np.ndarray:
        """Device addresses of ``maps`` (rows of 128 B), copied in."""
        n = len(maps)
        if n > self.SLOTS:
            raise MemoryError("more tensor maps than the store holds")
        if self.next + n > self.SLOTS:
            self.next = 0
        off = self.next
        self.next += n
        start = self.base - self.buf.data_ptr() + 128 * off
        self.ctx._staged(np.ascontiguousarray(maps).reshape(-1), self.buf[start:start + 128 * n])
        return (self.base + 128 * (off + np.arange(n, dtype=np.uint64))).astype(np.uint64)


def _regroup(conv: np.ndarray, conv_tma: np.ndarray, level: np.ndarray, bn: np.ndarray, k: np.ndarray):
    """Prepared conv rows (K/tiles/split-K filled) regrouped into one launch
    per (level, BN), long K first: tile_start prefixes and the split-K
    workspace / counter offsets (NULL-based bytes, rebased by the caller)
    recomputed per group, each descriptor's ksplit/kper kept."""
    order = np.lexsort((-k, -bn, level))
    conv, conv_tma = conv[order], conv_tma[order]
    key = np.stack([level[order], bn[order]], 1)
    launches = []
    ws_need = cnt_need = 0
    for lo, hi in _runs(key):
        g = conv[lo:hi]
        tiles = g["mtiles"].astype(np.int64) * g["ntiles"]
        units = tiles * g["ksplit"]
        start = np.zeros(hi - lo, np.int64)
        np.cumsum(units[:-1], out=start[1:])
        g["tile_start"] = start
        split = g["ksplit"] > 1
        b = int(key[lo, 1])
        wsf = np.where(split, units * kBM_ROWS * b, 0)
        cnts = np.where(split, tiles, 0)
        wo = np.zeros(hi - lo, np.int64)
        co = np.zeros(hi - lo, np.int64)
        np.cumsum(wsf[:-1], out=wo[1:])
        np.cumsum(cnts[:-1], out=co[1:])
        g["ws"] = np.where(split, 4 * wo, 0).astype(np.uint64)
        g["cnt"] = np.where(split, 4 * co, 0).astype(np.uint64)
        conv[lo:hi] = g
        ws_need, cnt_need = max(ws_need, int(wsf.sum())), max(cnt_need, int(cnts.sum()))
        tma_flag = (N.CONV_TMA | (N.CONV_TMA_ALL if TMA_ALL and conv_tma[lo:hi].all() else 0)) if conv_tma[lo:hi].any() else 0
        launches.append((int(key[lo, 0]), 0, "conv", lo, hi - lo, int(units.sum()), b | tma_flag))
    return conv, conv_tma, launches, ws_need, cnt_need


kBM_ROWS = 128  # rows of a conv tile (conv_tc.cu kBM): a split-K partial tile is kBM_ROWS x BN floats


class PlanTables:
    """Requirement tables of ForwardPlans resolved to device pointers, one
    plan at a time: packed weight images (cached per weight view in the
    context: every candidate reusing a vanilla layer, a branch slice of it or
    a shared knob constant shares one image), folded BatchNorms, staged
    constants. ``add`` may run while later plans are still being prepared
    (evaluate_records resolves each candidate as its worker result arrives);
    the pack / staging kernels it launches are stream-ordered before the
    forward."""

    def __init__(self, ctx: DeviceContext, refs: ArrayRefs):
        self.ctx, self.refs = ctx, refs
        if ctx.wimg_bytes > ctx.WIMG_LIMIT:
            ctx.reset_wimg()  # a long GA run: bound the packed-image cache between batches
        self.rows: list[tuple[list, list, list, list]] = []  # per plan: (wimg, affine, const, xcol) pointers
        # every device buffer a pointer was handed out for, held for the life of
        # the run: a context cache may drop its entry (size bound) mid-batch
        self.keep: list = []
        self._wimg_memo: dict = {}
        self._const_memo: dict = {}
        # im2col matrices of the staged input (geometry -> device buffer),
        # filled by PopulationRun.set_input before the forward reads them
        self.xcol: dict = {}

    def add(self, plans: list) -> None:
        aff = self._affine_ptrs(list({r for p in plans for r in p.affine}))
        wm, cm = self._wimg_memo, self._const_memo
        for p in plans:
            w = []
            for e in p.wimg:
                v = wm.get(e)
                if v is None:
                    v = wm[e] = self._wimg_ptr(e)
                w.append(v)
            c = []
            for e in p.const:
                v = cm.get(e)
                if v is None:
                    v = cm[e] = self._const_ptr(e)
                c.append(v)
            x = []
            for e in p.xcol:
                buf = self.xcol.get(e)
                if buf is None:
                    buf = self.xcol[e] = self._xcol_buffer(e)
                x.append(buf.data_ptr())
            self.rows.append((w, [aff[e] for e in p.affine], c, x))

    def table(self, i: int) -> tuple[np.ndarray, np.ndarray]:
        """Column ``i`` (0 wimg, 1 affine, 2 const, 3 xcol) of every plan concatenated
        (+ a 0 sentinel) and each plan's offset into it."""
        lens = np.array([len(r[i]) for r in self.rows], np.int64)
        offsets = np.zeros(len(self.rows), np.int64)
        np.cumsum(lens[:-1], out=offsets[1:])
        flat = [v for r in self.rows for v in r[i]]
        return np.array(flat + [0], np.uint64), offsets

    def _xcol_buffer(self, geom: tuple) -> torch.Tensor:
        """Device buffer of one input im2col matrix (batch*Ho*Wo rows of Kp),
        cached per geometry in the context (the runs are stream-ordered)."""
        batch, _, _, _, _, _, _, _, ho, wo, kp = geom
        cache = self.ctx.__dict__.setdefault("xcol_cache", {})
        buf = cache.get(geom)
        if buf is None:
            if len(cache) > 16:
                cache.clear()
            buf = cache[geom] = torch.empty(batch * ho * wo * kp, dtype=torch.float32, device=self.ctx.device)
        self.keep.append(buf)
        return buf

    def pair_image(self, entry: tuple) -> int:
        """Weight image of a paired stem (executor._pair_stems): the im2col
        weight of ``entry`` twice along N (rows 0-63 and 64-127 of one
        BN = 128 tile), cached like every image."""
        ref, is_conv, in_h, in_w, in_c, k1, k2, cp, j, bn, prec = entry
        hit = self._wimg_memo.get(("pair",) + entry)
        if hit is None:
            hit = self._wimg_memo[("pair",) + entry] = self._xcol_wimg_ptr(self.refs.resolve(ref), in_c, k1, k2, cp, j,
                                                                         128, prec, twice=True)
        return hit

    def _xcol_wimg_ptr(self, w, in_c, k1, k2, kp, j, bn, prec, twice: bool = False) -> int:
        """Weight image of an input conv run as a 1x1 GEMM over the input's
        im2col: K index (u*k2 + v)*c + ch of the (k1, k2, c, j) weight, packed
        through gather maps (the flattened (u, v, c) offsets; knob-derived
        weights compose their own maps and scales into them)."""
        ctx, lib = self.ctx, self.ctx.lib
        if isinstance(w, DerivedWeight):
            wptr, st = ctx.cached_view(w.base)
            mu, mv, mc, mn, s_c, s_n = w.maps()
            if (len(mu), len(mv), len(mc), len(mn)) != (k1, k2, in_c, j):
                raise ShapeMismatch(-1, f"derived weight maps {(len(mu), len(mv), len(mc), len(mn))} "
                                        f"!= conv geometry {(k1, k2, in_c, j)}")
            key = ("XD", wptr, st, w.key(), k1, k2, in_c, kp, j, bn, prec, twice)
        else:
            wptr, st = ctx.cached_view(w)
            mu, mv, mc, mn = np.arange(k1), np.arange(k2), np.arange(in_c), np.arange(j)
            s_c, s_n = np.ones(in_c, np.float32), np.ones(j, np.float32)
            key = ("X", wptr, st, k1, k2, in_c, kp, j, bn, prec, twice)
        if twice:  # the output channels twice: rows n and j + n of the image are channel n
            mn, s_n, j = np.concatenate([mn, mn]), np.concatenate([s_n, s_n]), 2 * j
        cache = ctx.__dict__.setdefault("wimg_cache", {})
        hit = cache.get(key)
        if hit is not None:
            self.keep.append(hit[0])
            return hit[0].data_ptr()
        su, sv, sc, sn = st
        mu, mv, mc = (np.asarray(m, np.int64) for m in (mu, mv, mc))
        off = (mu[:, None, None] * su + mv[None, :, None] * sv + mc[None, None, :] * sc)
        bad = (mu[:, None, None] < 0) | (mv[None, :, None] < 0) | (mc[None, None, :] < 0)
        flat = np.where(bad, -1, off).reshape(-1)
        kk = k1 * k2 * in_c
        imaps = np.concatenate([[0, 0], flat, np.asarray(mn, np.int64)]).astype(np.int32)
        scales = np.concatenate([np.tile(np.asarray(s_c, np.float32), k1 * k2), np.asarray(s_n, np.float32)])
        blob = ctx.upload_array(np.concatenate([imaps, scales.view(np.int32)]))
        maps, sdev = blob, blob[len(imaps):]
        nbytes = lib.tobf_wimg_bytes_ex(1, 1, kp, j, bn, prec)
        img = torch.empty(nbytes // 4, dtype=torch.float32, device=ctx.device)
        ctx.wimg_bytes += nbytes
        ctx.check(lib.tobf_pack_weights_ex(C.c_void_p(wptr), 1, 1, kk, kp, j, 0, 0, 1, sn,
                                           C.c_void_p(maps.data_ptr()), C.c_void_p(sdev.data_ptr()), bn, prec,
                                           C.c_void_p(img.data_ptr()), C.c_void_p(ctx.sp)), "pack im2col weights")
        ctx.launches += 1
        cache[key] = (img, maps, sdev)
        self.keep.append(img)
        return img.data_ptr()

    def _wimg_ptr(self, entry: tuple) -> int:
        ctx, lib = self.ctx, self.ctx.lib
        ref, is_conv, in_h, in_w, in_c, k1, k2, cp, j, bn, prec = entry
        w = self.refs.resolve(ref)
        if is_conv == 2:
            return self._xcol_wimg_ptr(w, in_c, k1, k2, cp, j, bn, prec)
        if isinstance(w, DerivedWeight):
            return self._derived_wimg_ptr(w, is_conv, in_h, in_w, in_c, k1, k2, cp, j, bn, prec)
        wptr, st = ctx.cached_view(w)
        if is_conv:
            su, sv, sc, sn = st
        else:
            r, cstride = st
            su, sv, sc, sn = in_w * r, r, in_h * in_w * r, cstride
        key = (wptr, su, sv, sc, sn, k1, k2, in_c, cp, j, bn, prec)
        cache = ctx.__dict__.setdefault("wimg_cache", {})
        hit = cache.get(key)
        if hit is not None:
            self.keep.append(hit)
            return hit.data_ptr()
        nbytes = lib.tobf_wimg_bytes_ex(k1, k2, cp, j, bn, prec)
        img = torch.empty(nbytes // 4, dtype=torch.float32, device=ctx.device)
        ctx.wimg_bytes += nbytes
        ctx.check(lib.tobf_pack_weights_ex(C.c_void_p(wptr), k1, k2, in_c, cp, j, su, sv, sc, sn, None, None, bn,
                                           prec, C.c_void_p(img.data_ptr()), C.c_void_p(ctx.sp)), "pack weights")
        ctx.launches += 1
        cache[key] = img
        self.keep.append(img)
        return img.data_ptr()

    def _derived_wimg_ptr(self, w: DerivedWeight, is_conv, in_h, in_w, in_c, k1, k2, cp, j, bn, prec) -> int:
        """Weight image of a knob-derived weight, packed on the device straight
        from the resident vanilla array through the gather maps (derived.py);
        only the maps (a few KB) cross PCIe."""
        ctx, lib = self.ctx, self.ctx.lib
        wptr, st = ctx.cached_view(w.base)
        if is_conv:
            su, sv, sc, sn = st
        else:
            r, cstride = st
            H, W = w.hw
            su, sv, sc, sn = W * r, r, H * W * r, cstride
        key = ("D", wptr, su, sv, sc, sn, w.key(), k1, k2, in_c, cp, j, bn, prec)
        cache = ctx.__dict__.setdefault("wimg_cache", {})
        hit = cache.get(key)
        if hit is not None:
            self.keep.append(hit[0])
            return hit[0].data_ptr()
        mu, mv, mc, mn, s_c, s_n = w.maps()
        if (len(mu), len(mv), len(mc), len(mn)) != (k1, k2, in_c, j):
            raise ShapeMismatch(-1, f"derived weight maps {(len(mu), len(mv), len(mc), len(mn))} "
                                    f"!= conv geometry {(k1, k2, in_c, j)}")
        # maps (int32) and scales (float32) in one upload
        imaps = np.concatenate([mu, mv, mc, mn]).astype(np.int32)
        blob = ctx.upload_array(np.concatenate([imaps, np.concatenate([s_c, s_n]).astype(np.float32).view(np.int32)]))
        maps, scales = blob, blob[len(imaps):]
        nbytes = lib.tobf_wimg_bytes_ex(k1, k2, cp, j, bn, prec)
        img = torch.empty(nbytes // 4, dtype=torch.float32, device=ctx.device)
        ctx.wimg_bytes += nbytes
        ctx.check(lib.tobf_pack_weights_ex(C.c_void_p(wptr), k1, k2, in_c, cp, j, su, sv, sc, sn,
                                           C.c_void_p(maps.data_ptr()), C.c_void_p(scales.data_ptr()), bn, prec,
                                           C.c_void_p(img.data_ptr()), C.c_void_p(ctx.sp)), "pack derived weights")
        ctx.launches += 1
        cache[key] = (img, maps, scales)  # maps stay alive until the (async) pack has run
        self.keep.append(img)
        return img.data_ptr()

    def _affine_ptrs(self, refs_needed: list) -> dict:
        """Fold every BatchNorm the epilogues use into (a, b) with
        a = scale/sqrt(var+eps), b = shift - mean*a (fp64 -> fp32), cached by
        weight-array identity; all misses go up in ONE H2D."""
        cache = self.ctx.__dict__.setdefault("affine_cache", {})
        out, misses = {}, {}
        for ref in refs_needed:
            w = self.refs.resolve(ref)
            hit = cache.get(id(w))
            if hit is not None and hit[0] is w:
                out[ref] = hit[2]
                self.keep.append(hit[1])
            else:
                misses[ref] = w
        if misses:
            blocks, offs, total = [], [], 0
            for w in misses.values():
                w64 = w.astype(np.float64)
                a = w64[0] / np.sqrt(w64[3] + BN_EPS)
                b = w64[1] - w64[2] * a
                cp = _rup4(w.shape[1])
                blk = np.zeros((2, cp), np.float32)
                blk[0, :w.shape[1]] = a
                blk[1, :w.shape[1]] = b
                offs.append(total)
                blocks.append(blk.reshape(-1))
                total += Arena.round(2 * cp)
            host = np.zeros(total, np.float32)
            for o, blk in zip(offs, blocks):
                host[o:o + blk.size] = blk
            dev = self.ctx.upload_array(host)
            self.keep.append(dev)
            if len(cache) > 200000:
                cache.clear()
            for (ref, w), o in zip(misses.items(), offs):
                cache[id(w)] = (w, dev, dev.data_ptr() + 4 * o)
                out[ref] = dev.data_ptr() + 4 * o
        return out

    def _const_ptr(self, entry: tuple) -> int:
        """Dummy-add constant in NHWC-padded layout, cached per array."""
        ref, b0, ch, h, w_, cp = entry
        w = self.refs.resolve(ref)
        cache = self.ctx.__dict__.setdefault("const_cache", {})
        hit = cache.get(id(w))
        if hit is not None and hit[0] is w:
            self.keep.append(hit[1])
            return hit[1].data_ptr()
        src_ptr, _ = self.ctx.cached_view(np.ascontiguousarray(w, dtype=np.float32))
        dev = torch.empty(b0 * h * w_ * cp, dtype=torch.float32, device=self.ctx.device)
        self.ctx.check(self.ctx.lib.tobf_nchw_to_nhwc(C.c_void_p(src_ptr), C.c_void_p(dev.data_ptr()), b0, ch, h,
                                                      w_, cp, C.c_void_p(self.ctx.sp)), "const staging")
        self.ctx.launches += 1
        cache[id(w)] = (w, dev)
        self.keep.append(dev)
        return dev.data_ptr()


class PopulationRun:
    """Runs the forward of several graphs on the same stacked input.

    Each graph is a ForwardPlan (built here, or in host worker processes);
    linking resolves the plans' requirement tables — packed weight images
    cached per weight view (every candidate that reuses a vanilla layer, a
    branch slice of it or a shared knob constant shares one image), folded
    BatchNorms, staged constants — lays the activation blocks out in one
    arena reused across runs, rewrites every symbolic pointer with
    vectorised numpy, groups rows into one launch per (level, BN) / level,
    and uploads all descriptors in one H2D.
    """

    conv_events = None  # optional list collecting (start, end) CUDA events per conv launch

    def __init__(self, ctx: DeviceContext, lowered: list[Lowered] | None, reps: int,
                 plans: list[ForwardPlan] | None = None, refs: ArrayRefs | None = None,
                 tables: "PlanTables | None" = None, prec: int = N.PREC_TF32X3):
        """``tables``: the plans' requirement tables already resolved (built
        incrementally while the plans arrive from host workers); resolved
        here otherwise. ``prec``: conv arithmetic of plans built here (given
        plans carry their own, and must agree)."""
        self.ctx = ctx
        self.reps = reps
        if plans is None:
            refs = ArrayRefs()
            plans = [plan_forward(lw, reps, refs, prec) for lw in lowered]
        precs = {p.prec for p in plans}
        if len(precs) != 1:
            raise ValueError(f"one run computes in one precision, got {sorted(precs)}")
        self.prec = precs.pop()
        self.plans, self.refs = plans, refs
        ishape = plans[0].input_shape
        for p in plans:
            if p.input_shape != ishape:
                raise ShapeMismatch(-1, "population graphs disagree on the input shape")
        self.input_shape = ishape
        self.batch = ishape.batch * reps
        if tables is None:
            tables = PlanTables(ctx, refs)
            tables.add(plans)
        elif len(tables.rows) != len(plans):
            raise ValueError(f"{len(tables.rows)} resolved tables for {len(plans)} plans")
        self._keep = tables.keep  # images / BatchNorms / constants this run's descriptors point at
        self._link_all(tables)

    # -------------------------------------------------------------- link
    def _link_all(self, tables: "PlanTables") -> None:
        ta = time.perf_counter()
        ctx, lib, plans = self.ctx, self.ctx.lib, self.plans
        s = self.input_shape
        in_floats = Arena.round(self.batch * s.height * s.width * _rup4(s.channels))
        total = 4 * in_floats + sum(p.arena_bytes for p in plans)
        self.arena = ctx_arena(ctx, total // 4 + 4096)
        self.x_ptr = self.arena.take(in_floats)
        bases = np.zeros(len(plans), np.int64)
        cur = self.x_ptr + 4 * in_floats
        for i, p in enumerate(plans):
            bases[i] = cur
            cur += p.arena_bytes
        self.arena.used = (cur - self.arena.base) // 4
        self.out_ptrs = [int(bases[i]) + p.out_off for i, p in enumerate(plans)]
        t0 = time.perf_counter()
        tabs = {sp: tables.table(i) for i, sp in enumerate((SP_WIMG, SP_AFFINE, SP_CONST, SP_XCOL))}
        # input im2col matrices this run's convs read: built in set_input
        self._xcol = [(g, tables.xcol[g]) for g in sorted({e for p in plans for e in p.xcol})]
        t1 = time.perf_counter()
        # rows of all plans, linked, grouped into launches
        conv = cat_records([p.conv for p in plans], CONV_DTYPE)
        ew = cat_records([p.ew for p in plans], EW_DTYPE)
        conv_plan = np.concatenate([np.full(len(p.conv), i, np.int64) for i, p in enumerate(plans)])
        ew_plan = np.concatenate([np.full(len(p.ew), i, np.int64) for i, p in enumerate(plans)])
        for arr, rp in ((conv, conv_plan), (ew, ew_plan)):
            if not len(arr):
                continue
            for f in ("x", "y") + (("wimg",) if arr.dtype == CONV_DTYPE else ()):
                arr[f] = _link(arr[f], rp, self.x_ptr, bases, tabs)
            arr["epi"]["ptr"] = _link(arr["epi"]["ptr"], rp, self.x_ptr, bases, tabs)
        conv_level = np.concatenate([p.conv_level for p in plans])
        conv_launch_level, ew_level = _aligned_levels(plans)
        conv_bn = np.concatenate([p.conv_bn for p in plans])
        conv_k = np.concatenate([p.conv_k for p in plans])
        if PAIR_STEMS and len(conv):
            keep = _pair_stems(plans, conv, conv_plan, conv_level, conv_launch_level, conv_bn, tables)
            if keep is not None:
                conv, conv_plan, conv_level, conv_launch_level, conv_bn, conv_k = (
                    a[keep] for a in (conv, conv_plan, conv_level, conv_launch_level, conv_bn, conv_k))
        # TMA im2col for the A operand of every conv: one 128-B tensor map per
        # problem, encoded on the host now that the input pointers are final
        conv_tma = np.zeros(len(conv), np.int64)
        if len(conv) and TMA_A:
            host_maps = np.zeros(128 * len(conv), np.uint8)
            ntma = C.c_int()
            # encoded against a 0 base (d.tmap = 128 * i), then placed in the
            # context's content-addressed store
            ctx.check(lib.tobf_conv_tmaps(C.c_void_p(conv.ctypes.data), len(conv), C.c_void_p(host_maps.ctypes.data),
                                          0, C.byref(ntma)), "conv tensor maps")
            conv_tma = (conv["tma"] > 0).astype(np.int64)
            if ntma.value:
                idx = np.nonzero(conv_tma)[0]
                store = ctx.__dict__.get("tmap_store")
                if store is None:
                    store = ctx.tmap_store = TensorMapStore(ctx)
                conv["tmap"][idx] = store.place(host_maps.reshape(-1, 128)[idx])
        # one launch per (level, BN), long K first (TMA-capable when any of its
        # problems is: the A mode is per tile); one ew launch per level
        order = np.lexsort((-conv_k, -conv_bn, conv_level))
        conv = conv[order]
        conv_tma = conv_tma[order]
        ckey = np.stack([conv_level[order], conv_bn[order]], 1) if len(conv) else np.zeros((0, 2), np.int64)
        eorder = np.argsort(ew_level, kind="stable")
        ew = ew[eorder]
        ekey = ew_level[eorder]
        t2 = time.perf_counter()
        launches = []
        ws_need = cnt_need = 0
        tot, wsf, cnts = C.c_int64(), C.c_int64(), C.c_int64()
        conv_ptr = conv.ctypes.data
        for lo, hi in _runs(ckey):
            bn = int(ckey[lo, 1])
            tma_flag = (N.CONV_TMA | (N.CONV_TMA_ALL if TMA_ALL and conv_tma[lo:hi].all() else 0)) if conv_tma[lo:hi].any() else 0
            # split-K for groups too small to fill the SMs; workspace offsets
            # now, one workspace shared by every (stream-ordered) conv launch
            ctx.check(lib.tobf_conv_prepare_split_ex(C.c_void_p(conv_ptr + lo * CONV_DTYPE.itemsize), hi - lo, bn,
                                                     self.prec, ctx.sms, SPLITK_MAX, None, None, C.byref(tot),
                                                     C.byref(wsf), C.byref(cnts)), "conv prepare")
            ws_need, cnt_need = max(ws_need, wsf.value), max(cnt_need, cnts.value)
            launches.append((int(ckey[lo, 0]), 0, "conv", lo, hi - lo, tot.value, bn | tma_flag))
        if len(conv) and not np.array_equal(conv_launch_level, conv_level):
            # tail alignment: the split-K decisions above were taken on the
            # as-soon-as-possible groups and stay with each problem, so every
            # problem's arithmetic (hence every output bit) is that of the
            # unaligned run; only the launch grouping changes
            conv, conv_tma, launches, ws_need, cnt_need = _regroup(conv, conv_tma, conv_launch_level[order], conv_bn[order],
                                                                  conv_k[order])
        if ws_need:
            ws, cnt = splitk_workspace(ctx, ws_need, cnt_need)
            split = conv["ksplit"] > 1
            conv["ws"][split] += np.uint64(ws.data_ptr())
            conv["cnt"][split] += np.uint64(cnt.data_ptr())
        ew_ptr = ew.ctypes.data
        for lo, hi in _runs(ekey.reshape(-1, 1)):
            ctx.check(lib.tobf_ew_prepare(C.c_void_p(ew_ptr + lo * EW_DTYPE.itemsize), hi - lo, C.byref(tot)),
                      "ew prepare")
            launches.append((int(ekey[lo]), 1, "ew", lo, hi - lo, tot.value, 0))
        launches.sort(key=lambda t: (t[0], t[1]))
        t3 = time.perf_counter()
        conv_bytes = conv.tobytes()
        pad = (-len(conv_bytes)) % 256
        host = conv_bytes + bytes(pad) + ew.tobytes()
        self.desc_dev = ctx.upload_bytes(host) if host else None
        self.conv_rows, self.ew_rows = conv, ew  # linked host copies (diagnostics: scripts/race_probe.py)
        base = self.desc_dev.data_ptr() if host else 0
        ew_base = base + len(conv_bytes) + pad
        self.launches = [(k, (base + lo * CONV_DTYPE.itemsize) if k == "conv" else (ew_base + lo * EW_DTYPE.itemsize),
                          n, tot, bn) for (_, _, k, lo, n, tot, bn) in launches]
        self.link_ms = {"arena": 1e3 * (t0 - ta), "tables": 1e3 * (t1 - t0), "rows": 1e3 * (t2 - t1), "prepare": 1e3 * (t3 - t2),
                        "upload": 1e3 * (time.perf_counter() - t3)}

    # -------------------------------------------------------------- run
    def set_input(self, x_nchw: torch.Tensor) -> None:
        """x: (batch, C, H, W) float32 on the device (batch = graph batch * reps)."""
        s = self.input_shape
        if tuple(x_nchw.shape) != (self.batch, s.channels, s.height, s.width):
            raise ShapeMismatch(-1, f"input shape {tuple(x_nchw.shape)} != stacked {(self.batch, *s.as_tuple()[1:])}")
        x = x_nchw.contiguous()
        self._x_keep = x
        self.ctx.check(self.ctx.lib.tobf_nchw_to_nhwc(C.c_void_p(x.data_ptr()), C.c_void_p(self.x_ptr), self.batch,
                                                      s.channels, s.height, s.width, _rup4(s.channels),
                                                      C.c_void_p(self.ctx.sp)), "input staging")
        self.ctx.launches += 1
        for (b, h, w, c, k1, k2, stride, pad, ho, wo, kp), buf in self._xcol:
            self.ctx.check(self.ctx.lib.tobf_im2col(C.c_void_p(self.x_ptr), b, h, w, _rup4(s.channels), c, k1, k2,
                                                    stride, pad, ho, wo, kp, C.c_void_p(buf.data_ptr()),
                                                    C.c_void_p(self.ctx.sp)), "input im2col")
            self.ctx.launches += 1

    def run(self) -> None:
        lib, sp = self.ctx.lib, C.c_void_p(self.ctx.sp)
        evs = self.conv_events
        sched = C.c_void_p(conv_sched(self.ctx).data_ptr())
        for kind, dptr, n, tot, bn in self.launches:
            if kind == "conv":
                if evs is not None:
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                rc = lib.tobf_conv_grouped_ex(C.c_void_p(dptr), n, tot, bn, self.prec, sched, sp)
                if evs is not None:
                    b.record()
                    evs.append((a, b))
            else:
                rc = lib.tobf_ew_grouped(C.c_void_p(dptr), n, tot, sp)
            self.ctx.check(rc, kind)
        self.ctx.launches += len(self.launches)

    def output_ptr(self, gi: int) -> tuple[int, TensorShape]:
        return self.out_ptrs[gi], self.plans[gi].out_shape

    def output_nchw(self, gi: int) -> torch.Tensor:
        ptr, s = self.output_ptr(gi)
        out = torch.empty((self.batch, s.channels, s.height, s.width), dtype=torch.float32, device=self.ctx.device)
        self.ctx.check(self.ctx.lib.tobf_nhwc_to_nchw(C.c_void_p(ptr), C.c_void_p(out.data_ptr()), self.batch,
                                                      s.channels, s.height, s.width, _rup4(s.channels),
                                                      C.c_void_p(self.ctx.sp)), "output staging")
        return out

    def gemm_flops(self) -> int:
        """Algorithmic conv/linear FLOPs of one run (all graphs, all reps): the
        emitted (obfuscated) layers, 2*M*N*K each; a fused sibling group counts
        exactly the sum of its parts."""
        return sum(p.flops_per_image for p in self.plans) * self.reps

    def gemm_bytes(self) -> int:
        """Algorithmic conv/linear HBM bytes of one run: every input and output
        activation once per stacked trial, every weight once (fp32)."""
        return sum(p.gemm_act_bytes_per_image for p in self.plans) * self.reps + \
            sum(p.gemm_weight_bytes for p in self.plans)


# ---------------------------------------------------------------------------
# Drop-in API (interpreter.py:75-118)
# ---------------------------------------------------------------------------

def trial_inputs(shape: TensorShape, trials: int, seed: int) -> np.ndarray:
    """The exact inputs equivalence_check draws: one default_rng(seed) stream,
    ``trials`` standard-normal draws of the input shape, cast to float32
    (interpreter.py:107-111), stacked along the batch dimension."""
    rng = np.random.default_rng(seed)
    xs = [rng.standard_normal(shape.as_tuple()).astype(np.float32) for _ in range(trials)]
    return np.concatenate(xs, axis=0)


def precision_code(precision) -> int:
    """'fp32' (3xTF32, the default) | 'bf16' -> N.PREC_*."""
    if isinstance(precision, (int, np.integer)) and int(precision) in N.PRECISIONS.values():
        return int(precision)
    try:
        return N.PRECISIONS[precision]
    except KeyError:
        raise ValueError(f"precision must be one of {sorted(N.PRECISIONS)}, got {precision!r}") from None


#: equivalence tolerance of each precision when the caller gives none: the
#: reference's tol (interpreter.py:93) in fp32, BASELINE's 2e-2 in bf16 mode
DEFAULT_TOL = {N.PREC_TF32X3: 1e-5, N.PREC_BF16: 2e-2}


def execute(graph: Graph, x: np.ndarray, *, precision="fp32") -> np.ndarray:
    """Run ``graph`` on ``x`` (NCHW float32) on the GPU; returns the output node's
    tensor as a numpy array (interpreter.py:75-90). ``precision='bf16'``:
    convs in the bf16 mode (tolerance 2e-2 against the fp32 reference)."""
    if tuple(x.shape) != graph.input_shape.as_tuple():
        raise ShapeMismatch(-1, f"input shape {x.shape} != {graph.input_shape.as_tuple()}")
    ctx = device()
    run = PopulationRun(ctx, [lower(graph)], reps=1, prec=precision_code(precision))
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(ctx.device)
    run.set_input(xd)
    run.run()
    out = run.output_nchw(0)
    ctx.sync()
    return out.cpu().numpy()


def equivalence_check(g1: Graph, g2: Graph, trials: int = 8, seed: int = 0,
                      tol: float | None = None, *, precision="fp32") -> tuple[bool, float]:
    """Seeded random-input functional comparison (interpreter.py:93-118): both
    graphs run all ``trials`` inputs stacked in one batch; verdict and worst
    relative difference use the reference's float32 formulas bit for bit."""
    if g1.input_shape != g2.input_shape:
        raise ShapeMismatch(-1, "input shapes differ")
    out1 = shape_map(g1)[g1.output_id]
    out2 = shape_map(g2)[g2.output_id]
    if out1 != out2:
        raise ShapeMismatch(-1, f"output shapes differ: {out1} vs {out2}")
    res = evaluate_equivalence(g1, [g2], trials=trials, seed=seed, tol=tol, precision=precision)
    return bool(res[0][0]), float(res[1][0])


def compare_outputs(ctx: DeviceContext, run: PopulationRun, ref_index: int, cand_indices: list[int],
                    tol: float) -> tuple[torch.Tensor, torch.Tensor]:
    """Device verdicts of candidates vs the reference graph output (a = ref,
    b = cand). Pointer tables are staged once per run and reused."""
    if not cand_indices:  # e.g. every plan of the batch was infeasible
        return (torch.zeros(0, dtype=torch.int32, device=ctx.device),
                torch.zeros(0, dtype=torch.float32, device=ctx.device))
    key = (ref_index, tuple(cand_indices))
    cache = run.__dict__.setdefault("_cmp", {})
    if key not in cache:
        ref_ptr, s = run.output_ptr(ref_index)
        a_list = np.array([ref_ptr] * len(cand_indices), dtype=np.uint64)
        b_list = np.array([run.output_ptr(i)[0] for i in cand_indices], dtype=np.uint64)
        ptrs = ctx.upload_bytes(a_list.tobytes() + b_list.tobytes())
        cache[key] = (ptrs, s)
    ptrs, s = cache[key]
    n = len(cand_indices)
    worst = torch.empty(n, dtype=torch.float32, device=ctx.device)
    ok = torch.empty(n, dtype=torch.int32, device=ctx.device)
    if n == 0:
        return ok, worst
    pixels = run.batch * s.height * s.width
    ctx.check(ctx.lib.tobf_equiv_compare(C.c_void_p(ptrs.data_ptr()), C.c_void_p(ptrs.data_ptr() + 8 * n), n,
                                         pixels, s.channels, _rup4(s.channels), C.c_float(tol),
                                         C.c_void_p(worst.data_ptr()), C.c_void_p(ok.data_ptr()),
                                         C.c_void_p(ctx.sp)), "equivalence compare")
    ctx.launches += 2
    return ok, worst


def evaluate_equivalence(reference: Graph, candidates: list[Graph], trials: int = 8, seed: int = 0,
                         tol: float | None = None, *, precision="fp32"):
    """Batched equivalence_check(reference, c) for every candidate c: one
    forward of the reference and of all candidates on the stacked trials.
    Returns (ok[np.bool_], worst[np.float64]) per candidate. ``tol`` defaults
    to the precision's (DEFAULT_TOL)."""
    ctx = device()
    prec = precision_code(precision)
    tol = DEFAULT_TOL[prec] if tol is None else tol
    run = PopulationRun(ctx, [lower(reference)] + [lower(g) for g in candidates], reps=trials, prec=prec)
    x = trial_inputs(reference.input_shape, trials, seed)
    run.set_input(torch.from_numpy(x).to(ctx.device))
    run.run()
    ok, worst = compare_outputs(ctx, run, 0, list(range(1, len(candidates) + 1)), tol)
    ctx.sync()
    return ok.cpu().numpy().astype(bool), worst.cpu().numpy().astype(np.float64)

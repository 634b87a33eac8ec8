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
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .engine import Arena, DeviceContext, _root, device
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
# Population run: allocate, pack, describe, launch
# ---------------------------------------------------------------------------

CONV_DTYPE = np.dtype(N.ConvDesc)
EW_DTYPE = np.dtype(N.EwDesc)
_NO_EPI = (0, 0, 0)


class PopulationRun:
    """Runs the forward of several lowered graphs on the same stacked input.

    Host preparation is table-driven: descriptor rows are numpy records
    (one H2D for all levels), packed weight images are cached per weight
    view (every candidate that reuses a vanilla layer — or a branch slice of
    it, or a shared knob constant — shares one image), activations live in
    one arena reused across runs on the engine stream.
    """

    conv_events = None  # optional list collecting (start, end) CUDA events per conv launch

    def __init__(self, ctx: DeviceContext, lowered: list[Lowered], reps: int):
        self.ctx = ctx
        self.lowered = lowered
        self.reps = reps
        self._keep: list = []
        g0 = lowered[0].graph
        for lw in lowered:
            if lw.graph.input_shape != g0.input_shape:
                raise ShapeMismatch(-1, "population graphs disagree on the input shape")
        ishape = g0.input_shape
        self.batch = ishape.batch * reps
        act = Arena.round(self.batch * ishape.height * ishape.width * _rup4(ishape.channels))
        for lw in lowered:
            for v in lw.values:
                sh = lw.shapes[v]
                act += Arena.round(self.batch * sh.height * sh.width * _rup4(sh.channels))
        self.arena = ctx_arena(ctx, act + 4096)
        self.x_ptr = self.arena.take(self.batch * ishape.height * ishape.width * _rup4(ishape.channels))
        self.bufs: list[dict[int, int]] = []
        for lw in lowered:
            b = {-1: self.x_ptr}
            for v in sorted(lw.values):
                sh = lw.shapes[v]
                b[v] = self.arena.take(self.batch * sh.height * sh.width * _rup4(sh.channels))
            self.bufs.append(b)
        self._stage_affines()
        self._prepare()

    # -------------------------------------------------------------- helpers
    @staticmethod
    def _in_shape(lw: Lowered, op: Op) -> TensorShape:
        return lw.shapes[op.src] if op.src >= 0 else lw.graph.input_shape

    def _gemm_geom(self, lw: Lowered, op: Op):
        n = lw.graph.nodes[op.node]
        s_in = self._in_shape(lw, op)
        j = op.j or n.attrs["j"]
        if n.kind is K.Conv2D:
            return n.attrs["k1"], n.attrs["k2"], _rup4(s_in.channels), j
        return s_in.height, s_in.width, _rup4(s_in.channels), j

    def _stage_affines(self) -> None:
        """Fold every BatchNorm the population's epilogues use into (a, b) with
        a = scale/sqrt(var+eps), b = shift - mean*a (fp64 -> fp32), caching the
        device copy by weight-array identity; all misses go up in ONE H2D."""
        cache = self.ctx.__dict__.setdefault("affine_cache", {})
        misses: dict[int, np.ndarray] = {}
        for lw in self.lowered:
            for op in lw.ops:
                for st in op.steps:
                    if st.op == "affine":
                        w = lw.graph.nodes[st.ref].weights
                        hit = cache.get(id(w))
                        if (hit is None or hit[0] is not w) and id(w) not in misses:
                            misses[id(w)] = w
        if not misses:
            return
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
        if len(cache) > 200000:
            cache.clear()
        for (key, w), o in zip(misses.items(), offs):
            cache[key] = (w, dev, dev.data_ptr() + 4 * o)

    def _affine(self, lw: Lowered, nid: int) -> int:
        return self.ctx.affine_cache[id(lw.graph.nodes[nid].weights)][2]

    def _const(self, lw: Lowered, nid: int) -> int:
        """Dummy-add constant in NHWC-padded layout, cached per array."""
        node = lw.graph.nodes[nid]
        cache = self.ctx.__dict__.setdefault("const_cache", {})
        hit = cache.get(id(node.weights))
        if hit is not None and hit[0] is node.weights:
            return hit[1].data_ptr()
        sh = lw.shapes[nid]
        b0 = lw.graph.input_shape.batch
        cp = _rup4(sh.channels)
        src_ptr, _ = self.ctx.cached_view(np.ascontiguousarray(node.weights, dtype=np.float32))
        dev = torch.empty(b0 * sh.height * sh.width * cp, dtype=torch.float32, device=self.ctx.device)
        self.ctx.check(self.ctx.lib.tobf_nchw_to_nhwc(C.c_void_p(src_ptr), C.c_void_p(dev.data_ptr()), b0,
                                                      sh.channels, sh.height, sh.width, cp, C.c_void_p(self.ctx.sp)),
                       "const staging")
        self.ctx.launches += 1
        cache[id(node.weights)] = (node.weights, dev)
        return dev.data_ptr()

    def _wimg(self, n, s_in: TensorShape, k1: int, k2: int, cp: int, j: int, bn: int, w=None) -> int:
        """Packed tf32 hi/lo operand image of a conv/linear weight view, cached
        by (device view, geometry): one pack per distinct view per cache life."""
        ctx, lib = self.ctx, self.ctx.lib
        wptr, st = ctx.cached_view(n.weights if w is None else w)
        if n.kind is K.Conv2D:
            su, sv, sc, sn = st
        else:
            r, cstride = st
            su, sv, sc, sn = s_in.width * r, r, s_in.height * s_in.width * r, cstride
        key = (wptr, su, sv, sc, sn, k1, k2, s_in.channels, cp, j, bn)
        cache = ctx.__dict__.setdefault("wimg_cache", {})
        hit = cache.get(key)
        if hit is not None:
            return hit.data_ptr()
        nbytes = lib.tobf_wimg_bytes(k1, k2, cp, j, bn)
        img = torch.empty(nbytes // 4, dtype=torch.float32, device=ctx.device)
        ctx.check(lib.tobf_pack_weights(C.c_void_p(wptr), k1, k2, s_in.channels, cp, j, su, sv, sc, sn, bn,
                                        C.c_void_p(img.data_ptr()), C.c_void_p(ctx.sp)), "pack weights")
        ctx.launches += 1
        cache[key] = img
        return img.data_ptr()

    def _epi_rows(self, lw: Lowered, bufs: dict, steps: list) -> list:
        out = []
        for st in steps:
            if st.op == "affine":
                out.append((N.EPI_AFFINE, _rup4(lw.shapes[st.ref].channels), self._affine(lw, st.ref)))
            elif st.op == "relu":
                out.append((N.EPI_RELU, 0, 0))
            elif st.op == "add":
                sh = lw.shapes[st.ref] if st.ref >= 0 else lw.graph.input_shape
                out.append((N.EPI_ADD_TENSOR, _rup4(sh.channels), bufs[st.ref]))
            elif st.op == "const":
                out.append((N.EPI_ADD_CONST, lw.graph.input_shape.batch, self._const(lw, st.ref)))
        return out

    # -------------------------------------------------------------- prepare
    def _prepare(self) -> None:
        ctx, lib = self.ctx, self.ctx.lib
        levels: dict[int, dict[str, list]] = {}
        for gi, lw in enumerate(self.lowered):
            bufs = self.bufs[gi]
            nodes = lw.graph.nodes
            for op in lw.ops:
                lvl = levels.get(op.level)
                if lvl is None:
                    lvl = levels[op.level] = {"g64": [], "g128": [], "ew": []}
                s_in = self._in_shape(lw, op)
                s_out = lw.shapes[op.out]
                if op.kind == "gemm":
                    n = nodes[op.node]
                    k1, k2, cp, j = self._gemm_geom(lw, op)
                    bn = 128 if j > 64 else 64
                    if n.kind is K.Conv2D:
                        stride, pad = n.attrs["stride"], n.attrs["padding"]
                    else:
                        stride, pad = 1, 0
                    epi = self._epi_rows(lw, bufs, op.steps)
                    row = (bufs[op.src], self._wimg(n, s_in, k1, k2, cp, j, bn, op.w), bufs[op.out],
                           self.batch, s_in.height, s_in.width, cp, s_out.height, s_out.width, _rup4(j), j,
                           k1, k2, stride, pad, 0, 0, 0, 0, 0, len(epi), cp, _rup4(j),
                           epi + [_NO_EPI] * (N.TOBF_MAX_EPI - len(epi)))
                    lvl["g128" if bn == 128 else "g64"].append((k1 * k2 * cp, row))
                    continue
                ldx, ldy = _rup4(s_in.channels), _rup4(s_out.channels)
                epi = []
                if op.kind == "pool":
                    n = nodes[op.node]
                    head = (N.OP_MAXPOOL, self.batch, s_in.height, s_in.width, s_in.channels, ldx, s_out.height,
                            s_out.width, ldy, n.attrs["window"], n.attrs["stride"])
                    cpo = _rup4(s_in.channels)
                elif op.kind == "epi":
                    epi = self._epi_rows(lw, bufs, op.steps)
                    head = (N.OP_EPI, self.batch, s_in.height, s_in.width, s_out.channels, ldx, s_out.height,
                            s_out.width, ldy, 0, 0)
                    cpo = _rup4(s_out.channels)
                elif op.kind == "copy":
                    total = s_out.channels
                    head = (N.OP_COPYCH, self.batch, s_in.height, s_in.width, op.cc, ldx, 0, 0, ldy, op.a0, op.a1)
                    cpo = _rup4(total) if op.a0 + op.cc == total else op.a0 + op.cc
                else:  # softmax
                    head = (N.OP_SOFTMAX, self.batch, s_in.height, s_in.width, s_in.channels, ldx, 0, 0, ldy, 0, 0)
                    cpo = _rup4(s_in.channels)
                lvl["ew"].append((bufs[op.src], bufs[op.out]) + head +
                                 (len(epi), 0, cpo, 0, epi + [_NO_EPI] * (N.TOBF_MAX_EPI - len(epi))))
        # one structured array per op class for the whole population (numpy's
        # nested-sequence parsing is the dominant host cost per call), then
        # one contiguous slice per launch
        conv_rows, conv_keys, ew_rows, ew_keys = [], [], [], []
        for lv in sorted(levels):
            grp = levels[lv]
            for key, bn in (("g128", 128), ("g64", 64)):
                if grp[key]:
                    rows = [r for _, r in sorted(grp[key], key=lambda t: -t[0])]  # long K first
                    conv_keys.append((lv, bn, len(conv_rows), len(rows)))
                    conv_rows += rows
            if grp["ew"]:
                ew_keys.append((lv, len(ew_rows), len(grp["ew"])))
                ew_rows += grp["ew"]
        conv_arr = np.array(conv_rows, dtype=CONV_DTYPE) if conv_rows else np.zeros(0, CONV_DTYPE)
        ew_arr = np.array(ew_rows, dtype=EW_DTYPE) if ew_rows else np.zeros(0, EW_DTYPE)
        launches = []
        for lv, bn, lo, n in conv_keys:
            tot = C.c_int64()
            ctx.check(lib.tobf_conv_prepare(C.c_void_p(conv_arr[lo:].ctypes.data), n, bn, C.byref(tot)),
                      "conv prepare")
            launches.append((lv, 0, "conv", lo, n, tot.value, bn))
        for lv, lo, n in ew_keys:
            tot = C.c_int64()
            ctx.check(lib.tobf_ew_prepare(C.c_void_p(ew_arr[lo:].ctypes.data), n, C.byref(tot)), "ew prepare")
            launches.append((lv, 1, "ew", lo, n, tot.value, 0))
        launches.sort(key=lambda t: (t[0], t[1]))
        conv_bytes = conv_arr.tobytes()
        pad = (-len(conv_bytes)) % 256
        host = conv_bytes + bytes(pad) + ew_arr.tobytes()
        self.desc_dev = ctx.upload_bytes(host) if host else None
        base = self.desc_dev.data_ptr() if host else 0
        ew_base = base + len(conv_bytes) + pad
        self.launches = [(k, (base + lo * CONV_DTYPE.itemsize) if k == "conv" else (ew_base + lo * EW_DTYPE.itemsize),
                          n, tot, bn) for (_, _, k, lo, n, tot, bn) in launches]

    # -------------------------------------------------------------- run
    def set_input(self, x_nchw: torch.Tensor) -> None:
        """x: (batch, C, H, W) float32 on the device (batch = graph batch * reps)."""
        s = self.lowered[0].graph.input_shape
        if tuple(x_nchw.shape) != (self.batch, s.channels, s.height, s.width):
            raise ShapeMismatch(-1, f"input shape {tuple(x_nchw.shape)} != stacked {(self.batch, *s.as_tuple()[1:])}")
        x = x_nchw.contiguous()
        self._x_keep = x
        self.ctx.check(self.ctx.lib.tobf_nchw_to_nhwc(C.c_void_p(x.data_ptr()), C.c_void_p(self.x_ptr), self.batch,
                                                      s.channels, s.height, s.width, _rup4(s.channels),
                                                      C.c_void_p(self.ctx.sp)), "input staging")
        self.ctx.launches += 1

    def run(self) -> None:
        lib, sp = self.ctx.lib, C.c_void_p(self.ctx.sp)
        evs = self.conv_events
        for kind, dptr, n, tot, bn in self.launches:
            if kind == "conv":
                if evs is not None:
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                rc = lib.tobf_conv_grouped(C.c_void_p(dptr), n, tot, bn, sp)
                if evs is not None:
                    b.record()
                    evs.append((a, b))
            else:
                rc = lib.tobf_ew_grouped(C.c_void_p(dptr), n, tot, sp)
            self.ctx.check(rc, kind)
        self.ctx.launches += len(self.launches)

    def output_ptr(self, gi: int) -> tuple[int, TensorShape]:
        lw = self.lowered[gi]
        return self.bufs[gi][lw.out_node], lw.shapes[lw.out_node]

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
        total = 0
        for lw in self.lowered:
            for op in lw.ops:
                if op.kind == "gemm":
                    n = lw.graph.nodes[op.node]
                    s = lw.shapes[op.node]
                    s_in = self._in_shape(lw, op)
                    j = op.j or n.attrs["j"]
                    if n.kind is K.Conv2D:
                        kk = n.attrs["k1"] * n.attrs["k2"] * s_in.channels
                        total += 2 * self.batch * s.height * s.width * j * kk
                    else:
                        total += 2 * self.batch * j * s_in.channels * s_in.height * s_in.width
        return total


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


def execute(graph: Graph, x: np.ndarray) -> np.ndarray:
    """Run ``graph`` on ``x`` (NCHW float32) on the GPU; returns the output node's
    tensor as a numpy array (interpreter.py:75-90)."""
    if tuple(x.shape) != graph.input_shape.as_tuple():
        raise ShapeMismatch(-1, f"input shape {x.shape} != {graph.input_shape.as_tuple()}")
    ctx = device()
    run = PopulationRun(ctx, [lower(graph)], reps=1)
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(ctx.device)
    run.set_input(xd)
    run.run()
    out = run.output_nchw(0)
    ctx.sync()
    return out.cpu().numpy()


def equivalence_check(g1: Graph, g2: Graph, trials: int = 8, seed: int = 0,
                      tol: float = 1e-5) -> tuple[bool, float]:
    """Seeded random-input functional comparison (interpreter.py:93-118): both
    graphs run all ``trials`` inputs stacked in one batch; verdict and worst
    relative difference use the reference's float32 formulas bit for bit."""
    if g1.input_shape != g2.input_shape:
        raise ShapeMismatch(-1, "input shapes differ")
    out1 = shape_map(g1)[g1.output_id]
    out2 = shape_map(g2)[g2.output_id]
    if out1 != out2:
        raise ShapeMismatch(-1, f"output shapes differ: {out1} vs {out2}")
    res = evaluate_equivalence(g1, [g2], trials=trials, seed=seed, tol=tol)
    return bool(res[0][0]), float(res[1][0])


def compare_outputs(ctx: DeviceContext, run: PopulationRun, ref_index: int, cand_indices: list[int],
                    tol: float) -> tuple[torch.Tensor, torch.Tensor]:
    """Device verdicts of candidates vs the reference graph output (a = ref,
    b = cand). Pointer tables are staged once per run and reused."""
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
                         tol: float = 1e-5):
    """Batched equivalence_check(reference, c) for every candidate c: one
    forward of the reference and of all candidates on the stacked trials.
    Returns (ok[np.bool_], worst[np.float64]) per candidate."""
    ctx = device()
    run = PopulationRun(ctx, [lower(reference)] + [lower(g) for g in candidates], reps=trials)
    x = trial_inputs(reference.input_shape, trials, seed)
    run.set_input(torch.from_numpy(x).to(ctx.device))
    run.run()
    ok, worst = compare_outputs(ctx, run, 0, list(range(1, len(candidates) + 1)), tol)
    ctx.sync()
    return ok.cpu().numpy().astype(bool), worst.cpu().numpy().astype(np.float64)

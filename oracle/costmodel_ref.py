"""Restated analytical cost model (oracle) — follows fusion.py:45-180 and
costmodel.py:108-293 with Python floats, so every feature is bit-exact by
construction. Operates on duck-typed graphs (``nodes``, ``output_id``,
``input_shape``) with integer shape tuples computed here.
"""

from __future__ import annotations

import math

from .interp_ref import _order

COMPLEX = {"Conv2D", "Linear", "MaxPool", "SoftMax"}   # graph.py:33-35
INJECTIVE = {"ReLU", "BatchNorm", "Add"}               # graph.py:38
FACTORS = (1, 2, 4, 8, 16, 32)                         # fusion.py:22
PROFILES = {  # costmodel.py:44-50: (macs/cycle, launch, l1, l2, sms)
    "default": (1024, 2000, 64 * 1024, 1024 * 1024, 4),
    "lean": (256, 500, 32 * 1024, 512 * 1024, 4),
}
FEATURES = ("cycles", "dram_read", "dram_write", "l1_tx", "l1_util", "l1_hit", "l2_tx", "l2_util", "l2_hit")


def shapes_of(graph) -> dict[int, tuple[int, int, int, int]]:
    """graph.py:174-254 shape rules, as NCHW tuples."""
    sh: dict[int, tuple] = {}
    ib = tuple(graph.input_shape.as_tuple())
    for nid in _order(graph):
        n = graph.nodes[nid]
        ins = [sh[p] for p in n.inputs] if n.inputs else [ib]
        k, a = n.kind.value, n.attrs
        b, c, h, w = ins[0]
        if k == "Conv2D":
            out = (b, a["j"], (h + 2 * a["padding"] - a["k1"]) // a["stride"] + 1,
                   (w + 2 * a["padding"] - a["k2"]) // a["stride"] + 1)
        elif k == "Linear":
            out = (b, a["j"], 1, 1)
        elif k == "MaxPool":
            out = (b, c, (h - a["window"]) // a["stride"] + 1, (w - a["window"]) // a["stride"] + 1)
        elif k == "Concat":
            out = (b, sum(s[1] for s in ins), h, w)
        elif k == "Slice":
            out = (b, a["stop"] - a["start"], h, w)
        else:
            out = ins[0]
        sh[nid] = out
    return sh


def fuse(graph, limits=None) -> list[tuple[int, ...]]:
    """fusion.py:45-80 (consumed is only checked for chain starts)."""
    limits = limits or {}
    cons: dict[int, list[int]] = {nid: [] for nid in graph.nodes}
    for n in graph.nodes.values():
        for p in set(n.inputs):
            if p in cons:
                cons[p].append(n.id)
    out, taken = [], set()
    for nid in _order(graph):
        if nid in taken:
            continue
        if graph.nodes[nid].kind.value not in COMPLEX:
            out.append((nid,))
            continue
        lim = limits.get(nid, 2)
        lim = 2 if lim < 0 else min(lim, 2)
        chain = [nid]
        while len(chain) - 1 < lim:
            nx = cons[chain[-1]]
            if len(nx) != 1 or graph.nodes[nx[0]].kind.value not in INJECTIVE:
                break
            chain.append(nx[0])
            taken.add(nx[0])
        out.append(tuple(chain))
    return out


def triples(extent: int) -> list[tuple[int, int, int]]:
    """fusion.py:137-156."""
    cap = 1 << max(0, (extent - 1).bit_length())
    return [(p, q, r) for p in FACTORS for q in FACTORS for r in FACTORS if p * q * r <= cap]


def _numel(s):
    return s[0] * s[1] * s[2] * s[3]


def _work(graph, sh, nid) -> int:
    n, s = graph.nodes[nid], sh[nid]
    k, a = n.kind.value, n.attrs
    if k == "Conv2D":
        return s[0] * a["k1"] * a["k2"] * a["c"] * a["j"] * s[2] * s[3]
    if k == "Linear":
        return s[0] * a["c"] * a["j"]
    if k == "MaxPool":
        return _numel(s) * a["window"] ** 2
    if k == "SoftMax":
        return 4 * _numel(s)
    if k == "BatchNorm":
        return 2 * _numel(s)
    return _numel(s)


def _footprint(kind, a, c, ey, ex) -> int:
    if kind == "Conv2D":
        s, k1, k2 = a["stride"], a["k1"], a["k2"]
        return 4 * (ey * ex + (ey * s + k1 - s) * (ex * s + k2 - s) * c + k1 * k2 * c)
    s, w = a["stride"], a["window"]
    return 4 * (ey * ex + (ey * s + w - s) * (ex * s + w - s) * c)


def profile_kernel(graph, sh, kern, ty, tx, unroll, prof):
    """costmodel.py:166-232 -> dict of the 9 features (Python floats)."""
    P, L, l1, l2, sms = prof
    anc = graph.nodes[kern[0]]
    s = sh[kern[0]]
    work = _work(graph, sh, kern[0])
    fw = sum(_work(graph, sh, q) for q in kern[1:])
    fb = 0
    for q in kern[1:]:
        nq = graph.nodes[q]
        if nq.weights is not None:
            fb += nq.weights.size * 4
        if nq.kind.value == "Add" and len(nq.inputs) > 1:
            fb += sum(_numel(sh[p]) * 4 for p in nq.inputs[1:])
    inb = sum(_numel(sh[p]) * 4 for p in anc.inputs) if anc.inputs else _numel(tuple(graph.input_shape.as_tuple())) * 4
    wb = anc.weights.size * 4 if anc.weights is not None else 0
    ob = _numel(sh[kern[-1]]) * 4
    ws = inb + wb + ob + fb
    kind = anc.kind.value
    if kind in ("Conv2D", "MaxPool"):
        iy, ix = ty[1] * ty[2], tx[1] * tx[2]
        fy, fx = ty[0] * iy, tx[0] * ix
        c = anc.attrs.get("c", s[1])
        fpi = _footprint(kind, anc.attrs, c, iy, ix)
        fpf = _footprint(kind, anc.attrs, c, fy, fx)
        blocks = (-(-s[2] // fy)) * (-(-s[3] // fx))
        occ = min(1.0, blocks / sms)
        eff = (min(fpf, l1) / l1) * occ
        eff = min(1.0, eff * (0.92 + 0.02 * unroll))
        eff = max(eff, 1.0 / 256.0)
        rw = (-(-s[2] // iy)) * (-(-s[3] // ix))
        rx = -(-anc.attrs.get("j", s[1]) // iy)
    else:
        fpi = fpf = min(8192, ws)
        eff = 1.0
        rw = 1
        rx = anc.attrs["j"] if kind == "Linear" else 1
    read = wb * rw + inb * rx + fb
    write = ob

    def hit(fp):
        return min(max(100.0 * (1.0 - fp / ws), 5.0), 99.0)

    return {"cycles": work / (P * eff) + fw / P + L, "dram_read": float(read), "dram_write": float(write),
            "l1_tx": read / 32, "l1_util": 100.0 * eff, "l1_hit": hit(fpi), "l2_tx": (read + write) / 32,
            "l2_util": 100.0 * min(fpf, l2) / l2, "l2_hit": hit(fpf)}


def default_schedule(graph, sh, kern, prof):
    """fusion.py:159-180: lexicographic (cycles, ty, tx) argmin."""
    if graph.nodes[kern[0]].kind.value not in COMPLEX:
        return (1, 1, 1), (1, 1, 1)
    s = sh[kern[0]]
    best = None
    for ty in triples(s[2]):
        for tx in triples(s[3]):
            key = (profile_kernel(graph, sh, kern, ty, tx, 4, prof)["cycles"], ty, tx)
            if best is None or key < best:
                best = key
    return best[1], best[2]


def _balanced(n):
    a = 1
    for d in range(1, math.isqrt(n) + 1):
        if n % d == 0:
            a = d
    return a, n // a


def modify(t, k):
    """fusion.py:105-134 for one triple."""
    if k == 0:
        return t
    a, b = _balanced(t[0] * t[1] * t[2])
    out = [1, 1, 1]
    rest = [i for i in range(3) if i != k - 1]
    out[rest[0]], out[rest[1]] = a, b
    return tuple(out)


class ScheduleMemo:
    """costmodel.py:248-256 _SCHEDULE_CACHE with first-seen semantics."""

    def __init__(self):
        self.table = {}

    def key(self, graph, sh, kern, prof_name):
        anc = graph.nodes[kern[0]]
        ins = sh[anc.inputs[0]] if anc.inputs else tuple(graph.input_shape.as_tuple())
        return (prof_name, anc.kind.value, tuple(sorted(anc.attrs.items())), ins, sh[kern[0]])


def profile_pipeline(graph, prof_name="default", limits=None, strategies=None, memo: ScheduleMemo | None = None):
    """costmodel.py:266-293 -> (kernels, schedules, feature rows, T)."""
    prof = PROFILES[prof_name]
    memo = memo if memo is not None else ScheduleMemo()
    strategies = strategies or {}
    sh = shapes_of(graph)
    kernels = fuse(graph, limits)
    scheds, rows = [], []
    for kern in kernels:
        k = memo.key(graph, sh, kern, prof_name)
        if k not in memo.table:
            memo.table[k] = default_schedule(graph, sh, kern, prof)
        ty, tx = memo.table[k]
        st = strategies.get(kern[0], 0)
        ty, tx = modify(ty, st), modify(tx, st)
        scheds.append((ty, tx))
        rows.append(profile_kernel(graph, sh, kern, ty, tx, 4, prof))
    T = sum(r["cycles"] for r in rows)   # CPython 3.12 sum(): Neumaier-compensated
    return kernels, scheds, rows, T

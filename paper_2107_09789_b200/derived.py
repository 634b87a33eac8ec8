"""Derived (lazily materialised) knob weights: SURVEY §8(f)1, device-side
knob weight synthesis.

Every weight the six knobs produce from a vanilla Conv2D / Linear weight is a
per-axis gather of it, scaled by powers of two, with zero rings:

  widen, producer   duplicate the first `extra` output channels at the end
                    (transforms.py:134-137 / knobs._widen)
  widen, consumer   scale the first `extra` input channels by 0.5 and append
                    0.5-scaled duplicates (transforms.py:148-165)
  kernel widen      zero rings on both spatial axes (transforms.py:319-335)
  branch            slices along j (out-branch) or c (in-branch)
                    (transforms.py:173-231)

(deepen / skip / dummy weights are shared identity / zero constants already).
A ``DerivedWeight`` records that gather instead of materialising it:

  out[u, v, c, n] = base4[mu[u], mv[v], mc[c], mn[n]] * sc[c] * sn[n]
                    (any map entry -1 -> 0)

with base4 the vanilla array viewed (k1, k2, c, j); a Linear (c*H*W, j)
weight in NCHW-flatten row order is viewed (H, W, c, j). Each axis map is a
short tuple of segments (src_start | -1, length, scale), so a derived weight
is a few hundred bytes: host workers ship it instead of ~1 GB of widened
VGG-16 weights per candidate, and the device packs the weight image straight
from the resident vanilla array (``tobf_pack_weights_gather``).

``materialize()`` (and ``np.asarray``) produce exactly the array the
reference's numpy code does (copies, x0.5 in float32, zeros), which the
tests pin against ``knobs.apply_plan``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

Seg = tuple  # (src_start or -1, length, scale)


def _segs_len(segs) -> int:
    return sum(s[1] for s in segs)


def _norm(segs) -> tuple:
    out = []
    for src, n, sc in segs:
        if n <= 0:
            continue
        if src < 0:
            src, sc = -1, 0.0
        if out:
            ps, pn, psc = out[-1]
            if psc == sc and ((ps < 0 and src < 0) or (ps >= 0 and src == ps + pn)):
                out[-1] = (ps, pn + n, psc)
                continue
        out.append((src, n, float(sc)))
    return tuple(out)


def seg_identity(n: int) -> tuple:
    return ((0, n, 1.0),)


def seg_slice(segs, a: int, b: int) -> tuple:
    out, pos = [], 0
    for src, n, sc in segs:
        lo, hi = max(a, pos), min(b, pos + n)
        if lo < hi:
            out.append((src + (lo - pos) if src >= 0 else -1, hi - lo, sc))
        pos += n
    return _norm(out)


def seg_scale(segs, s: float) -> tuple:
    return _norm([(src, n, sc * s if src >= 0 else 0.0) for src, n, sc in segs])


def seg_concat(*parts) -> tuple:
    return _norm([s for p in parts for s in p])


def seg_expand(segs) -> tuple[np.ndarray, np.ndarray]:
    idx = np.concatenate([np.arange(src, src + n, dtype=np.int32) if src >= 0 else np.full(n, -1, np.int32)
                          for src, n, _ in segs]) if segs else np.zeros(0, np.int32)
    scl = np.concatenate([np.full(n, sc, np.float32) for _, n, sc in segs]) if segs else np.zeros(0, np.float32)
    return idx, scl


@dataclass(frozen=True, eq=False)
class DerivedWeight:
    base: np.ndarray          # the vanilla root array: (k1, k2, c, j) conv or (c*H*W, j) linear
    kind: str                 # "conv" | "linear"
    hw: tuple                 # linear: (H, W) of the feeding activation; conv: (1, 1)
    segs: tuple               # 4 axis segment tuples: u, v, c, n

    # ------------------------------------------------------------ construction
    @staticmethod
    def of(base: np.ndarray, kind: str, hw: tuple = (1, 1)) -> "DerivedWeight":
        if kind == "conv":
            k1, k2, c, j = base.shape
            return DerivedWeight(base, kind, (1, 1), (seg_identity(k1), seg_identity(k2), seg_identity(c),
                                                      seg_identity(j)))
        H, W = hw
        rows, j = base.shape
        if rows % (H * W):
            raise ValueError(f"linear rows {rows} not a multiple of H*W={H * W}")
        return DerivedWeight(base, kind, (H, W), (seg_identity(H), seg_identity(W), seg_identity(rows // (H * W)),
                                                  seg_identity(j)))

    def _with(self, axis: int, segs) -> "DerivedWeight":
        s = list(self.segs)
        s[axis] = segs
        return DerivedWeight(self.base, self.kind, self.hw, tuple(s))

    # ------------------------------------------------------------ the knob ops
    def dup_tail(self, axis: int, extra: int, scale: float = 1.0) -> "DerivedWeight":
        """axis 2 (c) / 3 (n): the first ``extra`` entries scaled and appended."""
        segs = self.segs[axis]
        head = seg_scale(seg_slice(segs, 0, extra), scale)
        return self._with(axis, seg_concat(head, seg_slice(segs, extra, _segs_len(segs)), head))

    def pad_kernel(self, steps: int) -> "DerivedWeight":
        z = ((-1, steps, 0.0),)
        d = self._with(0, seg_concat(z, self.segs[0], z))
        return d._with(1, seg_concat(z, d.segs[1], z))

    def slice(self, axis: int, a: int, b: int) -> "DerivedWeight":
        return self._with(axis, seg_slice(self.segs[axis], a, b))

    # ------------------------------------------------------------ array protocol
    @property
    def channels(self) -> int:
        return _segs_len(self.segs[2])

    @property
    def shape(self) -> tuple:
        lu, lv, lc, ln = (_segs_len(s) for s in self.segs)
        if self.kind == "conv":
            return (lu, lv, lc, ln)
        return (lc * self.hw[0] * self.hw[1], ln)

    @property
    def ndim(self) -> int:
        return len(self.shape)

    @property
    def size(self) -> int:
        return int(np.prod(self.shape))

    @property
    def dtype(self):
        return np.dtype(np.float32)

    @property
    def nbytes(self) -> int:
        return 4 * self.size

    def is_identity(self) -> bool:
        full = tuple(seg_identity(n) for n in self._base4_shape())
        return self.segs == full

    def _base4_shape(self) -> tuple:
        if self.kind == "conv":
            return self.base.shape
        H, W = self.hw
        return (H, W, self.base.shape[0] // (H * W), self.base.shape[1])

    def key(self) -> tuple:
        """Hashable description of the gather (without the base)."""
        return (self.kind, self.hw, self.segs)

    def maps(self) -> tuple:
        """(mu, mv, mc, mn) int32 and (sc, sn) float32 expanded maps."""
        (mu, su), (mv, sv), (mc, sc), (mn, sn) = (seg_expand(s) for s in self.segs)
        if np.any(su[mu >= 0] != 1.0) or np.any(sv[mv >= 0] != 1.0):
            raise ValueError("spatial axes carry no scale")
        return mu, mv, mc, mn, sc, sn

    def materialize(self) -> np.ndarray:
        mu, mv, mc, mn, sc, sn = self.maps()
        if self.kind == "conv":
            b4 = self.base
        else:
            H, W = self.hw
            b4 = self.base.reshape(-1, H, W, self.base.shape[1]).transpose(1, 2, 0, 3)  # (H, W, c, j) view
        out = b4[np.ix_(np.maximum(mu, 0), np.maximum(mv, 0), np.maximum(mc, 0), np.maximum(mn, 0))]
        out = np.ascontiguousarray(out, dtype=np.float32)
        zero = (mu < 0)[:, None, None, None] | (mv < 0)[None, :, None, None] | \
            (mc < 0)[None, None, :, None] | (mn < 0)[None, None, None, :]
        if zero.any():
            out[np.broadcast_to(zero, out.shape)] = 0.0
        if np.any(sc != 1.0):
            cols = np.nonzero(sc != 1.0)[0]
            out[:, :, cols, :] *= sc[cols][None, None, :, None]
        if np.any(sn != 1.0):
            cols = np.nonzero(sn != 1.0)[0]
            out[:, :, :, cols] *= sn[cols][None, None, None, :]
        if self.kind == "conv":
            return out
        H, W = self.hw
        return np.ascontiguousarray(out.transpose(2, 0, 1, 3)).reshape(-1, out.shape[3])

    def __array__(self, dtype=None, copy=None):
        a = self.materialize()
        return a if dtype is None else a.astype(dtype)


def materialize(w):
    return w.materialize() if isinstance(w, DerivedWeight) else w


def consecutive_derived(ws: list, axis: int):
    """Sibling parts that are consecutive slices (along ``axis``: -1/3 = j,
    2 = c; Linear c axis) of one derived weight -> the merged derived weight, else None."""
    if not all(isinstance(w, DerivedWeight) for w in ws):
        return None
    w0 = ws[0]
    ax = 3 if axis in (-1, 3) or (w0.kind == "linear" and axis == 1) else 2
    if w0.kind == "linear" and axis == 0:
        ax = 2
    for w in ws:
        if w.base is not w0.base or w.kind != w0.kind or w.hw != w0.hw or \
                any(w.segs[i] != w0.segs[i] for i in range(4) if i != ax):
            return None
    merged = seg_concat(*[w.segs[ax] for w in ws])
    return w0._with(ax, merged)


__all__ = ["DerivedWeight", "materialize", "consecutive_derived", "seg_identity", "seg_slice", "seg_concat",
           "seg_scale", "seg_expand"]

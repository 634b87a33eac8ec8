"""ctypes front of oracle/fitness_ref.c (TEST ORACLE ONLY) + pure-Python pieces.

Builds oracle/_build/libfitness_ref.so with gcc on first use.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "fitness_ref.c"
LIB = HERE / "_build" / "libfitness_ref.so"

_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        LIB.parent.mkdir(parents=True, exist_ok=True)
        tmp = LIB.with_suffix(".tmp.so")
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", str(SRC),
                        "-o", str(tmp), "-lm"], check=True)
        tmp.replace(LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(build()))
        _lib.ref_lstm_ctc_one.restype = C.c_int
        _lib.ref_levenshtein.restype = C.c_int
        _lib.ref_py_sum.restype = C.c_double
        _lib.ref_eq10.restype = C.c_double
        _lib.ref_eq10.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double, C.c_double,
                                  C.c_void_p]
        _lib.ref_py_sum.argtypes = [C.c_void_p, C.c_int, C.c_int]
    return _lib


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def lstm_ctc(rows: np.ndarray, F: int, weights: dict) -> list[int]:
    """Decode one trace (rows: (T, 9) float64) with one predictor's weights
    (w_ihT [F,4H], w_hhT [H,4H], b [4H], w_out [NC,H], b_out [NC])."""
    L = lib()
    rows = np.ascontiguousarray(rows, dtype=np.float64)
    H = weights["w_hhT"].shape[0]
    NC = weights["w_out"].shape[0]
    ws = {k: np.ascontiguousarray(v, dtype=np.float32) for k, v in weights.items()}
    h = np.zeros(H, np.float32)
    c = np.zeros(H, np.float32)
    g = np.zeros(4 * H, np.float32)
    hn = np.zeros(H, np.float32)
    toks = np.zeros(max(rows.shape[0], 1), np.int8)
    n = L.ref_lstm_ctc_one(_p(rows), C.c_int(rows.shape[0]), C.c_int(F), C.c_int(H), C.c_int(NC), _p(ws["w_ihT"]),
                           _p(ws["w_hhT"]), _p(ws["b"]), _p(ws["w_out"]), _p(ws["b_out"]), _p(h), _p(c), _p(g),
                           _p(hn), _p(toks))
    return [int(t) for t in toks[:n]]


def levenshtein(a, b) -> int:
    """Unit-cost edit distance."""
    L = lib()
    a8 = np.asarray(list(a), dtype=np.int8)
    b8 = np.asarray(list(b), dtype=np.int8)
    r0 = np.zeros(len(b8) + 1, np.int32)
    r1 = np.zeros(len(b8) + 1, np.int32)
    return L.ref_levenshtein(_p(a8) if len(a8) else None, C.c_int(len(a8)), _p(b8) if len(b8) else None,
                             C.c_int(len(b8)), _p(r0), _p(r1))


def ler(pred, truth) -> float:
    """LER = ED / |L*|."""
    return levenshtein(pred, truth) / len(truth)


def eq10(lers, T: float, feasible: bool, Tstar: float, budget: float, eps: float = 0.05) -> tuple[float, float]:
    """Eq. 10 -> (R, mean LER)."""
    L = lib()
    v = np.ascontiguousarray(lers, dtype=np.float64)
    mean = np.zeros(1, np.float64)
    r = L.ref_eq10(_p(v), len(v), T, int(bool(feasible)), Tstar, budget, eps, _p(mean))
    return r, float(mean[0])

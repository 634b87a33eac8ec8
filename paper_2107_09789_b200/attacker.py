"""Attacker + fitness stage on the GPU: bagged LSTM sequence predictors, greedy CTC,
Levenshtein / LER and the Eq. 10 reward.

The reference package has no code for this stage (the attacker
and GA modules of SPEC.md:417-607 are absent); names follow the SPEC
(``levenshtein``, ``ler``, ``fitness``, ``FitnessReport``) and the paper's
attacker (PAPER.md:425-433: single-layer LSTM + CTC; :623 bagging of three
case-C predictors with H = 128/256/512). Predictor weights are seeded random
(training is a later row), drawn uniform(-1/sqrt(H), 1/sqrt(H))
as torch.nn.LSTM does and rounded to bf16-representable float32 values.

Decoded tokens, edit distances, LER and R are bit-exact against the CPU
restatement in oracle/fitness_ref.c (fixed-order fmaf, IEEE-only
transcendentals, see csrc/detmath.h).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from .engine import device
from .ir import OperatorKind as K

BLANK = 0
LABEL_CODES = {K.Conv2D: 1, K.Linear: 2, K.MaxPool: 3, K.SoftMax: 4}
CODE_LABELS = {v: k for k, v in LABEL_CODES.items()}
NUM_CLASSES = 5
EPSILON = 0.05


def encode_labels(seq) -> np.ndarray:
    """OperatorKind sequence (graph.label_sequence) -> int8 label codes."""
    return np.asarray([LABEL_CODES[k] for k in seq], dtype=np.int8)


def _bf16_round(a: np.ndarray) -> np.ndarray:
    u = a.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


@dataclass
class Predictor:
    """One single-layer LSTM + linear head (gate order i, f, g, o)."""

    hidden: int
    features: int
    w_ihT: np.ndarray   # [F][4H]
    w_hhT: np.ndarray   # [H][4H]
    b: np.ndarray       # [4H]
    w_out: np.ndarray   # [NC][H]
    b_out: np.ndarray   # [NC]
    _dev: dict = field(default_factory=dict, repr=False)

    def weights(self) -> dict:
        return {"w_ihT": self.w_ihT, "w_hhT": self.w_hhT, "b": self.b, "w_out": self.w_out, "b_out": self.b_out}

    def device_weights(self, ctx) -> dict:
        if not self._dev:
            self._dev = {k: torch.from_numpy(np.ascontiguousarray(v)).to(ctx.device)
                         for k, v in self.weights().items()}
        return self._dev


def init_predictor(hidden: int, features: int = 9, classes: int = NUM_CLASSES, seed: int = 0) -> Predictor:
    rng = np.random.default_rng(seed)
    bound = 1.0 / np.sqrt(hidden)
    u = lambda *shape: _bf16_round(rng.uniform(-bound, bound, shape))  # noqa: E731
    return Predictor(hidden, features, u(features, 4 * hidden), u(hidden, 4 * hidden), u(4 * hidden),
                     u(classes, hidden), u(classes))


def bagged_predictors(features: int = 9, hiddens=(128, 256, 512), seed: int = 0) -> list[Predictor]:
    """The three 'elite' case-C predictors of PAPER.md:623 (seeded init)."""
    return [init_predictor(h, features, seed=seed + i) for i, h in enumerate(hiddens)]


# ---------------------------------------------------------------------------
# device stages
# ---------------------------------------------------------------------------

def decode(feats: torch.Tensor, offsets: torch.Tensor, ntraces: int, t_max: int, pred: Predictor,
           stream: int | None = None):
    """LSTM + greedy CTC over device-resident trace rows -> (tokens[B,T_max] int8, ntok[B] int32).
    ``stream``: raw cudaStream_t to launch on (default: the engine stream)."""
    ctx = device()
    w = pred.device_weights(ctx)
    tokens = torch.zeros((ntraces, t_max), dtype=torch.int8, device=ctx.device)
    ntok = torch.empty(ntraces, dtype=torch.int32, device=ctx.device)
    ctx.check(ctx.lib.tobf_lstm_ctc(C.c_void_p(feats.data_ptr()), C.c_void_p(offsets.data_ptr()), ntraces,
                                    pred.features, pred.hidden, w["w_out"].shape[0],
                                    C.c_void_p(w["w_ihT"].data_ptr()), C.c_void_p(w["w_hhT"].data_ptr()),
                                    C.c_void_p(w["b"].data_ptr()), C.c_void_p(w["w_out"].data_ptr()),
                                    C.c_void_p(w["b_out"].data_ptr()), C.c_void_p(tokens.data_ptr()), t_max,
                                    C.c_void_p(ntok.data_ptr()), C.c_void_p(ctx.sp if stream is None else stream)),
              "lstm+ctc")
    ctx.launches += 1
    return tokens, ntok


def edit_distances(tokens: torch.Tensor, ntok: torch.Tensor, truth: np.ndarray, stream: int | None = None):
    """Warp-per-pair Levenshtein against one truth -> (ed int32, ler float64) on the device."""
    ctx = device()
    B, t_max = tokens.shape
    tr = truth if isinstance(truth, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(truth, dtype=np.int8)).to(ctx.device)
    ed = torch.empty(B, dtype=torch.int32, device=ctx.device)
    lr = torch.empty(B, dtype=torch.float64, device=ctx.device)
    ctx.check(ctx.lib.tobf_levenshtein(C.c_void_p(tokens.data_ptr()), C.c_void_p(ntok.data_ptr()), B, t_max,
                                       C.c_void_p(tr.data_ptr()), tr.numel(), C.c_void_p(ed.data_ptr()),
                                       C.c_void_p(lr.data_ptr()), C.c_void_p(ctx.sp if stream is None else stream)),
              "levenshtein")
    ctx.launches += 1
    return ed, lr, tr


def reward(lers: torch.Tensor, T: torch.Tensor, feasible: torch.Tensor, t_star: float, budget: float,
           eps: float = EPSILON):
    """Eq. 10 on the device. lers: (npred, ncand) float64."""
    ctx = device()
    npred, ncand = lers.shape
    R = torch.empty(ncand, dtype=torch.float64, device=ctx.device)
    mean = torch.empty(ncand, dtype=torch.float64, device=ctx.device)
    lers = lers.contiguous()
    ctx.check(ctx.lib.tobf_fitness_eq10(C.c_void_p(lers.data_ptr()), npred, ncand, C.c_void_p(T.data_ptr()),
                                        C.c_void_p(feasible.data_ptr()), float(t_star), float(budget), float(eps),
                                        C.c_void_p(R.data_ptr()), C.c_void_p(mean.data_ptr()),
                                        C.c_void_p(ctx.sp)), "eq10")
    ctx.launches += 1
    return R, mean


# ---------------------------------------------------------------------------
# SPEC-level API
# ---------------------------------------------------------------------------

def levenshtein(a, b) -> int:
    """Unit-cost edit distance between two token lists."""
    ctx = device()
    a8 = np.asarray([int(x) for x in a], dtype=np.int8)
    n = len(a8)
    toks = torch.zeros((1, max(n, 1)), dtype=torch.int8)
    toks[0, :n] = torch.from_numpy(a8)
    ed, _, _ = edit_distances(toks.to(ctx.device), torch.tensor([n], dtype=torch.int32, device=ctx.device),
                              np.asarray([int(x) for x in b], dtype=np.int8))
    return int(ed.cpu()[0])


class EmptyTruth(ValueError):
    pass


def ler(pred, truth) -> float:
    """LER = ED(L, L*) / |L*|."""
    if len(truth) == 0:
        raise EmptyTruth("truth sequence is empty")
    return levenshtein(pred, truth) / len(truth)


@dataclass
class FitnessReport:
    """SPEC.md:537-541."""

    plan: object
    latency: float
    clean_latency: float
    metrics: list[float]
    mean_metric: float
    reward: float
    feasible: bool = True
    equivalent: bool | None = None
    worst_rel: float | None = None


def eq10(mean_metric: float, T: float, t_star: float, budget: float, eps: float = EPSILON) -> float:
    """Eq. 10 on the host, for report checks."""
    return mean_metric / (eps + ((T - (1 + budget) * t_star) / t_star) ** 2)

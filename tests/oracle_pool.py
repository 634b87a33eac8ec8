"""Process-pool front of the CPU oracle for the full-size parity tests
(TEST INFRASTRUCTURE ONLY: the checker, never the thing measured).

The full-size configurations (ResNet-18 / VGG-16 at 224x224, 8 equivalence
trials, >= 1000 LSTM traces) are minutes of single-core numpy/C work; the jobs
are independent, so they are spread over the host's cores (one spawned worker
per core, single-threaded BLAS, like bench.py's cpu_baseline). The schedule
memo is NOT parallelised: the trace oracle runs in the parent, in candidate
order, with one memo (costmodel.py:248 first-seen semantics).
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

_S: dict = {}


def _init(vanilla, trials, seed):
    try:
        from threadpoolctl import threadpool_limits
        _S["limits"] = threadpool_limits(1)
    except ImportError:
        pass
    _S.update(vanilla=vanilla, trials=trials, seed=seed)


def equiv_job(plan):
    """(ok, worst, pre-softmax max rel diff vs fp64) for one plan, or None if infeasible."""
    from oracle import interp_ref as IR
    from paper_2107_09789_b200.knobs import TransformError, apply_plan
    try:
        og, _ = apply_plan(_S["vanilla"], plan)
    except TransformError:
        return None
    return IR.equivalence_check(_S["vanilla"], og, trials=_S["trials"], seed=_S["seed"])


def equiv64_job(plan):
    """equivalence_check's `worst` in float64 arithmetic (the exact-arithmetic
    yardstick) on the same float32 inputs."""
    from oracle import interp_ref as IR
    from paper_2107_09789_b200.knobs import apply_plan
    og, _ = apply_plan(_S["vanilla"], plan)
    worst = 0.0
    for x in IR.trial_inputs(tuple(_S["vanilla"].input_shape.as_tuple()), _S["trials"], _S["seed"]):
        a = IR.execute(_S["vanilla"], x, dtype=np.float64)
        b = IR.execute(og, x, dtype=np.float64)
        worst = max(worst, float((np.abs(a - b) / (1.0 + np.abs(b))).max()))
    return worst


def equiv_trial_job(args):
    """One (plan, trial index) of equivalence_check (interpreter.py:110-117):
    returns (worst, ok) of that trial so the parent folds them in trial order.
    The plan is applied in the worker (VGG-16 candidates are ~1 GB of weights)."""
    from oracle import interp_ref as IR
    from paper_2107_09789_b200.knobs import apply_plan
    plan, t = args
    key = repr(plan)
    if _S.get("plan_key") != key:
        _S["plan_key"], _S["og"] = key, apply_plan(_S["vanilla"], plan)[0]
    og = _S["og"]
    xs = IR.trial_inputs(tuple(_S["vanilla"].input_shape.as_tuple()), t + 1, _S["seed"])
    x = xs[t]
    a = IR.execute(_S["vanilla"], x)
    b = IR.execute(og, x)
    d = np.abs(a - b)
    den = 1.0 + np.abs(b)
    return float((d / den).max()), bool(np.all(d <= 1e-5 * den))


def execute_job(args):
    """Oracle output of one graph on one input."""
    from oracle import interp_ref as IR
    g, x = args
    return IR.execute(g, x)


def lstm_job(args):
    from oracle import fitness_ref as FR
    rows, F, w = args
    return FR.lstm_ctc(rows, F, w)


def pool(vanilla=None, trials: int = 8, seed: int = 0, procs: int | None = None):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    n = procs or max(1, len(os.sched_getaffinity(0)))
    return mp.get_context("spawn").Pool(n, initializer=_init, initargs=(vanilla, trials, seed))

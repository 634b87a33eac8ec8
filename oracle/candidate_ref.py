"""One GA candidate evaluated entirely on the CPU — the reference path restated
(TEST / BASELINE INFRASTRUCTURE ONLY; used by tests and by bench.py's
cpu_baseline and ``--impl reference`` arm).

Per candidate, exactly the work the reference would do:
  apply_plan                      transforms.py:400-474
  equivalence_check(vanilla, c)   interpreter.py:93-118 (``trials`` x 2 executes)
  profile_pipeline, cold memo     costmodel.py:266-293 (schedule brute force)
  3 bagged LSTM + greedy CTC      PAPER.md:425,623 (restated, oracle/fitness_ref.c)
  Levenshtein LER vs L*, Eq. 10

apply_plan uses the engine's host mirror (paper_2107_09789_b200.knobs, pure
numpy, node-for-node equal to the reference's and faster than it: this only
flatters the baseline). Workers run single-threaded BLAS.
"""

from __future__ import annotations

import os
import time

import numpy as np

_STATE = {}


def init_worker(vanilla, predictors, t_star, budget, trials, seed, blas_threads=1):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(blas_threads))
    try:
        from threadpoolctl import threadpool_limits
        _STATE["limits"] = threadpool_limits(blas_threads)
    except ImportError:
        pass
    from . import fitness_ref
    fitness_ref.lib()  # build/load once per worker
    from paper_2107_09789_b200.ir import label_sequence
    codes = {"Conv2D": 1, "Linear": 2, "MaxPool": 3, "SoftMax": 4}
    _STATE.update(vanilla=vanilla, predictors=predictors, t_star=t_star, budget=budget, trials=trials, seed=seed,
                  truth=[codes[k.value] for k in label_sequence(vanilla)])


def evaluate_candidate(plan) -> dict:
    from paper_2107_09789_b200.knobs import TransformError, apply_plan

    from . import costmodel_ref, fitness_ref, interp_ref
    st = _STATE
    t0 = time.perf_counter()
    try:
        og, d = apply_plan(st["vanilla"], plan)
    except TransformError:
        return {"reward": 0.0, "feasible": False, "seconds": time.perf_counter() - t0}
    t1 = time.perf_counter()
    ok, worst = interp_ref.equivalence_check(st["vanilla"], og, trials=st["trials"], seed=st["seed"])
    t2 = time.perf_counter()
    _, _, rows, T = costmodel_ref.profile_pipeline(og, "default", d.fusion_limits, d.schedule_strategies,
                                                   costmodel_ref.ScheduleMemo())
    t3 = time.perf_counter()
    feats = np.array([[r[f] for f in costmodel_ref.FEATURES] for r in rows], dtype=np.float64)
    lers = [fitness_ref.ler(fitness_ref.lstm_ctc(feats, p["F"], p["w"]), st["truth"]) for p in st["predictors"]]
    R, mean = fitness_ref.eq10(lers, T, ok, st["t_star"], st["budget"])
    t4 = time.perf_counter()
    return {"reward": R, "mean_ler": mean, "latency": T, "ok": ok, "worst": worst, "feasible": True,
            "seconds": t4 - t0, "stages": {"apply_plan": t1 - t0, "forward": t2 - t1, "trace": t3 - t2,
                                           "fitness": t4 - t3}}

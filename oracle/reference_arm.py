"""The reference's OWN candidate evaluation on the host CPU — BASELINE
INFRASTRUCTURE ONLY (bench.py's ``--impl reference`` arm and cpu_baseline).

Runs the unmodified reference package (traceobf 0.1.0, vendored into
baseline/_ref by scripts/vendor_reference.sh) through its public API, per
candidate exactly the work of one GA fitness evaluation:

  apply_plan                       transforms.py:400-474   (reference code)
  equivalence_check(vanilla, c)    interpreter.py:93-118   (reference code, ``trials`` x 2 executes)
  profile_pipeline, case C         costmodel.py:266-293    (reference code; its module-global
                                   _SCHEDULE_CACHE cold at every step, kept within a step)
  3 bagged LSTM + greedy CTC       PAPER.md:425,623 — no reference code: the C restatement
  Levenshtein LER vs L*, Eq. 10    SPEC.md:471-486, 563-571 — oracle/fitness_ref.c

Two modes: one process with the default BLAS threads, and one
worker process per core with single-threaded BLAS (candidates are
independent). Without baseline/_ref (not vendored) ``load_reference`` returns
None and the caller falls back to the restated port (candidate_ref.py).
"""

from __future__ import annotations

import importlib
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "baseline" / "_ref"

_STATE: dict = {}


def load_reference():
    """The vendored reference package, or None."""
    if not (REF_DIR / "traceobf" / "__init__.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    return importlib.import_module("traceobf")


def ref_graph(ref, g):
    """A graph (engine fixture) rebuilt in the reference's own classes."""
    nodes = {nid: ref.Node(n.id, ref.OperatorKind(n.kind.value), dict(n.attrs), n.weights, list(n.inputs))
             for nid, n in g.nodes.items()}
    s = g.input_shape
    return ref.Graph(nodes, g.output_id, ref.TensorShape(s.batch, s.channels, s.height, s.width))


def plan_wire(plan) -> tuple:
    return plan.mode, tuple(tuple(vars(e).items()) for e in plan.entries)


def init_worker(vanilla, predictors, t_star, budget, trials, seed, blas_threads=1):
    if blas_threads:
        os.environ["OPENBLAS_NUM_THREADS"] = str(blas_threads)
        try:
            from threadpoolctl import threadpool_limits
            _STATE["limits"] = threadpool_limits(blas_threads)
        except ImportError:
            pass
    from . import fitness_ref
    fitness_ref.lib()
    ref = load_reference()
    if ref is None:
        raise RuntimeError("baseline/_ref is not vendored (scripts/vendor_reference.sh)")
    g = ref_graph(ref, vanilla)
    codes = {"Conv2D": 1, "Linear": 2, "MaxPool": 3, "SoftMax": 4}
    _STATE.update(ref=ref, vanilla=g, predictors=predictors, t_star=t_star, budget=budget, trials=trials,
                  seed=seed, truth=[codes[k.value] for k in ref.label_sequence(g)], step=None)


def evaluate_candidate(job) -> dict:
    """job = (step id, plan_wire tuple): one candidate through the reference."""
    from . import fitness_ref
    step, (mode, entries) = job
    st = _STATE
    ref = st["ref"]
    if st["step"] != step:  # cold schedule memo at every step (bench.py's GPU arm: cold every step)
        ref.costmodel._SCHEDULE_CACHE.clear()
        st["step"] = step
    plan = ref.ObfuscationPlan(mode, tuple(ref.PlanEntry(**dict(e)) for e in entries))
    t0 = time.perf_counter()
    try:
        og, d = ref.apply_plan(st["vanilla"], plan)
    except ref.transforms.TransformError:
        return {"reward": 0.0, "feasible": False, "seconds": time.perf_counter() - t0}
    t1 = time.perf_counter()
    ok, worst = ref.equivalence_check(st["vanilla"], og, trials=st["trials"], seed=st["seed"])
    t2 = time.perf_counter()
    tr = ref.profile_pipeline(og, ref.LeakageCase.C, ref.BUILTIN_PROFILES["default"], d.fusion_limits,
                              d.schedule_strategies)
    T = tr.total_latency
    t3 = time.perf_counter()
    feats = tr.feature_matrix()
    lers = [fitness_ref.ler(fitness_ref.lstm_ctc(feats, p["F"], p["w"]), st["truth"]) for p in st["predictors"]]
    R, mean = fitness_ref.eq10(lers, T, ok, st["t_star"], st["budget"])
    t4 = time.perf_counter()
    return {"reward": R, "mean_ler": mean, "latency": T, "ok": bool(ok), "worst": float(worst), "feasible": True,
            "seconds": t4 - t0, "stages": {"apply_plan": t1 - t0, "forward": t2 - t1, "trace": t3 - t2,
                                           "fitness": t4 - t3}}


def vanilla_t_star(vanilla) -> float:
    """T* through the reference's own profile_pipeline (cold memo)."""
    ref = load_reference()
    g = ref_graph(ref, vanilla)
    ref.costmodel._SCHEDULE_CACHE.clear()
    t = ref.profile_pipeline(g, ref.LeakageCase.C, ref.BUILTIN_PROFILES["default"]).total_latency
    ref.costmodel._SCHEDULE_CACHE.clear()
    return t

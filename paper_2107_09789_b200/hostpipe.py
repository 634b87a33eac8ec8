"""Host preparation of candidate batches in worker processes.

The per-candidate host work of a GA generation — apply_plan
(transforms.py:441-474), lowering, forward descriptor rows and the trace's
kernel records (costmodel.py:248-285 host half) — is pure Python/numpy and
independent across candidates. A pool of worker processes (fresh
interpreters: they never touch CUDA) runs it and returns picklable,
device-free results:

  ForwardPlan      descriptor rows with symbolic pointers (executor.py)
  CandidateTrace   kernel records + schedule signatures (trace.py)
  new arrays       weight roots the candidate created itself (rare)

Weights cross the process boundary as references: ("v", nid) a vanilla
node's weight array, ("c", key) a shared knob constant (knobs._CONSTS), or
("n", cand, i) an array shipped with the result. The parent rebuilds views
on ITS arrays, so the device weight cache (keyed by root identity) still
uploads each vanilla array once per cache life.

The parent links, uploads and launches (PopulationRun, prepare_trace_records);
first-seen schedule-memo semantics are applied there, in candidate order.
"""

from __future__ import annotations

import dataclasses
import os
import subprocess
import sys
from multiprocessing.connection import Connection
from pathlib import Path

import numpy as np

from . import knobs
from .engine import _root
from .executor import ArrayRefs, ForwardPlan, lower, plan_forward
from .ir import Graph, analyze
from .knobs import ObfuscationPlan, PlanEntry, TransformError, apply_plan_analyzed
from .trace import CandidateTrace, trace_records


def _const_key_of(root: np.ndarray):
    for key, arr in knobs._CONSTS.items():
        if arr is root:
            return key
    return None


class WorkerRefs(ArrayRefs):
    """Worker side: name roots so the parent can rebuild them."""

    def __init__(self, vanilla_roots: dict, cand: int):
        super().__init__()
        self.vanilla_roots = vanilla_roots  # id(root) -> ("v", nid)
        self.cand = cand
        self.new: list[np.ndarray] = []
        self._new_ids: dict[int, int] = {}
        self._const_ids: dict[int, tuple] = {}

    def root_key(self, root: np.ndarray):
        rid = id(root)
        key = self.vanilla_roots.get(rid)
        if key is not None:
            return key
        key = self._const_ids.get(rid)
        if key is None:
            ck = _const_key_of(root)
            if ck is not None:
                key = self._const_ids[rid] = ("c",) + tuple(ck)
        if key is not None:
            return key
        i = self._new_ids.get(rid)
        if i is None:
            i = self._new_ids[rid] = len(self.new)
            self.new.append(np.ascontiguousarray(root))
        return ("n", self.cand, i)


class ParentRefs(ArrayRefs):
    """Parent side: resolve worker references onto the parent's arrays."""

    def __init__(self, vanilla: Graph):
        super().__init__()
        self.vanilla = {("v", nid): _root(n.weights) for nid, n in vanilla.nodes.items()
                        if isinstance(n.weights, np.ndarray)}
        self.new: dict[tuple, np.ndarray] = {}
        self.sig_table: dict[int, tuple] = {}  # digest -> schedule signature (workers send each once)

    def root(self, key) -> np.ndarray:
        tag = key[0]
        if tag == "v":
            return self.vanilla[key]
        if tag == "c":
            ck = tuple(key[1:])
            arr = knobs._CONSTS.get(ck)
            if arr is None:
                arr = knobs._shared_zeros(ck[1:]) if ck[0] == "zeros" else knobs._shared_identity(ck[1])
            return arr
        if tag == "n":
            return self.new[key]
        return super().root(key)

    def adopt(self, cand: int, arrays: list[np.ndarray]) -> None:
        for i, a in enumerate(arrays):
            self.new[("n", cand, i)] = a


# ------------------------------------------------------------------ worker
_W: dict = {}


def _worker_init(vanilla: Graph, reps: int, pname: str, prec: int = 0) -> None:
    _W["vanilla"] = vanilla
    _W["prec"] = prec
    _W["analysis"] = analyze(vanilla)
    _W["reps"] = reps
    _W["pname"] = pname
    _W["roots"] = {id(_root(n.weights)): ("v", nid) for nid, n in vanilla.nodes.items()
                   if isinstance(n.weights, np.ndarray)}
    _W["sent_sigs"] = set()  # signature digests this worker has sent to its parent


# knob weights as device-packed gathers (derived.py); TOBF_EAGER_KNOBS=1 ships
# materialised arrays instead (A/B measurements only)
LAZY_KNOBS = os.environ.get("TOBF_EAGER_KNOBS", "") != "1"


def encode_candidate(cand: int, plan: ObfuscationPlan, vanilla: Graph, vanilla_analysis, reps: int, pname: str,
                     roots: dict, sent_sigs: set | None = None, prec: int = 0):
    """(cand, error, payload): payload = (ForwardPlan, CandidateTrace, new arrays)."""
    try:
        g, d, ana = apply_plan_analyzed(vanilla, plan, vanilla_analysis, lazy=LAZY_KNOBS)
    except TransformError as exc:
        return cand, str(exc), None
    refs = WorkerRefs(roots, cand)
    fp = plan_forward(lower(g, ana), reps, refs, prec)
    ct, _, _ = trace_records(g, d.fusion_limits, d.schedule_strategies, pname, ana)
    if sent_sigs is not None:
        ct = ct.compact(sent_sigs)
    return cand, None, (fp, ct, refs.new)


_PLAN_FIELDS = tuple(f.name for f in dataclasses.fields(PlanEntry))


def plan_wire(plan: ObfuscationPlan) -> tuple:
    """A plan as nested plain tuples (pickles ~5x faster than the dataclasses:
    at P = 256 the job dealing alone took ~5 ms)."""
    return plan.mode, tuple(tuple(e.__dict__.values()) for e in plan.entries)  # field order (dataclass init)


def plan_unwire(w: tuple) -> ObfuscationPlan:
    return ObfuscationPlan(w[0], tuple(PlanEntry(*row) for row in w[1]))


def _worker_job(job: list[tuple[int, tuple]]) -> list:
    return [encode_candidate(c, plan_unwire(p), _W["vanilla"], _W["analysis"], _W["reps"], _W["pname"],
                             _W["roots"], _W["sent_sigs"], _W["prec"]) for c, p in job]


def _worker_main(rfd: int, wfd: int) -> None:
    rconn = Connection(rfd, writable=False)
    wconn = Connection(wfd, readable=False)
    vanilla, reps, pname, prec = rconn.recv()
    _worker_init(vanilla, reps, pname, prec)
    while True:
        msg = rconn.recv()
        if msg is None:
            break
        for jid, job in msg:  # this worker's jobs of one submit, answered one by one
            wconn.send((jid, _worker_job(job)))


class HostPool:
    """Worker processes preparing candidates of one vanilla graph.

    Each worker is a fresh interpreter (``python -m
    paper_2107_09789_b200.hostpipe``: no CUDA state, no re-import of the
    caller's __main__) talking over two pipes; no helper threads compete for
    the parent's GIL. Jobs are dealt round-robin and each worker answers its
    jobs in order, so a result is received on the parent's thread exactly
    when it is needed."""

    def __init__(self, vanilla: Graph, reps: int, pname: str, workers: int | None = None, prec: int = 0):
        n = workers if workers is not None else default_workers()
        self.workers = n
        self.procs, self.wconns, self.rconns = [], [], []
        env = dict(os.environ)
        root = str(Path(__file__).resolve().parents[1])
        env["PYTHONPATH"] = root + (os.pathsep + env["PYTHONPATH"] if env.get("PYTHONPATH") else "")
        env["CUDA_VISIBLE_DEVICES"] = ""  # workers never need a GPU
        for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            env[var] = "1"  # one core per worker: no BLAS / OpenMP thread pools oversubscribing the host
        for _ in range(n):
            to_r, to_w = os.pipe()      # parent -> worker
            from_r, from_w = os.pipe()  # worker -> parent
            p = subprocess.Popen([sys.executable, "-m", "paper_2107_09789_b200.hostpipe", str(to_r), str(from_w)],
                                 pass_fds=(to_r, from_w), env=env, cwd=root)
            os.close(to_r)
            os.close(from_w)
            self.procs.append(p)
            self.wconns.append(Connection(to_w, readable=False))
            self.rconns.append(Connection(from_r, writable=False))
        for c in self.wconns:
            c.send((vanilla, reps, pname, prec))
        self._next = 0
        self._jid = 0
        self._done: dict[int, list] = {}

    def submit(self, plans: list[ObfuscationPlan], first: int = 0, per_job: int = 1) -> list[tuple[int, int]]:
        """Deal jobs of ``per_job`` candidates round-robin, one message per
        worker (a send per job cost ~15 us of parent time each); returns
        handles (worker, job id) in order."""
        handles = []
        per_worker: list[list] = [[] for _ in range(self.workers)]
        for i in range(0, len(plans), per_job):
            job = [(first + i + q, plan_wire(plans[i + q])) for q in range(min(per_job, len(plans) - i))]
            w = self._next
            self._next = (self._next + 1) % self.workers
            per_worker[w].append((self._jid, job))
            handles.append((w, self._jid))
            self._jid += 1
        for w, jobs in enumerate(per_worker):
            if jobs:
                self.wconns[w].send(jobs)
        return handles

    def result(self, handle: tuple[int, int]) -> list:
        """encode_candidate tuples of one job (blocks until it is done)."""
        w, jid = handle
        while jid not in self._done:
            try:
                got, res = self.rconns[w].recv()
            except EOFError as exc:
                raise RuntimeError(f"host worker {w} exited (rc={self.procs[w].poll()})") from exc
            self._done[got] = res
        return self._done.pop(jid)

    def close(self) -> None:
        for c in self.wconns:
            try:
                c.send(None)
            except (BrokenPipeError, OSError):
                pass
        for p in self.procs:
            try:
                p.wait(timeout=10)
            except subprocess.TimeoutExpired:
                p.kill()
                p.wait()
        for c in self.wconns + self.rconns:
            c.close()
        self.procs, self.wconns, self.rconns = [], [], []

    def __del__(self):
        if self.procs:
            self.close()


def default_workers() -> int:
    env = os.environ.get("TOBF_HOST_WORKERS")
    if env:
        return max(1, int(env))
    # one GPU process per rank shares the host: split the cores the parents
    # leave free between the node's ranks (torchrun's LOCAL_WORLD_SIZE)
    ranks = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 2)
    return max(1, min(16, (cores - ranks - 1) // ranks))


__all__ = ["ForwardPlan", "CandidateTrace", "WorkerRefs", "ParentRefs", "HostPool", "encode_candidate",
           "default_workers"]


if __name__ == "__main__":
    _worker_main(int(sys.argv[1]), int(sys.argv[2]))

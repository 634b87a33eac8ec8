"""Multi-rank first-seen schedule memo on CPU (gloo, world size 2 and 3).

The reference memoises default schedules process-globally, first occurrence
wins (costmodel.py:248-285). Sharded over ranks, the engine
resolves that memo once per shard evaluation (trace.resolve_first_seen +
dist.exchange_signatures) and then runs the REAL host half of the trace stage,
trace.prepare_trace_records, per micro-batch (its device uploads go to a
CPU stand-in context here). Checked, against one process evaluating the whole
population in order:

  * exactly one collective per rank per evaluation, whatever the shard holds:
    P = 9 (uneven shards), P = 1 < world (empty shards), an all-infeasible
    shard — so no rank can hang waiting for a partner;
  * every signature is searched from its globally first descriptor (micro-
    batch splits differ per rank on purpose);
  * after folding the searched tables into the memos (finish_trace's rule),
    every rank's memo equals the single-process memo, so the next generation
    starts identical everywhere.
"""

import hashlib
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_2107_09789_b200 import dist as D
from paper_2107_09789_b200 import fixtures, ga, knobs
from paper_2107_09789_b200 import trace as T
from paper_2107_09789_b200.evaluate import _micro_bounds
from paper_2107_09789_b200.kernels import Schedule


class _HostCtx:
    """CPU stand-in for engine.Context's upload methods (no device needed)."""

    def upload_bytes(self, buf):
        return torch.from_numpy(np.frombuffer(bytes(buf), dtype=np.uint8).copy())

    def upload_array(self, a):
        return torch.from_numpy(np.ascontiguousarray(a).copy())


def _population(P: int, seed: int, infeasible: set):
    """Trace records of P ResNet-18 (64x64) sequence candidates in global order;
    None where the plan is infeasible (deepen of a layer whose activation
    chain has no ReLU raises NoActivation)."""
    g = fixtures.resnet18(size=64)
    rng = np.random.default_rng(seed)
    space = ga.search_space(g, "sequence")
    sizes = ga.domain_sizes("sequence", space)
    out = []
    for i, gen in enumerate(ga.random_genomes(rng, sizes, P)):
        plan = ga.decode_genome(g, "sequence", space, gen)
        if i in infeasible:
            out.append(None)
            continue
        og, d = knobs.apply_plan(g, plan)
        out.append(T.trace_records(og, d.fusion_limits, d.schedule_strategies, "default")[0])
    return out


def _search(blob: bytes) -> Schedule:
    """Stand-in for the device schedule search: a pure function of the descriptor."""
    h = hashlib.blake2b(blob, digest_size=6).digest()
    return Schedule(tuple(1 + v for v in h[:3]), tuple(1 + v for v in h[3:]), 4)


def _evaluate_shard(cts_all, P, ws, rank, micro, memo, exchange):
    """evaluate_records' trace-side flow for this rank's shard."""
    rng = D.shard(P, ws, rank)
    mine = [cts_all[i] for i in rng]
    ok = [k for k, ct in enumerate(mine) if ct is not None]
    glob = T.resolve_first_seen([mine[k] for k in ok], [rng.start + k for k in ok], memo, exchange)
    first_seen, extra = dict(glob), glob
    searched = {}
    bounds = _micro_bounds(len(mine), micro) if mine else [(0, 0)]
    for b, (lo, hi) in enumerate(bounds):
        cts = [ct for ct in mine[lo:hi] if ct is not None]
        ex = extra if b == 0 else None
        if not cts and not ex:
            continue
        tp = T.prepare_trace_records(cts, T.BUILTIN_PROFILES["default"], memo, first_seen=first_seen, extra=ex)
        table = tp.sigs.numpy().tobytes()
        size = T.KERN_DTYPE.itemsize
        for i, sig in tp.pending:
            got = _search(table[i * size:(i + 1) * size])
            assert searched.setdefault(sig, got) == got  # a re-search uses the same descriptor
    for sig, s in searched.items():  # finish_trace: first result wins
        memo.setdefault(sig, s)
    return {sig: s for sig, s in memo.items() if sig[1] in T._COMPLEX_VALUES}


CASES = [  # (P, infeasible global indices)
    (9, set()),
    (1, set()),
    (9, {0, 1, 2, 3, 4}),  # rank 0's whole shard (ws 2: 5 candidates; ws 3: 3) is infeasible
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, q):
    import paper_2107_09789_b200.trace as tr
    tr.device = lambda: _HostCtx()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    calls = [0]

    def counting_exchange(local):
        calls[0] += 1
        return D.exchange_signatures(local)

    try:
        out = []
        memo = {}  # persists across the cases, like the GA's memo across generations
        for case in CASES:
            P, bad = case
            cts = _population(P, 7, bad)
            before = calls[0]
            # rank-dependent micro-batch splits: must not matter
            got = _evaluate_shard(cts, P, ws, rank, (1 + rank, 2), memo, counting_exchange)
            out.append((calls[0] - before, {repr(k): repr(v) for k, v in got.items()}))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("ws", [2, 3])
def test_sharded_memo_matches_single_process(ws):
    import paper_2107_09789_b200.trace as tr
    saved = tr.device
    tr.device = lambda: _HostCtx()
    try:
        singles, memo = [], {}
        for case in CASES:  # one process, whole population, memo carried across cases
            P, bad = case
            singles.append({repr(k): repr(v) for k, v in
                            _evaluate_shard(_population(P, 7, bad), P, 1, 0, P, memo, None).items()})
    finally:
        tr.device = saved
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(ws):
        rank, out = q.get(timeout=500)
        res[rank] = out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(ws):
        for c, (ncoll, memo_r) in enumerate(res[rank]):
            assert ncoll == 1, (rank, c, ncoll)
            assert memo_r == singles[c], (rank, c)


def test_exchange_orders_by_global_index():
    """Lowest global candidate index wins, independent of rank order."""
    local = [(("a",), 5, b"late"), (("b",), 6, b"b6")]
    assert D.exchange_signatures(local) == {("a",): b"late", ("b",): b"b6"}
    # two ranks' parts merged as the collective would: rank 1 holds the earlier candidate for "a"
    import paper_2107_09789_b200.dist as dd
    saved = dd.world, dd.dist.all_gather_object
    try:
        dd.world = lambda: (2, 0)

        def fake_gather(out, obj):
            out[0], out[1] = obj, [(("a",), 2, b"early"), (("c",), 3, b"c3")]
        dd.dist.all_gather_object = fake_gather
        merged = D.exchange_signatures(local)
    finally:
        dd.world, dd.dist.all_gather_object = saved
    assert merged == {("a",): b"early", ("c",): b"c3", ("b",): b"b6"}
    assert list(merged) == [("a",), ("c",), ("b",)]

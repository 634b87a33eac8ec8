"""Population sharding across the GPUs of one box.

One process per GPU (torch.distributed; NCCL on GPUs, gloo for CPU tests).
GA candidates are independent: rank r evaluates the contiguous block
``shard(n, world, r)`` of each generation. The only exchanges are

  * ``gather_records``  — all-gather of the fixed-size fitness records
    (R, mean LER, T, verdict) so every rank holds the whole generation;
  * ``broadcast_genomes`` — rank 0's next-generation genomes to all ranks;
  * ``exchange_signatures`` — the schedule-memo first-seen exchange, once
    per shard evaluation: the reference memoises default schedules
    process-globally in candidate order (costmodel.py:248-285, SURVEY App.
    A-5). Each rank publishes, for its WHOLE shard (before any micro-batch
    runs), the signatures it has not memoised yet with the global index of
    the candidate they first occur in and that kernel's descriptor; every
    rank adopts, per signature, the descriptor of the lowest global index,
    searches the same union table and memoises all of it — so memos stay
    identical across ranks and every trace is bit-identical to one process
    evaluating the whole generation in order.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def shard(n: int, world_size: int, rank: int) -> range:
    """Contiguous block of candidates owned by ``rank`` (sizes differ by <= 1)."""
    base, extra = divmod(n, world_size)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def gather_records(local: np.ndarray, n_total: int) -> np.ndarray:
    """All-gather structured fitness records into global candidate order."""
    ws, rank = world()
    if ws == 1:
        return local
    raw = np.frombuffer(local.tobytes(), dtype=np.uint8)
    itemsize = local.dtype.itemsize
    cap = (n_total // ws + 1) * itemsize
    buf = np.zeros(cap, dtype=np.uint8)
    buf[:raw.size] = raw
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(buf).to(dev)
    out = torch.empty(ws * cap, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, t)
    allb = out.cpu().numpy().reshape(ws, cap)
    parts = []
    for r in range(ws):
        m = len(shard(n_total, ws, r))
        parts.append(np.frombuffer(allb[r, :m * itemsize].tobytes(), dtype=local.dtype))
    return np.concatenate(parts)


def broadcast_genomes(genomes: np.ndarray | None, shape: tuple[int, int]) -> np.ndarray:
    """Rank 0's genomes (int64 option indices) to every rank."""
    ws, rank = world()
    if ws == 1:
        return genomes
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(np.ascontiguousarray(genomes, dtype=np.int64)).to(dev) if rank == 0 else \
        torch.empty(shape, dtype=torch.int64, device=dev)
    dist.broadcast(t, 0)
    return t.cpu().numpy()


def exchange_signatures(local: list[tuple[tuple, int, bytes]]) -> dict[tuple, bytes]:
    """``local``: this rank's unmemoised (signature, global candidate index of
    its first occurrence, descriptor bytes), from ``trace.shard_first_seen``.
    Returns signature -> descriptor of the globally first occurrence (lowest
    candidate index; rank, then position break ties), for every signature any
    rank reported, in that global order. ONE collective per call: callers
    make exactly one call per shard evaluation on every rank, whatever the
    shard holds (trace.resolve_first_seen)."""
    ws, _ = world()
    parts = [local]
    if ws > 1:
        parts = [None] * ws
        dist.all_gather_object(parts, local)
    best: dict[tuple, tuple] = {}
    for r, part in enumerate(parts):
        for pos, (sig, gi, blob) in enumerate(part):
            key = (int(gi), r, pos)
            cur = best.get(sig)
            if cur is None or key < cur[0]:
                best[sig] = (key, blob)
    return {sig: kb[1] for sig, kb in sorted(best.items(), key=lambda it: it[1][0])}

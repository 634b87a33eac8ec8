"""Population sharding across the GPUs of one box.

One process per GPU (torch.distributed; NCCL on GPUs, gloo for CPU tests).
GA candidates are independent: rank r evaluates the contiguous block
``shard(n, world, r)`` of each generation. The only exchanges are

  * ``gather_records``  — all-gather of the fixed-size fitness records
    (R, mean LER, T, verdict) so every rank holds the whole generation;
  * ``broadcast_genomes`` — rank 0's next-generation genomes to all ranks;
  * ``exchange_signatures`` — the schedule-memo first-seen exchange: the
    reference memoises default schedules process-globally in candidate order
    (costmodel.py:248-285). Each rank publishes the
    signatures it has not memoised yet, with the kernel descriptor of its
    first occurrence; every rank then adopts, per signature, the descriptor
    of the globally first occurrence (rank order = candidate order), so the
    searched schedules — and hence every trace — are bit-identical to a
    single process evaluating the whole generation in order.
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


def exchange_signatures(local: list[tuple[tuple, bytes]]) -> dict[tuple, bytes]:
    """``local``: this rank's unmemoised (signature, descriptor bytes) in its
    first-seen order. Returns signature -> descriptor of the global first
    occurrence, for every signature any rank reported."""
    ws, _ = world()
    if ws == 1:
        return dict(local)
    gathered: list = [None] * ws
    dist.all_gather_object(gathered, local)
    first: dict[tuple, bytes] = {}
    for part in gathered:  # rank order == candidate order (contiguous shards)
        for sig, blob in part:
            first.setdefault(sig, blob)
    return first

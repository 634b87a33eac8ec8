"""N > 1 host-side path on CPU: world_size 2 over gloo (one process per rank),
checking that sharded evaluation + record all-gather + genome broadcast +
schedule-signature exchange reproduce the single-process result exactly."""

import socket
import zlib

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_2107_09789_b200 import dist as D
from paper_2107_09789_b200 import fixtures, ga
from paper_2107_09789_b200.evaluate import RECORD_DTYPE


def stable_eval(plans):
    rec = np.zeros(len(plans), dtype=RECORD_DTYPE)
    for i, p in enumerate(plans):
        h = zlib.crc32(repr(p.entries).encode())
        rec[i]["reward"] = (h % 1009) / 101.0
        rec[i]["mean_ler"] = (h % 37) / 10.0
        rec[i]["latency"] = 1e6 + (h % 5000)
        rec[i]["ok"] = 1
    return rec


def sharded_eval(plans):
    ws, rank = D.world()
    mine = [plans[i] for i in D.shard(len(plans), ws, rank)]
    return D.gather_records(stable_eval(mine), len(plans))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world_size, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world_size)
    try:
        g = fixtures.c1c2()
        params = ga.GaParams(population=8, generations=4, seed=5)
        res = ga.run_ga(g, "dimension", 0.02, params, sharded_eval)
        genomes = np.arange(12, dtype=np.int64).reshape(3, 4) * (rank + 1)
        got = D.broadcast_genomes(genomes if rank == 0 else None, (3, 4))
        local = [((f"sig{rank}",), 4 * rank, b"r%d" % rank), (("shared",), 4 * rank + 1, b"from%d" % rank)]
        merged = D.exchange_signatures(local)
        q.put((rank, res.best_genome.tolist(), res.best_reward, [x[2] for x in res.log], got.tolist(),
               sorted(merged.items())))
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for n in (1, 7, 32, 256):
        for ws in (1, 2, 3, 8):
            idx = [i for r in range(ws) for i in D.shard(n, ws, r)]
            assert idx == list(range(n))


@pytest.mark.timeout(300)
def test_two_rank_gloo_matches_single_process():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict()
    for _ in range(2):
        rank, *vals = q.get(timeout=240)
        out[rank] = vals
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = ga.run_ga(fixtures.c1c2(), "dimension", 0.02, ga.GaParams(population=8, generations=4, seed=5), stable_eval)
    for rank in (0, 1):
        best, reward, log, bcast, merged = out[rank]
        assert best == single.best_genome.tolist() and reward == single.best_reward
        assert log == [x[2] for x in single.log]
        assert bcast == (np.arange(12).reshape(3, 4)).tolist()
        # global first-seen: rank 0's descriptor wins for the shared signature
        assert merged == sorted({("sig0",): b"r0", ("sig1",): b"r1", ("shared",): b"from0"}.items())

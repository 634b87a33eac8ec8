"""Command-line GA driver (SURVEY §8(f)4; SPEC.md:572-607 search loop, :600 log).

    python -m paper_2107_09789_b200 ga --fixture resnet18 --mode sequence \
        --population 32 --generations 20 --out runs/rn18 [--resume]

One GA generation per step: the population is evaluated on the GPU(s) by
``PopulationEvaluator`` (forward + verdict, trace, bagged attackers, Eq. 10)
and the next generation is bred on the host (ga.py). Under torchrun
(``--nproc-per-node N``) every rank evaluates a contiguous shard of each
generation, records are all-gathered over NCCL, and every rank runs the same
deterministic GA step, so the search is identical for any number of GPUs.

After every generation rank 0 writes ``<out>/ckpt.pkl`` (GA state with the
RNG state, the schedule memo) atomically and appends to ``<out>/log.jsonl``;
``--resume`` continues bit-identically from the last checkpoint.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import pickle
import sys
import time
from pathlib import Path

import numpy as np


def _parse(argv):
    ap = argparse.ArgumentParser(prog="python -m paper_2107_09789_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("ga", help="run the obfuscation GA on a fixture network")
    g.add_argument("--fixture", choices=("resnet18", "vgg16", "c1c2"), default="resnet18")
    g.add_argument("--size", type=int, default=None, help="input resolution (fixture default if omitted)")
    g.add_argument("--mode", choices=("sequence", "dimension"), default="sequence")
    g.add_argument("--population", type=int, default=32)
    g.add_argument("--generations", type=int, default=20)
    g.add_argument("--budget", type=float, default=0.02)
    g.add_argument("--trials", type=int, default=8)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--micro", type=int, default=32, help="micro-batch size of the evaluator")
    g.add_argument("--out", type=Path, required=True)
    g.add_argument("--resume", action="store_true")
    g.add_argument("--attackers", type=Path, default=None,
                   help="npz of trained predictors (train-attacker); default: seeded random-init")
    t = sub.add_parser("train-attacker", help="train the bagged LSTM attackers on random architectures")
    t.add_argument("--n", type=int, default=2000, help="random networks in the dataset (4:1 split)")
    t.add_argument("--size", type=int, default=32, help="input resolution (32: CIFAR-like, 224: ImageNet-like)")
    t.add_argument("--epochs", type=int, default=30)
    t.add_argument("--seed", type=int, default=0)
    t.add_argument("--out", type=Path, required=True)
    return ap.parse_args(argv)


def train_attacker_cli(args) -> int:
    from .attacker_train import ArchGenConfig, save_predictors, train_bagged
    from .engine import device
    device()
    classes = 1000 if args.size >= 224 else 10
    cfg = ArchGenConfig(input_shape=(1, 3, args.size, args.size), num_classes=classes, seed=args.seed)
    preds, lers = train_bagged(args.n, cfg, epochs=args.epochs, seed=args.seed)
    save_predictors(args.out, preds)
    print(json.dumps({"out": str(args.out), "hiddens": [p.hidden for p in preds], "val_ler": lers}), flush=True)
    return 0


def _save(out: Path, state, memo: dict) -> None:
    tmp = out / "ckpt.pkl.tmp"
    with open(tmp, "wb") as f:
        pickle.dump({"state": state, "memo": dict(memo)}, f)
    os.replace(tmp, out / "ckpt.pkl")


def run_ga_cli(args) -> int:
    import torch
    import torch.distributed as dist

    from . import dist as tdist
    from . import fixtures, ga
    from .engine import device
    from .evaluate import Evaluator, PopulationEvaluator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device(local)
    kw = {} if args.size is None else {"size": args.size}
    vanilla = fixtures.FIXTURES[args.fixture](**kw)
    params = ga.GaParams(population=args.population, generations=args.generations, seed=args.seed)
    args.out.mkdir(parents=True, exist_ok=True)
    memo: dict = {}
    state = None
    ck = args.out / "ckpt.pkl"
    if args.resume and ck.exists():
        with open(ck, "rb") as f:
            blob = pickle.load(f)
        state, memo = blob["state"], blob["memo"]
        same = dataclasses.replace(state.params, generations=params.generations)
        if (state.mode, same) != (args.mode, params):
            raise SystemExit(f"checkpoint {ck} is for {state.mode} {state.params}, not {args.mode} {params}")
        state.params = params  # --generations may extend the run
    ev = Evaluator()
    if args.attackers is not None:
        from .attacker_train import load_predictors
        ev = Evaluator(predictors=load_predictors(args.attackers))
    pe = PopulationEvaluator(vanilla, ev, budget=args.budget, trials=args.trials, seed=args.seed,
                             memo=memo, exchange=tdist.exchange_signatures if world > 1 else None)

    def evaluate(plans):
        mine = [plans[i] for i in tdist.shard(len(plans), world, rank)]
        rec = pe.evaluate_records(mine, micro=args.micro, memo=memo)
        return tdist.gather_records(rec, len(plans)) if world > 1 else rec

    t0 = time.perf_counter()

    def checkpoint(st):
        if rank == 0:
            _save(args.out, st, memo)
            gen_rows = [r for r in st.log if r[0] == st.gen]
            line = {"generation": st.gen, "best_reward": st.best_reward,
                    "generation_best": max(r[2] for r in gen_rows) if gen_rows else None,
                    "generation_mean": float(np.mean([r[2] for r in gen_rows])) if gen_rows else None,
                    "survivor_rewards": [float(x) for x in st.rewards], "elapsed_s": time.perf_counter() - t0}
            with open(args.out / "log.jsonl", "a") as f:
                f.write(json.dumps(line) + "\n")
            print(json.dumps({k: line[k] for k in ("generation", "best_reward", "generation_mean", "elapsed_s")}),
                  flush=True)

    try:
        if state is None:
            state = ga.ga_init(vanilla, args.mode, params, evaluate)
            checkpoint(state)
        while state.gen < params.generations:
            state = ga.ga_step(vanilla, state, evaluate)
            checkpoint(state)
    finally:
        pe.close()
    res = ga.ga_result(vanilla, state)
    if rank == 0:
        out = {"best_reward": res.best_reward, "best_genome": [int(x) for x in res.best_genome],
               "best_plan": [e.__dict__ for e in res.best_plan.entries], "mode": args.mode,
               "fixture": args.fixture, "generations": params.generations, "population": params.population}
        (args.out / "result.json").write_text(json.dumps(out, indent=1) + "\n")
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None) -> int:
    args = _parse(sys.argv[1:] if argv is None else argv)
    if args.cmd == "ga":
        return run_ga_cli(args)
    if args.cmd == "train-attacker":
        return train_attacker_cli(args)
    return 2


if __name__ == "__main__":
    sys.exit(main())

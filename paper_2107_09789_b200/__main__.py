"""Command line (SURVEY §8(f)4; SPEC.md:609-659 cli_persistence, :572-607 GA loop).

    python -m paper_2107_09789_b200 ga --fixture resnet18 --mode sequence \
        --population 32 --generations 20 --out runs/rn18 [--resume]
    python -m paper_2107_09789_b200 obfuscate --graph net.graph --budget 0.02 --out runs/net
    python -m paper_2107_09789_b200 evaluate --graph net.graph [--plan p.plan] [--attackers a.npz]
    python -m paper_2107_09789_b200 profile --graph net.graph [--plan p.plan] --case C --out t.trace
    python -m paper_2107_09789_b200 train-attacker --n 2000 --out attackers.npz

Graph, plan and trace files are the reference's formats (formats.py). Exit
codes follow SPEC.md:659: 0 success, 1 usage, 2 data/model error.

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


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1, not argparse's 2
        self.print_usage(sys.stderr)
        self.exit(1, f"{self.prog}: error: {message}\n")


class DataError(Exception):
    """Unreadable graph / plan / model file or an inapplicable plan: exit 2."""


def _parse(argv):
    ap = _Parser(prog="python -m paper_2107_09789_b200")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    g = sub.add_parser("ga", help="run the obfuscation GA on a fixture network")
    o = sub.add_parser("obfuscate", help="run the GA on a graph file; write the obfuscated graph and plan")
    g.add_argument("--fixture", choices=("resnet18", "vgg16", "c1c2"), default="resnet18")
    g.add_argument("--size", type=int, default=None, help="input resolution (fixture default if omitted)")
    o.add_argument("--graph", type=Path, required=True)
    for g in (g, o):
        _ga_args(g)
    e = sub.add_parser("evaluate", help="attack a graph (or graph + plan): per-predictor LER, T/T*, reward")
    p = sub.add_parser("profile", help="write the case-masked cost-model trace of a graph (or graph + plan)")
    for x in (e, p):
        x.add_argument("--graph", type=Path, required=True)
        x.add_argument("--plan", type=Path, default=None)
        x.add_argument("--profile", default="default")
    e.add_argument("--attackers", type=Path, default=None)
    e.add_argument("--mode", choices=("sequence", "dimension"), default="sequence",
                   help="mode of the identity plan used when --plan is omitted")
    e.add_argument("--budget", type=float, default=0.02)
    e.add_argument("--trials", type=int, default=8)
    e.add_argument("--seed", type=int, default=0)
    p.add_argument("--case", choices=("A", "B", "C"), default="C")
    p.add_argument("--labels", action="store_true")
    p.add_argument("--out", type=Path, required=True)
    t = sub.add_parser("train-attacker", help="train the bagged LSTM attackers on random architectures")
    t.add_argument("--n", type=int, default=2000, help="random networks in the dataset (4:1 split)")
    t.add_argument("--size", type=int, default=32, help="input resolution (32: CIFAR-like, 224: ImageNet-like)")
    t.add_argument("--epochs", type=int, default=30)
    t.add_argument("--seed", type=int, default=0)
    t.add_argument("--dimension", action="store_true",
                   help="train the dimension attacker (bagged RF (c, j) regressors, 30/50/100/200 trees) instead")
    t.add_argument("--out", type=Path, required=True)
    e.add_argument("--dim-attackers", type=Path, default=None,
                   help="npz of dimension regressors (train-attacker --dimension): dimension plans score DER")
    return ap.parse_args(argv)


def _ga_args(g):
    g.add_argument("--mode", choices=("sequence", "dimension"), default="sequence")
    g.add_argument("--population", type=int, default=32)
    g.add_argument("--generations", type=int, default=20)
    g.add_argument("--budget", type=float, default=0.02)
    g.add_argument("--trials", type=int, default=8)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--micro", type=lambda v: v if v == "auto" else int(v), default="auto",
                   help="micro-batch size of the evaluator (auto: evaluate.auto_micro)")
    g.add_argument("--out", type=Path, required=True)
    g.add_argument("--resume", action="store_true")
    g.add_argument("--attackers", type=Path, default=None,
                   help="npz of trained predictors (train-attacker); default: seeded random-init")
    g.add_argument("--dim-attackers", type=Path, default=None,
                   help="npz of dimension regressors (train-attacker --dimension): dimension mode maximises DER")


def train_attacker_cli(args) -> int:
    from .attacker_train import ArchGenConfig, build_dataset, save_predictors, train_bagged
    from .engine import device
    device()
    classes = 1000 if args.size >= 224 else 10
    cfg = ArchGenConfig(input_shape=(1, 3, args.size, args.size), num_classes=classes, seed=args.seed)
    if args.dimension:
        from .dimattack import save_dim_regressors, train_dim_regressors
        regs, ders = train_dim_regressors(build_dataset(args.n, cfg), seed=args.seed)
        save_dim_regressors(args.out, regs)
        print(json.dumps({"out": str(args.out), "trees": [r.trees for r in regs], "val_der": ders}), flush=True)
        return 0
    preds, lers = train_bagged(args.n, cfg, epochs=args.epochs, seed=args.seed)
    save_predictors(args.out, preds)
    print(json.dumps({"out": str(args.out), "hiddens": [p.hidden for p in preds], "val_ler": lers}), flush=True)
    return 0


def _save(out: Path, state, memo: dict, run: dict) -> None:
    tmp = out / "ckpt.pkl.tmp"
    with open(tmp, "wb") as f:
        pickle.dump({"state": state, "memo": dict(memo), "run": run}, f)
    os.replace(tmp, out / "ckpt.pkl")


def _digest(path: Path | None) -> str | None:
    if path is None:
        return None
    import hashlib
    return hashlib.sha256(Path(path).read_bytes()).hexdigest()


def _run_config(args) -> dict:
    """Everything that fixes the reward scale of a run besides the GA params:
    a resumed run must match it exactly (mixing budgets, trial counts or
    attackers in one search would compare incomparable rewards)."""
    return {"budget": args.budget, "trials": args.trials, "seed": args.seed,
            "source": str(args.graph) if args.cmd == "obfuscate" else args.fixture,
            "source_digest": _digest(args.graph) if args.cmd == "obfuscate" else None,
            "size": getattr(args, "size", None),
            "attackers": _digest(args.attackers), "dim_attackers": _digest(args.dim_attackers)}


def run_ga_cli(args) -> int:
    import torch
    import torch.distributed as dist

    from . import dist as tdist
    from . import fixtures, ga
    from .engine import device
    from .evaluate import PopulationEvaluator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device(local)
    if args.cmd == "obfuscate":
        vanilla = _load_graph(args.graph)
    else:
        kw = {} if args.size is None else {"size": args.size}
        vanilla = fixtures.FIXTURES[args.fixture](**kw)
    params = ga.GaParams(population=args.population, generations=args.generations, seed=args.seed)
    args.out.mkdir(parents=True, exist_ok=True)
    memo: dict = {}
    state = None
    run_cfg = _run_config(args)
    ck = args.out / "ckpt.pkl"
    if args.resume and ck.exists():
        with open(ck, "rb") as f:
            blob = pickle.load(f)
        state, memo = blob["state"], blob["memo"]
        same = dataclasses.replace(state.params, generations=params.generations)
        if (state.mode, same) != (args.mode, params):
            raise SystemExit(f"checkpoint {ck} is for {state.mode} {state.params}, not {args.mode} {params}")
        if blob.get("run") != run_cfg:
            raise SystemExit(f"checkpoint {ck} was written with {blob.get('run')}, not {run_cfg}")
        state.params = params  # --generations may extend the run
    ev = _evaluator(args.attackers, args.dim_attackers)
    pe = PopulationEvaluator(vanilla, ev, budget=args.budget, trials=args.trials, seed=args.seed,
                             memo=memo, exchange=tdist.exchange_signatures if world > 1 else None)

    last_plans: list = []

    def evaluate(plans):
        last_plans[:] = [plans]
        rng = tdist.shard(len(plans), world, rank)
        mine = [plans[i] for i in rng]
        rec = pe.evaluate_records(mine, micro=args.micro, memo=memo, base=rng.start)
        return tdist.gather_records(rec, len(plans)) if world > 1 else rec

    t0 = time.perf_counter()

    def checkpoint(st):
        if rank == 0:
            _save(args.out, st, memo, run_cfg)
            gen_rows = [r for r in st.log if r[0] == st.gen]
            # one row per evaluated candidate: its genome, reward,
            # mean attack metric, latency T and the overhead ratio T/T*
            with open(args.out / "candidates.jsonl", "a") as f:
                for g_, i, r, m, T in gen_rows:
                    plan = last_plans[0][i] if last_plans and i < len(last_plans[0]) else None
                    f.write(json.dumps({"generation": g_, "index": i, "reward": r, "mean_metric": m, "latency": T,
                                        "overhead": T / pe.t_star,
                                        "plan": [dataclasses.asdict(e) for e in plan.entries] if plan else None})
                            + "\n")
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
               "source": str(args.graph) if args.cmd == "obfuscate" else args.fixture,
               "generations": params.generations, "population": params.population}
        if args.cmd == "obfuscate":
            from .formats import dump_graph, dump_plan
            from .knobs import apply_plan
            obf, _ = apply_plan(vanilla, res.best_plan)
            dump_plan(res.best_plan, args.out / "best.plan")
            dump_graph(obf, args.out / "obfuscated.graph")
            rep = pe.evaluate([res.best_plan]).reports[0] if world == 1 else None
            if rep is not None:
                out["report"] = _report_json(rep, args.budget)
                print(json.dumps({"mean_ler": rep.mean_metric, "overhead": out["report"]["overhead"]}), flush=True)
        (args.out / "result.json").write_text(json.dumps(out, indent=1) + "\n")
    if world > 1:
        dist.destroy_process_group()
    return 0


def _load_graph(path: Path):
    from .formats import GraphParseError, load_graph
    try:
        return load_graph(path)
    except (OSError, GraphParseError) as e:
        raise DataError(str(e)) from e


def _load_plan(path: Path | None, graph, mode: str = "sequence"):
    from .formats import load_plan
    from .knobs import identity_plan
    if path is None:
        return identity_plan(graph, mode)
    try:
        return load_plan(path)
    except (OSError, ValueError, TypeError) as e:
        raise DataError(f"{path}: {e}") from e


def _evaluator(attackers: Path | None, dim_attackers: Path | None = None):
    from .evaluate import Evaluator
    ev = Evaluator()
    try:
        if attackers is not None:
            from .attacker_train import load_predictors
            ev.predictors = load_predictors(attackers)
        if dim_attackers is not None:
            from .dimattack import load_dim_regressors
            ev.dim_regressors = load_dim_regressors(dim_attackers)
    except (OSError, KeyError, ValueError) as e:
        raise DataError(f"attacker models: {e}") from e
    return ev


def _report_json(rep, budget: float) -> dict:
    return {"feasible": rep.feasible, "equivalent": rep.equivalent, "worst_rel": rep.worst_rel,
            "latency": rep.latency, "clean_latency": rep.clean_latency,
            "overhead": rep.latency / rep.clean_latency - 1.0 if rep.feasible else None, "budget": budget,
            "lers": rep.metrics, "mean_ler": rep.mean_metric, "reward": rep.reward}


def evaluate_cli(args) -> int:
    """cmd_evaluate: the bagged attacker replayed against one
    graph (the identity plan) or graph + plan."""
    from .engine import device
    from .evaluate import PopulationEvaluator
    g = _load_graph(args.graph)
    plan = _load_plan(args.plan, g, args.mode)
    ev = _evaluator(args.attackers, args.dim_attackers)
    device()
    from .trace import BUILTIN_PROFILES
    ev.profile = BUILTIN_PROFILES[args.profile]
    pe = PopulationEvaluator(g, ev, budget=args.budget, trials=args.trials, seed=args.seed)
    try:
        rep = pe.evaluate([plan]).reports[0]
    finally:
        pe.close()
    if not rep.feasible:
        raise DataError(f"plan does not apply to {args.graph}")
    print(json.dumps(_report_json(rep, args.budget)), flush=True)
    return 0


def profile_cli(args) -> int:
    """cmd_profile: case-masked trace in the reference's
    trace format, from the device cost model."""
    from .engine import device
    from .formats import dump_trace
    from .knobs import TransformError, apply_plan
    from .trace import BUILTIN_PROFILES, LeakageCase, profile_pipeline
    g = _load_graph(args.graph)
    lim = strat = None
    if args.plan is not None:
        try:
            g, d = apply_plan(g, _load_plan(args.plan, g))
        except TransformError as e:
            raise DataError(str(e)) from e
        lim, strat = d.fusion_limits, d.schedule_strategies
    device()
    t = profile_pipeline(g, LeakageCase(args.case), BUILTIN_PROFILES[args.profile], lim, strat)
    dump_trace(t, args.out, include_labels=args.labels)
    print(json.dumps({"out": str(args.out), "kernels": len(t.steps), "total_latency": t.total_latency}), flush=True)
    return 0


def main(argv=None) -> int:
    args = _parse(sys.argv[1:] if argv is None else argv)
    cmds = {"ga": run_ga_cli, "obfuscate": run_ga_cli, "evaluate": evaluate_cli, "profile": profile_cli,
            "train-attacker": train_attacker_cli}
    try:
        return cmds[args.cmd](args)
    except DataError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

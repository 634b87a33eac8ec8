"""Knob search space and the genetic-algorithm obfuscator.

Absent from the reference package; restated from the SPEC and the paper
(PAPER.md:470-501, 555-556). Genomes are per-vanilla-layer option INDICES
into four per-layer domains ("perturb the option index"):

  sequence  mode: branching, fusion_limit, deepen, skip
  dimension mode: widen_factor, kernel_widen, dummy_count, schedule_strategy

Generation step (deterministic given the master seed and the rewards):
mating pool = top half by reward (stable: ties keep population order);
two rounds of uniform pairing without replacement (one permutation each)
with single-point crossover at a random pivot give ``population`` offspring;
each offspring gene gets N(0, sigma) noise, rounded and clipped to its
domain; merged parents+offspring are truncated to the best ``population``;
sigma halves every ``sigma_halving_period`` generations; best-so-far is the
first argmax ever seen. Evaluation never consumes randomness, so sharding
the population over GPUs cannot change the search.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .ir import Graph, OperatorKind as K, shape_map
from .knobs import BRANCH_MODES, WIDEN_FACTORS, ObfuscationPlan, PlanEntry, _Work, widenable

SEQ_GENES = ("branching", "fusion_limit", "deepen", "skip")
DIM_GENES = ("widen_factor", "kernel_widen", "dummy_count", "schedule_strategy")
FUSION_LIMITS = (-1, 0, 1, 2)
KERNEL_WIDEN = (0, 1, 2)
DUMMY_COUNTS = (0, 1, 2, 3, 4)
STRATEGIES = (0, 1, 2, 3)


def search_space(graph: Graph, mode: str) -> list[dict[str, tuple]]:
    """Per-vanilla-layer knob domains with infeasible options pruned."""
    shapes = shape_map(graph)
    w = _Work(graph)
    out = []
    for lid in graph.complex_layers():
        n = graph.nodes[lid]
        layer = n.kind in (K.Conv2D, K.Linear)
        if mode == "sequence":
            br = ["none"]
            if layer:
                j = n.attrs["j"]
                if n.kind is K.Conv2D:
                    cin = n.attrs["c"]
                else:
                    cin = shapes[n.inputs[0]].channels if n.inputs else graph.input_shape.channels
                for m in BRANCH_MODES[1:]:
                    parts = int(m[-1])
                    if (cin if m.startswith("in") else j) % parts == 0:
                        br.append(m)
            deep = (0, 1) if w.activation_site(lid) is not None else (0,)
            out.append({"branching": tuple(br), "fusion_limit": FUSION_LIMITS, "deepen": deep, "skip": (0, 1)})
        elif mode == "dimension":
            wf = WIDEN_FACTORS if (layer and widenable(graph, lid)) else (1.0,)
            kw = KERNEL_WIDEN if n.kind is K.Conv2D else (0,)
            out.append({"widen_factor": wf, "kernel_widen": kw, "dummy_count": DUMMY_COUNTS,
                        "schedule_strategy": STRATEGIES})
        else:
            raise ValueError(f"unknown mode {mode!r}")
    return out


def genes_of(mode: str) -> tuple[str, ...]:
    return SEQ_GENES if mode == "sequence" else DIM_GENES


def decode_genome(graph: Graph, mode: str, space: list[dict], genome: np.ndarray) -> ObfuscationPlan:
    names = genes_of(mode)
    entries = []
    for lid, dom, row in zip(graph.complex_layers(), space, genome.reshape(len(space), len(names))):
        kw = {name: dom[name][int(row[g])] for g, name in enumerate(names)}
        entries.append(PlanEntry(lid, **kw))
    return ObfuscationPlan(mode, tuple(entries))


def domain_sizes(mode: str, space: list[dict]) -> np.ndarray:
    return np.array([[len(dom[g]) for g in genes_of(mode)] for dom in space], dtype=np.int64).reshape(-1)


def random_genomes(rng: np.random.Generator, sizes: np.ndarray, count: int) -> np.ndarray:
    return np.stack([rng.integers(0, sizes) for _ in range(count)]).astype(np.int64)


@dataclass
class GaParams:
    """SPEC.md:542-546 (defaults)."""

    population: int = 16
    generations: int = 20
    sigma0: float = 8.0
    sigma_halving_period: int = 4
    elite_fraction: float = 0.5
    epsilon: float = 0.05
    seed: int = 0

    def __post_init__(self):
        if self.population % 2 or self.population < 2 or not (0 < self.elite_fraction <= 1):
            raise ValueError("population must be even and >= 2; 0 < elite_fraction <= 1")


def _order(rewards: np.ndarray) -> np.ndarray:
    """Descending reward, stable (ties keep list order)."""
    return np.argsort(-rewards, kind="stable")


def next_generation(rng: np.random.Generator, genomes: np.ndarray, rewards: np.ndarray, sizes: np.ndarray,
                    sigma: float, params: GaParams) -> np.ndarray:
    """Offspring of one generation (before evaluation)."""
    P, L = genomes.shape
    pool = genomes[_order(rewards)[:max(2, int(round(P * params.elite_fraction)))]]
    kids = []
    while len(kids) < P:
        perm = rng.permutation(len(pool))
        for a, b in zip(perm[0::2], perm[1::2]):
            pivot = int(rng.integers(1, L)) if L > 1 else 0
            kids.append(np.concatenate([pool[a][:pivot], pool[b][pivot:]]))
            kids.append(np.concatenate([pool[b][:pivot], pool[a][pivot:]]))
            if len(kids) >= P:
                break
    kids = np.stack(kids[:P]).astype(np.float64)
    kids += rng.normal(0.0, sigma, kids.shape)
    return np.clip(np.rint(kids), 0, sizes - 1).astype(np.int64)


@dataclass
class GaResult:
    best_genome: np.ndarray
    best_plan: ObfuscationPlan
    best_reward: float
    log: list = field(default_factory=list)   # (generation, index, reward, mean_ler, T) — raw latency T


@dataclass
class GaState:
    """Everything the search needs to continue after generation ``gen``: the
    surviving population and its rewards, the best-so-far, the log and the
    RNG state (a checkpoint is this object; resuming is bit-identical to an
    uninterrupted run, SPEC.md:600 generation log)."""

    mode: str
    params: GaParams
    gen: int
    pop: np.ndarray
    rewards: np.ndarray
    best_reward: float
    best_genome: np.ndarray
    rng_state: dict
    log: list = field(default_factory=list)   # (generation, index, reward, mean_ler, T)


def ga_init(graph: Graph, mode: str, params: GaParams, evaluate_fn) -> GaState:
    """Generation 0: random genomes from the master seed, evaluated."""
    rng = np.random.default_rng(params.seed)
    space = search_space(graph, mode)
    sizes = domain_sizes(mode, space)
    pop = random_genomes(rng, sizes, params.population)
    rec = evaluate_fn([decode_genome(graph, mode, space, g) for g in pop])
    rewards = rec["reward"].astype(np.float64)
    log = [(0, i, float(r["reward"]), float(r["mean_ler"]), float(r["latency"])) for i, r in enumerate(rec)]
    bi = int(_order(rewards)[0])
    return GaState(mode, params, 0, pop, rewards, float(rewards[bi]), pop[bi].copy(), rng.bit_generator.state, log)


def ga_step(graph: Graph, state: GaState, evaluate_fn) -> GaState:
    """One generation: offspring, evaluation, elitist truncation."""
    params, mode = state.params, state.mode
    rng = np.random.default_rng()
    rng.bit_generator.state = state.rng_state
    space = search_space(graph, mode)
    sizes = domain_sizes(mode, space)
    gen = state.gen + 1
    sigma = params.sigma0 / (2 ** ((gen - 1) // params.sigma_halving_period))
    kids = next_generation(rng, state.pop, state.rewards, sizes, sigma, params)
    krec = evaluate_fn([decode_genome(graph, mode, space, g) for g in kids])
    krew = krec["reward"].astype(np.float64)
    log = state.log + [(gen, i, float(r["reward"]), float(r["mean_ler"]), float(r["latency"]))
                       for i, r in enumerate(krec)]
    best_r, best_g = state.best_reward, state.best_genome
    ki = int(_order(krew)[0])
    if krew[ki] > best_r:
        best_r, best_g = float(krew[ki]), kids[ki].copy()
    merged = np.concatenate([state.pop, kids])
    mrew = np.concatenate([state.rewards, krew])
    keep = _order(mrew)[:params.population]
    return GaState(mode, params, gen, merged[keep], mrew[keep], best_r, best_g, rng.bit_generator.state, log)


def ga_result(graph: Graph, state: GaState) -> GaResult:
    space = search_space(graph, state.mode)
    return GaResult(state.best_genome, decode_genome(graph, state.mode, space, state.best_genome),
                    state.best_reward, state.log)


def run_ga(graph: Graph, mode: str, budget: float, params: GaParams, evaluate_fn, on_generation=None) -> GaResult:
    """SPEC.md:572-580. ``evaluate_fn(plans) -> records`` (RECORD_DTYPE) — the
    GPU population evaluator, possibly sharded across ranks. ``on_generation``
    (GaState) is called after every generation (checkpointing, logging)."""
    state = ga_init(graph, mode, params, evaluate_fn)
    if on_generation is not None:
        on_generation(state)
    while state.gen < params.generations:
        state = ga_step(graph, state, evaluate_fn)
        if on_generation is not None:
            on_generation(state)
    return ga_result(graph, state)

"""Attacker training data and LSTM training.

The reference package has no attacker; names and contracts
follow SPEC.md:417-470 (``generate_random_arch``, ``build_dataset``) and the
paper's attacker (a single-layer LSTM over the
per-kernel trace rows trained with CTC against the layer label sequence,
4:1 train/validation split).

* ``generate_random_arch`` — random networks in the reference IR: a random
  number of plain conv (+BN) + ReLU blocks, residual blocks and max-pools
  with random widths / kernel sizes / strides, then Linear layers with random
  neuron counts and the classification Linear + SoftMax (§V-A
  ordering). Deterministic per seed; every graph passes ``validate``.
* ``build_dataset`` — traces of n such networks from the device trace
  pipeline (``trace.trace_population``: generic fusion, default schedules,
  9 fp64 features per kernel) with their label sequences L*.
* ``train_predictor`` — torch ``nn.LSTM`` + linear head on the GPU over
  log1p-normalised features (the normalisation the decode kernel applies),
  trained FRAMEWISE: each trace step's target is its kernel anchor's label
  (complex kinds) or blank. The paper trains with CTC on
  profiler traces with several launches per layer; here a trace has one step
  per fused kernel, so a CTC alignment of consecutive same-kind layers (e.g.
  19 Conv2D in a row in ResNet-18, which need blanks between repeats) is
  infeasible — the step labels are known exactly instead. The greedy CTC
  decode then collapses such repeats, which bounds the attainable LER.
  The predictor is exported with weights rounded to bf16-representable fp32
  (the cluster decode kernel stores them as bf16), so the trained attacker
  runs through ``tobf_lstm_ctc`` bit-exactly against the CPU oracle.

Training is off the hot path (library autograd is fine here); the product
path is the inference kernels.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .attacker import NUM_CLASSES, Predictor, _bf16_round, encode_labels
from .fixtures import _Builder
from .ir import Graph, OperatorKind as K, TensorShape, label_sequence, shape_map, validate


@dataclass
class ArchGenConfig:
    """SPEC.md:422-426 (depthwise blocks omitted: the IR has no grouped conv)."""

    input_shape: tuple = (1, 3, 32, 32)
    num_classes: int = 10
    depth_range: tuple = (3, 10)          # complex feature layers (conv / pool / residual)
    block_mix: dict = field(default_factory=lambda: {"conv": 0.45, "residual": 0.25, "pool": 0.2, "bn": 0.1})
    max_linear: int = 2                   # hidden Linear layers before the classifier
    seed: int = 0

    def __post_init__(self):
        if abs(sum(self.block_mix.values()) - 1.0) > 1e-9 or self.depth_range[0] < 3:
            raise ValueError("block_mix must sum to 1 and depth >= 3")


WIDTHS = (16, 24, 32, 48, 64, 96, 128, 192, 256)


def generate_random_arch(config: ArchGenConfig, index: int = 0) -> Graph:
    """One random network; ``index`` selects it within the config's seed stream."""
    rng = np.random.default_rng([config.seed, index])
    b = _Builder(TensorShape(*config.input_shape), int(rng.integers(1 << 31)))
    kinds = list(config.block_mix)
    probs = np.array([config.block_mix[k] for k in kinds])
    cur, c, h = None, config.input_shape[1], config.input_shape[2]
    src = lambda: [] if cur is None else [cur]  # noqa: E731
    depth = int(rng.integers(config.depth_range[0], config.depth_range[1] + 1))
    for _ in range(depth):
        kind = kinds[int(rng.choice(len(kinds), p=probs))]
        if kind == "pool" and h >= 4 and cur is not None:
            cur = b.pool(cur, 2, 2)
            h //= 2
            continue
        if kind == "residual" and cur is not None and h >= 2:
            y = b.conv([cur], c, c, 3, 1, 1)
            y = b.relu(b.bn(y, c))
            y = b.bn(b.conv([y], c, c, 3, 1, 1), c)
            cur = b.relu(b.add([cur, y]))
            continue
        # plain conv (also the fallback for pool / residual where they do not fit)
        k = int(rng.choice([1, 3, 5]))
        stride = 2 if (h >= 8 and rng.random() < 0.25) else 1
        j = int(rng.choice(WIDTHS))
        y = b.conv(src(), c, j, k, stride, k // 2)
        h = (h + 2 * (k // 2) - k) // stride + 1
        if kind == "bn" or rng.random() < 0.5:
            y = b.bn(y, j)
        cur = b.relu(y)
        c = j
    feat = c * h * h
    for _ in range(int(rng.integers(0, config.max_linear + 1))):
        n = int(rng.choice([64, 128, 256, 512]))
        cur = b.relu(b.linear(cur, feat, n))
        feat = n
    cur = b.linear(cur, feat, config.num_classes)
    g = b.graph(b.softmax(cur))
    return g


@dataclass
class TraceDataset:
    """feature rows (fp64, 9 per kernel step) of every
    network, row offsets, and each network's label sequence (int8 codes)."""

    feats: np.ndarray       # (rows, 9) float64
    offsets: np.ndarray     # (n+1,) int32
    labels: list            # n arrays of int8 label codes (L*)
    graphs: list
    step_labels: np.ndarray | None = None  # (rows,) int8: each kernel anchor's code, 0 = not complex
    step_cj: np.ndarray | None = None      # (rows, 2) int32: a Conv2D anchor's (c, j), else 0 (dimension attacker)


def build_dataset(n: int, config: ArchGenConfig, profile=None, start: int = 0) -> TraceDataset:
    """n random networks, compiled with generic fusion and
    default schedules and profiled (on the device) with their labels."""
    from .trace import BUILTIN_PROFILES, trace_population
    profile = profile or BUILTIN_PROFILES["default"]
    graphs = [generate_random_arch(config, start + i) for i in range(n)]
    pt = trace_population([(g, None, None) for g in graphs], profile, memo={})
    feats = pt.feats.cpu().numpy()[: int(pt.offsets_host[-1])]
    labels = [encode_labels(label_sequence(g)) for g in graphs]
    from .attacker import LABEL_CODES
    anchors = [g.nodes[k.anchor] for g, cg in zip(graphs, pt.compiled) for k in cg.kernels]
    steps = np.array([LABEL_CODES.get(a.kind, 0) for a in anchors], dtype=np.int8)
    cj = np.array([(a.attrs["c"], a.attrs["j"]) if a.kind is K.Conv2D else (0, 0) for a in anchors],
                  dtype=np.int32).reshape(-1, 2)
    return TraceDataset(feats, pt.offsets_host.astype(np.int32), labels, graphs, steps, cj)


@dataclass
class TrainParams:
    hidden: int = 128
    features: int = 9
    epochs: int = 30
    batch: int = 64
    lr: float = 3e-3
    seed: int = 0
    val_fraction: float = 0.2   # PAPER.md §V-A "split each dataset into 4:1"


def _padded(ds: TraceDataset, idx: np.ndarray, features: int, dev):
    lens = np.diff(ds.offsets)[idx]
    T = int(lens.max())
    x = np.zeros((len(idx), T, features), np.float32)
    for r, i in enumerate(idx):
        lo, hi = ds.offsets[i], ds.offsets[i + 1]
        x[r, : hi - lo] = np.log1p(ds.feats[lo:hi, :features]).astype(np.float32)
    y = np.full((len(idx), T), -100, np.int64)  # ignore_index beyond each trace
    for r, i in enumerate(idx):
        lo, hi = ds.offsets[i], ds.offsets[i + 1]
        y[r, : hi - lo] = ds.step_labels[lo:hi]
    return torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)


def train_predictor(ds: TraceDataset, params: TrainParams, device=None) -> tuple[Predictor, dict]:
    """Framewise training of one single-layer LSTM sequence predictor
    (see the module note on CTC); returns the exported
    Predictor and the loss history."""
    dev = device or torch.device("cuda", torch.cuda.current_device())
    gen = torch.Generator(device="cpu").manual_seed(params.seed)
    n = len(ds.labels)
    perm = torch.randperm(n, generator=gen).numpy()
    nval = max(1, int(round(n * params.val_fraction)))
    val_idx, tr_idx = perm[:nval], perm[nval:]
    torch.manual_seed(params.seed)
    lstm = torch.nn.LSTM(params.features, params.hidden, batch_first=True).to(dev)
    head = torch.nn.Linear(params.hidden, NUM_CLASSES).to(dev)
    opt = torch.optim.Adam(list(lstm.parameters()) + list(head.parameters()), lr=params.lr)
    ce = torch.nn.CrossEntropyLoss(ignore_index=-100)
    hist = {"train": [], "val": []}

    def loss_of(idx):
        x, y = _padded(ds, idx, params.features, dev)
        out, _ = lstm(x)
        return ce(head(out).reshape(-1, NUM_CLASSES), y.reshape(-1))

    for _ in range(params.epochs):
        order = tr_idx[torch.randperm(len(tr_idx), generator=gen).numpy()]
        tot = 0.0
        for s in range(0, len(order), params.batch):
            loss = loss_of(order[s: s + params.batch])
            opt.zero_grad()
            loss.backward()
            opt.step()
            tot += loss.item() * len(order[s: s + params.batch])
        hist["train"].append(tot / max(1, len(order)))
        with torch.no_grad():
            hist["val"].append(float(loss_of(val_idx)))
    # export: torch gate order (i, f, g, o) is the kernel's; bias = b_ih + b_hh
    w_ih = lstm.weight_ih_l0.detach().float().cpu().numpy()   # (4H, F)
    w_hh = lstm.weight_hh_l0.detach().float().cpu().numpy()   # (4H, H)
    bias = (lstm.bias_ih_l0 + lstm.bias_hh_l0).detach().float().cpu().numpy()
    pred = Predictor(params.hidden, params.features, _bf16_round(w_ih.T.copy()), _bf16_round(w_hh.T.copy()),
                     _bf16_round(bias), _bf16_round(head.weight.detach().float().cpu().numpy()),
                     _bf16_round(head.bias.detach().float().cpu().numpy()))
    hist["val_idx"] = val_idx
    return pred, hist


def dataset_ler(ds: TraceDataset, pred: Predictor, idx: np.ndarray | None = None) -> float:
    """Mean LER of ``pred`` (through the device decode + Levenshtein kernels)
    over the dataset's networks ``idx`` against their own label sequences."""
    from .attacker import decode, edit_distances
    from .engine import device
    ctx = device()
    idx = np.arange(len(ds.labels)) if idx is None else np.asarray(idx)
    lers = []
    for i in idx:
        lo, hi = int(ds.offsets[i]), int(ds.offsets[i + 1])
        f = torch.from_numpy(np.ascontiguousarray(ds.feats[lo:hi])).to(ctx.device)
        offs = torch.tensor([0, hi - lo], dtype=torch.int32, device=ctx.device)
        toks, ntok = decode(f, offs, 1, hi - lo, pred)
        _, lr, _ = edit_distances(toks, ntok, ds.labels[i])
        lers.append(float(lr.cpu()[0]))
    return float(np.mean(lers))


def save_predictors(path, preds: list[Predictor]) -> None:
    """npz with each predictor's five weight arrays (p{i}_w_ihT ...)."""
    arrs = {f"p{i}_{k}": v for i, p in enumerate(preds) for k, v in p.weights().items()}
    arrs.update({f"p{i}_meta": np.array([p.hidden, p.features]) for i, p in enumerate(preds)})
    np.savez(path, **arrs)


def load_predictors(path) -> list[Predictor]:
    z = np.load(path)
    out, i = [], 0
    while f"p{i}_meta" in z:
        h, f = (int(x) for x in z[f"p{i}_meta"])
        out.append(Predictor(h, f, z[f"p{i}_w_ihT"], z[f"p{i}_w_hhT"], z[f"p{i}_b"], z[f"p{i}_w_out"],
                             z[f"p{i}_b_out"]))
        i += 1
    return out


def train_bagged(n: int = 2000, config: ArchGenConfig | None = None, hiddens=(128, 256, 512), epochs: int = 30,
                 seed: int = 0) -> tuple[list[Predictor], list[float]]:
    """The three case-C predictors of PAPER.md:623 trained on one dataset
    (each with its own seed / split); returns them with their validation LER."""
    ds = build_dataset(n, config or ArchGenConfig(seed=seed))
    preds, lers = [], []
    for i, h in enumerate(hiddens):
        p, hist = train_predictor(ds, TrainParams(hidden=h, epochs=epochs, seed=seed + i))
        preds.append(p)
        lers.append(dataset_ler(ds, p, hist["val_idx"]))
    return preds, lers


__all__ = ["ArchGenConfig", "generate_random_arch", "TraceDataset", "build_dataset", "TrainParams",
           "train_predictor", "dataset_ler", "save_predictors", "load_predictors", "train_bagged"]


def _self_check(g: Graph) -> None:  # used by tests
    assert not validate(g), validate(g)
    shape_map(g)

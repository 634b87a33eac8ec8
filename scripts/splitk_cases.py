"""Development aid: single-conv graphs, split-K on vs off vs the fp64 oracle."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import interp_ref as IR  # noqa: E402
from paper_2107_09789_b200 import executor  # noqa: E402
from paper_2107_09789_b200.ir import Graph, Node, OperatorKind, TensorShape  # noqa: E402

CASES = [  # b, c, h, j, k, s, p
    (1, 256, 8, 544, 5, 2, 2), (1, 256, 8, 512, 5, 2, 2), (1, 256, 8, 544, 5, 1, 2), (1, 256, 8, 544, 3, 2, 1),
    (1, 256, 8, 128, 5, 2, 2), (1, 256, 8, 64, 5, 2, 2), (8, 512, 7, 512, 3, 1, 1), (1, 512, 7, 512, 3, 1, 1),
    (1, 256, 4, 256, 5, 1, 2), (2, 256, 8, 256, 5, 2, 2),
]
for b, c, h, j, k, s, p in CASES:
    rng = np.random.default_rng(1)
    x = rng.standard_normal((b, c, h, h)).astype(np.float32)
    w = (rng.standard_normal((k, k, c, j)) * np.sqrt(2.0 / (k * k * c))).astype(np.float32)
    g = Graph({0: Node(0, OperatorKind.Conv2D, {"k1": k, "k2": k, "c": c, "j": j, "stride": s, "padding": p}, w, [])},
              0, TensorShape(b, c, h, h))
    ref = IR.conv2d(x, w, s, p).astype(np.float64)
    out = {}
    for sp in (1, 16):
        executor.SPLITK_MAX = sp
        out[sp] = executor.execute(g, x)
    e1 = np.abs(out[1] - ref).max() / (np.abs(ref).max())
    e16 = np.abs(out[16] - ref).max() / (np.abs(ref).max())
    bad = np.argwhere(np.abs(out[16] - ref) > 1e-3 * np.abs(ref).max())
    print((b, c, h, j, k, s, p), f"nosplit {e1:.2e} split {e16:.2e}", "bad idx sample", bad[:4].tolist(),
          "nbad", len(bad), flush=True)

"""cfg5 probe: one 10k-trace LSTM + CTC decode per predictor (the launch the
bench's kernels.cfg5_fitness times), for ncu capture of the real cfg5 grid."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_09789_b200 import attacker  # noqa: E402
from paper_2107_09789_b200.engine import device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--hidden", type=int, nargs="+", default=[128, 256, 512])
ap.add_argument("--traces", type=int, default=10_000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
ctx = device()
dev = ctx.device
gen = torch.Generator(device=dev)
gen.manual_seed(0)
tl = torch.randint(119, 170, (a.traces,), generator=gen, device=dev, dtype=torch.int32)
offs = torch.zeros(a.traces + 1, dtype=torch.int32, device=dev)
offs[1:] = torch.cumsum(tl, 0)
rows = int(offs[-1].item())
feats = torch.rand((rows, 9), generator=gen, device=dev, dtype=torch.float64) * 1e6
for h in a.hidden:
    p = attacker.init_predictor(h, 9, seed=h)
    attacker.decode(feats, offs, a.traces, 169, p)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        attacker.decode(feats, offs, a.traces, 169, p)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    fl = rows * 2 * 4 * h * (9 + h)
    print(f"H={h} traces={a.traces} rows={rows} ms={ms:.3f} TFLOP/s={fl / ms / 1e9:.2f}", flush=True)

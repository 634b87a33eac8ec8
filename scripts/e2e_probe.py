"""e2e (public API, host buffers) candidates/s vs micro-batch size, with the
parent's host-time split. usage: python scripts/e2e_probe.py [pop] [steps]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import population_plans  # noqa: E402
from paper_2107_09789_b200 import fixtures  # noqa: E402
from paper_2107_09789_b200.engine import device  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ctx = device(0)
g = fixtures.resnet18()
pe = PopulationEvaluator(g, Evaluator(), budget=0.02, trials=8, seed=0, memo={})
plans = population_plans(g, P * 40, 1)
k = 0
for micro in (32, 16, (8, 24)):
    for s in range(2):
        ctx.clear_cache()
        pe.evaluate_records(plans[k:k + P], micro=micro, memo={})
        k += P
    torch.cuda.synchronize()
    acc = {}
    t0 = time.perf_counter()
    for s in range(steps):
        ctx.clear_cache()
        pe.evaluate_records(plans[k:k + P], micro=micro, memo={})
        k += P
        for kk, v in pe.last_host_ms.items():
            acc[kk] = acc.get(kk, 0) + v / steps
    dt = (time.perf_counter() - t0) / steps
    print(f"micro {str(micro):12s}: {1e3 * dt:7.2f} ms/step  {P / dt:8.1f} cand/s  host " +
          " ".join(f"{kk}={v:.2f}" for kk, v in acc.items()), flush=True)
pe.close()

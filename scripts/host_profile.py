"""Development aid: cProfile of the end-to-end host path (evaluate_records on
cold caches, as bench.py's e2e leg runs it)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2107_09789_b200 import fixtures  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402


def main():
    g = fixtures.resnet18()
    pe = PopulationEvaluator(g, Evaluator(), budget=0.02, trials=8, seed=0, memo={})
    plans = bench.population_plans(g, 32 * 6, 1)
    steps = [plans[i * 32:(i + 1) * 32] for i in range(6)]
    for s in steps[:2]:
        pe.ctx.clear_cache()
        pe.evaluate_records(s, memo={})
    torch.cuda.synchronize()
    t = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    for s in steps[2:]:
        pe.ctx.clear_cache()
        pe.evaluate_records(s, memo={})
    pr.disable()
    torch.cuda.synchronize()
    print(f"{(time.perf_counter() - t) / 4 * 1e3:.1f} ms/step under cProfile; host split {pe.last_host_ms}")
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(40)
    st.sort_stats("cumtime").print_stats(50)


if __name__ == "__main__":
    main()

"""Development aid: cProfile of the cfg4 (VGG-16 dimension) end-to-end host
path, as bench.py's cfg4 e2e leg runs it (cold caches, 16 candidates/step)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_09789_b200 import fixtures, ga  # noqa: E402
from paper_2107_09789_b200.engine import device  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402

ctx = device()
P = 16
g = fixtures.vgg16()
space = ga.search_space(g, "dimension")
rng = np.random.default_rng(0)
plans = [ga.decode_genome(g, "dimension", space, x)
         for x in ga.random_genomes(rng, ga.domain_sizes("dimension", space), P * 6)]
pe = PopulationEvaluator(g, Evaluator(), budget=0.02, trials=8, seed=0, memo={})
for s in range(2):
    ctx.clear_cache()
    pe.evaluate_records(plans[P * s:P * (s + 1)], memo={})
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
for s in range(2, 6):
    ctx.clear_cache()
    pe.evaluate_records(plans[P * s:P * (s + 1)], memo={})
pr.disable()
torch.cuda.synchronize()
print(f"{(time.perf_counter() - t) / 4 * 1e3:.1f} ms/step under cProfile; {pe.last_host_ms}")
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
pe.close()

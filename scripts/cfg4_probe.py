"""cfg4: VGG-16 224x224, dimension-mode candidates (widen +
kernel widen + dummy), 8 equivalence trials. Device-resident candidates/s and
end-to-end (public API, host buffers, cold caches) candidates/s."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2107_09789_b200 import fixtures, ga  # noqa: E402
from paper_2107_09789_b200.engine import device  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = device(0)
g = fixtures.vgg16()
space = ga.search_space(g, "dimension")
sizes = ga.domain_sizes("dimension", space)
rng = np.random.default_rng(0)
plans = [ga.decode_genome(g, "dimension", space, x) for x in ga.random_genomes(rng, sizes, P * (steps + 2))]
pe = PopulationEvaluator(g, Evaluator(), budget=0.02, trials=8, seed=0, memo={})
t0 = time.perf_counter()
prep = pe.prepare(plans[:P], memo={})
t1 = time.perf_counter()
x = pe.x_host.to(ctx.device)
for _ in range(2):
    pe.run(prep, x_dev=x, cold_schedules=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    pe.run(prep, x_dev=x, cold_schedules=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
run = prep["run"]
print(f"cfg4 device: {P} candidates, {ms:.1f} ms/step -> {P / ms * 1e3:.1f} cand/s; "
      f"{run.gemm_flops() / ms / 1e9:.1f} TF/s conv-alg; prepare (in-process, lazy knobs) {1e3 * (t1 - t0):.0f} ms",
      flush=True)
for s in range(2):
    ctx.clear_cache()
    pe.evaluate_records(plans[P * (1 + s):P * (2 + s)], memo={})
torch.cuda.synchronize()
t0 = time.perf_counter()
for s in range(steps):
    ctx.clear_cache()
    pe.evaluate_records(plans[P * (1 + s):P * (2 + s)], memo={})
dt = (time.perf_counter() - t0) / steps
print(f"cfg4 e2e: {1e3 * dt:.0f} ms/step -> {P / dt:.1f} cand/s; host split {pe.last_host_ms}", flush=True)
pe.close()

"""Development aid: where the parent blocks in the streamed e2e path. Wraps
host-side calls of one process with wall-clock accumulators and runs the
bench's e2e stream (cold caches, 2 steps in flight). usage:
python scripts/e2e_stall_probe.py [steps]"""
import functools
import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import population_plans  # noqa: E402
from paper_2107_09789_b200 import attacker, engine, evaluate, executor, fixtures, trace  # noqa: E402
from paper_2107_09789_b200.engine import device  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402

ACC = defaultdict(float)
CNT = defaultdict(int)


def wrap(obj, name, label=None):
    f = getattr(obj, name)
    label = label or f"{getattr(obj, '__name__', type(obj).__name__)}.{name}"

    @functools.wraps(f)
    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            ACC[label] += time.perf_counter() - t
            CNT[label] += 1
    setattr(obj, name, g)


for cls, names in ((PopulationEvaluator, ("run_attack", "run_forward", "readback", "link_forward", "collect",
                                           "prepare_encoded", "receive", "complete", "launch")),
                   (executor.PlanTables, ("add", "_wimg_ptr", "_xcol_wimg_ptr", "_derived_wimg_ptr", "_affine_ptrs",
                                          "_const_ptr", "_xcol_buffer")),
                   (executor.PopulationRun, ("set_input", "run", "_link_all")),
                   (engine.DeviceContext, ("_staged", "cached_view", "_pinned_copy", "clear_cache", "upload_bytes",
                                           "side_streams"))):
    for n in names:
        if hasattr(cls, n):
            wrap(cls, n, f"{cls.__name__}.{n}")
for mod, names in ((evaluate, ("decode", "edit_distances", "reward", "compare_outputs", "run_trace", "readback_trace",
                               "finish_trace")),):
    for n in names:
        if hasattr(mod, n):
            wrap(mod, n, f"evaluate.{n}")

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ctx = device(0)
g = fixtures.resnet18()
pe = PopulationEvaluator(g, Evaluator(), budget=0.02, trials=8, seed=0, memo={})
P = 32
plans = population_plans(g, P * (steps + 4), 1)


def shards(lo, hi):
    for s in range(lo, hi):
        ctx.clear_cache()
        yield plans[s * P:(s + 1) * P]


for _ in pe.evaluate_stream(shards(0, 3), depth=2, cold=True):
    pass
torch.cuda.synchronize()
ACC.clear()
CNT.clear()
f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
f0.record()
for _ in pe.evaluate_stream(shards(3, 3 + steps), depth=2, cold=True):
    pass
f1.record()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"e2e {steps} steps: {1e3 * wall / steps:.2f} ms/step wall, {f0.elapsed_time(f1) / steps:.2f} device-event")
for k, v in sorted(ACC.items(), key=lambda x: -x[1]):
    print(f"  {k:40s} {1e3 * v / steps:8.2f} ms/step  calls/step {CNT[k] / steps:6.1f}")

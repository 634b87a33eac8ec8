"""Per-candidate host encode time (the hostpipe worker job) on this machine,
single process: apply_plan / lower+plan_forward / trace_records split."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os  # noqa: E402

from bench import population_plans  # noqa: E402
from paper_2107_09789_b200 import fixtures, hostpipe  # noqa: E402
from paper_2107_09789_b200.executor import lower, plan_forward  # noqa: E402
from paper_2107_09789_b200.knobs import apply_plan_analyzed  # noqa: E402
from paper_2107_09789_b200.trace import trace_records  # noqa: E402

g = fixtures.resnet18()
plans = population_plans(g, 64, 1)
hostpipe._worker_init(g, 8, "default")
W = hostpipe._W
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
acc = [0.0, 0.0, 0.0]
for rep in range(2):
    acc = [0.0, 0.0, 0.0]
    for i, p in enumerate(plans):
        t0 = time.perf_counter()
        try:
            og, d, ana = apply_plan_analyzed(g, p, W["analysis"])
        except Exception:
            continue
        t1 = time.perf_counter()
        refs = hostpipe.WorkerRefs(W["roots"], i)
        plan_forward(lower(og, ana), 8, refs)
        t2 = time.perf_counter()
        trace_records(og, d.fusion_limits, d.schedule_strategies, "default", ana)
        t3 = time.perf_counter()
        acc[0] += t1 - t0
        acc[1] += t2 - t1
        acc[2] += t3 - t2
n = len(plans)
print(f"ms/cand apply {1e3 * acc[0] / n:.2f} lower+plan {1e3 * acc[1] / n:.2f} trace {1e3 * acc[2] / n:.2f} "
      f"total {1e3 * sum(acc) / n:.2f}")

"""Development aid: repeat the headline population through the resident path
and the e2e path (host workers, micro-batches) and flag any candidate whose
`worst` is not fp32-noise (> 1e-3: a wrong forward). usage:
python scripts/stress_records.py [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from bench import population_plans  # noqa: E402
from paper_2107_09789_b200 import fixtures  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
g = fixtures.resnet18()
plans = population_plans(g, 32, 0)
pe = PopulationEvaluator(g, Evaluator(), budget=0.02, trials=8, seed=0, memo={})
bad = 0
try:
    for r in range(reps):
        runs = []
        if r % 4 == 0:
            prep = pe.prepare(plans, memo={})
            runs.append(("resident", pe.collect(pe.run(prep, cold_schedules=True))))
        runs.append(("e2e", pe.evaluate_records(plans, memo={})))
        for name, rr in runs:
            w = rr["worst"][rr["feasible"] != 0]
            idx = np.nonzero(rr["worst"] > 1e-3)[0]
            if len(idx):
                bad += 1
                print(f"rep {r} {name}: WRONG worst at {idx.tolist()}: {rr['worst'][idx].tolist()}", flush=True)
            else:
                print(f"rep {r} {name}: max worst {float(w.max()):.3e}", flush=True)
finally:
    pe.close()
print("BAD" if bad else "OK", bad)

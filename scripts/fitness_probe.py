"""Development aid: per-launch time of the fitness stage (LSTM+CTC per
predictor, Levenshtein, Eq. 10) for a 32-candidate RN18 sequence batch."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2107_09789_b200 import fixtures  # noqa: E402
from paper_2107_09789_b200.attacker import decode, edit_distances  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402


def main():
    g = fixtures.resnet18()
    pe = PopulationEvaluator(g, Evaluator(), trials=8, memo={})
    plans = bench.population_plans(g, 32, 1)
    prep = pe.prepare(plans, memo={})
    pe.run(prep)
    torch.cuda.synchronize()
    tp = prep["trace"]
    t_max = prep["t_max"]
    ncf = len(prep["feas"])
    print("traces", ncf, "t_max", t_max, "kernels", tp.nk)
    truth = pe.ctx.upload_array(pe.truth)
    for rep in range(2):
        for pred in pe.ev.predictors:
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            toks, ntok = decode(tp.feats, tp.offsets, ncf, t_max, pred)
            e1.record()
            edit_distances(toks, ntok, truth)
            e2.record()
            torch.cuda.synchronize()
            if rep:
                print(f"H={pred.hidden}: lstm+ctc {e0.elapsed_time(e1):.3f} ms  levenshtein {e1.elapsed_time(e2):.3f} ms")


if __name__ == "__main__":
    main()

"""Development aid: per-role wait/busy breakdown of the conv kernel per level
(needs the TOBF_CONV_PROF build: TOBF_LIB=scripts/_probe_libs/libtobf_prof.so)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_09789_b200 import fixtures, ga  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402

NAMES = {0: "A.info", 1: "A.empty", 2: "A.cpw", 3: "A.stw", 4: "A.issue", 5: "A.lds", 6: "A.sts", 7: "A.total", 8: "M.info", 9: "M.small", 10: "M.accE", 11: "M.full", 12: "M.issue",
         15: "M.total", 16: "D.info", 17: "D.accF", 18: "D.epi", 19: "D.bar1", 20: "D.setup", 21: "D.rows",
         22: "D.bar2", 23: "D.total", 24: "B.info", 25: "B.empty",
         31: "B.total"}


def main():
    g = fixtures.resnet18()
    space = ga.search_space(g, "sequence")
    sizes = ga.domain_sizes("sequence", space)
    plans = [ga.decode_genome(g, "sequence", space, x) for x in ga.random_genomes(np.random.default_rng(0), sizes, 32)]
    pe = PopulationEvaluator(g, Evaluator(), trials=8, memo={})
    prep = pe.prepare(plans, memo={})
    run = prep["run"]
    run.set_input(pe.x_host.cuda())
    run.run()
    torch.cuda.synchronize()
    lib = pe.ctx.lib
    lib.tobf_conv_prof_read.argtypes = [C.c_void_p, C.c_int]
    buf = np.zeros(32, np.uint64)
    lib.tobf_conv_prof_read(buf.ctypes.data, 1)
    sp = C.c_void_p(pe.ctx.sp)
    convs = [L for L in run.launches if L[0] == "conv"]
    for idx in [int(v) for v in (sys.argv[1].split(',') if len(sys.argv) > 1 else '0,1,2,4,14,20,22,29,34,38,44'.split(','))]:
        if idx >= len(convs):
            break
        _, dptr, n, tot, bn = convs[idx]
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        lib.tobf_conv_grouped(C.c_void_p(dptr), n, tot, bn, sp)
        ev1.record()
        torch.cuda.synchronize()
        lib.tobf_conv_prof_read(buf.ctypes.data, 1)
        ms = ev0.elapsed_time(ev1)
        ctas = min(tot, 148)
        per = {NAMES[k]: buf[k] / ctas / 1e3 for k in NAMES}  # kcycles per CTA
        tot_m = per["M.total"]
        t_first = (~int(buf[29])) & ((1 << 64) - 1)
        span = (int(buf[30]) - t_first) / 1e3
        start_skew = (int(buf[28]) - t_first) / 1e3
        life = int(buf[26]) / ctas / 1e3
        print(f"launch {idx}: {ms:.3f} ms probs {n} tiles {tot} BN {bn}  CTA span {span:.1f} us, start skew "
              f"{start_skew:.1f} us, mean CTA life {life:.1f} us  (kcycles/CTA)  " +
              "  ".join(f"{k}={v:.1f}" for k, v in per.items()))


if __name__ == "__main__":
    main()

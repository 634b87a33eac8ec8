"""Development aid: per-launch timing of the grouped conv over a real RN18
sequence population (CUDA events around each conv launch), printing the
problem mix, tile count, algorithmic FLOPs and achieved TFLOP/s per launch."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_09789_b200 import fixtures, ga  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402


def main(pop=32, reps=5, fixture="resnet18", mode="sequence", prec="fp32"):
    g = fixtures.FIXTURES[fixture]()
    space = ga.search_space(g, mode)
    sizes = ga.domain_sizes(mode, space)
    plans = [ga.decode_genome(g, mode, space, x) for x in ga.random_genomes(np.random.default_rng(0), sizes, pop)]
    pe = PopulationEvaluator(g, Evaluator(), trials=8, memo={}, precision=prec)
    prep = pe.prepare(plans, memo={})
    run = prep["run"]
    x = pe.x_host.cuda()
    run.set_input(x)
    for _ in range(2):
        run.run()
    torch.cuda.synchronize()
    times = np.zeros(sum(1 for L in run.launches if L[0] == "conv"))
    for _ in range(reps):
        run.conv_events = []
        run.run()
        torch.cuda.synchronize()
        times += np.array([a.elapsed_time(b) for a, b in run.conv_events])
    times /= reps
    run.conv_events = None
    # flops per launch from the host descriptor blobs
    import ctypes as C
    from paper_2107_09789_b200 import _native as N
    host = run.desc_dev.cpu().numpy().tobytes()
    base = run.desc_dev.data_ptr()
    rows = []
    ci = 0
    for kind, dptr, n, tot, bn in run.launches:
        if kind != "conv":
            continue
        arr = (N.ConvDesc * n).from_buffer_copy(host[dptr - base:dptr - base + n * C.sizeof(N.ConvDesc)])
        fl = sum(2.0 * d.batch * d.Ho * d.Wo * d.j * d.k1 * d.k2 * d.Cp for d in arr)
        kmax = max(d.kblocks for d in arr)
        kavg = sum(d.kblocks * d.mtiles * d.ntiles for d in arr) / max(tot, 1)
        geo = sorted({(d.k1, d.Cp, d.j, d.Ho) for d in arr})
        rows.append((times[ci], n, tot, bn & 0xFF, fl, kmax, arr[0].Ho, arr[0].j, ci, kavg, geo))
        ci += 1
    tot_t = sum(r[0] for r in rows)
    tot_f = sum(r[4] for r in rows)
    print(f"conv launches {len(rows)}  total {tot_t:.2f} ms  {tot_f/1e12:.3f} TFLOP(padded K)  {tot_f/tot_t/1e9:.1f} TF/s")
    by_order = "--order" in sys.argv
    for t, n, tot, bn, fl, kmax, ho, j, ci, kavg, geo in (rows if by_order else
                                                          sorted(rows, key=lambda r: -r[0])[:25]):
        print(f"#{ci:2d} {t:7.3f} ms  probs {n:3d} tiles {tot:5d} BN {bn:3d} kblk_max {kmax:4d} avg {kavg:6.1f} "
              f"Ho {ho:3d} j {j:4d}  {fl/1e9:8.1f} GF  {fl/t/1e9:6.1f} TF/s  us/tile/SM {t * 1e3 / (tot / 148):6.2f}"
              + (f"  (k1,Cp,j,Ho) {geo[:6]}" if by_order else ""))


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--pop", type=int, default=32)
    ap.add_argument("--fixture", default="resnet18")
    ap.add_argument("--mode", default="sequence")
    ap.add_argument("--prec", default="fp32")
    ap.add_argument("--order", action="store_true")
    a = ap.parse_args()
    main(a.pop, 5, a.fixture, a.mode, a.prec)
    sys.exit(0)
    main()

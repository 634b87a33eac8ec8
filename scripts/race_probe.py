"""Development aid: the forward of the headline population run repeatedly on
one prepared PopulationRun; every launch's outputs are checksummed (int32 sum
of their float bits) after the launch and compared with the first repetition.
Prints the first launch whose outputs differ in any repetition.
usage: python scripts/race_probe.py [reps]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import population_plans  # noqa: E402
from paper_2107_09789_b200 import fixtures  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402
from paper_2107_09789_b200.executor import CONV_DTYPE, EW_DTYPE, conv_sched  # noqa: E402

import argparse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("reps", type=int, nargs="?", default=30)
ap.add_argument("--prec", default="fp32")
ap.add_argument("--fixture", default="resnet18")
ap.add_argument("--mode", default="sequence")
ap.add_argument("--pop", type=int, default=32)
a = ap.parse_args()
reps = a.reps
g = getattr(fixtures, a.fixture)()
if a.mode == "sequence":
    plans = population_plans(g, a.pop, 0)
else:
    from paper_2107_09789_b200 import ga  # noqa: E402
    _rng = np.random.default_rng(0)
    _space = ga.search_space(g, a.mode)
    plans = [ga.decode_genome(g, a.mode, _space, x)
             for x in ga.random_genomes(_rng, ga.domain_sizes(a.mode, _space), a.pop)]
pe = PopulationEvaluator(g, Evaluator(), budget=0.02, trials=8, seed=0, memo={}, precision=a.prec)
prep = pe.prepare(plans, memo={})
run = prep["run"]
ctx = pe.ctx
lib = ctx.lib
x = pe.x_host.to(ctx.device)
base = run.desc_dev.data_ptr()
conv_bytes = len(run.conv_rows) * CONV_DTYPE.itemsize
ew_base = base + conv_bytes + ((-conv_bytes) % 256)
arena = run.arena


def regions(kind, dptr, n):
    out = []
    if kind == "conv":
        lo = (dptr - base) // CONV_DTYPE.itemsize
        for r in run.conv_rows[lo:lo + n]:
            out.append((int(r["y"]), int(r["batch"]) * int(r["Ho"]) * int(r["Wo"]) * int(r["ldy"])))
    else:
        lo = (dptr - ew_base) // EW_DTYPE.itemsize
        for r in run.ew_rows[lo:lo + n]:
            ho, wo = (int(r["Ho"]), int(r["Wo"])) if int(r["Ho"]) else (int(r["H"]), int(r["W"]))
            out.append((int(r["y"]), int(r["batch"]) * max(ho, 1) * max(wo, 1) * int(r["ldy"])))
    return out


def checksum(ptr, floats):
    t = arena.view(ptr, floats)
    return int(t.view(torch.int32).to(torch.int64).sum().item())


snap = {}  # (launch, problem) -> output copy of repetition 0


sp = C.c_void_p(ctx.sp)
sched = C.c_void_p(conv_sched(ctx).data_ptr())
ref = None
first_bad = {}
for rep in range(reps):
    run.set_input(x)
    sums = []
    for li, (kind, dptr, n, tot, bn) in enumerate(run.launches):
        if kind == "conv":
            rc = lib.tobf_conv_grouped_ex(C.c_void_p(dptr), n, tot, bn, run.prec, sched, sp)
        else:
            rc = lib.tobf_ew_grouped(C.c_void_p(dptr), n, tot, sp)
        ctx.check(rc, kind)
        torch.cuda.synchronize()
        regs = regions(kind, dptr, n)
        sums.append([checksum(p, f) for p, f in regs])
        if rep == 0 and kind == "conv":
            for i, (p, f) in enumerate(regs):
                snap[(li, i)] = arena.view(p, f).clone()
        elif kind == "conv" and ref is not None and sums[-1] != ref[li]:
            lo = (dptr - base) // CONV_DTYPE.itemsize
            for i, (u, v) in enumerate(zip(ref[li], sums[-1])):
                if u == v:
                    continue
                r = run.conv_rows[lo + i]
                ldy, j = int(r["ldy"]), int(r["j"])
                cur = arena.view(*regs[i]).view(-1, ldy)[:, :j]
                old = snap[(li, i)].view(-1, ldy)[:, :j]
                d = (cur != old).nonzero()
                rows, cols = d[:, 0], d[:, 1]
                tiles = sorted(set((rows // 128).tolist()))
                print(f"   launch {li} problem {i}: {len(d)} elements differ, rows {int(rows.min())}..{int(rows.max())}"
                      f" (M={int(r['batch']) * int(r['Ho']) * int(r['Wo'])}), m-tiles {tiles[:12]}{'...' if len(tiles) > 12 else ''},"
                      f" cols {int(cols.min())}..{int(cols.max())}, max |diff| {float((cur - old).abs().max()):.3e}"
                      f" x=0x{int(r['x']):x} y=0x{int(r['y']):x} tile_start={int(r['tile_start'])} mtiles={int(r['mtiles'])}"
                      f" epi={[(int(e['op']), int(e['aux'])) for e in r['epi'][:int(r['nepi'])]]}", flush=True)
    if ref is None:
        ref = sums
        continue
    for li, (a, b) in enumerate(zip(ref, sums)):
        if a != b:
            bad = [i for i, (u, v) in enumerate(zip(a, b)) if u != v]
            kind, dptr, n, tot, bn = run.launches[li]
            print(f"rep {rep}: launch {li} ({kind}, {n} problems, {tot} units, bn {bn}) differs in problems {bad}",
                  flush=True)
            first_bad[li] = first_bad.get(li, 0) + 1
            if kind == "conv":
                lo = (dptr - base) // CONV_DTYPE.itemsize
                for i in bad[:3]:
                    r = run.conv_rows[lo + i]
                    print("   ", {k: int(r[k]) for k in ("batch", "H", "W", "Cp", "Ho", "Wo", "j", "k1", "stride", "pad",
                                                      "ksplit", "kper", "tma", "nepi", "ldx", "ldy")}, flush=True)
            break
print("first differing launches:", first_bad)

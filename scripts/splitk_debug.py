"""Development aid: execute graphs with split-K enabled vs disabled
(executor.SPLITK_MAX) and report the first node whose output differs."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_09789_b200 import executor, fixtures, ga, knobs  # noqa: E402
from paper_2107_09789_b200.ir import Graph, topo_order  # noqa: E402


def run(g, x, split):
    executor.SPLITK_MAX = split
    return executor.execute(g, x)


g0 = fixtures.resnet18(size=64)
space = ga.search_space(g0, "dimension")
sizes = ga.domain_sizes("dimension", space)
rng = np.random.default_rng(11)
for t in range(2):
    plan = ga.decode_genome(g0, "dimension", space, rng.integers(0, sizes))
    og, _ = knobs.apply_plan(g0, plan)
    x = np.random.default_rng(5).standard_normal(og.input_shape.as_tuple()).astype(np.float32)
    for nid in topo_order(og):
        n = og.nodes[nid]
        sub = Graph(og.nodes, nid, og.input_shape)
        a = run(sub, x, 1)
        b = run(sub, x, 16)
        if not np.allclose(a, b, rtol=1e-4, atol=1e-4):
            print("plan", t, "first diff at node", nid, n.kind, n.attrs, "inputs", n.inputs,
                  "maxdiff", float(np.abs(a - b).max()), flush=True)
            break
    else:
        print("plan", t, "no diff")

# detail of the failing node (plan 0)
import ctypes as C  # noqa: E402
from paper_2107_09789_b200 import _native as N  # noqa: E402
rng = np.random.default_rng(11)
plan = ga.decode_genome(g0, "dimension", space, rng.integers(0, sizes))
og, _ = knobs.apply_plan(g0, plan)
sub = Graph(og.nodes, 50, og.input_shape)
lw = executor.lower(sub)
for op in lw.ops:
    if op.out == 50 or op.node == 50:
        print("op", op)
for nid in (48, 49, 50):
    n = og.nodes[nid]
    print(nid, n.kind, n.attrs, n.inputs, None if n.weights is None else (n.weights.shape, n.weights.strides))
executor.SPLITK_MAX = 16
run = executor.PopulationRun(executor.device(), [lw], reps=1)
host = run.desc_dev.cpu().numpy().tobytes()
base = run.desc_dev.data_ptr()
for kind, dptr, n, tot, bn in run.launches:
    if kind != "conv":
        continue
    arr = (N.ConvDesc * n).from_buffer_copy(host[dptr - base:dptr - base + n * C.sizeof(N.ConvDesc)])
    for d in arr:
        print(f"units {tot} bn {bn} HWC {d.H}x{d.W}x{d.Cp} ldx {d.ldx} -> {d.Ho}x{d.Wo} j {d.j} Cpo {d.Cpo} ldy {d.ldy} "
              f"k {d.k1}x{d.k2} s{d.stride} p{d.pad} kblocks {d.kblocks} mt {d.mtiles} nt {d.ntiles} split {d.ksplit}x{d.kper} "
              f"nepi {d.nepi} ops {[d.epi[i].op for i in range(d.nepi)]}")

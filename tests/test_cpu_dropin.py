"""The drop-in boundary with the reference's OWN objects.

The engine's public API is called with traceobf 0.1.0's classes (the real,
unmodified reference: baseline/_ref via scripts/vendor_reference.sh, else the
source tree) and must answer in those classes: apply_plan's graph equals the
reference's apply_plan result node for node (Graph.__eq__ compares weights
exactly, graph.py:102-110), kernels / labels / shapes / validation match, the
reference's exception classes are raised, and the lowered forward + trace
descriptors of a reference-typed graph are byte-identical to the engine's own.
INTEGRATION.md §3's maintainer patch (refcompat.install) is applied to the
real package and leaves it answering in its own types.
"""

from pathlib import Path

import numpy as np
import pytest

import paper_2107_09789_b200 as eng
from paper_2107_09789_b200 import executor, fixtures, ga, refcompat, trace
from paper_2107_09789_b200.executor import ArrayRefs, lower, plan_forward
from tests import refpkg

ref = refpkg.load()
pytestmark = pytest.mark.skipif(ref is None, reason="reference package not available")


def _plans(g, mode, n, seed):
    rng = np.random.default_rng(seed)
    space = ga.search_space(g, mode)
    sizes = ga.domain_sizes(mode, space)
    return [ga.decode_genome(g, mode, space, rng.integers(0, sizes)) for _ in range(n)]


@pytest.mark.parametrize("name,mode,size", [("resnet18", "sequence", 64), ("c1c2", "dimension", 24),
                                            ("vgg16", "dimension", 32)])
def test_apply_plan_with_reference_objects(name, mode, size):
    kw = {"hidden": 256} if name == "vgg16" else {}
    g = fixtures.FIXTURES[name](size=size, **kw)
    rg = refpkg.ref_graph(ref, g)
    for plan in _plans(g, mode, 3, seed=5):
        rp = refpkg.ref_plan(ref, plan)
        want, wdir = ref.apply_plan(rg, rp)
        got, gdir = eng.apply_plan(rg, rp)
        assert type(got) is ref.Graph and type(gdir) is type(wdir)
        assert got == want
        assert gdir.fusion_limits == wdir.fusion_limits and gdir.schedule_strategies == wdir.schedule_strategies
        # kernels, labels, shapes, validation of the obfuscated graph
        kern = eng.fuse(got, gdir.fusion_limits)
        assert all(type(k) is ref.Kernel for k in kern) and kern == ref.fuse(want, wdir.fusion_limits)
        assert eng.label_sequence(got) == ref.label_sequence(want)
        assert all(type(k) is ref.OperatorKind for k in eng.label_sequence(got))
        assert eng.infer_shapes(got) == ref.infer_shapes(want)
        assert eng.validate(got) == ref.validate(want) == []
        assert eng.topo_order(got) == ref.topo_order(want)


def test_lowered_descriptors_identical_for_reference_graphs():
    """Forward descriptor rows and trace kernel records of a reference-typed
    graph equal the engine-typed graph's byte for byte."""
    g = fixtures.resnet18(size=64)
    plan = _plans(g, "sequence", 1, seed=9)[0]
    og, d = eng.apply_plan(g, plan)
    rog, rd = ref.apply_plan(refpkg.ref_graph(ref, g), refpkg.ref_plan(ref, plan))
    conv = refcompat.engine_graph(rog)
    ra, rb = ArrayRefs(), ArrayRefs()
    a = plan_forward(lower(og), 8, ra)
    b = plan_forward(lower(conv), 8, rb)
    for f in ("conv_level", "conv_bn", "conv_k", "ew_level"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.ew.tobytes() == b.ew.tobytes()
    # conv rows: identical except the weight-image pointer, an index into each
    # plan's table of weight views (deduplicated by array identity) — compare
    # what it points at: the same geometry and bit-identical weights
    ca, cb = a.conv.copy(), b.conv.copy()
    low = np.uint64((1 << 56) - 1)
    ia, ib = (ca["wimg"] & low).astype(int), (cb["wimg"] & low).astype(int)
    ca["wimg"] = cb["wimg"] = 0
    assert ca.tobytes() == cb.tobytes()
    for x, y in zip(ia, ib):
        ea, eb = a.wimg[x], b.wimg[y]
        assert ea[1:] == eb[1:]
        assert np.array_equal(np.asarray(ra.resolve(ea[0])), np.asarray(rb.resolve(eb[0])))
    ta, _, _ = trace.trace_records(og, d.fusion_limits, d.schedule_strategies, "default")
    tb, _, _ = trace.trace_records(conv, rd.fusion_limits, rd.schedule_strategies, "default")
    assert ta.recs.tobytes() == tb.recs.tobytes() and ta.sigs == tb.sigs


def test_reference_exception_classes():
    g = fixtures.c1c2(size=16)
    rg = refpkg.ref_graph(ref, g)
    bad = ref.ObfuscationPlan("dimension", tuple(ref.PlanEntry(lid, widen_factor=0.5)
                                                 for lid in rg.complex_layers()))
    from traceobf.transforms import PlanApplicationError, TransformError
    with pytest.raises(PlanApplicationError) as ei:
        eng.apply_plan(rg, bad)
    assert isinstance(ei.value, TransformError) and ei.value.failures
    from traceobf.transforms import NoActivation
    r18 = refpkg.ref_graph(ref, fixtures.resnet18(size=64))
    with pytest.raises(NoActivation):
        ref.deepen_layer(r18, 7)   # BN -> Add -> ReLU: no BN-only link to an activation
    with pytest.raises(NoActivation):
        eng.deepen_layer(r18, 7)
    from traceobf.fusion import InvalidStrategy
    with pytest.raises(InvalidStrategy):
        eng.modify_schedule(ref.Schedule((4, 8, 4), (2, 4, 2)), 7)


def test_schedule_helpers_answer_in_reference_types():
    s = ref.Schedule((4, 8, 4), (2, 4, 2))
    got = eng.modify_schedule(s, 1)
    assert type(got) is ref.Schedule and got == ref.modify_schedule(s, 1)


def test_maintainer_patch_installs_on_the_real_package():
    saved = refcompat.install(ref)
    try:
        for n in refcompat.HOT_PATH:
            assert getattr(ref, n) is getattr(eng, n) and getattr(ref, n).__dropin__
    finally:
        refcompat.uninstall(ref, saved)
    assert ref.execute is ref.interpreter.execute


def test_integration_md_patch_applied_to_a_copy_of_the_reference(tmp_path):
    """The maintainer patch exactly as INTEGRATION.md §3 prints it, appended to
    a copy of the real package's __init__.py: the patched package imports,
    its hot entry points are the engine's drop-in wrappers, the rest is the
    reference's own code."""
    import re
    import shutil
    import subprocess
    import sys
    src = Path(ref.__file__).resolve().parent
    dst = tmp_path / "traceobf"
    shutil.copytree(src, dst, ignore=shutil.ignore_patterns("__pycache__"))
    md = (refpkg.ROOT / "INTEGRATION.md").read_text()
    patch = re.search(r"```python\n(# traceobf/__init__.py \(maintainer patch.*?)```", md, re.S).group(1)
    with open(dst / "__init__.py", "a") as f:
        f.write("\n" + patch)
    code = ("import traceobf, paper_2107_09789_b200 as eng\n"
            "hot = ('execute', 'equivalence_check', 'compile_graph', 'profile_pipeline')\n"
            "assert all(getattr(getattr(traceobf, n), '__dropin__', False) for n in hot)\n"
            "assert traceobf.apply_plan is traceobf.transforms.apply_plan\n"
            "assert traceobf.__file__.startswith(%r)\n"
            "print('patched ok')\n") % str(tmp_path)
    env = dict(__import__("os").environ)
    env["PYTHONPATH"] = f"{tmp_path}:{refpkg.ROOT}"
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and "patched ok" in r.stdout, r.stderr[-2000:]

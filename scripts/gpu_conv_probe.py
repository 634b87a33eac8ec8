"""Standalone GPU probe of the tcgen05 conv kernel (development aid).

Runs a handful of conv problems through tobf_conv_grouped and compares
against a float64 torch reference on the CPU. Prints one line per case.
"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_09789_b200 import _native as N  # noqa: E402

lib = C.CDLL(str(N.LIB_PATH))
for name in ("tobf_conv_prepare", "tobf_wimg_bytes", "tobf_pack_weights", "tobf_conv_grouped",
             "tobf_last_error", "tobf_check_fault"):
    res, args = N.SIGNATURES[name]
    getattr(lib, name).restype = res
    getattr(lib, name).argtypes = args


def chk(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: {rc} {lib.tobf_last_error().decode()}")


def rup(a, b):
    return (a + b - 1) // b * b


def run_case(cases, block_n, seed=0):
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda")
    keep = []
    descs = (N.ConvDesc * len(cases))()
    refs = []
    for i, cs in enumerate(cases):
        b, c, h, w, j, k, s, p = cs["shape"]
        Cp, Cpo = rup(c, 4), rup(j, 4)
        x = rng.standard_normal((b, c, h, w)).astype(np.float32)
        wt = (rng.standard_normal((k, k, c, j)) * np.sqrt(2.0 / (k * k * c))).astype(np.float32)
        xn = np.zeros((b, h, w, Cp), np.float32)
        xn[..., :c] = x.transpose(0, 2, 3, 1)
        xd = torch.from_numpy(xn).to(dev)
        wd = torch.from_numpy(wt).to(dev)
        nbytes = lib.tobf_wimg_bytes(k, k, Cp, j, block_n)
        img = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
        chk(lib.tobf_pack_weights(wd.data_ptr(), k, k, c, Cp, j, k * c * j, c * j, j, 1, block_n,
                                  img.data_ptr(), None), "pack")
        ho = (h + 2 * p - k) // s + 1
        wo = (w + 2 * p - k) // s + 1
        y = torch.full((b, ho, wo, Cpo), float("nan"), dtype=torch.float32, device=dev)
        ref = torch.nn.functional.conv2d(torch.from_numpy(x).double(),
                                         torch.from_numpy(wt).double().permute(3, 2, 0, 1), stride=s,
                                         padding=p).numpy()
        d = descs[i]
        d.x, d.wimg, d.y = xd.data_ptr(), img.data_ptr(), y.data_ptr()
        d.batch, d.H, d.W, d.Cp = b, h, w, Cp
        d.Ho, d.Wo, d.Cpo, d.j = ho, wo, Cpo, j
        d.k1, d.k2, d.stride, d.pad = k, k, s, p
        d.ldx, d.ldy = Cp, Cpo
        nepi = 0
        if cs.get("epi"):
            scale = rng.uniform(0.5, 1.5, j).astype(np.float32)
            shift = rng.normal(0, 0.1, j).astype(np.float32)
            aff = np.zeros((2, Cpo), np.float32)
            aff[0, :j], aff[1, :j] = scale, shift
            affd = torch.from_numpy(aff).to(dev)
            res = rng.standard_normal((b, ho, wo, Cpo)).astype(np.float32)
            res[..., j:] = 0
            resd = torch.from_numpy(res).to(dev)
            cst = rng.standard_normal((1, ho, wo, Cpo)).astype(np.float32)
            cstd = torch.from_numpy(cst).to(dev)
            keep += [affd, resd, cstd]
            steps = [(N.EPI_AFFINE, Cpo, affd.data_ptr()), (N.EPI_RELU, 0, 0),
                     (N.EPI_ADD_TENSOR, Cpo, resd.data_ptr()), (N.EPI_ADD_CONST, 1, cstd.data_ptr()),
                     (N.EPI_RELU, 0, 0)]
            for si, (op, aux, ptr) in enumerate(steps):
                d.epi[si].op, d.epi[si].aux, d.epi[si].ptr = op, aux, ptr
            nepi = len(steps)
            r = ref * scale.astype(np.float64)[None, :, None, None] + shift[None, :, None, None]
            r = np.maximum(r, 0)
            r = r + res[..., :j].transpose(0, 3, 1, 2)
            r = r + cst[..., :j].transpose(0, 3, 1, 2)
            ref = np.maximum(r, 0)
        d.nepi = nepi
        keep += [xd, wd, img, y]
        refs.append((ref, y, j))
    total = C.c_int64(0)
    chk(lib.tobf_conv_prepare(descs, len(cases), block_n, C.byref(total)), "prepare")
    dd = torch.frombuffer(bytearray(bytes(descs)), dtype=torch.uint8).to(dev)
    torch.cuda.synchronize()
    chk(lib.tobf_conv_grouped(dd.data_ptr(), len(cases), total.value, block_n, None), "conv")
    torch.cuda.synchronize()
    chk(lib.tobf_check_fault(None), "fault")
    out = []
    for (ref, y, j), cs in zip(refs, cases):
        got = y.cpu().numpy()
        pad_ok = bool(np.all(got[..., j:] == 0))
        got = got[..., :j].transpose(0, 3, 1, 2).astype(np.float64)
        err = np.abs(got - ref)
        rel = float((err / (1 + np.abs(ref))).max())
        nrm = float(err.max() / max(np.abs(ref).max(), 1e-30))
        out.append((cs["shape"], cs.get("epi", False), rel, nrm, pad_ok, bool(np.isfinite(got).all())))
    # timing of the whole group
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        lib.tobf_conv_grouped(dd.data_ptr(), len(cases), total.value, block_n, None)
    t0.record()
    iters = 10
    for _ in range(iters):
        lib.tobf_conv_grouped(dd.data_ptr(), len(cases), total.value, block_n, None)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / iters
    flops = 0
    for cs in cases:
        b, c, h, w, j, k, s, p = cs["shape"]
        ho = (h + 2 * p - k) // s + 1
        wo = (w + 2 * p - k) // s + 1
        flops += 2 * b * ho * wo * j * k * k * c
    return out, ms, flops / ms / 1e9


def main():
    torch.cuda.init()
    groups = [
        (128, [{"shape": (2, 64, 56, 56, 128, 3, 1, 1)}]),
        (64, [{"shape": (1, 3, 64, 64, 64, 7, 2, 3)}]),
        (64, [{"shape": (2, 128, 14, 14, 68, 1, 1, 0)}]),
        (64, [{"shape": (1, 20, 9, 9, 17, 5, 1, 2)}]),
        (128, [{"shape": (2, 64, 20, 20, 96, 3, 2, 1), "epi": True},
               {"shape": (1, 17, 11, 11, 144, 3, 1, 1), "epi": True},
               {"shape": (3, 256, 7, 7, 512, 3, 1, 1)}]),
        (128, [{"shape": (8, 512, 7, 7, 512, 3, 1, 1)}] * 4),
        (128, [{"shape": (8, 64, 56, 56, 128, 3, 1, 1)}] * 4),
    ]
    worst = 0.0
    for bn, cases in groups:
        t = time.time()
        res, ms, tflops = run_case(cases, bn)
        for shape, epi, rel, nrm, pad_ok, fin in res:
            worst = max(worst, rel)
            print(f"BN={bn} shape={shape} epi={epi} rel={rel:.3e} nrm={nrm:.3e} pad0={pad_ok} finite={fin}")
        print(f"  group: {ms:.3f} ms  {tflops:.1f} GFLOP/s algorithmic  (wall {time.time()-t:.1f}s)")
    print("WORST", worst)


if __name__ == "__main__":
    main()

"""Development aid: per-tile cost of the conv epilogue as a function of the
fused chain (1 K-block problems, so the epilogue dominates). Run with
TOBF_LIB=scripts/_probe_libs/libtobf_prof.so for the role breakdown."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_09789_b200 import _native as N  # noqa: E402


def main():
    lib = N.load()
    prof = hasattr(lib, "tobf_conv_prof_read")
    if prof:
        lib.tobf_conv_prof_read.argtypes = [C.c_void_p, C.c_int]
    dev = torch.device("cuda")
    for bn, j in ((128, 128), (64, 64)):
        b, h, w, cp, k = 8, 56, 56, 32, 1
        nprob = 32
        x = torch.randn(b * h * w * cp, device=dev)
        wt = torch.randn(k * k * cp * j, device=dev)
        img = torch.empty(lib.tobf_wimg_bytes(k, k, cp, j, bn) // 4, device=dev)
        N.check(lib.tobf_pack_weights(C.c_void_p(wt.data_ptr()), k, k, cp, cp, j, 0, 0, j, 1, bn,
                                      C.c_void_p(img.data_ptr()), None))
        ys = [torch.empty(b * h * w * j, device=dev) for _ in range(nprob)]
        res = torch.randn(b * h * w * j, device=dev)
        cst = torch.randn(h * w * j, device=dev)
        aff = torch.randn(2 * j, device=dev)
        variants = {
            "none": [],
            "relu": [(N.EPI_RELU, 0, 0)],
            "affine+relu": [(N.EPI_AFFINE, j, aff.data_ptr()), (N.EPI_RELU, 0, 0)],
            "affine+add+relu": [(N.EPI_AFFINE, j, aff.data_ptr()), (N.EPI_ADD_TENSOR, j, res.data_ptr()),
                                (N.EPI_RELU, 0, 0)],
            "const": [(N.EPI_ADD_CONST, 1, cst.data_ptr())],
        }
        for name, epi in variants.items():
            arr = (N.ConvDesc * nprob)()
            for i in range(nprob):
                d = arr[i]
                d.x, d.wimg, d.y = x.data_ptr(), img.data_ptr(), ys[i].data_ptr()
                d.batch, d.H, d.W, d.Cp = b, h, w, cp
                d.Ho, d.Wo, d.Cpo, d.j = h, w, j, j
                d.k1 = d.k2 = k
                d.stride, d.pad, d.ldx, d.ldy = 1, 0, cp, j
                for si, (op, aux, ptr) in enumerate(epi):
                    d.epi[si].op, d.epi[si].aux, d.epi[si].ptr = op, aux, ptr
                d.nepi = len(epi)
            tot = C.c_int64()
            N.check(lib.tobf_conv_prepare(arr, nprob, bn, C.byref(tot)))
            dd = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(dev)
            for _ in range(2):
                lib.tobf_conv_grouped(C.c_void_p(dd.data_ptr()), nprob, tot.value, bn, None)
            torch.cuda.synchronize()
            buf = np.zeros(32, np.uint64)
            if prof:
                lib.tobf_conv_prof_read(buf.ctypes.data, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lib.tobf_conv_grouped(C.c_void_p(dd.data_ptr()), nprob, tot.value, bn, None)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            tiles_per_cta = tot.value / 148
            line = f"BN={bn} {name:16s} {ms:.3f} ms  tiles {tot.value}  {ms * 1e3 / tiles_per_cta:.2f} us/tile/SM"
            if prof:
                lib.tobf_conv_prof_read(buf.ctypes.data, 1)
                f = lambda i: buf[i] / 148 / tiles_per_cta  # noqa: E731  cycles per tile
                line += (f"   D.rows {f(21):.0f}  D.setup {f(20):.0f}  D.accF {f(17):.0f}  M.full {f(11):.0f}"
                         f"  M.accE {f(10):.0f}  A.empty {f(1):.0f}  M.total {f(15):.0f}")
            print(line, flush=True)


if __name__ == "__main__":
    main()

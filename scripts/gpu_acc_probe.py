"""Development aid: error growth of the tcgen05 tf32 conv vs K for MMA variants.

1x1 convolutions are plain GEMMs (K = channels). Compares each library
variant (scripts/_probe_libs/libconv_m{0,1,2}.so) against float64 and against
a float32 CPU matmul (the reference's own arithmetic class).
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_09789_b200 import _native as N  # noqa: E402

LIBS = Path(__file__).resolve().parent / "_probe_libs"


def bind(path):
    lib = C.CDLL(str(path))
    for name in ("tobf_conv_prepare", "tobf_wimg_bytes", "tobf_pack_weights", "tobf_conv_grouped",
                 "tobf_last_error", "tobf_check_fault"):
        res, args = N.SIGNATURES[name]
        getattr(lib, name).restype = res
        getattr(lib, name).argtypes = args
    return lib


def gemm(lib, x, w, bn=128):
    # x: (M, K) -> NHWC (M,1,1,K); w: (K, J) -> (1,1,K,J)
    dev = torch.device("cuda")
    M, K = x.shape
    J = w.shape[1]
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    wd = torch.from_numpy(np.ascontiguousarray(w)).to(dev)
    img = torch.empty(lib.tobf_wimg_bytes(1, 1, K, J, bn) // 4, dtype=torch.float32, device=dev)
    assert lib.tobf_pack_weights(wd.data_ptr(), 1, 1, K, K, J, 0, 0, J, 1, bn, img.data_ptr(), None) == 0
    y = torch.empty((M, J), dtype=torch.float32, device=dev)
    d = (N.ConvDesc * 1)()
    d[0].x, d[0].wimg, d[0].y = xd.data_ptr(), img.data_ptr(), y.data_ptr()
    d[0].batch, d[0].H, d[0].W, d[0].Cp = M, 1, 1, K
    d[0].Ho, d[0].Wo, d[0].Cpo, d[0].j = 1, 1, J, J
    d[0].k1, d[0].k2, d[0].stride, d[0].pad = 1, 1, 1, 0
    d[0].ldx, d[0].ldy, d[0].nepi = K, J, 0
    tot = C.c_int64()
    assert lib.tobf_conv_prepare(d, 1, bn, C.byref(tot)) == 0
    dd = torch.frombuffer(bytearray(bytes(d)), dtype=torch.uint8).to(dev)
    assert lib.tobf_conv_grouped(dd.data_ptr(), 1, tot.value, bn, None) == 0
    torch.cuda.synchronize()
    assert lib.tobf_check_fault(None) == 0
    return y.cpu().numpy()


def main():
    libs = {m: bind(LIBS / f"libconv_m{m}.so") for m in (0,)}
    rng = np.random.default_rng(1)
    for K in (32, 128, 512, 2048, 4608, 16384):
        M, J = 512, 128
        x = rng.standard_normal((M, K)).astype(np.float32)
        w = (rng.standard_normal((K, J)) / np.sqrt(K)).astype(np.float32)
        ref = x.astype(np.float64) @ w.astype(np.float64)
        scale = np.abs(ref).max()
        f32 = (x @ w).astype(np.float64)
        naive = np.zeros_like(ref, dtype=np.float32)  # strict sequential fp32 accumulate over K
        acc = np.zeros((M, J), np.float32)
        for k in range(K):
            acc = (acc + x[:, k:k + 1] * w[k:k + 1, :]).astype(np.float32)
        naive = acc.astype(np.float64)
        line = [f"K={K:6d}", f"blas_f32={np.abs(f32-ref).max()/scale:.2e}",
                f"seq_f32={np.abs(naive-ref).max()/scale:.2e}"]
        for m, lib in libs.items():
            got = gemm(lib, x, w).astype(np.float64)
            err = got - ref
            line.append(f"m{m}: max={np.abs(err).max()/scale:.2e} mean={err.mean()/scale:+.1e}")
        print("  ".join(line), flush=True)


if __name__ == "__main__":
    main()

"""The C ABI boundary without a GPU: libtobf.so loads, exports every symbol
include/tobf.h declares, its struct layouts match the ctypes mirror, and the
host-only entry points (descriptor preparation, sizes, errors) behave."""

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2107_09789_b200 import _native as N

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "tobf.h"


@pytest.fixture(scope="module")
def lib():
    from paper_2107_09789_b200 import build_native
    build_native.build()
    return N.load()


def declared_functions() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(tobf_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} missing from the ctypes mirror"
    assert set(N.SIGNATURES) == set(names)


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(f'#include "{HEADER}"\n#include <stdio.h>\n#include <stddef.h>\n'
                   "int main(void){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(tobf_conv_desc),"
                   " sizeof(tobf_ew_desc), sizeof(tobf_kern_desc), offsetof(tobf_conv_desc, epi),"
                   " offsetof(tobf_ew_desc, work_start), offsetof(tobf_kern_desc, ty));"
                   " printf(\"%zu %zu\\n\", offsetof(tobf_conv_desc, ws), offsetof(tobf_conv_desc, kper)); return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got == [C.sizeof(N.ConvDesc), C.sizeof(N.EwDesc), C.sizeof(N.KernDesc), N.ConvDesc.epi.offset,
                   N.EwDesc.work_start.offset, N.KernDesc.ty.offset, N.ConvDesc.ws.offset, N.ConvDesc.kper.offset]


def test_conv_prepare_tiles_and_validation(lib):
    arr = (N.ConvDesc * 2)()
    for d, (b, h, j) in zip(arr, ((8, 56, 128), (1, 7, 512))):
        d.batch, d.H, d.W, d.Cp = b, h, h, 64
        d.Ho, d.Wo, d.Cpo, d.j = h, h, j, j
        d.k1 = d.k2 = 3
        d.stride, d.pad, d.ldx, d.ldy = 1, 1, 64, j
    tot = C.c_int64()
    assert lib.tobf_conv_prepare(arr, 2, 128, C.byref(tot)) == 0
    assert arr[0].K == 576 and arr[0].kblocks == 18
    assert arr[0].mtiles == (8 * 56 * 56 + 127) // 128 and arr[0].ntiles == 1
    assert arr[1].tile_start == arr[0].mtiles and arr[1].ntiles == 4
    assert tot.value == arr[0].mtiles + arr[1].mtiles * 4
    arr[0].Cp = 6  # not a multiple of 4 -> rejected, message recorded
    assert lib.tobf_conv_prepare(arr, 2, 128, C.byref(tot)) == N.TOBF_E_INVALID
    assert b"layout" in lib.tobf_last_error()
    assert lib.tobf_conv_prepare(arr, 2, 96, C.byref(tot)) != 0


def test_wimg_bytes(lib):
    # RN18 layer4 conv: K = 3*3*512 = 4608 -> 144 K-blocks, j = 512 -> 4 tiles of 128
    assert lib.tobf_wimg_bytes(3, 3, 512, 512, 128) == 4 * 144 * 2 * 128 * 128
    assert lib.tobf_wimg_bytes(7, 7, 4, 64, 64) == 1 * 7 * 2 * 64 * 128  # stem: K = 196 -> 7 blocks


def test_ew_prepare(lib):
    arr = (N.EwDesc * 3)()
    arr[0].op, arr[0].batch, arr[0].Ho, arr[0].Wo, arr[0].Cpo, arr[0].ldx, arr[0].ldy = N.OP_MAXPOOL, 2, 3, 3, 8, 8, 8
    arr[0].a0, arr[0].a1 = 2, 2
    arr[1].op, arr[1].batch, arr[1].H, arr[1].W, arr[1].C, arr[1].Cpo, arr[1].a0 = N.OP_COPYCH, 1, 2, 2, 17, 36, 17
    arr[2].op, arr[2].batch, arr[2].H, arr[2].W = N.OP_SOFTMAX, 4, 1, 1
    tot = C.c_int64()
    assert lib.tobf_ew_prepare(arr, 3, C.byref(tot)) == 0
    # each descriptor's range is padded to a multiple of 32 items (no warp
    # straddles two descriptors: the softmax reduces with full-warp shuffles)
    assert arr[1].work_start == 64  # 2*3*3*2 = 36 maxpool items
    assert arr[2].work_start == arr[1].work_start + 96  # 4*(36-17) = 76 channel copies
    assert tot.value == arr[2].work_start + 4 * 32
    arr[0].op = 99
    assert lib.tobf_ew_prepare(arr, 3, C.byref(tot)) != 0


def test_invalid_arguments_never_throw(lib):
    assert lib.tobf_conv_grouped(None, 1, 10, 128, None) != 0
    assert lib.tobf_lstm_ctc(None, None, 4, 9, 128, 5, None, None, None, None, None, None, 8, None, None) != 0
    assert lib.tobf_levenshtein(None, None, 4, 8, None, 3, None, None, None) != 0
    assert lib.tobf_version() >= 1


def _descs(shapes):
    arr = (N.ConvDesc * len(shapes))()
    for d, (b, h, c, j, k) in zip(arr, shapes):
        d.batch, d.H, d.W, d.Cp = b, h, h, c
        d.Ho, d.Wo, d.Cpo, d.j = h, h, j, j
        d.k1 = d.k2 = k
        d.stride, d.pad, d.ldx, d.ldy = 1, k // 2, c, j
    return arr


def test_conv_prepare_split_policy(lib):
    """Split-K only for groups with < 2 tiles per SM; units of >= 16 K blocks,
    no empty unit, tile_start counts units, workspace offsets per split tile."""
    tot, wsf, cnt = C.c_int64(), C.c_int64(), C.c_int64()
    # many tiles: no split, identical to tobf_conv_prepare
    big = _descs([(8, 56, 64, 64, 3)] * 2)
    assert lib.tobf_conv_prepare_split(big, 2, 64, 148, 16, None, None, C.byref(tot), C.byref(wsf), C.byref(cnt)) == 0
    assert tot.value == 2 * 196 and wsf.value == 0 and cnt.value == 0
    assert all(d.ksplit == 1 and d.kper == d.kblocks and not d.ws for d in big)
    # stage-4 shaped tail: 3 problems of 4 x 4 tiles, K = 4608 (144 blocks) / 512 (16 blocks)
    small = _descs([(8, 7, 512, 512, 3), (8, 7, 512, 512, 3), (8, 7, 512, 512, 1)])
    base = 1 << 20
    assert lib.tobf_conv_prepare_split(small, 3, 128, 148, 16, C.c_void_p(base), C.c_void_p(base * 4),
                                       C.byref(tot), C.byref(wsf), C.byref(cnt)) == 0
    units = 0
    for d in small:
        assert d.kper >= 16 or d.ksplit == 1
        assert (d.ksplit - 1) * d.kper < d.kblocks <= d.ksplit * d.kper
        assert d.tile_start == units
        units += d.mtiles * d.ntiles * d.ksplit
    assert tot.value == units
    assert small[0].ksplit > 1 and small[2].ksplit == 1 and not small[2].ws
    assert small[0].ws == base and small[0].cnt == base * 4
    assert small[1].ws == base + 4 * 16 * small[0].ksplit * 128 * 128
    assert wsf.value == 16 * 128 * 128 * (small[0].ksplit + small[1].ksplit)
    assert cnt.value == 32
    # NULL bases: byte offsets for the caller to rebase (executor.py does)
    assert lib.tobf_conv_prepare_split(small, 3, 128, 148, 16, None, None, C.byref(tot), C.byref(wsf),
                                       C.byref(cnt)) == 0
    assert not small[0].ws and small[1].ws == 4 * 16 * small[0].ksplit * 128 * 128 and small[1].cnt == 4 * 16
    # max_split caps the units per tile
    assert lib.tobf_conv_prepare_split(small, 3, 128, 148, 2, None, None, C.byref(tot), C.byref(wsf),
                                       C.byref(cnt)) == 0
    assert max(d.ksplit for d in small) == 2

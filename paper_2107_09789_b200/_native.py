"""ctypes binding of libtobf.so (include/tobf.h).

The product path has no CPU fallback: if the shared library is missing or
fails to load, importing the engine raises NativeUnavailable.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libtobf.so"

TOBF_OK = 0
TOBF_E_INVALID, TOBF_E_CUDA, TOBF_E_FAULT = -1, -2, -3
TOBF_MAX_EPI = 6
EPI_NONE, EPI_AFFINE, EPI_RELU, EPI_ADD_TENSOR, EPI_ADD_CONST = 0, 1, 2, 3, 4
OP_MAXPOOL, OP_EPI, OP_COPYCH, OP_SOFTMAX = 1, 2, 3, 4
PREC_TF32X3, PREC_BF16 = 0, 1
CONV_TMA = 0x100  # block_n flag of a TMA-capable conv launch (include/tobf.h TOBF_CONV_TMA)
CONV_TMA_ALL = 0x200  # ... whose problems all take A by TMA (TOBF_CONV_TMA_ALL)
PRECISIONS = {"fp32": PREC_TF32X3, "bf16": PREC_BF16}


class NativeUnavailable(RuntimeError):
    """libtobf.so is not built or cannot be loaded; there is no fallback."""


class NativeError(RuntimeError):
    pass


class EpiStep(C.Structure):
    _fields_ = [("op", C.c_int32), ("aux", C.c_int32), ("ptr", C.c_void_p)]


class ConvDesc(C.Structure):
    _fields_ = [
        ("x", C.c_void_p), ("wimg", C.c_void_p), ("y", C.c_void_p),
        ("batch", C.c_int32), ("H", C.c_int32), ("W", C.c_int32), ("Cp", C.c_int32),
        ("Ho", C.c_int32), ("Wo", C.c_int32), ("Cpo", C.c_int32), ("j", C.c_int32),
        ("k1", C.c_int32), ("k2", C.c_int32), ("stride", C.c_int32), ("pad", C.c_int32),
        ("K", C.c_int32), ("kblocks", C.c_int32), ("mtiles", C.c_int32), ("ntiles", C.c_int32),
        ("tile_start", C.c_int32), ("nepi", C.c_int32), ("ldx", C.c_int32), ("ldy", C.c_int32),
        ("epi", EpiStep * TOBF_MAX_EPI),
        ("ws", C.c_void_p), ("cnt", C.c_void_p), ("ksplit", C.c_int32), ("kper", C.c_int32),
        ("tmap", C.c_void_p), ("tma", C.c_int32), ("pair", C.c_int32), ("y2", C.c_void_p), ("aff2", C.c_void_p),
    ]


class EwDesc(C.Structure):
    _fields_ = [
        ("x", C.c_void_p), ("y", C.c_void_p),
        ("op", C.c_int32), ("batch", C.c_int32), ("H", C.c_int32), ("W", C.c_int32),
        ("C", C.c_int32), ("ldx", C.c_int32), ("Ho", C.c_int32), ("Wo", C.c_int32),
        ("ldy", C.c_int32), ("a0", C.c_int32), ("a1", C.c_int32), ("nepi", C.c_int32),
        ("work_start", C.c_int64),
        ("Cpo", C.c_int32), ("pad_", C.c_int32),
        ("epi", EpiStep * TOBF_MAX_EPI),
    ]


class KernDesc(C.Structure):
    _fields_ = [
        ("work", C.c_int64), ("fused_work", C.c_int64), ("fused_bytes", C.c_int64),
        ("in_bytes", C.c_int64), ("w_bytes", C.c_int64), ("out_bytes", C.c_int64),
        ("tiled", C.c_int32), ("is_conv", C.c_int32),
        ("c", C.c_int32), ("k1", C.c_int32), ("k2", C.c_int32), ("s", C.c_int32),
        ("H", C.c_int32), ("W", C.c_int32), ("channel_like", C.c_int32),
        ("reuse_x_stream", C.c_int32),
        ("ty", C.c_int32 * 3), ("tx", C.c_int32 * 3),
        ("unroll", C.c_int32), ("label", C.c_int32),
        ("has_shape", C.c_int32), ("strategy", C.c_int32),
        ("sig_index", C.c_int32), ("resolved", C.c_int32),
    ]


class DeviceProfileC(C.Structure):
    _fields_ = [
        ("macs_per_cycle", C.c_int64), ("launch_overhead", C.c_int64),
        ("l1_bytes", C.c_int64), ("l2_bytes", C.c_int64), ("sm_count", C.c_int64),
    ]


assert C.sizeof(ConvDesc) == 256, C.sizeof(ConvDesc)  # <= one 256-B tile-info ring slot (conv_tc.cu)
assert C.sizeof(EwDesc) == 176, C.sizeof(EwDesc)
assert C.sizeof(KernDesc) == 136, C.sizeof(KernDesc)

_vp, _i32, _i64, _f32, _f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_double

# name -> (restype, argtypes); mirrors include/tobf.h one to one.
SIGNATURES = {
    "tobf_conv_prepare": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_i64)]),
    "tobf_conv_prepare_split": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp, C.POINTER(_i64),
                                          C.POINTER(_i64), C.POINTER(_i64)]),
    "tobf_wimg_bytes": (_i64, [_i32, _i32, _i32, _i32, _i32]),
    "tobf_pack_weights": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i64, _i64, _i64, _i64, _i32, _vp, _vp]),
    "tobf_pack_weights_gather": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i64, _i64, _i64, _i64, _vp, _vp, _i32,
                                           _vp, _vp]),
    "tobf_conv_grouped": (C.c_int, [_vp, C.c_int, _i64, C.c_int, _vp]),
    "tobf_conv_prepare_ex": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(_i64)]),
    "tobf_conv_prepare_split_ex": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp,
                                             C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]),
    "tobf_wimg_bytes_ex": (_i64, [_i32, _i32, _i32, _i32, _i32, _i32]),
    "tobf_pack_weights_ex": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i64, _i64, _i64, _i64, _vp, _vp, _i32,
                                       _i32, _vp, _vp]),
    "tobf_conv_grouped_ex": (C.c_int, [_vp, C.c_int, _i64, C.c_int, C.c_int, _vp, _vp]),
    "tobf_conv_tmaps": (C.c_int, [_vp, C.c_int, _vp, C.c_uint64, C.POINTER(C.c_int)]),
    "tobf_ew_prepare": (C.c_int, [_vp, C.c_int, C.POINTER(_i64)]),
    "tobf_ew_grouped": (C.c_int, [_vp, C.c_int, _i64, _vp]),
    "tobf_equiv_compare": (C.c_int, [_vp, _vp, C.c_int, _i64, _i32, _i32, _f32, _vp, _vp, _vp]),
    "tobf_nhwc_to_nchw": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp]),
    "tobf_nchw_to_nhwc": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp]),
    "tobf_im2col": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "tobf_schedule_search": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "tobf_resolve_schedules": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "tobf_profile_kernels": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp]),
    "tobf_trace_totals": (C.c_int, [_vp, _vp, C.c_int, _vp, _vp]),
    "tobf_lstm_ctc": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp]),
    "tobf_levenshtein": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _i32, _vp, _vp, _vp]),
    "tobf_fitness_eq10": (C.c_int, [_vp, _i32, _i32, _vp, _vp, _f64, _f64, _f64, _vp, _vp, _vp]),
    "tobf_forest_der": (C.c_int, [_vp, _i32, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32,
                                  _vp, _vp, _vp]),
    "tobf_last_error": (C.c_char_p, []),
    "tobf_version": (C.c_int, []),
    "tobf_check_fault": (C.c_int, [_vp]),
    "tobf_fault_async": (C.c_int, [_vp, _vp]),
    "tobf_device_sync": (C.c_int, []),
}

_LIB = None


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load (once) and type the shared library; raises NativeUnavailable."""
    global _LIB
    if _LIB is not None:
        return _LIB
    p = Path(path) if path else Path(os.environ.get("TOBF_LIB", LIB_PATH))  # TOBF_LIB: debug builds
    if not p.exists():
        raise NativeUnavailable(
            f"{p} is missing: build it with `python -m paper_2107_09789_b200.build_native` "
            "(there is no CPU fallback)")
    try:
        lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
    except OSError as exc:
        raise NativeUnavailable(f"cannot load {p}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError here = ABI drift, fail loudly
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc != TOBF_OK:
        msg = _LIB.tobf_last_error().decode(errors="replace") if _LIB else "?"
        raise NativeError(f"{what or 'libtobf'} failed ({rc}): {msg}")

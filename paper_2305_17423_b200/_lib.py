"""ctypes binding of libfisedit.so (the C ABI declared in include/fisedit.h).

This is the thin boundary between the Python host mirror of the reference API
and the sm_100a kernels. It fails loudly: there is no CPU fallback anywhere in
the product path.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import torch

from .errors import CacheMissError, ContractViolation

import os as _os

# FIS_LIB (profiling experiments): load an alternative in-tree build, e.g. libfisedit_vm6.so
_LIB_PATH = Path(__file__).resolve().parent / _os.environ.get("FIS_LIB", "libfisedit.so")
_lib = None

F32, BF16 = 0, 1
A_ROWS, A_CONV3X3 = 0, 1
EPI_NONE, EPI_GN_SILU, EPI_STEP = 0, 1, 2
MAX_LEVELS = 8


class Ref(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("step_stride", C.c_longlong), ("ld", C.c_int), ("dtype", C.c_int)]


class Src(C.Structure):
    _fields_ = [("fresh", Ref), ("cache", Ref), ("index", C.c_void_p), ("h", C.c_int), ("w", C.c_int),
                ("c", C.c_int), ("up", C.c_int)]


class GemmArgs(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int), ("k", C.c_int), ("a_mode", C.c_int), ("a", Ref),
                ("rows", C.c_void_p), ("out_h", C.c_int), ("out_w", C.c_int), ("nsrc", C.c_int),
                ("src", Src * 2), ("b", Ref), ("alpha", C.c_float), ("bias", C.c_void_p), ("bias2", Ref),
                ("pre", Ref), ("epi", C.c_int), ("gn_mean", Ref), ("gn_var", Ref), ("gamma", C.c_void_p),
                ("beta", C.c_void_p), ("groups", C.c_int), ("eps", C.c_float), ("pre2", Ref), ("lat", Ref),
                ("step_scale", C.c_float), ("res", Ref), ("d", Ref), ("d_trans", C.c_int), ("n_split", C.c_int), ("d2", Ref), ("d2_trans", C.c_int),
                ("d_rows", C.c_void_p), ("splits", C.c_int), ("ws", C.c_void_p), ("ws_floats", C.c_longlong), ("counters", C.c_void_p),
                ("step", C.c_void_p), ("impl", C.c_int), ("static_meta", C.c_int),
                ("m_halo", C.c_int)]


class GnStatsArgs(C.Structure):
    _fields_ = [("hw", C.c_int), ("c", C.c_int), ("groups", C.c_int), ("x", Ref), ("mean", Ref), ("var", Ref),
                ("step", C.c_void_p), ("n_img", C.c_int)]


class GnApplyArgs(C.Structure):
    _fields_ = [("rows", C.c_int), ("c", C.c_int), ("groups", C.c_int), ("eps", C.c_float), ("x", Ref),
                ("x_rows", C.c_void_p), ("mean", Ref), ("var", Ref), ("gamma", C.c_void_p), ("beta", C.c_void_p),
                ("y_norm", Ref), ("y_silu", Ref), ("y_rows", C.c_void_p), ("step", C.c_void_p),
                ("img_rows", C.c_int), ("row_img", C.c_void_p)]


class SoftmaxArgs(C.Structure):
    _fields_ = [("rows", C.c_int), ("cols", C.c_int), ("pad_cols", C.c_int), ("s", Ref), ("scale", C.c_float),
                ("p", Ref), ("map", Ref), ("cached", Ref), ("verbatim", C.c_int), ("npairs", C.c_int),
                ("pair_old", C.c_void_p), ("pair_new", C.c_void_p), ("step", C.c_void_p)]


class AttnArgs(C.Structure):
    _fields_ = [("m", C.c_int), ("n_keys", C.c_int), ("d", C.c_int), ("dv", C.c_int), ("q", Ref), ("k", Ref),
                ("vt", Ref), ("scale", C.c_float), ("res", Ref), ("pre", Ref), ("out", Ref), ("step", C.c_void_p),
                ("nseg", C.c_int), ("max_seg_q", C.c_int), ("q_seg", C.c_void_p), ("k_seg", C.c_void_p),
                ("max_seg_k", C.c_int), ("ws", C.c_void_p), ("ws_bytes", C.c_longlong)]


class PoolArgs(C.Structure):
    _fields_ = [("n", C.c_int), ("c", C.c_int), ("src", Src), ("rows", C.c_void_p), ("out", Ref),
                ("step", C.c_void_p)]


class MaterializeArgs(C.Structure):
    _fields_ = [("c", C.c_int), ("src", Src), ("out", Ref), ("step", C.c_void_p)]


class MaskDetectArgs(C.Structure):
    _fields_ = [("h", C.c_int), ("w", C.c_int), ("c", C.c_int), ("t1", C.c_int), ("t2", C.c_int),
                ("radius", C.c_int), ("x", Ref), ("y", Ref), ("values", C.c_void_p), ("raw_mask", C.c_void_p),
                ("mask", C.c_void_p), ("result", C.c_void_p), ("flags", C.c_void_p),
                ("values_in", C.c_void_p)]


class MaskPlanArgs(C.Structure):
    _fields_ = [("h", C.c_int), ("w", C.c_int), ("levels", C.c_int), ("radius", C.c_int), ("mask", C.c_void_p),
                ("bits", C.c_void_p * MAX_LEVELS), ("rows", C.c_void_p * MAX_LEVELS),
                ("index", C.c_void_p * MAX_LEVELS), ("tiles", C.c_void_p * MAX_LEVELS), ("counts", C.c_void_p)]



_SIGS = {
    "fis_gemm": GemmArgs, "fis_attn": AttnArgs, "fis_gn_stats": GnStatsArgs, "fis_gn_apply": GnApplyArgs, "fis_gn": GnApplyArgs, "fis_softmax": SoftmaxArgs,
    "fis_pool2": PoolArgs, "fis_up2": PoolArgs, "fis_materialize": MaterializeArgs, "fis_mask_detect": MaskDetectArgs,
    "fis_mask_plan": MaskPlanArgs,
}

EXPORTS = tuple(_SIGS) + ("fis_attn_launches", "fis_attn_ws_bytes", "fis_gn_launches", "fis_gemm_kernel_kind", "fis_gemm_big_launch_count", "fis_gemm_pair_launch_count", "fis_gemm_ws_floats", "fis_gemm_counters", "fis_mask_detect_smem", "fis_abi_version",
                          "fis_last_error", "fis_device_sm_count")


def lib():
    """Load libfisedit.so (built in-tree). Raises if it is missing."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(f"{_LIB_PATH} is missing: build it with `python -m paper_2305_17423_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(str(_LIB_PATH))
        for name, st in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = [C.POINTER(st), C.c_void_p]
            fn.restype = C.c_int
        L.fis_gemm_ws_floats.argtypes = [C.c_int, C.c_int, C.c_int]
        L.fis_gemm_ws_floats.restype = C.c_longlong
        L.fis_gemm_counters.argtypes = [C.c_int, C.c_int]
        L.fis_gemm_counters.restype = C.c_int
        L.fis_mask_detect_smem.argtypes = [C.c_int, C.c_int]
        L.fis_mask_detect_smem.restype = C.c_longlong
        L.fis_gemm_kernel_kind.argtypes = [C.POINTER(GemmArgs)]
        L.fis_gemm_kernel_kind.restype = C.c_int
        L.fis_gemm_big_launch_count.restype = C.c_longlong
        L.fis_gemm_pair_launch_count.restype = C.c_longlong
        L.fis_gn_launches.argtypes = [C.POINTER(GnApplyArgs)]
        L.fis_gn_launches.restype = C.c_int
        L.fis_trace_launches.argtypes = [C.c_void_p]
        L.fis_trace_launches.restype = C.c_int
        L.fis_attn_ws_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
        L.fis_attn_ws_bytes.restype = C.c_longlong
        L.fis_attn_launches.argtypes = [C.POINTER(AttnArgs)]
        L.fis_attn_launches.restype = C.c_int
        L.fis_abi_version.restype = C.c_int
        L.fis_last_error.restype = C.c_char_p
        L.fis_device_sm_count.restype = C.c_int
        if L.fis_abi_version() != 1:
            raise RuntimeError("libfisedit ABI mismatch")
        _lib = L
    return _lib


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2305_17423_b200 needs a CUDA device (B200); there is no CPU fallback")
    lib()


def stream_ptr():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def call(name, args):
    st = getattr(lib(), name)(C.byref(args), stream_ptr())
    if st == 0:
        return
    if st == 2:
        raise CacheMissError("?", "?", f"{name}: required cached tensor missing")
    if st in (1, 3):
        raise ContractViolation(f"{name}: invalid or unsupported arguments (status {st})")
    raise RuntimeError(f"{name}: CUDA launch failed: {lib().fis_last_error().decode()}")


def dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise ContractViolation(f"unsupported dtype {t.dtype}")


def ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())

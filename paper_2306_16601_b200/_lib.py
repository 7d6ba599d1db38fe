"""ctypes binding of libsparseinfer_b200.so (include/sparseinfer_b200.h).

This is the product's only route to compute: there is no CPU fallback.  If
the library is missing or fails to load, ``lib()`` raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

SI_OK, SI_EINVAL, SI_EFORMAT, SI_ECUDA, SI_EUNSUPPORTED, SI_ENOSPACE = range(6)
KERNELS = {"auto": 0, "gather": 1, "tc": 2, "ref": 3, "sp": 4, "ws": 5}
LAYOUTS = {"kn": 0, "nk": 1}

_vp, _i32, _i64, _u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64


class SiWeight(ctypes.Structure):
    _fields_ = [("rows", _i32), ("cols", _i32), ("logical_rows", _i32),
                ("group_ptr", _vp), ("idx", _vp), ("vals", _vp)]


class SiProgram(ctypes.Structure):
    _fields_ = [("m", _i32), ("scale_in", _vp), ("a_zp", _i32), ("n_ops", _i32), ("ops", _vp),
                ("fparams", _vp), ("iparams", _vp), ("n_luts", _i32), ("luts", _vp),
                ("n_chans", _i32), ("chans", _vp), ("out_dtype", _i32), ("n_sides", _i32)]


class SiPlanInfo(ctypes.Structure):
    _fields_ = [("m", _i32), ("k", _i32), ("groups", _i32), ("out_dtype", _i32), ("epi_mode", _i32),
                ("exact", _i32), ("nnz_blocks", _i64), ("padded_blocks", _i64),
                ("image_bytes", _u64)]


ABI_VERSION = 2   # include/sparseinfer_b200.h SI_ABI_VERSION


class SiHostJob(ctypes.Structure):
    _fields_ = [("host_image", _vp), ("dev_image", _vp), ("x_host", _vp), ("x_layout", _i32), ("ldx", _i64),
                ("n", _i64), ("out_host", _vp), ("ldo", _i64), ("sides_host", _vp)]


_lib = None


def lib():
    """Load (building in-tree first if this is a source checkout with nvcc)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SI_LIB") or _build.LIB_PATH   # SI_LIB: experiment builds only
    if not os.path.exists(path):
        try:
            path = _build.build()
        except Exception as e:  # no nvcc on this host and no prebuilt library
            raise RuntimeError(f"sparseinfer_b200 native library unavailable: {e}") from e
    L = ctypes.CDLL(path)
    L.si_abi_version.restype = _i32
    L.si_last_error.restype = ctypes.c_char_p
    L.si_plan_image_size.argtypes = [ctypes.POINTER(SiWeight), ctypes.POINTER(SiProgram),
                                     ctypes.POINTER(_u64)]
    L.si_plan_image_build.argtypes = [ctypes.POINTER(SiWeight), ctypes.POINTER(SiProgram), _vp, _vp, _u64]
    L.si_plan_info_get.argtypes = [_vp, ctypes.POINTER(SiPlanInfo)]
    L.si_plan_image_validate.argtypes = [_vp, _u64]
    L.si_spmm_workspace_size.argtypes = [_vp, _i64, _i32, _i32, ctypes.POINTER(_u64)]
    L.si_spmm_launch_count.argtypes = [_vp, _i64, _i32, _i32]
    L.si_spmm.argtypes = [_vp, _vp, _vp, _i32, _i64, _i64, _vp, _vp, _i64, _vp, _u64, _i32, _vp]
    L.si_spmm_host_workspace_size.argtypes = [_vp, _i64, _i32, _i32, ctypes.POINTER(_u64)]
    L.si_spmm_host.argtypes = [_vp, _vp, _vp, _i32, _i64, _i64, _vp, _vp, _i64, _vp, _u64, _i64, _i32, _vp]
    L.si_spmm_host_batch_workspace_size.argtypes = [ctypes.POINTER(SiHostJob), _i32, _i64, ctypes.POINTER(_u64)]
    L.si_spmm_host_batch.argtypes = [ctypes.POINTER(SiHostJob), _i32, _vp, _u64, _i64, _i32, _vp]
    L.si_softmax_rows_f32.argtypes = [_vp, _vp, _i64, _i64, _vp]
    L.si_layer_norm_f32.argtypes = [_vp, _vp, _vp, ctypes.c_double, _vp, _i64, _i64, _vp]
    L.si_bmm_f32.argtypes = [_vp, _vp, _vp] + [_i64] * 14 + [_i32, ctypes.c_float, _vp]
    L.si_quantize_f32.argtypes = [_vp, _i64, ctypes.c_float, _i32, _i32, _i32, _vp, _vp]
    L.si_attention_f32.argtypes = [_vp, _vp] + [_i64] * 6 + [ctypes.c_float, _vp]
    for f in ("si_plan_image_size", "si_plan_image_build", "si_plan_info_get", "si_plan_image_validate",
              "si_spmm_workspace_size", "si_spmm_launch_count", "si_spmm",
              "si_spmm_host_workspace_size", "si_spmm_host",
              "si_spmm_host_batch_workspace_size", "si_spmm_host_batch",
              "si_softmax_rows_f32", "si_layer_norm_f32", "si_bmm_f32", "si_quantize_f32", "si_attention_f32"):
        getattr(L, f).restype = _i32
    if L.si_abi_version() != ABI_VERSION:
        raise RuntimeError("libsparseinfer_b200 ABI version mismatch")
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc == SI_OK:
        return
    msg = lib().si_last_error().decode(errors="replace")
    if rc == SI_EFORMAT:
        from .sparse import SparseFormatError
        raise SparseFormatError(msg)
    if rc == SI_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed ({rc}): {msg}")


def ptr(a: np.ndarray | None):
    return None if a is None or a.size == 0 else a.ctypes.data_as(_vp)


class HostWeight:
    """Contiguous numpy views of a Sparse4x1Weight + the ctypes struct."""

    def __init__(self, sw):
        self.group_ptr = np.ascontiguousarray(sw.group_ptr, np.int32)
        self.idx = np.ascontiguousarray(sw.idx, np.int32)
        self.vals = np.ascontiguousarray(sw.vals, np.int8)
        self.s = SiWeight(int(sw.rows), int(sw.cols), int(sw.logical_rows), ptr(self.group_ptr),
                          ptr(self.idx), ptr(self.vals))


class HostProgram:
    """Contiguous numpy views of an EpilogueProgram + the ctypes struct."""

    def __init__(self, prog):
        self.scale_in = np.ascontiguousarray(prog.scale_in, np.float32)
        self.ops = np.ascontiguousarray(prog.ops, np.int32)
        self.fparams = np.ascontiguousarray(prog.fparams, np.float32)
        self.iparams = np.ascontiguousarray(prog.iparams, np.int32).reshape(-1)
        self.luts = np.ascontiguousarray(prog.luts, np.uint8).reshape(-1)
        self.chans = np.ascontiguousarray(prog.chans, np.float32).reshape(-1)
        dt = prog.out_dtype
        code = {"f32": 0, "s8": 1, "u8": 2, "s32": 3}[getattr(dt, "value", dt)]
        self.s = SiProgram(int(self.scale_in.shape[0]), ptr(self.scale_in), int(prog.a_zp),
                           int(self.ops.shape[0]), ptr(self.ops), ptr(self.fparams), ptr(self.iparams),
                           int(self.luts.size // 256), ptr(self.luts),
                           int(self.chans.size // max(1, self.scale_in.shape[0])), ptr(self.chans),
                           code, int(getattr(prog, "n_sides", 0)))

"""ctypes binding of the C ABI in ``include/lpradon_gpu.h``.

The shared library is built in-tree (``paper_1506_00014_b200/build.py``);
loading fails loudly when it is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

LIB_PATH = os.environ.get("LPR_GPU_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                         "liblpradon_gpu.so")

LPR_OK, LPR_ERR_ARG, LPR_ERR_CUDA, LPR_ERR_OOM = 0, 1, 2, 3


class Geometry(ctypes.Structure):
    """Mirror of ``lpr_geometry`` / ``lpr::GeometryPlan`` (geometry.hpp:23-43)."""

    _fields_ = [(n, ctypes.c_int) for n in ("N", "M", "n_theta", "nts", "n_rho", "refine")] + [
        (n, ctypes.c_double) for n in ("beta", "a_R", "a_r", "log_ar", "dtheta_p", "dtheta_lp", "drho", "ds")]

    def __repr__(self):
        return ("Geometry(" + ", ".join(f"{n}={getattr(self, n)!r}" for n, _ in self._fields_) + ")")


EXPORTS = {
    "lpr_geometry_make": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(Geometry)]),
    "lpr_smooth_n_rho": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "lpr_spectrum_quadrature": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.c_int, ctypes.c_void_p]),
    "lpr_gpu_plan_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(Geometry), ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "lpr_gpu_plan_create_ex": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(Geometry), ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_int, ctypes.c_uint,
                                              ctypes.POINTER(ctypes.c_void_p)]),
    "lpr_gpu_plan_destroy": (None, [ctypes.c_void_p]),
    "lpr_gpu_radon": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                     ctypes.c_void_p]),
    "lpr_gpu_backproject": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                           ctypes.c_void_p]),
    "lpr_gpu_radon_transpose": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                               ctypes.c_void_p]),
    "lpr_gpu_radon_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "lpr_gpu_backproject_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "lpr_gpu_radon_transpose_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                    ctypes.c_int]),
    "lpr_gpu_profile_stages": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_char_p)]),
    "lpr_gpu_filter": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.c_void_p]),
    "lpr_gpu_fbp": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                   ctypes.c_void_p]),
    "lpr_gpu_fbp_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "lpr_gpu_profile_stages_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                                   ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                                   ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_char_p)]),
    "lpr_gpu_lp_convolve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "lpr_gpu_lp_convolve_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_int]),
    "lpr_gpu_radon_backproject_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                      ctypes.c_void_p, ctypes.c_int]),
    "lpr_gpu_launch_count": (ctypes.c_longlong, [ctypes.c_void_p]),
    "lpr_gpu_fft_count": (ctypes.c_longlong, [ctypes.c_void_p]),
    "lpr_gpu_last_error": (ctypes.c_char_p, []),
    "lpr_gpu_spectrum_quadrature": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "lpr_spectrum_cache_dir": (ctypes.c_int, [ctypes.c_char_p]),
    "lpr_spectrum_cache_hits": (ctypes.c_longlong, []),
    "lpr_spectrum_cache_stores": (ctypes.c_longlong, []),
    "lpr_gpu_sensitivity": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "lpr_gpu_sensitivity_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "lpr_gpu_em": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "lpr_gpu_em_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_void_p]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == LPR_OK:
        return
    msg = lib().lpr_gpu_last_error().decode(errors="replace")
    if rc == LPR_ERR_ARG:
        raise ValueError(msg)  # the reference's std::invalid_argument
    if rc == LPR_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(msg)

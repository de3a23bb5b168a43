"""ctypes binding of the C ABI in ``include/hexbench_b200.h``.

The library is built in-tree (``build.py``) and loaded from the package
directory.  There is no fallback: if the library is missing or fails to load,
every operator call raises ``NativeLibraryError``.
"""

import ctypes
import os

from .mesh import DegenerateGeometryError

HERE = os.path.dirname(os.path.abspath(__file__))
# HX_LIB_PATH selects an alternative build (tuning experiments only)
LIB_PATH = os.environ.get("HX_LIB_PATH", os.path.join(HERE, "libhexbench_b200.so"))

HX_OK, HX_EINVAL, HX_ENONFINITE, HX_EDEGENERATE, HX_ECUDA, HX_ENOMEM = range(6)
HX_BP1, HX_BP35, HX_BP3 = 10, 35, 30
HX_FLAG_NONFINITE, HX_FLAG_DEGENERATE = 1, 2
HX_HOST_OVERLAP = 1  # hx_apply_host_ex: back-to-back pipelining (include/hexbench_b200.h)

# every symbol include/hexbench_b200.h declares, with its ctypes signature
_c = ctypes
_P = _c.c_void_p
_D = _c.POINTER(_c.c_double)
SIGNATURES = {
    "hx_plan_create": (_c.c_int, [_c.c_int, _c.c_int, _c.c_double, _P, _P, _P, _P,
                                  _c.POINTER(_P)]),
    "hx_plan_destroy": (None, [_P]),
    "hx_plan_factor_layout": (_c.c_int, [_P, _c.POINTER(_c.c_int),
                                         _c.POINTER(_c.c_int64), _c.POINTER(_c.c_int64)]),
    "hx_geometric_factors": (_c.c_int, [_P, _P, _c.c_int64, _c.c_int, _P, _P, _P]),
    "hx_repack_factors": (_c.c_int, [_P, _P, _c.c_int64, _P, _c.c_int, _P]),
    "hx_apply": (_c.c_int, [_P, _P, _P, _P, _c.c_int64, _P, _P]),
    "hx_apply_range": (_c.c_int, [_P, _P, _P, _P, _c.c_int64, _c.c_int64, _P, _P]),
    "hx_apply_host_workspace": (_c.c_int64, [_P, _c.c_int64]),
    "hx_apply_host": (_c.c_int, [_P, _P, _P, _P, _c.c_int64, _c.c_int64, _P, _P, _P]),
    "hx_apply_host_ex": (_c.c_int, [_P, _P, _P, _P, _c.c_int64, _c.c_int64, _P, _P, _c.c_uint,
                                    _P]),
    "hx_apply_host_staging_bytes": (_c.c_int64, [_P, _c.c_int64]),
    "hx_apply_host_staged": (_c.c_int, [_P, _P, _P, _P, _c.c_int64, _c.c_int64, _P, _P, _P,
                                        _P]),
    "hx_check_finite": (_c.c_int, [_P, _c.c_int64, _P, _P]),
    "hx_host_all_finite": (_c.c_int, [_P, _c.c_int64]),
    "hx_plan_kernel_shape": (_c.c_int, [_P, _c.POINTER(_c.c_int), _c.POINTER(_c.c_int),
                                        _c.POINTER(_c.c_int)]),
    "hx_measure_smem_bandwidth": (_c.c_int, [_c.POINTER(_c.c_double), _P]),
    "hx_apply_baseline_workspace": (_c.c_int64, [_P, _c.c_int64]),
    "hx_apply_baseline": (_c.c_int, [_P, _P, _P, _P, _c.c_int64, _P, _P, _P]),
    "hx_interp_elements": (_c.c_int, [_c.c_int, _P, _c.c_int, _P, _P, _c.c_int64, _P, _P]),
    "hx_energy_partials": (_c.c_int64, []),
    "hx_apply_energy": (_c.c_int, [_P, _P, _P, _P, _c.c_int64, _P, _c.c_int64, _P, _P, _P]),
    "hx_apply_energy_dir": (_c.c_int, [_P, _P, _P, _P, _P, _P, _P, _c.c_int64, _P, _c.c_int64,
                                       _P, _P, _P]),
    "hx_dot": (_c.c_int, [_P, _P, _c.c_int64, _P, _c.c_int64, _P, _P]),
    "hx_cg_update": (_c.c_int, [_P, _P, _P, _P, _c.c_int64, _P, _P, _P, _c.c_int64, _P, _P]),
    "hx_cg_direction": (_c.c_int, [_P, _P, _c.c_int64, _P, _P, _P]),
    "hx_dss": (_c.c_int, [_P, _P, _c.c_int, _c.c_int, _c.c_int, _c.c_int64, _c.c_int64,
                          _c.c_int64, _P]),
    "hx_dot_dss": (_c.c_int, [_P, _P, _c.c_int, _c.c_int, _c.c_int64, _c.c_int64, _P,
                              _c.c_int64, _P, _P]),
    "hx_dss_inplace": (_c.c_int, [_P, _c.c_int, _c.c_int, _c.c_int64, _c.c_int64, _P]),
    "hx_cg_update_assembled": (_c.c_int, [_P, _P, _P, _P, _c.c_int, _c.c_int, _c.c_int,
                                          _c.c_int64, _c.c_int64, _c.c_int64, _c.c_int64,
                                          _P, _P, _P, _c.c_int64, _P, _P]),
    "hx_strerror": (_c.c_char_p, [_c.c_int]),
    "hx_device_ok": (_c.c_int, []),
}


class NativeLibraryError(RuntimeError):
    """The sm_100a library is missing or unusable (there is no CPU fallback)."""


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not built; run `python -m paper_1711_00903_b200.build` "
                "(or __graft_entry__.build()) -- there is no CPU fallback")
        try:
            handle = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status, what="native call"):
    if status == HX_OK:
        return
    msg = lib().hx_strerror(status).decode()
    if status in (HX_EINVAL, HX_ENONFINITE):
        raise ValueError(f"{what}: {msg}")
    if status == HX_EDEGENERATE:
        raise DegenerateGeometryError(f"{what}: {msg}")
    if status == HX_ENOMEM:
        raise MemoryError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


def ptr(arr):
    """Raw address of a numpy array or torch tensor (None -> NULL)."""
    if arr is None:
        return None
    if hasattr(arr, "data_ptr"):
        return arr.data_ptr()
    return arr.ctypes.data


class Plan:
    """Owns one ``hx_plan``; immutable after creation."""

    def __init__(self, bp_id, degree, lam, interp, diff, nodes, weights):
        import numpy as np

        keep = []

        def as_c(a):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            return a.ctypes.data

        handle = ctypes.c_void_p()
        check(lib().hx_plan_create(bp_id, degree, float(lam), as_c(interp), as_c(diff),
                                   as_c(nodes), as_c(weights), ctypes.byref(handle)),
              "hx_plan_create")
        self.handle = handle
        ns, sst, est = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
        check(lib().hx_plan_factor_layout(handle, ctypes.byref(ns), ctypes.byref(sst),
                                          ctypes.byref(est)))
        self.n_slots, self.slot_stride, self.elem_stride = ns.value, sst.value, est.value
        epb, nt, sm = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(lib().hx_plan_kernel_shape(handle, ctypes.byref(epb), ctypes.byref(nt),
                                         ctypes.byref(sm)))
        self.elements_per_tile, self.threads, self.smem_bytes = epb.value, nt.value, sm.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.hx_plan_destroy(h)
            self.handle = None

"""CPU: the C-ABI library loads, exports every symbol include/hexbench_b200.h
declares, and validates plans like make_operator does -- no device work."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1711_00903_b200 import _native, basis, quadrature

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "hexbench_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hx_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 12
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_native.SIGNATURES), "ctypes table out of sync with the header"


def test_library_is_sm100a_only():
    """The shared object carries sm_100a SASS (no PTX/JIT fallback)."""
    import subprocess
    res = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    assert "sm_100a" in res.stdout
    arches = set(re.findall(r"sm_\d+a?", res.stdout))
    assert arches == {"sm_100a"}, arches


def _plan_args(bp, deg):
    if bp == _native.HX_BP35:
        rule = quadrature.gll_rule(deg + 1)
        return None, basis.diff_matrix_gll(deg).entries, rule
    rule = quadrature.gl_rule(deg + 2)
    diff = None if bp == _native.HX_BP1 else basis.diff_matrix_gl(deg).entries
    return basis.interp_matrix(deg).entries, diff, rule


@pytest.mark.parametrize("bp", [_native.HX_BP1, _native.HX_BP35, _native.HX_BP3])
@pytest.mark.parametrize("deg", [1, 2, 7, 15])
def test_plan_layout_and_shape(bp, deg):
    interp, diff, rule = _plan_args(bp, deg)
    plan = _native.Plan(bp, deg, 1.0, interp, diff, rule.nodes, rule.weights)
    q3 = rule.n ** 3
    assert plan.slot_stride == q3 + (q3 & 1)
    assert plan.n_slots == (1 if bp == _native.HX_BP1 else 7)
    assert plan.elem_stride == plan.n_slots * plan.slot_stride
    assert plan.elem_stride * 8 % 16 == 0  # every element slab 16-byte aligned
    assert plan.threads % 32 == 0 and plan.threads <= 1024
    assert 0 < plan.smem_bytes <= 227 * 1024
    lines = (deg + 1) ** 2 if bp == _native.HX_BP35 else (deg + 2) ** 2
    if bp == _native.HX_BP1:  # BP1.0 CTAs may walk several lines per thread
        assert plan.elements_per_tile >= 1
    else:                     # BP3.5 / BP3.0 keep one line per thread
        assert plan.elements_per_tile * lines <= plan.threads


def test_plan_create_rejects_bad_arguments():
    lib = _native.lib()
    interp, diff, rule = _plan_args(_native.HX_BP3, 3)
    arrs = [np.ascontiguousarray(a) for a in (interp, diff, rule.nodes, rule.weights)]
    ptrs = [a.ctypes.data for a in arrs]
    h = ctypes.c_void_p()
    assert lib.hx_plan_create(99, 3, 0.0, *ptrs, ctypes.byref(h)) == _native.HX_EINVAL
    assert lib.hx_plan_create(_native.HX_BP3, 0, 0.0, *ptrs, ctypes.byref(h)) == _native.HX_EINVAL
    assert lib.hx_plan_create(_native.HX_BP3, 16, 0.0, *ptrs, ctypes.byref(h)) == _native.HX_EINVAL
    assert lib.hx_plan_create(_native.HX_BP3, 3, -1.0, *ptrs, ctypes.byref(h)) == _native.HX_EINVAL
    assert lib.hx_plan_create(_native.HX_BP3, 3, float("nan"), *ptrs,
                              ctypes.byref(h)) == _native.HX_EINVAL
    assert lib.hx_plan_create(_native.HX_BP3, 3, 0.0, None, ptrs[1], ptrs[2], ptrs[3],
                              ctypes.byref(h)) == _native.HX_EINVAL
    assert lib.hx_plan_create(_native.HX_BP3, 3, 0.0, *ptrs, None) == _native.HX_EINVAL
    # matrices that are not (anti-)centro-symmetric would be mis-applied by the
    # folded kernels: rejected
    bad_i = arrs[0].copy()
    bad_i[0, 0] += 1e-3
    assert lib.hx_plan_create(_native.HX_BP3, 3, 0.0, bad_i.ctypes.data, *ptrs[1:],
                              ctypes.byref(h)) == _native.HX_EINVAL
    bad_d = arrs[1].copy()
    bad_d[1, 2] += 1e-3
    assert lib.hx_plan_create(_native.HX_BP3, 3, 0.0, ptrs[0], bad_d.ctypes.data, *ptrs[2:],
                              ctypes.byref(h)) == _native.HX_EINVAL
    assert lib.hx_plan_create(_native.HX_BP3, 3, 0.5, *ptrs, ctypes.byref(h)) == _native.HX_OK
    # pointers to doubles must be 8-byte aligned (checked before any launch)
    assert lib.hx_apply(h, 8, 16, 3, 1, None, None) == _native.HX_EINVAL
    assert lib.hx_apply(h, None, None, None, -1, None, None) == _native.HX_EINVAL
    assert lib.hx_apply(h, None, None, None, 4, None, None) == _native.HX_EINVAL
    assert lib.hx_apply(None, None, None, None, 0, None, None) == _native.HX_EINVAL
    lib.hx_plan_destroy(h)
    lib.hx_plan_destroy(None)


def test_strerror_and_exception_mapping():
    lib = _native.lib()
    assert lib.hx_strerror(_native.HX_OK) == b"success"
    assert b"non-finite" in lib.hx_strerror(_native.HX_ENONFINITE)
    with pytest.raises(ValueError):
        _native.check(_native.HX_EINVAL)
    with pytest.raises(ValueError):
        _native.check(_native.HX_ENONFINITE)
    from paper_1711_00903_b200.mesh import DegenerateGeometryError
    with pytest.raises(DegenerateGeometryError):
        _native.check(_native.HX_EDEGENERATE)
    with pytest.raises(RuntimeError):
        _native.check(_native.HX_ECUDA)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(_native.NativeLibraryError):
        _native.lib()


def test_host_finite_scan_runs_on_host_threads():
    """hx_host_all_finite (the up-front np.isfinite scan of operators.py:317,
    for apply_operator(..., out=)) is host-only: no GPU needed."""
    x = np.random.default_rng(0).standard_normal(3_000_001)
    lib = _native.lib()
    assert lib.hx_host_all_finite(x.ctypes.data, x.size) == 1
    assert lib.hx_host_all_finite(x.ctypes.data, 0) == 1
    for pos in (0, 1_500_000, 3_000_000):
        for v in (np.inf, -np.inf, np.nan):
            y = x.copy()
            y[pos] = v
            assert lib.hx_host_all_finite(y.ctypes.data, y.size) == 0

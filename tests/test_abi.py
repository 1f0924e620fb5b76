"""The C-ABI library: loads without a GPU, exports every declared symbol,
validates arguments before touching CUDA (no compute calls here)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO

import paper_1601_00072_b200 as pkg
from paper_1601_00072_b200 import _lib


def header_symbols():
    text = open(os.path.join(REPO, "include", "fcm_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(fcm_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"


def test_abi_version_and_status_strings():
    L = _lib.lib()
    assert L.fcm_abi_version() == 1
    assert L.fcm_status_string(_lib.FCM_E_DEGENERATE) == b"degenerate cluster"
    assert L.fcm_status_string(99) == b"unknown status"


def test_argument_validation_is_host_side():
    L = _lib.lib()
    h = ctypes.c_void_p()
    # c < 2, n < c, bad kind, bad shard count: rejected before any CUDA call
    assert L.fcm_plan_create(ctypes.byref(h), 10, 1, 0, 1, None) == _lib.FCM_E_ARG
    assert L.fcm_plan_create(ctypes.byref(h), 2, 3, 0, 1, None) == _lib.FCM_E_ARG
    assert L.fcm_plan_create(ctypes.byref(h), 100, 3, 7, 1, None) == _lib.FCM_E_ARG
    assert L.fcm_plan_create(ctypes.byref(h), 100, 3, 0, 3, None) == _lib.FCM_E_ARG
    assert L.fcm_plan_create(ctypes.byref(h), 100, 33, 0, 1, None) == _lib.FCM_E_ARG
    assert L.fcm_plan_create_rank(ctypes.byref(h), 100, 3, 0, 0, 2, 2, None) == _lib.FCM_E_ARG
    assert L.fcm_set_option(None, 1, 8) == _lib.FCM_E_ARG
    assert L.fcm_max_abs_diff(None, None, 4, 0, None) == _lib.FCM_E_ARG


def test_no_gpu_means_loud_failure_not_fallback():
    cnt = ctypes.c_int32(-1)
    st = _lib.lib().fcm_device_count(ctypes.byref(cnt))
    if st == _lib.FCM_OK and cnt.value > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(pkg.DeviceError):
        pkg.run_fcm_gpu(pkg.GrayImage(4, 1, [1.0, 2.0, 3.0, 4.0]), pkg.FcmConfig(c=2))


def test_pixel_kind_selection():
    # host-only: fcm_narrow_pixels needs no GPU
    k, a = pkg.pixel_kind(np.array([0.0, 17.0, 255.0]))
    assert k == _lib.FCM_X_U8 and a.dtype == np.uint8 and a.tolist() == [0, 17, 255]
    k, a = pkg.pixel_kind(np.array([0.0, 256.0, 65535.0]))
    assert k == _lib.FCM_X_U16 and a.dtype == np.uint16 and a.tolist() == [0, 256, 65535]
    for bad in ([0.5, 2.0], [0.0, 65536.0], [1.0, np.nan], [1.0, -1.0], [1.0, np.inf]):
        k, a = pkg.pixel_kind(np.array(bad))
        assert k == _lib.FCM_X_F64 and a.dtype == np.float64
    k, a = pkg.pixel_kind(np.array([3, 200], dtype=np.uint16))  # 16-bit raster, 8-bit values
    assert k == _lib.FCM_X_U8 and a.dtype == np.uint8
    k, a = pkg.pixel_kind(np.array([3, 300], dtype=np.uint16))
    assert k == _lib.FCM_X_U16 and a.dtype == np.uint16


def test_narrow_pixels_large_multithreaded():
    rng = np.random.default_rng(3)
    x = rng.integers(0, 256, 3_000_001).astype(np.float64)
    k, a = pkg.pixel_kind(x)
    assert k == _lib.FCM_X_U8 and np.array_equal(a, x.astype(np.uint8))
    x[2_999_999] = 255.5  # one bad value in the last thread's block
    assert pkg.pixel_kind(x)[0] == _lib.FCM_X_F64
    x[2_999_999] = 4095.0
    k, a = pkg.pixel_kind(x)
    assert k == _lib.FCM_X_U16 and np.array_equal(a, x.astype(np.uint16))


def test_product_path_does_not_import_oracle():
    import sys
    import subprocess
    code = ("import sys; sys.path.insert(0, %r); import paper_1601_00072_b200 as p; "
            "import paper_1601_00072_b200.engine; "
            "bad=[m for m in sys.modules if m.startswith('oracle')]; assert not bad, bad") % REPO
    subprocess.run([sys.executable, "-c", code], check=True)


def test_pixel_kind_staging_buffer():
    """run_fcm_gpu / _iterate narrow float64 pixels into this thread's reused
    staging buffer (page-locked when a GPU is present, pageable otherwise):
    same kind and values as a fresh array, and the buffer is reused, not
    reallocated, for a same-size or smaller image."""
    from paper_1601_00072_b200 import engine
    rng = np.random.default_rng(3)
    x = rng.integers(0, 256, 1_000_003).astype(np.float64)
    k0, a0 = pkg.pixel_kind(x)
    k1, a1 = engine.pixel_kind(x, staging=True)
    assert k0 == k1 == _lib.FCM_X_U8 and np.array_equal(a0, a1)
    base = engine._scratch.buf
    k2, a2 = engine.pixel_kind(x[:500_000] * 200.0, staging=True)  # 16-bit values now
    assert k2 == _lib.FCM_X_U16 and np.array_equal(a2, (x[:500_000] * 200).astype(np.uint16))
    assert engine._scratch.buf is base

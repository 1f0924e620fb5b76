"""ctypes binding of libfcm_b200.so (declared in include/fcm_b200.h).

The library is built in-tree by __graft_entry__.build() (make -C
paper_1601_00072_b200/csrc).  There is no fallback: if the library is missing
or no GPU is usable, every compute call raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DegenerateClusterError, DeviceError, FcmError, InvalidConfigError

LIB_PATH = os.environ.get("FCM_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfcm_b200.so")

FCM_OK, FCM_E_ARG, FCM_E_CUDA, FCM_E_NCCL, FCM_E_DEGENERATE, FCM_E_STATE, FCM_E_NOMEM = range(7)
FCM_X_U8, FCM_X_U16, FCM_X_F64 = 0, 1, 2
FCM_OPT_BATCH, FCM_OPT_TIMING, FCM_OPT_GRID, FCM_OPT_KERNEL, FCM_OPT_GRAPH = 1, 2, 3, 4, 5
FCM_OPT_LOOP, FCM_OPT_L2, FCM_OPT_PROFILE, FCM_OPT_SEED_PASS = 6, 7, 8, 9
FCM_OPT_RECOMPUTE, FCM_OPT_DEBUG_DELAY, FCM_OPT_DEBUG_SHARED_PARTIALS, FCM_OPT_PEER_TIMEOUT_MS = 11, 12, 13, 14
FCM_OPT_DEBUG_SOLO_RANK = 15

# Every symbol the header declares (tests/test_abi.py checks the .so exports them).
SIGNATURES = {
    "fcm_abi_version": ([], ctypes.c_int),
    "fcm_status_string": ([ctypes.c_int], ctypes.c_char_p),
    "fcm_device_count": ([ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
    "fcm_plan_create": ([ctypes.POINTER(ctypes.c_void_p), ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                         ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
    "fcm_plan_create_rank": ([ctypes.POINTER(ctypes.c_void_p), ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                              ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p], ctypes.c_int),
    "fcm_nccl_unique_id": ([ctypes.c_void_p], ctypes.c_int),
    "fcm_label_confusion": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p], ctypes.c_int),
    "fcm_mask_overlap": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "fcm_mailbox_handle": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "fcm_connect_peers": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32], ctypes.c_int),
    "fcm_geometry": ([ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                      ctypes.c_int32], ctypes.c_int),
    "fcm_plan_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "fcm_last_error": ([ctypes.c_void_p], ctypes.c_char_p),
    "fcm_set_option": ([ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64], ctypes.c_int),
    "fcm_plan_info": ([ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32], ctypes.c_int),
    "fcm_upload_pixels": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "fcm_init_membership": ([ctypes.c_void_p, ctypes.c_uint64], ctypes.c_int),
    "fcm_upload_membership": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "fcm_run": ([ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_void_p,
                 ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                 ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
    "fcm_download": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "fcm_download_table": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32],
                           ctypes.c_int),
    "fcm_last_timing": ([ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int32], ctypes.c_int),
    "fcm_delta_trace": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32], ctypes.c_int),
    "fcm_result_table": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "fcm_narrow_pixels": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32],
                          ctypes.c_int),
    "fcm_last_profile": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int32),
                          ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
    "fcm_host_register": ([ctypes.c_void_p, ctypes.c_int64], ctypes.c_int),
    "fcm_host_unregister": ([ctypes.c_void_p], ctypes.c_int),
    "fcm_fill_membership_random": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64,
                                    ctypes.c_int32], ctypes.c_int),
    "fcm_update_centers": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                            ctypes.c_double, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
    "fcm_update_membership": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                               ctypes.c_int32, ctypes.c_double, ctypes.c_int32], ctypes.c_int),
    "fcm_objective": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                       ctypes.c_double, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "fcm_max_abs_diff": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                          ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "fcm_check_rcp": ([ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p], ctypes.c_int),
    "fcm_argmax_rows": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32],
                        ctypes.c_int),
}

_lib = None


def lib():
    """Load libfcm_b200.so once; raise DeviceError when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        if L.fcm_abi_version() != 1:
            raise DeviceError("libfcm_b200.so ABI mismatch")
        _lib = L
    return _lib


def check(status: int, plan=None, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception classes."""
    if status == FCM_OK:
        return
    detail = ""
    if plan:
        msg = lib().fcm_last_error(plan)
        detail = msg.decode() if msg else ""
    text = f"{what}: {lib().fcm_status_string(status).decode()}" + (f" ({detail})" if detail else "")
    if status == FCM_E_ARG:
        raise InvalidConfigError(text)
    if status in (FCM_E_CUDA, FCM_E_NCCL, FCM_E_NOMEM):
        raise DeviceError(text)
    raise FcmError(text)


def ptr(a) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


GEOMETRY_KEYS = ("n_local", "voxel0", "tile", "T", "M", "levels", "oct0", "noct", "tile0", "tiles_local")


def geometry(n: int, nranks: int = 1, rank: int = 0) -> dict:
    """Voxel range and tree geometry of one rank (host-only, no GPU)."""
    buf = (ctypes.c_int64 * len(GEOMETRY_KEYS))()
    check(lib().fcm_geometry(int(n), int(nranks), int(rank), buf, len(GEOMETRY_KEYS)), None, "fcm_geometry")
    return dict(zip(GEOMETRY_KEYS, list(buf)))

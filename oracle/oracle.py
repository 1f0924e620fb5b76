"""ctypes front-end of the CPU parity oracle (oracle/fcm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product package
(paper_1601_00072_b200), which has no CPU fallback.

Each wrapper restates the matching reference entry point:

* kernels    -> /root/reference/pkg/src/fcmseg/_kernels.pyx (line cited per function)
* sequential -> core._iterate / run_fcm_sequential (core.py:105-171)
* parallel   -> parallel._iterate (parallel.py:257-331)

The C library is built with the reference's own flags (-O2 -ffp-contract=off,
pkg/setup.py:14) and the same libm, so results are bit-identical to the
reference; tests/test_oracle.py pins that against tests/golden/ fixtures that
were produced by the reference itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_fcm.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64


def build() -> str:
    """Compile liboracle_fcm.so in place (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "fcm_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_splitmix64.argtypes = [_u64, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]
        L.oracle_fill_membership_random.argtypes = [_dp, _i64, _i64, _u64]
        L.oracle_fill_membership_random.restype = ctypes.c_int
        L.oracle_update_centers_linear.argtypes = [_dp, _dp, _dp, _i64, _i64, ctypes.c_double]
        L.oracle_update_centers_linear.restype = _i64
        L.oracle_update_membership_range.argtypes = [_dp, _dp, _dp, _i64, ctypes.c_double, _i64, _i64]
        L.oracle_center_terms_range.argtypes = [_dp, _dp, _dp, _dp, _i64, _i64, ctypes.c_double, _i64, _i64]
        L.oracle_block_reduce_range.argtypes = [_dp, _dp, _i64, _i64, _i64, _i64]
        L.oracle_block_reduce_range.restype = ctypes.c_int
        L.oracle_linear_sum.argtypes = [_dp, _i64]
        L.oracle_linear_sum.restype = ctypes.c_double
        L.oracle_objective_linear.argtypes = [_dp, _dp, _dp, _i64, _i64, ctypes.c_double]
        L.oracle_objective_linear.restype = ctypes.c_double
        L.oracle_objective_terms_range.argtypes = [_dp, _dp, _dp, _dp, _i64, ctypes.c_double, _i64, _i64]
        L.oracle_max_abs_diff.argtypes = [_dp, _dp, _i64, _i64]
        L.oracle_max_abs_diff.restype = ctypes.c_double
        L.oracle_argmax_rows.argtypes = [_dp, ctypes.POINTER(ctypes.c_int32), _i64, _i64]
        it_args = [_dp, _dp, _i64, _i64, ctypes.c_double, ctypes.c_double, _i64]
        L.oracle_iterate_sequential.argtypes = it_args + [
            _dp, _dp, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_int32)]
        L.oracle_iterate_sequential.restype = _i64
        L.oracle_iterate_parallel.argtypes = it_args + [
            _i64, _dp, _dp, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_int32)]
        L.oracle_iterate_parallel.restype = _i64
        L.oracle_last_deltas.argtypes = [_dp]
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(_dp)


class OracleDegenerate(ArithmeticError):
    """Oracle counterpart of DegenerateClusterError (core.py:121-123)."""

    def __init__(self, cluster):
        self.cluster = cluster
        super().__init__(f"cluster {cluster} has zero total membership weight")


def splitmix64(state: int):
    """_kernels.pyx:33-41."""
    s, z = _u64(), _u64()
    lib().oracle_splitmix64(state & 0xFFFFFFFFFFFFFFFF, ctypes.byref(s), ctypes.byref(z))
    return s.value, z.value


def fill_membership_random(n: int, c: int, seed: int) -> np.ndarray:
    """_kernels.pyx:44-69 (core.init_membership, core.py:24-39)."""
    u = np.empty(n * c, dtype=np.float64)
    lib().oracle_fill_membership_random(_p(u), n, c, seed & 0xFFFFFFFFFFFFFFFF)
    return u


def update_centers_linear(x, u, c: int, m: float):
    """_kernels.pyx:72-90; returns (v, dead) with dead == -1 when all centers exist."""
    x, u = _f64(x), _f64(u)
    v = np.zeros(c, dtype=np.float64)
    dead = lib().oracle_update_centers_linear(_p(x), _p(u), _p(v), x.shape[0], c, m)
    return v, int(dead)


def update_membership(x, v, m: float) -> np.ndarray:
    """_kernels.pyx:93-120 over the whole image."""
    x, v = _f64(x), _f64(v)
    u = np.empty(x.shape[0] * v.shape[0], dtype=np.float64)
    lib().oracle_update_membership_range(_p(x), _p(v), _p(u), v.shape[0], m, 0, x.shape[0])
    return u


def center_terms(x, u, c: int, j: int, m: float):
    """_kernels.pyx:123-134."""
    x, u = _f64(x), _f64(u)
    n = x.shape[0]
    num, den = np.empty(n), np.empty(n)
    lib().oracle_center_terms_range(_p(x), _p(u), _p(num), _p(den), c, j, m, 0, n)
    return num, den


def block_reduce(a, block_size: int) -> np.ndarray:
    """_kernels.pyx:137-165 over every block."""
    a = _f64(a)
    n = a.shape[0]
    nb = -(-n // (2 * block_size))
    out = np.empty(nb)
    lib().oracle_block_reduce_range(_p(a), _p(out), n, block_size, 0, nb)
    return out


def linear_sum(a) -> float:
    """_kernels.pyx:168-175."""
    a = _f64(a)
    return lib().oracle_linear_sum(_p(a), a.shape[0])


def objective_linear(x, u, v, m: float) -> float:
    """_kernels.pyx:178-191."""
    x, u, v = _f64(x), _f64(u), _f64(v)
    return lib().oracle_objective_linear(_p(x), _p(u), _p(v), x.shape[0], v.shape[0], m)


def max_abs_diff(a, b) -> float:
    """_kernels.pyx:211-220."""
    a, b = _f64(a), _f64(b)
    return lib().oracle_max_abs_diff(_p(a), _p(b), 0, a.shape[0])


def argmax_rows(u, c: int) -> np.ndarray:
    """_kernels.pyx:223-238."""
    u = _f64(u)
    n = u.shape[0] // c
    labels = np.empty(n, dtype=np.int32)
    lib().oracle_argmax_rows(_p(u), labels.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n, c)
    return labels


def last_deltas() -> np.ndarray:
    """(delta_{k-1}, delta_k) of the last two iterations of the last
    iterate()/run_fcm() call (max |u_k - u_{k-1}|, core.py:128-130)."""
    out = np.zeros(2)
    lib().oracle_last_deltas(_p(out))
    return out


def iterate(x, u0, c: int, m: float, epsilon: float, max_iters: int, engine="sequential",
            block_size: int = 128):
    """core._iterate (core.py:105-132) or parallel._iterate (parallel.py:257-331).

    Returns (v, u_final, iterations, trace, converged); raises OracleDegenerate
    where the reference raises DegenerateClusterError.
    """
    x = _f64(x)
    u = np.array(u0, dtype=np.float64, copy=True)
    n = x.shape[0]
    v = np.zeros(c)
    trace = np.zeros(max_iters)
    iters = _i64()
    conv = ctypes.c_int32()
    if engine == "sequential":
        st = lib().oracle_iterate_sequential(_p(x), _p(u), n, c, m, epsilon, max_iters,
                                             _p(v), _p(trace), ctypes.byref(iters), ctypes.byref(conv))
    elif engine == "parallel":
        st = lib().oracle_iterate_parallel(_p(x), _p(u), n, c, m, epsilon, max_iters, block_size,
                                           _p(v), _p(trace), ctypes.byref(iters), ctypes.byref(conv))
    else:
        raise ValueError(engine)
    if st < 0:
        raise MemoryError("oracle allocation failed")
    if st > 0:
        raise OracleDegenerate(int(st) - 1)
    k = iters.value
    return v, u, k, trace[:k].copy(), bool(conv.value)


def run_fcm(x, c: int, m: float = 2.0, epsilon: float = 0.005, max_iters: int = 500, seed: int = 0,
            initial_membership=None, engine="sequential"):
    """run_fcm_sequential / run_fcm_parallel (core.py:146-171, parallel.py:334-362) on raw pixels.

    Returns a dict with centers, membership (AoS f64), labels, iterations,
    objective_trace, converged.
    """
    x = _f64(x)
    n = x.shape[0]
    if n < c:
        raise ValueError(f"need at least {c} pixels for {c} clusters, got {n}")
    u0 = fill_membership_random(n, c, seed) if initial_membership is None else _f64(initial_membership)
    v, u, k, trace, conv = iterate(x, u0, c, m, epsilon, max_iters, engine)
    return {
        "centers": v,
        "membership": u,
        "labels": argmax_rows(u, c),
        "iterations": k,
        "objective_trace": trace,
        "converged": conv,
    }

"""The GPU engine inside the reference package itself (fcmseg).

`register(fcmseg)` applies the patches of INTEGRATION.md section 3 to an
imported reference package:

* `cli.ENGINES["gpu"]` (cli.py:23-26): `segment --engine gpu`;
* `bench.ENGINES` gains "gpu" (bench.py:22, enforced at :43-44), and
  `bench._timed_loop` (bench.py:49-59) times `_iterate` for it exactly as it
  times `core._iterate` -- u0 copied before the clock, the loop alone inside.

The engine hands back the reference's own result types (fcmseg.types), built
from the GPU arrays, so every reference consumer -- `write_pgm`'s isinstance
checks, `metrics`, the CLI printouts -- runs unchanged.  Nothing here imports
the reference; the caller passes the module in.
"""

from __future__ import annotations

import time

from .engine import _iterate, run_fcm_gpu


def reference_engine(types_mod):
    """run_fcm_gpu with the signature and result types of the reference's
    run_fcm_sequential / run_fcm_parallel (core.py:146-171, parallel.py:334-362)."""

    def run_fcm_gpu_reference(img, cfg, initial_membership=None):
        res = run_fcm_gpu(img, cfg, initial_membership=initial_membership)
        n, c = res.membership.n, res.membership.c
        return types_mod.FcmResult(
            centers=types_mod.ClusterCenters(res.centers.v),
            membership=types_mod.MembershipMatrix(n, c, res.membership.u),
            labels=types_mod.LabelMap(img.width, img.height, res.labels.labels, c),
            iterations=res.iterations,
            objective_trace=res.objective_trace,
            converged=res.converged,
        )

    run_fcm_gpu_reference.__name__ = "run_fcm_gpu"
    return run_fcm_gpu_reference


def register(fcmseg) -> None:
    """Register "gpu" in the reference's CLI and benchmark harness (idempotent)."""
    from importlib import import_module

    cli = import_module(fcmseg.__name__ + ".cli")
    bench = import_module(fcmseg.__name__ + ".bench")
    types_mod = import_module(fcmseg.__name__ + ".types")
    cli.ENGINES["gpu"] = reference_engine(types_mod)
    if "gpu" not in bench.ENGINES:
        bench.ENGINES = tuple(bench.ENGINES) + ("gpu",)
    if getattr(bench._timed_loop, "_fcm_gpu", False):
        return
    cpu_timed_loop = bench._timed_loop

    def _timed_loop(engine, x, u0, cfg, workers):
        if engine != "gpu":
            return cpu_timed_loop(engine, x, u0, cfg, workers)
        u = u0.copy()
        t0 = time.perf_counter()
        _, _, iterations, _, _ = _iterate(x, u, cfg)
        return time.perf_counter() - t0, iterations, None

    _timed_loop._fcm_gpu = True
    bench._timed_loop = _timed_loop

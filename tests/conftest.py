"""Shared test plumbing.

* registers the ``gpu`` marker (tests that need a B200; run with -m gpu),
* puts the repo root on sys.path (package, oracle/),
* restates the reference's synthetic-image generator
  (/root/reference/pkg/tests/conftest.py:9-22) so the GPU box can rebuild the
  same inputs without /root/reference, and loads the golden fixtures.
"""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


def mixture_pixels(n_pixels, n_groups, seed):
    """Well-separated integer intensity groups plus integer noise +-10."""
    rng = np.random.default_rng(seed)
    levels = np.linspace(25, 230, n_groups)
    base = rng.choice(levels, size=n_pixels)
    noise = rng.integers(-10, 11, size=n_pixels)
    return np.clip(np.rint(base + noise), 0.0, 255.0).astype(np.float64)


def small_fixture_params(count=10):
    """(n, c, m, image seed, init seed) of the reference's small_fixtures (conftest.py:58-67)."""
    return [(64 * (i + 1), 2 + i % 3, (1.5, 2.0, 3.0)[i % 3], 300 + i, 50 + i) for i in range(count)]


_cache = {}


def golden(name):
    if name not in _cache:
        _cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    return _cache[name]


def run_cases():
    """Names of the reference run records in tests/golden/runs.npz."""
    return [str(s) for s in golden("runs")["names"]]


def run_case(name):
    r = golden("runs")
    cfg = r[name + "_cfg"]
    return {
        "x": r[name + "_x"],
        "c": int(cfg[0]), "m": float(cfg[1]), "epsilon": float(cfg[2]),
        "max_iters": int(cfg[3]), "seed": int(cfg[4]),
        "v": r[name + "_v"], "labels": r[name + "_labels"], "trace": r[name + "_trace"],
        "iterations": int(r[name + "_iters"][0]), "converged": bool(r[name + "_conv"][0]),
        "u": r.get(name + "_u"),
    }

"""Synthetic BrainWeb-shaped inputs.

A nested-ellipsoid phantom with the tissue levels of the reference's test
phantom (background 15, CSF-like 70, GM-like 140, WM-like 215; reference
pkg/tests/conftest.py:25-37) plus per-slice integer noise U{-6..6}, stored
as uint8.  These are the configs of BASELINE.json:

* C1 = phantom_slice(181, 217)                    (39,277 px)
* C2 = phantom3d(181, 217, 181)                   (7,109,137 vox)
* C3 = enlarge_dataset(C1, 40 KB .. 1 MB)         (78,554 .. 1,178,310 px)
* C4 = phantom3d(512, 512, 512)                   (134,217,728 vox)
* C5 = phantom3d(1024, 1024, 512)                 (536,870,912 vox)
"""

from __future__ import annotations

import math

import numpy as np


def phantom_slice(nx: int, ny: int, zfrac: float = 0.0, seed: int = 5) -> np.ndarray:
    """One (ny, nx) uint8 slice at normalised depth zfrac."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:ny, 0:nx]
    r = np.sqrt(((yy - ny / 2) / ny) ** 2 + ((xx - nx / 2) / nx) ** 2 + zfrac ** 2)
    v = np.full((ny, nx), 15.0)
    v[r < 0.45] = 70.0
    v[r < 0.32] = 140.0
    v[r < 0.18] = 215.0
    v += rng.integers(-6, 7, size=(ny, nx))
    return np.clip(np.rint(v), 0, 255).astype(np.uint8)


def phantom3d(nx: int, ny: int, nz: int, seed: int = 5, out: np.ndarray | None = None) -> np.ndarray:
    """(nz, ny, nx) uint8 volume; slice z uses seed*100003 + z."""
    vol = np.empty((nz, ny, nx), dtype=np.uint8) if out is None else out
    for z in range(nz):
        vol[z] = phantom_slice(nx, ny, (z - nz / 2) / nz, seed=seed * 100003 + z)
    return vol


def enlarge(slice2d: np.ndarray, target_bytes: int) -> np.ndarray:
    """Whole-copy tiling to >= target_bytes pixels (reference imgio.py:196-217)."""
    h, w = slice2d.shape
    cur = h * w
    if target_bytes < cur:
        raise ValueError(f"target of {target_bytes} bytes is below the current size {cur}")
    tiles = -(-target_bytes // cur)
    if tiles == 1:
        return slice2d
    gx = math.isqrt(tiles)
    if gx * gx < tiles:
        gx += 1
    gy = -(-tiles // gx)
    return np.tile(slice2d, (gy, gx))


CONFIGS = {
    "C1": dict(shape=(217, 181), c=3, m=2.0),
    "C2": dict(shape=(181, 217, 181), c=3, m=2.0),
    "C4": dict(shape=(512, 512, 512), c=3, m=2.0),
    "C5": dict(shape=(512, 1024, 1024), c=8, m=1.5),
}

C3_SIZES = (40_000, 100_000, 200_000, 500_000, 1_000_000)


def make_config(name: str) -> np.ndarray:
    """Flat uint8 voxels for config C1/C2/C4/C5, or C3@<bytes>."""
    if name == "C1":
        return phantom_slice(181, 217).reshape(-1)
    if name == "C2":
        return phantom3d(181, 217, 181).reshape(-1)
    if name == "C4":
        return phantom3d(512, 512, 512).reshape(-1)
    if name == "C5":
        return phantom3d(1024, 1024, 512).reshape(-1)
    if name.startswith("C3@"):
        return enlarge(phantom_slice(181, 217), int(name[3:])).reshape(-1)
    raise KeyError(name)

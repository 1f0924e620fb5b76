"""Shard geometry and the fixed reduction tree, on the CPU.

* fcm_geometry (C ABI, host-only) partitions the voxels into tile-aligned
  contiguous rank ranges for N in {1,2,4,8}.
* The restated tree (tests/tree_model.py) gives a bit-identical global root
  for every N -- the property behind the GPU-count invariance test on the
  B200 (tests/test_gpu_parity.py) and the analogue of the reference's
  worker-count invariance (reference test_parallel.py:214-264).
* A world_size-2 gloo job exchanges rank roots like the NCCL path does
  (all-gather, rank-ordered combine) and reproduces the 1-rank root.
"""

import os

import numpy as np
import pytest

from conftest import REPO
from paper_1601_00072_b200._lib import geometry
from tree_model import combine_ranks, rank_root

SIZES = [3, 64, 1000, 39277, 78554, 1_178_310, 7_109_137, 134_217_728, 536_870_912]


@pytest.mark.parametrize("n", SIZES)
def test_geometry_partitions_voxels(n):
    g1 = geometry(n, 1, 0)
    tile = g1["tile"]
    assert g1["n_local"] == n and g1["voxel0"] == 0
    assert g1["T"] == -(-n // tile) and g1["T"] <= 8 * 32 ** 3
    assert 1 <= g1["levels"] <= 3 and g1["M"] <= 32 ** g1["levels"]
    assert g1["levels"] == 1 or g1["M"] > 32 ** (g1["levels"] - 1)
    assert tile >= 1024 and tile & (tile - 1) == 0
    for N in (2, 4, 8):
        covered = 0
        for r in range(N):
            g = geometry(n, N, r)
            assert g["tile"] == tile and g["T"] == g1["T"] and g["M"] == g1["M"]
            if g["n_local"]:
                assert g["voxel0"] == covered and g["voxel0"] % tile == 0
            covered += g["n_local"]
            assert g["noct"] == 8 // N and g["oct0"] == r * (8 // N)
        assert covered == n


def _partials(T, nf, seed=0):
    rng = np.random.default_rng(seed)
    p = rng.random((T, nf)) * 10.0 ** rng.integers(-3, 6, size=(T, nf))
    p[:, -1] = rng.random(T) * 1e-3  # max field
    return p


@pytest.mark.parametrize("n", [64, 39277, 7_109_137, 134_217_728])
def test_tree_root_is_rank_count_invariant(n):
    g1 = geometry(n, 1, 0)
    parts = _partials(g1["T"], 8, seed=n % 97)
    ref = rank_root(parts, g1)
    for N in (2, 4, 8):
        roots = [rank_root(parts, geometry(n, N, r)) for r in range(N)]
        got = combine_ranks(roots)
        assert got.tobytes() == ref.tobytes(), N


def _gloo_worker(rank, world, port, n, out_path):
    import torch
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.join(REPO, "tests"))
    sys.path.insert(0, REPO)
    from tree_model import combine_ranks as cr, rank_root as rr
    from paper_1601_00072_b200._lib import geometry as geo
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = geo(n, world, rank)
    parts = _partials(geo(n, 1, 0)["T"], 8, seed=5)
    mine = torch.from_numpy(rr(parts, g))
    gathered = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    total = cr([t.numpy() for t in gathered])
    if rank == 0:
        np.save(out_path, total)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_exchange_matches_single(tmp_path):
    import socket
    import torch.multiprocessing as mp
    n = 1_178_310
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "root.npy")
    mp.spawn(_gloo_worker, args=(2, port, n, out), nprocs=2, join=True)
    got = np.load(out)
    ref = rank_root(_partials(geometry(n, 1, 0)["T"], 8, seed=5), geometry(n, 1, 0))
    assert got.tobytes() == ref.tobytes()


@pytest.mark.parametrize("n,tile", [(39277, 1024), (78554, 1024), (235662, 2048), (628432, 4096),
                                    (1178310, 8192), (7109137, 8192), (134217728, 8192), (536870912, 32768)])
def test_tile_size_rule(n, tile):
    """Tile sizes chosen by base_geometry (DESIGN 3.4; measured with tools/tile_sweep.py):
    8192 voxels, halved while fewer than 100 tiles remain (>= 1024), doubled above 64 tiles per CTA."""
    g = geometry(n)
    assert g["tile"] == tile
    assert g["T"] <= 64 * 296 or tile == 1024


import pytest  # noqa: E402


@pytest.mark.parametrize("m", [5, 7, 9, 13, 17, 33, 65])
def test_butterfly_is_one_stride_tree_per_field(m):
    """The consumer warps' tile-end butterfly (fcm_device.cuh::bfly_level,
    restated in tree_model.bfly_reduce) leaves every field on exactly one lane,
    and each field's value is exactly the stride tree over its 32 lane values
    -- one fixed shape whichever lane adds, for every field count the kernels
    instantiate (2c+1 sum fields, c = 2..32)."""
    import random
    from tree_model import bfly_reduce, stride_tree
    rnd = random.Random(m)
    lanes = [[rnd.uniform(0, 1) * 2.0 ** rnd.randint(-30, 30) for _ in range(m)] for _ in range(32)]
    got = bfly_reduce(lanes)
    assert sorted(got) == list(range(m))
    for f in range(m):
        assert got[f] == stride_tree([lanes[i][f] for i in range(32)])

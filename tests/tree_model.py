"""Python restatement of the device reduction tree (test helper).

Mirrors fcm_device.cuh::warp_tree and fcm_kernels.cuh::tile_finish /
fcm_dispatch.cu::finalize_kernel so the CPU suite can prove, without a GPU,
that the tree shape makes the global root independent of the rank count.
"""

import numpy as np


def warp_tree(vals, is_max):
    x = list(vals) + [0.0] * (32 - len(vals))
    s = 1
    while s < 32:
        for i in range(0, 32, 2 * s):
            x[i] = max(x[i], x[i + s]) if is_max else x[i] + x[i + s]
        s *= 2
    return x[0]


def group_real_tiles(geo, o, g):
    lo = o * geo["M"] + g * 32
    hi = min(o * geo["M"] + min((g + 1) * 32, geo["M"]), geo["T"])
    return max(0, hi - lo)


def rank_root(tile_part, geo):
    """tile_part: (T, nf) float64 partials of ALL global tiles; geo: one rank's geometry."""
    T, M, gpo = geo["T"], geo["M"], geo["gpo"]
    nf = tile_part.shape[1]
    oct_roots = []
    for o in range(geo["oct0"], geo["oct0"] + geo["noct"]):
        groups = []
        for g in range(gpo):
            fields = []
            for f in range(nf):
                leaves = []
                for lane in range(32):
                    leaf = g * 32 + lane
                    real = leaf < M and o * M + leaf < T
                    leaves.append(float(tile_part[o * M + leaf, f]) if real else 0.0)
                fields.append(warp_tree(leaves, f == nf - 1))
            groups.append(fields)
        fields = []
        for f in range(nf):
            leaves = [groups[g][f] if (g < gpo and group_real_tiles(geo, o, g) > 0) else 0.0 for g in range(32)]
            fields.append(warp_tree(leaves, f == nf - 1))
        oct_roots.append(fields if o * M < T else [0.0] * nf)
    return np.array([warp_tree([r[f] for r in oct_roots], f == nf - 1) for f in range(nf)])


def combine_ranks(roots):
    roots = np.asarray(roots)
    nf = roots.shape[1]
    return np.array([warp_tree(list(roots[:, f]), f == nf - 1) for f in range(nf)])

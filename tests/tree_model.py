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


def octant_real_nodes(geo, o, level):
    rt = min(geo["M"], geo["T"] - o * geo["M"])
    if rt <= 0:
        return 0
    span = 32 ** level
    return -(-rt // span)


def rank_root(tile_part, geo):
    """tile_part: (T, nf) float64 partials of ALL global tiles; geo: one rank's geometry.

    Per octant a 32-ary tree of geo["levels"] levels over its M tiles (node j of
    level l reduces children 32j..32j+31 of level l-1 with warp_tree; unreal
    children contribute 0.0), then a warp tree over the rank's octant roots.
    """
    T, M, L = geo["T"], geo["M"], geo["levels"]
    nf = tile_part.shape[1]
    oct_roots = []
    for o in range(geo["oct0"], geo["oct0"] + geo["noct"]):
        if o * M >= T:
            oct_roots.append([0.0] * nf)
            continue
        level = [tile_part[o * M + t] for t in range(octant_real_nodes(geo, o, 0))]
        for lv in range(1, L + 1):
            n_nodes = -(-M // 32 ** lv)
            nxt = []
            for j in range(n_nodes):
                if j >= octant_real_nodes(geo, o, lv):
                    break
                kids = [level[k] if k < len(level) else None for k in range(32 * j, 32 * j + 32)]
                nxt.append([warp_tree([kd[f] if kd is not None else 0.0 for kd in kids], f == nf - 1)
                            for f in range(nf)])
            level = nxt
        oct_roots.append(level[0])
    return np.array([warp_tree([r[f] for r in oct_roots], f == nf - 1) for f in range(nf)])


def combine_ranks(roots):
    roots = np.asarray(roots)
    nf = roots.shape[1]
    return np.array([warp_tree(list(roots[:, f]), f == nf - 1) for f in range(nf)])

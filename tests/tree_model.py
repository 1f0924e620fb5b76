"""Python restatement of the device reduction tree (test helper).

Mirrors fcm_device.cuh::warp_tree, bfly_level (the tile-internal lane tree) and fcm_kernels.cuh::tile_finish /
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


def bfly_reduce(lanes):
    """Python restatement of fcm_device.cuh::bfly_level / bfly_field: lanes is
    a list of 32 lists of M field values.  Returns {field: value} as the
    lanes hold them after the five halving levels."""
    m = len(lanes[0])
    v = [list(x) for x in lanes]
    size = m
    for s in (16, 8, 4, 2, 1):
        h = (size + 1) // 2
        nv = []
        for lane in range(32):
            hi = bool(lane & s)
            partner = lane ^ s
            cur = []
            for k in range(h):
                a = v[lane][k]
                b = v[lane][h + k] if h + k < size else 0.0
                pa = v[partner][k]
                pb = v[partner][h + k] if h + k < size else 0.0
                keep = b if hi else a
                recv = pb if hi else pa  # the partner gives the half this lane keeps
                cur.append(keep + recv)
            nv.append(cur)
        v = nv
        size = h
    out = {}
    for lane in range(32):
        off, mm, real = 0, m, m
        for s in (16, 8, 4, 2, 1):
            h = (mm + 1) // 2
            if lane & s:
                off += h
                real = max(real - h, 0)
            else:
                real = min(real, h)
            mm = h
        for k in range(size):
            if k < real:
                assert off + k not in out, "two lanes hold one field"
                out[off + k] = v[lane][k]
    return out


def stride_tree(vals):
    """The tile-internal lane tree the butterfly evaluates: level 1 pairs lanes
    i and i ^ 16, level 2 the results of i and i ^ 8, ...."""
    x = list(vals)
    for s in (16, 8, 4, 2, 1):
        x = [x[i] + x[i + s] for i in range(s)]  # lane i < s keeps i, partner i + s
    return x[0]

"""Single GPU ops vs the reference's known answers and golden kernel outputs
(reference test_core.py:20-207, test_backends.py:42-150)."""

import numpy as np
import pytest

from conftest import golden

import paper_1601_00072_b200 as pkg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,c,seed", [(257, 3, 77), (1000, 4, 7), (33, 8, 2**64 - 1), (5, 2, 424242), (1, 2, 0)])
def test_init_membership_bitwise(n, c, seed):
    u = pkg.init_membership(n, pkg.FcmConfig(c=c, seed=seed if seed < 2**63 else seed - 2**64))
    assert u.u.tobytes() == golden("kernels")[f"init_{n}_{c}_{seed}"].tobytes()


def test_init_rows_exactly_one():
    u = pkg.init_membership(200, pkg.FcmConfig(c=4, seed=9)).as_rows()
    for row in u:
        t = 0.0
        for val in row.tolist():
            t += val
        assert t == 1.0


@pytest.mark.parametrize("m", [1.5, 2.0, 3.0])
def test_kernel_outputs_vs_reference(m):
    k = golden("kernels")
    x, u, v = k["k_x"], k["k_u"], k["k_v"]
    img = pkg.GrayImage(x.shape[0], 1, x)
    mm = pkg.MembershipMatrix(x.shape[0], 3, u)
    assert np.allclose(pkg.update_centers(img, mm, m).v, k[f"k_centers_m{m}"], rtol=1e-12)
    got = pkg.update_membership(img, pkg.ClusterCenters(v), m).u
    assert np.abs(got - k[f"k_memb_m{m}"]).max() <= 1e-13
    assert pkg.objective(img, mm, pkg.ClusterCenters(v), m) == pytest.approx(k[f"k_obj_m{m}"][0], rel=1e-12)


def test_known_answers():
    G, M, C = pkg.GrayImage, pkg.MembershipMatrix, pkg.ClusterCenters
    assert pkg.update_centers(G(2, 1, [0.0, 10.0]), M(2, 1, [1.0, 1.0]), 2.0).v[0] == 5.0
    v = pkg.update_centers(G(3, 1, [0.0, 1.0, 2.0]), M(3, 2, [0.8, 0.2, 0.5, 0.5, 0.2, 0.8]), 2.0)
    assert v.v[0] == pytest.approx(11.0 / 31.0, abs=1e-12)
    u7 = pkg.init_membership(4, pkg.FcmConfig(c=2, seed=3))
    assert np.allclose(pkg.update_centers(G(4, 1, [7.0] * 4), u7, 2.0).v, 7.0, rtol=1e-12, atol=0)
    with pytest.raises(pkg.DegenerateClusterError) as e:
        pkg.update_centers(G(2, 1, [1.0, 2.0]), M(2, 2, [1.0, 0.0, 1.0, 0.0]), 2.0)
    assert e.value.cluster == 1
    assert pkg.update_membership(G(1, 1, [0.5]), C([0.0, 1.0]), 2.0).u.tolist() == [0.5, 0.5]
    assert pkg.update_membership(G(1, 1, [0.0]), C([0.0, 1.0]), 2.0).u.tolist() == [1.0, 0.0]
    u = pkg.update_membership(G(1, 1, [0.25]), C([0.0, 1.0]), 2.0).u
    assert u[0] == pytest.approx(0.9, abs=1e-12) and u[1] == pytest.approx(0.1, abs=1e-12)
    assert pkg.update_membership(G(1, 1, [3.0]), C([3.0, 5.0, 3.0]), 2.0).u.tolist() == [0.5, 0.0, 0.5]
    assert pkg.objective(G(2, 1, [0.0, 1.0]), M(2, 2, [1, 0, 0, 1]), C([0.0, 1.0]), 2.0) == 0.0
    assert pkg.objective(G(2, 1, [0.0, 1.0]), M(2, 1, [1.0, 1.0]), C([0.5]), 2.0) == 0.5
    a = M(2, 2, [0.3, 0.7, 0.6, 0.4])
    assert pkg.membership_delta(a, a) == 0.0
    assert pkg.membership_delta(a, M(2, 2, [0.6, 0.4, 0.6, 0.4])) == pytest.approx(0.3, abs=1e-15)
    assert pkg.defuzzify(M(1, 2, [0.5, 0.5]), 1, 1).labels.tolist() == [0]
    assert pkg.defuzzify(M(3, 3, [0.1, 0.2, 0.7, 0.8, 0.1, 0.1, 0.2, 0.6, 0.2]), 3, 1).labels.tolist() == [2, 0, 1]


def test_rows_sum_to_one_general_m():
    from conftest import mixture_pixels
    img = pkg.GrayImage(500, 1, mixture_pixels(500, 3, seed=2))
    u = pkg.update_membership(img, pkg.ClusterCenters([10.0, 100.0, 250.0]), 1.7)
    assert np.abs(u.as_rows().sum(axis=1) - 1.0).max() <= 1e-9


def test_delta_and_argmax_vs_reference():
    k = golden("kernels")
    u = k["k_u"]
    a = pkg.MembershipMatrix(257, 3, u)
    b = pkg.MembershipMatrix(257, 3, u[::-1].copy())
    assert pkg.membership_delta(a, b) == k["k_maxdiff"][0]
    assert np.array_equal(pkg.defuzzify(a, 257, 1).labels, k["k_argmax"])


@pytest.mark.parametrize("n,c,seed", [(3_000_000, 3, 0), (700_000, 8, 12345), (500_000, 5, 2**63 + 7)])
def test_init_membership_large_bitwise(n, c, seed):
    """Device SplitMix64 rows (shared-reciprocal IEEE quotients) == reference generator, bit for bit."""
    from oracle import oracle as O
    s = seed if seed < 2**63 else seed - 2**64
    got = pkg.init_membership(n, pkg.FcmConfig(c=c, seed=s)).u
    ref = O.fill_membership_random(n, c, seed)
    assert got.tobytes() == ref.tobytes()


def test_branch_free_reciprocal_matches_drcp_rn():
    """The seeded start forms each row's IEEE quotients from one correctly
    rounded reciprocal of the row total; the loop kernel's copy is CUDA's
    __drcp_rn fast path without the range test and slow-path call (so four
    rows interleave).  2^31 pseudo-random totals over the whole range a row
    total can take ([2^-53, 64)): bit-identical to __drcp_rn."""
    import ctypes
    from paper_1601_00072_b200 import _lib
    bad = ctypes.c_int64(-1)
    assert _lib.lib().fcm_check_rcp(1 << 31, 0x5EED, 0, ctypes.byref(bad)) == 0
    assert bad.value == 0


def test_seeded_pass_equals_uploaded_reference_rows():
    """The loop kernel's pass 0 (strength-reduced SplitMix64 state, branch-free
    reciprocal) against the same solve started from the reference
    generator's rows uploaded as fp64 (prologue kernel, same tree): 4M voxels,
    c = 3 and 5, three passes -- centers, objective and delta traces
    identical bit for bit, so every u_0 row was."""
    from oracle import oracle as O
    from paper_1601_00072_b200 import _lib
    rng = np.random.default_rng(7)
    n = 4_000_037
    x = rng.integers(0, 256, n).astype(np.uint8)
    for c in (3, 5):
        with pkg.FcmPlan(n, c, _lib.FCM_X_U8) as plan:
            plan.upload_pixels(x)
            plan.init_membership(12345)
            v, trace, k, conv = plan.run(2.0, 1e-300, 3)
            assert plan.timing()["passes_launched"] == 1  # one loop-kernel launch, seeded in pass 0
        with pkg.FcmPlan(n, c, _lib.FCM_X_U8) as plan:
            plan.upload_pixels(x)
            plan.upload_membership(O.fill_membership_random(n, c, 12345))
            v2, trace2, k2, conv2 = plan.run(2.0, 1e-300, 3)
        assert k == k2 == 3
        assert v.tobytes() == v2.tobytes() and trace.tobytes() == trace2.tobytes()


@pytest.mark.parametrize("n,c,m", [(1_000_003, 5, 2.0), (300_001, 20, 1.5), (70_000, 1, 2.0)])
def test_update_centers_seam_large(n, c, m):
    """The seam's Eq. 3 (one op, no plan; 2c sums per CTA range and fixed
    trees, update_centers_linear, _kernels.pyx:72-90) against the oracle's
    restatement of the reference on the same AoS rows, up to c = 20."""
    from oracle import oracle as O
    rng = np.random.default_rng(n)
    x = rng.integers(0, 256, n).astype(np.float64)
    u = O.fill_membership_random(n, c, 99) if c > 1 else np.ones(n)
    v, dead = O.update_centers_linear(x, u.reshape(-1), c, m)
    got = pkg.update_centers(pkg.GrayImage(n, 1, x), pkg.MembershipMatrix(n, c, u.reshape(-1)), m).v
    assert dead < 0
    assert np.allclose(got, v, rtol=1e-11, atol=0)

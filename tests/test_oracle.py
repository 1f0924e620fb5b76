"""Pin the CPU oracle (oracle/fcm_oracle.c) against the reference's own outputs.

Fixtures in tests/golden/ were produced by the reference package itself
(tests/golden/make_golden.py); the oracle must reproduce them BITWISE,
because it restates the same double expressions in the same order with the
same libm (reference _kernels.pyx, built -O2 -ffp-contract=off).
Known answers mirror reference pkg/tests/test_core.py and test_parallel.py.
"""

import numpy as np
import pytest

from conftest import golden, mixture_pixels, run_case, run_cases, small_fixture_params
from oracle import oracle as O


def test_splitmix64_published_stream():
    # reference test_backends.py:23-32
    st, got = 0, []
    for _ in range(3):
        st, z = O.splitmix64(st)
        got.append(z)
    assert got == [16294208416658607535, 7960286522194355700, 487617019471545679]
    k = golden("kernels")
    st, got = 987654321, []
    for _ in range(100):
        st, z = O.splitmix64(st)
        got.append(z)
    assert np.array_equal(np.array(got, dtype=np.uint64), k["splitmix_987654321"])


@pytest.mark.parametrize("n,c,seed", [(257, 3, 77), (1000, 4, 7), (33, 8, 2**64 - 1), (5, 2, 424242), (1, 2, 0)])
def test_init_bitwise(n, c, seed):
    assert O.fill_membership_random(n, c, seed).tobytes() == golden("kernels")[f"init_{n}_{c}_{seed}"].tobytes()


def test_init_rows_sum_exactly_one_left_to_right():
    # reference test_core.py:48-55
    u = O.fill_membership_random(200, 4, 9).reshape(200, 4)
    for row in u:
        t = 0.0
        for val in row.tolist():
            t += val
        assert t == 1.0


@pytest.mark.parametrize("m", [1.5, 2.0, 3.0])
def test_kernels_bitwise(m):
    k = golden("kernels")
    x, u, v = k["k_x"], k["k_u"], k["k_v"]
    vv, dead = O.update_centers_linear(x, u, 3, m)
    assert dead == -1 and vv.tobytes() == k[f"k_centers_m{m}"].tobytes()
    assert O.update_membership(x, v, m).tobytes() == k[f"k_memb_m{m}"].tobytes()
    assert O.objective_linear(x, u, v, m) == k[f"k_obj_m{m}"][0]


def test_delta_argmax_reduce_bitwise():
    k = golden("kernels")
    u = k["k_u"]
    assert O.max_abs_diff(u, u[::-1].copy()) == k["k_maxdiff"][0]
    assert np.array_equal(O.argmax_rows(u, 3), k["k_argmax"])
    for length in (1, 5, 16, 255, 1024, 1025):
        out = O.block_reduce(k[f"br_in_{length}"], 8)
        assert out.tobytes() == k[f"br_out_{length}"].tobytes()
        assert O.linear_sum(out) == k[f"br_sum_{length}"][0]


@pytest.mark.parametrize("name", [n for n in run_cases()])
def test_full_runs_bitwise(name):
    r = run_case(name)
    engine = "parallel" if name.endswith("_par") else "sequential"
    res = O.run_fcm(r["x"], r["c"], r["m"], r["epsilon"], r["max_iters"], r["seed"], engine=engine)
    assert res["iterations"] == r["iterations"]
    assert res["converged"] == r["converged"]
    assert res["centers"].tobytes() == r["v"].tobytes()
    assert res["objective_trace"].tobytes() == r["trace"].tobytes()
    assert np.array_equal(res["labels"], r["labels"])
    if r["u"] is not None:
        assert res["membership"].tobytes() == r["u"].tobytes()


def test_generator_restatement_matches_reference_inputs():
    r = golden("runs")
    for idx, (n, c, m, s_img, s_init) in enumerate(small_fixture_params()):
        assert np.array_equal(mixture_pixels(n, c, s_img), r[f"small{idx}_seq_x"])
        cfg = r[f"small{idx}_seq_cfg"]
        assert (int(cfg[0]), float(cfg[1]), int(cfg[4])) == (c, m, s_init)


def test_phantom_c1_matches_fixture():
    from paper_1601_00072_b200.phantom import make_config
    assert np.array_equal(make_config("C1").astype(np.float64), golden("runs")["C1_x"])


class TestKnownAnswers:
    """Reference test_core.py:62-207 / test_parallel.py:71-143 values, on the oracle."""

    def test_centers(self):
        assert O.update_centers_linear([0.0, 10.0], [1.0, 1.0], 1, 2.0)[0][0] == 5.0
        v, _ = O.update_centers_linear([0.0, 1.0, 2.0], [0.8, 0.2, 0.5, 0.5, 0.2, 0.8], 2, 2.0)
        assert v[0] == pytest.approx(11.0 / 31.0, abs=1e-12)
        assert O.update_centers_linear([1.0, 2.0], [1.0, 0.0, 1.0, 0.0], 2, 2.0)[1] == 1

    def test_membership(self):
        assert O.update_membership([0.5], [0.0, 1.0], 2.0).tolist() == [0.5, 0.5]
        assert O.update_membership([0.0], [0.0, 1.0], 2.0).tolist() == [1.0, 0.0]
        u = O.update_membership([0.25], [0.0, 1.0], 2.0)
        assert u[0] == pytest.approx(0.9, abs=1e-12) and u[1] == pytest.approx(0.1, abs=1e-12)
        assert O.update_membership([3.0], [3.0, 5.0, 3.0], 2.0).tolist() == [0.5, 0.0, 0.5]

    def test_objective_delta_argmax(self):
        assert O.objective_linear([0.0, 1.0], [1.0, 0.0, 0.0, 1.0], [0.0, 1.0], 2.0) == 0.0
        assert O.objective_linear([0.0, 1.0], [1.0, 1.0], [0.5], 2.0) == 0.5
        assert O.max_abs_diff([0.3, 0.7, 0.6, 0.4], [0.6, 0.4, 0.6, 0.4]) == pytest.approx(0.3, abs=1e-15)
        assert O.argmax_rows([0.5, 0.5], 2).tolist() == [0]
        assert O.argmax_rows([0.1, 0.2, 0.7, 0.8, 0.1, 0.1, 0.2, 0.6, 0.2], 3).tolist() == [2, 0, 1]

    def test_reductions(self):
        assert O.block_reduce(np.ones(16), 4).tolist() == [8.0, 8.0]
        out = O.block_reduce(np.ones(1 << 20), 128)
        assert out.shape == (4096,) and np.all(out == 256.0)
        assert O.linear_sum(O.block_reduce(np.arange(1.0, 101.0), 128)) == 5050.0

    def test_degenerate_raises(self):
        with pytest.raises(O.OracleDegenerate) as e:
            O.iterate([1.0, 2.0], [1.0, 0.0, 1.0, 0.0], 2, 2.0, 0.005, 10)
        assert e.value.cluster == 1

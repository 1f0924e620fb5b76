"""Domain contracts mirror reference types.py (validation rules and errors)."""

import numpy as np
import pytest

import paper_1601_00072_b200 as pkg


def test_config_validation():
    for bad in (dict(c=1), dict(c=2, m=1.0), dict(c=2, m=float("nan")), dict(c=2, epsilon=0.0),
                dict(c=2, epsilon=1.0), dict(c=2, max_iters=0), dict(c=2, block_size=6), dict(c=2, seed=1.5)):
        with pytest.raises(pkg.InvalidConfigError):
            pkg.FcmConfig(**bad)
    cfg = pkg.FcmConfig(c=3, seed=-1)
    assert cfg.seed64 == 2**64 - 1 and cfg.m == 2.0 and cfg.epsilon == 0.005 and cfg.max_iters == 500


def test_membership_row_sum_tolerance():
    pkg.MembershipMatrix(1, 2, [0.5, 0.5 + 0.9e-9])
    with pytest.raises(ValueError):
        pkg.MembershipMatrix(1, 2, [0.5, 0.5 + 2e-9])
    with pytest.raises(ValueError):
        pkg.MembershipMatrix(1, 2, [-0.1, 1.1])


def test_image_and_labels():
    with pytest.raises(ValueError):
        pkg.GrayImage(2, 1, [1.0, -1.0])
    with pytest.raises(ValueError):
        pkg.GrayImage(2, 1, [1.0, np.inf])
    img = pkg.GrayImage.from_array(np.arange(6.0).reshape(2, 3))
    assert img.width == 3 and img.height == 2 and img.pixel_count == 6
    with pytest.raises(ValueError):
        pkg.LabelMap(2, 1, [0, 2], 2)


def test_result_trace_length():
    img_u = pkg.MembershipMatrix(1, 2, [0.5, 0.5])
    with pytest.raises(ValueError):
        pkg.FcmResult(pkg.ClusterCenters([1.0, 2.0]), img_u, pkg.LabelMap(1, 1, [0], 2), 2, (1.0,), True)


def test_errors_hierarchy():
    e = pkg.DegenerateClusterError(3)
    assert e.cluster == 3 and isinstance(e, ArithmeticError) and isinstance(e, pkg.FcmError)
    assert issubclass(pkg.InvalidConfigError, ValueError)
    assert issubclass(pkg.DimensionMismatchError, ValueError)


def test_engine_validation_before_device():
    img = pkg.GrayImage(1, 1, [3.0])
    with pytest.raises(pkg.InvalidConfigError):
        pkg.run_fcm_gpu(img, pkg.FcmConfig(c=2))
    img = pkg.GrayImage(4, 1, [1.0, 2.0, 3.0, 4.0])
    with pytest.raises(pkg.DimensionMismatchError):
        pkg.run_fcm_gpu(img, pkg.FcmConfig(c=2), initial_membership=pkg.MembershipMatrix(2, 2, [1, 0, 0, 1]))
    with pytest.raises(pkg.InvalidConfigError):
        pkg.run_fcm_gpu(pkg.GrayImage(40, 1, np.arange(40.0)), pkg.FcmConfig(c=33))

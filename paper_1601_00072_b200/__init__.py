"""B200-native Fuzzy C-Means hot path (arXiv 1601.00072), drop-in for fcmseg.

The reference package (fcmseg) runs the FCM loop on the CPU; this package runs
the same loop as one fused sm_100a streaming kernel per iteration behind the
C ABI in include/fcm_b200.h.  The Python surface mirrors the reference's
names and contracts (fcmseg/__init__.py re-exports):

    from paper_1601_00072_b200 import FcmConfig, GrayImage, run_fcm_gpu
    result = run_fcm_gpu(img, FcmConfig(c=3, m=2.0, epsilon=1e-5))

There is no CPU fallback: without libfcm_b200.so or a GPU, calls raise
DeviceError.
"""

from .engine import (
    C_MAX,
    ENGINES,
    FcmPlan,
    _iterate,
    defuzzify,
    init_membership,
    membership_delta,
    objective,
    pixel_kind,
    release_cached_plans,
    run_fcm_gpu,
    update_centers,
    update_membership,
)
from .errors import (DegenerateClusterError, DeviceError, DimensionMismatchError, FcmError, InvalidConfigError,
                     MalformedHeaderError, MissingClassError, PgmError, PgmValueError, TruncatedRasterError,
                     UnsupportedMagicError)
from .imgio import PgmImage, label_intensity, parse_pgm, read_ground_truth, read_pgm, read_pgm_raster, write_pgm
from .metrics import BinaryMask, DscReport, dsc, dsc_report_gpu, mask_for_class, match_clusters, match_clusters_gpu
from .types import ROW_SUM_TOL, ClusterCenters, FcmConfig, FcmResult, GrayImage, LabelMap, MembershipMatrix

__version__ = "0.1.0"

__all__ = [
    "C_MAX", "ENGINES", "FcmPlan", "_iterate", "defuzzify", "init_membership", "membership_delta",
    "objective", "pixel_kind", "release_cached_plans", "run_fcm_gpu", "update_centers", "update_membership",
    "DegenerateClusterError", "DeviceError", "DimensionMismatchError", "FcmError", "InvalidConfigError",
    "ROW_SUM_TOL", "ClusterCenters", "FcmConfig", "FcmResult", "GrayImage", "LabelMap", "MembershipMatrix",
    "MalformedHeaderError", "MissingClassError", "PgmError", "PgmValueError", "TruncatedRasterError",
    "UnsupportedMagicError", "PgmImage", "label_intensity", "parse_pgm", "read_ground_truth", "read_pgm",
    "read_pgm_raster", "write_pgm", "BinaryMask", "DscReport", "dsc", "dsc_report_gpu", "mask_for_class",
    "match_clusters", "match_clusters_gpu",
]

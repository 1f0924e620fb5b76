"""Segmentation metrics of the drop-in (reference metrics.py:1-97), with the
counting on the device.

The labels of a solve are already in HBM after `FcmPlan.download`; the c x c
confusion matrix against a reference label map and the per-cluster overlaps
with a ground-truth mask are counted there (`fcm_label_confusion`,
`fcm_mask_overlap`), and only c^2 integers come back.  Dice and the greedy
cluster matching are then exact integer arithmetic on the host, with the
reference's formulas, tie rules and errors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatchError
from .types import LabelMap


@dataclass(frozen=True)
class BinaryMask:
    """Flat boolean raster marking one tissue class."""

    width: int
    height: int
    bits: np.ndarray

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError("mask dimensions must be at least 1x1")
        bits = np.ascontiguousarray(self.bits, dtype=bool)
        if bits.ndim != 1 or bits.shape[0] != self.width * self.height:
            raise ValueError("bit buffer length must equal width*height")
        object.__setattr__(self, "bits", bits)

    @property
    def count(self) -> int:
        return int(np.count_nonzero(self.bits))


@dataclass(frozen=True)
class DscReport:
    """Per-class Dice similarity values, each in [0, 1]."""

    per_class: dict

    def __post_init__(self):
        for name, value in self.per_class.items():
            if not (0.0 <= value <= 1.0):
                raise ValueError(f"DSC for {name!r} is {value}, outside [0, 1]")


def dice_from_counts(inter: int, a: int, b: int) -> float:
    """2|A and B| / (|A| + |B|); two empty sets agree perfectly (1.0)."""
    return 1.0 if a + b == 0 else 2.0 * inter / (a + b)


def dsc(pr: BinaryMask, gt: BinaryMask) -> float:
    """Dice similarity of two masks (reference metrics.py:46-61)."""
    if (pr.width, pr.height) != (gt.width, gt.height):
        raise DimensionMismatchError(f"masks are {pr.width}x{pr.height} and {gt.width}x{gt.height}")
    return dice_from_counts(int(np.count_nonzero(pr.bits & gt.bits)), pr.count, gt.count)


def mask_for_class(labels: LabelMap, j: int) -> BinaryMask:
    """Binary mask of the pixels assigned to cluster j."""
    if not 0 <= j < labels.c:
        raise IndexError(f"cluster index {j} out of range [0, {labels.c})")
    return BinaryMask(labels.width, labels.height, labels.labels == j)


def greedy_match(conf: np.ndarray) -> tuple:
    """The reference's greedy assignment on a c x c confusion matrix: repeatedly
    take the unassigned (pred, ref) pair with the largest count, ties toward the
    lowest flat index (metrics.py:78-97).  perm[p] = r."""
    work = np.array(conf, dtype=np.int64, copy=True)
    c = work.shape[0]
    perm = [-1] * c
    for _ in range(c):
        p, r = divmod(int(np.argmax(work)), c)
        perm[p] = r
        work[p, :] = -1
        work[:, r] = -1
    return tuple(perm)


def confusion(pred: LabelMap, ref: LabelMap, c: int) -> np.ndarray:
    """Host c x c confusion counts (pred row, ref column)."""
    if (pred.width, pred.height) != (ref.width, ref.height):
        raise DimensionMismatchError(f"label maps are {pred.width}x{pred.height} and {ref.width}x{ref.height}")
    if pred.c > c or ref.c > c:
        raise DimensionMismatchError(f"label maps use more than {c} clusters")
    return np.bincount(pred.labels.astype(np.int64) * c + ref.labels.astype(np.int64),
                       minlength=c * c).reshape(c, c)


def match_clusters(pred: LabelMap, ref: LabelMap, c: int) -> tuple:
    """Permutation aligning predicted clusters to reference classes (metrics.py:78-97)."""
    return greedy_match(confusion(pred, ref, c))


def match_clusters_gpu(plan, ref: LabelMap, c: int) -> tuple:
    """match_clusters for the labels of `plan`'s last solve, counted on the device."""
    if ref.c > c or plan.c > c:
        raise DimensionMismatchError(f"label maps use more than {c} clusters")
    conf = np.zeros((c, c), dtype=np.int64)  # rows of clusters the plan does not have stay 0,
    conf[: plan.c, :] = plan.confusion(ref.labels, c)  # as in the reference's c x c bincount
    return greedy_match(conf)


def dsc_report_gpu(plan, truth: dict, classes) -> DscReport:
    """The reference CLI's per-class Dice (cli.py cmd_dsc): reference labels from
    the ground-truth masks (uncovered -> background, overlaps -> lowest index),
    greedy matching, then Dice of each matched cluster against its mask -- every
    count taken on the device from the plan's resident labels."""
    c = len(classes)
    first = truth[classes[0]]
    n = first.width * first.height
    if n != plan.n:
        raise DimensionMismatchError(f"prediction has {plan.n} pixels, ground truth {n}")
    background = classes.index("background")
    ref = np.full(n, background, dtype=np.int32)
    for idx in range(c - 1, -1, -1):
        ref[truth[classes[idx]].bits] = idx
    perm = greedy_match(plan.confusion(ref, c))
    out = {}
    for idx, name in enumerate(classes):
        p = perm.index(idx)
        counts, total = plan.mask_overlap(truth[name].bits)
        pred_count = int(plan.label_counts()[p])
        out[name] = dice_from_counts(int(counts[p]), pred_count, total)
    return DscReport(out)

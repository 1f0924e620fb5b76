"""The GPU engine: drop-in for the reference's FCM entry points.

Reference surface (fcmseg, /root/reference/pkg/src/fcmseg):

* run_fcm_sequential / run_fcm_parallel (core.py:146-171, parallel.py:334-362)
  -> run_fcm_gpu(img, cfg, devices=None, initial_membership=None), same
  validation, same FcmResult.
* core._iterate / parallel._iterate (core.py:105-132, parallel.py:257-331), the
  region the reference benchmark times (bench.py:49-59) -> _iterate(x, u0, cfg,
  devices=None) returning (v, u, iterations, trace, converged).
* the single-step operations init_membership, update_centers,
  update_membership, objective, membership_delta, defuzzify (core.py:24-102)
  -> same names on the GPU.

Every call goes through libfcm_b200.so (include/fcm_b200.h); nothing here
computes on the CPU except argument validation and result packaging.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _lib
from ._lib import check, lib, ptr
from .errors import DegenerateClusterError, DimensionMismatchError, FcmError, InvalidConfigError
from .types import ClusterCenters, FcmConfig, FcmResult, GrayImage, LabelMap, MembershipMatrix

C_MAX = 32


_scratch = threading.local()


def _pinned_scratch(nbytes: int) -> np.ndarray:
    """This thread's page-locked staging buffer (cudaHostRegister'ed once and
    reused): run_fcm_gpu narrows float64 pixels straight into it, so the
    upload runs at pinned-copy speed.  Falls back to pageable memory when
    registration fails."""
    buf = getattr(_scratch, "buf", None)
    if buf is None or buf.nbytes < nbytes:
        if buf is not None and getattr(_scratch, "pinned", False):
            lib().fcm_host_unregister(ptr(buf))
        buf = np.empty(max(nbytes, 1), dtype=np.uint8)
        _scratch.pinned = lib().fcm_host_register(ptr(buf), buf.nbytes) == _lib.FCM_OK
        _scratch.buf = buf
    return buf[:nbytes]


def pixel_kind(pixels: np.ndarray, staging: bool = False):
    """Pick the narrowest exact device representation of the pixels.

    Integer intensities 0..255 travel and live in HBM as uint8 (every
    BASELINE config), 256..65535 as uint16 (16-bit PGM rasters,
    imgio.py:102-110); anything else stays float64 (types.py:38-41 accepts
    any finite non-negative value).  float64 input is checked and narrowed in
    one multi-threaded pass in the library (fcm_narrow_pixels).  Returns
    (FCM_X_*, contiguous array).  staging=True narrows into this thread's
    pinned staging buffer (valid until the next call; run_fcm_gpu uses it).
    """
    if pixels.dtype == np.uint8:
        return _lib.FCM_X_U8, np.ascontiguousarray(pixels)
    if pixels.dtype == np.uint16:
        x = np.ascontiguousarray(pixels)
        if x.size and int(x.max()) > 255:
            return _lib.FCM_X_U16, x
        return _lib.FCM_X_U8, x.astype(np.uint8)
    x = np.ascontiguousarray(pixels, dtype=np.float64)
    n = x.shape[0]
    for kind, dt in ((_lib.FCM_X_U8, np.uint8), (_lib.FCM_X_U16, np.uint16)):
        out = _pinned_scratch(n * np.dtype(dt).itemsize).view(dt) if staging else np.empty(n, dtype=dt)
        if lib().fcm_narrow_pixels(ptr(x), n, kind, ptr(out), 0) == _lib.FCM_OK:
            return kind, out
    return _lib.FCM_X_F64, x


def _devices(devices):
    if devices is None:
        return [0]
    if isinstance(devices, int):
        if devices < 1:
            raise InvalidConfigError(f"device count must be >= 1, got {devices!r}")
        return list(range(devices))
    devs = [int(d) for d in devices]
    if len(devs) not in (1, 2, 4, 8):
        raise InvalidConfigError(f"shard count must be 1, 2, 4 or 8, got {len(devs)}")
    return devs


class FcmPlan:
    """Device-resident FCM problem: pixels, memberships and reduction state.

    One plan per host thread (the C plan is not re-entrant).  Single-process
    plans shard over `devices` (repeats allowed); rank plans (FcmPlan.for_rank)
    own one rank's voxel range of a multi-process job and exchange the
    2c+2-double reduction roots over NCCL.
    """

    def __init__(self, n: int, c: int, x_kind: int, devices=None, _handle=None):
        if _handle is not None:
            self._h = _handle
        else:
            devs = _devices(devices)
            arr = (ctypes.c_int32 * len(devs))(*devs)
            h = ctypes.c_void_p()
            check(lib().fcm_plan_create(ctypes.byref(h), int(n), int(c), int(x_kind), len(devs), arr),
                  None, "fcm_plan_create")
            self._h = h
        self.n, self.c, self.x_kind = int(n), int(c), int(x_kind)
        info = self.info()
        self.n_local, self.voxel0 = info["n_local"], info["voxel0"]

    @staticmethod
    def _locate_nccl():
        """Point the C library at the wheel's libnccl (it dlopens on first use)."""
        if os.environ.get("FCM_NCCL_LIB"):
            return
        try:
            import nvidia.nccl
            for d in nvidia.nccl.__path__:
                cand = os.path.join(d, "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["FCM_NCCL_LIB"] = cand
                    return
        except ImportError:
            pass

    @classmethod
    def for_rank(cls, n_global: int, c: int, x_kind: int, device: int, nranks: int, rank: int,
                 nccl_id: bytes | None = None):
        cls._locate_nccl()
        h = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        check(lib().fcm_plan_create_rank(ctypes.byref(h), int(n_global), int(c), int(x_kind), int(device),
                                         int(nranks), int(rank), idbuf), None, "fcm_plan_create_rank")
        return cls(n_global, c, x_kind, _handle=h)

    def mailbox_handle(self) -> bytes:
        """64-byte CUDA IPC handle of this rank's root mailbox (fused exchange)."""
        buf = ctypes.create_string_buffer(64)
        check(lib().fcm_mailbox_handle(self._h, buf), self._h, "fcm_mailbox_handle")
        return buf.raw

    def connect_peers(self, handles: bytes, nranks: int):
        """Map every rank's mailbox (handles of all ranks, rank order): the loop kernel then
        exchanges the per-pass roots with NVLink peer stores instead of NCCL."""
        buf = ctypes.create_string_buffer(bytes(handles), 64 * nranks)
        check(lib().fcm_connect_peers(self._h, buf, int(nranks)), self._h, "fcm_connect_peers")

    @staticmethod
    def nccl_unique_id() -> bytes:
        FcmPlan._locate_nccl()
        buf = ctypes.create_string_buffer(128)
        check(lib().fcm_nccl_unique_id(buf), None, "fcm_nccl_unique_id")
        return buf.raw

    # -- lifecycle -------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().fcm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- configuration ---------------------------------------------------
    def set_option(self, key: int, value: int):
        check(lib().fcm_set_option(self._h, key, int(value)), self._h, "fcm_set_option")

    def info(self) -> dict:
        keys = ("n_global", "n_local", "voxel0", "tile", "tiles", "tiles_local", "grid", "nshards", "dev_bytes")
        buf = (ctypes.c_int64 * len(keys))()
        check(lib().fcm_plan_info(self._h, buf, len(keys)), self._h, "fcm_plan_info")
        return dict(zip(keys, list(buf)))

    # -- data ------------------------------------------------------------
    def upload_pixels(self, x: np.ndarray):
        """Pixels of this plan's voxel range: uint8 (FCM_X_U8), uint16 (FCM_X_U16) or float64."""
        want = {_lib.FCM_X_U8: np.uint8, _lib.FCM_X_U16: np.uint16}.get(self.x_kind, np.float64)
        x = np.ascontiguousarray(x, dtype=want)
        check(lib().fcm_upload_pixels(self._h, ptr(x)), self._h, "fcm_upload_pixels")

    def init_membership(self, seed: int):
        """Seeded SplitMix64 start, generated on the device (core.init_membership)."""
        check(lib().fcm_init_membership(self._h, int(seed) & 0xFFFFFFFFFFFFFFFF), self._h, "fcm_init_membership")

    def upload_membership(self, u0: np.ndarray):
        """Explicit AoS float64 start (initial_membership=, core.py:135-143)."""
        u0 = np.ascontiguousarray(u0, dtype=np.float64)
        check(lib().fcm_upload_membership(self._h, ptr(u0)), self._h, "fcm_upload_membership")

    # -- the loop --------------------------------------------------------
    def run(self, m: float, epsilon: float, max_iters: int):
        """Returns (v, trace, iterations, converged); raises DegenerateClusterError."""
        v = np.zeros(self.c, dtype=np.float64)
        trace = np.zeros(max_iters, dtype=np.float64)
        it, conv, dead = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        st = lib().fcm_run(self._h, float(m), float(epsilon), int(max_iters), ptr(v), ptr(trace),
                           ctypes.byref(it), ctypes.byref(conv), ctypes.byref(dead))
        if st == _lib.FCM_E_DEGENERATE:
            raise DegenerateClusterError(int(dead.value))
        check(st, self._h, "fcm_run")
        k = int(it.value)
        return v, trace[:k].copy(), k, bool(conv.value)

    def download(self, membership: bool = True, labels: bool = True, u_out=None, labels_out=None):
        """Final membership (AoS float64) and labels of this plan's voxel range."""
        u = None
        lab = None
        if membership:
            u = u_out if u_out is not None else np.empty(self.n_local * self.c, dtype=np.float64)
        if labels:
            lab = labels_out if labels_out is not None else np.empty(self.n_local, dtype=np.int32)
        check(lib().fcm_download(self._h, ptr(u), ptr(lab)), self._h, "fcm_download")
        return u, lab

    def download_table(self, x: np.ndarray, membership: bool = True, labels: bool = True, u_out=None,
                       labels_out=None, threads: int = 0):
        """download() for uint8 plans through the 256-row intensity table: the same arrays bit for
        bit, 256*(8c+4) bytes over PCIe, rows expanded on the host along `x` (the uploaded pixels)."""
        x = np.ascontiguousarray(x, dtype=np.uint8)
        if x.shape[0] != self.n_local:
            raise DimensionMismatchError(f"pixels cover {x.shape[0]} voxels, expected {self.n_local}")
        u = lab = None
        if membership:
            u = u_out if u_out is not None else np.empty(self.n_local * self.c, dtype=np.float64)
        if labels:
            lab = labels_out if labels_out is not None else np.empty(self.n_local, dtype=np.int32)
        check(lib().fcm_download_table(self._h, ptr(x), ptr(u), ptr(lab), int(threads)), self._h,
              "fcm_download_table")
        return u, lab

    def result_table(self):
        """(u_tab [256, c] float64, l_tab [256] int32): the result table of the last download_table."""
        u = np.empty(256 * self.c, dtype=np.float64)
        lab = np.empty(256, dtype=np.int32)
        check(lib().fcm_result_table(self._h, ptr(u), ptr(lab)), self._h, "fcm_result_table")
        return u.reshape(256, self.c), lab

    def profile(self) -> np.ndarray:
        """Loop-kernel timeline of the last run (FCM_OPT_PROFILE): array [pass, cta, slot]
        with slots 0 start, 1 claims done, 2 consumers done, 3 barrier arrival (ns), 4 tiles, ...
        21 / 22 multi-shard root exchange: all roots here / last rank's publication
        (tools/pass_phases.py, tools/exchange_latency.py)."""
        slots = 24  # kProbeSlots (fcm_kernels.h)
        cap = 64 * 8 * 1024 * slots
        buf = np.zeros(cap, dtype=np.uint64)
        passes, grid = ctypes.c_int32(), ctypes.c_int32()
        check(lib().fcm_last_profile(self._h, ptr(buf), cap, ctypes.byref(passes), ctypes.byref(grid)),
              self._h, "fcm_last_profile")
        return buf[: passes.value * grid.value * slots].reshape(passes.value, grid.value, slots)

    # -- label statistics (metrics on the device) ------------------------
    def confusion(self, ref_labels: np.ndarray, c_ref: int) -> np.ndarray:
        """[c, c_ref] counts |pred==p & ref==r| of the last solve's labels (after download)."""
        ref = np.ascontiguousarray(ref_labels, dtype=np.int32)
        if ref.shape[0] != self.n_local:
            raise DimensionMismatchError(f"reference labels cover {ref.shape[0]} voxels, expected {self.n_local}")
        if ref.size and (ref.min() < 0 or ref.max() >= c_ref):
            raise InvalidConfigError(f"reference labels must lie in [0, {c_ref})")
        out = np.zeros(self.c * c_ref, dtype=np.int64)
        check(lib().fcm_label_confusion(self._h, ptr(ref), int(c_ref), ptr(out)), self._h, "fcm_label_confusion")
        return out.reshape(self.c, c_ref)

    def _mask_stats(self, mask) -> np.ndarray:
        m = np.ascontiguousarray(np.asarray(mask, dtype=bool)).view(np.uint8)
        if m.shape[0] != self.n_local:
            raise DimensionMismatchError(f"mask covers {m.shape[0]} voxels, expected {self.n_local}")
        out = np.zeros(2 * self.c + 1, dtype=np.int64)
        check(lib().fcm_mask_overlap(self._h, ptr(m), ptr(out)), self._h, "fcm_mask_overlap")
        return out

    def mask_overlap(self, mask):
        """(|pred==p & mask| for each cluster p, |mask|) for the last solve's labels."""
        st = self._mask_stats(mask)
        return st[: self.c], int(st[self.c])

    def label_counts(self) -> np.ndarray:
        """|pred==p| for each cluster p."""
        return self._mask_stats(np.zeros(self.n_local, dtype=bool))[self.c + 1:]

    def delta_trace(self, iterations: int) -> np.ndarray:
        """delta_1..delta_k of the last run (what the stop test compared with epsilon)."""
        d = np.zeros(iterations, dtype=np.float64)
        check(lib().fcm_delta_trace(self._h, ptr(d), int(iterations)), self._h, "fcm_delta_trace")
        return d

    def timing(self) -> dict:
        keys = ("loop_ms", "pass_ms", "prologue_ms", "passes_launched", "passes", "seeded_in_loop",
                "loop_fallbacks")
        buf = (ctypes.c_double * len(keys))()
        check(lib().fcm_last_timing(self._h, buf, len(keys)), self._h, "fcm_last_timing")
        return dict(zip(keys, list(buf)))


# ----------------------------------------------------------------- engine --
def _check_c(c: int):
    if c > C_MAX:
        raise InvalidConfigError(f"the GPU path supports c <= {C_MAX} (kernel payload), got {c}")


# One cached plan per host thread (plans are not re-entrant): repeated solves
# of the same shape -- the reference's bench loop (bench.py:49-59, 96-106)
# and every caller that segments a series of same-sized volumes -- reuse the
# device buffers instead of allocating and freeing them per call.
_plans = threading.local()


def _cached_plan(n: int, c: int, kind: int, devices) -> FcmPlan:
    key = (int(n), int(c), int(kind), tuple(_devices(devices)))
    ent = getattr(_plans, "entry", None)
    if ent is not None and ent[0] == key and ent[1]._h:
        return ent[1]
    release_cached_plans()
    plan = FcmPlan(n, c, kind, devices)
    _plans.entry = (key, plan)
    return plan


def release_cached_plans() -> None:
    """Free the device memory of this thread's cached plan (run_fcm_gpu / _iterate)."""
    ent = getattr(_plans, "entry", None)
    _plans.entry = None
    if ent is not None:
        ent[1].close()


def _solve(plan: FcmPlan, xx, kind, cfg: FcmConfig, u0=None):
    """Upload, run and download on `plan`; returns (v, trace, k, conv, u, labels, table).
    A failed run (other than a dead cluster) drops the plan from the cache."""
    try:
        plan.upload_pixels(xx)
        if u0 is None:
            plan.init_membership(cfg.seed64)
        else:
            plan.upload_membership(u0)
        v, trace, k, conv = plan.run(cfg.m, cfg.epsilon, cfg.max_iters)
        table = None
        if kind == _lib.FCM_X_U8:
            # 8-bit pixels: at most 256 distinct result rows -- copy the table,
            # expand on the host (identical arrays, ~n*8c fewer PCIe bytes)
            u, labels = plan.download_table(xx)
            table = plan.result_table()
        else:
            u, labels = plan.download()
    except DegenerateClusterError:
        raise
    except BaseException:
        ent = getattr(_plans, "entry", None)
        if ent is not None and ent[1] is plan:
            release_cached_plans()
        raise
    return v, trace, k, conv, u, labels, table


def _iterate(x: np.ndarray, u0: np.ndarray | None, cfg: FcmConfig, devices=None, seed: int | None = None):
    """Device counterpart of core._iterate (core.py:105-132).

    x: pixels (float64, uint8 or uint16); u0: AoS float64 start (consumed
    like the reference's scratch, here only read), or None with `seed` to
    generate the reference's seeded start on the device.  Returns
    (v, u_final, iterations, trace, converged) like the reference.
    """
    _check_c(cfg.c)
    kind, xx = pixel_kind(np.asarray(x), staging=True)
    n = xx.shape[0]
    if u0 is not None:
        u0 = np.ascontiguousarray(u0, dtype=np.float64)
        if u0.shape[0] != n * cfg.c:
            raise DimensionMismatchError(f"initial membership has {u0.shape[0]} entries, expected {n * cfg.c}")
    if u0 is None and seed is not None:
        cfg = FcmConfig(c=cfg.c, m=cfg.m, epsilon=cfg.epsilon, max_iters=cfg.max_iters, seed=seed,
                        block_size=cfg.block_size)
    plan = _cached_plan(n, cfg.c, kind, devices)
    v, trace, k, conv, u, _, _ = _solve(plan, xx, kind, cfg, u0)
    return v, u, k, list(trace), conv


def run_fcm_gpu(img: GrayImage, cfg: FcmConfig, devices=None,
                initial_membership: MembershipMatrix | None = None, keep_plan: bool = False):
    """Cluster an image on the GPU; drop-in for run_fcm_sequential / run_fcm_parallel.

    `img` is a GrayImage or an imgio.PgmImage (integer raster, no float64
    expansion).  keep_plan=True returns (FcmResult, FcmPlan) with the plan's
    labels still resident for the device-side metrics (metrics.dsc_report_gpu);
    the caller closes the plan.  Otherwise the thread's cached plan is reused
    (release_cached_plans() frees it).

    Same seeded initialization as the reference engines (SplitMix64, generated
    on the device), same convergence rule, same result contract.  `devices`
    shards the voxels (1, 2, 4 or 8 shards; results are bit-identical for any
    shard count, mirroring workers= invariance, parallel.py:1-11).
    """
    n = img.pixel_count
    if n < cfg.c:
        raise InvalidConfigError(f"need at least {cfg.c} pixels for {cfg.c} clusters, got {n}")
    _check_c(cfg.c)
    if initial_membership is not None and (initial_membership.n != n or initial_membership.c != cfg.c):
        raise DimensionMismatchError(
            f"initial membership is {initial_membership.n}x{initial_membership.c}, expected {n}x{cfg.c}")
    # a PgmImage (imgio.read_pgm_raster) hands its integer raster over as is:
    # 8-bit images reach HBM at 1 B per voxel, 16-bit at 2 B, without a float64 copy
    from .imgio import PgmImage
    kind, xx = pixel_kind(img.raster if isinstance(img, PgmImage) else img.pixels, staging=True)
    plan = FcmPlan(n, cfg.c, kind, devices) if keep_plan else _cached_plan(n, cfg.c, kind, devices)
    try:
        v, trace, k, conv, u, labels, table = _solve(
            plan, xx, kind, cfg, None if initial_membership is None else initial_membership.u)
    except BaseException:
        if keep_plan:
            plan.close()
        raise
    if table is not None:
        # every row / label is a copy of a table entry: validating the 256
        # table rows validates the result (types.py:82-85) without n*c passes
        membership = MembershipMatrix.from_table_rows(n, cfg.c, u, table[0])
        label_map = LabelMap.from_table_labels(img.width, img.height, labels, cfg.c, table[1])
    else:
        membership = MembershipMatrix(n, cfg.c, u)
        label_map = LabelMap(img.width, img.height, labels, cfg.c)
    result = FcmResult(
        centers=ClusterCenters(v),
        membership=membership,
        labels=label_map,
        iterations=k,
        objective_trace=tuple(float(t) for t in trace),
        converged=conv,
    )
    return (result, plan) if keep_plan else result


ENGINES = {"gpu": run_fcm_gpu}


# ------------------------------------------------------ single operations --
def _require_fuzzifier(m: float) -> float:
    m = float(m)
    if not np.isfinite(m) or m <= 1.0:
        raise InvalidConfigError(f"fuzzifier must be a finite real > 1, got {m!r}")
    return m


def init_membership(n: int, cfg: FcmConfig, device: int = 0) -> MembershipMatrix:
    """Seeded start on the GPU, bit-identical to core.init_membership (core.py:24-39)."""
    if not isinstance(n, int) or n < 1:
        raise InvalidConfigError(f"pixel count must be an integer >= 1, got {n!r}")
    _check_c(cfg.c)
    u = np.empty(n * cfg.c, dtype=np.float64)
    check(lib().fcm_fill_membership_random(ptr(u), n, cfg.c, cfg.seed64, device), None, "fill_membership_random")
    matrix = MembershipMatrix(n, cfg.c, u)
    if n > cfg.c:
        cols = matrix.as_rows().sum(axis=0)
        if np.any(cols <= 0.0) or np.any(cols >= n):
            raise FcmError("randomized initialization produced an empty or saturated cluster")
    return matrix


def update_centers(img: GrayImage, u: MembershipMatrix, m: float, device: int = 0) -> ClusterCenters:
    """Eq. 3 on the GPU (core.update_centers, core.py:42-57)."""
    m = _require_fuzzifier(m)
    if u.n != img.pixel_count:
        raise DimensionMismatchError(f"membership covers {u.n} pixels but the image has {img.pixel_count}")
    _check_c(u.c)
    v = np.zeros(u.c, dtype=np.float64)
    dead = ctypes.c_int32(-1)
    check(lib().fcm_update_centers(ptr(img.pixels), ptr(u.u), ptr(v), u.n, u.c, m, device, ctypes.byref(dead)),
          None, "update_centers")
    if dead.value >= 0:
        raise DegenerateClusterError(int(dead.value))
    return ClusterCenters(v)


def update_membership(img: GrayImage, v: ClusterCenters, m: float, device: int = 0) -> MembershipMatrix:
    """Eq. 4 on the GPU (core.update_membership, core.py:60-70)."""
    m = _require_fuzzifier(m)
    _check_c(v.c)
    n = img.pixel_count
    u = np.empty(n * v.c, dtype=np.float64)
    check(lib().fcm_update_membership(ptr(img.pixels), ptr(v.v), ptr(u), n, v.c, m, device), None,
          "update_membership")
    return MembershipMatrix(n, v.c, u)


def objective(img: GrayImage, u: MembershipMatrix, v: ClusterCenters, m: float, device: int = 0) -> float:
    """J = sum_i sum_j u_ij^m (x_i - v_j)^2 on the GPU (core.objective, core.py:73-82)."""
    m = _require_fuzzifier(m)
    if u.n != img.pixel_count:
        raise DimensionMismatchError(f"membership covers {u.n} pixels but the image has {img.pixel_count}")
    if u.c != v.c:
        raise DimensionMismatchError(f"membership has {u.c} clusters but centers have {v.c}")
    out = ctypes.c_double()
    check(lib().fcm_objective(ptr(img.pixels), ptr(u.u), ptr(v.v), u.n, u.c, m, device, ctypes.byref(out)),
          None, "objective")
    return float(out.value)


def membership_delta(u_new: MembershipMatrix, u_old: MembershipMatrix, device: int = 0) -> float:
    """max |u_new - u_old| on the GPU (core.membership_delta, core.py:85-91)."""
    if (u_new.n, u_new.c) != (u_old.n, u_old.c):
        raise DimensionMismatchError(f"memberships are {u_new.n}x{u_new.c} and {u_old.n}x{u_old.c}")
    out = ctypes.c_double()
    check(lib().fcm_max_abs_diff(ptr(u_new.u), ptr(u_old.u), u_new.n * u_new.c, device, ctypes.byref(out)),
          None, "max_abs_diff")
    return float(out.value)


def defuzzify(u: MembershipMatrix, width: int, height: int, device: int = 0) -> LabelMap:
    """Argmax per row, ties to the lowest index (core.defuzzify, core.py:94-102)."""
    if u.n != width * height:
        raise DimensionMismatchError(f"membership covers {u.n} pixels but the map is {width}x{height}")
    labels = np.empty(u.n, dtype=np.int32)
    check(lib().fcm_argmax_rows(ptr(u.u), ptr(labels), u.n, u.c, device), None, "argmax_rows")
    return LabelMap(width, height, labels, u.c)

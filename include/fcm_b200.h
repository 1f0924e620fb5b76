/*
 * fcm_b200.h -- C ABI of the B200 Fuzzy C-Means hot path (libfcm_b200.so).
 *
 * Drop-in boundary for the reference package fcmseg (/root/reference/pkg).
 * The reference has no FFI of its own: its hot path is the Python engine loop
 * core._iterate / parallel._iterate calling a kernel module chosen by
 * backend.active() (backend.py:11-52).  Two cuts are exported:
 *
 *   1. the ENGINE-LOOP boundary (the one the product uses): a plan holding
 *      device-resident pixels and memberships runs the whole
 *      centers -> membership -> delta -> objective loop on the GPU and
 *      returns what _iterate returns (v, u, iterations, trace, converged).
 *      Replaces core._iterate (core.py:105-132), parallel._iterate
 *      (parallel.py:257-331), core.init_membership (core.py:24-39) and
 *      core.defuzzify (core.py:94-102).
 *   2. the KERNEL seam: the functions of _kernels.pyx (:33-238) that have a
 *      meaning on their own, on caller-owned host buffers with the
 *      reference's conventions (flat float64, membership AoS u[i*c + j],
 *      int32 labels, -1 / cluster-index return for a dead cluster).
 *
 * All functions return an fcm_status.  Host buffers stay caller-owned; the
 * plan owns every device buffer.  A plan is not re-entrant: use one plan per
 * host thread.  There is no CPU fallback: without a usable sm_100 GPU every
 * entry point that computes returns FCM_E_CUDA.
 */
#ifndef FCM_B200_H
#define FCM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FCM_ABI_VERSION 1

typedef enum {
  FCM_OK = 0,
  FCM_E_ARG = 1,        /* invalid argument            -> InvalidConfigError / DimensionMismatchError */
  FCM_E_CUDA = 2,       /* CUDA runtime failure / no GPU */
  FCM_E_NCCL = 3,       /* NCCL failure (multi-process plans) */
  FCM_E_DEGENERATE = 4, /* a cluster got zero weight   -> DegenerateClusterError(dead_cluster), core.py:121-123 */
  FCM_E_STATE = 5,      /* call order violated (e.g. run before upload) */
  FCM_E_NOMEM = 6       /* device allocation failed */
} fcm_status;

typedef enum {
  FCM_X_U8 = 0,  /* integer intensities 0..255 (every BASELINE config): 1 byte per voxel in HBM */
  FCM_X_U16 = 1, /* integer intensities 0..65535 (16-bit PGM rasters, imgio.py:102-110): 2 bytes per voxel */
  FCM_X_F64 = 2  /* any finite, non-negative intensity (types.py:38-41) */
} fcm_x_kind;

typedef enum {
  FCM_OPT_BATCH = 1,   /* passes launched between host checks of the done flag (default 8) */
  FCM_OPT_TIMING = 2,  /* 1: record per-pass CUDA events for fcm_last_timing (default 0) */
  FCM_OPT_GRID = 3,    /* force CTAs per pass launch (0 = occupancy-derived, default) */
  FCM_OPT_KERNEL = 4,  /* pass kernel: 0 = TMA bulk-copy pipeline, automatic per-voxel math (default:
                          product form for m == 2, per-pass intensity table for other m on uint8),
                          1 = register-staged LDG/STG (the kernel of 17 <= c <= 32; FCM_E_ARG for c <= 16,
                          where it lost its A/B and is not built), 2 = TMA + intensity table for every m (uint8),
                          3 = TMA + per-voxel math for every m */
  FCM_OPT_GRAPH = 5,   /* 1 (default): when the loop kernel is off, single-shard runs launch
                          prologue + a device-side while loop (CUDA graph conditional node);
                          0: host-driven batches.  FCM_OPT_TIMING forces the host-driven path. */
  FCM_OPT_LOOP = 6,    /* 1 (default): single-shard, single-rank runs launch the prologue and ONE
                          persistent cooperative kernel that runs every pass, with a grid barrier
                          between passes; 0: one launch per pass (graph or host-driven) */
  FCM_OPT_L2 = 7,      /* 0: stream x/u with evict-first stores; 1 (default): keep them in L2
                          (evict_last policy) when they fit; 2: always */
  FCM_OPT_PROFILE = 8, /* 1: the loop kernel records a per-CTA timeline (fcm_last_profile) */
  FCM_OPT_SEED_PASS = 9, /* seeded start: 1 = the loop kernel generates u_0 as its pass 0, 0 = a
                           separate prologue kernel does, 2 (default) = auto: pass 0 for volumes of
                           <= 1024 tiles and in recompute mode, the prologue kernel above */
  FCM_OPT_RECOMPUTE = 11, /* 1: "effective" mode (uint8 pixels, m == 2, seeded start, loop kernel):
                           passes >= 2 read x only and write u_k; delta_k is taken between the fp64
                           intensity tables of passes k-1 and k over the intensities present
                           (u_{k-1} is recomputed from (x, v_{k-1}), never read back).  0: default */
  FCM_OPT_DEBUG_DELAY = 12, /* diagnostics: after every grid barrier of the loop kernel one CTA (a
                              different one each pass) sleeps this many ns (<= 10 ms) before it reads
                              the pass's partials -- results must not change (race test).  0: default */
  FCM_OPT_DEBUG_SHARED_PARTIALS = 13, /* diagnostics: 1 = every pass of the loop kernel's small-volume
                              path publishes its tile partials into the same buffer (the round-1
                              layout, racy under FCM_OPT_DEBUG_DELAY; shows the race test can fail).
                              0: default (two buffers alternated by pass parity) */
  FCM_OPT_PEER_TIMEOUT_MS = 14 /* multi-rank loop kernel: how long a rank waits for a peer's per-pass
                              root before failing fcm_run with FCM_E_NCCL naming the missing rank and
                              pass (default 4000).  Single-process multi-shard plans retry such a
                              failure with one launch per pass (fcm_last_timing out[6] counts it). */,
  FCM_OPT_DEBUG_SOLO_RANK = 15 /* diagnostics: a rank plan runs its slice alone (no root exchange; the
                              centers are the slice's, not the job's) -- the per-rank pass of an
                              N-GPU job timed on one GPU (tools/rank_proxy.py) */
} fcm_option;

typedef struct fcm_plan fcm_plan;

int fcm_abi_version(void);
const char* fcm_status_string(int status);
int fcm_device_count(int32_t* count);

/* ------------------------------------------------------------------------
 * Engine loop (replaces core._iterate / parallel._iterate)
 * ---------------------------------------------------------------------- */

/* Single-process plan over n voxels and c clusters (2 <= c <= 32), sharded
 * over nshards in {1,2,4,8} shards placed on devices[0..nshards-1] (a device
 * may repeat: shards on one GPU exercise the multi-GPU reduction exactly).
 * Mirrors run_fcm_parallel's workers= (parallel.py:334-362): results are
 * bit-identical for every shard count. */
int fcm_plan_create(fcm_plan** out, int64_t n, int32_t c, int32_t x_kind, int32_t nshards,
                    const int32_t* devices);

/* One rank of an nranks-process job (one process per GPU): the plan owns the
 * rank's contiguous voxel range (query it with fcm_plan_info) and exchanges
 * the 2c+2 reduction roots with ncclAllGather, or -- after fcm_connect_peers --
 * inside the loop kernel through peer-memory mailboxes.  nccl_id is the
 * 128-byte ncclUniqueId from fcm_nccl_unique_id on rank 0, or NULL for a
 * mailbox-only plan (a one-rank id still routes the roots through NCCL,
 * which tests use). */
int fcm_plan_create_rank(fcm_plan** out, int64_t n_global, int32_t c, int32_t x_kind,
                         int32_t device, int32_t nranks, int32_t rank, const void* nccl_id);
int fcm_nccl_unique_id(void* out128);

/* Multi-process ranks, fused exchange (loop kernel): the 64-byte CUDA IPC
 * handle of this rank's rank-root mailbox, and the connection of a rank plan
 * to every rank's mailbox (handles: nranks x 64 bytes, rank order, gathered
 * by the caller, e.g. torch.distributed.all_gather).  Once connected, fcm_run
 * runs the whole solve in one loop-kernel launch per rank and exchanges the
 * 2c+2-double roots with NVLink peer stores inside the kernel instead of an
 * ncclAllGather per pass. */
int fcm_mailbox_handle(fcm_plan* plan, void* out64);
int fcm_connect_peers(fcm_plan* plan, const void* handles, int32_t nranks);

/* Host-only: the voxel range and reduction-tree geometry of `rank` in an
 * nranks job over n voxels (no GPU needed).  out[0..]: n_local, voxel0,
 * tile voxels, tiles T, tiles per octant M, tree levels per octant, first octant,
 * octants, first tile, tiles_local. */
int fcm_geometry(int64_t n, int32_t nranks, int32_t rank, int64_t* out, int32_t count);

int fcm_plan_destroy(fcm_plan* plan);
const char* fcm_last_error(const fcm_plan* plan);
int fcm_set_option(fcm_plan* plan, int32_t key, int64_t value);

/* info[0..]: n_global, n_local (voxels of the plan's range: the whole image
 * for fcm_plan_create, the rank's slice for fcm_plan_create_rank), voxel0
 * (first voxel of that range), tile voxels, tiles (global), tiles of the
 * plan, grid of the last pass, nshards, bytes of device memory held. */
int fcm_plan_info(const fcm_plan* plan, int64_t* info, int32_t count);

/* Pixels of the plan's voxel range (whole image for fcm_plan_create, the
 * rank's [voxel0, voxel0 + n_local) slice for fcm_plan_create_rank), in the
 * plan's x_kind (uint8_t or double). */
int fcm_upload_pixels(fcm_plan* plan, const void* x);

/* Initial membership, exactly one of:
 *   fcm_init_membership  -- seeded SplitMix64 rows generated on the device,
 *                           bit-identical to core.init_membership
 *                           (_kernels.pyx:44-69); nothing crosses PCIe.
 *   fcm_upload_membership-- caller-provided AoS float64 rows of the plan's
 *                           voxel range (initial_membership=, core.py:135-143). */
int fcm_init_membership(fcm_plan* plan, uint64_t seed);
int fcm_upload_membership(fcm_plan* plan, const double* u0_aos);

/* Run the loop to convergence (delta < epsilon) or max_iters passes.
 * v_out[c] receives the centers that produced the final membership
 * (core.py:132), trace_out[max_iters] the objective per iteration.
 * Returns FCM_E_DEGENERATE with *dead_cluster set when a cluster weight sum
 * is exactly zero.  Each fcm_run restarts from the initial membership. */
int fcm_run(fcm_plan* plan, double m, double epsilon, int32_t max_iters, double* v_out,
            double* trace_out, int32_t* iterations, int32_t* converged, int32_t* dead_cluster);

/* Final membership (AoS float64, rows sum to 1 within 1e-9; types.py:82-85)
 * and defuzzified labels (argmax, ties -> lowest index; _kernels.pyx:223-238)
 * of the plan's voxel range.  Either pointer may be NULL. */
int fcm_download(fcm_plan* plan, double* u_aos_out, int32_t* labels_out);

/* fcm_download for uint8 plans without moving n*c doubles over PCIe: u_final
 * and the labels depend only on (x_i, v_final), so the epilogue is evaluated
 * for the 256 intensities (same kernel: bit-identical rows), 256*(8c+4) bytes
 * are copied back, and `nthreads` host threads (<= 0: all cores) expand the
 * rows along x_host -- the same pixels the plan uploaded (its voxel range) --
 * with streaming stores.  Output identical to fcm_download; the device labels
 * are still written for fcm_label_confusion / fcm_mask_overlap.
 * FCM_E_ARG for float64 plans.  Reference: core.py:132 / defuzzify core.py:94-102
 * (the FcmResult arrays); no reference counterpart for the table itself. */
int fcm_download_table(fcm_plan* plan, const uint8_t* x_host, double* u_aos_out, int32_t* labels_out,
                       int32_t nthreads);

/* Label statistics of the last solve, counted on the device from the labels
 * fcm_download left there (metrics.py:46-97: Dice and match_clusters need
 * only these integers).  ref_labels: int32 class per voxel of the plan's
 * range in [0, c_ref); conf_out[p*c_ref + r] = |pred==p & ref==r|.
 * mask: one byte per voxel (nonzero = set); counts_out[0..c) = |pred==p &
 * mask|, counts_out[c] = |mask|, counts_out[c+1+p] = |pred==p|. */
int fcm_label_confusion(fcm_plan* plan, const int32_t* ref_labels, int32_t c_ref, int64_t* conf_out);
int fcm_mask_overlap(fcm_plan* plan, const uint8_t* mask, int64_t* counts_out);

/* out[0..]: ms of the last fcm_run's device loop (start + passes, CUDA
 * events), ms per pass (FCM_OPT_TIMING: mean pass-kernel time; loop kernel:
 * its duration / passes, the seeded start included), prologue-kernel ms
 * (0 when the loop kernel generated u_0 itself), kernel launches of the
 * loop (1 for the loop kernel), passes that did work, 1 if the loop kernel
 * ran the seeded start as its pass 0, solves of this plan that fell back
 * from the multi-shard loop kernel to per-pass launches. */
int fcm_last_timing(const fcm_plan* plan, double* out, int32_t count);

/* delta_1..delta_k of the last fcm_run (out[0..min(count, iterations))):
 * max |u_k - u_{k-1}| per pass, as the stop test compared it with epsilon
 * (core.py:128-130).  Taken in fp64 against the fp32-stored u_{k-1} (within
 * 3e-8 of the reference's fp64 delta) and rounded UP to 20 mantissa bits, so
 * the stop test never fires early; parity tests log |delta - epsilon| of the
 * last two passes against that error. */
int fcm_delta_trace(const fcm_plan* plan, double* out, int32_t count);

/* Loop-kernel timeline of the last fcm_run with FCM_OPT_PROFILE (diagnostics):
 * out[(pass * grid + cta) * 16 + k], k = 0 pass start, 1 producer done claiming,
 * 2 consumers done, 3 grid barrier released (globaltimer ns), 4 tiles claimed.
 * count must be >= passes * grid * 16; passes <= min(max_iters, 64). */
int fcm_last_profile(const fcm_plan* plan, uint64_t* out, int64_t count, int32_t* passes, int32_t* grid);

/* The 256-row result table of the last fcm_download_table: u_tab[b*c + j] is
 * the fp64 membership row and l_tab[b] the label of intensity b.  Every row
 * of the expanded result is a copy of one of these, so validating the table
 * validates the result (types.py:82-85) without a pass over n*c doubles. */
int fcm_result_table(const fcm_plan* plan, double* u_tab, int32_t* l_tab);

/* Host-only: float64 intensities -> x_kind (FCM_X_U8: every value an integer
 * in 0..255; FCM_X_U16: in 0..65535) on nthreads threads (<= 0: all cores),
 * check and conversion in one pass.  FCM_E_ARG (out unspecified) when any
 * value does not convert exactly.  The drop-in uses it to pick the narrowest
 * exact device representation of GrayImage.pixels (types.py:38-41). */
int fcm_narrow_pixels(const double* x, int64_t n, int32_t x_kind, void* out, int32_t nthreads);

/* Page-lock caller memory so uploads/downloads run at full PCIe speed. */
int fcm_host_register(void* ptr, int64_t bytes);
int fcm_host_unregister(void* ptr);

/* ------------------------------------------------------------------------
 * Kernel seam (_kernels.pyx), host buffers, one call = one GPU op
 * ---------------------------------------------------------------------- */
int fcm_fill_membership_random(double* u_out, int64_t n, int32_t c, uint64_t seed, int32_t device);
int fcm_update_centers(const double* x, const double* u, double* v_out, int64_t n, int32_t c,
                       double m, int32_t device, int32_t* dead_out);
int fcm_update_membership(const double* x, const double* v, double* u_out, int64_t n, int32_t c,
                          double m, int32_t device);
int fcm_objective(const double* x, const double* u, const double* v, int64_t n, int32_t c,
                  double m, int32_t device, double* out);
int fcm_max_abs_diff(const double* a, const double* b, int64_t count, int32_t device, double* out);
int fcm_argmax_rows(const double* u, int32_t* labels_out, int64_t n, int32_t c, int32_t device);

/* Diagnostics (no reference counterpart): the seeded start's branch-free
 * correctly rounded reciprocal against CUDA's __drcp_rn on n pseudo-random
 * row totals in [2^-53, 64); *mismatches = how many differ (expected 0). */
int fcm_check_rcp(int64_t n, uint64_t seed, int32_t device, int64_t* mismatches);

#ifdef __cplusplus
}
#endif
#endif /* FCM_B200_H */

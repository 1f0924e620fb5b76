// fcm_api.cu -- host runtime behind include/fcm_b200.h.
//
// A plan owns, per shard: the pixels (uint8 or fp64, padded to whole tiles),
// two fp32 SoA membership buffers (u_{k-1}, u_k), the reduction tree scratch
// and a Control block.  fcm_run enqueues prologue + passes in batches on the
// shard streams and only syncs once per batch to read the device `done` flag
// (core._iterate's Python loop, core.py:105-132, becomes a device loop).
#include <dlfcn.h>
#include <sys/mman.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include <emmintrin.h>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost nothing without a tool attached

#include "../../include/fcm_b200.h"
#include "fcm_kernels.h"
#include "fcm_ops.h"

using namespace fcm;

static size_t xkind_bytes(int xkind) {  // bytes per voxel of x in HBM
  return xkind == XK_U8 ? 1 : (xkind == XK_U16 ? 2 : 8);
}

// Host-only: float64 intensities -> the narrowest exact plan kind.  Every
// value must be an integer in range (NaN, negatives and fractions fail);
// the check and the conversion are one pass on `nthreads` threads.
namespace {
template <typename T>
bool narrow_block(const double* x, int64_t i0, int64_t i1, T* out) {
  const double hi = (double)std::numeric_limits<T>::max();
  bool ok = true;
  for (int64_t i = i0; i < i1; ++i) {
    const double v = x[i];
    const bool in = v >= 0.0 && v <= hi;  // false for NaN
    const T t = in ? (T)v : (T)0;
    ok &= in && (double)t == v;
    out[i] = t;
  }
  return ok;
}
}  // namespace


// ------------------------------------------------------------------ NCCL ---
// Loaded on first use so the library (and single-GPU plans) do not depend on
// libnccl being present.
namespace {
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

bool load_nccl() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  const char* names[] = {"libnccl.so.2", "libnccl.so", nullptr};
  void* h = nullptr;
  const char* env = getenv("FCM_NCCL_LIB");
  if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  for (int i = 0; !h && names[i]; ++i) h = dlopen(names[i], RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllGather && g_nccl.CommDestroy;
  return g_nccl.ok;
}
}  // namespace

// ------------------------------------------------------------------ plan ---
namespace {
struct Shard {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_pass = nullptr;
  Geometry g{};
  void* x = nullptr;
  float* u = nullptr;  // fp32 SoA membership, updated in place pass after pass
  int keep_l2 = 0;     // x + u fit in L2 (evict_last policy on the stream)
  double* u0_aos = nullptr;
  double* tile_part = nullptr;
  double* node_part[kMaxLevels + 1] = {};  // level l >= 1: [noct][nodes[l]][nf]
  uint8_t* tab_x = nullptr;                // fcm_download_table: intensities 0..255
  double* tab_u = nullptr;                 //   their fp64 membership rows
  int32_t* tab_l = nullptr;                //   and labels
  double* l1_buf = nullptr;                // loop kernel: [3][noct][nodes[1]][nf] (pass generation mod 3)
  Mailbox* mbox = nullptr;                 // loop kernel: rank-root mailbox (own allocation: IPC-exportable)
  double* rank_root = nullptr;  // [2][nf], double-buffered by pass parity
  double* gathered = nullptr;   // [nranks][nf] (NCCL)
  unsigned* node_cnt[kMaxLevels + 1] = {};
  size_t cnt_total = 0;  // counters of all levels, one allocation (node_cnt[1] is its base)
  Control* ctl = nullptr;
  double* trace = nullptr;
  int trace_cap = 0;
  double* out_u = nullptr;
  int32_t* out_labels = nullptr;
  int last_grid = 0;
  std::vector<void*> allocs;
};
}  // namespace

struct fcm_plan {
  int64_t n_global = 0;
  int c = 0;
  int xkind = XK_U8;
  int nshards = 1;     // shards driven by this process
  int nranks = 1;      // ranks of the whole job (== nshards for single-process plans)
  int rank = 0;        // rank of shard 0 (NCCL plans)
  bool use_nccl = false;
  ncclComm_t comm = nullptr;
  Shard sh[kOctants];
  int init_src = 0;  // 0 none, 1 seed, 2 uploaded AoS
  uint64_t seed = 0;
  bool x_ready = false;
  bool run_ok = false;
  int mode = MODE_M2;
  Powers pw{};
  int batch = 8;
  int timing = 0;
  int force_grid = 0;
  int variant = 0;  // pass kernel: 0 TMA pipeline (auto), 1 register-staged LDG, 2 TMA + intensity table
  // graph mode: prologue + while(!done) { pass; pass } as ONE CUDA graph with a
  // device-side conditional loop -- no host round trip per iteration
  int use_graph = 1;
  // loop mode: prologue + ONE persistent cooperative kernel running every
  // pass with grid barriers in between (single-shard, single-rank plans)
  int use_loop = 1;
  int l2_mode = 1;  // 0 never keep x/u in L2, 1 when they fit (default), 2 always
  int profile = 0;  // record the loop kernel's per-CTA timeline
  int seed_pass = 2;  // seeded u_0: 1 = loop kernel's pass 0, 0 = prologue kernel, 2 = auto (by volume)
  int recompute = 0;  // loop kernel: "effective" mode, passes >= 2 stream x only
  std::vector<double> deltas;  // delta_1..delta_k of the last fcm_run
  std::vector<double> res_tab_u;  // the 256-row result table of the last fcm_download_table
  int32_t res_tab_l[256] = {};
  unsigned debug_delay_ns = 0;  // loop kernel: one CTA per pass sleeps after the grid barrier (tests)
  int debug_shared_parts = 0;   // loop kernel: single tile-partial buffer (the racy round-1 layout; tests)
  int solo_rank = 0;            // diagnostics: a rank plan solves its slice without the exchange
  int64_t peer_timeout_ms = 4000;  // loop kernel, multi-rank: how long to wait for a peer's root
  bool force_per_pass = false;  // fcm_run retry after a failed multi-shard loop (shards sharing a device)
  bool looped_last = false;     // the last run_impl ran the loop kernel
  int loop_fallbacks = 0;       // solves that fell back to per-pass launches
  bool labels_valid = false;    // device labels belong to the last successful fcm_run
  unsigned run_counter = 0;  // fcm_run calls (mailbox tags); identical on every rank
  bool p2p_ready = false;    // multi-process ranks: peer mailboxes mapped (fcm_connect_peers)
  Mailbox* peer_mbox[kOctants] = {};
  bool peer_opened[kOctants] = {};
  uint64_t* prof = nullptr;
  int prof_passes = 0, prof_grid = 0;
  bool capturing = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraphConditionalHandle gcond = 0;
  struct GraphKey {
    double m, eps;
    int max_iters, init_src, variant, force_grid, l2_mode;
    uint64_t seed;
  } gkey{};
  Control* host_ctl = nullptr;   // pinned: device -> host reads of the control block
  Control* host_tmpl = nullptr;  // pinned: reset template copied to every shard
  // pageable host -> device uploads (fcm_upload_pixels / _membership):
  // kStageThreads host threads, each with its own stream and two pinned slots
  char* stage_pinned = nullptr;
  cudaStream_t stage_st[16] = {};
  cudaEvent_t stage_ev[16][2] = {};
  std::vector<cudaEvent_t> ev_t0, ev_t1;
  cudaEvent_t ev_start = nullptr, ev_pro = nullptr, ev_end = nullptr;
  double t_loop_ms = 0, t_pass_ms = 0, t_pro_ms = 0;
  int passes_launched = 0, passes_done = 0;
  int seeded_in_loop = 0;  // last run: the loop kernel generated u_0 itself (pass 0)
  int64_t dev_bytes = 0;
  std::string err;
};

namespace {
int fail(fcm_plan* p, int code, const char* fmt, ...) {
  if (p) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    p->err = buf;
  }
  return code;
}

#define CK(expr)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(p, FCM_E_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),      \
                  __FILE__, __LINE__);                                                        \
  } while (0)

// NVTX range for the host-side phases (Nsight Systems / ncu --nvtx timelines):
// uploads, the solve (prologue, loop-kernel launch, per-pass launches),
// downloads and the host table expansion.  Per-pass phases
// inside the persistent loop kernel come from its device timeline
// (FCM_OPT_PROFILE, tools/pass_phases.py) instead.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

int nf_of(int c) { return 2 * c + 2; }

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Global tile tree ("Deterministic reduction").  Depends only on n.
// Tile = 8192 voxels (8 TMA chunks) unless that leaves fewer than 100 tiles,
// then halved down to 1024; above 64 tiles per CTA of a full B200 (2 x 148
// CTAs) it doubles.  Measured per-pass times (tools/tile_sweep.py, C2/C4
// bench): the per-tile reduction handoff costs more than the end-of-pass
// imbalance of larger tiles down to ~100 tiles per volume (C1 1024, C3-200K
// 2048, C3-1M/C2/C4 8192).  Beyond 8 * 32^3 tiles they grow further.
void base_geometry(int64_t n, Geometry& g) {
  int64_t tile = 8192;
  while (tile > 1024 && ceil_div(n, tile) < 100) tile >>= 1;
  while (ceil_div(n, tile) > int64_t(64) * 296) tile <<= 1;
  if (const char* e = getenv("FCM_TILE_EXPERIMENT")) tile = std::max<int64_t>(1024, atoll(e));  // A/B only
  const int64_t cap = (int64_t)kOctants << (5 * kMaxLevels);
  while (ceil_div(n, tile) > cap) tile <<= 1;
  int shift = 0;
  while ((int64_t(1) << shift) < tile) ++shift;
  g.n_global = n;
  g.tile_shift = shift;
  g.T = (int)ceil_div(n, tile);
  const int T8 = (int)ceil_div(g.T, kOctants) * kOctants;
  g.M = T8 / kOctants;
  g.levels = 1;
  while ((int64_t(1) << (5 * g.levels)) < g.M) ++g.levels;
  for (int l = 0; l <= kMaxLevels; ++l)
    g.nodes[l] = l <= g.levels ? (int)ceil_div(g.M, int64_t(1) << (5 * l)) : 0;
}

void rank_geometry(Geometry& g, int nranks, int rank) {
  const int64_t tile = int64_t(1) << g.tile_shift;
  g.nranks = nranks;
  g.rank = rank;
  g.noct = kOctants / nranks;
  g.oct0 = rank * g.noct;
  g.tile0 = g.oct0 * g.M;
  const int tend = std::min((g.oct0 + g.noct) * g.M, g.T);
  g.tiles_local = std::max(0, tend - g.tile0);
  g.voxel0 = (int64_t)g.tile0 * tile;
  const int64_t vend = std::min((int64_t)tend * tile, g.n_global);
  g.n_local = std::max<int64_t>(0, vend - g.voxel0);
  if (g.tiles_local == 0) g.voxel0 = std::min(g.voxel0, g.n_global);
  g.plane = (int64_t)std::max(g.tiles_local, 1) * tile;
}

template <typename T>
int dalloc(fcm_plan* p, Shard& s, T** ptr, size_t count) {
  void* q = nullptr;
  size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(p, FCM_E_NOMEM, "cudaMalloc(%zu bytes) on device %d failed: %s", bytes, s.device,
                cudaGetErrorString(e));
  }
  s.allocs.push_back(q);
  p->dev_bytes += (int64_t)bytes;
  *ptr = (T*)q;
  return FCM_OK;
}

int setup_shard(fcm_plan* p, Shard& s) {
  CK(cudaSetDevice(s.device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, s.device));
  if (prop.major < 10)
    return fail(p, FCM_E_CUDA, "device %d is sm_%d%d; this build targets sm_100a", s.device,
                prop.major, prop.minor);
  s.sms = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&s.ev_pass, cudaEventDisableTiming));
  const int nf = nf_of(p->c);
  const size_t xsz = xkind_bytes(p->xkind);
  int rc;
  uint8_t* xb = nullptr;
  if ((rc = dalloc(p, s, &xb, s.g.plane * xsz))) return rc;
  s.x = xb;
  CK(cudaMemsetAsync(s.x, 0, s.g.plane * xsz, s.stream));
  if ((rc = dalloc(p, s, &s.u, (size_t)s.g.plane * p->c))) return rc;
  const double resident = (double)s.g.plane * (double)(xsz + 4 * p->c);
  s.keep_l2 = resident <= 0.8 * (double)prop.l2CacheSize ? 1 : 0;
  if ((rc = dalloc(p, s, &s.tile_part, (size_t)3 * std::max(s.g.tiles_local, 1) * nf))) return rc;
  size_t cnt_total = 0;
  for (int l = 1; l <= s.g.levels; ++l) {
    if ((rc = dalloc(p, s, &s.node_part[l], (size_t)s.g.noct * s.g.nodes[l] * nf))) return rc;
    cnt_total += (size_t)s.g.noct * s.g.nodes[l];
  }
  if ((rc = dalloc(p, s, &s.rank_root, (size_t)2 * nf))) return rc;
  if ((rc = dalloc(p, s, &s.gathered, (size_t)p->nranks * nf))) return rc;
  if ((rc = dalloc(p, s, &s.l1_buf, (size_t)3 * s.g.noct * s.g.nodes[1] * nf))) return rc;
  if ((rc = dalloc(p, s, &s.mbox, 1))) return rc;
  CK(cudaMemsetAsync(s.mbox, 0, sizeof(Mailbox), s.stream));
  unsigned* cnt = nullptr;
  if ((rc = dalloc(p, s, &cnt, cnt_total))) return rc;
  s.cnt_total = cnt_total;
  for (int l = 1; l <= s.g.levels; ++l) {
    s.node_cnt[l] = cnt;
    cnt += (size_t)s.g.noct * s.g.nodes[l];
  }
  if ((rc = dalloc(p, s, &s.ctl, 1))) return rc;
  CK(cudaMemsetAsync(s.node_cnt[1], 0, sizeof(unsigned) * s.cnt_total, s.stream));
  CK(cudaMemsetAsync(s.ctl, 0, sizeof(Control), s.stream));
  // every tree slot starts unpublished (all-ones NaN pattern, see fcm_kernels.cuh)
  CK(cudaMemsetAsync(s.tile_part, 0xff, sizeof(double) * 3 * std::max(s.g.tiles_local, 1) * nf, s.stream));
  for (int l = 1; l <= s.g.levels; ++l)
    CK(cudaMemsetAsync(s.node_part[l], 0xff, sizeof(double) * s.g.noct * s.g.nodes[l] * nf, s.stream));
  return FCM_OK;
}

void drop_graph(fcm_plan* p);
void release(fcm_plan* p) {
  for (int i = 0; i < p->nshards; ++i) {
    Shard& s = p->sh[i];
    cudaSetDevice(s.device);
    if (s.stream) cudaStreamSynchronize(s.stream);
    for (void* q : s.allocs) cudaFree(q);
    s.allocs.clear();
    if (s.ev_pass) cudaEventDestroy(s.ev_pass);
    if (s.stream) cudaStreamDestroy(s.stream);
  }
  if (p->nshards > 0) cudaSetDevice(p->sh[0].device);
  for (auto e : p->ev_t0) cudaEventDestroy(e);
  for (auto e : p->ev_t1) cudaEventDestroy(e);
  if (p->ev_start) cudaEventDestroy(p->ev_start);
  if (p->ev_pro) cudaEventDestroy(p->ev_pro);
  if (p->ev_end) cudaEventDestroy(p->ev_end);
  if (p->host_ctl) cudaFreeHost(p->host_ctl);
  if (p->host_tmpl) cudaFreeHost(p->host_tmpl);
  if (p->stage_pinned) {
    cudaFreeHost(p->stage_pinned);
    for (int t = 0; t < 16; ++t) {
      if (p->stage_st[t]) cudaStreamDestroy(p->stage_st[t]);
      for (int k = 0; k < 2; ++k)
        if (p->stage_ev[t][k]) cudaEventDestroy(p->stage_ev[t][k]);
    }
  }
  drop_graph(p);
  for (int r = 0; r < kOctants; ++r)
    if (p->peer_opened[r]) cudaIpcCloseMemHandle(p->peer_mbox[r]);
  if (p->comm && g_nccl.ok) g_nccl.CommDestroy(p->comm);
}

int common_setup(fcm_plan* p) {
  int rc;
  for (int i = 0; i < p->nshards; ++i)
    if ((rc = setup_shard(p, p->sh[i]))) return rc;
  // Peer access for single-process multi-device plans: each finalize reads
  // every shard's 2c+2-double root directly over NVLink.
  for (int i = 0; i < p->nshards; ++i)
    for (int j = 0; j < p->nshards; ++j) {
      const int di = p->sh[i].device, dj = p->sh[j].device;
      if (di == dj) continue;
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, di, dj));
      if (!can) return fail(p, FCM_E_CUDA, "device %d cannot access peer %d", di, dj);
      CK(cudaSetDevice(di));
      cudaError_t e = cudaDeviceEnablePeerAccess(dj, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
      cudaGetLastError();
    }
  CK(cudaSetDevice(p->sh[0].device));
  CK(cudaMallocHost(&p->host_ctl, sizeof(Control)));
  CK(cudaMallocHost(&p->host_tmpl, sizeof(Control)));
  CK(cudaEventCreate(&p->ev_start));
  CK(cudaEventCreate(&p->ev_pro));
  CK(cudaEventCreate(&p->ev_end));
  for (int i = 0; i < p->nshards; ++i) {
    CK(cudaSetDevice(p->sh[i].device));
    CK(cudaStreamSynchronize(p->sh[i].stream));
  }
  return FCM_OK;
}

void set_powers(fcm_plan* p, double m) {
  Powers& w = p->pw;
  w.m = m;
  w.p = 2.0 / (m - 1.0);  // _kernels.pyx:96
  const double pr = std::nearbyint(w.p);
  if (w.p == pr && pr >= 1.0 && pr <= 64.0) {
    w.pkind = PK_INT;
    w.pint = (int)pr;
  } else {
    w.pkind = PK_REAL;
    w.pint = 0;
  }
  const double mr = std::nearbyint(m), m2 = std::nearbyint(2.0 * m);
  if (m == mr && m <= 64.0) {
    w.mkind = MK_INT;
    w.mint = (int)mr;
  } else if (2.0 * m == m2 && m <= 64.0) {
    w.mkind = MK_HALF;
    w.mint = (int)std::floor(m);
  } else {
    w.mkind = MK_REAL;
    w.mint = 0;
  }
  p->mode = (m == 2.0) ? MODE_M2 : MODE_GEN;
}

PassArgs make_args(fcm_plan* p, Shard& s, int seq, double eps, int max_iters) {
  PassArgs a{};
  const int nf = nf_of(p->c);
  a.x = s.x;
  a.u_cur = s.u;  // in place: each element is read before the same thread rewrites it
  a.u_nxt = s.u;
  a.u0_aos = s.u0_aos;
  a.seed = p->seed;
  a.c = p->c;
  a.m = p->pw.m;
  a.p = p->pw.p;
  a.pkind = p->pw.pkind;
  a.pint = p->pw.pint;
  a.mkind = p->pw.mkind;
  a.mint = p->pw.mint;
  a.eps = eps;
  a.max_iters = max_iters;
  a.seq = seq;
  a.g = s.g;
  a.tile_part = s.tile_part;
  for (int l = 0; l <= kMaxLevels; ++l) {
    a.node_part[l] = s.node_part[l];
    a.node_cnt[l] = s.node_cnt[l];
  }
  a.rank_root = s.rank_root + (seq & 1) * nf;
  a.ctl = s.ctl;
  a.trace = s.trace;
  a.cond = p->gcond;
  a.use_cond = p->capturing ? 1 : 0;
  a.finalize_local = (p->nranks == 1 && !p->use_nccl) ? 1 : 0;
  a.keep_l2 = p->l2_mode == 2 ? 1 : (p->l2_mode == 1 ? s.keep_l2 : 0);
  a.l1_buf = s.l1_buf;
  return a;
}

// Launch one prologue (seq == 0) or pass on every shard, then -- when the
// job has more than one rank -- exchange the roots and finalize everywhere.
int step(fcm_plan* p, int seq, double eps, int max_iters) {
  char label[32];
  snprintf(label, sizeof label, seq == 0 ? "fcm prologue" : "fcm pass %d", seq);
  NvtxRange nv(label);
  const int nf = nf_of(p->c);
  const bool prologue = seq == 0;
  for (int i = 0; i < p->nshards; ++i) {
    Shard& s = p->sh[i];
    CK(cudaSetDevice(s.device));
    const PassArgs a = make_args(p, s, seq, eps, max_iters);
    if (s.g.tiles_local == 0) {
      CK(cudaMemsetAsync(a.rank_root, 0, sizeof(double) * nf, s.stream));
    } else if (prologue) {
      CK(launch_prologue(p->xkind, p->c, p->mode, p->init_src == 1, a, s.sms, s.stream));
    } else {
      int grid = 0;
      const bool t = p->timing && i == 0;
      if (t) {
        size_t k = (size_t)p->passes_launched;
        while (p->ev_t0.size() <= k) {
          cudaEvent_t e0, e1;
          CK(cudaEventCreate(&e0));
          CK(cudaEventCreate(&e1));
          p->ev_t0.push_back(e0);
          p->ev_t1.push_back(e1);
        }
        CK(cudaEventRecord(p->ev_t0[k], s.stream));
      }
      PassArgs b = a;
      CK(launch_pass(p->xkind, p->c, p->mode, b, s.sms, s.stream, &grid, p->variant, p->force_grid));
      if (t) CK(cudaEventRecord(p->ev_t1[(size_t)p->passes_launched], s.stream));
      s.last_grid = grid;
    }
  }
  if (!prologue) p->passes_launched++;
  if (p->nranks == 1 && !p->use_nccl) return FCM_OK;

  FinalizeArgs f{};
  f.nranks = p->nranks;
  f.c = p->c;
  f.eps = eps;
  f.max_iters = max_iters;
  f.prologue = prologue ? 1 : 0;
  f.cond = p->gcond;
  f.use_cond = p->capturing ? 1 : 0;
  if (p->use_nccl) {
    Shard& s = p->sh[0];
    ncclResult_t r = g_nccl.AllGather(s.rank_root + (seq & 1) * nf, s.gathered, (size_t)nf,
                                      ncclDouble, p->comm, s.stream);
    if (r != ncclSuccess)
      return fail(p, FCM_E_NCCL, "ncclAllGather: %s", g_nccl.GetErrorString(r));
    for (int r2 = 0; r2 < p->nranks; ++r2) f.roots[r2] = s.gathered + r2 * nf;
    f.ctl = s.ctl;
    f.trace = s.trace;
    CK(launch_finalize(f, s.stream));
    return FCM_OK;
  }
  for (int i = 0; i < p->nshards; ++i) {
    CK(cudaSetDevice(p->sh[i].device));
    CK(cudaEventRecord(p->sh[i].ev_pass, p->sh[i].stream));
  }
  for (int r2 = 0; r2 < p->nshards; ++r2) f.roots[r2] = p->sh[r2].rank_root + (seq & 1) * nf;
  for (int i = 0; i < p->nshards; ++i) {
    Shard& s = p->sh[i];
    CK(cudaSetDevice(s.device));
    for (int j = 0; j < p->nshards; ++j)
      if (j != i) CK(cudaStreamWaitEvent(s.stream, p->sh[j].ev_pass, 0));
    f.ctl = s.ctl;
    f.trace = s.trace;
    CK(launch_finalize(f, s.stream));
  }
  return FCM_OK;
}

int check_plan(fcm_plan* p) { return p ? FCM_OK : FCM_E_ARG; }

void drop_graph(fcm_plan* p) {
  if (p->gexec) cudaGraphExecDestroy(p->gexec);
  if (p->graph) cudaGraphDestroy(p->graph);
  p->gexec = nullptr;
  p->graph = nullptr;
}

// prologue -> while (cond) { pass(odd); pass(even) } on shard 0's stream.
// The conditional handle defaults to 1 at every launch; whichever kernel
// observes `done` (finalize, or an early-exiting pass) sets it to 0.
int build_graph(fcm_plan* p, double eps, int max_iters) {
  drop_graph(p);
  Shard& s = p->sh[0];
  CK(cudaSetDevice(s.device));
  CK(cudaGraphCreate(&p->graph, 0));
  CK(cudaGraphConditionalHandleCreate(&p->gcond, p->graph, 1u, cudaGraphCondAssignDefault));
  p->capturing = true;
  int rc = FCM_OK;
  cudaGraph_t g_out = nullptr;
  if (cudaStreamBeginCaptureToGraph(s.stream, p->graph, nullptr, nullptr, 0,
                                    cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    p->capturing = false;
    return fail(p, FCM_E_CUDA, "cudaStreamBeginCaptureToGraph failed");
  }
  rc = step(p, 0, eps, max_iters);
  cudaError_t ec = cudaStreamEndCapture(s.stream, &g_out);
  if (rc || ec != cudaSuccess) {
    p->capturing = false;
    drop_graph(p);
    return rc ? rc : fail(p, FCM_E_CUDA, "prologue capture: %s", cudaGetErrorString(ec));
  }
  size_t nn = 0;
  CK(cudaGraphGetNodes(p->graph, nullptr, &nn));
  std::vector<cudaGraphNode_t> deps(nn);
  CK(cudaGraphGetNodes(p->graph, deps.data(), &nn));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = p->gcond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  CK(cudaGraphAddNode(&cnode, p->graph, deps.data(), nn, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if (cudaStreamBeginCaptureToGraph(s.stream, body, nullptr, nullptr, 0,
                                    cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    p->capturing = false;
    drop_graph(p);
    return fail(p, FCM_E_CUDA, "body capture failed");
  }
  rc = step(p, 1, eps, max_iters);
  if (!rc) rc = step(p, 2, eps, max_iters);
  ec = cudaStreamEndCapture(s.stream, &g_out);
  p->capturing = false;
  if (rc || ec != cudaSuccess) {
    drop_graph(p);
    return rc ? rc : fail(p, FCM_E_CUDA, "body capture: %s", cudaGetErrorString(ec));
  }
  ec = cudaGraphInstantiate(&p->gexec, p->graph, 0);
  if (ec != cudaSuccess) {
    drop_graph(p);
    return fail(p, FCM_E_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ec));
  }
  return FCM_OK;
}
}  // namespace

constexpr int kSmallTilesHost = 1024;  // = kSmallTiles (fcm_tma_pipe.cuh): the loop kernel's small-volume bound

// ================================================================== C ABI ==
// host-side row expansion for fcm_download_table (below)
namespace {

// madvise(MADV_HUGEPAGE) on the 2 MB-aligned interior of [p, p + bytes).
void advise_huge(void* p, size_t bytes) {
  static const bool off = getenv("FCM_NO_HUGEPAGE") != nullptr;  // A/B switch (diagnostics)
  if (off || !p || bytes < ((size_t)4 << 20)) return;
  const uintptr_t a = ((uintptr_t)p + ((1u << 21) - 1)) & ~(uintptr_t)((1u << 21) - 1);
  const uintptr_t e = ((uintptr_t)p + bytes) & ~(uintptr_t)((1u << 21) - 1);
  if (e > a) madvise((void*)a, e - a, MADV_HUGEPAGE);
}

// SM count of a device, cached (the seam ops size their grids by it).
int device_sms(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v < 1) v = 148;
    cache[device] = v;
  }
  return cache[device];
}

template <int C>
void expand_u_c(const uint8_t* x, int64_t i0, int64_t i1, const double* tab, double* u) {
  double* o = u + i0 * C;
  int64_t i = i0;
  if (C % 2 == 0) {
    for (; i < i1; ++i) {
      const double* t = tab + (int)x[i] * C;
      for (int k = 0; k < C / 2; ++k) _mm_stream_pd(o + 2 * k, _mm_loadu_pd(t + 2 * k));
      o += C;
    }
  } else {
    for (; i + 2 <= i1; i += 2) {  // two rows = C aligned 16-byte stores
      double r[2 * C];
      const double* t0 = tab + (int)x[i] * C;
      const double* t1 = tab + (int)x[i + 1] * C;
      for (int k = 0; k < C; ++k) {
        r[k] = t0[k];
        r[C + k] = t1[k];
      }
      for (int k = 0; k < C; ++k) _mm_stream_pd(o + 2 * k, _mm_loadu_pd(r + 2 * k));
      o += 2 * C;
    }
    for (; i < i1; ++i, o += C) std::memcpy(o, tab + (int)x[i] * C, sizeof(double) * C);
  }
}

void expand_block(const uint8_t* x, int64_t i0, int64_t i1, int c, const double* tab, const int32_t* ltab,
                  double* u, int32_t* lab) {
  if (u) {
    const bool aligned = (reinterpret_cast<uintptr_t>(u + i0 * c) & 15) == 0;
    switch (aligned ? c : 0) {
      case 2: expand_u_c<2>(x, i0, i1, tab, u); break;
      case 3: expand_u_c<3>(x, i0, i1, tab, u); break;
      case 4: expand_u_c<4>(x, i0, i1, tab, u); break;
      case 5: expand_u_c<5>(x, i0, i1, tab, u); break;
      case 6: expand_u_c<6>(x, i0, i1, tab, u); break;
      case 7: expand_u_c<7>(x, i0, i1, tab, u); break;
      case 8: expand_u_c<8>(x, i0, i1, tab, u); break;
      default:
        for (int64_t i = i0; i < i1; ++i) std::memcpy(u + i * c, tab + (int)x[i] * c, sizeof(double) * c);
    }
  }
  if (lab) {
    int64_t i = i0;
    for (; i < i1 && (reinterpret_cast<uintptr_t>(lab + i) & 15); ++i) lab[i] = ltab[x[i]];
    for (; i + 4 <= i1; i += 4)
      _mm_stream_si128(reinterpret_cast<__m128i*>(lab + i),
                       _mm_set_epi32(ltab[x[i + 3]], ltab[x[i + 2]], ltab[x[i + 1]], ltab[x[i]]));
    for (; i < i1; ++i) lab[i] = ltab[x[i]];
  }
  _mm_sfence();
}

}  // namespace

extern "C" {

int fcm_abi_version(void) { return FCM_ABI_VERSION; }

const char* fcm_status_string(int status) {
  switch (status) {
    case FCM_OK: return "ok";
    case FCM_E_ARG: return "invalid argument";
    case FCM_E_CUDA: return "CUDA error";
    case FCM_E_NCCL: return "NCCL error";
    case FCM_E_DEGENERATE: return "degenerate cluster";
    case FCM_E_STATE: return "invalid call order";
    case FCM_E_NOMEM: return "out of device memory";
    default: return "unknown status";
  }
}

int fcm_device_count(int32_t* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (count) *count = 0;
    return FCM_E_CUDA;
  }
  if (count) *count = n;
  return FCM_OK;
}

static int validate_create(int64_t n, int32_t c, int32_t x_kind) {
  if (n < 1 || c < 2 || c > kCMaxSupported || n < c) return FCM_E_ARG;
  if (x_kind != FCM_X_U8 && x_kind != FCM_X_U16 && x_kind != FCM_X_F64) return FCM_E_ARG;
  if (n > (int64_t)8192 * (int64_t(1) << 30)) return FCM_E_ARG;
  return FCM_OK;
}

int fcm_plan_create(fcm_plan** out, int64_t n, int32_t c, int32_t x_kind, int32_t nshards,
                    const int32_t* devices) {
  if (!out) return FCM_E_ARG;
  *out = nullptr;
  if (validate_create(n, c, x_kind)) return FCM_E_ARG;
  if (nshards != 1 && nshards != 2 && nshards != 4 && nshards != 8) return FCM_E_ARG;
  fcm_plan* p = new fcm_plan();
  p->n_global = n;
  p->c = c;
  p->xkind = x_kind == FCM_X_U8 ? XK_U8 : (x_kind == FCM_X_U16 ? XK_U16 : XK_F64);
  p->nshards = nshards;
  p->nranks = nshards;
  Geometry base{};
  base_geometry(n, base);
  for (int i = 0; i < nshards; ++i) {
    p->sh[i].device = devices ? devices[i] : 0;
    p->sh[i].g = base;
    rank_geometry(p->sh[i].g, nshards, i);
  }
  int rc = common_setup(p);
  if (rc) {
    fprintf(stderr, "fcm_plan_create: %s\n", p->err.c_str());
    release(p);
    delete p;
    return rc;
  }
  *out = p;
  return FCM_OK;
}

int fcm_geometry(int64_t n, int32_t nranks, int32_t rank, int64_t* out, int32_t count) {
  if (!out || n < 1 || (nranks != 1 && nranks != 2 && nranks != 4 && nranks != 8) || rank < 0 ||
      rank >= nranks)
    return FCM_E_ARG;
  Geometry g{};
  base_geometry(n, g);
  rank_geometry(g, nranks, rank);
  const int64_t v[] = {g.n_local, g.voxel0, int64_t(1) << g.tile_shift, g.T, g.M,
                       g.levels, g.oct0, g.noct, g.tile0, g.tiles_local};
  for (int i = 0; i < count && i < (int)(sizeof v / sizeof v[0]); ++i) out[i] = v[i];
  return FCM_OK;
}

int fcm_nccl_unique_id(void* out128) {
  if (!out128) return FCM_E_ARG;
  if (!load_nccl()) return FCM_E_NCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return FCM_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out128, &id, sizeof id);
  return FCM_OK;
}

int fcm_plan_create_rank(fcm_plan** out, int64_t n_global, int32_t c, int32_t x_kind,
                         int32_t device, int32_t nranks, int32_t rank, const void* nccl_id) {
  if (!out) return FCM_E_ARG;
  *out = nullptr;
  if (validate_create(n_global, c, x_kind)) return FCM_E_ARG;
  if (nranks != 1 && nranks != 2 && nranks != 4 && nranks != 8) return FCM_E_ARG;
  if (rank < 0 || rank >= nranks) return FCM_E_ARG;
  fcm_plan* p = new fcm_plan();
  p->n_global = n_global;
  p->c = c;
  p->xkind = x_kind == FCM_X_U8 ? XK_U8 : (x_kind == FCM_X_U16 ? XK_U16 : XK_F64);
  p->nshards = 1;
  p->nranks = nranks;
  p->rank = rank;
  p->sh[0].device = device;
  base_geometry(n_global, p->sh[0].g);
  rank_geometry(p->sh[0].g, nranks, rank);
  int rc = common_setup(p);
  // nranks == 1 with an id still builds a (one-rank) communicator: the NCCL
  // exchange path then runs end to end on a single GPU (tests).  nranks > 1
  // without an id: a mailbox-only plan (fcm_connect_peers before fcm_run).
  if (!rc && nccl_id) {
    if (!nccl_id || !load_nccl()) {
      rc = fail(p, FCM_E_NCCL, "NCCL unavailable (set FCM_NCCL_LIB) or no unique id");
    } else {
      ncclUniqueId id;
      memcpy(&id, nccl_id, sizeof id);
      cudaSetDevice(device);
      ncclResult_t r = g_nccl.CommInitRank(&p->comm, nranks, id, rank);
      if (r != ncclSuccess) rc = fail(p, FCM_E_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
      else p->use_nccl = true;
    }
  }
  if (rc) {
    fprintf(stderr, "fcm_plan_create_rank: %s\n", p->err.c_str());
    release(p);
    delete p;
    return rc;
  }
  *out = p;
  return FCM_OK;
}

int fcm_plan_destroy(fcm_plan* p) {
  if (!p) return FCM_OK;
  release(p);
  delete p;
  return FCM_OK;
}

const char* fcm_last_error(const fcm_plan* p) { return p ? p->err.c_str() : "null plan"; }

int fcm_set_option(fcm_plan* p, int32_t key, int64_t value) {
  if (check_plan(p)) return FCM_E_ARG;
  switch (key) {
    case FCM_OPT_BATCH:
      if (value < 1 || value > 4096) return FCM_E_ARG;
      p->batch = (int)value;
      return FCM_OK;
    case FCM_OPT_TIMING: p->timing = value ? 1 : 0; return FCM_OK;
    case FCM_OPT_GRID:
      if (value < 0) return FCM_E_ARG;
      p->force_grid = (int)value;
      return FCM_OK;
    case FCM_OPT_GRAPH: p->use_graph = value ? 1 : 0; return FCM_OK;
    case FCM_OPT_LOOP: p->use_loop = value ? 1 : 0; return FCM_OK;
    case FCM_OPT_PROFILE: p->profile = value ? 1 : 0; return FCM_OK;
    case FCM_OPT_SEED_PASS:
      if (value < 0 || value > 2) return FCM_E_ARG;
      p->seed_pass = (int)value;
      return FCM_OK;
    case FCM_OPT_RECOMPUTE: p->recompute = value ? 1 : 0; return FCM_OK;
    case FCM_OPT_DEBUG_DELAY:
      if (value < 0 || value > 10000000) return FCM_E_ARG;  // <= 10 ms
      p->debug_delay_ns = (unsigned)value;
      return FCM_OK;
    case FCM_OPT_DEBUG_SHARED_PARTIALS: p->debug_shared_parts = value ? 1 : 0; return FCM_OK;
    case FCM_OPT_DEBUG_SOLO_RANK: p->solo_rank = value ? 1 : 0; return FCM_OK;
    case FCM_OPT_PEER_TIMEOUT_MS:
      if (value < 0 || value > 3600000) return FCM_E_ARG;
      p->peer_timeout_ms = value;
      return FCM_OK;
    case FCM_OPT_L2:
      if (value < 0 || value > 2) return FCM_E_ARG;
      p->l2_mode = (int)value;
      return FCM_OK;
    case FCM_OPT_KERNEL:
      if (value < 0 || value > 3) return FCM_E_ARG;
      if (value == 1 && p->c <= 16)  // the register-staged kernel is built for 17 <= c <= 32 only
        return fail(p, FCM_E_ARG, "FCM_OPT_KERNEL = 1 (register-staged pass kernel) needs c > 16");
      p->variant = (int)value;
      return FCM_OK;
    default: return FCM_E_ARG;
  }
}

int fcm_plan_info(const fcm_plan* p, int64_t* info, int32_t count) {
  if (!p || !info) return FCM_E_ARG;
  // The plan's voxel range: the whole image for single-process plans, the
  // rank's slice for NCCL rank plans.
  const Geometry& g = p->sh[0].g;
  int64_t n_plan = 0, tiles_plan = 0;
  for (int i = 0; i < p->nshards; ++i) {
    n_plan += p->sh[i].g.n_local;
    tiles_plan += p->sh[i].g.tiles_local;
  }
  const int64_t v[] = {p->n_global, n_plan, g.voxel0, int64_t(1) << g.tile_shift, g.T,
                       tiles_plan, p->sh[0].last_grid, p->nshards, p->dev_bytes};
  for (int i = 0; i < count && i < (int)(sizeof v / sizeof v[0]); ++i) info[i] = v[i];
  return FCM_OK;
}

// Host -> device copy of `bytes` from a caller buffer.  Pinned (or small)
// sources go straight to the copy engine; a large pageable source is split
// over kStageThreads host threads, each copying its range through two 8 MB
// page-locked slots of the plan (memcpy into one slot while the other's DMA
// runs on the thread's own stream) -- the driver's own pageable path stages
// through one buffer on one thread (~11 GB/s here).  Synchronous.
constexpr int kStageThreads = 16;
constexpr size_t kStageSlot = (size_t)8 << 20;
static int h2d_from_host(fcm_plan* p, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  cudaPointerAttributes at{};
  const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  int cur = 0;
  cudaGetDevice(&cur);
  // (the staging streams live on shard 0's device)
  if (pinned || bytes < ((size_t)64 << 20) || cur != p->sh[0].device) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return FCM_OK;
  }
  if (!p->stage_pinned) {
    if (cudaMallocHost(&p->stage_pinned, kStageSlot * 2 * kStageThreads) != cudaSuccess) {
      cudaGetLastError();  // no page-locked memory to spare: the driver's own pageable path
      p->stage_pinned = nullptr;
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
      return FCM_OK;
    }
    for (int t = 0; t < kStageThreads; ++t) {
      CK(cudaStreamCreateWithFlags(&p->stage_st[t], cudaStreamNonBlocking));
      for (int k = 0; k < 2; ++k) CK(cudaEventCreateWithFlags(&p->stage_ev[t][k], cudaEventDisableTiming));
    }
  }
  CK(cudaStreamSynchronize(st));  // (the destination's earlier users on the plan stream)
  const int dev = cur;
  const size_t per = ((bytes + kStageThreads - 1) / kStageThreads + 4095) & ~(size_t)4095;
  std::vector<char> ok(kStageThreads, 1);
  auto work = [&](int t) {
    cudaSetDevice(dev);
    const size_t b0 = std::min(bytes, t * per), b1 = std::min(bytes, b0 + per);
    char* slot[2] = {p->stage_pinned + (size_t)(2 * t) * kStageSlot, p->stage_pinned + (size_t)(2 * t + 1) * kStageSlot};
    int k = 0;
    for (size_t o = b0; o < b1; o += kStageSlot, k ^= 1) {
      const size_t len = std::min(kStageSlot, b1 - o);
      if (cudaEventSynchronize(p->stage_ev[t][k]) != cudaSuccess) ok[t] = 0;  // the slot's last DMA
      memcpy(slot[k], (const char*)src + o, len);
      if (cudaMemcpyAsync((char*)dst + o, slot[k], len, cudaMemcpyHostToDevice, p->stage_st[t]) != cudaSuccess ||
          cudaEventRecord(p->stage_ev[t][k], p->stage_st[t]) != cudaSuccess)
        ok[t] = 0;
    }
    if (cudaStreamSynchronize(p->stage_st[t]) != cudaSuccess) ok[t] = 0;
  };
  std::vector<std::thread> th;
  for (int t = 1; t < kStageThreads; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& t : th) t.join();
  for (char o : ok)
    if (!o) return fail(p, FCM_E_CUDA, "staged host-to-device copy failed");
  return FCM_OK;
}

int fcm_upload_pixels(fcm_plan* p, const void* x) {
  NvtxRange nv("fcm_upload_pixels");
  if (check_plan(p) || !x) return FCM_E_ARG;
  const size_t xsz = xkind_bytes(p->xkind);
  const int64_t host0 = p->nranks > p->nshards ? p->sh[0].g.voxel0 : 0;  // rank plans: host buffers hold the rank slice
  for (int i = 0; i < p->nshards; ++i) {
    Shard& s = p->sh[i];
    if (s.g.n_local == 0) continue;
    CK(cudaSetDevice(s.device));
    const char* src = (const char*)x + (s.g.voxel0 - host0) * xsz;
    if (int rc = h2d_from_host(p, s.x, src, s.g.n_local * xsz, s.stream)) return rc;
  }
  for (int i = 0; i < p->nshards; ++i) {
    CK(cudaSetDevice(p->sh[i].device));
    CK(cudaStreamSynchronize(p->sh[i].stream));
  }
  p->x_ready = true;
  return FCM_OK;
}

int fcm_init_membership(fcm_plan* p, uint64_t seed) {
  if (check_plan(p)) return FCM_E_ARG;
  p->init_src = 1;
  p->seed = seed;
  return FCM_OK;
}

int fcm_upload_membership(fcm_plan* p, const double* u0) {
  NvtxRange nv("fcm_upload_membership");
  if (check_plan(p) || !u0) return FCM_E_ARG;
  const int64_t host0 = p->nranks > p->nshards ? p->sh[0].g.voxel0 : 0;  // rank plans: host buffers hold the rank slice
  for (int i = 0; i < p->nshards; ++i) {
    Shard& s = p->sh[i];
    if (s.g.n_local == 0) continue;
    CK(cudaSetDevice(s.device));
    if (!s.u0_aos) {
      int rc = dalloc(p, s, &s.u0_aos, (size_t)s.g.n_local * p->c);
      if (rc) return rc;
    }
    if (int rc = h2d_from_host(p, s.u0_aos, u0 + (s.g.voxel0 - host0) * p->c,
                               sizeof(double) * s.g.n_local * p->c, s.stream))
      return rc;
  }
  for (int i = 0; i < p->nshards; ++i) {
    CK(cudaSetDevice(p->sh[i].device));
    CK(cudaStreamSynchronize(p->sh[i].stream));
  }
  p->init_src = 2;
  return FCM_OK;
}

static int run_impl(fcm_plan* p, double m, double eps, int32_t max_iters, double* v_out,
                    double* trace_out, int32_t* iterations, int32_t* converged, int32_t* dead_cluster) {
  if (check_plan(p)) return FCM_E_ARG;
  p->run_ok = false;
  p->labels_valid = false;
  p->looped_last = false;
  if (!(m > 1.0) || !std::isfinite(m)) return fail(p, FCM_E_ARG, "fuzzifier must be > 1");
  if (!(eps > 0.0 && eps < 1.0)) return fail(p, FCM_E_ARG, "epsilon must lie in (0, 1)");
  if (max_iters < 1) return fail(p, FCM_E_ARG, "max_iters must be >= 1");
  if (!p->x_ready) return fail(p, FCM_E_STATE, "fcm_upload_pixels has not been called");
  if (!p->init_src) return fail(p, FCM_E_STATE, "no initial membership (init or upload)");
  if (p->nshards == 1 && p->nranks > 1 && !p->use_nccl && !p->p2p_ready && !p->solo_rank)
    return fail(p, FCM_E_STATE, "rank plan without NCCL: call fcm_connect_peers first");
  set_powers(p, m);

  Control tmpl;
  memset(&tmpl, 0, sizeof tmpl);
  tmpl.dead = -1;
  tmpl.stuck_rank = 0x7fffffff;  // lowest rank whose root never arrived (atomicMin)
  *p->host_tmpl = tmpl;
  for (int i = 0; i < p->nshards; ++i) {
    Shard& s = p->sh[i];
    CK(cudaSetDevice(s.device));
    if (s.trace_cap < max_iters) {
      int rc = dalloc(p, s, &s.trace, (size_t)2 * max_iters);  // objective, then delta trace
      if (rc) return rc;
      s.trace_cap = max_iters;
    }
    CK(cudaMemcpyAsync(s.ctl, p->host_tmpl, sizeof(Control), cudaMemcpyHostToDevice, s.stream));
    CK(cudaMemsetAsync(s.node_cnt[1], 0, sizeof(unsigned) * s.cnt_total, s.stream));
    const int nf = nf_of(p->c);
    CK(cudaMemsetAsync(s.tile_part, 0xff, sizeof(double) * 3 * std::max(s.g.tiles_local, 1) * nf, s.stream));
    for (int l = 1; l <= s.g.levels; ++l)
      CK(cudaMemsetAsync(s.node_part[l], 0xff, sizeof(double) * s.g.noct * s.g.nodes[l] * nf, s.stream));
    CK(cudaMemsetAsync(s.l1_buf, 0xff, sizeof(double) * 3 * s.g.noct * s.g.nodes[1] * nf, s.stream));
  }
  Shard& s0 = p->sh[0];
  CK(cudaSetDevice(s0.device));
  p->passes_launched = 0;
  int rc = FCM_OK;
  const bool single = p->nshards == 1 && !p->use_nccl && !p->timing;
  // loop kernel: single-process plans (mailboxes in process for >1 shard) or
  // multi-process ranks whose peer mailboxes are mapped
  // (17 <= c <= 32: per-pass register-staged kernels only -- no stage ring
  // holds that many membership planes)
  bool loop = p->use_loop && !p->force_per_pass && !p->timing && p->variant != 1 && p->c <= 16 &&
              (!p->use_nccl || p->p2p_ready);
  for (int i = 0; i < p->nshards; ++i) loop = loop && p->sh[i].g.tiles_local > 0;
  const bool graph = !loop && single && p->use_graph;
  if (!loop && p->nranks > p->nshards && !p->use_nccl)
    return fail(p, FCM_E_STATE, "a mailbox-only rank plan runs the loop kernel only (no NCCL for per-pass launches)");
  bool looped = false;
  p->seeded_in_loop = 0;
  if (loop) {
    CK(cudaEventRecord(p->ev_start, s0.stream));
    // seeded start: pass 0 of the loop kernel (no prologue launch);
    // uploaded start: the prologue kernel reads the AoS rows first
    // auto: small volumes generate u_0 inside the loop kernel (no second
    // launch); large ones in the prologue kernel, which runs the
    // SplitMix64-bound work at 4 CTAs per SM instead of the loop kernel's 2
    // (C4: 0.75 vs 0.84 ms; same v_1 bit for bit); recompute mode needs the
    // in-loop pass 0 (it records the intensities present)
    // (the prologue kernel's root meets the other shards' only through the
    // per-pass exchange machinery: multi-shard and multi-rank plans keep the
    // seeded start inside the loop kernel, whose pass 0 exchanges like any pass)
    const bool small = p->sh[0].g.tiles_local <= kSmallTilesHost;
    const bool alone = p->nshards == 1 && p->nranks == 1;
    const bool seed_pass = p->init_src == 1 &&
                           (p->seed_pass == 1 || (p->seed_pass == 2 && (small || p->recompute || !alone)));
    if (!seed_pass && (rc = step(p, 0, eps, max_iters))) return rc;
    for (int i = 1; i < p->nshards; ++i) {  // shards start together with shard 0
      CK(cudaSetDevice(p->sh[i].device));
      CK(cudaStreamWaitEvent(p->sh[i].stream, p->ev_start, 0));
    }
    CK(cudaSetDevice(s0.device));
    CK(cudaEventRecord(p->ev_pro, s0.stream));
    const unsigned run = ++p->run_counter & 0xffffu;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < p->nshards && e == cudaSuccess; ++i) {
      Shard& s = p->sh[i];
      CK(cudaSetDevice(s.device));
      PassArgs a = make_args(p, s, 1, eps, max_iters);
      a.seed_pass = seed_pass ? 1 : 0;
      // recompute needs the intensity set, tracked by the seeded pass 0
      a.recompute = (p->recompute && seed_pass && p->xkind == XK_U8 && p->mode == MODE_M2 && p->c <= 8 &&
                     p->variant == 0) ? 1 : 0;
      a.mb_ranks = p->solo_rank ? 1 : p->nranks;
      a.mb_rank = p->solo_rank ? 0 : (p->nshards > 1 ? i : p->rank);
      a.mb_run = run ? run : 1;
      a.mbox_local = s.mbox;
      for (int r = 0; r < p->nranks; ++r) a.mbox_peer[r] = p->nshards > 1 ? p->sh[r].mbox : p->peer_mbox[r];
      a.finalize_local = 1;  // every rank finalizes from the exchanged global root
      a.debug_delay_ns = p->debug_delay_ns;
      a.debug_shared_parts = p->debug_shared_parts;
      a.peer_timeout_ns = (uint64_t)p->peer_timeout_ms * 1000000ull;
      if (p->profile && i == 0) {
        const int passes = std::min(max_iters, 64);
        if (!p->prof) {
          int rc2 = dalloc(p, s0, &p->prof, (size_t)64 * 2 * s0.sms * 4 * kProbeSlots);
          if (rc2) return rc2;
        }
        CK(cudaMemsetAsync(p->prof, 0, sizeof(uint64_t) * 64 * 2 * s0.sms * 4 * kProbeSlots, s0.stream));
        a.prof = p->prof;
        a.prof_passes = passes;
        p->prof_passes = passes;
      }
      // shards sharing a device split its SMs so every loop kernel is resident at once
      int share = 0;
      for (int j = 0; j < p->nshards; ++j) share += p->sh[j].device == s.device ? 1 : 0;
      int grid = 0;
      NvtxRange nv3("fcm loop kernel launch");
      e = launch_loop(p->xkind, p->c, p->mode, a, s.sms, s.stream, &grid, p->variant, p->force_grid, share);
      if (e == cudaSuccess) {
        s.last_grid = grid;
        if (i == 0) p->prof_grid = grid;
      }
    }
    CK(cudaSetDevice(s0.device));
    if (e == cudaSuccess) {
      p->passes_launched = 1;
      looped = true;
      p->looped_last = true;
      p->seeded_in_loop = seed_pass ? 1 : 0;
      for (int i = 1; i < p->nshards; ++i) {  // ev_end on shard 0 covers every shard
        CK(cudaSetDevice(p->sh[i].device));
        CK(cudaEventRecord(p->sh[i].ev_pass, p->sh[i].stream));
        CK(cudaSetDevice(s0.device));
        CK(cudaStreamWaitEvent(s0.stream, p->sh[i].ev_pass, 0));
      }
    } else if ((e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported) && p->nshards == 1 &&
               !p->use_nccl) {
      cudaGetLastError();  // grid cannot be co-resident: host-driven passes below
      if (seed_pass && (rc = step(p, 0, eps, max_iters))) return rc;
    } else {
      CK(e);
    }
  }
  if (looped) {
    // nothing else to enqueue: the loop kernel ran every pass
  } else if (graph) {
    fcm_plan::GraphKey key;
    memset(&key, 0, sizeof key);  // padding takes part in the memcmp below
    key.m = m;
    key.eps = eps;
    key.max_iters = max_iters;
    key.init_src = p->init_src;
    key.variant = p->variant;
    key.force_grid = p->force_grid;
    key.l2_mode = p->l2_mode;
    key.seed = p->seed;
    if (!p->gexec || memcmp(&key, &p->gkey, sizeof key) != 0) {
      if ((rc = build_graph(p, eps, max_iters))) return rc;
      p->gkey = key;
    }
    CK(cudaEventRecord(p->ev_start, s0.stream));
    CK(cudaGraphLaunch(p->gexec, s0.stream));
    CK(cudaEventRecord(p->ev_pro, s0.stream));
  } else {
    if (!loop) {
      CK(cudaEventRecord(p->ev_start, s0.stream));
      rc = step(p, 0, eps, max_iters);
      if (rc) return rc;
      CK(cudaSetDevice(s0.device));
      CK(cudaEventRecord(p->ev_pro, s0.stream));
    }
    int seq = 1;
    while (seq <= max_iters) {
      const int nb = std::min(p->batch, max_iters - seq + 1);
      for (int b = 0; b < nb; ++b, ++seq)
        if ((rc = step(p, seq, eps, max_iters))) return rc;
      CK(cudaSetDevice(s0.device));
      CK(cudaMemcpyAsync(p->host_ctl, s0.ctl, sizeof(Control), cudaMemcpyDeviceToHost, s0.stream));
      CK(cudaStreamSynchronize(s0.stream));
      if (p->host_ctl->done) break;
    }
  }
  CK(cudaSetDevice(s0.device));
  CK(cudaEventRecord(p->ev_end, s0.stream));
  for (int i = 0; i < p->nshards; ++i) {
    CK(cudaSetDevice(p->sh[i].device));
    CK(cudaStreamSynchronize(p->sh[i].stream));
  }
  CK(cudaSetDevice(s0.device));
  CK(cudaMemcpy(p->host_ctl, s0.ctl, sizeof(Control), cudaMemcpyDeviceToHost));
  const Control& h = *p->host_ctl;
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, p->ev_start, p->ev_end));
  p->t_loop_ms = ms;
  CK(cudaEventElapsedTime(&ms, p->ev_start, p->ev_pro));
  p->t_pro_ms = ms;
  p->passes_done = h.iter;
  if (graph) p->passes_launched = (int)h.launches;
  p->t_pass_ms = 0;
  if (looped && h.iter > 0) {
    // the loop kernel's own duration per pass (barriers included)
    CK(cudaEventElapsedTime(&ms, p->ev_pro, p->ev_end));
    p->t_pass_ms = ms / h.iter;
  }
  if (p->timing && h.iter > 0) {
    double tot = 0;
    for (int k = 0; k < h.iter && k < (int)p->ev_t0.size(); ++k) {
      CK(cudaEventElapsedTime(&ms, p->ev_t0[k], p->ev_t1[k]));
      tot += ms;
    }
    p->t_pass_ms = tot / h.iter;
  }
  if (iterations) *iterations = h.iter;
  if (converged) *converged = h.converged;
  if (dead_cluster) *dead_cluster = h.dead;
  if (v_out) memcpy(v_out, h.v, sizeof(double) * p->c);
  if (trace_out && h.iter > 0)
    CK(cudaMemcpy(trace_out, s0.trace, sizeof(double) * h.iter, cudaMemcpyDeviceToHost));
  p->deltas.assign((size_t)std::max(h.iter, 0), 0.0);
  if (h.iter > 0)
    CK(cudaMemcpy(p->deltas.data(), s0.trace + max_iters, sizeof(double) * h.iter, cudaMemcpyDeviceToHost));
  if (!h.done) return fail(p, FCM_E_STATE, "loop ended without the done flag");
  if (h.dead == -2) return fail(p, FCM_E_STATE, "device loop watchdog fired (internal error)");
  if (h.dead == -3) return fail(p, FCM_E_STATE, "loop kernel grid barrier timed out (internal error)");
  if (h.dead == -4)
    return fail(p, FCM_E_NCCL,
                "rank %d: the pass-%u root of rank %d did not arrive within %lld ms (peer process dead or stuck)",
                p->nshards > 1 ? 0 : p->rank, h.stuck_pass, h.stuck_rank, (long long)p->peer_timeout_ms);
  if (h.dead >= 0) return fail(p, FCM_E_DEGENERATE, "cluster %d has zero total membership weight", h.dead);
  p->run_ok = true;
  return FCM_OK;
}

// Single-process multi-shard plans run one loop kernel per shard; shards on
// the same device rely on those kernels being co-scheduled, which CUDA does
// not promise (MPS limits, sanitizers, CUDA_LAUNCH_BLOCKING).  If the
// in-kernel exchange or barrier times out there, the solve is redone with
// one launch per pass (same tree, same bits).  Multi-process ranks and
// single-shard plans report the failure instead.
int fcm_run(fcm_plan* p, double m, double eps, int32_t max_iters, double* v_out,
            double* trace_out, int32_t* iterations, int32_t* converged, int32_t* dead_cluster) {
  NvtxRange nv("fcm_run");
  int rc = run_impl(p, m, eps, max_iters, v_out, trace_out, iterations, converged, dead_cluster);
  if (rc != FCM_OK && rc != FCM_E_DEGENERATE && rc != FCM_E_ARG && p && p->looped_last && p->nshards > 1 &&
      p->nranks == p->nshards && p->host_ctl && (p->host_ctl->dead == -3 || p->host_ctl->dead == -4)) {
    ++p->loop_fallbacks;
    p->force_per_pass = true;
    rc = run_impl(p, m, eps, max_iters, v_out, trace_out, iterations, converged, dead_cluster);
    p->force_per_pass = false;
  }
  return rc;
}

int fcm_download(fcm_plan* p, double* u_out, int32_t* labels_out) {
  NvtxRange nv("fcm_download");
  if (check_plan(p)) return FCM_E_ARG;
  if (!p->run_ok) return fail(p, FCM_E_STATE, "no successful fcm_run to download");
  const int64_t host0 = p->nranks > p->nshards ? p->sh[0].g.voxel0 : 0;  // rank plans: host buffers hold the rank slice
  for (int i = 0; i < p->nshards; ++i) {
    Shard& s = p->sh[i];
    if (s.g.n_local == 0) continue;
    CK(cudaSetDevice(s.device));
    int rc;
    if (u_out && !s.out_u && (rc = dalloc(p, s, &s.out_u, (size_t)s.g.n_local * p->c))) return rc;
    if (labels_out && !s.out_labels && (rc = dalloc(p, s, &s.out_labels, (size_t)s.g.n_local)))
      return rc;
    EpilogueArgs e{};
    e.x = s.x;
    e.n = s.g.n_local;
    e.c = p->c;
    e.v = s.ctl->v;
    e.m = p->pw.m;
    e.p = p->pw.p;
    e.pkind = p->pw.pkind;
    e.pint = p->pw.pint;
    e.mkind = p->pw.mkind;
    e.mint = p->pw.mint;
    e.u_out = u_out ? s.out_u : nullptr;
    e.labels = labels_out ? s.out_labels : nullptr;
    CK(launch_epilogue(p->xkind, p->c, p->mode, e, s.sms, s.stream));
    if (u_out)
      CK(cudaMemcpyAsync(u_out + (s.g.voxel0 - host0) * p->c, s.out_u,
                         sizeof(double) * s.g.n_local * p->c, cudaMemcpyDeviceToHost, s.stream));
    if (labels_out)
      CK(cudaMemcpyAsync(labels_out + (s.g.voxel0 - host0), s.out_labels,
                         sizeof(int32_t) * s.g.n_local, cudaMemcpyDeviceToHost, s.stream));
  }
  for (int i = 0; i < p->nshards; ++i) {
    CK(cudaSetDevice(p->sh[i].device));
    CK(cudaStreamSynchronize(p->sh[i].stream));
  }
  if (labels_out) p->labels_valid = true;
  return FCM_OK;
}

// ---------------------------------------------------------------------------
// Download by intensity table (uint8 pixels).  u_final and the labels are a
// pure function of (x_i, v_final) -- the epilogue evaluates exactly that per
// voxel -- so for 8-bit pixels the n x c result has at most 256 distinct
// rows.  The epilogue runs once over the 256 intensities (same kernel, same
// arithmetic: bit-identical rows), 256 x (8c + 4) bytes cross PCIe, and the
// host expands the rows along its own copy of the pixels with streaming
// stores on every core.  The device labels are still written (resident for
// fcm_label_confusion / fcm_mask_overlap).

int fcm_download_table(fcm_plan* p, const uint8_t* x_host, double* u_out, int32_t* labels_out,
                       int32_t nthreads) {
  NvtxRange nv("fcm_download_table");
  if (check_plan(p)) return FCM_E_ARG;
  if (!p->run_ok) return fail(p, FCM_E_STATE, "no successful fcm_run to download");
  if (p->xkind != XK_U8) return fail(p, FCM_E_ARG, "fcm_download_table needs a uint8 plan");
  if (!x_host && (u_out || labels_out)) return fail(p, FCM_E_ARG, "x_host is NULL");
  // device labels stay resident (metrics); the 256-row table from shard 0
  for (int i = 0; i < p->nshards; ++i) {
    Shard& s = p->sh[i];
    if (s.g.n_local == 0) continue;
    CK(cudaSetDevice(s.device));
    int rc;
    if (!s.out_labels && (rc = dalloc(p, s, &s.out_labels, (size_t)s.g.n_local))) return rc;
    EpilogueArgs e{};
    e.x = s.x;
    e.n = s.g.n_local;
    e.c = p->c;
    e.v = s.ctl->v;
    e.m = p->pw.m;
    e.p = p->pw.p;
    e.pkind = p->pw.pkind;
    e.pint = p->pw.pint;
    e.mkind = p->pw.mkind;
    e.mint = p->pw.mint;
    e.u_out = nullptr;
    e.labels = s.out_labels;
    CK(launch_epilogue(p->xkind, p->c, p->mode, e, s.sms, s.stream));
  }
  Shard& s0 = p->sh[0];
  CK(cudaSetDevice(s0.device));
  int rc;
  if (!s0.tab_x) {
    if ((rc = dalloc(p, s0, &s0.tab_x, 256))) return rc;
    if ((rc = dalloc(p, s0, &s0.tab_u, (size_t)256 * p->c))) return rc;
    if ((rc = dalloc(p, s0, &s0.tab_l, 256))) return rc;
    uint8_t ramp[256];
    for (int b = 0; b < 256; ++b) ramp[b] = (uint8_t)b;
    CK(cudaMemcpy(s0.tab_x, ramp, 256, cudaMemcpyHostToDevice));
  }
  EpilogueArgs e{};
  e.x = s0.tab_x;
  e.n = 256;
  e.c = p->c;
  e.v = s0.ctl->v;
  e.m = p->pw.m;
  e.p = p->pw.p;
  e.pkind = p->pw.pkind;
  e.pint = p->pw.pint;
  e.mkind = p->pw.mkind;
  e.mint = p->pw.mint;
  e.u_out = s0.tab_u;
  e.labels = s0.tab_l;
  CK(launch_epilogue(p->xkind, p->c, p->mode, e, s0.sms, s0.stream));
  std::vector<double> tab((size_t)256 * p->c);
  int32_t ltab[256];
  CK(cudaMemcpyAsync(tab.data(), s0.tab_u, sizeof(double) * tab.size(), cudaMemcpyDeviceToHost, s0.stream));
  CK(cudaMemcpyAsync(ltab, s0.tab_l, sizeof(ltab), cudaMemcpyDeviceToHost, s0.stream));
  CK(cudaStreamSynchronize(s0.stream));
  p->res_tab_u = tab;  // fcm_result_table
  memcpy(p->res_tab_l, ltab, sizeof ltab);
  // host expansion over the plan's voxel range (rank plans: the rank slice)
  int64_t n = 0;
  for (int i = 0; i < p->nshards; ++i) n += p->sh[i].g.n_local;
  if (u_out || labels_out) {
    // freshly allocated result arrays (the drop-in returns new arrays every
    // call) fault in 2 MB pages instead of 4 KB ones where the kernel allows
    // transparent huge pages on request -- advice only, ignored otherwise
    NvtxRange nv2("host table expansion");
    advise_huge(u_out, (size_t)n * p->c * sizeof(double));
    advise_huge(labels_out, (size_t)n * sizeof(int32_t));
    int T = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
    T = (int)std::max<int64_t>(1, std::min<int64_t>(T, std::max<int64_t>(1, n >> 16)));
    const int64_t chunk = ((n + T - 1) / T + 63) & ~int64_t(63);  // even starts keep the u rows 16-B aligned
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) {
      const int64_t i0 = t * chunk, i1 = std::min(n, i0 + chunk);
      if (i0 < i1) th.emplace_back(expand_block, x_host, i0, i1, p->c, tab.data(), ltab, u_out, labels_out);
    }
    expand_block(x_host, 0, std::min(n, chunk), p->c, tab.data(), ltab, u_out, labels_out);
    for (auto& t : th) t.join();
  }
  for (int i = 0; i < p->nshards; ++i) {
    CK(cudaSetDevice(p->sh[i].device));
    CK(cudaStreamSynchronize(p->sh[i].stream));
  }
  p->labels_valid = true;  // the full-size epilogue wrote the device labels
  return FCM_OK;
}

int fcm_result_table(const fcm_plan* p, double* u_tab, int32_t* l_tab) {
  if (!p || (!u_tab && !l_tab)) return FCM_E_ARG;
  if (p->res_tab_u.empty()) return FCM_E_STATE;
  if (u_tab) memcpy(u_tab, p->res_tab_u.data(), sizeof(double) * p->res_tab_u.size());
  if (l_tab) memcpy(l_tab, p->res_tab_l, sizeof p->res_tab_l);
  return FCM_OK;
}


int fcm_narrow_pixels(const double* x, int64_t n, int32_t x_kind, void* out, int32_t nthreads) {
  if ((!x || !out) && n > 0) return FCM_E_ARG;
  if (n < 0 || (x_kind != XK_U8 && x_kind != XK_U16)) return FCM_E_ARG;
  int T = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
  T = (int)std::max<int64_t>(1, std::min<int64_t>(T, std::max<int64_t>(1, n >> 18)));
  const int64_t chunk = (n + T - 1) / T;
  std::vector<char> ok(T, 1);
  auto work = [&](int t) {
    const int64_t i0 = t * chunk, i1 = std::min(n, i0 + chunk);
    if (i0 >= i1) return;
    ok[t] = x_kind == XK_U8 ? narrow_block(x, i0, i1, (uint8_t*)out) : narrow_block(x, i0, i1, (uint16_t*)out);
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& t : th) t.join();
  for (int t = 0; t < T; ++t)
    if (!ok[t]) return FCM_E_ARG;
  return FCM_OK;
}

int fcm_last_timing(const fcm_plan* p, double* out, int32_t count) {
  if (!p || !out) return FCM_E_ARG;
  const double v[] = {p->t_loop_ms, p->t_pass_ms, p->t_pro_ms, (double)p->passes_launched,
                      (double)p->passes_done, (double)p->seeded_in_loop, (double)p->loop_fallbacks};
  for (int i = 0; i < count && i < (int)(sizeof v / sizeof v[0]); ++i) out[i] = v[i];
  return FCM_OK;
}

int fcm_delta_trace(const fcm_plan* p, double* out, int32_t count) {
  if (!p || !out || count < 0) return FCM_E_ARG;
  if (p->deltas.empty()) return FCM_E_STATE;
  for (int i = 0; i < count && i < (int)p->deltas.size(); ++i) out[i] = p->deltas[i];
  return FCM_OK;
}

// Label statistics of the last solve on the device (metrics.py:46-97 counts).
static int label_stats(fcm_plan* p, const int32_t* ref, int32_t cref, const uint8_t* mask, int64_t* out,
                       int nbins) {
  if (check_plan(p) || !out) return FCM_E_ARG;
  if (!p->run_ok) return fail(p, FCM_E_STATE, "no successful fcm_run");
  const int64_t host0 = p->nranks > p->nshards ? p->sh[0].g.voxel0 : 0;
  std::vector<unsigned long long> total(nbins, 0ull), part(nbins);
  for (int i = 0; i < p->nshards; ++i) {
    Shard& s = p->sh[i];
    if (s.g.n_local == 0) continue;
    if (!s.out_labels || !p->labels_valid)
      return fail(p, FCM_E_STATE, "download the labels of the last fcm_run (fcm_download / fcm_download_table) first");
    CK(cudaSetDevice(s.device));
    int32_t* dref = nullptr;
    uint8_t* dmask = nullptr;
    unsigned long long* dbins = nullptr;
    CK(cudaMallocAsync(&dbins, sizeof(unsigned long long) * nbins, s.stream));
    CK(cudaMemsetAsync(dbins, 0, sizeof(unsigned long long) * nbins, s.stream));
    if (ref) {
      CK(cudaMallocAsync(&dref, sizeof(int32_t) * s.g.n_local, s.stream));
      CK(cudaMemcpyAsync(dref, ref + (s.g.voxel0 - host0), sizeof(int32_t) * s.g.n_local, cudaMemcpyHostToDevice,
                         s.stream));
    } else {
      CK(cudaMallocAsync(&dmask, s.g.n_local, s.stream));
      CK(cudaMemcpyAsync(dmask, mask + (s.g.voxel0 - host0), s.g.n_local, cudaMemcpyHostToDevice, s.stream));
    }
    CK(op_label_counts(s.out_labels, dref, dmask, s.g.n_local, p->c, cref, dbins, s.stream));
    CK(cudaMemcpyAsync(part.data(), dbins, sizeof(unsigned long long) * nbins, cudaMemcpyDeviceToHost, s.stream));
    if (dref) CK(cudaFreeAsync(dref, s.stream));
    if (dmask) CK(cudaFreeAsync(dmask, s.stream));
    CK(cudaFreeAsync(dbins, s.stream));
    CK(cudaStreamSynchronize(s.stream));
    for (int b = 0; b < nbins; ++b) total[b] += part[b];
  }
  for (int b = 0; b < nbins; ++b) out[b] = (int64_t)total[b];
  return FCM_OK;
}

int fcm_label_confusion(fcm_plan* p, const int32_t* ref_labels, int32_t c_ref, int64_t* conf_out) {
  if (check_plan(p) || !ref_labels || c_ref < 1 || c_ref > kCMaxSupported) return FCM_E_ARG;
  return label_stats(p, ref_labels, c_ref, nullptr, conf_out, p->c * c_ref);
}

int fcm_mask_overlap(fcm_plan* p, const uint8_t* mask, int64_t* counts_out) {
  if (check_plan(p) || !mask) return FCM_E_ARG;
  return label_stats(p, nullptr, 0, mask, counts_out, 2 * p->c + 1);
}

int fcm_mailbox_handle(fcm_plan* p, void* out64) {
  if (check_plan(p) || !out64) return FCM_E_ARG;
  if (p->nshards != 1) return fail(p, FCM_E_STATE, "mailbox handles belong to rank plans");
  cudaIpcMemHandle_t h;
  CK(cudaSetDevice(p->sh[0].device));
  CK(cudaIpcGetMemHandle(&h, p->sh[0].mbox));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(out64, &h, sizeof h);
  return FCM_OK;
}

int fcm_connect_peers(fcm_plan* p, const void* handles, int32_t nranks) {
  if (check_plan(p) || !handles) return FCM_E_ARG;
  if (p->nshards != 1 || nranks != p->nranks) return fail(p, FCM_E_ARG, "connect needs a rank plan of %d ranks", p->nranks);
  CK(cudaSetDevice(p->sh[0].device));
  for (int r = 0; r < nranks; ++r) {
    if (r == p->rank) {
      p->peer_mbox[r] = p->sh[0].mbox;
      continue;
    }
    if (p->peer_opened[r]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + 64 * r, sizeof h);
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    p->peer_mbox[r] = (Mailbox*)ptr;
    p->peer_opened[r] = true;
  }
  p->p2p_ready = true;
  return FCM_OK;
}

int fcm_last_profile(const fcm_plan* p, uint64_t* out, int64_t count, int32_t* passes, int32_t* grid) {
  if (!p || !out) return FCM_E_ARG;
  if (!p->prof || !p->prof_grid) return FCM_E_STATE;
  const int64_t want = (int64_t)p->prof_passes * p->prof_grid * kProbeSlots;
  if (count < want) return FCM_E_ARG;
  if (cudaMemcpy(out, p->prof, sizeof(uint64_t) * want, cudaMemcpyDeviceToHost) != cudaSuccess) return FCM_E_CUDA;
  if (passes) *passes = p->prof_passes;
  if (grid) *grid = p->prof_grid;
  return FCM_OK;
}

int fcm_host_register(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return FCM_E_ARG;
  cudaError_t e = cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return FCM_E_CUDA;
  }
  return FCM_OK;
}

int fcm_host_unregister(void* ptr) {
  if (!ptr) return FCM_E_ARG;
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return FCM_E_CUDA;
  }
  return FCM_OK;
}

// ----------------------------------------------------------- kernel seam --
namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};
#define CKS(expr)                  \
  do {                             \
    if ((expr) != cudaSuccess) {   \
      cudaGetLastError();          \
      return FCM_E_CUDA;           \
    }                              \
  } while (0)
}  // namespace

int fcm_fill_membership_random(double* u_out, int64_t n, int32_t c, uint64_t seed, int32_t device) {
  if (!u_out || n < 1 || c < 1 || c > kCMaxSupported) return FCM_E_ARG;
  CKS(cudaSetDevice(device));
  DevBuf d;
  CKS(cudaMalloc(&d.p, sizeof(double) * n * c));
  CKS(op_init_aos((double*)d.p, n, c, seed, 0));
  CKS(cudaMemcpy(u_out, d.p, sizeof(double) * n * c, cudaMemcpyDeviceToHost));
  return FCM_OK;
}

int fcm_update_centers(const double* x, const double* u, double* v_out, int64_t n, int32_t c,
                       double m, int32_t device, int32_t* dead_out) {
  if (!x || !u || !v_out || n < 1 || c < 1 || c > kCMaxSupported || !(m > 1.0)) return FCM_E_ARG;
  // One seam op, no plan: the 2c sums of Eq. 3 over the caller's AoS rows
  // (op_center_sums: per-CTA voxel ranges, fixed trees), then the
  // reference's control flow -- the first cluster with zero total weight is
  // dead and ends the update (_kernels.pyx:79-89).
  CKS(cudaSetDevice(device));
  DevBuf dx, du, ds, dw;
  CKS(cudaMalloc(&dx.p, sizeof(double) * n));
  CKS(cudaMalloc(&du.p, sizeof(double) * n * c));
  CKS(cudaMalloc(&ds.p, sizeof(double) * kCenterScratch));
  CKS(cudaMalloc(&dw.p, sizeof(double) * 2 * c));
  CKS(cudaMemcpy(dx.p, x, sizeof(double) * n, cudaMemcpyHostToDevice));
  CKS(cudaMemcpy(du.p, u, sizeof(double) * n * c, cudaMemcpyHostToDevice));
  CKS(op_center_sums((const double*)dx.p, (const double*)du.p, n, c, m, (double*)ds.p, (double*)dw.p,
                     device_sms(device), 0));
  std::vector<double> sums(2 * c);
  CKS(cudaMemcpy(sums.data(), dw.p, sizeof(double) * 2 * c, cudaMemcpyDeviceToHost));
  int dead = -1;
  for (int j = 0; j < c; ++j) {
    if (sums[c + j] == 0.0) {
      dead = j;
      break;
    }
    v_out[j] = sums[j] / sums[c + j];
  }
  if (dead_out) *dead_out = dead;
  return FCM_OK;
}

int fcm_update_membership(const double* x, const double* v, double* u_out, int64_t n, int32_t c,
                          double m, int32_t device) {
  if (!x || !v || !u_out || n < 1 || c < 1 || c > kCMaxSupported || !(m > 1.0)) return FCM_E_ARG;
  CKS(cudaSetDevice(device));
  fcm_plan tmp;  // only for powers
  set_powers(&tmp, m);
  DevBuf dx, dv, du;
  CKS(cudaMalloc(&dx.p, sizeof(double) * n));
  CKS(cudaMalloc(&dv.p, sizeof(double) * c));
  CKS(cudaMalloc(&du.p, sizeof(double) * n * c));
  CKS(cudaMemcpy(dx.p, x, sizeof(double) * n, cudaMemcpyHostToDevice));
  CKS(cudaMemcpy(dv.p, v, sizeof(double) * c, cudaMemcpyHostToDevice));
  EpilogueArgs e{};
  e.x = dx.p;
  e.n = n;
  e.c = c;
  e.v = (const double*)dv.p;
  e.m = tmp.pw.m;
  e.p = tmp.pw.p;
  e.pkind = tmp.pw.pkind;
  e.pint = tmp.pw.pint;
  e.mkind = tmp.pw.mkind;
  e.mint = tmp.pw.mint;
  e.u_out = (double*)du.p;
  e.labels = nullptr;
  if (c == 1) {
    // single cluster: every voxel belongs fully (or equally on a tie) to it
    std::vector<double> ones(n, 1.0);
    memcpy(u_out, ones.data(), sizeof(double) * n);
    return FCM_OK;
  }
  CKS(launch_epilogue(XK_F64, c, tmp.mode, e, device_sms(device), 0));
  CKS(cudaMemcpy(u_out, du.p, sizeof(double) * n * c, cudaMemcpyDeviceToHost));
  return FCM_OK;
}

int fcm_objective(const double* x, const double* u, const double* v, int64_t n, int32_t c,
                  double m, int32_t device, double* out) {
  if (!x || !u || !v || !out || n < 1 || c < 1) return FCM_E_ARG;
  CKS(cudaSetDevice(device));
  DevBuf dx, du, dv, ds;
  CKS(cudaMalloc(&dx.p, sizeof(double) * n));
  CKS(cudaMalloc(&du.p, sizeof(double) * n * c));
  CKS(cudaMalloc(&dv.p, sizeof(double) * c));
  CKS(cudaMalloc(&ds.p, sizeof(double) * (kOpsScratch + 1)));
  CKS(cudaMemcpy(dx.p, x, sizeof(double) * n, cudaMemcpyHostToDevice));
  CKS(cudaMemcpy(du.p, u, sizeof(double) * n * c, cudaMemcpyHostToDevice));
  CKS(cudaMemcpy(dv.p, v, sizeof(double) * c, cudaMemcpyHostToDevice));
  double* s = (double*)ds.p;
  CKS(op_reduce(0, (double*)dx.p, (double*)du.p, (double*)dv.p, n, c, m, nullptr, nullptr, s,
                s + kOpsScratch, 0));
  CKS(cudaMemcpy(out, s + kOpsScratch, sizeof(double), cudaMemcpyDeviceToHost));
  return FCM_OK;
}

int fcm_max_abs_diff(const double* a, const double* b, int64_t count, int32_t device, double* out) {
  if (!a || !b || !out || count < 0) return FCM_E_ARG;
  if (count == 0) {
    *out = 0.0;
    return FCM_OK;
  }
  CKS(cudaSetDevice(device));
  DevBuf da, db, ds;
  CKS(cudaMalloc(&da.p, sizeof(double) * count));
  CKS(cudaMalloc(&db.p, sizeof(double) * count));
  CKS(cudaMalloc(&ds.p, sizeof(double) * (kOpsScratch + 1)));
  CKS(cudaMemcpy(da.p, a, sizeof(double) * count, cudaMemcpyHostToDevice));
  CKS(cudaMemcpy(db.p, b, sizeof(double) * count, cudaMemcpyHostToDevice));
  double* s = (double*)ds.p;
  CKS(op_reduce(1, nullptr, nullptr, nullptr, count, 0, 0.0, (double*)da.p, (double*)db.p, s,
                s + kOpsScratch, 0));
  CKS(cudaMemcpy(out, s + kOpsScratch, sizeof(double), cudaMemcpyDeviceToHost));
  return FCM_OK;
}

int fcm_check_rcp(int64_t n, uint64_t seed, int32_t device, int64_t* mismatches) {
  if (n < 0 || !mismatches) return FCM_E_ARG;
  CKS(cudaSetDevice(device));
  DevBuf d;
  CKS(cudaMalloc(&d.p, sizeof(unsigned long long)));
  CKS(cudaMemset(d.p, 0, sizeof(unsigned long long)));
  CKS(op_rcp_check(n, seed, (unsigned long long*)d.p, 0));
  unsigned long long h = 0;
  CKS(cudaMemcpy(&h, d.p, sizeof h, cudaMemcpyDeviceToHost));
  *mismatches = (int64_t)h;
  return FCM_OK;
}

int fcm_argmax_rows(const double* u, int32_t* labels_out, int64_t n, int32_t c, int32_t device) {
  if (!u || !labels_out || n < 1 || c < 1) return FCM_E_ARG;
  CKS(cudaSetDevice(device));
  DevBuf du, dl;
  CKS(cudaMalloc(&du.p, sizeof(double) * n * c));
  CKS(cudaMalloc(&dl.p, sizeof(int32_t) * n));
  CKS(cudaMemcpy(du.p, u, sizeof(double) * n * c, cudaMemcpyHostToDevice));
  CKS(op_argmax((double*)du.p, (int32_t*)dl.p, n, c, 0));
  CKS(cudaMemcpy(labels_out, dl.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  return FCM_OK;
}

}  // extern "C"

// fcm_tma_pipe.cuh -- the streaming half of the TMA pass: PTX glue, stage
// ring layout, producer (bulk copies), intensity tables and the consumer
// warps (per-voxel Eq. 4 / Eq. 3 terms, tile-end hand-off to the reducer).
// Part of the TMA pass (fcm_tma_kernels.cuh).
#pragma once
#include <climits>

#include "fcm_kernels.cuh"

namespace fcm {

constexpr int kChunk = kThreads * kVec;  // voxels per stage (1024)
constexpr int kTmaThreads = kThreads + 64;  // consumers | producer warp | reducer warp
constexpr int kProducerTid = kThreads;
constexpr int kReducerWarp = kThreads / 32 + 1;
constexpr int kSlots = 8;  // tile-partial slots between consumers and the reducer (<= 32)
constexpr int kSmallTiles = 1024;  // loop kernel: up to this many tiles every CTA reduces level 1 itself

// Consumer -> reducer handoff: per slot, the 8 warp-tree values of every
// field of one tile (tile = -1: end of pass).  full: one arrival per
// consumer thread (after the butterfly several lanes of a warp write fields,
// and each releases its own writes); empty: 1 reducer arrival.
template <int NF>
struct RedSlots {
  double w[kSlots][kWarps][NF];
  int tile[kSlots];
  double root[NF];
  uint64_t full[kSlots];
  uint64_t empty[kSlots];
};
constexpr int kStageBudget = 100 * 1024;  // smem bytes of ring per CTA

// ------------------------------------------------------------- PTX glue ---
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// try_wait with a suspend-time hint: the thread sleeps in hardware until the
// phase completes or about `ns` nanoseconds pass (no busy polling).
__device__ __forceinline__ bool mbar_wait_for(uint32_t bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Blocking wait.  The try_wait carries a long suspend-time hint: the warp
// sleeps in hardware until the phase completes instead of re-issuing the
// probe -- the producer (empty stages) and the reducer (full slots) spend
// most of a pass waiting, and on an issue-bound pass (C2) their spin loops
// were ~6 % of all issued instructions, taken from the consumer warps
// sharing their schedulers.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(bar),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// fp32 -> fp64 with integer ops (exact for normal floats; zero and denormals
// land below 1.2e-38).  Keeps the conversion unit free for the u_k stores.
__device__ __forceinline__ double f32_to_f64_fast(float f) {
  const uint32_t b = __float_as_uint(f);
  return __hiloint2double((int)((b >> 3) + 0x38000000u), (int)(b << 29));
}

// uint8 (or any 32-bit unsigned) intensity -> double via the 2^52 magic
// constant (one DADD).
__device__ __forceinline__ double u8_to_f64(uint32_t byte) {
  return __hiloint2double(0x43300000, (int)byte) - 4503599627370496.0;
}

// ------------------------------------------------------- m == 2, uint8 ---
// Eq. 4 at p = 2 in product form: u_j = P_j / sum_k P_k with
// P_j = prod_{k != j} D_k, D_k = (x - v_k)^2.  For uint8 pixels every
// nonzero D is >= ~1e-27, so the products neither under- nor overflow and
// prod_k D_k == 0 exactly when some x == v_k (then the reference's
// equal-share rule applies, _kernels.pyx:103-113).  The objective term
// sum_j u_j^2 D_j collapses to prod_k D_k / sum_k P_k.
template <int C>
__device__ __forceinline__ void m2_membership(double xd, const double* v, double* u, double& obj) {
  double D[C];
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const double d = xd - v[j];
    D[j] = d * d;
  }
  double pre[C];
  pre[0] = D[0];
#pragma unroll
  for (int j = 1; j < C; ++j) pre[j] = pre[j - 1] * D[j];
  double P[C];
  double suf = D[C - 1];
  P[C - 1] = pre[C - 2];
#pragma unroll
  for (int j = C - 2; j >= 1; --j) {
    P[j] = pre[j - 1] * suf;
    suf *= D[j];
  }
  P[0] = suf;
  const double all = pre[C - 1];
  if (all != 0.0) {
    double Q = P[0];
#pragma unroll
    for (int j = 1; j < C; ++j) Q += P[j];
    const double R = rcp64(Q);
#pragma unroll
    for (int j = 0; j < C; ++j) u[j] = P[j] * R;
    obj = all * R;
  } else {
    int zc = 0;
#pragma unroll
    for (int j = 0; j < C; ++j) zc += D[j] == 0.0 ? 1 : 0;
    const double share = 1.0 / (double)zc;
#pragma unroll
    for (int j = 0; j < C; ++j) u[j] = D[j] == 0.0 ? share : 0.0;
    obj = 0.0;  // sum_j u_j^2 D_j with every weight on a zero distance
  }
}

// Eq. 3 / delta / store terms of one voxel from its fp64 memberships.
template <int C>
__device__ __forceinline__ void m2_fold(double xd, const double* u, double obj, const float* uo_f, float* un,
                                        double* acc, uint32_t& dmax_hi, bool valid) {
  if (valid) acc[2 * C] += obj;
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const double w = u[j] * u[j];
    const double dl = u[j] - f32_to_f64_fast(uo_f[j]);
    if (valid) {
      acc[j] = fma(w, xd, acc[j]);
      acc[C + j] += w;
      dmax_hi = max(dmax_hi, (uint32_t)__double2hiint(dl) & 0x7fffffffu);
    }
    un[j] = (float)u[j];
  }
}

template <int C>
__device__ __forceinline__ void voxel_m2_u8(double xd, const double* v, float uo_f[C], float* un,
                                            double* acc, uint32_t& dmax_hi, bool valid) {
  double u[C], obj;
  m2_membership<C>(xd, v, u, obj);
  m2_fold<C>(xd, u, obj, uo_f, un, acc, dmax_hi, valid);
}

// General path: robust normalised form (membership()) and the reference's
// w = u^m, objective sum_j w_j (x - v_j)^2.
template <int C, int MODE>
__device__ __forceinline__ void voxel_general(double xd, const double* v, int c, const Powers& pw,
                                              float uo_f[C], float* un, double* acc,
                                              uint32_t& dmax_hi, bool valid) {
  double u[C];
  membership<C, MODE>(xd, v, c, pw, u);
#pragma unroll
  for (int j = 0; j < C; ++j) {
    if (j < c) {
      const double w = pow_m<MODE>(u[j], pw);
      const double dj = xd - v[j];
      const double dl = u[j] - f32_to_f64_fast(uo_f[j]);
      if (valid) {
        acc[j] = fma(w, xd, acc[j]);
        acc[C + j] += w;
        acc[2 * C] = fma(w, dj * dj, acc[2 * C]);
        dmax_hi = max(dmax_hi, (uint32_t)__double2hiint(dl) & 0x7fffffffu);
      }
      un[j] = (float)u[j];
    }
  }
}

// Per-pass intensity table for uint8 pixels (MODE_LUT, any m): Eq. 4 is a
// function of the intensity alone, so each CTA evaluates the robust fp64
// form once per pass for the 256 intensities.  The stream gathers u (fp32 +
// fp32 residual, for the stores and an exact-to-1e-12 delta) and counts the
// tile's intensities in per-warp shared-memory histograms; Eq. 3's sums and
// the objective of a tile are then sum_b count_b * (w_b * b, w_b, J_b), with
// thread b holding w_b = u_b^m and J_b in registers for the whole pass -- no
// fp64 work per voxel.  Integer counts are exact, so a tile partial is a
// pure function of the tile's intensity multiset.  Rows are interleaved by
// 16-byte chunk (chunk k of intensity b at (k*256 + b)*16) so lanes with
// different intensities spread over the banks and equal intensities
// broadcast.  Histograms are double-buffered by tile parity.
template <int C>
struct LutLayout {
  static constexpr int K4 = (C + 3) / 4;  // float4 chunks of u (fp32) and of its residual
  static constexpr int kUfOff = 0;
  static constexpr int kDuOff = kUfOff + K4 * 256 * 16;
  static constexpr int kHistOff = kDuOff + K4 * 256 * 16;  // uint32 [2][kWarps][256]
  static constexpr int kBytes = kHistOff + 2 * kWarps * 256 * 4;
};

// m == 2 table (MODE_LUT2): per intensity the fp64 product-form memberships
// u_0..u_{C-1} and the objective term, as double2 chunks interleaved like
// LutLayout (chunk k of intensity b at (k*256 + b)*16).  Entries are exactly
// what m2_membership returns, so the table path is bit-identical to the
// per-voxel product form while the stream does no division per voxel.
template <int C>
struct Lut2Layout {
  static constexpr int K2 = (C + 2) / 2;  // C memberships + objective term
  static constexpr int kBytes = K2 * 256 * 16;
};

template <typename XT, int C, int MODE = MODE_M2>
struct TmaLayout {
  static constexpr int kXBytes = kChunk * (int)sizeof(XT);
  static constexpr int kUBytes = kChunk * 4;
  static constexpr int kStageBytes = kXBytes + C * kUBytes;
  static constexpr int kLutBytes =
      MODE == MODE_LUT ? LutLayout<C>::kBytes : (MODE == MODE_LUT2 ? Lut2Layout<C>::kBytes : 0);
  static constexpr int kStages0 = (kStageBudget - kLutBytes) / kStageBytes;
  static constexpr int kStages = kStages0 < 2 ? 2 : (kStages0 > 8 ? 8 : kStages0);
  static constexpr int kRingBytes = kStages * kStageBytes;
  // ring | lut | full[S] | empty[S] | meta[S]
  static constexpr int kLutOff = kRingBytes;
  static constexpr int kBarOff = kLutOff + kLutBytes;
  static constexpr int kMetaOff = kBarOff + 16 * kStages;
  static constexpr int kSmemBytes = kMetaOff + 16 * kStages;
};

struct StageMeta {
  int tile;   // local tile, -1 = end of work
  int chunk;  // chunk within the tile
  int last;   // 1 if this is the tile's last chunk
  int pad;
};

// Pipeline position of one role (producer or consumers).  Both sides walk
// the ring in the same order, including the end-of-pass marker stage, so the
// persistent loop kernel can run pass after pass on the same ring.
struct Pipe {
  int stage = 0;
  uint32_t phase = 0;
  template <int S>
  __device__ __forceinline__ void advance() {
    if (++stage == S) {
      stage = 0;
      phase ^= 1u;
    }
  }
};

// L2 residency: when x and the c membership planes fit in L2 (BrainWeb-sized
// volumes, SURVEY config 2), loads and stores carry an evict_last policy so
// the next pass -- the next iteration of the loop kernel -- hits L2 instead
// of HBM.  Larger volumes stream with evict-first stores.
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_keep(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_u4(float4* p, float4 v, bool keep, uint64_t pol) {
  if (keep)
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
  else
    __stcs(p, v);
}
// Pass-end barrier of the loop kernel (named barrier 2 over the whole CTA):
// producer and consumers wait on it, the reducer warp only arrives (then
// goes on reducing its level-1 nodes while thread 0 is in the grid barrier).
__device__ __forceinline__ void bar_sync_end() {
  asm volatile("barrier.sync 2, %0;" ::"n"(kTmaThreads) : "memory");  // non-aligned: see red_sync
}
__device__ __forceinline__ void bar_arrive_end() {
  asm volatile("barrier.arrive 2, %0;" ::"n"(kTmaThreads) : "memory");
}

// Orders this thread's generic-proxy view (u_k written by other CTAs, made
// visible by the grid barrier) before its following TMA (async-proxy) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Device-scope release reduction: publishes everything this thread has
// written or observed (cumulativity through the preceding CTA barrier), then
// adds -- one MEMBAR.ALL.GPU + a fire-and-forget REDG, no SC fence.
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Optional per-CTA timeline of the loop kernel (FCM_OPT_PROFILE): slot k of
// record (pass, CTA) -- 0 pass start, 1 producer done claiming, 2 consumers
// done, 3 barrier released, 4 tiles claimed.
__device__ __forceinline__ void probe(const PassArgs& a, unsigned it, int k, uint64_t v) {
  if (a.prof && it >= 1 && it <= (unsigned)a.prof_passes)
    a.prof[((uint64_t)(it - 1) * gridDim.x + blockIdx.x) * kProbeSlots + k] = v;
}

// ------------------------------------------------------------ producer ----
// One elected thread: claim tiles from `counter` until the rank's tiles are
// exhausted, stream every chunk of x and of the c planes of u_{k-1} into the
// ring, then post the end-of-pass marker.
// `first_static` (loop kernel): CTA b's first tile of every pass is tile b,
// the counter hands out tiles G.. -- the pass starts streaming without an
// atomic round trip on the one counter every producer hits at once.
// `gate` (loop kernel, small volumes): tile b's u_{k-1} was written by this
// CTA, so its copies go out at once; before the first claimed tile -- whose
// u_{k-1} another CTA may have written -- the producer waits for the grid
// barrier of the previous pass (ctl->bar_count >= gate->target, acquire; 0 =
// none), then arrives on the CTA's gate mbarrier (one phase per pass) for the
// reducer.  The barrier is thereby off the critical path: it completes while
// the static tile streams.  Returns -1 on a barrier timeout (the run is
// flagged).
struct ProduceGate {
  const unsigned* bar_count;
  unsigned target;
  uint32_t mbar;  // shared-memory mbarrier, count 1
};
__device__ __forceinline__ bool wait_count(unsigned* ctr, unsigned target);

// Large-volume loop kernel (loop_tma_kernel<..., PF = true>): as soon as
// this CTA's own stream is done (after the pass-end CTA barrier, which orders
// the consumers' u_k stores before this warp; the proxy fence hands them to
// the bulk copies) the producer warp issues the first stages of the NEXT
// pass's static tile b -- data this CTA wrote itself -- so they land while
// the root is polled and the next table is built.  Lane k issues chunk k into
// ring stage (stage + k); lane 0 owns the pipe position.  Returns the chunks
// issued.
template <typename XT, int C, int MODE>
__device__ __forceinline__ int prefetch_static(const PassArgs& a, uint8_t* smem, Pipe& ps, bool x_only) {
  using L = TmaLayout<XT, C, MODE>;
  constexpr int S = L::kStages;
  const int lane = threadIdx.x & 31;
  const uint32_t bar0 = smem_u32(smem + L::kBarOff);
  StageMeta* meta = reinterpret_cast<StageMeta*>(smem + L::kMetaOff);
  const bool keep = a.keep_l2 != 0;
  const uint64_t pol = keep ? l2_keep_policy() : 0ull;
  const int c = C <= 8 ? C : a.c;
  const int lt = (int)blockIdx.x;
  const int64_t tile = int64_t(1) << a.g.tile_shift;
  const int64_t nch64 = (a.g.n_local - (int64_t)lt * tile + kChunk - 1) / kChunk;
  const int per = (int)(tile / kChunk);
  const int nch = nch64 < per ? (int)nch64 : per;
  const int pre = nch < S ? nch : S;
  const int st0 = __shfl_sync(0xffffffffu, ps.stage, 0);
  const uint32_t ph0 = __shfl_sync(0xffffffffu, ps.phase, 0);
  fence_proxy_async_global();
  if (lane < pre) {
    const int stg = (st0 + lane) % S;
    const uint32_t ph = ph0 ^ (uint32_t)(((st0 + lane) / S) & 1);
    mbar_wait(bar0 + 8u * (S + stg), ph ^ 1u);
    meta[stg].tile = lt;
    meta[stg].chunk = lane;
    meta[stg].last = lane == nch - 1;
    const uint32_t fb = bar0 + 8u * stg;
    mbar_arrive_tx(fb, (uint32_t)(L::kXBytes + (x_only ? 0 : c * L::kUBytes)));
    const int64_t i0 = (int64_t)lt * tile + (int64_t)lane * kChunk;
    uint8_t* sp = smem + stg * L::kStageBytes;
    const void* xs = reinterpret_cast<const XT*>(a.x) + i0;
    if (keep) bulk_g2s_keep(smem_u32(sp), xs, L::kXBytes, fb, pol);
    else bulk_g2s(smem_u32(sp), xs, L::kXBytes, fb);
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (j < c && !x_only) {
        const uint32_t dst = smem_u32(sp + L::kXBytes + j * L::kUBytes);
        const float* src = a.u_cur + j * a.g.plane + i0;
        if (keep) bulk_g2s_keep(dst, src, L::kUBytes, fb, pol);
        else bulk_g2s(dst, src, L::kUBytes, fb);
      }
  }
  if (lane == 0)
    for (int k = 0; k < pre; ++k) ps.advance<S>();
  __syncwarp();
  return pre;
}

template <typename XT, int C, int MODE>
__device__ __forceinline__ int tma_produce(const PassArgs& a, uint8_t* smem, Pipe& ps, unsigned* counter,
                                           unsigned it = 0, bool x_only = false, unsigned base = 0,
                                           bool first_static = false, const ProduceGate* gate = nullptr,
                                           int pre = 0) {
  using L = TmaLayout<XT, C, MODE>;
  constexpr int S = L::kStages;
  const uint32_t bar0 = smem_u32(smem + L::kBarOff);
  StageMeta* meta = reinterpret_cast<StageMeta*>(smem + L::kMetaOff);
  const int64_t tile = int64_t(1) << a.g.tile_shift;
  const int chunks_per_tile = (int)(tile / kChunk);
  const int c = C <= 8 ? C : a.c;
  const bool keep = a.keep_l2 != 0;
  const uint64_t pol = keep ? l2_keep_policy() : 0ull;
  const int ntiles = a.g.tiles_local;
  int claimed = 0;
  const int off = first_static ? (int)gridDim.x : 0;
  bool aborted = false;
  // one tile per CTA (grid == tiles): nothing to claim -- the end-of-pass
  // marker follows the static tile at once and the gate comes after it
  const bool static_only = first_static && ntiles <= (int)gridDim.x;
  auto pass_gate = [&]() {  // the previous pass's barrier, then the reducer's gate
    if (gate->target && !wait_count(const_cast<unsigned*>(gate->bar_count), gate->target)) aborted = true;
    fence_proxy_async_global();  // other CTAs' u_{k-1} (acquired above) before the bulk copies
    mbar_arrive(gate->mbar);     // (release, CTA scope) -> the reducer may reset slots
  };
  for (;;) {
    if (gate && claimed == 1 && !static_only) pass_gate();  // the static tile is out
    // (mod 2^32: a monotone counter)
    const int lt = (first_static && claimed == 0) ? (int)blockIdx.x
                   : (aborted || static_only)    ? ntiles
                                                 : (int)(atomicAdd(counter, 1u) - base) + off;
    if (lt >= ntiles) {
      mbar_wait(bar0 + 8u * (S + ps.stage), ps.phase ^ 1u);
      meta[ps.stage].tile = -1;
      mbar_arrive(bar0 + 8u * ps.stage);
      ps.advance<S>();
      if (gate && static_only) pass_gate();
      return aborted ? -1 : claimed;
    }
    ++claimed;
    if (it) probe(a, it, 5, global_ns());
    const int64_t base = (int64_t)lt * tile;
    const int64_t left = a.g.n_local - base;
    const int64_t nch64 = (left + kChunk - 1) / kChunk;
    const int nch = nch64 < chunks_per_tile ? (int)nch64 : chunks_per_tile;
    // (the static tile's first `pre` chunks went out at the end of the last pass)
    for (int ch = (first_static && claimed == 1) ? pre : 0; ch < nch; ++ch) {
      mbar_wait(bar0 + 8u * (S + ps.stage), ps.phase ^ 1u);
      meta[ps.stage].tile = lt;
      meta[ps.stage].chunk = ch;
      meta[ps.stage].last = ch == nch - 1;
      const uint32_t fb = bar0 + 8u * ps.stage;
      mbar_arrive_tx(fb, (uint32_t)(L::kXBytes + (x_only ? 0 : c * L::kUBytes)));
      const int64_t i0 = base + (int64_t)ch * kChunk;
      uint8_t* st = smem + ps.stage * L::kStageBytes;
      const void* xs = reinterpret_cast<const XT*>(a.x) + i0;
      if (keep) bulk_g2s_keep(smem_u32(st), xs, L::kXBytes, fb, pol);
      else bulk_g2s(smem_u32(st), xs, L::kXBytes, fb);
#pragma unroll
      for (int j = 0; j < C; ++j)
        if (j < c && !x_only) {
          const uint32_t dst = smem_u32(st + L::kXBytes + j * L::kUBytes);
          const float* src = a.u_cur + j * a.g.plane + i0;
          if (keep) bulk_g2s_keep(dst, src, L::kUBytes, fb, pol);
          else bulk_g2s(dst, src, L::kUBytes, fb);
        }
      ps.advance<S>();
    }
  }
}

// ------------------------------------------------------- intensity table --
// Entry b = tid: the same robust Eq. 4 evaluation as the direct path, so
// table values equal per-voxel evaluation.  Ends with a consumer barrier.
// Entry b = tid: the same robust Eq. 4 evaluation as the direct path.
// Returns w_b * b, w_b and the objective term J_b (registers of thread b) and
// clears thread b's histogram bins.  Ends with a consumer barrier.
template <int C>
__device__ __forceinline__ void tma_build_lut(uint8_t* lut, const double* v, int c, const Powers& pw,
                                              double* wx, double* wb, double& jb) {
  using LL = LutLayout<C>;
  const int tid = threadIdx.x;
  const double xb = (double)tid;
  double u[C];
  membership<C, MODE_GEN>(xb, v, c, pw, u);
  double jt = 0.0;
  float ufv[4 * LL::K4], duv[4 * LL::K4];
#pragma unroll
  for (int j = 0; j < 4 * LL::K4; ++j) ufv[j] = duv[j] = 0.0f;
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const double w = j < c ? pow_m<MODE_GEN>(u[j], pw) : 0.0;
    const double d = xb - v[j];
    jt = fma(w, d * d, jt);
    wb[j] = w;
    wx[j] = w * xb;
    ufv[j] = (float)u[j];
    duv[j] = (float)(u[j] - (double)ufv[j]);
  }
  jb = jt;
#pragma unroll
  for (int k = 0; k < LL::K4; ++k) {
    reinterpret_cast<float4*>(lut + LL::kUfOff)[k * 256 + tid] =
        make_float4(ufv[4 * k], ufv[4 * k + 1], ufv[4 * k + 2], ufv[4 * k + 3]);
    reinterpret_cast<float4*>(lut + LL::kDuOff)[k * 256 + tid] =
        make_float4(duv[4 * k], duv[4 * k + 1], duv[4 * k + 2], duv[4 * k + 3]);
  }
  uint32_t* hist = reinterpret_cast<uint32_t*>(lut + LL::kHistOff);
#pragma unroll
  for (int w = 0; w < 2 * kWarps; ++w) hist[w * 256 + tid] = 0u;
  red_sync<true>();
}

// m == 2 table: entry b = tid is m2_membership at x = b (the per-voxel
// product form, bit for bit).  Ends with a consumer barrier.
template <int C>
__device__ __forceinline__ void tma_build_lut2(uint8_t* lut, const double* v) {
  constexpr int K2 = Lut2Layout<C>::K2;
  const int tid = threadIdx.x;
  double e[2 * K2];
#pragma unroll
  for (int j = 0; j < 2 * K2; ++j) e[j] = 0.0;
  double obj;
  m2_membership<C>((double)tid, v, e, obj);
  e[C] = obj;
#pragma unroll
  for (int k = 0; k < K2; ++k)
    reinterpret_cast<double2*>(lut)[k * 256 + tid] = make_double2(e[2 * k], e[2 * k + 1]);
  red_sync<true>();
}

// ------------------------------------------------------------ consumers ---
// The 8 consumer warps: per stage, copy 4 voxels per thread to registers,
// release the stage, evaluate Eq. 4, store u_k (in place over u_{k-1}: each
// element is in the stage before the same thread overwrites it) and fold the
// Eq. 3 / objective / delta terms; at the end of each tile run the fixed
// reduction tree.  Returns after the end-of-pass marker.
// Consumers of the loop kernel's seeded start (pass 0): the stage carries x
// only; u_0 is generated per voxel (seed_quad: bit-exact SplitMix64 rows),
// stored as the first fp32 membership and folded into Eq. 3's sums; tile
// partials go to the reducer like any pass.  Same thread -> voxel map and
// tree as prologue_kernel, so both starts give the same v_1 bit for bit.
template <typename XT, int C, int MODE>
__device__ __forceinline__ void tma_consume_seed(const PassArgs& a, uint8_t* smem, Pipe& ps,
                                                 RedSlots<2 * C + 2>& rs, Pipe& sp, const Powers& pw) {
  using L = TmaLayout<XT, C, MODE>;
  constexpr int S = L::kStages;
  constexpr int NS = 2 * C + 2;
  const int tid = threadIdx.x;
  const uint32_t bar0 = smem_u32(smem + L::kBarOff);
  const StageMeta* meta = reinterpret_cast<const StageMeta*>(smem + L::kMetaOff);
  const int64_t tile = int64_t(1) << a.g.tile_shift;
  const int c = C <= 8 ? C : a.c;
  const bool keep = a.keep_l2 != 0;
  const uint64_t pol = keep ? l2_keep_policy() : 0ull;
  double acc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) acc[s] = 0.0;
  // recompute mode: which intensities occur (256 bits per thread, OR-reduced
  // into ctl->present at the end of the pass)
  const bool track = a.recompute && sizeof(XT) == 1;
  uint32_t pm[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) pm[k] = 0u;
  for (;;) {
    mbar_wait(bar0 + 8u * ps.stage, ps.phase);
    const StageMeta mt = meta[ps.stage];
    const uint8_t* st = smem + ps.stage * L::kStageBytes;
    if (mt.tile < 0) {
      mbar_arrive(bar0 + 8u * (S + ps.stage));  // every consumer thread (count kThreads)
      ps.advance<S>();
      if (track) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t w = __reduce_or_sync(0xffffffffu, pm[k]);
          if ((tid & 31) == 0 && w) atomicOr(&a.ctl->present[k], w);
        }
      }
      mbar_wait(smem_u32(&rs.empty[sp.stage]), sp.phase ^ 1u);
      if (tid == 0) rs.tile[sp.stage] = -1;
      mbar_arrive(smem_u32(&rs.full[sp.stage]));  // every consumer thread: its own slot writes
      sp.advance<kSlots>();
      return;
    }
    const int64_t i0 = (int64_t)mt.tile * tile + (int64_t)mt.chunk * kChunk + tid * kVec;
    double xd[4];
    if (sizeof(XT) == 1) {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(st + tid * 4);
#pragma unroll
      for (int q = 0; q < 4; ++q) xd[q] = u8_to_f64((w >> (8 * q)) & 0xffu);
      if (track) {
        const int64_t nv = a.g.n_local - i0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t b = (w >> (8 * q)) & 0xffu;
          const uint32_t bit = q < nv ? 1u << (b & 31u) : 0u;
#pragma unroll
          for (int k = 0; k < 8; ++k) pm[k] |= (b >> 5) == (uint32_t)k ? bit : 0u;
        }
      }
    } else if (sizeof(XT) == 2) {
      const uint2 w = *reinterpret_cast<const uint2*>(st + tid * 8);
      xd[0] = u8_to_f64(w.x & 0xffffu);  // (exact for any 32-bit unsigned value)
      xd[1] = u8_to_f64(w.x >> 16);
      xd[2] = u8_to_f64(w.y & 0xffffu);
      xd[3] = u8_to_f64(w.y >> 16);
    } else {
      const double2 p0 = *reinterpret_cast<const double2*>(st + tid * 32);
      const double2 p1 = *reinterpret_cast<const double2*>(st + tid * 32 + 16);
      xd[0] = p0.x;
      xd[1] = p0.y;
      xd[2] = p1.x;
      xd[3] = p1.y;
    }
    mbar_arrive(bar0 + 8u * (S + ps.stage));  // every consumer thread (count kThreads)
    ps.advance<S>();
    float4 un[C];
    seed_quad<C, MODE>(a, pw, c, i0, xd, a.g.n_local - i0, un, acc);
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (j < c) st_u4(reinterpret_cast<float4*>(a.u_nxt + j * a.g.plane + i0), un[j], keep, pol);
    if (mt.last) {
      // the sum fields through the halving butterfly (bfly_level); the
      // pass-0 delta and objective fields are 0.0
      constexpr int NSUM = NS - 1;
      double v[NSUM];
#pragma unroll
      for (int s2 = 0; s2 < NSUM; ++s2) v[s2] = acc[s2];
      bfly_level<NSUM, 16>(v, tid & 31);
      mbar_wait(smem_u32(&rs.empty[sp.stage]), sp.phase ^ 1u);
#pragma unroll
      for (int k = 0; k < bfly_slots(NSUM); ++k) {
        const int s2 = bfly_field(tid & 31, NSUM, k);
        const int f = s2 >= 0 ? field_of<C>(s2, c) : -1;
        if (f >= 0) rs.w[sp.stage][tid >> 5][f] = v[k];
      }
      if ((tid & 31) == 0) {
        rs.w[sp.stage][tid >> 5][field_of<C>(NS - 1, c)] = 0.0;
        if (tid == 0) rs.tile[sp.stage] = mt.tile;
      }
      mbar_arrive(smem_u32(&rs.full[sp.stage]));  // every consumer thread: its own slot writes
      sp.advance<kSlots>();
#pragma unroll
      for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    }
  }
}

template <typename XT, int C, int MODE, bool XONLY = false>
__device__ __forceinline__ void tma_consume(const PassArgs& a, uint8_t* smem, Pipe& ps,
                                            RedSlots<2 * C + 2>& rs, Pipe& sp, const double* v,
                                            const Powers& pw, const double* lwx = nullptr,
                                            const double* lwb = nullptr, double ljb = 0.0, unsigned it = 0) {
  constexpr bool LUT = MODE == MODE_LUT;
  constexpr bool LUT2 = MODE == MODE_LUT2;
  using L = TmaLayout<XT, C, MODE>;
  using LL = LutLayout<C>;
  constexpr int S = L::kStages;
  const int tid = threadIdx.x;
  const uint32_t bar0 = smem_u32(smem + L::kBarOff);
  const StageMeta* meta = reinterpret_cast<const StageMeta*>(smem + L::kMetaOff);
  const uint8_t* lut = smem + L::kLutOff;
  const int64_t tile = int64_t(1) << a.g.tile_shift;
  const int c = C <= 8 ? C : a.c;
  const bool keep = a.keep_l2 != 0;
  const uint64_t pol = keep ? l2_keep_policy() : 0ull;
  float dmax_f = 0.0f;
  double acc[2 * C + 2];
#pragma unroll
  for (int s = 0; s < 2 * C + 2; ++s) acc[s] = 0.0;
  uint32_t dmax_hi = 0;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L::kLutOff + (LUT ? LL::kHistOff : 0));
  int hpar = 0;  // histogram buffer of the current tile
  bool first = true;
  if (it && tid == 0) probe(a, it, 13, global_ns());
  for (;;) {
    mbar_wait(bar0 + 8u * ps.stage, ps.phase);
    if (first && it && tid == 0) probe(a, it, 12, global_ns());
    first = false;
    const StageMeta mt = meta[ps.stage];
    const uint8_t* st = smem + ps.stage * L::kStageBytes;
    if (mt.tile < 0) {
      if (it && tid == 0) probe(a, it, 19, global_ns());
      mbar_arrive(bar0 + 8u * (S + ps.stage));  // every consumer thread (count kThreads)
      ps.advance<S>();
      // end-of-pass slot for the reducer
      mbar_wait(smem_u32(&rs.empty[sp.stage]), sp.phase ^ 1u);
      if (tid == 0) rs.tile[sp.stage] = -1;
      mbar_arrive(smem_u32(&rs.full[sp.stage]));  // every consumer thread: its own slot writes
      sp.advance<kSlots>();
      return;
    }
    const int64_t i0 = (int64_t)mt.tile * tile + (int64_t)mt.chunk * kChunk + tid * kVec;
    const int64_t nleft = a.g.n_local - i0;
    double xd[4];
    uint32_t xw = 0;  // uint8: the 4 intensities, also the table rows (no fp64 -> int conversion)
    if (sizeof(XT) == 1) {
      xw = *reinterpret_cast<const uint32_t*>(st + tid * 4);
#pragma unroll
      for (int q = 0; q < 4; ++q) xd[q] = u8_to_f64((xw >> (8 * q)) & 0xffu);
    } else if (sizeof(XT) == 2) {
      const uint2 w = *reinterpret_cast<const uint2*>(st + tid * 8);
      xd[0] = u8_to_f64(w.x & 0xffffu);  // (exact for any 32-bit unsigned value)
      xd[1] = u8_to_f64(w.x >> 16);
      xd[2] = u8_to_f64(w.y & 0xffffu);
      xd[3] = u8_to_f64(w.y >> 16);
    } else {
      const double2 p0 = *reinterpret_cast<const double2*>(st + tid * 32);
      const double2 p1 = *reinterpret_cast<const double2*>(st + tid * 32 + 16);
      xd[0] = p0.x;
      xd[1] = p0.y;
      xd[2] = p1.x;
      xd[3] = p1.y;
    }
    float4 uo[C];
#pragma unroll
    for (int j = 0; j < C; ++j) {
      uo[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j < c && !XONLY) uo[j] = *reinterpret_cast<const float4*>(st + L::kXBytes + j * L::kUBytes + tid * 16);
    }
    mbar_arrive(bar0 + 8u * (S + ps.stage));  // every consumer thread (count kThreads)
    ps.advance<S>();
    float4 un[C];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float uq[C], nq[C];
#pragma unroll
      for (int j = 0; j < C; ++j) uq[j] = f4get(uo[j], q);
      const bool valid = q < nleft;
      if (LUT) {
        const int b = (int)((xw >> (8 * q)) & 0xffu);
        const int br = b;
        float ufv[4 * LL::K4], duv[4 * LL::K4];
#pragma unroll
        for (int k = 0; k < LL::K4; ++k) {
          const float4 f = reinterpret_cast<const float4*>(lut + LL::kUfOff)[k * 256 + br];
          const float4 e = reinterpret_cast<const float4*>(lut + LL::kDuOff)[k * 256 + br];
          ufv[4 * k] = f.x; ufv[4 * k + 1] = f.y; ufv[4 * k + 2] = f.z; ufv[4 * k + 3] = f.w;
          duv[4 * k] = e.x; duv[4 * k + 1] = e.y; duv[4 * k + 2] = e.z; duv[4 * k + 3] = e.w;
        }
        if (valid) atomicAdd(hist + (hpar * kWarps + (tid >> 5)) * 256 + b, 1u);
#pragma unroll
        for (int j = 0; j < C; ++j) {
          // |u - u_old| = |(fl32(u) - u_old) + (u - fl32(u))|, both fp32-exact to ~1e-12
          const float dl = fabsf((ufv[j] - uq[j]) + duv[j]);
          if (valid) dmax_f = fmaxf(dmax_f, dl);
          nq[j] = ufv[j];
        }
      } else if (LUT2) {
        const int br = (int)((xw >> (8 * q)) & 0xffu);
        constexpr int K2 = Lut2Layout<C>::K2;
        double e[2 * K2];
#pragma unroll
        for (int k = 0; k < K2; ++k) {
          const double2 w2 = reinterpret_cast<const double2*>(lut)[k * 256 + br];
          e[2 * k] = w2.x;
          e[2 * k + 1] = w2.y;
        }
        if (XONLY) {  // recompute mode: delta comes from the tables, not from u_{k-1}
          uint32_t none = 0;
          m2_fold<C>(xd[q], e, e[C], uq, nq, acc, none, valid);
        } else {
          m2_fold<C>(xd[q], e, e[C], uq, nq, acc, dmax_hi, valid);
        }
      } else if (MODE == MODE_M2 && sizeof(XT) == 1 && C <= 8)
        voxel_m2_u8<C>(xd[q], v, uq, nq, acc, dmax_hi, valid);
      else
        voxel_general<C, MODE>(xd[q], v, c, pw, uq, nq, acc, dmax_hi, valid);
#pragma unroll
      for (int j = 0; j < C; ++j) f4set(un[j], q, nq[j]);
    }
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (j < c) st_u4(reinterpret_cast<float4*>(a.u_nxt + j * a.g.plane + i0), un[j], keep, pol);
    if (mt.last) {
      if (LUT) {
        // every consumer warp has counted the tile: thread b folds bin b
        // (exact count) into the tile's sums and clears it
        red_sync<true>();
        uint32_t cnt = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          uint32_t* h = hist + (hpar * kWarps + w) * 256 + tid;
          cnt += *h;
          *h = 0u;
        }
        const double cd = (double)cnt;
#pragma unroll
        for (int j = 0; j < C; ++j) {
          acc[j] = cd * lwx[j];
          acc[C + j] = cd * lwb[j];
        }
        acc[2 * C] = cd * ljb;
        hpar ^= 1;
      }
      // lanes -> warp value per field: the sum fields through the halving
      // butterfly (bfly_level: the tile-internal tree), the delta as one
      // max reduction of its order-preserving 32-bit key (the fp32 delta, or
      // the high word of the fp64 one) -- then hand the 8 warp values to the
      // reducer through a slot
      constexpr int NS = 2 * C + 2;
      constexpr int NSUM = NS - 1;
      double v[NSUM];
#pragma unroll
      for (int s2 = 0; s2 < NSUM; ++s2) v[s2] = acc[s2];
      bfly_level<NSUM, 16>(v, tid & 31);
      const uint32_t dkey = __reduce_max_sync(0xffffffffu, LUT ? __float_as_uint(dmax_f) : dmax_hi);
      mbar_wait(smem_u32(&rs.empty[sp.stage]), sp.phase ^ 1u);
#pragma unroll
      for (int k = 0; k < bfly_slots(NSUM); ++k) {
        const int s2 = bfly_field(tid & 31, NSUM, k);
        const int f = s2 >= 0 ? field_of<C>(s2, c) : -1;
        if (f >= 0) rs.w[sp.stage][tid >> 5][f] = v[k];
      }
      if ((tid & 31) == 0) {
        rs.w[sp.stage][tid >> 5][field_of<C>(NS - 1, c)] =
            LUT ? (double)__uint_as_float(dkey) : __hiloint2double((int)dkey, (int)0xffffffffu);
        if (tid == 0) rs.tile[sp.stage] = mt.tile;
      }
      mbar_arrive(smem_u32(&rs.full[sp.stage]));  // every consumer thread: its own slot writes
      sp.advance<kSlots>();
#pragma unroll
      for (int s = 0; s < 2 * C + 2; ++s) acc[s] = 0.0;
      dmax_hi = 0;
      dmax_f = 0.0f;
    }
  }
}

}  // namespace fcm

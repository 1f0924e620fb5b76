// fcm_pass_tma.cuh -- the production FCM pass: TMA bulk-copy pipeline.
//
// One CTA = 8 consumer warps + 1 producer warp + 1 reducer warp.  The
// producer claims tiles from the dynamic scheduler and streams each
// 1024-voxel chunk of x and of the c planes of u_{k-1} into a ring of
// shared-memory stages with cp.async.bulk (TMA, completion counted on an
// mbarrier).  Consumers wait on the stage's full barrier, evaluate Eq. 4 for
// 4 voxels per thread, store u_k with 128-bit STG and fold the Eq. 3 /
// objective / delta terms into fp64 registers; at the end of each tile every
// consumer warp reduces its lanes (warp tree) into a shared-memory slot and
// moves on.  The reducer warp combines the 8 warp values of each slot (the
// top of the tile's fixed binary tree), publishes the tile partial and climbs
// the global tree -- the device-scope fences and L2 round trips of the tree
// never stall a consumer.  Bytes in flight per SM are set by the ring depth,
// not by registers, which is what an HBM-bound stream needs.
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
// field of one tile (tile = -1: end of pass).  full: 8 warp arrivals;
// empty: 1 reducer arrival.
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
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(bar),
      "r"(parity)
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

// uint8 intensity -> double via the 2^52 magic constant (one DADD).
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
  asm volatile("bar.sync 2, %0;" ::"n"(kTmaThreads) : "memory");
}
__device__ __forceinline__ void bar_arrive_end() {
  asm volatile("bar.arrive 2, %0;" ::"n"(kTmaThreads) : "memory");
}

// Orders this thread's generic-proxy view (u_k written by other CTAs, made
// visible by the grid barrier) before its following TMA (async-proxy) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
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
template <typename XT, int C, int MODE>
__device__ __forceinline__ int tma_produce(const PassArgs& a, uint8_t* smem, Pipe& ps, unsigned* counter,
                                           unsigned it = 0, bool x_only = false) {
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
  for (;;) {
    const int lt = (int)atomicAdd(counter, 1u);
    if (lt >= ntiles) {
      mbar_wait(bar0 + 8u * (S + ps.stage), ps.phase ^ 1u);
      meta[ps.stage].tile = -1;
      mbar_arrive(bar0 + 8u * ps.stage);
      ps.advance<S>();
      return claimed;
    }
    ++claimed;
    if (it) probe(a, it, 5, global_ns());
    const int64_t base = (int64_t)lt * tile;
    const int64_t left = a.g.n_local - base;
    const int64_t nch64 = (left + kChunk - 1) / kChunk;
    const int nch = nch64 < chunks_per_tile ? (int)nch64 : chunks_per_tile;
    for (int ch = 0; ch < nch; ++ch) {
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
  for (;;) {
    mbar_wait(bar0 + 8u * ps.stage, ps.phase);
    const StageMeta mt = meta[ps.stage];
    const uint8_t* st = smem + ps.stage * L::kStageBytes;
    if (mt.tile < 0) {
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(bar0 + 8u * (S + ps.stage));
      ps.advance<S>();
      mbar_wait(smem_u32(&rs.empty[sp.stage]), sp.phase ^ 1u);
      if (tid == 0) rs.tile[sp.stage] = -1;
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(smem_u32(&rs.full[sp.stage]));
      sp.advance<kSlots>();
      return;
    }
    const int64_t i0 = (int64_t)mt.tile * tile + (int64_t)mt.chunk * kChunk + tid * kVec;
    double xd[4];
    if (sizeof(XT) == 1) {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(st + tid * 4);
#pragma unroll
      for (int q = 0; q < 4; ++q) xd[q] = u8_to_f64((w >> (8 * q)) & 0xffu);
    } else {
      const double2 p0 = *reinterpret_cast<const double2*>(st + tid * 32);
      const double2 p1 = *reinterpret_cast<const double2*>(st + tid * 32 + 16);
      xd[0] = p0.x;
      xd[1] = p0.y;
      xd[2] = p1.x;
      xd[3] = p1.y;
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(bar0 + 8u * (S + ps.stage));
    ps.advance<S>();
    float4 un[C];
    seed_quad<C, MODE>(a, pw, c, i0, xd, a.g.n_local - i0, un, acc);
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (j < c) st_u4(reinterpret_cast<float4*>(a.u_nxt + j * a.g.plane + i0), un[j], keep, pol);
    if (mt.last) {
      double r[NS];
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2) r[s2] = warp_tree(acc[s2], s2 == NS - 1);
      mbar_wait(smem_u32(&rs.empty[sp.stage]), sp.phase ^ 1u);
      if ((tid & 31) == 0) {
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) {
          const int f = field_of<C>(s2, c);
          if (f >= 0) rs.w[sp.stage][tid >> 5][f] = r[s2];
        }
        if (tid == 0) rs.tile[sp.stage] = mt.tile;
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(smem_u32(&rs.full[sp.stage]));
      sp.advance<kSlots>();
#pragma unroll
      for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    }
  }
}

template <typename XT, int C, int MODE>
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
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(bar0 + 8u * (S + ps.stage));
      ps.advance<S>();
      // end-of-pass slot for the reducer
      mbar_wait(smem_u32(&rs.empty[sp.stage]), sp.phase ^ 1u);
      if (tid == 0) rs.tile[sp.stage] = -1;
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(smem_u32(&rs.full[sp.stage]));
      sp.advance<kSlots>();
      return;
    }
    const int64_t i0 = (int64_t)mt.tile * tile + (int64_t)mt.chunk * kChunk + tid * kVec;
    const int64_t nleft = a.g.n_local - i0;
    double xd[4];
    if (sizeof(XT) == 1) {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(st + tid * 4);
#pragma unroll
      for (int q = 0; q < 4; ++q) xd[q] = u8_to_f64((w >> (8 * q)) & 0xffu);
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
    for (int j = 0; j < C; ++j)
      if (j < c) uo[j] = *reinterpret_cast<const float4*>(st + L::kXBytes + j * L::kUBytes + tid * 16);
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(bar0 + 8u * (S + ps.stage));
    ps.advance<S>();
    float4 un[C];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float uq[C], nq[C];
#pragma unroll
      for (int j = 0; j < C; ++j) uq[j] = f4get(uo[j], q);
      const bool valid = q < nleft;
      if (LUT) {
        const int b = (int)(xd[q] - 0.0);
        float ufv[4 * LL::K4], duv[4 * LL::K4];
#pragma unroll
        for (int k = 0; k < LL::K4; ++k) {
          const float4 f = reinterpret_cast<const float4*>(lut + LL::kUfOff)[k * 256 + b];
          const float4 e = reinterpret_cast<const float4*>(lut + LL::kDuOff)[k * 256 + b];
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
        const int b = (int)(xd[q] - 0.0);
        constexpr int K2 = Lut2Layout<C>::K2;
        double e[2 * K2];
#pragma unroll
        for (int k = 0; k < K2; ++k) {
          const double2 w2 = reinterpret_cast<const double2*>(lut)[k * 256 + b];
          e[2 * k] = w2.x;
          e[2 * k + 1] = w2.y;
        }
        m2_fold<C>(xd[q], e, e[C], uq, nq, acc, dmax_hi, valid);
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
      acc[2 * C + 1] = LUT ? (double)dmax_f : __hiloint2double((int)dmax_hi, (int)0xffffffffu);
      // lanes -> warp value per field (adjacent-pair tree), then hand the
      // 8 warp values to the reducer through a slot
      constexpr int NS = 2 * C + 2;
      double r[NS];
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2) r[s2] = warp_tree(acc[s2], s2 == NS - 1);
      mbar_wait(smem_u32(&rs.empty[sp.stage]), sp.phase ^ 1u);
      if ((tid & 31) == 0) {
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) {
          const int f = field_of<C>(s2, c);
          if (f >= 0) rs.w[sp.stage][tid >> 5][f] = r[s2];
        }
        if (tid == 0) rs.tile[sp.stage] = mt.tile;
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(smem_u32(&rs.full[sp.stage]));
      sp.advance<kSlots>();
#pragma unroll
      for (int s = 0; s < 2 * C + 2; ++s) acc[s] = 0.0;
      dmax_hi = 0;
      dmax_f = 0.0f;
    }
  }
}

// ------------------------------------------------------------- reducer ----
// Poll-and-reduce of one tree node by one warp: lane i reads child i's NF
// fields (children < nreal; the rest count as 0.0).  Returns false, without
// side effects, while any child is unpublished; otherwise resets the children
// to unpublished and leaves the per-field adjacent-pair warp tree in lane 0
// of out[f] (out in shared or global memory, written by lane 0).
template <int NF, bool GLOBAL_OUT>
__device__ __forceinline__ bool try_node(double* child0, int nreal, int nf, double* out) {
  const int lane = threadIdx.x & 31;
  const bool real = lane < nreal;
  double* src = child0 + (int64_t)lane * nf;
  // one round trip: every field of every child in flight at once, then check
  double v[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) v[f] = (f < nf && real) ? ld_relaxed(src + f) : 0.0;
  bool ok = true;
#pragma unroll
  for (int f = 0; f < NF; ++f)
    if (f < nf && real) ok = ok && !is_sentinel(v[f]);
  if (!__all_sync(0xffffffffu, ok)) return false;
#pragma unroll
  for (int f = 0; f < NF; ++f)
    if (f < nf) {
      if (real) st_relaxed(src + f, sentinel());
      const double r = warp_tree(v[f], f == nf - 1);
      if (lane == 0) {
        if (GLOBAL_OUT) st_relaxed(out + f, r);
        else out[f] = r;
      }
    }
  return true;
}

template <int NF, bool GLOBAL_OUT>
__device__ __forceinline__ void wait_node(double* child0, int nreal, int nf, double* out) {
  while (!try_node<NF, GLOBAL_OUT>(child0, nreal, nf, out)) __nanosleep(32);
}

// Node k of CTA 0's upper-level list -- levels 2..L, octant by octant, each
// octant's level-2 nodes before its level-3 node -- as (level, octant, j).
__device__ __forceinline__ void upper_node(const Geometry& g, int k, int& l, int& lo, int& j) {
  int per = 0;
  for (int m = 2; m <= g.levels; ++m) per += g.nodes[m];
  lo = k / per;
  j = k - lo * per;
  l = 2;
  while (j >= g.nodes[l]) {
    j -= g.nodes[l];
    ++l;
  }
}

// One warp per CTA.  It (1) drains the consumers' slots: per slot the 8-warp
// pair tree per field (the top three levels of the tile's binary tree over
// its 256 threads) and a relaxed publish of the tile partial -- no fence, no
// atomic on the streaming path; (2) in the gaps, reduces the level-1 nodes
// this CTA owns once the scheduler has handed out all their tiles and every
// child is visibly published (fixed owners: no last-arriver races, no
// feedback onto slow CTAs).
//   LOOP (persistent kernel): level-1 node z belongs to CTA z mod G and its
//     result goes to l1_out (plain stores; the grid barrier that follows
//     publishes it, every CTA then reduces the levels above redundantly);
//   per-pass kernels: node z belongs to CTA 1 + z mod (G-1), results are
//     published with the sentinel protocol, and CTA 0 owns the levels above
//     (octant by octant), the rank root and the finalize.
template <int C, bool LOOP>
__device__ __forceinline__ void tma_reduce(const PassArgs& a, RedSlots<2 * C + 2>& rs, Pipe& sp,
                                           const unsigned* counter, double* l1_out, unsigned it = 0,
                                           bool no_owners = false) {
  constexpr int NF = 2 * C + 2;
  const int lane = threadIdx.x & 31;
  const int nf = 2 * a.c + 2;
  const Geometry& g = a.g;
  const int G = gridDim.x;
  const bool cta0 = blockIdx.x == 0;
  const int NA = no_owners ? 0 : g.noct * g.nodes[1];  // list A: level-1 nodes
  int per = 0;
  for (int m = 2; m <= g.levels; ++m) per += g.nodes[m];
  const int NB = (!LOOP && cta0) ? g.noct * per : 0;  // list B: CTA 0's upper levels
  int strideA, za;
  if (LOOP || G == 1) {
    strideA = G;
    za = blockIdx.x;
  } else {
    strideA = G - 1;
    za = cta0 ? NA : (int)blockIdx.x - 1;
  }
  int zb = 0;
  bool slots_done = false;
  uint64_t n_poll = 0, n_node = 0;

  uint32_t backoff = 64;
  bool node_hot = false;  // the pending node's tiles have all been handed out
  while (!slots_done || za < NA || zb < NB) {
    // next slot: sleep in hardware until it fills (bounded while a node is
    // pending, so the node is still polled about every microsecond)
    // (a node whose tiles are all handed out is "hot": poll it every ~200 ns)
    const bool pending = za < NA || zb < NB;
    const uint32_t hint = pending && node_hot ? 200u : 1000u;
    if (!slots_done && (pending ? mbar_wait_for(smem_u32(&rs.full[sp.stage]), sp.phase, hint)
                                : (mbar_wait(smem_u32(&rs.full[sp.stage]), sp.phase), true))) {
      const int t = rs.tile[sp.stage];
      if (t >= 0) {
        for (int f = lane; f < nf; f += 32) {  // nf <= 34
          const bool mx = f == nf - 1;
          const double(*w)[NF] = rs.w[sp.stage];
          const double q0 = combine(w[0][f], w[1][f], mx);
          const double q1 = combine(w[2][f], w[3][f], mx);
          const double q2 = combine(w[4][f], w[5][f], mx);
          const double q3 = combine(w[6][f], w[7][f], mx);
          st_relaxed(a.tile_part + (int64_t)t * nf + f, combine(combine(q0, q1, mx), combine(q2, q3, mx), mx));
        }
      } else {
        slots_done = true;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&rs.empty[sp.stage]));
      sp.advance<kSlots>();
      if (LOOP && slots_done) {
        bar_arrive_end();  // the CTA may enter the grid barrier now
        if (it && lane == 0) probe(a, it, 15, global_ns());
      }
      continue;
    }
    int l, lo, j;
    if (za < NA) {
      l = 1;
      lo = za / g.nodes[1];
      j = za - lo * g.nodes[1];
    } else if (zb < NB) {
      upper_node(g, zb, l, lo, j);
    } else {
      continue;
    }
    const int oct = g.oct0 + lo;
    const int nreal = node_real_children(g, oct, l, j);
    bool advance = nreal == 0;  // unreal node: nothing to do
    if (!advance) {
      // every tile under the node handed out?  (local index of its last tile)
      const long long r0 = octant_real_nodes(g, oct, 0);
      const long long last = min(((long long)j + 1) << (5 * l), r0) - 1;
      const int last_lt = (int)((long long)oct * g.M - g.tile0 + last);
      // (loop kernel, after this CTA's slots: the barrier may already have
      // re-armed the scheduler, so poll without the hand-out check)
      node_hot = (LOOP && slots_done) || (int)ld_relaxed_u32(counter) > last_lt;
      if (node_hot) {
        ++n_poll;
        double* child0 = l == 1 ? a.tile_part + ((int64_t)oct * g.M - g.tile0 + (int64_t)j * kFan) * nf
                                : a.node_part[l - 1] + ((int64_t)lo * g.nodes[l - 1] + (int64_t)j * kFan) * nf;
        if (LOOP) {  // publish, then count it (readers wait for the count after the grid barrier)
          advance = try_node<NF, false>(child0, nreal, nf, l1_out + ((int64_t)lo * g.nodes[1] + j) * nf);
          if (advance && lane == 0) {
            __threadfence();
            atomicAdd(&a.ctl->l1_done, 1u);
          }
        }
        else
          advance = try_node<NF, true>(child0, nreal, nf, a.node_part[l] + ((int64_t)lo * g.nodes[l] + j) * nf);
        n_node += advance;
      }
    }
    if (advance) {
      if (za < NA) za += strideA;
      else ++zb;
      backoff = 64;
      node_hot = false;
    } else if (slots_done) {
      __nanosleep(backoff);  // pass drained: poll the pending node with a short backoff
      backoff = min(backoff * 2, 128u);
    }
  }
  if (!LOOP && cta0) {
    // octant roots (one level-L node per octant; real octants are a prefix)
    wait_node<NF, false>(a.node_part[g.levels], rank_real_octants(g), nf, rs.root);
    __syncwarp();
    for (int f = lane; f < nf; f += 32) a.rank_root[f] = rs.root[f];
    __syncwarp();
    if (lane == 0) {
      if (a.finalize_local)
        finalize(a.ctl, rs.root, a.c, a.eps, a.max_iters, a.trace, false, a.cond, a.use_cond);
      __threadfence();
    }
  }
  if (it && lane == 0) {
    probe(a, it, 8, n_poll);
    probe(a, it, 9, n_node);
  }
}

// The adjacent-pair tree over 32 children (identical association to
// warp_tree: ((c0+c1)+(c2+c3))+... up to (c0..15)+(c16..31)), evaluated by ONE
// thread from memory (child i at p[i*stride]; children >= nreal count as
// 0.0): no shuffles, all loads in flight at once.
template <bool GLOBAL>
__device__ __forceinline__ double tree32(const double* p, int64_t stride, int nreal, bool mx) {
  double v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i)
    v[i] = i < nreal ? (GLOBAL ? __ldcg(p + (int64_t)i * stride) : p[(int64_t)i * stride]) : 0.0;

#pragma unroll
  for (int s2 = 1; s2 < 32; s2 <<= 1)
#pragma unroll
    for (int i = 0; i < 32; i += 2 * s2) v[i] = combine(v[i], v[i + s2], mx);
  return v[0];
}

// Loop kernel, after the grid barrier of pass `it`: every CTA reduces the
// levels above 1 from the published level-1 results (l1, [noct][nodes[1]][nf]),
// the same fixed tree as everywhere else, into root[] -- redundantly, so no
// further cross-CTA hop is needed.  Each (node, field) pair is one thread's
// tree32; all kTmaThreads threads call it; scratch is the (idle) stage ring.
template <int NF>
__device__ __forceinline__ void loop_upper(const PassArgs& a, const double* l1, double* scratch,
                                           double (*oroot)[NF], double* root, unsigned it = 0,
                                           bool from_tiles = false) {
  const int tid = threadIdx.x;
  const int nf = 2 * a.c + 2;
  const Geometry& g = a.g;
  const int per = g.levels == 3 ? g.nodes[2] : 1;
  // step 0 (small volumes, no level-1 owners): the level-1 nodes themselves,
  // from the tile partials the grid barrier published, into shared memory
  if (from_tiles) {
    double* l1s = scratch;
    scratch += (int64_t)g.noct * g.nodes[1] * NF;
    for (int pr = tid; pr < g.noct * g.nodes[1] * nf; pr += kTmaThreads) {
      const int z = pr / nf, f = pr - z * nf;
      const int lo = z / g.nodes[1], j = z - lo * g.nodes[1];
      const int oct = g.oct0 + lo;
      const int nreal = (int64_t)oct * g.M < g.T ? node_real_children(g, oct, 1, j) : 0;
      const double* src = a.tile_part + ((int64_t)oct * g.M - g.tile0 + (int64_t)j * kFan) * nf + f;
      l1s[(int64_t)z * NF + f] = nreal ? tree32<true>(src, nf, nreal, f == nf - 1) : 0.0;
    }
    __syncthreads();
    l1 = l1s;
  }
  const int ls = from_tiles ? NF : nf;  // row stride of the level-1 results
  // step 1: level-2 nodes (L == 3) or octant roots (L == 2) from level-1 results
  if (g.levels >= 2) {
    for (int pr = tid; pr < g.noct * per * nf; pr += kTmaThreads) {
      const int item = pr / nf, f = pr - item * nf;
      const int lo = item / per, k = item - lo * per;
      const int oct = g.oct0 + lo;
      const int nreal = (int64_t)oct * g.M < g.T ? node_real_children(g, oct, 2, k) : 0;
      const double* src = l1 + ((int64_t)lo * g.nodes[1] + (int64_t)k * kFan) * ls + f;
      double r = 0.0;
      if (nreal) r = from_tiles ? tree32<false>(src, ls, nreal, f == nf - 1) : tree32<true>(src, ls, nreal, f == nf - 1);
      scratch[(int64_t)item * NF + f] = r;
    }
    __syncthreads();
    if (tid == 0) probe(a, it, 11, global_ns());
  }
  // step 2: octant roots
  for (int pr = tid; pr < g.noct * nf; pr += kTmaThreads) {
    const int lo = pr / nf, f = pr - lo * nf;
    const int oct = g.oct0 + lo;
    double r = 0.0;
    if ((int64_t)oct * g.M < g.T) {
      if (g.levels == 1)  // the level-1 node is the octant root
        r = from_tiles ? l1[(int64_t)lo * ls + f] : __ldcg(l1 + (int64_t)lo * ls + f);
      else if (g.levels == 2) r = scratch[(int64_t)lo * NF + f];
      else r = tree32<false>(scratch + (int64_t)lo * per * NF + f, NF, (int)octant_real_nodes(g, oct, 2), f == nf - 1);
    }
    oroot[lo][f] = r;
  }
  __syncthreads();
  // step 3: the rank root over the rank's octants (a pair tree over 8 leaves)
  for (int f = tid; f < nf; f += kTmaThreads) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (i < g.noct && (int64_t)(g.oct0 + i) * g.M < g.T) ? oroot[i][f] : 0.0;
    const bool mx = f == nf - 1;
    root[f] = combine(combine(combine(v[0], v[1], mx), combine(v[2], v[3], mx), mx),
                      combine(combine(v[4], v[5], mx), combine(v[6], v[7], mx), mx), mx);
  }
  __syncthreads();
}

template <typename XT, int C, int MODE>
__device__ __forceinline__ void tma_init_barriers(uint8_t* smem, RedSlots<2 * C + 2>& rs) {
  using L = TmaLayout<XT, C, MODE>;
  const uint32_t bar0 = smem_u32(smem + L::kBarOff);
  for (int s = 0; s < L::kStages; ++s) {
    mbar_init(bar0 + 8u * s, 1);
    mbar_init(bar0 + 8u * (L::kStages + s), kWarps);
  }
  for (int s = 0; s < kSlots; ++s) {
    mbar_init(smem_u32(&rs.full[s]), kWarps);
    mbar_init(smem_u32(&rs.empty[s]), 1);
  }
  mbar_fence_init();
}

template <int C>
__device__ __forceinline__ void load_centers(const Control* ctl, int c, double* v) {
#pragma unroll
  for (int j = 0; j < C; ++j) v[j] = j < c ? __ldcg(&ctl->v[j]) : 0.0;
}

// ------------------------------------------------- one pass per launch ----
template <typename XT, int C, int MODE>
__global__ void __launch_bounds__(kTmaThreads, 2) pass_tma_kernel(PassArgs a) {
  constexpr bool LUT = MODE == MODE_LUT;
  using L = TmaLayout<XT, C, MODE>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ RedSlots<2 * C + 2> rs;
  __shared__ int s_done;
  const int tid = threadIdx.x;
  if (tid == 0) {
    int done = *(volatile int*)&a.ctl->done;
    if (blockIdx.x == 0 && a.seq != 0) {
      const unsigned launched = a.ctl->launches++;
      if (!done && a.use_cond && launched > (unsigned)a.max_iters + 8u) {
        a.ctl->dead = -2;  // watchdog: a device loop may never outlive max_iters passes
        a.ctl->done = 1;
        done = 1;
      }
      if (done && a.use_cond) cudaGraphSetConditional(a.cond, 0u);
    }
    s_done = done;
    if (!done) {
      tma_init_barriers<XT, C, MODE>(smem, rs);
      if (blockIdx.x == 0) a.ctl->tile_next[(a.seq + 1) & 1] = 0u;
    }
  }
  __syncthreads();
  if (s_done) return;
  Pipe ps, sp;
  if (tid >= kThreads) {
    if (tid == kProducerTid) tma_produce<XT, C, MODE>(a, smem, ps, &a.ctl->tile_next[a.seq & 1]);
    else if ((tid >> 5) == kReducerWarp)
      tma_reduce<C, false>(a, rs, sp, &a.ctl->tile_next[a.seq & 1], nullptr);
    return;
  }
  const int c = C <= 8 ? C : a.c;
  double v[C];
  load_centers<C>(a.ctl, c, v);
  const Powers pw = load_powers(a);
  double lwx[C], lwb[C], ljb = 0.0;
  if (LUT) tma_build_lut<C>(smem + L::kLutOff, v, c, pw, lwx, lwb, ljb);
  if (MODE == MODE_LUT2) tma_build_lut2<C>(smem + L::kLutOff, v);
  tma_consume<XT, C, MODE>(a, smem, ps, rs, sp, v, pw, lwx, lwb, ljb);
}

// -------------------------------------------------------- grid barrier ----
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Called by thread 0 of every CTA after a CTA barrier that follows the CTA's
// last tile of pass `it`.  The last arriver knows every tile of the pass is
// finished (so the reduction root and its finalize are published) and every
// producer has stopped claiming, so it re-arms the tile scheduler and
// releases generation `it`.  A stuck barrier (which co-residency rules out)
// times out after 4 s, flags the run, and lets every CTA leave.
__device__ __forceinline__ bool grid_barrier(Control* ctl, unsigned it, unsigned ncta) {
  __threadfence();
  const unsigned prev = atomicAdd(&ctl->bar_count, 1u);
  if (prev == it * ncta - 1u) {
    ctl->tile_next[1] = 0u;
    __threadfence();
    st_release_u32(&ctl->epoch, it);
    return true;
  }
  const uint64_t t0 = global_ns();
  while (ld_acquire_u32(&ctl->epoch) < it) {
    __nanosleep(32);
    if (global_ns() - t0 > 4000000000ull) {
      ctl->dead = -3;
      ctl->done = 1;
      __threadfence();
      return false;
    }
  }
  return true;
}

// Wait (thread 0) until a monotone device counter reaches `target`; false on
// a 4 s timeout (flags the run like a stuck grid barrier).
__device__ __forceinline__ bool wait_count(unsigned* ctr, unsigned target) {
  const uint64_t t0 = global_ns();
  while (ld_acquire_u32(ctr) < target) {
    __nanosleep(32);
    if (global_ns() - t0 > 4000000000ull) return false;
  }
  return true;
}

// Loop kernel, thread 0 of every CTA after the redundant root of pass `it`:
// the same decisions as finalize_body (core.py:120-131: converged, max_iters,
// DegenerateClusterError(j), else v_{k+1}) on the CTA's own copy; CTA 0 also
// publishes them to the control block and the trace.
__device__ __forceinline__ void finalize_loop(const PassArgs& a, const double* root, unsigned it, double* vsh,
                                              const double* vnew, int* s_done) {
  const int c = a.c;
  if (it == 0) {  // seeded start: v_1 or DegenerateClusterError (core.py:121-123)
    int dead = -1;
    for (int j = 0; j < c; ++j)
      if (root[c + j] == 0.0) {
        dead = j;
        break;
      }
    if (dead < 0)
      for (int j = 0; j < c; ++j) vsh[j] = vnew[j];  // root[j] / root[c + j]
    *s_done = dead >= 0 ? 1 : 0;
    if (blockIdx.x == 0) {
      Control* ctl = a.ctl;
      for (int f = 0; f < 2 * c + 2; ++f) ctl->root[f] = root[f];
      ctl->dead = dead;
      if (dead < 0)
        for (int j = 0; j < c; ++j) ctl->v[j] = vsh[j];
      ctl->done = dead >= 0 ? 1 : 0;
    }
    return;
  }
  const int k = (int)it;
  const double delta = root[2 * c + 1];
  const bool conv = delta < a.eps;
  bool done = conv || k >= a.max_iters;
  int dead = -1;
  if (!done)
    for (int j = 0; j < c; ++j)
      if (root[c + j] == 0.0) {
        dead = j;
        done = true;
        break;
      }
  if (!done)
    for (int j = 0; j < c; ++j) vsh[j] = vnew[j];  // root[j] / root[c + j], computed side by side
  *s_done = done ? 1 : 0;
  if (blockIdx.x == 0) {
    Control* ctl = a.ctl;
    for (int f = 0; f < 2 * c + 2; ++f) {
      ctl->root[f] = root[f];
      a.rank_root[f] = root[f];
    }
    ctl->iter = k;
    a.trace[k - 1] = root[2 * c];
    ctl->delta = delta;
    ctl->converged = conv ? 1 : 0;
    ctl->dead = dead;
    if (!done)
      for (int j = 0; j < c; ++j) ctl->v[j] = vsh[j];
    ctl->done = done ? 1 : 0;
  }
}

// Loop kernel, multi-rank: publish this rank's root (in root[], every CTA
// has it) to every rank's mailbox, wait for all ranks' roots of this pass in
// the local mailbox, and replace root[] by the rank-ordered pair tree over
// them -- the same tree the octants use (tree_model.combine_ranks), so the
// global root is the single-rank root bit for bit.  All threads call it.
// Returns false on a 4 s timeout (a peer died): the run is flagged.
__device__ __forceinline__ bool exchange_roots(const PassArgs& a, double* root, unsigned gen) {
  const int tid = threadIdx.x;
  const int nf = 2 * a.c + 2;
  const int par = gen & 1;
  const unsigned tag = (a.mb_run << 16) | (gen & 0xffffu);
  if (blockIdx.x == 0 && tid < a.mb_ranks) {  // thread p writes rank p's copy (NVLink stores)
    Mailbox* mb = a.mbox_peer[tid];
    for (int f = 0; f < nf; ++f) mb->root[par][a.mb_rank][f] = root[f];
    __threadfence_system();
    st_release_sys_u32(&mb->tag[par][a.mb_rank], tag);
  }
  __shared__ int s_ok;
  if (tid == 0) {
    s_ok = 1;
    const uint64_t t0 = global_ns();
    for (int r = 0; r < a.mb_ranks && s_ok; ++r)
      while (ld_acquire_sys_u32(&a.mbox_local->tag[par][r]) != tag) {
        __nanosleep(64);
        if (global_ns() - t0 > 4000000000ull) {
          s_ok = 0;
          break;
        }
      }
  }
  __syncthreads();
  if (!s_ok) return false;
  for (int f = tid; f < nf; f += kTmaThreads) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = i < a.mb_ranks ? ld_relaxed_sys(&a.mbox_local->root[par][i][f]) : 0.0;
    const bool mx = f == nf - 1;
    root[f] = combine(combine(combine(v[0], v[1], mx), combine(v[2], v[3], mx), mx),
                      combine(combine(v[4], v[5], mx), combine(v[6], v[7], mx), mx), mx);
  }
  __syncthreads();
  return true;
}

// --------------------------------------------- persistent loop kernel -----
// The whole device loop of core._iterate (core.py:118-131) in ONE launch:
// every CTA stays resident (cooperative launch), runs pass after pass over
// the dynamic tile scheduler, and meets the others at a grid barrier between
// passes; the CTA that completes a pass's reduction tree finalizes v_{k+1}
// and the stop test before it arrives.  u is updated in place.  No
// per-iteration launch, no host round trip, ring barriers initialised once.
template <typename XT, int C, int MODE>
__global__ void __launch_bounds__(kTmaThreads, 2) loop_tma_kernel(PassArgs a) {
  constexpr bool LUT = MODE == MODE_LUT;
  constexpr int NF = 2 * C + 2;
  using L = TmaLayout<XT, C, MODE>;
  static_assert(L::kRingBytes >= (kOctants * kFan + kSmallTiles / kFan + kOctants) * NF * 8,
                "ring too small for the upper-level scratch");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ RedSlots<NF> rs;
  __shared__ double oroot[kOctants][NF];
  __shared__ double vsh[C];
  __shared__ double vnew[C];
  __shared__ int s_done;
  const int tid = threadIdx.x;
  const int c = C <= 8 ? C : a.c;
  if (tid == 0) {
    tma_init_barriers<XT, C, MODE>(smem, rs);
    s_done = *(volatile int*)&a.ctl->done;
    for (int j = 0; j < c; ++j) vsh[j] = __ldcg(&a.ctl->v[j]);
  }
  const Powers pw = load_powers(a);
  const int64_t l1_len = (int64_t)a.g.noct * a.g.nodes[1] * (2 * a.c + 2);  // one of 3 buffers
  // small volumes (<= 1024 tiles): no level-1 owners -- every CTA reduces
  // the level-1 nodes itself after the grid barrier (one hop less per pass)
  const bool from_tiles = a.g.tiles_local <= kSmallTiles;
  unsigned l1_real = 0;  // real level-1 nodes of this rank (published once per pass)
  if (!from_tiles)
    for (int lo = 0; lo < a.g.noct; ++lo) l1_real += (unsigned)octant_real_nodes(a.g, a.g.oct0 + lo, 1);
  Pipe ps, sp;
  unsigned gen = 0;  // grid-barrier generations
  __syncthreads();
  for (unsigned it = a.seed_pass ? 0u : 1u; !s_done && it <= (unsigned)a.max_iters; ++it) {
    if (tid == 0) probe(a, it, 0, global_ns());
    // level-1 results of this pass: buffer (gen+1) % 3; owners publish them
    // after their CTA has entered the grid barrier and count them in
    // ctl->l1_done (fence + atomic per node); readers wait for the count
    const unsigned gnext = gen + 1;
    double* l1 = a.l1_buf + (gnext % 3) * l1_len;
    if (tid >= kThreads) {
      if (tid == kProducerTid) {
        fence_proxy_async_global();
        const int n = tma_produce<XT, C, MODE>(a, smem, ps, &a.ctl->tile_next[1], it, it == 0);
        probe(a, it, 1, global_ns());
        probe(a, it, 4, (uint64_t)n);
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        probe(a, it, 6, smid);
      }
      if ((tid >> 5) == kReducerWarp) {
        // slots first (then arrive at the pass-end barrier), owned level-1
        // nodes after -- overlapping the grid barrier
        tma_reduce<C, true>(a, rs, sp, &a.ctl->tile_next[1], l1, it, from_tiles);
        if ((tid & 31) == 0) probe(a, it, 7, global_ns());
      } else {
        bar_sync_end();
      }
    } else {
      if (it == 0) {
        tma_consume_seed<XT, C, MODE>(a, smem, ps, rs, sp, pw);
      } else {
        double v[C];
#pragma unroll
        for (int j = 0; j < C; ++j) v[j] = j < c ? vsh[j] : 0.0;
        double lwx[C], lwb[C], ljb = 0.0;
        if (LUT) tma_build_lut<C>(smem + L::kLutOff, v, c, pw, lwx, lwb, ljb);
        if (MODE == MODE_LUT2) tma_build_lut2<C>(smem + L::kLutOff, v);
        tma_consume<XT, C, MODE>(a, smem, ps, rs, sp, v, pw, lwx, lwb, ljb, it);
        if (tid == 0) probe(a, it, 2, global_ns());
      }
      bar_sync_end();
    }
    gen = gnext;
    if (tid == 0) {
      if (!grid_barrier(a.ctl, gen, gridDim.x) || !wait_count(&a.ctl->l1_done, gen * l1_real)) {
        a.ctl->dead = -3;  // a stuck CTA (cannot happen with co-resident CTAs): flag the run
        a.ctl->done = 1;
        s_done = 1;
      }
      probe(a, it, 3, global_ns());
    }
    __syncthreads();
    if (s_done) break;
    loop_upper<NF>(a, l1, reinterpret_cast<double*>(smem), oroot, rs.root, it, from_tiles);
    if (tid == 0) probe(a, it, 10, global_ns());
    if (a.mb_ranks > 1 && !exchange_roots(a, rs.root, gen)) {
      if (tid == 0) {
        a.ctl->dead = -3;
        a.ctl->done = 1;
      }
      break;
    }
    if (tid < c) vnew[tid] = rs.root[tid] / rs.root[c + tid];  // the c divisions side by side
    __syncthreads();
    if (tid == 0) {
      finalize_loop(a, rs.root, it, vsh, vnew, &s_done);
      probe(a, it, 14, global_ns());
    }
    __syncthreads();
  }
}

template <typename XT, int C, int MODE>
inline cudaError_t launch_pass_tma(const PassArgs& a, int sms, cudaStream_t st, int* grid_out,
                                   int force_grid) {
  using L = TmaLayout<XT, C, MODE>;
  auto k = pass_tma_kernel<XT, C, MODE>;
  int dev = 0;
  cudaGetDevice(&dev);
  static unsigned configured = 0;  // per instantiation, bit per device
  if (dev >= 32 || !(configured & (1u << dev))) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemBytes);
    if (e != cudaSuccess) return e;
    if (dev < 32) configured |= 1u << dev;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kTmaThreads, L::kSmemBytes);
  if (per_sm < 1) per_sm = 1;
  long long g = force_grid > 0 ? force_grid : (long long)per_sm * sms;
  if (g > a.g.tiles_local) g = a.g.tiles_local;
  if (g < 1) g = 1;
  k<<<(int)g, kTmaThreads, L::kSmemBytes, st>>>(a);
  if (grid_out) *grid_out = (int)g;
  return cudaGetLastError();
}

// The persistent loop kernel needs every CTA resident at once: cooperative
// launch (fails instead of deadlocking when the grid cannot be co-resident).
template <typename XT, int C, int MODE>
inline cudaError_t launch_loop_tma(const PassArgs& a, int sms, cudaStream_t st, int* grid_out,
                                   int force_grid, int share = 1) {
  using L = TmaLayout<XT, C, MODE>;
  auto k = loop_tma_kernel<XT, C, MODE>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemBytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kTmaThreads, L::kSmemBytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  // kernels sharing a device (multi-shard plans on one GPU) each take at most
  // half their fair share of CTA slots: concurrent cooperative launches are
  // not co-scheduled by contract, so leave slack for imperfect packing
  long long g = (long long)per_sm * sms;
  if (share > 1) g = std::max(1LL, g / (2LL * share));
  if (force_grid > 0 && force_grid < g) g = force_grid;
  if (g > a.g.tiles_local) g = a.g.tiles_local;
  if (g < 1) g = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g);
  cfg.blockDim = dim3(kTmaThreads);
  cfg.dynamicSmemBytes = L::kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, k, a);
  if (grid_out) *grid_out = (int)g;
  return e;
}

}  // namespace fcm

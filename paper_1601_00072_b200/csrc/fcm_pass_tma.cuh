// fcm_pass_tma.cuh -- the production FCM pass: TMA bulk-copy pipeline.
//
// One CTA = 8 consumer warps + 1 producer warp.  The producer claims tiles
// from the dynamic scheduler and streams each 1024-voxel chunk of x and of
// the c planes of u_{k-1} into a ring of shared-memory stages with
// cp.async.bulk (TMA, completion counted on an mbarrier).  Consumers wait on
// the stage's full barrier, evaluate Eq. 4 for 4 voxels per thread, store
// u_k with 128-bit STG, fold the Eq. 3 / objective / delta terms into fp64
// registers, release the stage, and at the end of each tile run the fixed
// reduction tree (tile_finish).  Bytes in flight per SM are set by the ring
// depth, not by registers, which is what an HBM-bound stream needs.
#pragma once
#include "fcm_kernels.cuh"

namespace fcm {

constexpr int kChunk = kThreads * kVec;  // voxels per stage (1024)
constexpr int kTmaThreads = kThreads + 32;
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
__device__ __forceinline__ void voxel_m2_u8(double xd, const double* v, float uo_f[C], float* un,
                                            double* acc, uint32_t& dmax_hi, bool valid) {
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
  double u[C];
  if (all != 0.0) {
    double Q = P[0];
#pragma unroll
    for (int j = 1; j < C; ++j) Q += P[j];
    const double R = rcp64(Q);
#pragma unroll
    for (int j = 0; j < C; ++j) u[j] = P[j] * R;
    if (valid) acc[2 * C] += all * R;
  } else {
    int zc = 0;
#pragma unroll
    for (int j = 0; j < C; ++j) zc += D[j] == 0.0 ? 1 : 0;
    const double share = 1.0 / (double)zc;
#pragma unroll
    for (int j = 0; j < C; ++j) u[j] = D[j] == 0.0 ? share : 0.0;
  }
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

// Per-pass intensity table for uint8 pixels (MODE_LUT): the Eq. 4 / Eq. 3
// per-voxel terms are a function of the intensity alone, so each CTA
// evaluates them once per pass for the 256 intensities (the same robust
// fp64 formula the direct path uses, so values are identical) and the
// stream then gathers them.  Rows are interleaved by 16-byte chunk
// (chunk k of intensity b at (k*256 + b)*16) so lanes with different
// intensities spread over the banks and equal intensities broadcast.
template <int C>
struct LutLayout {
  static constexpr int K4 = (C + 3) / 4;  // float4 chunks of u (fp32) and of its residual
  static constexpr int K2 = (C + 1) / 2;  // double2 chunks of w = u^m
  static constexpr int kUfOff = 0;
  static constexpr int kDuOff = kUfOff + K4 * 256 * 16;
  static constexpr int kWOff = kDuOff + K4 * 256 * 16;
  static constexpr int kJOff = kWOff + K2 * 256 * 16;
  static constexpr int kBytes = kJOff + 256 * 8;
};

template <typename XT, int C, bool LUT = false>
struct TmaLayout {
  static constexpr int kXBytes = kChunk * (int)sizeof(XT);
  static constexpr int kUBytes = kChunk * 4;
  static constexpr int kStageBytes = kXBytes + C * kUBytes;
  static constexpr int kLutBytes = LUT ? LutLayout<C>::kBytes : 0;
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

template <typename XT, int C, int MODE>
__global__ void __launch_bounds__(kTmaThreads, 2) pass_tma_kernel(PassArgs a) {
  constexpr bool LUT = MODE == MODE_LUT;
  using L = TmaLayout<XT, C, LUT>;
  constexpr int S = L::kStages;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ SmemRedT<2 * C + 2> sm;
  if (pass_done(a, sm)) return;

  const int tid = threadIdx.x;
  const uint32_t bar0 = smem_u32(smem + L::kBarOff);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (S + s); };
  StageMeta* meta = reinterpret_cast<StageMeta*>(smem + L::kMetaOff);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), kWarps);
    }
    mbar_fence_init();
    if (blockIdx.x == 0) a.ctl->tile_next[(a.seq + 1) & 1] = 0u;
  }
  __syncthreads();

  const int64_t tile = int64_t(1) << a.g.tile_shift;
  const int chunks_per_tile = (int)(tile / kChunk);
  const int c = C <= 8 ? C : a.c;

  if (tid >= kThreads) {
    // ---------------------------------------------------------- producer --
    if (tid == kThreads) {
      int stage = 0;
      uint32_t phase = 0;
      const int ntiles = a.g.tiles_local;
      for (;;) {
        const int lt = (int)atomicAdd(&a.ctl->tile_next[a.seq & 1], 1u);
        if (lt >= ntiles) {
          mbar_wait(empty_bar(stage), phase ^ 1u);
          meta[stage].tile = -1;
          mbar_arrive(full_bar(stage));
          break;
        }
        const int64_t base = (int64_t)lt * tile;
        const int64_t left = a.g.n_local - base;
        const int64_t nch64 = (left + kChunk - 1) / kChunk;
        const int nch = nch64 < chunks_per_tile ? (int)nch64 : chunks_per_tile;
        for (int ch = 0; ch < nch; ++ch) {
          mbar_wait(empty_bar(stage), phase ^ 1u);
          meta[stage].tile = lt;
          meta[stage].chunk = ch;
          meta[stage].last = ch == nch - 1;
          const uint32_t fb = full_bar(stage);
          mbar_arrive_tx(fb, (uint32_t)(L::kXBytes + c * L::kUBytes));
          const int64_t i0 = base + (int64_t)ch * kChunk;
          uint8_t* st = smem + stage * L::kStageBytes;
          bulk_g2s(smem_u32(st), reinterpret_cast<const XT*>(a.x) + i0, L::kXBytes, fb);
#pragma unroll
          for (int j = 0; j < C; ++j)
            if (j < c)
              bulk_g2s(smem_u32(st + L::kXBytes + j * L::kUBytes), a.u_cur + j * a.g.plane + i0,
                       L::kUBytes, fb);
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers --
  double v[C];
#pragma unroll
  for (int j = 0; j < C; ++j) v[j] = j < c ? a.ctl->v[j] : 0.0;
  const Powers pw = load_powers(a);
  using LL = LutLayout<C>;
  uint8_t* lut = smem + L::kLutOff;
  if (LUT) {
    // entry b = tid: the same robust Eq. 4 evaluation as the direct path
    const double xb = (double)tid;
    double u[C];
    membership<C, MODE_GEN>(xb, v, c, pw, u);
    double jt = 0.0;
    float ufv[4 * LL::K4], duv[4 * LL::K4];
    double wv[2 * LL::K2];
#pragma unroll
    for (int j = 0; j < 4 * LL::K4; ++j) ufv[j] = duv[j] = 0.0f;
#pragma unroll
    for (int j = 0; j < 2 * LL::K2; ++j) wv[j] = 0.0;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const double w = pow_m<MODE_GEN>(u[j], pw);
      const double d = xb - v[j];
      jt = fma(w, d * d, jt);
      wv[j] = w;
      ufv[j] = (float)u[j];
      duv[j] = (float)(u[j] - (double)ufv[j]);
    }
#pragma unroll
    for (int k = 0; k < LL::K4; ++k) {
      reinterpret_cast<float4*>(lut + LL::kUfOff)[k * 256 + tid] =
          make_float4(ufv[4 * k], ufv[4 * k + 1], ufv[4 * k + 2], ufv[4 * k + 3]);
      reinterpret_cast<float4*>(lut + LL::kDuOff)[k * 256 + tid] =
          make_float4(duv[4 * k], duv[4 * k + 1], duv[4 * k + 2], duv[4 * k + 3]);
    }
#pragma unroll
    for (int k = 0; k < LL::K2; ++k)
      reinterpret_cast<double2*>(lut + LL::kWOff)[k * 256 + tid] = make_double2(wv[2 * k], wv[2 * k + 1]);
    reinterpret_cast<double*>(lut + LL::kJOff)[tid] = jt;
    red_sync<true>();
  }
  float dmax_f = 0.0f;
  int tile_parity = 0;
  double acc[2 * C + 2];
#pragma unroll
  for (int s = 0; s < 2 * C + 2; ++s) acc[s] = 0.0;
  uint32_t dmax_hi = 0;
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    mbar_wait(full_bar(stage), phase);
    const StageMeta mt = meta[stage];
    if (mt.tile < 0) break;
    const uint8_t* st = smem + stage * L::kStageBytes;
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
    if ((tid & 31) == 0) mbar_arrive(empty_bar(stage));
    if (++stage == S) {
      stage = 0;
      phase ^= 1u;
    }
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
        double wv[2 * LL::K2];
#pragma unroll
        for (int k = 0; k < LL::K4; ++k) {
          const float4 f = reinterpret_cast<const float4*>(lut + LL::kUfOff)[k * 256 + b];
          const float4 e = reinterpret_cast<const float4*>(lut + LL::kDuOff)[k * 256 + b];
          ufv[4 * k] = f.x; ufv[4 * k + 1] = f.y; ufv[4 * k + 2] = f.z; ufv[4 * k + 3] = f.w;
          duv[4 * k] = e.x; duv[4 * k + 1] = e.y; duv[4 * k + 2] = e.z; duv[4 * k + 3] = e.w;
        }
#pragma unroll
        for (int k = 0; k < LL::K2; ++k) {
          const double2 w2 = reinterpret_cast<const double2*>(lut + LL::kWOff)[k * 256 + b];
          wv[2 * k] = w2.x;
          wv[2 * k + 1] = w2.y;
        }
        if (valid) acc[2 * C] += reinterpret_cast<const double*>(lut + LL::kJOff)[b];
#pragma unroll
        for (int j = 0; j < C; ++j) {
          // |u - u_old| = |(fl32(u) - u_old) + (u - fl32(u))|, both fp32-exact to ~1e-12
          const float dl = fabsf((ufv[j] - uq[j]) + duv[j]);
          if (valid) {
            acc[j] = fma(wv[j], xd[q], acc[j]);
            acc[C + j] += wv[j];
            dmax_f = fmaxf(dmax_f, dl);
          }
          nq[j] = ufv[j];
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
      if (j < c) __stcs(reinterpret_cast<float4*>(a.u_nxt + j * a.g.plane + i0), un[j]);
    if (mt.last) {
      acc[2 * C + 1] = LUT ? (double)dmax_f : __hiloint2double((int)dmax_hi, (int)0xffffffffu);
      tile_finish<C, true>(a, mt.tile, acc, sm, false, tile_parity);
      tile_parity ^= 1;
#pragma unroll
      for (int s = 0; s < 2 * C + 2; ++s) acc[s] = 0.0;
      dmax_hi = 0;
      dmax_f = 0.0f;
    }
  }
}

template <typename XT, int C, int MODE>
inline cudaError_t launch_pass_tma(const PassArgs& a, int sms, cudaStream_t st, int* grid_out,
                                   int force_grid) {
  using L = TmaLayout<XT, C, MODE == MODE_LUT>;
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

}  // namespace fcm

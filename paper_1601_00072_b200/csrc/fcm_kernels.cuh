// fcm_kernels.cuh -- the B200 FCM loop: one fused streaming pass per iteration.
//
// Replaces the reference's per-iteration sequence (core._iterate,
// core.py:105-132; parallel._iterate, parallel.py:257-331):
//     v_k  = centers(u_{k-1})          (update_centers_linear, _kernels.pyx:72-90)
//     u_k  = membership(x, v_k)        (update_membership_range, :93-120)
//     d_k  = max |u_k - u_{k-1}|       (max_abs_diff, :211-220)
//     J_k  = objective(x, u_k, v_k)    (objective_linear, :178-191)
// with ONE kernel per iteration that reads x and u_{k-1} (fp32 SoA), writes
// u_k (fp32 SoA), and reduces the 2c+2 doubles {sum u_k^m x, sum u_k^m, J_k,
// d_k} through a fixed tile tree.  The CTA that completes the tree computes
// v_{k+1} (the "finalize" step) so the next pass needs no host round trip.
#pragma once
#include <algorithm>
#include <cstdio>

#include "fcm_device.cuh"
#include "fcm_kernels.h"

namespace fcm {

template <int NF>
struct SmemRedT {
  double w[2][kWarps][NF];
  double part[NF];
  double root[NF];
  int tile;
  int flag;
};
using SmemRed = SmemRedT<kNFMax>;

// Barrier over the kThreads reduction threads: the whole CTA for the plain
// kernels, the consumer warps (named barrier 1) for the TMA pipeline whose
// producer warp never joins.
template <bool NAMED>
__device__ __forceinline__ void red_sync() {
  // barrier.sync (not bar.sync == barrier.sync.aligned): threads of a warp may
  // arrive from different branches (compute-sanitizer synccheck)
  if (NAMED) asm volatile("barrier.sync 1, %0;" ::"n"(kThreads) : "memory");
  else __syncthreads();
}

// Register slot s (0..2C+1) -> payload field for runtime c <= C.
template <int C>
__device__ __forceinline__ int field_of(int s, int c) {
  if (s < C) return s < c ? s : -1;
  if (s < 2 * C) return (s - C) < c ? c + (s - C) : -1;
  return s == 2 * C ? 2 * c : 2 * c + 1;
}

// ----------------------------------------------------------- finalize -----
// Consumes the global root of pass k (or of the prologue) and prepares the
// centers of the next pass; mirrors the control flow of core._iterate.
__device__ inline void finalize_body(Control* ctl, const double* root, int c, double eps, int max_iters,
                                     double* trace, bool prologue) {
  const int nf = 2 * c + 2;
  for (int f = 0; f < nf; ++f) ctl->root[f] = root[f];
  if (!prologue) {
    const int k = ctl->iter + 1;
    ctl->iter = k;
    trace[k - 1] = root[2 * c];
    trace[max_iters + k - 1] = root[2 * c + 1];  // delta trace (second half of the buffer)
    ctl->delta = root[2 * c + 1];
    if (root[2 * c + 1] < eps) {  // core.py:129-131
      ctl->converged = 1;
      ctl->done = 1;
      return;
    }
    if (k >= max_iters) {  // core.py:120
      ctl->done = 1;
      return;
    }
  }
  for (int j = 0; j < c; ++j) {  // core.py:121-123 -> DegenerateClusterError(j)
    if (root[c + j] == 0.0) {
      ctl->dead = j;
      ctl->done = 1;
      return;
    }
  }
  for (int j = 0; j < c; ++j) ctl->v[j] = root[j] / root[c + j];
}

// finalize + stop the device-side while loop (graph mode) once done.
__device__ inline void finalize(Control* ctl, const double* root, int c, double eps, int max_iters,
                                double* trace, bool prologue, cudaGraphConditionalHandle cond,
                                int use_cond) {
  finalize_body(ctl, root, c, eps, max_iters, trace, prologue);
  if (use_cond && ctl->done) cudaGraphSetConditional(cond, 0u);
}

// Uniform early exit of a pass launched after the loop finished; CTA 0 also
// closes the device-side loop so a graph never spins on finished work.
template <typename SM>
__device__ __forceinline__ bool pass_done(const PassArgs& a, SM& sm) {
  if (threadIdx.x == 0) {
    int done = *(volatile int*)&a.ctl->done;
    if (blockIdx.x == 0 && a.seq != 0) {
      const unsigned launched = a.ctl->launches++;
      if (!done && a.use_cond && launched > (unsigned)a.max_iters + 8u) {
        // watchdog: a device loop may never outlive max_iters passes
        a.ctl->dead = -2;
        a.ctl->done = 1;
        done = 1;
      }
      if (done && a.use_cond) cudaGraphSetConditional(a.cond, 0u);
    }
    sm.flag = done;
  }
  __syncthreads();
  return sm.flag != 0;
}

// ----------------------------------------------------------- tile tree ----
// acq_rel device-scope counter increment: publishes this thread's stores (and
// everything it observed) and, for the last arriver, makes the other
// arrivals' stores visible.  Replaces a full __threadfence on every thread.
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// ---------------------------------------------------- publish protocol ----
// Every tree node slot (tile partials and node results) holds the all-ones
// NaN bit pattern while unpublished: no tree value can be that NaN (sums of
// finite terms and a max of |differences|).  The TMA kernels publish with
// relaxed device-scope stores and their fixed owners poll for the pattern to
// disappear -- no fence or atomic per tile; every reader writes the pattern
// back once it has consumed a slot, so the next pass starts clean.
__device__ __forceinline__ double sentinel() { return __longlong_as_double(-1ll); }
__device__ __forceinline__ bool is_sentinel(double v) { return __double_as_longlong(v) == -1ll; }
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ----------------------------------------------------------- the climb ----
// One warp completes node `node` of level l >= 1 in octant `oct` (it made the
// last arrival on the node's counter): reduce the node's <= 32 children
// (adjacent-pair warp tree), publish it, arrive at the parent, and so on up
// to the octant root; the warp completing the rank's last octant reduces the
// rank root (and, in a single-rank job, finalizes v_{k+1} / the stop test).
// Arrivals are acq_rel device-scope counters -- no spin-waits anywhere.
// Lane 0 writes every node it publishes, so its acq_rel update orders exactly
// the stores it covers.
__device__ __forceinline__ void climb(const PassArgs& a, int oct, int l, int node, double* root_smem,
                                      bool prologue) {
  const int lane = threadIdx.x & 31;
  const int nf = 2 * a.c + 2;
  const Geometry& g = a.g;
  const int loct = oct - g.oct0;
  unsigned prev = 0;
  for (;;) {
    if (lane == 0) a.node_cnt[l][(int64_t)loct * g.nodes[l] + node] = 0u;
    const int child = node * kFan + lane;
    const bool real = child < octant_real_nodes(g, oct, l - 1);
    const double* src = l == 1 ? a.tile_part + ((int64_t)oct * g.M - g.tile0 + child) * nf
                               : a.node_part[l - 1] + ((int64_t)loct * g.nodes[l - 1] + child) * nf;
    double* dst = a.node_part[l] + ((int64_t)loct * g.nodes[l] + node) * nf;
    for (int f = 0; f < nf; ++f) {
      double v = real ? __ldcg(src + f) : 0.0;
      if (real) const_cast<double*>(src)[f] = sentinel();  // consumed: back to unpublished
      v = warp_tree(v, f == nf - 1);
      if (lane == 0) dst[f] = v;
    }
    if (l == g.levels) break;
    node >>= 5;
    ++l;
    if (lane == 0) prev = atom_add_acq_rel(&a.node_cnt[l][(int64_t)loct * g.nodes[l] + node], 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if ((int)prev != node_real_children(g, oct, l, node) - 1) return;
  }
  // octant root published: arrive at the rank
  if (lane == 0) prev = atom_add_acq_rel(&a.ctl->rank_cnt, 1u);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if ((int)prev != rank_real_octants(g) - 1) return;
  if (lane == 0) a.ctl->rank_cnt = 0u;
  {
    const bool real = lane < g.noct && (int64_t)(g.oct0 + lane) * g.M < g.T;
    double* oroot = a.node_part[g.levels];  // one node per octant at the top level
    for (int f = 0; f < nf; ++f) {
      double v = real ? __ldcg(&oroot[lane * nf + f]) : 0.0;
      if (real) oroot[lane * nf + f] = sentinel();
      v = warp_tree(v, f == nf - 1);
      if (lane == 0) {
        a.rank_root[f] = v;
        root_smem[f] = v;
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    if (a.finalize_local) finalize(a.ctl, root_smem, a.c, a.eps, a.max_iters, a.trace, prologue, a.cond, a.use_cond);
    __threadfence();
  }
}

// Octant / level-1 node of local tile lt.
__device__ __forceinline__ void tile_node(const Geometry& g, int lt, int& oct, int& node) {
  const int gt = g.tile0 + lt;
  oct = gt / g.M;
  node = (gt - oct * g.M) >> 5;
}

// One warp publishes the partial of local tile lt (part[f], shared memory),
// arrives at its level-1 node and climbs when it completes it.
__device__ __forceinline__ void publish_climb(const PassArgs& a, int lt, const double* part, double* root_smem,
                                              bool prologue) {
  const int lane = threadIdx.x & 31;
  const int nf = 2 * a.c + 2;
  if (lane == 0)
    for (int f = 0; f < nf; ++f) a.tile_part[(int64_t)lt * nf + f] = part[f];
  int oct, node;
  tile_node(a.g, lt, oct, node);
  unsigned prev = 0;
  if (lane == 0) prev = atom_add_acq_rel(&a.node_cnt[1][(int64_t)(oct - a.g.oct0) * a.g.nodes[1] + node], 1u);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if ((int)prev != node_real_children(a.g, oct, 1, node) - 1) return;
  climb(a, oct, 1, node, root_smem, prologue);
}

// Whole-CTA version (prologue and register-staged pass kernels): reduce the
// per-thread payload of local tile lt to the tile partial, then warp 0
// publishes and climbs while the other warps return to the stream; `buf`
// double-buffers the per-warp scratch for that reason.
template <int C, bool NAMED = false, typename SM>
__device__ __forceinline__ void tile_finish(const PassArgs& a, int lt, const double* acc, SM& sm,
                                            bool prologue, int buf = 0) {
  constexpr int NS = 2 * C + 2;
  const int c = C <= 8 ? C : a.c, nf = 2 * c + 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // lanes -> warp value: the sum fields through the halving butterfly (the
  // same tile-internal tree as the TMA consumers), the max field through a
  // warp tree (max is order-free)
  constexpr int NSUM = NS - 1;
  double v[NSUM];
#pragma unroll
  for (int s = 0; s < NSUM; ++s) v[s] = acc[s];
  bfly_level<NSUM, 16>(v, lane);
#pragma unroll
  for (int k = 0; k < bfly_slots(NSUM); ++k) {
    const int s = bfly_field(lane, NSUM, k);
    const int f = s >= 0 ? field_of<C>(s, c) : -1;
    if (f >= 0) sm.w[buf][warp][f] = v[k];
  }
  const double dm = warp_tree(acc[NS - 1], true);
  if (lane == 0) sm.w[buf][warp][field_of<C>(NS - 1, c)] = dm;
  red_sync<NAMED>();
  if (warp != 0) return;
  for (int f = lane; f < nf; f += 32) {  // nf <= 34
    const bool mx = f == nf - 1;
    const double q0 = combine(sm.w[buf][0][f], sm.w[buf][1][f], mx);
    const double q1 = combine(sm.w[buf][2][f], sm.w[buf][3][f], mx);
    const double q2 = combine(sm.w[buf][4][f], sm.w[buf][5][f], mx);
    const double q3 = combine(sm.w[buf][6][f], sm.w[buf][7][f], mx);
    sm.part[f] = combine(combine(q0, q1, mx), combine(q2, q3, mx), mx);
  }
  __syncwarp();
  publish_climb(a, lt, sm.part, sm.root, prologue);
}

// ---------------------------------------------------------------- loads ---
template <typename XT>
struct XLoad;
template <>
struct XLoad<uint8_t> {
  static __device__ __forceinline__ void load4(const uint8_t* x, int64_t i, double* xd) {
    unsigned w = __ldg(reinterpret_cast<const unsigned*>(x + i));
#pragma unroll
    for (int q = 0; q < 4; ++q) xd[q] = (double)((w >> (8 * q)) & 0xffu);
  }
  static __device__ __forceinline__ double load1(const uint8_t* x, int64_t i) { return (double)x[i]; }
};
template <>
struct XLoad<uint16_t> {
  static __device__ __forceinline__ void load4(const uint16_t* x, int64_t i, double* xd) {
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(x + i));
    xd[0] = (double)(w.x & 0xffffu);
    xd[1] = (double)(w.x >> 16);
    xd[2] = (double)(w.y & 0xffffu);
    xd[3] = (double)(w.y >> 16);
  }
  static __device__ __forceinline__ double load1(const uint16_t* x, int64_t i) { return (double)x[i]; }
};
template <>
struct XLoad<double> {
  static __device__ __forceinline__ void load4(const double* x, int64_t i, double* xd) {
    double2 a = __ldg(reinterpret_cast<const double2*>(x + i));
    double2 b = __ldg(reinterpret_cast<const double2*>(x + i + 2));
    xd[0] = a.x;
    xd[1] = a.y;
    xd[2] = b.x;
    xd[3] = b.y;
  }
  static __device__ __forceinline__ double load1(const double* x, int64_t i) { return x[i]; }
};

__device__ __forceinline__ float f4get(const float4& v, int q) {
  return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
}
__device__ __forceinline__ void f4set(float4& v, int q, float s) {
  if (q == 0) v.x = s;
  else if (q == 1) v.y = s;
  else if (q == 2) v.z = s;
  else v.w = s;
}

__device__ __forceinline__ Powers load_powers(const PassArgs& a) {
  Powers p;
  p.m = a.m;
  p.p = a.p;
  p.pkind = a.pkind;
  p.pint = a.pint;
  p.mkind = a.mkind;
  p.mint = a.mint;
  return p;
}

// ------------------------------------------------------------ the pass ----
// Four voxels per thread per step; u planes move as float4 (128-bit) loads
// and stores, x as one 32-bit (u8) / 64-bit (u16) / 2x128-bit (f64) load.
template <typename XT, int C, int MODE, bool MASK>
__device__ __forceinline__ void pass_tile(const PassArgs& a, int lt, const double* v,
                                          const Powers& pw, double* acc) {
  const int c = a.c;
  const int64_t base = (int64_t)lt << a.g.tile_shift;
  const int steps = (1 << a.g.tile_shift) / (kThreads * kVec);
  const float* ucur = a.u_cur;  // may alias unxt (in-place update)
  float* unxt = a.u_nxt;
  const int64_t plane = a.g.plane;
#pragma unroll 1
  for (int r = 0; r < steps; ++r) {
    const int64_t i0 = base + ((int64_t)r * kThreads + threadIdx.x) * kVec;
    if (MASK && i0 >= a.g.n_local) break;
    double xd[4];
    XLoad<XT>::load4(reinterpret_cast<const XT*>(a.x), i0, xd);
    float4 uo[C], un[C];
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (j < c) uo[j] = __ldcs(reinterpret_cast<const float4*>(ucur + j * plane + i0));
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double u[C];
      membership<C, MODE>(xd[q], v, c, pw, u);
      const bool valid = !MASK || (i0 + q < a.g.n_local);
#pragma unroll
      for (int j = 0; j < C; ++j) {
        if (j < c) {
          const double w = pow_m<MODE>(u[j], pw);
          const double dj = xd[q] - v[j];
          const double dl = fabs(u[j] - (double)f4get(uo[j], q));
          if (valid) {
            acc[j] = fma(w, xd[q], acc[j]);
            acc[C + j] += w;
            acc[2 * C] = fma(w, dj * dj, acc[2 * C]);
            acc[2 * C + 1] = fmax(acc[2 * C + 1], dl);
          }
          f4set(un[j], q, (float)u[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (j < c) __stcs(reinterpret_cast<float4*>(unxt + j * plane + i0), un[j]);
  }
}

template <typename XT, int C, int MODE>
__global__ void __launch_bounds__(kThreads) pass_kernel(PassArgs a) {
  __shared__ SmemRed sm;
  if (pass_done(a, sm)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ctl->tile_next[(a.seq + 1) & 1] = 0u;
  double v[C];
#pragma unroll
  for (int j = 0; j < C; ++j) v[j] = j < a.c ? a.ctl->v[j] : 0.0;
  const Powers pw = load_powers(a);
  const int ntiles = a.g.tiles_local;
  for (;;) {
    if (threadIdx.x == 0) sm.tile = (int)atomicAdd(&a.ctl->tile_next[a.seq & 1], 1u);
    __syncthreads();
    const int lt = sm.tile;
    __syncthreads();
    if (lt >= ntiles) break;
    double acc[2 * C + 2];
#pragma unroll
    for (int s = 0; s < 2 * C + 2; ++s) acc[s] = 0.0;
    const bool full = ((int64_t)(lt + 1) << a.g.tile_shift) <= a.g.n_local;
    if (full) pass_tile<XT, C, MODE, false>(a, lt, v, pw, acc);
    else pass_tile<XT, C, MODE, true>(a, lt, v, pw, acc);
    tile_finish<C>(a, lt, acc, sm, false);
    __syncthreads();
  }
}

// ------------------------------------------------------------ prologue ----
// Builds u_0 (fp32 SoA, for delta_1) and the sums of u_0^m x / u_0^m that
// give v_1, from either the seeded generator (bit-exact with
// core.init_membership) or an uploaded fp64 AoS initial membership.
// Seeded start for the 4 consecutive voxels i0..i0+3 of this rank (the same
// thread -> voxel map as the streaming pass): u_0 rows bit-exact with
// core.init_membership (init_row_state), w = u^m folded into acc in voxel
// order, u_0 returned as fp32 for the plane stores.
template <int C, int MODE>
__device__ __forceinline__ void seed_quad(const PassArgs& a, const Powers& pw, int c, int64_t i0,
                                          const double* xd, int64_t nvalid, float4* un, double* acc) {
  constexpr int PM = (MODE == MODE_M2 || MODE == MODE_LUT2) ? MODE_M2 : MODE_GEN;
  // SplitMix64 state before voxel i0's first draw; each row advances it by c*GAMMA
  uint64_t st = a.seed + (uint64_t)(a.g.voxel0 + i0) * ((uint64_t)c * kGamma);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double u[C];
    init_row_advance<C>(st, c, u);
    const bool valid = q < nvalid;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      if (j < c) {
        const double w = pow_m<PM>(u[j], pw);  // the reference's pow(u, m)
        if (valid) {
          acc[j] = fma(w, xd[q], acc[j]);
          acc[C + j] += w;
        }
        f4set(un[j], q, (float)u[j]);
      }
    }
  }
}

template <typename XT, int C, int MODE, bool FROM_SEED>
__global__ void __launch_bounds__(kThreads, C <= 4 ? 4 : 2) prologue_kernel(PassArgs a) {
  __shared__ SmemRedT<2 * C + 2> sm;
  if (pass_done(a, sm)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ctl->tile_next[(a.seq + 1) & 1] = 0u;
  const Powers pw = load_powers(a);
  const int c = C <= 8 ? C : a.c;
  const int ntiles = a.g.tiles_local;
  const int chunks = (1 << a.g.tile_shift) / (kThreads * kVec);
  for (;;) {
    if (threadIdx.x == 0) sm.tile = (int)atomicAdd(&a.ctl->tile_next[a.seq & 1], 1u);
    __syncthreads();
    const int lt = sm.tile;
    __syncthreads();
    if (lt >= ntiles) break;
    double acc[2 * C + 2];
#pragma unroll
    for (int s = 0; s < 2 * C + 2; ++s) acc[s] = 0.0;
    const int64_t base = (int64_t)lt << a.g.tile_shift;
    // 4 consecutive voxels per thread per 1024-voxel chunk, chunk by chunk:
    // the TMA pass's map, so both give the same tile partials bit for bit.
    // The next chunk's pixels are loaded before this chunk's rows are
    // generated (x is padded to whole tiles), so the load latency hides
    // behind the SplitMix64 work instead of stalling it.
    double xn[4];
    XLoad<XT>::load4(reinterpret_cast<const XT*>(a.x), base + threadIdx.x * kVec, xn);
    for (int ch = 0; ch < chunks; ++ch) {
      const int64_t i0 = base + (int64_t)ch * (kThreads * kVec) + threadIdx.x * kVec;
      const int64_t nvalid = a.g.n_local - i0;
      if (nvalid <= 0) break;
      double xd[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) xd[q] = xn[q];
      if (ch + 1 < chunks) XLoad<XT>::load4(reinterpret_cast<const XT*>(a.x), i0 + kThreads * kVec, xn);
      float4 un[C];
      if (FROM_SEED) {
        seed_quad<C, MODE>(a, pw, c, i0, xd, nvalid, un, acc);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool valid = q < nvalid;
#pragma unroll
          for (int j = 0; j < C; ++j) {
            if (j < c) {
              const double u = valid ? a.u0_aos[(i0 + q) * c + j] : 0.0;
              const double w = pow_m<MODE>(u, pw);
              if (valid) {
                acc[j] = fma(w, xd[q], acc[j]);
                acc[C + j] += w;
              }
              f4set(un[j], q, (float)u);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < C; ++j)
        if (j < c) __stcg(reinterpret_cast<float4*>(a.u_nxt + j * a.g.plane + i0), un[j]);
    }
    tile_finish<C>(a, lt, acc, sm, true);
    __syncthreads();
  }
}

// ------------------------------------------------------------ epilogue ----
// u_final = membership(x, v_final) in fp64 AoS (what the reference returns,
// core.py:132) and labels = argmax with ties to the lowest index.
template <typename XT, int C, int MODE>
__global__ void __launch_bounds__(kThreads) epilogue_kernel(EpilogueArgs a) {
  double v[C];
#pragma unroll
  for (int j = 0; j < C; ++j) v[j] = j < a.c ? a.v[j] : 0.0;
  Powers pw;
  pw.m = a.m; pw.p = a.p; pw.pkind = a.pkind; pw.pint = a.pint; pw.mkind = a.mkind; pw.mint = a.mint;
  const int c = a.c;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xd = XLoad<XT>::load1(reinterpret_cast<const XT*>(a.x), i);
    double u[C];
    membership<C, MODE>(xd, v, c, pw, u);
    if (a.u_out) {
#pragma unroll
      for (int j = 0; j < C; ++j)
        if (j < c) a.u_out[i * c + j] = u[j];
    }
    if (a.labels) {
      double best = u[0];
      int bj = 0;
#pragma unroll
      for (int j = 1; j < C; ++j)
        if (j < c && u[j] > best) {
          best = u[j];
          bj = j;
        }
      a.labels[i] = bj;
    }
  }
}

}  // namespace fcm
#include "fcm_tma_kernels.cuh"
namespace fcm {

// ------------------------------------------------------------ launchers ---
template <typename KernelPtr>
inline int occupancy_grid(KernelPtr k, int tiles, int sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  long long g = (long long)per_sm * sms;
  if (g > tiles) g = tiles;
  return g < 1 ? 1 : (int)g;
}

// One translation unit per cluster count C instantiates these (fcm_inst_c*.cu).
// Per-voxel math of a plan: m == 2 product form (C <= 8) or the general
// robust form.  C == 32 (17 <= c <= 32) runs the register-staged pass kernel
// only: no shared-memory stage holds 17..32 membership planes of a chunk.
// For C <= 16 that kernel lost its A/B against the TMA pipeline (round 1:
// 0.60-0.66 vs 0.51 ms per C4 pass) and is not instantiated (the plan
// rejects FCM_OPT_KERNEL = 1 there).
template <int C>
cudaError_t launch_pass_c(int xkind, int mode, const PassArgs& a, int sms, cudaStream_t st,
                          int* grid_out, int variant, int force_grid) {
  constexpr int MD = C <= 8 ? MODE_M2 : MODE_GEN;
  const bool m2 = (mode == MODE_M2) && C <= 8;
  if constexpr (C <= 16) {
    if (variant == 0 || variant == 2 || variant == 3) {  // TMA bulk pipeline (production)
      if (xkind == XK_U8) {
        // uint8 pixels: m == 2 -> fused product form; any other m (or variant 2)
        // -> per-pass intensity table (C <= 8); variant 3 -> direct math always.
        if (C <= 8 && variant != 3 && (variant == 2 || !m2))
          return launch_pass_tma<uint8_t, C, (C <= 8 ? MODE_LUT : MODE_GEN)>(a, sms, st, grid_out, force_grid);
        if (C <= 8 && m2 && variant == 0)
          return launch_pass_tma<uint8_t, C, (C <= 8 ? MODE_LUT2 : MODE_GEN)>(a, sms, st, grid_out, force_grid);
        return m2 ? launch_pass_tma<uint8_t, C, MD>(a, sms, st, grid_out, force_grid)
                  : launch_pass_tma<uint8_t, C, MODE_GEN>(a, sms, st, grid_out, force_grid);
      }
      if (xkind == XK_U16)
        return m2 ? launch_pass_tma<uint16_t, C, MD>(a, sms, st, grid_out, force_grid)
                  : launch_pass_tma<uint16_t, C, MODE_GEN>(a, sms, st, grid_out, force_grid);
      return m2 ? launch_pass_tma<double, C, MD>(a, sms, st, grid_out, force_grid)
                : launch_pass_tma<double, C, MODE_GEN>(a, sms, st, grid_out, force_grid);
    }
  }
  if constexpr (C <= 16) {
    return cudaErrorNotSupported;  // variant 1 (register-staged) is built for C == 32 only
  } else {
  int grid = 0;  // C == 32: register-staged LDG/STG kernel
  auto go = [&](auto k) {
    grid = force_grid > 0 ? std::min(force_grid, a.g.tiles_local) : occupancy_grid(k, a.g.tiles_local, sms);
    k<<<grid, kThreads, 0, st>>>(a);
  };
  if (xkind == XK_U8) {
    if (m2) go(pass_kernel<uint8_t, C, MD>);
    else go(pass_kernel<uint8_t, C, MODE_GEN>);
  } else if (xkind == XK_U16) {
    if (m2) go(pass_kernel<uint16_t, C, MD>);
    else go(pass_kernel<uint16_t, C, MODE_GEN>);
  } else {
    if (m2) go(pass_kernel<double, C, MD>);
    else go(pass_kernel<double, C, MODE_GEN>);
  }
  if (grid_out) *grid_out = grid;
  return cudaGetLastError();
  }
}

template <int C>
cudaError_t launch_loop_c(int xkind, int mode, const PassArgs& a, int sms, cudaStream_t st, int* grid_out,
                          int variant, int force_grid, int share) {
  if constexpr (C > 16) {
    return cudaErrorNotSupported;  // per-pass launches (register-staged kernel)
  } else {
    constexpr int MD = C <= 8 ? MODE_M2 : MODE_GEN;
    const bool m2 = (mode == MODE_M2) && C <= 8;
    if (variant == 1) return cudaErrorNotSupported;  // the LDG kernel has no loop form
    if (xkind == XK_U8) {
      if (C <= 8 && variant != 3 && (variant == 2 || !m2))
        return launch_loop_tma<uint8_t, C, (C <= 8 ? MODE_LUT : MODE_GEN)>(a, sms, st, grid_out, force_grid, share);
      if (C <= 8 && m2 && variant == 0)  // large volumes: the prefetching instantiation
        return a.g.tiles_local > kSmallTiles
                   ? launch_loop_tma<uint8_t, C, (C <= 8 ? MODE_LUT2 : MODE_GEN), true>(a, sms, st, grid_out,
                                                                                       force_grid, share)
                   : launch_loop_tma<uint8_t, C, (C <= 8 ? MODE_LUT2 : MODE_GEN)>(a, sms, st, grid_out, force_grid,
                                                                                 share);
      return m2 ? launch_loop_tma<uint8_t, C, MD>(a, sms, st, grid_out, force_grid, share)
                : launch_loop_tma<uint8_t, C, MODE_GEN>(a, sms, st, grid_out, force_grid, share);
    }
    if (xkind == XK_U16)
      return m2 ? launch_loop_tma<uint16_t, C, MD>(a, sms, st, grid_out, force_grid, share)
                : launch_loop_tma<uint16_t, C, MODE_GEN>(a, sms, st, grid_out, force_grid, share);
    return m2 ? launch_loop_tma<double, C, MD>(a, sms, st, grid_out, force_grid, share)
              : launch_loop_tma<double, C, MODE_GEN>(a, sms, st, grid_out, force_grid, share);
  }
}

template <int C>
cudaError_t launch_prologue_c(int xkind, int mode, bool from_seed, const PassArgs& a, int sms,
                              cudaStream_t st) {
  auto go = [&](auto k) { k<<<occupancy_grid(k, a.g.tiles_local, sms), kThreads, 0, st>>>(a); };
  constexpr int MD = C <= 8 ? MODE_M2 : MODE_GEN;
  const bool m2 = mode == MODE_M2 && C <= 8;
  if (xkind == XK_U8) {
    if (from_seed) m2 ? go(prologue_kernel<uint8_t, C, MD, true>) : go(prologue_kernel<uint8_t, C, MODE_GEN, true>);
    else m2 ? go(prologue_kernel<uint8_t, C, MD, false>) : go(prologue_kernel<uint8_t, C, MODE_GEN, false>);
  } else if (xkind == XK_U16) {
    if (from_seed) m2 ? go(prologue_kernel<uint16_t, C, MD, true>) : go(prologue_kernel<uint16_t, C, MODE_GEN, true>);
    else m2 ? go(prologue_kernel<uint16_t, C, MD, false>) : go(prologue_kernel<uint16_t, C, MODE_GEN, false>);
  } else {
    if (from_seed) m2 ? go(prologue_kernel<double, C, MD, true>) : go(prologue_kernel<double, C, MODE_GEN, true>);
    else m2 ? go(prologue_kernel<double, C, MD, false>) : go(prologue_kernel<double, C, MODE_GEN, false>);
  }
  return cudaGetLastError();
}

template <int C>
cudaError_t launch_epilogue_c(int xkind, int mode, const EpilogueArgs& a, int sms, cudaStream_t st) {
  long long want = (a.n + kThreads - 1) / kThreads;
  long long cap = (long long)sms * 8;
  int grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  const bool m2 = (mode == MODE_M2) && C <= 8;
  constexpr int MD = C <= 8 ? MODE_M2 : MODE_GEN;
  if (xkind == XK_U8) {
    if (m2) epilogue_kernel<uint8_t, C, MD><<<grid, kThreads, 0, st>>>(a);
    else epilogue_kernel<uint8_t, C, MODE_GEN><<<grid, kThreads, 0, st>>>(a);
  } else if (xkind == XK_U16) {
    if (m2) epilogue_kernel<uint16_t, C, MD><<<grid, kThreads, 0, st>>>(a);
    else epilogue_kernel<uint16_t, C, MODE_GEN><<<grid, kThreads, 0, st>>>(a);
  } else {
    if (m2) epilogue_kernel<double, C, MD><<<grid, kThreads, 0, st>>>(a);
    else epilogue_kernel<double, C, MODE_GEN><<<grid, kThreads, 0, st>>>(a);
  }
  return cudaGetLastError();
}

#define FCM_INSTANTIATE(C)                                                                        \
  template cudaError_t launch_pass_c<C>(int, int, const PassArgs&, int, cudaStream_t, int*, int, int); \
  template cudaError_t launch_loop_c<C>(int, int, const PassArgs&, int, cudaStream_t, int*, int, int, int); \
  template cudaError_t launch_prologue_c<C>(int, int, bool, const PassArgs&, int, cudaStream_t); \
  template cudaError_t launch_epilogue_c<C>(int, int, const EpilogueArgs&, int, cudaStream_t);

}  // namespace fcm

// fcm_tma_kernels.cuh -- the TMA kernels: one pass per launch
// (pass_tma_kernel) and the persistent loop kernel, plus their launchers.
// The pass is split in three headers: the stream (fcm_tma_pipe.cuh:
// producer, tables, consumers), the tree (fcm_tma_tree.cuh: reducer,
// publication, pass end, exchange) and these kernels.
//
// The production FCM pass: TMA bulk-copy pipeline.
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
// top of the tile's fixed binary tree), publishes the tile partial with a
// relaxed store and reduces the level-1 tree nodes its CTA owns -- the
// device-scope fences and L2 round trips of the tree never stall a
// consumer.  Bytes in flight per SM are set by the ring depth, not by
// registers, which is what an HBM-bound stream needs.  The persistent loop
// kernel runs every pass of a solve this way.

#pragma once
#include "fcm_tma_tree.cuh"

namespace fcm {

template <typename XT, int C, int MODE>
__device__ __forceinline__ void tma_init_barriers(uint8_t* smem, RedSlots<2 * C + 2>& rs) {
  using L = TmaLayout<XT, C, MODE>;
  const uint32_t bar0 = smem_u32(smem + L::kBarOff);
  for (int s = 0; s < L::kStages; ++s) {
    mbar_init(bar0 + 8u * s, 1);
    mbar_init(bar0 + 8u * (L::kStages + s), kThreads);
  }
  for (int s = 0; s < kSlots; ++s) {
    mbar_init(smem_u32(&rs.full[s]), kThreads);
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

// --------------------------------------------- persistent loop kernel -----
// The whole device loop of core._iterate (core.py:118-131) in ONE launch:
// every CTA stays resident (cooperative launch), runs pass after pass over
// the dynamic tile scheduler, and meets the others at a grid barrier between
// passes; the CTA that completes a pass's reduction tree finalizes v_{k+1}
// and the stop test before it arrives.  u is updated in place.  No
// per-iteration launch, no host round trip, ring barriers initialised once.
// PF (large volumes, uint8 tables): the next pass's static tile is issued at
// the pass end (prefetch_static) and the post-pass scratch lives in the
// table region; a separate instantiation, so the small-volume kernel keeps
// its register allocation (same-box A/B, profiles/ab_r02/variants.txt).
template <typename XT, int C, int MODE, bool PF = false>
__global__ void __launch_bounds__(kTmaThreads, 2) loop_tma_kernel(PassArgs a) {
  constexpr bool LUT = MODE == MODE_LUT;
  constexpr int NF = 2 * C + 2;
  using L = TmaLayout<XT, C, MODE>;
  static_assert(L::kRingBytes >= (kOctants * kFan + kSmallTiles / kFan + kOctants) * NF * 8,
                "ring too small for the upper-level scratch");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ RedSlots<NF> rs;
  __shared__ double oroot[kOctants][NF];
  __shared__ double vsh[C];        // centers at launch (ctl->v)
  __shared__ double vprev[C];      // recompute mode: centers of the previous pass
  __shared__ double sdelta;       // recompute mode: delta of this pass from the tables
  __shared__ uint32_t spresent[8];
  __shared__ int s_done;
  __shared__ volatile int s_abort;  // producer: the previous pass's barrier timed out
  __shared__ __align__(8) uint64_t gatebar;  // producer -> reducer: previous pass's barrier seen
  __shared__ __align__(8) uint64_t upbar;    // bulk copy of the tile partials (small volumes)
  const int tid = threadIdx.x;
  const int c = C <= 8 ? C : a.c;
  if (tid == 0) {
    s_abort = 0;
    mbar_init(smem_u32(&gatebar), 1);  // (tma_init_barriers' fence publishes both)
    mbar_init(smem_u32(&upbar), 1);
    tma_init_barriers<XT, C, MODE>(smem, rs);
    s_done = *(volatile int*)&a.ctl->done;
    for (int j = 0; j < c; ++j) vsh[j] = __ldcg(&a.ctl->v[j]);
  }
  const Powers pw = load_powers(a);
  const int64_t l1_len = (int64_t)a.g.noct * a.g.nodes[1] * (2 * a.c + 2);  // one of 3 buffers
  // small volumes (<= 1024 tiles): no level-1 owners -- every CTA reduces
  // the level-1 nodes itself after the grid barrier (one hop less per pass),
  // in one fused step when the geometry fits a warp (loop_root_small)
  const bool from_tiles = a.g.tiles_local <= kSmallTiles;
  const int fusedP = from_tiles ? fused_lanes_per_octant(a.g) : 0;
  // fence-free pass end (small volumes whose tree fits one warp, loop_root_small):
  // tile partials rotate over THREE buffers by pass generation g (buffer
  // g % 3); the reducer publishing tile t in pass g also resets t's slot in
  // buffer (g+1) % 3 -- last read in pass g-2, i.e. before every CTA arrived
  // at the barrier of pass g-1, which the producer has observed first.  Each
  // CTA arrives at the grid barrier after its stream and immediately polls
  // the published partials for the root (no wait); the barrier is awaited by
  // the producer of the next pass, after its static first tile (whose
  // u_{k-1} this CTA wrote itself), before it claims tiles other CTAs wrote.
  const bool proto_s = fusedP != 0 && !a.debug_shared_parts;
  // the same for large volumes (level-1 owners): owners read this pass's
  // tile-partial buffer without resetting it, publish each level-1 result
  // with relaxed stores into l1_buf[g % 3] and reset the node's slot of
  // l1_buf[(g+1) % 3] (after the gate); after its stream every CTA arrives
  // at the grid barrier and polls the level-1 results for the levels above
  const bool proto_l = !from_tiles && !a.debug_shared_parts;
  const bool proto = proto_s || proto_l;
  // PF: prefetch only when the owner path runs and its scratch fits the table region
  const bool pf = PF && proto_l &&
                  (int64_t)a.g.noct * (a.g.levels == 3 ? a.g.nodes[2] : 1) * NF * 8 <= (int64_t)L::kLutBytes;
  int pre = 0;  // producer: chunks of this pass's static tile already issued
  Pipe pfp;     // producer: ring position of the last prefetch (drained at exit)
  const int64_t tlen = (int64_t)a.g.tiles_local * (2 * a.c + 2);
  // recompute mode (SURVEY 8(d) "effective"): passes >= 2 stream x only;
  // u_{k-1} is never read back -- delta_k = max over the intensities present
  // of |u_k(b) - u_{k-1}(b)| from the two pass tables (fp64, exact)
  const bool recomp = a.recompute && MODE == MODE_LUT2 && sizeof(XT) == 1;
  unsigned l1_real = 0;  // real level-1 nodes of this rank (published once per pass)
  if (!from_tiles && !proto_l)
    for (int lo = 0; lo < a.g.noct; ++lo) l1_real += (unsigned)octant_real_nodes(a.g, a.g.oct0 + lo, 1);
  Pipe ps, sp;
  // monotone tile scheduler: CTA b starts every pass with tile b (no claim),
  // the counter hands out tiles G..T-1 and every producer makes exactly one
  // failing claim, so pass p takes counter values [pT, pT+T) -- no per-pass
  // reset (grid <= tiles, launch_loop_tma)
  // (loop-carried counters are derived from `it`, not kept in registers: the
  // kernel sits at the 96-register cap of 2 CTAs x 320 threads per SM)
  const unsigned sched_step = (unsigned)a.g.tiles_local;
  __syncthreads();
  const unsigned it0 = a.seed_pass ? 0u : 1u;
  for (unsigned it = it0; !s_done && it <= (unsigned)a.max_iters; ++it) {
    if (tid == 0) probe(a, it, 0, global_ns());
    // level-1 results of this pass: buffer (gen+1) % 3; owners publish them
    // after their CTA has entered the grid barrier and count them in
    // ctl->l1_done (release reduction per node); readers wait for the count
    const unsigned gnext = it - it0 + 1;  // grid-barrier generation closing this pass
    const unsigned sched = (it - it0) * sched_step;
    double* l1 = a.l1_buf + (gnext % 3) * l1_len;
    // small volumes: this pass's tile partials go to the half of tile_part of
    // its parity.  Every CTA reads them after the grid barrier while early
    // CTAs may already publish the next pass's partials -- into the other
    // half; pass it+2 reuses this half only after the barrier of pass it+1,
    // which no CTA passes before every CTA has finished reading.
    // (formed where used: a pointer live across the stream would cost the
    // consumers a register at the cap)
    auto tpart_of = [&](unsigned g) {
      return a.tile_part + (proto ? (int64_t)(g % 3u) * tlen
                            : from_tiles && !a.debug_shared_parts ? (int64_t)(g & 1u) * tlen : 0);
    };
    if (tid >= kThreads) {
      if (tid == kProducerTid) {
        fence_proxy_async_global();
        const ProduceGate gate{&a.ctl->bar_count, (gnext - 1u) * gridDim.x, smem_u32(&gatebar)};
        const int n = tma_produce<XT, C, MODE>(a, smem, ps, &a.ctl->tile_next[1], it, it == 0 || (recomp && it >= 2),
                                                     sched, true, proto ? &gate : nullptr, pre);
        pre = 0;
        if (n < 0) {
          a.ctl->dead = -3;  // a stuck CTA (cannot happen with co-resident CTAs): flag the run
          a.ctl->done = 1;
          s_abort = 1;
        }
        probe(a, it, 1, global_ns());
        probe(a, it, 4, (uint64_t)n);
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        probe(a, it, 6, smid);
      }
      if ((tid >> 5) == kReducerWarp) {
        // slots first (then arrive at the pass-end barrier), owned level-1
        // nodes after -- overlapping the grid barrier
        tma_reduce<C, true>(a, rs, sp, &a.ctl->tile_next[1], l1, it, from_tiles, sched, tpart_of(gnext),
                            proto ? tpart_of(gnext + 1u) : nullptr, smem_u32(&gatebar), (gnext - 1u) & 1u,
                            proto_l ? a.l1_buf + ((gnext + 1u) % 3u) * l1_len : nullptr);
        if ((tid & 31) == 0) probe(a, it, 7, global_ns());
      } else {
        bar_sync_end();
        if (PF && pf && it < (unsigned)a.max_iters) {  // the producer warp (drained at exit if unused)
          pfp = ps;
          const int n = prefetch_static<XT, C, MODE>(a, smem, ps, recomp && it + 1u >= 2u);
          if (tid == kProducerTid) pre = n;
        }
      }
    } else {
      if (it == 0) {
        tma_consume_seed<XT, C, MODE>(a, smem, ps, rs, sp, pw);
      } else {
        // centers of this pass: v_{k} = root[j] / root[c + j] of the previous
        // pass (the IEEE quotient loop_decide publishes), formed by every
        // consumer from the shared root -- rs.root is rewritten only after
        // this pass's grid barrier; the run's first pass takes ctl->v
        double v[C];
#pragma unroll
        for (int j = 0; j < C; ++j) v[j] = j >= c ? 0.0 : it == it0 ? vsh[j] : rs.root[j] / rs.root[c + j];
        double lwx[C], lwb[C], ljb = 0.0;
        if (LUT) tma_build_lut<C>(smem + L::kLutOff, v, c, pw, lwx, lwb, ljb);
        if (MODE == MODE_LUT2) tma_build_lut2<C>(smem + L::kLutOff, v);
        if (recomp && it >= 2) {
          if (tid < 8) spresent[tid] = __ldcg(&a.ctl->present[tid]);
          red_sync<true>();
          table_delta<C>(v, vprev, spresent, c, &sdelta);  // (vprev: v_{k-1}, stored below last pass)
          tma_consume<XT, C, MODE, true>(a, smem, ps, rs, sp, v, pw, lwx, lwb, ljb, it);
        } else {
          tma_consume<XT, C, MODE>(a, smem, ps, rs, sp, v, pw, lwx, lwb, ljb, it);
        }
        if (recomp) {  // read after the next grid barrier (constant indices: v stays in registers)
#pragma unroll
          for (int j = 0; j < C; ++j)
            if (tid == j && j < c) vprev[j] = v[j];
        }
        if (tid == 0) probe(a, it, 2, global_ns());
      }
      bar_sync_end();
    }
    const unsigned gen = gnext;
    uint32_t upphase = (it - it0) & 1u;  // bulk copies of the tile partials so far (one per pass)
    const double* tpart = tpart_of(gnext);
    if (proto_s) {
      // arrive (release: this CTA's u_k and tile partials), do not wait
      if (tid == 0) {
        red_release_add(&a.ctl->bar_count, 1u);
        probe(a, it, 3, global_ns());
      }
      if (a.debug_delay_ns) {  // race test: one CTA (a different one each pass) reads late
        if (tid == 0 && blockIdx.x == (it * 7u + 1u) % gridDim.x) {
          const uint64_t t0 = global_ns();
          while (global_ns() - t0 < a.debug_delay_ns) __nanosleep(1000);
        }
        __syncthreads();
      }
      const double xdelta = (recomp && it >= 2) ? sdelta : 0.0;
      const bool ok = loop_root_small<NF>(a, reinterpret_cast<double*>(smem), L::kRingBytes / 8, tpart, fusedP,
                                          rs.root, it, xdelta, 0u, &upphase, true);
      if (!ok || s_abort) {
        if (tid == 0) {
          a.ctl->dead = -3;
          a.ctl->done = 1;
        }
        break;
      }
    } else if (proto_l) {
      if (tid == 0) {  // arrive (release: u_k and the owned level-1 results come later,
        red_release_add(&a.ctl->bar_count, 1u);  // published by their own pattern), do not wait
        probe(a, it, 3, global_ns());
      }
      if (a.debug_delay_ns) {  // race test: one CTA (a different one each pass) reads late
        if (tid == 0 && blockIdx.x == (it * 7u + 1u) % gridDim.x) {
          const uint64_t t0 = global_ns();
          while (global_ns() - t0 < a.debug_delay_ns) __nanosleep(1000);
        }
        __syncthreads();
      }
      const double xdelta = (recomp && it >= 2) ? sdelta : 0.0;
      const bool ok = loop_upper<NF>(a, l1, reinterpret_cast<double*>(smem + (PF && pf ? L::kLutOff : 0)), oroot,
                                     rs.root, it, false, xdelta, 0u, &upphase, L::kRingBytes / 8, nullptr, true);
      if (!ok || s_abort) {
        if (tid == 0) {
          a.ctl->dead = -3;
          a.ctl->done = 1;
        }
        break;
      }
    } else {
      if (tid == 0) {
        if (!grid_barrier(a.ctl, gen, gridDim.x) || (l1_real && !wait_count(&a.ctl->l1_done, gen * l1_real))) {
          a.ctl->dead = -3;  // a stuck CTA (cannot happen with co-resident CTAs): flag the run
          a.ctl->done = 1;
          s_done = 1;
        }
        probe(a, it, 3, global_ns());
      }
      __syncthreads();
      if (s_done) break;
      if (a.debug_delay_ns) {  // race test: one CTA (a different one each pass) reads late
        if (tid == 0 && blockIdx.x == (it * 7u + 1u) % gridDim.x) {
          const uint64_t t0 = global_ns();
          while (global_ns() - t0 < a.debug_delay_ns) __nanosleep(1000);
        }
        __syncthreads();
      }
      const double xdelta = (recomp && it >= 2) ? sdelta : 0.0;
      if (fusedP)
        loop_root_small<NF>(a, reinterpret_cast<double*>(smem), L::kRingBytes / 8, tpart, fusedP, rs.root, it,
                            xdelta, smem_u32(&upbar), &upphase);
      else
        loop_upper<NF>(a, l1, reinterpret_cast<double*>(smem), oroot, rs.root, it, from_tiles, xdelta,
                       smem_u32(&upbar), &upphase, L::kRingBytes / 8, tpart);
    }
    if (tid == 0) probe(a, it, 10, global_ns());
    if (a.mb_ranks > 1 && !exchange_roots(a, rs.root, gen)) {
      if (tid == 0) {
        a.ctl->dead = -4;  // a peer's root never arrived (ctl->stuck_rank / stuck_pass)
        a.ctl->done = 1;
      }
      break;
    }
    // stop test and v_{k+1}: every thread from the same root (no barrier);
    // rs.root is next written after the next grid barrier
    if (loop_decide(a, rs.root, it)) break;
    if (tid == 0) probe(a, it, 14, global_ns());
  }
  // a prefetch for a pass that never ran: its bulk copies must land before
  // the CTA's shared memory goes away
  if (PF && tid == kProducerTid && pre > 0) {
    const uint32_t bar0 = smem_u32(smem + L::kBarOff);
    for (int k = 0; k < pre; ++k) {
      mbar_wait(bar0 + 8u * pfp.stage, pfp.phase);
      pfp.advance<L::kStages>();
    }
  }
  // (the scheduler counter and the barrier count are reset by fcm_run's
  // control-block upload before the next launch)
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
template <typename XT, int C, int MODE, bool PF = false>
inline cudaError_t launch_loop_tma(const PassArgs& a, int sms, cudaStream_t st, int* grid_out,
                                   int force_grid, int share = 1) {
  using L = TmaLayout<XT, C, MODE>;
  auto k = loop_tma_kernel<XT, C, MODE, PF>;
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

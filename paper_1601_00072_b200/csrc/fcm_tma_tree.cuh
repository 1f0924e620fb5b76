// fcm_tma_tree.cuh -- the reduction half of the TMA pass: reducer warp,
// fence-free publication of tile partials, level-1 owners, the upper tree
// levels, the grid barrier, the loop kernel's stop test and the multi-rank
// mailbox exchange.  Part of the TMA pass (fcm_tma_kernels.cuh).
#pragma once
#include "fcm_tma_pipe.cuh"

namespace fcm {

// ------------------------------------------------------------- reducer ----
// Poll-and-reduce of one tree node by one warp: lane i reads child i's NF
// fields (children < nreal; the rest count as 0.0).  Returns false, without
// side effects, while any child is unpublished; otherwise resets the children
// to unpublished and leaves the per-field adjacent-pair warp tree in lane 0
// of out[f] (out in shared or global memory, written by lane 0).
template <int NF, bool GLOBAL_OUT, bool RESET = true>
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
      if (RESET && real) st_relaxed(src + f, sentinel());
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

// Recompute mode, consumer threads (thread b = intensity b): this pass's
// delta = max over the intensities present in the rank of
// max_j |u_k(b)_j - u_{k-1}(b)_j|, both from the m == 2 product form in
// fp64 (v = v_k, vprev = v_{k-1}).  max is order-independent, so every CTA
// gets the same value.  Ends with a consumer barrier.
template <int C>
__device__ __forceinline__ void table_delta(const double* v, const double* vprev, const uint32_t* present, int c,
                                            double* out) {
  __shared__ double wmax[kWarps];
  const int b = threadIdx.x;
  double d = 0.0;
  if ((present[b >> 5] >> (b & 31)) & 1u) {
    double uk[C], up[C], ok, op;
    m2_membership<C>((double)b, v, uk, ok);
    m2_membership<C>((double)b, vprev, up, op);
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (j < c) d = fmax(d, fabs(uk[j] - up[j]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
  if ((b & 31) == 0) wmax[b >> 5] = d;
  red_sync<true>();
  if (b == 0) {
    double m = 0.0;
    for (int w = 0; w < kWarps; ++w) m = fmax(m, wmax[w]);
    *out = m;
  }
  red_sync<true>();
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
                                           bool no_owners = false, unsigned base = 0,
                                           double* tile_out = nullptr, double* tile_reset = nullptr,
                                           uint32_t gate_mbar = 0u, uint32_t gate_parity = 0u,
                                           double* l1_reset = nullptr) {
  constexpr int NF = 2 * C + 2;
  const int lane = threadIdx.x & 31;
  const int nf = 2 * a.c + 2;
  const Geometry& g = a.g;
  const int G = gridDim.x;
  const bool cta0 = blockIdx.x == 0;
  const int NA = no_owners ? 0 : g.noct * g.nodes[1];  // list A: level-1 nodes
  // tile partials go to half 0 of tile_part, or (loop kernel, small volumes)
  // to the half of this pass's parity
  double* const tpart = tile_out ? tile_out : a.tile_part;
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
  bool slots_done = false, reset_ok = false;
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
          st_relaxed(tpart + (int64_t)t * nf + f, combine(combine(q0, q1, mx), combine(q2, q3, mx), mx));
        }
      } else {
        slots_done = true;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&rs.empty[sp.stage]));
      sp.advance<kSlots>();
      // (loop kernel, small volumes: the slot tile t takes two passes from
      // now is reset to unpublished -- after the partial is out, and once the
      // producer has seen the previous pass's grid barrier, i.e. every CTA
      // has finished reading the pass that last used it; before this CTA's
      // own barrier arrival, which the resets must precede)
      if (tile_reset && t >= 0) {
        if (!reset_ok) {
          mbar_wait(gate_mbar, gate_parity);  // this pass's phase of the producer's gate
          reset_ok = true;
        }
        for (int f = lane; f < nf; f += 32) st_relaxed(tile_reset + (int64_t)t * nf + f, sentinel());
      }
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
      // (loop kernel: tiles 0..G-1 are every CTA's static first tile, the
      // counter hands out G..)
      node_hot = (LOOP && slots_done) || (int)(ld_relaxed_u32(counter) - base) + (LOOP ? G : 0) > last_lt;
      if (node_hot && l1_reset && !reset_ok) {  // rotation: the node's slots are known reset only
        mbar_wait(gate_mbar, gate_parity);     // once the previous pass's barrier is seen
        reset_ok = true;
      }
      if (node_hot) {
        ++n_poll;
        double* child0 = l == 1 ? tpart + ((int64_t)oct * g.M - g.tile0 + (int64_t)j * kFan) * nf
                                : a.node_part[l - 1] + ((int64_t)lo * g.nodes[l - 1] + (int64_t)j * kFan) * nf;
        double* out = l1_out + ((int64_t)lo * g.nodes[1] + j) * nf;
        if (LOOP && l1_reset) {
          // fence-free (loop kernel, large volumes): the tile partials rotate
          // (their writers reset them), the level-1 result is published with
          // relaxed stores into this pass's buffer and the node's slot of the
          // buffer two passes ahead is reset -- readers poll the results
          advance = try_node<NF, true, false>(child0, nreal, nf, out);
          if (advance)
            for (int f = lane; f < nf; f += 32)
              st_relaxed(l1_reset + ((int64_t)lo * g.nodes[1] + j) * nf + f, sentinel());
        } else if (LOOP) {  // publish, then count it (readers wait for the count after the grid barrier)
          advance = try_node<NF, false>(child0, nreal, nf, out);
          if (advance) {  // (warp-uniform) every lane's sentinel resets, then lane 0's release
            __syncwarp();
            if (lane == 0) red_release_add(&a.ctl->l1_done, 1u);
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

// The adjacent-pair tree over 16 published slots (relaxed loads of global
// memory; children >= nreal count as 0.0), retried until no real child holds
// the unpublished pattern.  False on a 4 s timeout.
__device__ __forceinline__ bool poll_tree16(const double* p, int64_t stride, int nreal, bool mx, double* out) {
  const uint64_t t0 = global_ns();
  for (;;) {
    double v[16];
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = i < nreal ? ld_relaxed(p + (int64_t)i * stride) : 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) ok = ok && !(i < nreal && is_sentinel(v[i]));
    if (ok) {
#pragma unroll
      for (int s2 = 1; s2 < 16; s2 <<= 1)
#pragma unroll
        for (int i = 0; i < 16; i += 2 * s2) v[i] = combine(v[i], v[i + s2], mx);
      *out = v[0];
      return true;
    }
    __nanosleep(64);
    if (global_ns() - t0 > 4000000000ull) return false;
  }
}

// tree32 over published slots: the 32-leaf adjacent-pair tree is
// (children 0..15) + (children 16..31), each half polled as above.
__device__ __forceinline__ bool poll_tree32(const double* p, int64_t stride, int nreal, bool mx, double* out) {
  double lo = 0.0, hi = 0.0;
  if (!poll_tree16(p, stride, nreal < 16 ? nreal : 16, mx, &lo)) return false;
  if (nreal > 16 && !poll_tree16(p + 16 * stride, stride, nreal - 16, mx, &hi)) return false;
  *out = combine(lo, hi, mx);
  return true;
}

// Loop kernel, after the grid barrier of pass `it`: every CTA reduces the
// levels above 1 from the published level-1 results (l1, [noct][nodes[1]][nf]),
// the same fixed tree as everywhere else, into root[] -- redundantly, so no
// further cross-CTA hop is needed.  Each (node, field) pair is one thread's
// tree32; all kTmaThreads threads call it; scratch is the (idle) stage ring.
template <int NF>
__device__ __forceinline__ bool loop_upper(const PassArgs& a, const double* l1, double* scratch,
                                           double (*oroot)[NF], double* root, unsigned it = 0,
                                           bool from_tiles = false, double extra_delta = 0.0,
                                           uint32_t upbar = 0u, uint32_t* upphase = nullptr,
                                           int64_t scratch_doubles = 0, const double* tparts = nullptr,
                                           bool poll = false) {
  const int tid = threadIdx.x;
  const int nf = 2 * a.c + 2;
  const Geometry& g = a.g;
  const int per = g.levels == 3 ? g.nodes[2] : 1;
  // step 0 (small volumes, no level-1 owners): the level-1 nodes themselves,
  // from the tile partials the grid barrier published, into shared memory
  if (tid == 0) probe(a, it, 16, global_ns());
  if (from_tiles) {
    const double* tp = tparts ? tparts : a.tile_part;  // this pass's half of the tile partials
    double* l1s = scratch;
    scratch += (int64_t)g.noct * g.nodes[1] * NF;
    // the rank's tile partials in one bulk copy (TMA) into the idle ring when
    // they fit: one request stream per CTA instead of 32 dependent loads per
    // thread against the same hot L2 lines
    double* tcopy = scratch + kOctants * NF;  // after the upper scratch (levels <= 2 here)
    const int64_t tdoubles = (int64_t)g.tiles_local * nf;
    const bool bulk = upbar != 0u && tdoubles > 0 && (tcopy - l1s) + tdoubles <= scratch_doubles;
    if (bulk) {
      if (tid == 0) {
        fence_proxy_async_global();  // partials: generic stores published by the grid barrier
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_tx(upbar, (uint32_t)(tdoubles * 8));
        bulk_g2s(smem_u32(tcopy), tp, (uint32_t)(tdoubles * 8), upbar);
      }
      mbar_wait(upbar, *upphase);
      *upphase ^= 1u;
    }
    for (int pr = tid; pr < g.noct * g.nodes[1] * nf; pr += kTmaThreads) {
      const int z = pr / nf, f = pr - z * nf;
      const int lo = z / g.nodes[1], j = z - lo * g.nodes[1];
      const int oct = g.oct0 + lo;
      const int nreal = (int64_t)oct * g.M < g.T ? node_real_children(g, oct, 1, j) : 0;
      const int64_t off = ((int64_t)oct * g.M - g.tile0 + (int64_t)j * kFan) * nf + f;
      l1s[(int64_t)z * NF + f] = nreal == 0 ? 0.0
                                 : bulk   ? tree32<false>(tcopy + off, nf, nreal, f == nf - 1)
                                          : tree32<true>(tp + off, nf, nreal, f == nf - 1);
    }
    __syncthreads();
    if (tid == 0) probe(a, it, 17, global_ns());
    l1 = l1s;
  }
  const int ls = from_tiles ? NF : nf;  // row stride of the level-1 results
  // step 1: level-2 nodes (L == 3) or octant roots (L == 2) from level-1
  // results (fence-free protocol: polled until published)
  bool ok = true;
  if (g.levels >= 2) {
    for (int pr = tid; pr < g.noct * per * nf; pr += kTmaThreads) {
      const int item = pr / nf, f = pr - item * nf;
      const int lo = item / per, k = item - lo * per;
      const int oct = g.oct0 + lo;
      const int nreal = (int64_t)oct * g.M < g.T ? node_real_children(g, oct, 2, k) : 0;
      const double* src = l1 + ((int64_t)lo * g.nodes[1] + (int64_t)k * kFan) * ls + f;
      double r = 0.0;
      if (nreal) {
        if (poll) ok = ok && poll_tree32(src, ls, nreal, f == nf - 1, &r);
        else r = from_tiles ? tree32<false>(src, ls, nreal, f == nf - 1) : tree32<true>(src, ls, nreal, f == nf - 1);
      }
      scratch[(int64_t)item * NF + f] = r;
    }
    ok = __syncthreads_and(ok) != 0;
    if (tid == 0) probe(a, it, 11, global_ns());
    if (!ok) return false;
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
    if (mx) root[f] = fmax(root[f], extra_delta);  // recompute mode: the table delta
  }
  __syncthreads();
  return true;
}

// Loop kernel, small volumes (<= kSmallTiles tiles), after the grid barrier
// of pass `it`: the rank root from this pass's tile partials with two CTA
// barriers.  Step A (every thread, one (level-1 node, field) pair each): the
// node's 32-leaf tree over the tile partials (tree32), into shared memory.
// Step B (warp w: fields w, w + 10, ...): lane L is (octant lo = L / P,
// level-1 node j = L % P), P = nodes[1] rounded up to a power of two; the P
// lanes of an octant meet in the adjacent-pair shuffle tree (the 32-ary
// level-2 node: children past the real ones are 0.0, and x + 0.0 == x,
// max(x, 0.0) == x for these non-negative sums), the octant roots (lanes 0,
// P, .., 7P; missing octants 0.0) in the 8-leaf pair tree -- exactly
// loop_upper's association, two barriers instead of four.  Eligible when
// levels <= 2 and noct * P <= 32 (fused_lanes_per_octant > 0); otherwise the
// caller uses loop_upper.
__device__ __forceinline__ int fused_lanes_per_octant(const Geometry& g) {
  if (g.levels > 2) return 0;
  int P = 1;
  while (P < g.nodes[1]) P <<= 1;
  return g.noct * P <= 32 ? P : 0;
}

// `poll` (the fence-free protocol of the loop kernel): called right after
// this CTA's own stream, before any grid barrier -- step A reads the slots
// with relaxed loads and waits for every real one to be published (the tile
// partials rotate over three buffers, see loop_tma_kernel).  Returns false on
// a timeout.
template <int NF>
__device__ __forceinline__ bool loop_root_small(const PassArgs& a, double* scratch, int64_t scratch_doubles,
                                                const double* tp, int P, double* root, unsigned it,
                                                double extra_delta, uint32_t upbar, uint32_t* upphase,
                                                bool poll = false) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nf = 2 * a.c + 2;
  const Geometry& g = a.g;
  const int n1 = g.nodes[1];
  if (tid == 0) probe(a, it, 16, global_ns());
  // the rank's tile partials in one bulk copy (TMA) into the idle ring when
  // they fit: one request stream per CTA instead of 32 loads per thread
  const int64_t tdoubles = (int64_t)g.tiles_local * nf;
  const int64_t tpad = (tdoubles + 15) & ~(int64_t)15;
  const bool bulk = !poll && upbar != 0u && tdoubles > 0 && tpad + 32 * NF <= scratch_doubles;
  double* l1s = bulk ? scratch + tpad : scratch;  // [noct * n1][NF]
  bool ok = true;
  if (bulk) {
    if (tid == 0) {
      fence_proxy_async_global();  // partials: generic stores published by the grid barrier
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_tx(upbar, (uint32_t)(tdoubles * 8));
      bulk_g2s(smem_u32(scratch), tp, (uint32_t)(tdoubles * 8), upbar);
    }
    mbar_wait(upbar, *upphase);
    *upphase ^= 1u;
  }
  // step A: level-1 nodes (consecutive threads take consecutive fields of a node)
  for (int pr = tid; pr < g.noct * n1 * nf; pr += kTmaThreads) {
    const int z = pr / nf, f = pr - z * nf;
    const int lo = z / n1, j = z - lo * n1;
    const int oct = g.oct0 + lo;
    const int nreal = (int64_t)oct * g.M < g.T ? node_real_children(g, oct, 1, j) : 0;
    const int64_t off = ((int64_t)oct * g.M - g.tile0 + (int64_t)j * kFan) * nf + f;
    double r = 0.0;
    if (nreal) {
      if (poll) ok = ok && poll_tree32(tp + off, nf, nreal, f == nf - 1, &r);
      else r = bulk ? tree32<false>(scratch + off, nf, nreal, f == nf - 1) : tree32<true>(tp + off, nf, nreal, f == nf - 1);
    }
    l1s[(int64_t)z * NF + f] = r;
  }
  const bool all_ok = __syncthreads_and(ok);
  if (tid == 0) probe(a, it, 17, global_ns());
  if (!all_ok) return false;
  // step B: level 2 and the rank root, one warp per field, shuffles only
  const int lo = lane / P, j = lane - lo * P;
  const bool lane_real = lo < g.noct && j < n1;
  for (int f = warp; f < nf; f += kTmaThreads / 32) {
    const bool mx = f == nf - 1;
    double v = lane_real ? l1s[(int64_t)(lo * n1 + j) * NF + f] : 0.0;
    for (int s = 1; s < P; s <<= 1) {  // level 2: the octant's level-1 nodes
      const double o = __shfl_down_sync(0xffffffffu, v, s);
      if ((lane & (2 * s - 1)) == 0) v = combine(v, o, mx);
    }
    for (int s = P; s < 8 * P; s <<= 1) {  // the rank root over the octants
      const double o = __shfl_down_sync(0xffffffffu, v, s & 31);
      if ((lane & (2 * s - 1)) == 0 && lane + s < 32) v = combine(v, o, mx);
    }
    if (lane == 0) root[f] = mx ? fmax(v, extra_delta) : v;  // recompute mode: the table delta
  }
  __syncthreads();
  return true;
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
__device__ __forceinline__ bool grid_barrier(Control* ctl, unsigned gen, unsigned ncta) {
  // release this CTA's writes (tile partials, u), arrive, then wait until the
  // monotone count reaches gen * ncta -- no last-arriver hop, no reset.
  // red.release (MEMBAR.ALL.GPU + REDG) instead of __threadfence + atomicAdd
  // (MEMBAR.SC.GPU + CCTL.IVALL + ATOMG with a return trip)
  red_release_add(&ctl->bar_count, 1u);
  const unsigned target = gen * ncta;
  const uint64_t t0 = global_ns();
  while ((int)(ld_acquire_u32(&ctl->bar_count) - target) < 0) {
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
  while ((int)(ld_acquire_u32(ctr) - target) < 0) {  // modular: counts may wrap on very long runs
    __nanosleep(32);
    if (global_ns() - t0 > 4000000000ull) return false;
  }
  return true;
}

// Loop kernel, EVERY thread once the root of pass `it` is in root[] (shared
// memory): the decisions of finalize_body (core.py:120-131: converged,
// max_iters, DegenerateClusterError(j)) evaluated redundantly -- every thread
// reads the same root, so all decide alike and no CTA barrier or serial
// thread-0 step sits between the root and the next pass.  Thread 0 of CTA 0
// publishes the outcome (control block, objective and delta traces, v_{k+1}
// = root[j] / root[c + j], the IEEE quotient every thread also forms).
__device__ __forceinline__ bool loop_decide(const PassArgs& a, const double* root, unsigned it) {
  const int c = a.c;
  bool conv = false, done = false;
  if (it != 0) {  // (it == 0: the seeded start -- v_1 or DegenerateClusterError, core.py:121-123)
    conv = root[2 * c + 1] < a.eps;
    done = conv || (int)it >= a.max_iters;
  }
  int dead = -1;
  if (!done)
    for (int j = 0; j < c; ++j)
      if (root[c + j] == 0.0) {
        dead = j;
        done = true;
        break;
      }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Control* ctl = a.ctl;
    for (int f = 0; f < 2 * c + 2; ++f) ctl->root[f] = root[f];
    if (it != 0) {
      const int k = (int)it;
      for (int f = 0; f < 2 * c + 2; ++f) a.rank_root[f] = root[f];
      ctl->iter = k;
      a.trace[k - 1] = root[2 * c];
      a.trace[a.max_iters + k - 1] = root[2 * c + 1];  // delta trace (second half of the buffer)
      ctl->delta = root[2 * c + 1];
      ctl->converged = conv ? 1 : 0;
    }
    ctl->dead = dead;
    if (!done)
      for (int j = 0; j < c; ++j) ctl->v[j] = root[j] / root[c + j];
    ctl->done = done ? 1 : 0;
  }
  return done;
}

// Loop kernel, multi-rank: publish this rank's root (in root[], every CTA
// has it) to every rank's mailbox, wait for all ranks' roots of this pass in
// the local mailbox, and replace root[] by the rank-ordered pair tree over
// them -- the same tree the octants use (tree_model.combine_ranks), so the
// global root is the single-rank root bit for bit.  All threads call it.
// Returns false when a peer's root does not arrive within peer_timeout_ns
// (a peer died or is stuck): the rank and pass are recorded for the host.
__device__ __forceinline__ bool exchange_roots(const PassArgs& a, double* root, unsigned gen) {
  const int tid = threadIdx.x;
  const int nf = 2 * a.c + 2;
  const int par = gen & 1;
  const unsigned tag = (a.mb_run << 16) | (gen & 0xffffu);
  if (blockIdx.x == 0 && tid < a.mb_ranks) {  // thread p writes rank p's copy (NVLink stores)
    Mailbox* mb = a.mbox_peer[tid];
    for (int f = 0; f < nf; ++f) mb->root[par][a.mb_rank][f] = root[f];
    // (timeline runs: the publication time rides in the slot's unused last
    // field, so the receiver can time the exchange -- one device, one clock)
    if (a.prof) mb->root[par][a.mb_rank][kNFMax - 1] = __longlong_as_double((long long)global_ns());
    // the release orders this thread's own root stores before the tag: no
    // separate system fence
    st_release_sys_u32(&mb->tag[par][a.mb_rank], tag);
  }
  // every rank's tag polled at once (thread r waits for rank r): one
  // round trip after the last publication, not one per rank
  bool ok = true;
  if (tid < a.mb_ranks) {
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys_u32(&a.mbox_local->tag[par][tid]) != tag) {
      __nanosleep(32);
      if (global_ns() - t0 > a.peer_timeout_ns) {  // rank tid is dead or stuck: name it
        ok = false;
        atomicMin(&a.ctl->stuck_rank, tid);  // (the lowest missing rank is named)
        a.ctl->stuck_pass = gen;
        break;
      }
    }
  }
  const bool all_ok = __syncthreads_and(ok) != 0;
  if (a.prof && all_ok && tid == 0) {  // 21: every root here; 22: the last rank's publication
    const uint64_t t_all = global_ns();
    uint64_t t_pub = 0;
    for (int r = 0; r < a.mb_ranks; ++r)
      t_pub = max(t_pub, (uint64_t)__double_as_longlong(ld_relaxed_sys(&a.mbox_local->root[par][r][kNFMax - 1])));
    probe(a, gen - (a.seed_pass ? 1u : 0u), 21, t_all);
    probe(a, gen - (a.seed_pass ? 1u : 0u), 22, t_pub);
  }
  if (!all_ok) return false;
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

}  // namespace fcm

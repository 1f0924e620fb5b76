// fcm_kernels.h -- internal interface between the C-ABI host code and the
// CUDA kernels (not part of the public ABI; see include/fcm_b200.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fcm_device.cuh"

namespace fcm {

enum { XK_U8 = 0, XK_U16 = 1, XK_F64 = 2 };

struct PassArgs {
  const void* x;          // pixels of this rank, padded to the plane length
  const float* u_cur;     // u_{k-1}, fp32 SoA: plane j at u_cur + j * plane
  float* u_nxt;           // u_k (== u_cur: updated in place)
  const double* u0_aos;   // prologue source when not seeded
  uint64_t seed;          // prologue source when seeded
  int c;
  double m, p;
  int pkind, pint, mkind, mint;
  double eps;
  int max_iters;
  int seq;                // pass sequence number in this run (tile-scheduler parity)
  Geometry g;
  double* tile_part;      // level 0: [3][tiles_local][nf] (the loop kernel's small-volume path
                          // rotates the three buffers by pass generation; every other path uses buffer 0)
  double* node_part[kMaxLevels + 1];  // level l >= 1: [noct][nodes[l]][nf]
  unsigned* node_cnt[kMaxLevels + 1]; // level l >= 1: [noct][nodes[l]] arrival counters
  double* rank_root;      // [nf]
  Control* ctl;
  double* trace;          // [2][max_iters]: objective J_k, then delta_k
  cudaGraphConditionalHandle cond;  // device-side loop: while(cond) { pass } (graph mode)
  int use_cond;
  int finalize_local;     // 1: the CTA completing the rank root finalizes (single-rank jobs)
  int keep_l2;            // 1: x + u fit in L2 -> evict_last loads/stores (next pass hits L2)
  double* l1_buf;         // loop kernel: level-1 node results [3][noct][nodes[1]][nf] (generation mod 3)
  int seed_pass;          // loop kernel: 1 = run the seeded start as pass 0 (no prologue kernel)
  int recompute;          // loop kernel: passes >= 2 stream x only; delta from the intensity tables
  int mb_ranks;           // loop kernel: ranks exchanging roots through mailboxes (1 = none)
  int mb_rank;            // this rank's slot
  unsigned mb_run;        // run tag (fcm_run counter, identical on every rank)
  Mailbox* mbox_local;              // this rank's mailbox (device memory of this rank)
  Mailbox* mbox_peer[kOctants];     // every rank's mailbox as mapped here (peer / IPC pointers)
  uint64_t* prof;         // loop-kernel timeline [prof_passes][grid][kProbeSlots] or null
  int prof_passes;
  unsigned debug_delay_ns;  // FCM_OPT_DEBUG_DELAY: one CTA per pass sleeps this long after the grid
                            // barrier (race-detection test; 0 in production)
  int debug_shared_parts;   // FCM_OPT_DEBUG_SHARED_PARTIALS: one tile-partial buffer for every pass
  uint64_t peer_timeout_ns; // loop kernel, multi-rank: wait this long for a peer's root (FCM_OPT_PEER_TIMEOUT_MS)
};
constexpr int kProbeSlots = 24;

struct FinalizeArgs {
  const double* roots[kOctants];  // rank r's reduction root (peer, local or NCCL-gathered)
  int nranks, c;
  double eps;
  int max_iters;
  int prologue;
  Control* ctl;
  double* trace;
  cudaGraphConditionalHandle cond;
  int use_cond;
};

struct EpilogueArgs {
  const void* x;
  int64_t n;
  int c;
  const double* v;
  double m, p;
  int pkind, pint, mkind, mint;
  double* u_out;    // AoS fp64 [n][c] or null
  int32_t* labels;  // [n] or null
};

// variant 0: TMA bulk-copy pipeline (default); 1: register-staged LDG kernel.
cudaError_t launch_pass(int xkind, int c, int mode, const PassArgs& a, int sms, cudaStream_t st,
                        int* grid_out, int variant = 0, int force_grid = 0);
// Persistent loop kernel (all passes of a run in one cooperative launch);
// returns cudaErrorCooperativeLaunchTooLarge when the grid cannot be resident.
cudaError_t launch_loop(int xkind, int c, int mode, const PassArgs& a, int sms, cudaStream_t st,
                        int* grid_out, int variant = 0, int force_grid = 0, int share = 1);
cudaError_t launch_prologue(int xkind, int c, int mode, bool from_seed, const PassArgs& a, int sms,
                            cudaStream_t st);
cudaError_t launch_epilogue(int xkind, int c, int mode, const EpilogueArgs& a, int sms,
                            cudaStream_t st);
cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st);

}  // namespace fcm

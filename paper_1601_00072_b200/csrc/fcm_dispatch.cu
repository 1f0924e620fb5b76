// fcm_dispatch.cu -- runtime (x kind, c, m) -> kernel instantiation, and the
// multi-rank finalize kernel.  Instantiations live in fcm_inst_c*.cu so the
// build compiles them in parallel.
#include "fcm_kernels.cuh"

namespace fcm {

#define FCM_EXTERN(C)                                                                                \
  extern template cudaError_t launch_pass_c<C>(int, int, const PassArgs&, int, cudaStream_t, int*, int, int); \
  extern template cudaError_t launch_loop_c<C>(int, int, const PassArgs&, int, cudaStream_t, int*, int, int, int); \
  extern template cudaError_t launch_prologue_c<C>(int, int, bool, const PassArgs&, int, cudaStream_t); \
  extern template cudaError_t launch_epilogue_c<C>(int, int, const EpilogueArgs&, int, cudaStream_t);
FCM_EXTERN(2) FCM_EXTERN(3) FCM_EXTERN(4) FCM_EXTERN(5) FCM_EXTERN(6) FCM_EXTERN(7) FCM_EXTERN(8) FCM_EXTERN(16)
FCM_EXTERN(32)

__global__ void finalize_kernel(FinalizeArgs a) {
  // Combine the N rank roots (already gathered, rank-major) in the binary
  // tree that continues each rank's octant tree, then finalize.
  __shared__ double root[kNFMax];
  const int nf = 2 * a.c + 2;
  const int lane = threadIdx.x;
  if (*(volatile int*)&a.ctl->done) {
    if (a.use_cond && lane == 0) cudaGraphSetConditional(a.cond, 0u);
    return;
  }
  for (int f = 0; f < nf; ++f) {
    double v = lane < a.nranks ? __ldcg(&a.roots[lane][f]) : 0.0;
    v = warp_tree(v, f == nf - 1);
    if (lane == 0) root[f] = v;
  }
  __syncwarp();
  if (lane == 0)
    finalize(a.ctl, root, a.c, a.eps, a.max_iters, a.trace, a.prologue != 0, a.cond, a.use_cond);
}


#define FCM_SWITCH(CALL)          \
  switch (c <= 8 ? c : (c <= 16 ? 16 : 32)) { \
    case 2: return CALL(2);       \
    case 3: return CALL(3);       \
    case 4: return CALL(4);       \
    case 5: return CALL(5);       \
    case 6: return CALL(6);       \
    case 7: return CALL(7);       \
    case 8: return CALL(8);       \
    case 16: return CALL(16);     \
    case 32: return CALL(32);     \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_pass(int xkind, int c, int mode, const PassArgs& a, int sms, cudaStream_t st,
                        int* grid_out, int variant, int force_grid) {
  if (c < 2 || c > kCMaxSupported) return cudaErrorInvalidValue;
#define CALL(C) launch_pass_c<C>(xkind, mode, a, sms, st, grid_out, variant, force_grid)
  FCM_SWITCH(CALL)
#undef CALL
}

cudaError_t launch_loop(int xkind, int c, int mode, const PassArgs& a, int sms, cudaStream_t st,
                        int* grid_out, int variant, int force_grid, int share) {
  if (c < 2 || c > kCMaxSupported) return cudaErrorInvalidValue;
#define CALL(C) launch_loop_c<C>(xkind, mode, a, sms, st, grid_out, variant, force_grid, share)
  FCM_SWITCH(CALL)
#undef CALL
}

cudaError_t launch_prologue(int xkind, int c, int mode, bool from_seed, const PassArgs& a, int sms,
                            cudaStream_t st) {
  if (c < 2 || c > kCMaxSupported) return cudaErrorInvalidValue;
#define CALL(C) launch_prologue_c<C>(xkind, mode, from_seed, a, sms, st)
  FCM_SWITCH(CALL)
#undef CALL
}

cudaError_t launch_epilogue(int xkind, int c, int mode, const EpilogueArgs& a, int sms,
                            cudaStream_t st) {
  if (c < 2 || c > kCMaxSupported) return cudaErrorInvalidValue;
#define CALL(C) launch_epilogue_c<C>(xkind, mode, a, sms, st)
  FCM_SWITCH(CALL)
#undef CALL
}

cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st) {
  finalize_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace fcm

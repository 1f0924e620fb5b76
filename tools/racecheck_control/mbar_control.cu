// Control experiment for compute-sanitizer racecheck on this toolchain: a
// minimal, correct producer/consumer hand-off through shared memory ordered
// ONLY by an mbarrier (the pattern of the FCM pipeline: TMA bulk copy or
// plain stores by one producer thread -> mbarrier -> consumer reads), next
// to the same hand-off ordered by __syncthreads.  If racecheck reports the
// mbarrier variant, its reports on the FCM kernels' mbarrier hand-offs are
// tool limitations, not races.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mbar_control mbar_control.cu
//   compute-sanitizer --tool racecheck ./mbar_control {sync|mbar|tma|ring|relaunch}
#include <cstdio>
#include <cstring>
#include <cstdint>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void handoff(int mode, const float* src, float* out) {
  __shared__ __align__(128) float buf[256];
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int round = 0; round < 4; ++round) {
    if (mode == 0) {  // __syncthreads ordering
      if (t == 0)
        for (int i = 0; i < 256; ++i) buf[i] = src[i] + round;
      __syncthreads();
    } else if (mode == 1) {  // mbarrier ordering, plain stores by one thread
      if (t == 0) {
        for (int i = 0; i < 256; ++i) buf[i] = src[i] + round;
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(s32(&bar)) : "memory");
      }
    } else {  // mbarrier ordering, TMA bulk copy
      if (t == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 1024;" ::"r"(s32(&bar)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];"
                     ::"r"(s32(buf)), "l"(src), "r"(s32(&bar)) : "memory");
      }
    }
    if (mode != 0) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, P;\n\t}" : "=r"(ok) : "r"(s32(&bar)), "r"(round & 1) : "memory");
    }
    out[round * 256 + t] = buf[t];
    __syncthreads();  // every reader done before the next round's writes
  }
}

// The FCM ring: one producer thread (its own warp) fills stage s and
// arrives on full[s]; 8 consumer warps wait on full[s], read, __syncwarp,
// and lane 0 of each warp arrives on empty[s] (count 8); the producer waits
// on empty[s] before it rewrites the stage.  Correct by the PTX memory model
// (__syncwarp orders the lanes' reads before lane 0's release-arrive).
__global__ void ring(const float* src, float* out, int rounds) {
  __shared__ __align__(128) float stage[2][256];
  __shared__ int meta[2];
  __shared__ __align__(8) uint64_t full[2], empty[2];
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < 2; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(s32(&empty[s])) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 256) {  // producer
    for (int r = 0; r < rounds; ++r) {
      const int s = r & 1;
      const uint32_t ph = ((r >> 1) & 1) ^ 1;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, P;\n\t}" : "=r"(ok) : "r"(s32(&empty[s])), "r"(ph) : "memory");
      for (int i = 0; i < 256; ++i) stage[s][i] = src[i] + r;
      meta[s] = r;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&full[s])) : "memory");
    }
  } else if (t < 256) {  // consumers
    for (int r = 0; r < rounds; ++r) {
      const int s = r & 1;
      const uint32_t ph = (r >> 1) & 1;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, P;\n\t}" : "=r"(ok) : "r"(s32(&full[s])), "r"(ph) : "memory");
      out[r * 256 + t] = stage[s][t] + meta[s];
      __syncwarp();
      if ((t & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[s])) : "memory");
    }
  }
}

int main(int argc, char** argv) {
  const char* m = argc > 1 ? argv[1] : "mbar";
  const int mode = !strcmp(m, "sync") ? 0 : (!strcmp(m, "mbar") ? 1 : 2);
  float *src, *out;
  cudaMalloc(&src, 1024);
  cudaMalloc(&out, 4 * 1024);
  cudaMemset(src, 0, 1024);
  if (!strcmp(m, "ring") || !strcmp(m, "relaunch")) {
    float* o2;
    cudaMalloc(&o2, 16 * 1024);
    for (int l = 0; l < (!strcmp(m, "relaunch") ? 3 : 1); ++l) ring<<<1, 288>>>(src, o2, 16);
  } else {
    handoff<<<1, 256>>>(mode, src, out);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("mode %s: %s\n", m, cudaGetErrorString(e));
  return e != cudaSuccess;
}

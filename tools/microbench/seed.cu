// Throughput of the seeded start's per-voxel work (seed_quad: SplitMix64
// rows, correctly rounded quotients, Eq. 3 terms, fp32 stores) in isolation,
// at 16 / 32 / 48 / 64 resident warps per SM, to tell a pipe bound from a
// latency bound (the loop kernel runs it with 16 consumer warps per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1601_00072_b200/csrc seed.cu -o seed
#include <cstdio>
#include "fcm_kernels.cuh"
using namespace fcm;

template <int C>
__global__ void __launch_bounds__(256) seedk(PassArgs a, float* u, double* out, int64_t n) {
  const Powers pw = load_powers(a);
  double acc[2 * C + 2];
  for (int s = 0; s < 2 * C + 2; ++s) acc[s] = 0.0;
  for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i0 < n;
       i0 += (int64_t)gridDim.x * blockDim.x * 4) {
    double xd[4] = {(double)(i0 & 255), (double)((i0 + 1) & 255), (double)((i0 + 2) & 255), (double)((i0 + 3) & 255)};
    float4 un[C];
    seed_quad<C, MODE_LUT2>(a, pw, C, i0, xd, 4, un, acc);
#pragma unroll
    for (int j = 0; j < C; ++j) __stcs(reinterpret_cast<float4*>(u + (int64_t)j * n + i0), un[j]);
  }
  double s = 0;
  for (int k = 0; k < 2 * C + 2; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  const int64_t n = 134217728;
  float* u; double* out;
  cudaMalloc(&u, sizeof(float) * 3 * n);
  cudaMalloc(&out, sizeof(double) * 148 * 8 * 256);
  PassArgs a = {};
  a.seed = 0; a.c = 3; a.m = 2.0; a.p = 2.0; a.pkind = PK_INT; a.pint = 2; a.mkind = MK_INT; a.mint = 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int per_sm = 2; per_sm <= 8; per_sm += 2) {
    const int grid = 148 * per_sm;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      seedk<3><<<grid, 256>>>(a, u, out, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, seedk<3>, 256, 0);
    printf("c=3, %d CTAs x 8 warps per SM (occupancy limit %d): %.3f ms for 512^3 voxels (%s)\n", per_sm, occ, best,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

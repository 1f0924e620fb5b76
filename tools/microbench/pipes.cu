// Per-SM throughput of the instruction classes on the seeded start's path
// (B200, sm_100a): 64-bit integer mixing, fp64 <-> integer / fp32
// conversions, DFMA.  One kernel per class, 8 independent chains per thread,
// 16 warps per SM (the loop kernel's consumer occupancy); prints warp
// instructions per clock per SM.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 pipes.cu -o pipes
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
template <int K>
__global__ void bench(uint64_t* out, long long* clk, uint64_t seed) {
  uint64_t a[8];
  double d[8];
  float f[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed + threadIdx.x * 8 + i; d[i] = 1.0 + 1e-9 * (threadIdx.x + i); f[i] = 0.f; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (K == 0) a[i] = (a[i] ^ (a[i] >> 30)) * 0xBF58476D1CE4E5B9ULL;   // xorshift-multiply (2 SHF, 2 LOP3, 3 IMAD)
      if (K == 1) d[i] = (double)(a[i] + (uint64_t)it) + d[i];            // I2F.F64.U64 (+DADD, IADD)
      if (K == 2) f[i] += __double2float_rn(d[i] * 1.0000001);            // F2F.F32.F64 (+DMUL, FADD)
      if (K == 3) d[i] = fma(d[i], 1.0000001, 1e-9);                     // DFMA
      if (K == 4) a[i] = a[i] * 0xBF58476D1CE4E5B9ULL + 1;                // 64-bit IMAD only
      if (K == 5) a[i] = (a[i] ^ (a[i] >> 30)) + 0x9E3779B97F4A7C15ULL;   // ALU only (SHF, LOP3, IADD3)
    }
  }
  long long t1 = clock64();
  uint64_t s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + (uint64_t)d[i] + (uint64_t)f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  uint64_t* out; long long* clk;
  const int blocks = 148 * 2, threads = 256;
  cudaMalloc(&out, sizeof(uint64_t) * blocks * threads);
  cudaMalloc(&clk, sizeof(long long) * blocks);
  const char* names[] = {"xorshift-mul64 (per op)", "I2F.F64.U64+DADD", "F2F.F32.F64+DMUL+FADD", "DFMA", "IMAD64 mul+add", "SHF/LOP3/IADD (xorshift+add)"};
  for (int k = 0; k < 6; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (k) {
        case 0: bench<0><<<blocks, threads>>>(out, clk, 1); break;
        case 1: bench<1><<<blocks, threads>>>(out, clk, 1); break;
        case 2: bench<2><<<blocks, threads>>>(out, clk, 1); break;
        case 3: bench<3><<<blocks, threads>>>(out, clk, 1); break;
        case 4: bench<4><<<blocks, threads>>>(out, clk, 1); break;
        case 5: bench<5><<<blocks, threads>>>(out, clk, 1); break;
      }
    }
    cudaDeviceSynchronize();
    long long h[blocks];
    cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost);
    double mean = 0; for (int b = 0; b < blocks; ++b) mean += h[b]; mean /= blocks;
    // ops per SM per clock: 2 CTAs per SM x 8 warps x 8 chains x kIters / cycles
    const double ops = 2.0 * 8 * 8 * kIters / mean;
    printf("%-34s %.3f warp-ops/clk/SM  (%.1f cycles per op per warp-chain)\n", names[k], ops, mean / kIters);
  }
  return 0;
}

// fcm_ops.cu -- the kernel seam: single GPU ops on the reference's buffer
// conventions (flat float64, AoS memberships), one call = one op.
// Mirrors _kernels.pyx:44-69 (fill_membership_random), :178-191
// (objective_linear), :211-220 (max_abs_diff), :223-238 (argmax_rows).
// Sums use a fixed two-level tree (per-CTA chunk tree, then one CTA over the
// partials) so every result is deterministic.
#include <algorithm>

#include "fcm_device.cuh"
#include "fcm_ops.h"

namespace fcm {

constexpr int kOpsBlocks = 1024;

__global__ void init_aos_kernel(double* u, int64_t n, int c, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double row[kCMaxSupported];
    init_row<kCMaxSupported>(seed, i, c, row);
    for (int j = 0; j < c; ++j) u[i * c + j] = row[j];
  }
}

// Block tree: thread partials -> warp trees -> adjacent pairs over warps.
__device__ double block_tree(double x, bool is_max) {
  __shared__ double w[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  x = warp_tree(x, is_max);
  if (lane == 0) w[warp] = x;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = warp_tree(lane < nw ? w[lane] : 0.0, is_max);
  }
  __syncthreads();
  return r;
}

// kind 0: objective terms sum_j pow(u_ij, m) (x_i - v_j)^2 ; kind 1: |a_i - b_i| (max)
__global__ void terms_kernel(int kind, const double* x, const double* u, const double* v, int64_t n,
                             int c, double m, const double* a, const double* b, double* partials) {
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    if (kind == 0) {
      double t = 0.0;
      for (int j = 0; j < c; ++j) {
        const double d = x[i] - v[j];
        t += pow(u[i * c + j], m) * (d * d);
      }
      acc += t;
    } else {
      acc = fmax(acc, fabs(a[i] - b[i]));
    }
  }
  const double r = block_tree(acc, kind == 1);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

// Eq. 3 sums of the seam (update_centers_linear, _kernels.pyx:72-90) on the
// reference's AoS fp64 membership: fields [f0, f0 + 16) of the 2c sums
// (f < c: sum pow(u_if, m) x_i; f >= c: sum pow(u_i(f-c), m)), each CTA over
// one contiguous voxel range, block tree per field -> partials[block][16].
constexpr int kCenterFields = 16;
__global__ void centers_terms_kernel(const double* x, const double* u, int64_t n, int c, double m, int f0,
                                     double* partials) {
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  const int nfk = min(kCenterFields, 2 * c - f0);
  double acc[kCenterFields];
#pragma unroll
  for (int k = 0; k < kCenterFields; ++k) acc[k] = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double xi = x[i];
#pragma unroll
    for (int k = 0; k < kCenterFields; ++k) {
      const int f = f0 + k;
      if (k < nfk) {
        const double w = pow(u[i * c + (f < c ? f : f - c)], m);
        acc[k] += f < c ? w * xi : w;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kCenterFields; ++k) {
    const double r = block_tree(acc[k], false);
    if (threadIdx.x == 0) partials[blockIdx.x * kCenterFields + k] = r;
  }
}

// One CTA per field: fold the per-CTA partials of field k (stride 16) in a fixed order.
__global__ void centers_fold_kernel(const double* partials, int np, int f0, int nfk, double* out) {
  const int k = blockIdx.x;
  if (k >= nfk) return;
  double acc = 0.0;
  const int per = (np + blockDim.x - 1) / blockDim.x;
  for (int q = 0; q < per; ++q) {
    const int i = threadIdx.x * per + q;
    if (i < np) acc += partials[i * kCenterFields + k];
  }
  const double r = block_tree(acc, false);
  if (threadIdx.x == 0) out[f0 + k] = r;
}

cudaError_t op_center_sums(const double* x, const double* u, int64_t n, int c, double m, double* scratch,
                           double* sums, int sms, cudaStream_t st) {
  int blocks = (int)std::min<int64_t>((n + 4095) / 4096, (int64_t)sms * 4);
  if (blocks > kOpsBlocks) blocks = kOpsBlocks;
  if (blocks < 1) blocks = 1;
  for (int f0 = 0; f0 < 2 * c; f0 += kCenterFields) {
    centers_terms_kernel<<<blocks, kThreads, 0, st>>>(x, u, n, c, m, f0, scratch);
    centers_fold_kernel<<<kCenterFields, kThreads, 0, st>>>(scratch, blocks, f0, std::min(kCenterFields, 2 * c - f0),
                                                            sums);
  }
  return cudaGetLastError();
}

__global__ void partials_kernel(const double* partials, int np, bool is_max, double* out) {
  // np <= blockDim.x * k: each thread folds a contiguous run, then the block tree.
  double acc = 0.0;
  const int per = (np + blockDim.x - 1) / blockDim.x;
  for (int k = 0; k < per; ++k) {
    const int i = threadIdx.x * per + k;
    if (i < np) acc = is_max ? fmax(acc, partials[i]) : acc + partials[i];
  }
  const double r = block_tree(acc, is_max);
  if (threadIdx.x == 0) *out = r;
}

__global__ void argmax_kernel(const double* u, int32_t* labels, int64_t n, int c) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double best = u[i * c];
    int bj = 0;
    for (int j = 1; j < c; ++j) {
      const double w = u[i * c + j];
      if (w > best) {
        best = w;
        bj = j;
      }
    }
    labels[i] = bj;
  }
}

// Diagnostics: drcp_rn_normal (the seeded init's branch-free reciprocal) vs
// CUDA's __drcp_rn on n SplitMix64-drawn b = 2^e * (1 + f), e uniform in
// [-53, 5], f uniform in [0, 1) -- the row totals' range.  Counts mismatches.
__global__ void rcp_check_kernel(int64_t n, uint64_t seed, unsigned long long* bad) {
  unsigned long long nb = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (uint64_t)(i + 1) * kGamma;
    z = (z ^ (z >> 30)) * kMix1;
    z = (z ^ (z >> 27)) * kMix2;
    z ^= z >> 31;
    const int e = (int)((z >> 52) % 59u) - 53;
    const double b = __hiloint2double((int)(((uint32_t)(e + 1023) << 20) | ((uint32_t)(z >> 32) & 0xfffffu)),
                                      (int)(uint32_t)z);
    if (__double_as_longlong(drcp_rn_normal(b)) != __double_as_longlong(__drcp_rn(b))) ++nb;
  }
  if (nb) atomicAdd(bad, nb);
}

cudaError_t op_rcp_check(int64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t st) {
  rcp_check_kernel<<<148 * 8, kThreads, 0, st>>>(n, seed, bad);
  return cudaGetLastError();
}

static int grid_for(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : (int)g;
}

cudaError_t op_init_aos(double* u, int64_t n, int c, uint64_t seed, cudaStream_t st) {
  init_aos_kernel<<<grid_for(n), kThreads, 0, st>>>(u, n, c, seed);
  return cudaGetLastError();
}

cudaError_t op_reduce(int kind, const double* x, const double* u, const double* v, int64_t n, int c,
                      double m, const double* a, const double* b, double* scratch, double* out,
                      cudaStream_t st) {
  int blocks = (int)((n + 4095) / 4096);
  if (blocks > kOpsBlocks) blocks = kOpsBlocks;
  if (blocks < 1) blocks = 1;
  terms_kernel<<<blocks, kThreads, 0, st>>>(kind, x, u, v, n, c, m, a, b, scratch);
  partials_kernel<<<1, kThreads, 0, st>>>(scratch, blocks, kind == 1, out);
  return cudaGetLastError();
}

cudaError_t op_argmax(const double* u, int32_t* labels, int64_t n, int c, cudaStream_t st) {
  argmax_kernel<<<grid_for(n), kThreads, 0, st>>>(u, labels, n, c);
  return cudaGetLastError();
}

// Integer label statistics: shared-memory bins per
// CTA, one 64-bit global atomic per bin per CTA.  Counts are exact.
__global__ void label_counts_kernel(const int32_t* pred, const int32_t* ref, const uint8_t* mask, int64_t n,
                                    int c, int cref, unsigned long long* bins) {
  __shared__ unsigned sb[kCMaxSupported * kCMaxSupported + 2 * kCMaxSupported + 1];
  const int nb = ref ? c * cref : 2 * c + 1;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sb[b] = 0u;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int p = pred[i];
    if (ref) {
      atomicAdd(&sb[p * cref + ref[i]], 1u);
    } else {
      atomicAdd(&sb[c + 1 + p], 1u);
      if (mask[i]) {
        atomicAdd(&sb[p], 1u);
        atomicAdd(&sb[c], 1u);
      }
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (sb[b]) atomicAdd(&bins[b], (unsigned long long)sb[b]);
}

cudaError_t op_label_counts(const int32_t* pred, const int32_t* ref, const uint8_t* mask, int64_t n, int c,
                            int cref, unsigned long long* bins, cudaStream_t st) {
  int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  if (grid < 1) grid = 1;
  label_counts_kernel<<<grid, 256, 0, st>>>(pred, ref, mask, n, c, cref, bins);
  return cudaGetLastError();
}

}  // namespace fcm

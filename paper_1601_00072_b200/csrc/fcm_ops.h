// fcm_ops.h -- single-op kernels behind the kernel-seam half of the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fcm {
constexpr int kOpsScratch = 1024;  // doubles of scratch op_reduce needs
cudaError_t op_init_aos(double* u, int64_t n, int c, uint64_t seed, cudaStream_t st);
// kind 0: objective (x, u, v, m); kind 1: max |a - b| over n elements
cudaError_t op_reduce(int kind, const double* x, const double* u, const double* v, int64_t n, int c,
                      double m, const double* a, const double* b, double* scratch, double* out,
                      cudaStream_t st);
// Eq. 3 sums of update_centers_linear on AoS fp64 u: sums[0..c) = sum pow(u_ij, m) x_i,
// sums[c..2c) = sum pow(u_ij, m); scratch holds kOpsBlocks * 16 doubles.
constexpr int kCenterScratch = 1024 * 16;
cudaError_t op_center_sums(const double* x, const double* u, int64_t n, int c, double m, double* scratch,
                           double* sums, int sms, cudaStream_t st);
cudaError_t op_argmax(const double* u, int32_t* labels, int64_t n, int c, cudaStream_t st);
// Label statistics of a solve (metrics): bins[p*cref + r] += |pred==p & ref==r| when ref is set;
// bins[p] += |pred==p & mask|, bins[c] += |mask|, bins[c+1+p] += |pred==p| when mask is set.
cudaError_t op_label_counts(const int32_t* pred, const int32_t* ref, const uint8_t* mask, int64_t n, int c,
                            int cref, unsigned long long* bins, cudaStream_t st);
// Diagnostics: mismatches of the seeded init's branch-free reciprocal against __drcp_rn.
cudaError_t op_rcp_check(int64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t st);
}  // namespace fcm

// synthetic.cu -- the separable benchmark objective and its exact bounder on the
// device (the paper's d = 50..300 synthetic benchmark):
//   f(u) = sum_j 5 u_j^2 + cos(50 u_j) on [-1, 1]^d
//     reference SyntheticObjective::evaluate, proj/src/objective.cpp:86-98
//   lower(box) = sum_j min over {a_j, b_j, critical points of the 1-d term in
//     (a_j, b_j)} of 5 x^2 + cos(50 x)
//     reference SeparableBounder::term_min / lower, proj/src/bab.cpp:70-83
// Both are FP64 (the reference's arithmetic); one warp per row / box, lanes over
// the coordinates, a fixed lane-strided order and a fixed shuffle tree, so a row's
// value never depends on the batch it is evaluated in (graph.hpp:102-103's
// guarantee for the unrolled objectives).
#include <cuda_runtime.h>

#include <cstdint>

namespace bp {

namespace {

__device__ __forceinline__ double term(double x) { return 5.0 * x * x + cos(50.0 * x); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  return v;
}

// costs[r] = f(actions[r]) for n_rows rows of d FP32 values; a non-finite row marks its
// subdomain (rows_per_sub consecutive rows) failed, like the rollout kernels.
__global__ void synthetic_eval_kernel(const float* __restrict__ actions, float* __restrict__ costs, int* failed,
                                      long long n_rows, int d, int rows_per_sub) {
  const int lane = threadIdx.x & 31;
  const long long row = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n_rows) return;
  const float* u = actions + row * d;
  double acc = 0.0;
  for (int j = lane; j < d; j += 32) acc += term(static_cast<double>(__ldg(u + j)));
  acc = warp_sum(acc);
  if (lane == 0) {
    const float c = static_cast<float>(acc);
    costs[row] = c;
    if (failed != nullptr && !isfinite(c)) atomicOr(failed + row / rows_per_sub, 1);
  }
}

// lf[i] = sum_j term_min(lo[i][j], hi[i][j]) over the sorted critical points of the
// 1-d term (bab.cpp:32-68, computed once on the host); use[i] == 0 leaves -inf.
__global__ void separable_bound_kernel(const double* __restrict__ lo, const double* __restrict__ hi, int n, int d,
                                       const double* __restrict__ crit, int ncrit, const int* use, double* lf) {
  const int lane = threadIdx.x & 31;
  const int box = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (box >= n) return;
  double acc = 0.0;
  for (int j = lane; j < d; j += 32) {
    const double a = lo[static_cast<size_t>(box) * d + j], b = hi[static_cast<size_t>(box) * d + j];
    double m = fmin(term(a), term(b));
    // first critical point > a (binary search), then every one below b
    int l = 0, r = ncrit;
    while (l < r) {
      const int mid = (l + r) >> 1;
      if (crit[mid] > a) r = mid; else l = mid + 1;
    }
    for (int k = l; k < ncrit && crit[k] < b; ++k) m = fmin(m, term(crit[k]));
    acc += m;
  }
  acc = warp_sum(acc);
  if (lane == 0) lf[box] = (use == nullptr || use[box]) ? acc : -INFINITY;
}

}  // namespace

cudaError_t launch_synthetic_eval(const float* actions, float* costs, int* failed, long long n_rows, int d,
                                  int rows_per_sub, cudaStream_t st) {
  if (n_rows <= 0) return cudaSuccess;
  constexpr int kWarps = 8;
  const long long grid = (n_rows + kWarps - 1) / kWarps;
  synthetic_eval_kernel<<<static_cast<unsigned>(grid), 32 * kWarps, 0, st>>>(actions, costs, failed, n_rows, d,
                                                                              rows_per_sub);
  return cudaGetLastError();
}

cudaError_t launch_separable_bound(const double* lo, const double* hi, int n, int d, const double* crit, int ncrit,
                                   const int* use, double* lf, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  constexpr int kWarps = 8;
  separable_bound_kernel<<<(n + kWarps - 1) / kWarps, 32 * kWarps, 0, st>>>(lo, hi, n, d, crit, ncrit, use, lf);
  return cudaGetLastError();
}

}  // namespace bp

// pool.cu -- branching on the device: the subdomain pool's payload (boxes, incumbent
// actions, top-sample lists) lives in HBM, and the split of picked parents and the
// merge of each child's search report run as kernels.
//
//   split_kernel   split (bab.cpp:155-223): axis choice from the parent's top-k
//                  samples (count below the midpoint per axis, score w_j |2 n_lo - k|,
//                  lowest axis on ties, width fallback), bisection at the midpoint,
//                  stable routing of the parent's top list into the two children.
//                  One CTA per parent.  Children go to this rank's search inputs and
//                  staging, or into shipped records for another rank.
//   unpack_kernel  shipped child records -> search inputs / staging / slot.
//   merge_kernel   merge_report (bab.cpp:245-262): the routed list merged with the
//                  search's list (std::merge order: ties keep the routed samples first),
//                  truncated to the capacity; the incumbent replaced when the search
//                  found a strictly lower value.  One CTA per child.
//
// Everything here is comparisons, integer counts and copies of FP32/FP64 values, so
// the results are bit-identical to the host restatement (pick_out stays on the host:
// its softmax must use the same exp() as the reference to pick the same records).
// Traffic per parent is its top list read once and written once (K x (d+1) floats)
// plus the top-k x d axis-count reads; per child the two lists read and the merged
// one written: HBM-bound, microseconds per iteration at the bench sizes.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "bp_common.cuh"

namespace bp {

namespace {

constexpr int kPoolThreads = 256;
constexpr int kPoolWarps = kPoolThreads / 32;

struct AxisPick {
  double score;
  int axis;
};
__device__ __forceinline__ AxisPick better(AxisPick a, AxisPick b) {  // higher score, then lower axis
  if (b.axis < 0) return a;
  if (a.axis < 0) return b;
  if (b.score > a.score || (b.score == a.score && b.axis < a.axis)) return b;
  return a;
}
__device__ AxisPick block_best(AxisPick v, AxisPick* red) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    AxisPick o{__shfl_xor_sync(0xffffffffu, v.score, s), __shfl_xor_sync(0xffffffffu, v.axis, s)};
    v = better(v, o);
  }
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  AxisPick r{-1.0, -1};
  for (int i = 0; i < kPoolWarps; ++i) r = better(r, red[i]);
  return r;
}

// Exclusive prefix count of `flag` over the block and the block total.
__device__ int block_scan(bool flag, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, flag);
  __syncthreads();
  if (lane == 0) warp_tot[w] = __popc(m);
  __syncthreads();
  int before = 0, all = 0;
  for (int i = 0; i < kPoolWarps; ++i) {
    before += i < w ? warp_tot[i] : 0;
    all += warp_tot[i];
  }
  *total = all;
  return before + __popc(m & ((1u << lane) - 1u));
}

__device__ __forceinline__ void copy_row(float* dst, const float* src, int d, int lane) {
  for (int j = lane; j < d; j += 32) dst[j] = src[j];
}

// Destination of one child: this rank's staging at local index i, or a shipped record.
struct ChildOut {
  float* val;
  float* act;
  double* lo;   // slot or record box
  double* hi;
  double* lo_d;  // search inputs (local children)
  double* hi_d;
  float* lo_f;
  float* hi_f;
  float* warm;
  int* n;        // staging count (local); records store it as a double
  double* rec_n;
};

__device__ ChildOut child_out(const PoolArgs& P, const StageArgs& S, unsigned char* pack, const SplitTask& t, int b) {
  const int d = P.d, K = P.K;
  ChildOut o{};
  if (t.dst[b] >= 0) {
    const size_t i = static_cast<size_t>(t.dst[b]);
    o.val = S.val + i * K;
    o.act = S.act + i * K * d;
    o.lo = pool_lo(P, t.slot[b]);
    o.hi = pool_hi(P, t.slot[b]);
    o.lo_d = S.lo_d + i * d;
    o.hi_d = S.hi_d + i * d;
    o.lo_f = S.lo_f + i * d;
    o.hi_f = S.hi_f + i * d;
    o.warm = S.warm_f + i * d;
    o.n = S.n + i;
  } else {
    unsigned char* r = pack + static_cast<size_t>(t.pack[b]) * pool_record_bytes(d, K);
    double* h = reinterpret_cast<double*>(r);
    if (threadIdx.x == 0) h[0] = static_cast<double>(t.key[b]);
    o.rec_n = h + 1;
    o.lo = h + 2;
    o.hi = h + 2 + d;
    o.val = reinterpret_cast<float*>(h + 2 + 2 * d);
    o.act = o.val + K;
  }
  return o;
}

__global__ void __launch_bounds__(kPoolThreads) split_kernel(PoolArgs P, const SplitTask* __restrict__ tasks, StageArgs S,
                                                         unsigned char* pack, double min_width, int* axis_out) {
  extern __shared__ int route[];  // [K]: >= 0 position in the lo child, else ~position in the hi child
  __shared__ AxisPick red[kPoolWarps];
  __shared__ int warp_tot[kPoolWarps];
  const SplitTask t = tasks[blockIdx.x];
  const int d = P.d, K = P.K;
  const double* lo = pool_lo(P, t.parent);
  const double* hi = pool_hi(P, t.parent);
  const float* pval = pool_val(P, t.parent);
  const float* pact = pool_act(P, t.parent);
  const int n_top = *pool_n(P, t.parent);
  long long k = 0;
  if (n_top > 0 && t.k_round != -2)
    k = t.k_round == -1 ? n_top : (t.k_round < 1 ? 1 : t.k_round > n_top ? n_top : t.k_round);
  // axis (bab.cpp:166-195): per axis above the width floor, the sample score and the width
  AxisPick by_samples{-1.0, -1}, by_width{-1.0, -1};
  for (int j = threadIdx.x; j < d; j += kPoolThreads) {  // ascending j per thread: first max kept
    const double wj = hi[j] - lo[j];
    if (wj <= min_width) continue;
    if (k > 0) {
      const double mid = 0.5 * (lo[j] + hi[j]);
      int n_lo = 0;
      for (long long i = 0; i < k; ++i) n_lo += static_cast<double>(pact[i * d + j]) <= mid ? 1 : 0;
      const int diff = 2 * n_lo - static_cast<int>(k);
      by_samples = better(by_samples, AxisPick{wj * static_cast<double>(diff < 0 ? -diff : diff), j});
    }
    by_width = better(by_width, AxisPick{wj, j});
  }
  const AxisPick s = block_best(by_samples, red);
  const AxisPick w = block_best(by_width, red);
  int axis = k > 0 ? s.axis : w.axis;
  if (k > 0 && axis >= 0 && s.score == 0.0) axis = w.axis;
  if (threadIdx.x == 0) axis_out[blockIdx.x] = axis;
  if (axis < 0) return;  // uniform over the block; the host reports the error
  const double mid = 0.5 * (lo[axis] + hi[axis]);
  // stable routing: u[axis] <= mid -> lo child, in list order
  int base_lo = 0, base_hi = 0;
  for (int c0 = 0; c0 < n_top; c0 += kPoolThreads) {
    const int i = c0 + threadIdx.x;
    const bool in = i < n_top;
    const bool to_lo = in && static_cast<double>(pact[static_cast<size_t>(i) * d + axis]) <= mid;
    int tot_lo = 0;
    const int before_lo = block_scan(to_lo, warp_tot, &tot_lo);
    if (in) route[i] = to_lo ? base_lo + before_lo : ~(base_hi + (i - c0) - before_lo);
    base_lo += tot_lo;
    base_hi += min(kPoolThreads, n_top - c0) - tot_lo;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int b = 0; b < 2; ++b) {
    const ChildOut o = child_out(P, S, pack, t, b);
    const int nb = b == 0 ? base_lo : base_hi;
    for (int j = threadIdx.x; j < d; j += kPoolThreads) {
      double l = lo[j], h = hi[j];
      if (j == axis) (b == 0 ? h : l) = mid;
      o.lo[j] = l;
      o.hi[j] = h;
      if (o.lo_d) {
        o.lo_d[j] = l;
        o.hi_d[j] = h;
        o.lo_f[j] = static_cast<float>(l);
        o.hi_f[j] = static_cast<float>(h);
        if (nb == 0) o.warm[j] = __int_as_float(0x7fc00000);  // no warm start
      }
    }
    if (threadIdx.x == 0) {
      if (o.n) *o.n = nb;
      else *o.rec_n = static_cast<double>(nb);
    }
  }
  for (int i = wid; i < n_top; i += kPoolWarps) {  // one warp per routed row
    const int r = route[i];
    const int b = r >= 0 ? 0 : 1, p = r >= 0 ? r : ~r;
    const ChildOut o = child_out(P, S, pack, t, b);
    if (lane == 0) o.val[p] = pval[i];
    copy_row(o.act + static_cast<size_t>(p) * d, pact + static_cast<size_t>(i) * d, d, lane);
    if (p == 0 && o.warm) copy_row(o.warm, pact + static_cast<size_t>(i) * d, d, lane);  // best = routed front
  }
}

__global__ void __launch_bounds__(kPoolThreads) unpack_kernel(PoolArgs P, StageArgs S, const unsigned char* __restrict__ recv,
                                                          const int* __restrict__ dst, const int* __restrict__ slot) {
  const int d = P.d, K = P.K;
  const double* h = reinterpret_cast<const double*>(recv + static_cast<size_t>(blockIdx.x) * pool_record_bytes(d, K));
  const size_t i = static_cast<size_t>(dst[blockIdx.x]);
  double* plo = pool_lo(P, slot[blockIdx.x]);
  double* phi = pool_hi(P, slot[blockIdx.x]);
  const int nb = static_cast<int>(h[1]);
  const float* val = reinterpret_cast<const float*>(h + 2 + 2 * d);
  const float* act = val + K;
  for (int j = threadIdx.x; j < d; j += kPoolThreads) {
    const double l = h[2 + j], u = h[2 + d + j];
    plo[j] = l;
    phi[j] = u;
    S.lo_d[i * d + j] = l;
    S.hi_d[i * d + j] = u;
    S.lo_f[i * d + j] = static_cast<float>(l);
    S.hi_f[i * d + j] = static_cast<float>(u);
    S.warm_f[i * d + j] = nb > 0 ? act[j] : __int_as_float(0x7fc00000);
  }
  if (threadIdx.x == 0) S.n[i] = nb;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int r = wid; r < nb; r += kPoolWarps) {
    if (lane == 0) S.val[i * K + r] = val[r];
    copy_row(S.act + (i * K + r) * d, act + static_cast<size_t>(r) * d, d, lane);
  }
}

// count of v[0, n) < x (strict) / <= x, v ascending
__device__ __forceinline__ int count_less(const float* v, int n, float x, bool or_equal) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (or_equal ? v[m] <= x : v[m] < x) lo = m + 1;
    else hi = m;
  }
  return lo;
}

__global__ void __launch_bounds__(kPoolThreads) merge_kernel(PoolArgs P, StageArgs S, const int* __restrict__ slots,
                                                         const float* __restrict__ s_val, const float* __restrict__ s_act,
                                                         const int* __restrict__ s_cnt, const float* __restrict__ s_uf,
                                                         const float* __restrict__ s_best, const int* __restrict__ failed,
                                                         int capacity, float* out_uf, double* out_maxw) {
  extern __shared__ float sm[];  // A (routed) values [K], B (search) values [K], source of each output [K]
  const int d = P.d, K = P.K;
  float* av = sm;
  float* bv = sm + K;
  int* src = reinterpret_cast<int*>(sm + 2 * K);
  __shared__ double wred[kPoolWarps];
  const size_t i = blockIdx.x;
  const int s = slots[i];
  const int na = S.n[i];
  const bool ok = failed[i] == 0;
  const int nb = ok ? s_cnt[i] : 0;
  const float* aact = S.act + i * K * d;
  const float* bact = s_act + i * K * d;
  for (int q = threadIdx.x; q < na; q += kPoolThreads) av[q] = S.val[i * K + q];
  for (int q = threadIdx.x; q < nb; q += kPoolThreads) bv[q] = s_val[i * K + q];
  __syncthreads();
  // merge_report (bab.cpp:248-261): an empty list takes the other whole; otherwise the
  // first `capacity` of the stable merge
  const int keep = na == 0 ? nb : nb == 0 ? na : min(na + nb, capacity);
  for (int q = threadIdx.x; q < na; q += kPoolThreads) {
    const int p = q + count_less(bv, nb, av[q], false);
    if (p < keep) src[p] = q;
  }
  for (int q = threadIdx.x; q < nb; q += kPoolThreads) {
    const int p = q + count_less(av, na, bv[q], true);
    if (p < keep) src[p] = K + q;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* oval = pool_val(P, s);
  float* oact = pool_act(P, s);
  for (int p = wid; p < keep; p += kPoolWarps) {
    const int q = src[p];
    const bool from_a = q < K;
    if (lane == 0) oval[p] = from_a ? av[q] : bv[q - K];
    copy_row(oact + static_cast<size_t>(p) * d, from_a ? aact + static_cast<size_t>(q) * d
                                                       : bact + static_cast<size_t>(q - K) * d, d, lane);
  }
  // incumbent: the routed front, replaced by the search's best when strictly lower
  const float a_uf = na > 0 ? av[0] : __int_as_float(0x7f800000);
  const float r_uf = ok ? s_uf[i] : __int_as_float(0x7f800000);
  const bool take = r_uf < a_uf;
  const float* bsrc = take ? s_best + i * d : aact;
  const bool has = take || na > 0;
  float* pbest = pool_best(P, s);
  const double* plo = pool_lo(P, s);
  const double* phi = pool_hi(P, s);
  for (int j = threadIdx.x; j < d && has; j += kPoolThreads) pbest[j] = bsrc[j];
  double w = 0.0;
  for (int j = threadIdx.x; j < d; j += kPoolThreads) w = fmax(w, phi[j] - plo[j]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) w = fmax(w, __shfl_xor_sync(0xffffffffu, w, o));
  if (lane == 0) wred[wid] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int q = 0; q < kPoolWarps; ++q) m = fmax(m, wred[q]);
    out_maxw[i] = m;
    out_uf[i] = take ? r_uf : a_uf;
    *pool_n(P, s) = keep;
    *pool_has(P, s) = has ? 1 : 0;
  }
}

}  // namespace

cudaError_t launch_pool_split(const PoolArgs& P, const SplitTask* tasks, int n_tasks, const StageArgs& S,
                              unsigned char* pack, double min_width, int* axis_out, cudaStream_t st) {
  if (n_tasks <= 0) return cudaSuccess;
  const size_t smem = sizeof(int) * static_cast<size_t>(P.K);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  split_kernel<<<n_tasks, kPoolThreads, smem, st>>>(P, tasks, S, pack, min_width, axis_out);
  return cudaGetLastError();
}

cudaError_t launch_pool_unpack(const PoolArgs& P, const StageArgs& S, const unsigned char* recv, const int* dst,
                               const int* slot, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  unpack_kernel<<<n, kPoolThreads, 0, st>>>(P, S, recv, dst, slot);
  return cudaGetLastError();
}

cudaError_t launch_pool_merge(const PoolArgs& P, const StageArgs& S, const int* slots, int n, const float* s_val,
                              const float* s_act, const int* s_cnt, const float* s_uf, const float* s_best,
                              const int* failed, int capacity, float* out_uf, double* out_maxw, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = sizeof(float) * 3 * static_cast<size_t>(P.K);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  merge_kernel<<<n, kPoolThreads, smem, st>>>(P, S, slots, s_val, s_act, s_cnt, s_uf, s_best, failed, capacity, out_uf,
                                          out_maxw);
  return cudaGetLastError();
}

}  // namespace bp

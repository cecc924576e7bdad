// gradient.cu -- reverse-mode gradient of the unrolled objective with respect to the
// action sequence, for the GD searcher.
//
// Restates gradient (reference proj/src/graph.cpp:403-564) on the build_objective
// graph: exact adjoints, ReLU subgradient 0 at the kink (x > 0 ? 1 : 0), squared
// distance 2 w (x - t), penalty hinge -penalty (x - c) / |x - c| inside the radius
// (0 at the centre and outside), Linear W^T, Slice / Sum / ScalarAffine routing.
// FP64 like the reference.  One warp per row: the forward pass checkpoints x_t per
// step (global scratch); the backward pass recomputes each step's layer inputs from
// its checkpoint, runs the step's cost program forward and in reverse, then the MLP
// transposed (lanes over the input coordinates, coalesced W rows), so memory stays
// O(H * ks) per row.  The synthetic objective's gradient is elementwise
// (objective.cpp:100-107).
#include <cuda_runtime.h>

#include <cstdint>

#include "bp_common.cuh"

namespace bp {

namespace {

constexpr int kGradWarps = 4;

// Per-warp shared-memory plan (doubles): activations of every layer of one step
// (widths[0] .. widths[L]), the op values of the cost program, two adjoint buffers
// of the widest layer, the step's u / p / adjoints.
__host__ __device__ inline int grad_warp_doubles(const DevObjective& o) {
  int acts = 0, maxw = 0;
  for (int l = 0; l <= o.L; ++l) {
    acts += o.widths[l];
    maxw = maxw > o.widths[l] ? maxw : o.widths[l];
  }
  return acts + 2 * o.S + 2 * maxw + 64 + o.ks;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  return v;
}

// out[j] = b[j] + sum_k W[j][k] in[k] (W row-major [N][K], FP64), relu if asked.
__device__ void warp_affine(const double* W, const double* b, int N, int K, const double* in, double* out) {
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < N; ++j) {
    double acc = 0.0;
    for (int k = lane; k < K; k += 32) acc += W[static_cast<size_t>(j) * K + k] * in[k];
    acc = warp_sum_d(acc);
    if (lane == 0) out[j] = acc + b[j];
  }
  __syncwarp();
}

// Value pointers of the cost program's sources (0 x_t, 1 u_t, 2 p_t, 3+i op i).
__device__ __forceinline__ double* val_of(const DevObjective& o, double* x, double* u, double* p, double* ov, int id) {
  if (id == 0) return x;
  if (id == 1) return u;
  if (id == 2) return p;
  return ov + o.ops[id - 3].col;
}

__global__ void __launch_bounds__(32 * kGradWarps) gradient_kernel(const DevObjective o, const float* __restrict__ act,
                                                                   float* __restrict__ grad, double* ckpt,
                                                                   long long n_rows) {
  extern __shared__ __align__(16) double gsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long row = static_cast<long long>(blockIdx.x) * kGradWarps + wid;
  if (row >= n_rows) return;
  const int ks = o.ks, ka = o.ka, kd = o.kd, H = o.H, L = o.L, S = o.S;
  double* base = gsm + static_cast<size_t>(wid) * grad_warp_doubles(o);
  double* a[kMaxLayers + 1];  // a[0] features, a[l+1] output of layer l (pre-activation for hidden layers)
  {
    double* q = base;
    for (int l = 0; l <= L; ++l) {
      a[l] = q;
      q += o.widths[l];
    }
  }
  double* ov = a[L] + o.widths[L];  // op values [S]
  double* gv = ov + S;              // op adjoints [S]
  int maxw = 0;
  for (int l = 0; l <= L; ++l) maxw = max(maxw, o.widths[l]);
  double* lam = gv + S;   // [maxw]
  double* lam2 = lam + maxw;
  double* small = lam2 + maxw;  // x_prev adj [16], u[16], p[16], gu[16]... within 64
  double* u = small;       // u_t
  double* p = small + 16;  // p_t
  double* lp = small + 32; // adjoint of p_t
  double* gu = small + 48; // adjoint of u_t
  double* xadj = small + 64;  // [ks] adjoint of x_t (from step t+1, then the step's cost program)
  const float* ur = act + row * o.d;
  double* ck = ckpt + row * static_cast<long long>(H) * ks;
  const double* x0 = o.dd + o.x0d;
  const double* p0 = o.dd + o.p0d;

  // ---- forward with checkpoints of x_t
  auto features = [&](const double* xprev, const double* pprev, int t) {
    for (int j = lane; j < ks; j += 32) a[0][j] = o.rel ? xprev[j] - pprev[j % kd] : xprev[j];
    for (int j = lane; j < ka; j += 32) a[0][ks + j] = static_cast<double>(ur[t * ka + j]);
    __syncwarp();
  };
  auto mlp = [&]() {  // a[l+1] = W_l relu(a[l]) + b_l with relu on hidden inputs
    for (int l = 0; l < L; ++l) {
      const int K = o.widths[l], N = o.widths[l + 1];
      double* in = a[l];
      if (l > 0 && o.relu[l - 1]) {  // apply relu in a scratch copy so a[l] keeps the pre-activation
        for (int k = lane; k < K; k += 32) lam2[k] = fmax(in[k], 0.0);
        __syncwarp();
        in = lam2;
      }
      warp_affine(o.dd + o.wd[l], o.dd + o.bd[l], N, K, in, a[l + 1]);
    }
  };
  for (int j = lane; j < kd; j += 32) p[j] = p0[j];
  __syncwarp();
  for (int t = 0; t < H; ++t) {
    const double* xprev = t == 0 ? x0 : ck + static_cast<long long>(t - 1) * ks;
    features(xprev, p, t);
    mlp();
    for (int j = lane; j < ks; j += 32) ck[static_cast<long long>(t) * ks + j] = a[L][j];
    for (int j = lane; j < kd; j += 32) p[j] += j < ka ? static_cast<double>(ur[t * ka + j]) : 0.0;
    __syncwarp();
  }

  // ---- backward
  double* lx = xadj;
  for (int j = lane; j < ks; j += 32) xadj[j] = 0.0;
  for (int j = lane; j < 16; j += 32) lp[j] = 0.0;
  __syncwarp();
  for (int t = H - 1; t >= 0; --t) {
    // p_{t-1} = p0 + sum_{tau < t} u_tau, in the forward pass's order
    for (int j = lane; j < kd; j += 32) {
      double v = p0[j];
      for (int tau = 0; tau < t; ++tau) v += j < ka ? static_cast<double>(ur[tau * ka + j]) : 0.0;
      p[j] = v;
    }
    __syncwarp();
    const double* xprev = t == 0 ? x0 : ck + static_cast<long long>(t - 1) * ks;
    features(xprev, p, t);
    mlp();
    // u_t, p_t, x_t = a[L]; cost program forward (lane 0: small ops)
    for (int j = lane; j < ka; j += 32) u[j] = static_cast<double>(ur[t * ka + j]);
    for (int j = lane; j < kd; j += 32) p[j] += j < ka ? u[j] : 0.0;
    for (int j = lane; j < S; j += 32) gv[j] = 0.0;
    for (int j = lane; j < 16; j += 32) gu[j] = 0.0;
    __syncwarp();
    double* x = a[L];
    if (lane == 0) {
      for (int i = 0; i < o.n_ops; ++i) {
        const DevOp& op = o.ops[i];
        const double* s0 = val_of(o, x, u, p, ov, op.src0);
        double* out = ov + op.col;
        switch (op.kind) {
          case 0: {
            const double* W = o.dd + op.wd;
            for (int r = 0; r < op.dim; ++r) {
              double acc = 0.0;
              for (int k = 0; k < op.in_dim; ++k) acc += W[r * op.in_dim + k] * s0[k];
              out[r] = acc + o.dd[op.bd + r];
            }
            break;
          }
          case 1:
            for (int k = 0; k < op.dim; ++k) out[k] = fmax(s0[k], 0.0);
            break;
          case 2: {
            const double* s1 = op.src1 >= 0 ? val_of(o, x, u, p, ov, op.src1) : nullptr;
            for (int k = 0; k < op.dim; ++k) out[k] = s1 ? s0[k] + s1[k] : s0[k];
            break;
          }
          case 3:
            for (int k = 0; k < op.dim; ++k) out[k] = op.scaled * s0[k] + op.offsetd;
            break;
          case 4: {
            const double* tg = o.dd + op.tgtd;
            const double* wt = o.dd + op.wtd + (op.weight_by_step ? t * op.in_dim : 0);
            double acc = 0.0;
            for (int k = 0; k < op.in_dim; ++k) {
              const double dd = s0[k] - tg[k];
              acc += wt[k] * dd * dd;
            }
            out[0] = acc;
            break;
          }
          case 5: {
            const double* c = o.dd + op.ctrd;
            double d2 = 0.0;
            for (int k = 0; k < op.in_dim; ++k) d2 += (s0[k] - c[k]) * (s0[k] - c[k]);
            const double m = op.radiusd - sqrt(d2);
            out[0] = m > 0.0 ? op.penaltyd * m : 0.0;
            break;
          }
          default:
            for (int k = 0; k < op.dim; ++k) out[k] = s0[op.begin + k];
            break;
        }
      }
      // reverse: every term has adjoint 1
      for (int i = 0; i < o.n_ops; ++i)
        if (o.ops[i].is_term) gv[o.ops[i].col] += 1.0;
    }
    __syncwarp();
    // adjoint of x_t: the next step's (in xadj) plus the cost program's
    if (lane == 0) {
      for (int i = o.n_ops - 1; i >= 0; --i) {
        const DevOp& op = o.ops[i];
        const double* g = gv + op.col;
        const double* s0 = val_of(o, x, u, p, ov, op.src0);
        // adjoint target of src0 (x: lx, u: gu, p: lp, op: gv)
        double* d0 = op.src0 == 0 ? lx : op.src0 == 1 ? gu : op.src0 == 2 ? lp : gv + o.ops[op.src0 - 3].col;
        switch (op.kind) {
          case 0: {
            const double* W = o.dd + op.wd;
            for (int k = 0; k < op.in_dim; ++k) {
              double acc = 0.0;
              for (int r = 0; r < op.dim; ++r) acc += g[r] * W[r * op.in_dim + k];
              d0[k] += acc;
            }
            break;
          }
          case 1:
            for (int k = 0; k < op.dim; ++k) d0[k] += s0[k] > 0.0 ? g[k] : 0.0;
            break;
          case 2: {
            double* d1 = op.src1 < 0 ? nullptr
                         : op.src1 == 0 ? lx : op.src1 == 1 ? gu : op.src1 == 2 ? lp : gv + o.ops[op.src1 - 3].col;
            for (int k = 0; k < op.dim; ++k) {
              d0[k] += g[k];
              if (d1) d1[k] += g[k];
            }
            break;
          }
          case 3:
            for (int k = 0; k < op.dim; ++k) d0[k] += op.scaled * g[k];
            break;
          case 4: {
            if (g[0] == 0.0) break;
            const double* tg = o.dd + op.tgtd;
            const double* wt = o.dd + op.wtd + (op.weight_by_step ? t * op.in_dim : 0);
            for (int k = 0; k < op.in_dim; ++k) d0[k] += g[0] * 2.0 * wt[k] * (s0[k] - tg[k]);
            break;
          }
          case 5: {
            if (g[0] == 0.0) break;
            const double* c = o.dd + op.ctrd;
            double d2 = 0.0;
            for (int k = 0; k < op.in_dim; ++k) d2 += (s0[k] - c[k]) * (s0[k] - c[k]);
            const double dn = sqrt(d2);
            if (dn <= 0.0 || op.radiusd - dn <= 0.0) break;
            for (int k = 0; k < op.in_dim; ++k) d0[k] -= (g[0] * op.penaltyd / dn) * (s0[k] - c[k]);
            break;
          }
          default:
            for (int k = 0; k < op.dim; ++k) d0[op.begin + k] += g[k];
            break;
        }
      }
    }
    __syncwarp();
    for (int j = lane; j < ks; j += 32) lam[j] = xadj[j];
    __syncwarp();
    // MLP transposed: lam (on a[L]) -> features
    for (int l = L - 1; l >= 0; --l) {
      const int K = o.widths[l], N = o.widths[l + 1];
      const double* W = o.dd + o.wd[l];
      for (int k = lane; k < K; k += 32) {
        double acc = 0.0;
        for (int j = 0; j < N; ++j) acc += lam[j] * W[static_cast<size_t>(j) * K + k];
        if (l > 0 && o.relu[l - 1]) acc = a[l][k] > 0.0 ? acc : 0.0;  // subgradient 0 at the kink
        lam2[k] = acc;
      }
      __syncwarp();
      for (int k = lane; k < K; k += 32) lam[k] = lam2[k];
      __syncwarp();
    }
    // features -> x_{t-1}, p_{t-1}, u_t; p_t = p_{t-1} + u_t
    for (int j = lane; j < ka; j += 32) {
      const double g = gu[j] + lam[ks + j] + (j < kd ? lp[j] : 0.0);
      grad[row * o.d + t * ka + j] = static_cast<float>(g);
    }
    __syncwarp();
    for (int j = lane; j < kd; j += 32) {
      double v = lp[j];
      if (o.rel)
        for (int k = 0; k < ks / kd; ++k) v -= lam[k * kd + j];
      lp[j] = v;
    }
    for (int j = lane; j < ks; j += 32) xadj[j] = lam[j];  // adjoint of x_{t-1}
    __syncwarp();
  }
}

__global__ void synthetic_gradient_kernel(const float* __restrict__ act, float* __restrict__ grad, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double x = static_cast<double>(act[i]);
    grad[i] = static_cast<float>(10.0 * x - 50.0 * sin(50.0 * x));
  }
}

}  // namespace

size_t gradient_smem_bytes(const DevObjective& o) {
  return sizeof(double) * static_cast<size_t>(grad_warp_doubles(o)) * kGradWarps;
}
int gradient_rows_per_cta() { return kGradWarps; }

// grad[r][:] = d objective / d actions[r][:]; ckpt: n_rows * H * ks doubles of scratch.
cudaError_t launch_gradient(const DevObjective& o, const float* actions, float* grad, double* ckpt, long long n_rows,
                            cudaStream_t st) {
  if (n_rows <= 0) return cudaSuccess;
  const size_t smem = gradient_smem_bytes(o);
  cudaError_t e = cudaFuncSetAttribute(gradient_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const long long grid = (n_rows + kGradWarps - 1) / kGradWarps;
  gradient_kernel<<<static_cast<unsigned>(grid), 32 * kGradWarps, smem, st>>>(o, actions, grad, ckpt, n_rows);
  return cudaGetLastError();
}

cudaError_t launch_synthetic_gradient(const float* actions, float* grad, long long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long long grid = (n + 255) / 256;
  synthetic_gradient_kernel<<<static_cast<unsigned>(grid < 4096 ? grid : 4096), 256, 0, st>>>(actions, grad, n);
  return cudaGetLastError();
}

}  // namespace bp

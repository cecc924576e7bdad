// bound.cu -- K7: batched early-stop CROWN lower bound per subdomain, with
// the K6 interval forward pass as the fallback source of intermediate bounds.
//
// Restates, per subdomain and for the unrolled rollout graph:
//   lower_bound (reference proj/src/crown.cpp:440-469) in the early-stop modes,
//   backward_propagate (crown.cpp:92-292) -- lower form only, the only one
//   lower_bound reads (crown.cpp:466-468) --, relax_relu (crown.cpp:10-39),
//   quad_envelope (crown.cpp:72-88), concretize_lower (crown.cpp:296-319),
//   interval_forward (graph.cpp:566-684) for the fallback / interval mode.
//
// The unrolled graph is a chain over steps, so the reference's countdown /
// LIFO traversal reduces to one backward sweep t = H..1: cost program in
// reverse op order, stop anchors, the MLP layers L..1 with the ReLU
// relaxation in between, then the feature split into (x_{t-1}, p_{t-1}, u_t).
// The bound work is ~1/5000 of the rollout, so it runs in FP64 (one CTA per
// subdomain): with the same sample extrema it matches the FP64 reference to
// rounding, instead of adding FP32 cancellation error to lf.
#include <cuda_runtime.h>

#include <cstdint>

#include "bp_common.cuh"

namespace bp {

// BoundArgs: bp_common.cuh

namespace {

constexpr int kMaxW = 1024;  // widest supported layer / scratch row (the kernel is instantiated at 128 .. 1024)

template <int MW>
struct Smem {
  double a_lo[MW], a_hi[MW];   // interval pass: current layer in/out
  double b_lo[MW], b_hi[MW];
  double x_lo[MW], x_hi[MW];   // interval x_t (ks)
  double p_lo[16], p_hi[16];
  double o_lo[MW], o_hi[MW];   // interval op values (by op col)
  double lam[MW], lam2[MW];    // backward coefficients
  double lx[MW];                  // coefficient on x_t
  double lops[MW];                // coefficients on op values (by op col)
  double lu[16], lp[16], lpt[16];
  double red[kThreads / 32];
};

__device__ __forceinline__ double relu_lower_slope(double l, double u, int alpha) {
  if (l >= 0.0) return 1.0;
  if (u <= 0.0) return 0.0;
  return alpha == 1 ? 0.0 : alpha == 2 ? 1.0 : (u >= -l ? 1.0 : 0.0);
}

struct Bounds {
  const DevObjective& o;
  const BoundArgs& a;
  long long base;  // s * H * SP
  bool emp;
  __device__ double lo(int t, int off) const {
    const long long i = base + static_cast<long long>(t) * o.SP + off;
    return emp ? static_cast<double>(dec_f(a.stat_min[i])) : a.ivl_lo[i];
  }
  __device__ double hi(int t, int off) const {
    const long long i = base + static_cast<long long>(t) * o.SP + off;
    return emp ? static_cast<double>(dec_f(a.stat_max[i])) : a.ivl_hi[i];
  }
};

// y = W x + b interval over [in_lo, in_hi] (graph.cpp:587-605, sequential in j).
__device__ void interval_linear(const double* W, const double* b, int N, int K, const double* in_lo,
                                const double* in_hi, double* out_lo, double* out_hi) {
  for (int r = threadIdx.x; r < N; r += kThreads) {
    double l = b[r], h = b[r];
    const double* w = W + static_cast<size_t>(r) * K;
    for (int j = 0; j < K; ++j) {
      const double wj = w[j];
      if (wj >= 0.0) {
        l += wj * in_lo[j];
        h += wj * in_hi[j];
      } else {
        l += wj * in_hi[j];
        h += wj * in_lo[j];
      }
    }
    out_lo[r] = l;
    out_hi[r] = h;
  }
}

template <int MW>
__device__ __forceinline__ const double* ival_lo(const DevObjective& o, Smem<MW>& sm, int id, int t, const BoundArgs& a,
                                                 long long boxoff) {
  if (id == 0) return sm.x_lo;
  if (id == 1) return a.lo + boxoff + t * o.ka;
  if (id == 2) return sm.p_lo;
  return sm.o_lo + o.ops[id - 3].col;
}
template <int MW>
__device__ __forceinline__ const double* ival_hi(const DevObjective& o, Smem<MW>& sm, int id, int t, const BoundArgs& a,
                                                 long long boxoff) {
  if (id == 0) return sm.x_hi;
  if (id == 1) return a.hi + boxoff + t * o.ka;
  if (id == 2) return sm.p_hi;
  return sm.o_hi + o.ops[id - 3].col;
}

// K6: interval_forward over the unrolled graph; records every watched slot.
template <int MW>
__device__ void interval_pass(const DevObjective& o, const BoundArgs& a, Smem<MW>& sm, int s) {
  const int tid = threadIdx.x;
  const long long boxoff = static_cast<long long>(s) * o.d;
  const long long base = static_cast<long long>(s) * o.H * o.SP;
  for (int j = tid; j < o.ks; j += kThreads) sm.x_lo[j] = sm.x_hi[j] = o.dd[o.x0d + j];
  for (int j = tid; j < o.kd; j += kThreads) sm.p_lo[j] = sm.p_hi[j] = o.dd[o.p0d + j];
  __syncthreads();
  for (int t = 0; t < o.H; ++t) {
    const double* ulo = a.lo + boxoff + t * o.ka;
    const double* uhi = a.hi + boxoff + t * o.ka;
    // features: concat(x - tile(p), u_t), concat(x, u_t), or u_t alone (bare network)
    const int uoff = o.net ? 0 : o.ks;
    for (int j = tid; j < o.ks && !o.net; j += kThreads) {
      sm.a_lo[j] = o.rel ? sm.x_lo[j] - sm.p_hi[j % o.kd] : sm.x_lo[j];
      sm.a_hi[j] = o.rel ? sm.x_hi[j] - sm.p_lo[j % o.kd] : sm.x_hi[j];
    }
    for (int j = tid; j < o.ka; j += kThreads) {
      sm.a_lo[uoff + j] = ulo[j];
      sm.a_hi[uoff + j] = uhi[j];
    }
    __syncthreads();
    double *in_lo = sm.a_lo, *in_hi = sm.a_hi, *out_lo = sm.b_lo, *out_hi = sm.b_hi;
    for (int l = 0; l < o.L; ++l) {
      const int K = o.widths[l], N = o.widths[l + 1];
      interval_linear(o.dd + o.wd[l], o.dd + o.bd[l], N, K, in_lo, in_hi, out_lo, out_hi);
      __syncthreads();
      if (o.relu[l]) {
        for (int j = tid; j < N; j += kThreads) {
          if (o.pre_stat[l] >= 0) {
            a.ivl_lo[base + t * o.SP + o.pre_stat[l] + j] = out_lo[j];
            a.ivl_hi[base + t * o.SP + o.pre_stat[l] + j] = out_hi[j];
          }
          out_lo[j] = fmax(out_lo[j], 0.0);
          out_hi[j] = fmax(out_hi[j], 0.0);
        }
        __syncthreads();
      }
      double* tl = in_lo; in_lo = out_lo; out_lo = tl;
      double* th = in_hi; in_hi = out_hi; out_hi = th;
    }
    for (int j = tid; j < o.ks; j += kThreads) {
      sm.x_lo[j] = in_lo[j];
      sm.x_hi[j] = in_hi[j];
      if (o.x_stat >= 0) {
        a.ivl_lo[base + t * o.SP + o.x_stat + j] = in_lo[j];
        a.ivl_hi[base + t * o.SP + o.x_stat + j] = in_hi[j];
      }
    }
    for (int j = tid; j < o.kd; j += kThreads) {  // p_t = p_{t-1} + u_t
      sm.p_lo[j] = sm.p_lo[j] + ulo[j];
      sm.p_hi[j] = sm.p_hi[j] + uhi[j];
      if (o.p_stat >= 0) {
        a.ivl_lo[base + t * o.SP + o.p_stat + j] = sm.p_lo[j];
        a.ivl_hi[base + t * o.SP + o.p_stat + j] = sm.p_hi[j];
      }
    }
    if (o.u_stat >= 0)
      for (int j = tid; j < o.ka; j += kThreads) {
        a.ivl_lo[base + t * o.SP + o.u_stat + j] = ulo[j];
        a.ivl_hi[base + t * o.SP + o.u_stat + j] = uhi[j];
      }
    __syncthreads();
    // cost program intervals (graph.cpp:587-663)
    for (int i = 0; i < o.n_ops; ++i) {
      const DevOp& op = o.ops[i];
      const double* sl = ival_lo(o, sm, op.src0, t, a, boxoff);
      const double* sh = ival_hi(o, sm, op.src0, t, a, boxoff);
      double* dl = sm.o_lo + op.col;
      double* dh = sm.o_hi + op.col;
      switch (op.kind) {
        case 0:
          interval_linear(o.dd + op.wd, o.dd + op.bd, op.dim, op.in_dim, sl, sh, dl, dh);
          break;
        case 1:
          for (int j = tid; j < op.dim; j += kThreads) {
            dl[j] = fmax(sl[j], 0.0);
            dh[j] = fmax(sh[j], 0.0);
          }
          break;
        case 2: {
          const double* s1l = op.src1 >= 0 ? ival_lo(o, sm, op.src1, t, a, boxoff) : nullptr;
          const double* s1h = op.src1 >= 0 ? ival_hi(o, sm, op.src1, t, a, boxoff) : nullptr;
          for (int j = tid; j < op.dim; j += kThreads) {
            dl[j] = s1l ? (0.0 + sl[j]) + s1l[j] : 0.0 + sl[j];
            dh[j] = s1h ? (0.0 + sh[j]) + s1h[j] : 0.0 + sh[j];
          }
          break;
        }
        case 3:
          for (int j = tid; j < op.dim; j += kThreads) {
            if (op.scaled >= 0.0) {
              dl[j] = op.scaled * sl[j] + op.offsetd;
              dh[j] = op.scaled * sh[j] + op.offsetd;
            } else {
              dl[j] = op.scaled * sh[j] + op.offsetd;
              dh[j] = op.scaled * sl[j] + op.offsetd;
            }
          }
          break;
        case 4:
          if (tid == 0) {
            const double* tg = o.dd + op.tgtd;
            const double* wt = o.dd + op.wtd + (op.weight_by_step ? t * op.in_dim : 0);
            double l = 0.0, h = 0.0;
            for (int j = 0; j < op.in_dim; ++j) {
              const double x = sl[j] - tg[j], y = sh[j] - tg[j];
              const double mx = fmax(x * x, y * y);
              const double mn = (x <= 0.0 && y >= 0.0) ? 0.0 : fmin(x * x, y * y);
              l += wt[j] * mn;
              h += wt[j] * mx;
            }
            dl[0] = l;
            dh[0] = h;
          }
          break;
        case 5:
          if (tid == 0) {
            const double* c = o.dd + op.ctrd;
            double d2l = 0.0, d2h = 0.0;
            for (int j = 0; j < op.in_dim; ++j) {
              const double x = sl[j] - c[j], y = sh[j] - c[j];
              d2h += fmax(x * x, y * y);
              d2l += (x <= 0.0 && y >= 0.0) ? 0.0 : fmin(x * x, y * y);
            }
            const double ml = op.radiusd - sqrt(d2h), mh = op.radiusd - sqrt(d2l);
            dl[0] = ml > 0.0 ? op.penaltyd * ml : 0.0;
            dh[0] = mh > 0.0 ? op.penaltyd * mh : 0.0;
          }
          break;
        case 6:
          for (int j = tid; j < op.dim; j += kThreads) {
            dl[j] = sl[op.begin + j];
            dh[j] = sh[op.begin + j];
          }
          break;
      }
      __syncthreads();
      if (op.stat >= 0)
        for (int j = tid; j < op.dim; j += kThreads) {
          a.ivl_lo[base + t * o.SP + op.stat + j] = dl[j];
          a.ivl_hi[base + t * o.SP + op.stat + j] = dh[j];
        }
    }
    __syncthreads();
  }
}

template <int MW>
__device__ __forceinline__ double* lam_of(const DevObjective& o, Smem<MW>& sm, int id) {
  if (id == 0) return sm.lx;
  if (id == 1) return sm.lu;
  if (id == 2) return sm.lpt;
  return sm.lops + o.ops[id - 3].col;
}

// Stat offset of a value id (for its bounds), -1 when not recorded.
__device__ __forceinline__ int stat_of(const DevObjective& o, int id) {
  if (id == 0) return o.x_stat;
  if (id == 1) return o.u_stat;
  if (id == 2) return o.p_stat;
  return o.ops[id - 3].stat;
}

// One backward sweep (backward_propagate's lower form, crown.cpp:92-292) of a scalar:
// the objective's output (start_kind < 0) or `sign` times row `row` of a start node.
// Returns the concretised lower bound (crown.cpp:296-319) on every thread.
template <int MW>
__device__ double sweep(const DevObjective& o, const BoundArgs& a, Smem<MW>& sm, const Bounds& B, int s, int row,
                        double sign) {
  const int tid = threadIdx.x;
  const long long boxoff = static_cast<long long>(s) * o.d;
  const bool node = a.start_kind >= 0;
  const bool stops = a.mode != 0;  // full CROWN: no stop set (crown.cpp:463-464)
  const int t_top = node ? a.start_t : o.H - 1;
  double bacc = 0.0;  // this thread's share of the offset
  for (int j = tid; j < MW; j += kThreads) sm.lx[j] = 0.0;
  for (int j = tid; j < 16; j += kThreads) sm.lp[j] = 0.0;
  __syncthreads();

  for (int t = t_top; t >= 0; --t) {
    const bool last = t == o.H - 1;
    const bool top = t == t_top;
    // 1. cost program, reverse op order; terms enter with coefficient 1 (output pass),
    //    or the start row of a cost-op node with coefficient `sign`.
    for (int j = tid; j < MW; j += kThreads) sm.lops[j] = 0.0;
    for (int j = tid; j < 16; j += kThreads) {
      sm.lu[j] = 0.0;
      sm.lpt[j] = j < o.kd ? sm.lp[j] : 0.0;  // from step t+1's relative features
    }
    __syncthreads();
    if (tid == 0) {
      if (!node) {
        for (int i = 0; i < o.n_ops; ++i)
          if (o.ops[i].is_term) sm.lops[o.ops[i].col] += 1.0;
      } else if (top) {
        if (a.start_kind == 4) sm.lops[o.ops[a.start_index].col + row] = sign;
        if (a.start_kind == 1) sm.lx[row] = sign;
        if (a.start_kind == 2) sm.lu[row] = sign;
        if (a.start_kind == 3) sm.lpt[row] = sign;
      }
    }
    __syncthreads();
    const bool ops_live = !node || (top && a.start_kind == 4);  // earlier steps' ops feed nothing upstream
    for (int i = o.n_ops - 1; i >= 0 && ops_live; --i) {
      const DevOp& op = o.ops[i];
      if (node && top && i > a.start_index) continue;  // only the start op's ancestors
      const double* lam = sm.lops + op.col;
      double* ls = lam_of(o, sm, op.src0);
      const int st = stat_of(o, op.src0);
      switch (op.kind) {
        case 0: {  // LINEAR: lam_src += lam W ; offset += lam . b
          const double* W = o.dd + op.wd;
          for (int j = tid; j < op.in_dim; j += kThreads) {
            double acc = 0.0;
            for (int r = 0; r < op.dim; ++r) acc += lam[r] * W[r * op.in_dim + j];
            ls[j] += acc;
          }
          for (int r = tid; r < op.dim; r += kThreads) bacc += lam[r] * o.dd[op.bd + r];
          break;
        }
        case 1:  // RELU: anchor (last-ReLU stop) or sign-selected relaxation
          for (int j = tid; j < op.dim; j += kThreads) {
            const double c = lam[j], l = B.lo(t, st + j), u = B.hi(t, st + j);
            if (stops && op.stop && last) {
              bacc += c * (c >= 0.0 ? fmax(l, 0.0) : fmax(u, 0.0));
            } else if (c >= 0.0) {
              ls[j] += c * relu_lower_slope(l, u, a.alpha);
            } else if (l >= 0.0) {
              ls[j] += c;
            } else if (u > 0.0) {
              ls[j] += c * (u / (u - l));
              bacc += c * (-u * l / (u - l));
            }
          }
          break;
        case 2:
          for (int j = tid; j < op.dim; j += kThreads) {
            ls[j] += lam[j];
            if (op.src1 >= 0) lam_of(o, sm, op.src1)[j] += lam[j];
          }
          break;
        case 3: {
          for (int j = tid; j < op.dim; j += kThreads) {
            ls[j] += op.scaled * lam[j];
            bacc += op.offsetd * lam[j];
          }
          break;
        }
        case 4: {  // SQDIST: tangent at the midpoint (below) / chord (above)
          const double c = lam[0];
          const double* tg = o.dd + op.tgtd;
          const double* wt = o.dd + op.wtd + (op.weight_by_step ? t * op.in_dim : 0);
          for (int j = tid; j < op.in_dim; j += kThreads) {
            const double l = B.lo(t, st + j), u = B.hi(t, st + j), w = wt[j], tj = tg[j];
            if (c >= 0.0) {
              const double m = 0.5 * (l + u);
              ls[j] += c * (2.0 * w * (m - tj));
              bacc += c * (-w * (m - tj) * (m + tj));
            } else {
              const double sl = w * (l + u - 2.0 * tj);
              ls[j] += c * sl;
              bacc += c * (w * (l - tj) * (l - tj) - sl * l);
            }
          }
          break;
        }
        case 5:  // HINGE: anchor on its own output bounds
          if (tid == 0) {
            const double c = lam[0];
            bacc += c * (c >= 0.0 ? B.lo(t, op.stat) : B.hi(t, op.stat));
          }
          break;
        case 6:
          for (int j = tid; j < op.dim; j += kThreads) ls[op.begin + j] += lam[j];
          break;
      }
      __syncthreads();
    }
    // 2. x_t as a stop node: anchor on its extrema, nothing flows below.
    const bool xstop = stops && o.iv[o.xstop + t] != 0;
    const bool mlp_live = !node || !top || a.start_kind <= 1 || a.start_kind == 4;
    for (int j = tid; j < o.ks; j += kThreads) {
      sm.lam[j] = mlp_live ? sm.lx[j] : 0.0;
      if (xstop) {
        const double c = sm.lx[j];
        bacc += c * (c >= 0.0 ? B.lo(t, o.x_stat + j) : B.hi(t, o.x_stat + j));
        sm.lam[j] = 0.0;
      }
    }
    // a pre-activation node starts inside the MLP: lam on the output of layer start_index
    const int l_top = (node && top && a.start_kind == 0) ? a.start_index : o.L - 1;
    if (node && top && a.start_kind == 0) {
      __syncthreads();
      for (int j = tid; j < o.widths[l_top + 1]; j += kThreads) sm.lam[j] = j == row ? sign : 0.0;
    }
    __syncthreads();
    // 3. MLP layers l_top..1
    bool cut = xstop || !mlp_live;
    for (int l = l_top; l >= 0 && !cut; --l) {
      const int K = o.widths[l], N = o.widths[l + 1];
      const double* W = o.dd + o.wd[l];
      for (int j = tid; j < K; j += kThreads) {
        double acc = 0.0;
        for (int r = 0; r < N; ++r) acc += sm.lam[r] * W[static_cast<size_t>(r) * K + j];
        sm.lam2[j] = acc;
      }
      for (int r = tid; r < N; r += kThreads) bacc += sm.lam[r] * o.dd[o.bd[l] + r];
      __syncthreads();
      if (l > 0 && o.relu[l - 1]) {
        const int st = o.pre_stat[l - 1];
        const bool anchor = stops && last && o.stop_layer == l - 1;
        for (int j = tid; j < K; j += kThreads) {
          const double c = sm.lam2[j], lo = B.lo(t, st + j), hi = B.hi(t, st + j);
          double out = 0.0;
          if (anchor) {
            bacc += c * (c >= 0.0 ? fmax(lo, 0.0) : fmax(hi, 0.0));
          } else if (c >= 0.0) {
            out = c * relu_lower_slope(lo, hi, a.alpha);
          } else if (lo >= 0.0) {
            out = c;
          } else if (hi > 0.0) {
            out = c * (hi / (hi - lo));
            bacc += c * (-hi * lo / (hi - lo));
          }
          sm.lam[j] = out;
        }
        if (anchor) cut = true;
      } else {
        for (int j = tid; j < K; j += kThreads) sm.lam[j] = sm.lam2[j];
      }
      __syncthreads();
    }
    // 4. features -> x_{t-1}, p_{t-1}, u_t ; p_t = p_{t-1} + u_t.  A bare network (o.net:
    //    build_network_objective, model.cpp:389-405) reads u_t only.
    const int uoff = o.net ? 0 : o.ks;
    for (int j = tid; j < o.ks; j += kThreads) sm.lx[j] = (cut || o.net) ? 0.0 : sm.lam[j];
    for (int j = tid; j < o.ka; j += kThreads) {
      double lu = sm.lu[j] + sm.lpt[j] + (cut ? 0.0 : sm.lam[uoff + j]);
      // concretize the input slice u_t on the box (crown.cpp:461, 296-319)
      bacc += lu * (lu >= 0.0 ? a.lo[boxoff + t * o.ka + j] : a.hi[boxoff + t * o.ka + j]);
    }
    for (int j = tid; j < o.kd; j += kThreads) {
      double lp = sm.lpt[j];
      if (o.rel && !cut)
        for (int k = 0; k < o.ks / o.kd; ++k) lp -= sm.lam[k * o.kd + j];
      sm.lp[j] = lp;
    }
    __syncthreads();
  }
  // constants x0, p0 fold into the offset
  for (int j = tid; j < o.ks; j += kThreads) bacc += sm.lx[j] * o.dd[o.x0d + j];
  for (int j = tid; j < o.kd; j += kThreads) bacc += sm.lp[j] * o.dd[o.p0d + j];
  // deterministic block reduction
  for (int off = 16; off > 0; off >>= 1) bacc += __shfl_down_sync(0xffffffffu, bacc, off);
  if ((tid & 31) == 0) sm.red[tid >> 5] = bacc;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < kThreads / 32; ++w) tot += sm.red[w];
  __syncthreads();
  return tot;
}

template <int MW>
__global__ void __launch_bounds__(kThreads) bound_kernel(const DevObjective o, const BoundArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem<MW>& sm = *reinterpret_cast<Smem<MW>*>(smraw);
  if (a.start_kind >= 0) {  // full-CROWN node pass: CTA = (subdomain, row)
    const int s = blockIdx.x / a.start_dim, row = blockIdx.x % a.start_dim;
    const Bounds B{o, a, static_cast<long long>(s) * o.H * o.SP, false};
    double lo = sweep(o, a, sm, B, s, row, 1.0);
    double hi = -sweep(o, a, sm, B, s, row, -1.0);  // upper(v) = -lower(-v): every relaxation is by sign
    if (lo > hi) {  // guard against rounding inversions on degenerate coordinates (crown.cpp:406-407)
      const double tmp = lo;
      lo = hi;
      hi = tmp;
    }
    if (threadIdx.x == 0) {
      const long long i = static_cast<long long>(s) * o.H * o.SP + static_cast<long long>(a.start_t) * o.SP +
                          a.start_slot + row;
      a.ivl_lo[i] = lo;
      a.ivl_hi[i] = hi;
    }
    return;
  }
  const int s = blockIdx.x;
  const bool emp = a.mode == 1 && a.use_stats != nullptr && a.use_stats[s] != 0 && a.stat_min != nullptr;
  if (!emp && a.mode != 0) interval_pass(o, a, sm, s);  // full CROWN: node bounds already in ivl
  const Bounds B{o, a, static_cast<long long>(s) * o.H * o.SP, emp};
  const double tot = sweep(o, a, sm, B, s, 0, 1.0);
  if (threadIdx.x == 0) a.lf[s] = tot;
}

// Hinge outputs under full CROWN: enclosed from their argument's bounds, never
// propagated (crown_node_bounds, crown.cpp:393-400; hinge_interval :360-375).
__global__ void hinge_bounds_kernel(const DevObjective o, const BoundArgs a, int t, int op_index) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.start_dim) return;  // start_dim = subdomains here
  const DevOp& op = o.ops[op_index];
  const long long base = static_cast<long long>(s) * o.H * o.SP + static_cast<long long>(t) * o.SP;
  const int st = stat_of(o, op.src0);
  const double* c = o.dd + op.ctrd;
  double d2l = 0.0, d2h = 0.0;
  for (int j = 0; j < op.in_dim; ++j) {
    const double x = a.ivl_lo[base + st + j] - c[j], y = a.ivl_hi[base + st + j] - c[j];
    d2h += fmax(x * x, y * y);
    d2l += (x <= 0.0 && y >= 0.0) ? 0.0 : fmin(x * x, y * y);
  }
  const double ml = op.radiusd - sqrt(d2h), mh = op.radiusd - sqrt(d2l);
  a.ivl_lo[base + op.stat] = ml > 0.0 ? op.penaltyd * ml : 0.0;
  a.ivl_hi[base + op.stat] = mh > 0.0 ? op.penaltyd * mh : 0.0;
}

}  // namespace

// Scratch width the bound kernel needs: the widest layer and the per-row scratch (op values by column).
int bound_width(const DevObjective& o) {
  int w = o.bw;  // compile(): max(widest layer, ks, end of the last op column) -- what Smem<MW> is indexed by
  for (int l = 0; l <= o.L; ++l) w = o.widths[l] > w ? o.widths[l] : w;
  return w;
}
size_t bound_smem_bytes() { return sizeof(Smem<kMaxW>); }

// Instantiated at the smallest width class that holds the objective: shared memory of
// 12 x width doubles per CTA, so narrow objectives keep several CTAs per SM.
cudaError_t launch_bound(const DevObjective& o, const BoundArgs& a, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long long grid = a.start_kind >= 0 ? static_cast<long long>(n) * a.start_dim : n;
  auto go = [&](auto kern, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(grid), kThreads, smem, st>>>(o, a);
    return cudaGetLastError();
  };
  const int w = bound_width(o);
  if (w <= 128) return go(bound_kernel<128>, sizeof(Smem<128>));
  if (w <= 256) return go(bound_kernel<256>, sizeof(Smem<256>));
  if (w <= 512) return go(bound_kernel<512>, sizeof(Smem<512>));
  if (w <= kMaxW) return go(bound_kernel<kMaxW>, sizeof(Smem<kMaxW>));
  return cudaErrorInvalidValue;
}

cudaError_t launch_hinge_bounds(const DevObjective& o, const BoundArgs& a, int t, int op_index, cudaStream_t st) {
  if (a.start_dim <= 0) return cudaSuccess;
  hinge_bounds_kernel<<<(a.start_dim + 127) / 128, 128, 0, st>>>(o, a, t, op_index);
  return cudaGetLastError();
}

}  // namespace bp

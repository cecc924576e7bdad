// rollout_common.cuh -- pieces shared by the SIMT (rollout.cu) and the
// tcgen05 (rollout_tc.cu) rollout kernels: launch arguments, the per-tile
// subdomain split, the column extrema pass and the per-row cost program
// (reference node semantics, proj/src/graph.cpp:293-347).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "bp_common.cuh"

namespace bp {

struct RolloutArgs {
  const float* actions;  // [n_rows][d]
  float* costs;          // [n_rows]
  float* states;         // optional [n_rows][H][ks]
  int* stat_min;         // [n_sub][H*SP] (enc_f), may be null
  int* stat_max;
  int* failed;           // [n_sub], may be null: set when a row's objective is non-finite
  long long n_rows;
  int rows_per_sub;
  int kslab;             // streamed mode: K rows per weight slab
  long long* timeline;   // optional (BP_TC_TIMELINE): clock64 marks of CTA 0, see rollout_tc.cu
};

// Rows of a tile split into at most two subdomains: rows [0, bnd) belong to
// subdomain seg0, rows [bnd, nvalid) to seg0 + 1 (bnd = nvalid when one).
struct TileSeg {
  long long seg0;
  int bnd, nvalid;
  bool two;  // the tile fits the two-segment form (rows_per_sub >= R)
};

// Column pass over act[:, col0 : col0+ncols): per-subdomain extrema of the
// valid rows into the global record (stat >= 0) and optional in-place ReLU.
// segl[r] is the tile-local subdomain of row r (-1 past the last valid row);
// seg0 the subdomain of the tile's first row.
// Barrier of the threads running the row work: the whole CTA (BAR = 0), or
// named barrier 1 over the 128 row threads of a warp-specialized CTA.
template <int BAR>
__device__ __forceinline__ void row_sync() {
  if constexpr (BAR == 0)
    __syncthreads();
  else
    asm volatile("bar.sync 1, 128;" ::: "memory");
}

template <int R, int BAR = 0>
__device__ void column_pass(const DevObjective& o, const RolloutArgs& a, float* act, int S, const int* segl,
                            long long seg0, int col0, int ncols, int stat, bool relu, int t) {
  const bool rec = stat >= 0 && a.stat_min != nullptr;
  if (ncols <= 0 || (!rec && !relu)) return;  // uniform across the CTA
  const int nthr = BAR == 0 ? static_cast<int>(blockDim.x) : 128;
  const int groups = max(1, min(R, nthr / ncols));
  const int rpg = (R + groups - 1) / groups;
  const long long SPH = static_cast<long long>(o.SP) * o.H;
  const int soff = t * o.SP + stat;
  for (int item = threadIdx.x; item < ncols * groups; item += nthr) {
    const int c = item % ncols, g = item / ncols;
    const int rb = g * rpg, re = min(R, rb + rpg);
    float mn = INFINITY, mx = -INFINITY;
    int seg = -1;
    float* p = act + rb * S + col0 + c;
    for (int r = rb; r < re; ++r, p += S) {
      const float v = *p;
      if (rec) {
        const int s = segl[r];
        if (s != seg) {
          if (seg >= 0) {
            const long long idx = (seg0 + seg) * SPH + soff + c;
            atomicMin(a.stat_min + idx, enc_f(mn));
            atomicMax(a.stat_max + idx, enc_f(mx));
          }
          seg = s;
          mn = INFINITY;
          mx = -INFINITY;
        }
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
      }
      if (relu) *p = fmaxf(v, 0.f);
    }
    if (rec && seg >= 0) {
      const long long idx = (seg0 + seg) * SPH + soff + c;
      atomicMin(a.stat_min + idx, enc_f(mn));
      atomicMax(a.stat_max + idx, enc_f(mx));
    }
  }
  row_sync<BAR>();
}

__device__ __forceinline__ const float* val_ptr(const DevObjective& o, const DevOp* ops, const float* row, int id) {
  if (id == 0) return row;                 // x_t
  if (id == 1) return row + o.ucol;        // u_t
  if (id == 2) return row + o.pcol;        // p_t
  return row + ops[id - 3].col;            // op output
}

// The step's cost program for one row (reference node semantics, graph.cpp:293-347).
// ops: the objective's op table (kernel parameters, or a shared-memory copy);
// cf: base such that cf + op.<offset> addresses the op constants (o.f, or a
// shared-memory copy of the arena range [cost_f0, cost_f1) shifted by -cost_f0).
__device__ __forceinline__ float cost_program(const DevObjective& o, const DevOp* ops, const float* cf, float* row,
                                             int t) {
  float cost = 0.f;
  for (int i = 0; i < o.n_ops; ++i) {
    const DevOp& op = ops[i];
    const float* src = val_ptr(o, ops, row, op.src0);
    float* dst = row + op.col;
    float v = 0.f;
    switch (op.kind) {
      case 0: {  // LINEAR
        const float* W = cf + op.w;
        const float* b = cf + op.b;
        for (int r = 0; r < op.dim; ++r) {
          float s = 0.f;
          for (int j = 0; j < op.in_dim; ++j) s = fmaf(W[r * op.in_dim + j], src[j], s);
          dst[r] = s + b[r];
        }
        v = dst[0];
        break;
      }
      case 1:  // RELU
        for (int j = 0; j < op.dim; ++j) dst[j] = fmaxf(src[j], 0.f);
        v = dst[0];
        break;
      case 2: {  // SUM
        const float* s1 = op.src1 >= 0 ? val_ptr(o, ops, row, op.src1) : nullptr;
        for (int j = 0; j < op.dim; ++j) dst[j] = s1 ? src[j] + s1[j] : src[j];
        v = dst[0];
        break;
      }
      case 3:  // SCALAR_AFFINE
        for (int j = 0; j < op.dim; ++j) dst[j] = op.scale * src[j] + op.offset;
        v = dst[0];
        break;
      case 4: {  // SQDIST
        const float* tg = cf + op.tgt;
        const float* wt = cf + op.wt + (op.weight_by_step ? t * op.in_dim : 0);
        float acc = 0.f;
        for (int j = 0; j < op.in_dim; ++j) {
          const float d = src[j] - tg[j];
          acc += wt[j] * d * d;
        }
        dst[0] = v = acc;
        break;
      }
      case 5: {  // HINGE
        const float* c = cf + op.ctr;
        float acc = 0.f;
        for (int j = 0; j < op.in_dim; ++j) {
          const float d = src[j] - c[j];
          acc += d * d;
        }
        const float m = op.radius - sqrtf(acc);
        dst[0] = v = m > 0.f ? op.penalty * m : 0.f;
        break;
      }
      case 6:  // SLICE
        for (int j = 0; j < op.dim; ++j) dst[j] = src[op.begin + j];
        v = dst[0];
        break;
    }
    if (op.is_term) cost += v;
  }
  return cost;
}


}  // namespace bp

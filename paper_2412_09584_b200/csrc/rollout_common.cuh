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

// Forward-only op record (80 B): what the cost program reads of a DevOp, loaded
// with five 16-byte shared-memory loads issued back to back.
struct alignas(16) FwdOp {
  int kind, c0, c1, col, dim, in_dim, begin, is_term;
  int weight_by_step, w, b, tgt, wt, ctr, pad0, pad1;
  float scale, offset, radius, penalty;
};

__device__ __forceinline__ FwdOp to_fwd(const DevOp& d) {
  FwdOp f;
  f.kind = d.kind, f.c0 = d.c0, f.c1 = d.c1, f.col = d.col, f.dim = d.dim, f.in_dim = d.in_dim, f.begin = d.begin;
  f.is_term = d.is_term, f.weight_by_step = d.weight_by_step, f.w = d.w, f.b = d.b, f.tgt = d.tgt, f.wt = d.wt;
  f.ctr = d.ctr, f.pad0 = 0, f.pad1 = 0;
  f.scale = d.scale, f.offset = d.offset, f.radius = d.radius, f.penalty = d.penalty;
  return f;
}

__device__ __forceinline__ FwdOp load_op(const FwdOp* p) {
  FwdOp r;
  const int4* s = reinterpret_cast<const int4*>(p);
  int4* d = reinterpret_cast<int4*>(&r);
#pragma unroll
  for (int q = 0; q < 5; ++q) d[q] = s[q];
  return r;
}
__device__ __forceinline__ const DevOp& load_op(const DevOp* p) { return *p; }

// The step's cost program for NR rows of one thread, interleaved so the rows'
// dependent chains overlap (reference node semantics, graph.cpp:293-347).
// ops: the objective's op table (kernel parameters, or a shared-memory copy);
// cf: base such that cf + op.<offset> addresses the op constants (o.f, or a
// shared-memory copy of the arena range [cost_f0, cost_f1) shifted by -cost_f0).
template <int NR, class OpT>
__device__ __forceinline__ void cost_program_n(const DevObjective& o, const OpT* ops, const float* cf,
                                               float* const (&row)[NR], int t, float (&cost)[NR]) {
  for (int i = 0; i < o.n_ops; ++i) {
    const auto& op = load_op(ops + i);
    const int c0 = op.c0, c1 = op.c1, oc = op.col, dim = op.dim, in = op.in_dim;
    float v[NR];
    switch (op.kind) {
      case 0: {  // LINEAR
        const float* W = cf + op.w;
        const float* b = cf + op.b;
        if (op.ctr) {  // CSR of a sparse weight matrix (host compile): the fma chain over the nonzeros
          const int* rp = reinterpret_cast<const int*>(cf + op.tgt);
          const int* ci = rp + dim + 1;
          const float* val = reinterpret_cast<const float*>(ci + rp[dim]);
#pragma unroll 4
          for (int r = 0; r < dim; ++r) {
            float s[NR];
#pragma unroll
            for (int q = 0; q < NR; ++q) s[q] = 0.f;
#pragma unroll 4
            for (int k = rp[r]; k < rp[r + 1]; ++k) {
              const float w = val[k];
              const int j = ci[k];
#pragma unroll
              for (int q = 0; q < NR; ++q) s[q] = fmaf(w, row[q][c0 + j], s[q]);
            }
#pragma unroll
            for (int q = 0; q < NR; ++q) row[q][oc + r] = s[q] + b[r];
          }
#pragma unroll
          for (int q = 0; q < NR; ++q) v[q] = row[q][oc];
          break;
        }
#pragma unroll 4
        for (int r = 0; r < dim; ++r) {
          float s[NR];
#pragma unroll
          for (int q = 0; q < NR; ++q) s[q] = 0.f;
#pragma unroll 4
          for (int j = 0; j < in; ++j) {
            const float w = W[r * in + j];
#pragma unroll
            for (int q = 0; q < NR; ++q) s[q] = fmaf(w, row[q][c0 + j], s[q]);
          }
#pragma unroll
          for (int q = 0; q < NR; ++q) row[q][oc + r] = s[q] + b[r];
        }
#pragma unroll
        for (int q = 0; q < NR; ++q) v[q] = row[q][oc];
        break;
      }
      case 1:  // RELU
#pragma unroll 4
        for (int j = 0; j < dim; ++j)
#pragma unroll
          for (int q = 0; q < NR; ++q) row[q][oc + j] = fmaxf(row[q][c0 + j], 0.f);
#pragma unroll
        for (int q = 0; q < NR; ++q) v[q] = row[q][oc];
        break;
      case 2:  // SUM
#pragma unroll 4
        for (int j = 0; j < dim; ++j)
#pragma unroll
          for (int q = 0; q < NR; ++q) row[q][oc + j] = c1 >= 0 ? row[q][c0 + j] + row[q][c1 + j] : row[q][c0 + j];
#pragma unroll
        for (int q = 0; q < NR; ++q) v[q] = row[q][oc];
        break;
      case 3: {  // SCALAR_AFFINE
        const float sc = op.scale, of = op.offset;
#pragma unroll 4
        for (int j = 0; j < dim; ++j)
#pragma unroll
          for (int q = 0; q < NR; ++q) row[q][oc + j] = sc * row[q][c0 + j] + of;
#pragma unroll
        for (int q = 0; q < NR; ++q) v[q] = row[q][oc];
        break;
      }
      case 4: {  // SQDIST
        const float* tg = cf + op.tgt;
        const float* wt = cf + op.wt + (op.weight_by_step ? t * in : 0);
        float acc[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) acc[q] = 0.f;
#pragma unroll 4
        for (int j = 0; j < in; ++j) {
          const float g = tg[j], w = wt[j];
#pragma unroll
          for (int q = 0; q < NR; ++q) {
            const float dd = row[q][c0 + j] - g;
            acc[q] += w * dd * dd;
          }
        }
#pragma unroll
        for (int q = 0; q < NR; ++q) row[q][oc] = v[q] = acc[q];
        break;
      }
      case 5: {  // HINGE
        const float* c = cf + op.ctr;
        float acc[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) acc[q] = 0.f;
#pragma unroll 4
        for (int j = 0; j < in; ++j) {
          const float g = c[j];
#pragma unroll
          for (int q = 0; q < NR; ++q) {
            const float dd = row[q][c0 + j] - g;
            acc[q] += dd * dd;
          }
        }
        const float rad = op.radius, pen = op.penalty;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const float mg = rad - sqrtf(acc[q]);
          row[q][oc] = v[q] = mg > 0.f ? pen * mg : 0.f;
        }
        break;
      }
      case 7: {  // a LINEAR on x_t folded into the output layer's MMA (rollout_tc2.cu): its values are in the scratch
#pragma unroll
        for (int q = 0; q < NR; ++q) v[q] = row[q][oc];
        break;
      }
      default: {  // SLICE
        const int b0 = c0 + op.begin;
#pragma unroll 4
        for (int j = 0; j < dim; ++j)
#pragma unroll
          for (int q = 0; q < NR; ++q) row[q][oc + j] = row[q][b0 + j];
#pragma unroll
        for (int q = 0; q < NR; ++q) v[q] = row[q][oc];
        break;
      }
    }
    if (op.is_term)
#pragma unroll
      for (int q = 0; q < NR; ++q) cost[q] += v[q];
  }
}

__device__ __forceinline__ float cost_program(const DevObjective& o, const DevOp* ops, const float* cf, float* row,
                                             int t) {
  float* const rows[1] = {row};
  float c[1] = {0.f};
  cost_program_n<1>(o, ops, cf, rows, t, c);
  return c[0];
}


}  // namespace bp

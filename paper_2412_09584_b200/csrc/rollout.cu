// rollout.cu -- K1: fused H-step rollout of the ReLU-MLP dynamics with the
// step cost program and the per-subdomain sample extrema of every watched
// coordinate (the empirical pre-activation bounds).
//
// Restates, for a whole batch of subdomains at once:
//   evaluate / forward_chunk  (reference proj/src/graph.cpp:252-401) on the
//   graph build_objective unrolls (proj/src/model.cpp:310-387), and the
//   watch-stat recording (graph.cpp:270-281, 361-374).
//
// Layout.  A CTA owns a tile of R = 16*TM consecutive rows (samples) of the
// flat [n_sub x rows_per_sub] batch; a tile may straddle two subdomains.
// The activations of its rows live in shared memory as [R][S] floats
// (row-major, stride S = 4 mod 8 words so the two row-groups a warp reads
// fall in different banks) and are updated in place layer by layer: the
// whole layer accumulates in registers before one barrier and the write-back.
// Weights sit in shared memory transposed to [K][N] (k-major), either all
// layers resident for the whole kernel or streamed per layer in K-slabs.
// Every output of a row is a fixed-order FMA chain over k, so a row's
// result never depends on the tile it lands in (graph.hpp:102-103).
#include <cuda_runtime.h>

#include <cstdint>

#include "rollout_common.cuh"

namespace bp {

namespace {

__device__ __forceinline__ float f4get(const float4& v, int k) {
  return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}

// Register-tiled layer: rows ty + 16 i (i < TM), columns q*64 + tx*4 + c.
// FULL: every column quad q < NQ holds live columns (no per-quad predicate).
template <int TM, int NQ, bool FULL>
__device__ __forceinline__ void kloop_wide(const float* __restrict__ act, int S, const float* __restrict__ W,
                                           int NS, int k0, int k1, float (&acc)[TM][NQ * 4]) {
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  const float* xr = act + ty * S;
  const float* wr = W + tx * 4;
#pragma unroll 1
  for (int k = k0; k < k1; k += 4) {
    float4 xv[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) xv[i] = *reinterpret_cast<const float4*>(xr + 16 * i * S + k);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      float4 wv[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        wv[q] = (FULL || q * 64 < NS) ? *reinterpret_cast<const float4*>(wr + (k - k0 + kk) * NS + q * 64)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const float xs = f4get(xv[i], kk);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          if (FULL || q * 64 < NS) {
            acc[i][q * 4 + 0] = fmaf(xs, wv[q].x, acc[i][q * 4 + 0]);
            acc[i][q * 4 + 1] = fmaf(xs, wv[q].y, acc[i][q * 4 + 1]);
            acc[i][q * 4 + 2] = fmaf(xs, wv[q].z, acc[i][q * 4 + 2]);
            acc[i][q * 4 + 3] = fmaf(xs, wv[q].w, acc[i][q * 4 + 3]);
          }
        }
      }
    }
  }
}

template <int TM, int NQ>
__device__ __forceinline__ void kloop_any(const float* act, int S, const float* W, int NS, int k0, int k1,
                                          float (&acc)[TM][NQ * 4]) {
  if (NS > 64 * (NQ - 1))
    kloop_wide<TM, NQ, true>(act, S, W, NS, k0, k1, acc);
  else
    kloop_wide<TM, NQ, false>(act, S, W, NS, k0, k1, acc);
}

// Cooperative global -> shared copy of n floats (16B aligned).
__device__ __forceinline__ void copy_f4(float* dst, const float* __restrict__ src, int n) {
  const int n4 = n >> 2;
  for (int i = threadIdx.x; i < n4; i += kThreads)
    reinterpret_cast<float4*>(dst)[i] = __ldg(reinterpret_cast<const float4*>(src) + i);
}

// Wide layer with the fused epilogue: bias in the accumulator, per-column
// extrema of the pre-activations (register -> xor-16 shuffle -> shared
// atomics -> one global atomic per column and subdomain), ReLU applied on
// the way back to shared memory.
template <int TM, int NQ, bool STREAM>
__device__ void layer_wide(const DevObjective& o, const RolloutArgs& a, float* act, float* wsm, int* red, int l,
                           const TileSeg& ts, int t) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4, lane = threadIdx.x & 31;
  const int K4 = o.kpad[l], NS = o.nstr[l], S = o.S, N = o.widths[l + 1], RW = o.red_w;
  const float* __restrict__ bias = o.f + o.bias[l];
  float acc[TM][NQ * 4];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int col = q * 64 + tx * 4;
    const float4 bq = col < NS ? __ldg(reinterpret_cast<const float4*>(bias + col)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      acc[i][q * 4 + 0] = bq.x;
      acc[i][q * 4 + 1] = bq.y;
      acc[i][q * 4 + 2] = bq.z;
      acc[i][q * 4 + 3] = bq.w;
    }
  }
  if constexpr (!STREAM) {
    kloop_any<TM, NQ>(act, S, wsm + o.w_smem_off[l], NS, 0, K4, acc);
  } else {
    const float* __restrict__ wg = o.f + o.wt[l];
    for (int k0 = 0; k0 < K4; k0 += a.kslab) {
      const int k1 = min(K4, k0 + a.kslab);
      __syncthreads();  // previous slab fully consumed
      copy_f4(wsm, wg + static_cast<size_t>(k0) * NS, (k1 - k0) * NS);
      __syncthreads();
      kloop_any<TM, NQ>(act, S, wsm, NS, k0, k1, acc);
    }
  }
  const bool relu = o.relu[l] != 0;
  const int stat = o.pre_stat[l];
  const bool rec = ts.two && relu && stat >= 0 && a.stat_min != nullptr;
  const bool apply_relu = relu && ts.two;  // otherwise the column pass records, then rectifies
  if (rec) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (q * 64 >= NS) continue;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float mn0 = INFINITY, mx0 = -INFINITY, mn1 = INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const int r = ty + 16 * i;
          const float v = acc[i][q * 4 + c];
          if (r < ts.bnd) {
            mn0 = fminf(mn0, v);
            mx0 = fmaxf(mx0, v);
          } else if (r < ts.nvalid) {
            mn1 = fminf(mn1, v);
            mx1 = fmaxf(mx1, v);
          }
        }
        mn0 = fminf(mn0, __shfl_xor_sync(0xffffffffu, mn0, 16));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 16));
        mn1 = fminf(mn1, __shfl_xor_sync(0xffffffffu, mn1, 16));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 16));
        const int col = q * 64 + tx * 4 + c;
        if (lane < 16 && col < N) {
          atomicMin(red + col, enc_f(mn0));
          atomicMax(red + RW + col, enc_f(mx0));
          atomicMin(red + 2 * RW + col, enc_f(mn1));
          atomicMax(red + 3 * RW + col, enc_f(mx1));
        }
      }
    }
  }
  __syncthreads();  // every row's inputs consumed: write in place
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int col = q * 64 + tx * 4;
    if (col < NS) {
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        float4 v = make_float4(acc[i][q * 4 + 0], acc[i][q * 4 + 1], acc[i][q * 4 + 2], acc[i][q * 4 + 3]);
        if (apply_relu) {
          v.x = fmaxf(v.x, 0.f);
          v.y = fmaxf(v.y, 0.f);
          v.z = fmaxf(v.z, 0.f);
          v.w = fmaxf(v.w, 0.f);
        }
        *reinterpret_cast<float4*>(act + (ty + 16 * i) * S + col) = v;
      }
    }
  }
  if (rec) {  // flush this layer's extrema and reset the shared buffer
    const long long SPH = static_cast<long long>(o.SP) * o.H;
    for (int item = threadIdx.x; item < 2 * N; item += kThreads) {
      const int sg = item / N, col = item % N;
      const int vmin = red[2 * sg * RW + col], vmax = red[(2 * sg + 1) * RW + col];
      red[2 * sg * RW + col] = enc_f(INFINITY);
      red[(2 * sg + 1) * RW + col] = enc_f(-INFINITY);
      if (sg == 1 && ts.bnd >= ts.nvalid) continue;
      const long long idx = (ts.seg0 + sg) * SPH + t * o.SP + stat + col;
      atomicMin(a.stat_min + idx, vmin);
      atomicMax(a.stat_max + idx, vmax);
    }
  }
  __syncthreads();
}

// Narrow layer (N <= 16): one thread per row, all columns.
template <int R, bool STREAM>
__device__ void layer_narrow(const DevObjective& o, float* act, float* wsm, int l, int kslab) {
  const int K4 = o.kpad[l], NS = o.nstr[l], S = o.S;
  const int r = threadIdx.x;
  const float* __restrict__ bias = o.f + o.bias[l];
  float acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = c < NS ? __ldg(bias + c) : 0.f;
  auto kl = [&](const float* W, int k0, int k1) {
    if (r < R) {
      for (int k = k0; k < k1; k += 4) {
        const float4 xv = *reinterpret_cast<const float4*>(act + r * S + k);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float xs = f4get(xv, kk);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (q * 4 < NS) {
              const float4 w = *reinterpret_cast<const float4*>(W + (k - k0 + kk) * NS + q * 4);
              acc[q * 4 + 0] = fmaf(xs, w.x, acc[q * 4 + 0]);
              acc[q * 4 + 1] = fmaf(xs, w.y, acc[q * 4 + 1]);
              acc[q * 4 + 2] = fmaf(xs, w.z, acc[q * 4 + 2]);
              acc[q * 4 + 3] = fmaf(xs, w.w, acc[q * 4 + 3]);
            }
          }
        }
      }
    }
  };
  if constexpr (!STREAM) {
    kl(wsm + o.w_smem_off[l], 0, K4);
  } else {
    const float* __restrict__ wg = o.f + o.wt[l];
    for (int k0 = 0; k0 < K4; k0 += kslab) {
      const int k1 = min(K4, k0 + kslab);
      __syncthreads();
      copy_f4(wsm, wg + static_cast<size_t>(k0) * NS, (k1 - k0) * NS);
      __syncthreads();
      kl(wsm, k0, k1);
    }
  }
  __syncthreads();
  if (r < R) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q * 4 < NS)
        *reinterpret_cast<float4*>(act + r * S + q * 4) =
            make_float4(acc[q * 4 + 0], acc[q * 4 + 1], acc[q * 4 + 2], acc[q * 4 + 3]);
  }
  __syncthreads();
}

template <int TM, int NQ, bool STREAM>
__global__ void __launch_bounds__(kThreads, 1) rollout_kernel(const DevObjective o, const RolloutArgs a) {
  constexpr int R = 16 * TM;
  extern __shared__ __align__(16) float smem[];
  float* act = smem;                                // [R][S]
  float* prow = act + R * o.S;                      // [R][8] effector
  int* segl = reinterpret_cast<int*>(prow + R * 8);  // [R] tile-local subdomain per row
  int* red = segl + R;                              // [2 seg][min|max][red_w] fused-extrema scratch
  float* wsm = prow + R * 9 + 4 * o.red_w;          // weights (resident image or slab)
  const long long row0 = static_cast<long long>(blockIdx.x) * R;
  const long long rem_rows = a.n_rows - row0;
  const int nvalid = static_cast<int>(rem_rows < R ? rem_rows : R);
  const int tid = threadIdx.x;
  const int ks = o.ks, ka = o.ka, kd = o.kd, d = o.d;

  // Skip tiles whose subdomains already failed (their search is abandoned).
  if (a.failed != nullptr) {
    const long long s0 = row0 / a.rows_per_sub, s1 = (row0 + nvalid - 1) / a.rows_per_sub;
    bool all_failed = true;
    for (long long s = s0; s <= s1; ++s) all_failed = all_failed && a.failed[s] != 0;
    if (all_failed) return;
  }

  for (int i = tid; i < R * o.S; i += kThreads) act[i] = 0.f;
  const long long seg0 = row0 / a.rows_per_sub;
  if (tid < R) segl[tid] = tid < nvalid ? static_cast<int>((row0 + tid) / a.rows_per_sub - seg0) : -1;
  for (int i = tid; i < 4 * o.red_w; i += kThreads) red[i] = enc_f(((i / o.red_w) & 1) ? -INFINITY : INFINITY);
  TileSeg ts;
  ts.seg0 = seg0;
  ts.nvalid = nvalid;
  {
    const long long first_next = (seg0 + 1) * a.rows_per_sub;  // first row of the next subdomain
    const long long b = first_next - row0;
    ts.bnd = static_cast<int>(b < nvalid ? b : nvalid);
    ts.two = (row0 + nvalid - 1) / a.rows_per_sub - seg0 <= 1;
  }
  if constexpr (!STREAM) copy_f4(wsm, o.f + o.wt[0] - o.w_smem_off[0], o.w_smem_total);
  __syncthreads();

  // Initial features from x0 / p0 and u_1.
  float cost = 0.f;
  const bool row_ok = tid < R && tid < nvalid;
  const float* urow = row_ok ? a.actions + (row0 + tid) * d : nullptr;
  if (tid < R) {
    float* row = act + tid * o.S;
    for (int j = 0; j < kd; ++j) prow[tid * 8 + j] = o.f[o.p0 + j];
    for (int j = 0; j < ks; ++j) row[j] = o.f[o.x0 + j] - (o.rel ? o.f[o.p0 + j % kd] : 0.f);
    for (int j = 0; j < ka; ++j) row[ks + j] = row_ok ? __ldg(urow + j) : 0.f;
  }
  __syncthreads();

  for (int t = 0; t < o.H; ++t) {
    for (int l = 0; l < o.L; ++l) {
      if (o.nstr[l] <= 16)
        layer_narrow<R, STREAM>(o, act, wsm, l, a.kslab);
      else
        layer_wide<TM, NQ, STREAM>(o, a, act, wsm, red, l, ts, t);
      // narrow hidden layers, or tiles spanning more than two subdomains
      if (o.relu[l] && (o.nstr[l] <= 16 || !ts.two))
        column_pass<R>(o, a, act, o.S, segl, seg0, 0, o.widths[l + 1], o.pre_stat[l], true, t);
    }
    // x_t in act[:, 0:ks).  Cost program with u_t, p_t in the row scratch.
    if (tid < R) {
      float* row = act + tid * o.S;
      for (int j = 0; j < ka; ++j) {
        const float u = row_ok ? __ldg(urow + t * ka + j) : 0.f;
        row[o.ucol + j] = u;
        const float p = prow[tid * 8 + j] + u;
        prow[tid * 8 + j] = p;
        row[o.pcol + j] = p;
      }
      cost += cost_program(o, o.ops, o.f, row, t);
    }
    __syncthreads();
    column_pass<R>(o, a, act, o.S, segl, seg0, 0, ks, o.x_stat, false, t);
    if (o.u_stat >= 0) column_pass<R>(o, a, act, o.S, segl, seg0, o.ucol, ka, o.u_stat, false, t);
    if (o.p_stat >= 0) column_pass<R>(o, a, act, o.S, segl, seg0, o.pcol, kd, o.p_stat, false, t);
    for (int i = 0; i < o.n_ops; ++i)
      if (o.ops[i].stat >= 0) column_pass<R>(o, a, act, o.S, segl, seg0, o.ops[i].col, o.ops[i].dim, o.ops[i].stat, false, t);
    if (tid < R) {
      float* row = act + tid * o.S;
      if (a.states != nullptr && row_ok)
        for (int j = 0; j < ks; ++j) a.states[((row0 + tid) * o.H + t) * ks + j] = row[j];
      if (t + 1 < o.H) {
        if (o.rel)
          for (int j = 0; j < ks; ++j) row[j] -= prow[tid * 8 + j % kd];
        for (int j = 0; j < ka; ++j) row[ks + j] = row_ok ? __ldg(urow + (t + 1) * ka + j) : 0.f;
        for (int j = ks + ka; j < o.kpad[0]; ++j) row[j] = 0.f;
      }
    }
    __syncthreads();
  }
  if (row_ok) {
    a.costs[row0 + tid] = cost;
    if (a.failed != nullptr && !isfinite(cost)) atomicOr(a.failed + (row0 + tid) / a.rows_per_sub, 1);
  }
}

template <int TM, int NQ, bool STREAM>
cudaError_t launch_t(const DevObjective& o, const RolloutArgs& a, size_t smem, cudaStream_t st) {
  constexpr int R = 16 * TM;
  auto k = rollout_kernel<TM, NQ, STREAM>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const long long grid = (a.n_rows + R - 1) / R;
  if (grid <= 0) return cudaSuccess;
  k<<<static_cast<unsigned>(grid), kThreads, smem, st>>>(o, a);
  return cudaGetLastError();
}

}  // namespace

// Tile shape for the widest layer: R = 16*TM rows, 64*NQ columns, 64 accumulators per thread.
int rollout_rows_per_tile(int nq) { return nq == 1 ? 256 : nq == 2 ? 128 : nq == 4 ? 64 : 32; }

cudaError_t launch_rollout(const DevObjective& o, const RolloutArgs& a, int nq, bool stream, size_t smem,
                           cudaStream_t st) {
  switch (nq) {
    case 1: return stream ? launch_t<16, 1, true>(o, a, smem, st) : launch_t<16, 1, false>(o, a, smem, st);
    case 2: return stream ? launch_t<8, 2, true>(o, a, smem, st) : launch_t<8, 2, false>(o, a, smem, st);
    case 4: return stream ? launch_t<4, 4, true>(o, a, smem, st) : launch_t<4, 4, false>(o, a, smem, st);
    case 8: return stream ? launch_t<2, 8, true>(o, a, smem, st) : launch_t<2, 8, false>(o, a, smem, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace bp

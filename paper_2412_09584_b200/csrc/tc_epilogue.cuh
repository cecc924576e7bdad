// tc_epilogue.cuh -- epilogue pieces shared by the tcgen05 rollout kernels with
// in-place TMEM operands (rollout_tc2.cu, rollout_tc3.cu): warp-butterfly column
// extrema of the recorded pre-activations, scratch-column extrema, the hi / lo
// 3xTF32 operand store and the K-block publish.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "rollout_common.cuh"
#include "tc_common.cuh"

namespace bp {
namespace tc {

// Transposing butterfly over the warp for 16 columns: v = this lane's values (one
// row, columns c0..c0+15); returns in (mn, mx) the min / max over all 32 lanes of
// column c0 + (lane & 15).  MASK: lanes with incl == false contribute nothing.
template <bool MASK>
__device__ __forceinline__ void warp_col_extrema16(const float* v, bool incl, float& mn, float& mx) {
  const int lane = threadIdx.x & 31;
  float a[8], b[8];
  {
    const bool up = (lane & 8) != 0;
    if constexpr (MASK) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float l0 = incl ? v[j] : INFINITY, h0 = incl ? v[j + 8] : INFINITY;
        const float l1 = incl ? v[j] : -INFINITY, h1 = incl ? v[j + 8] : -INFINITY;
        a[j] = fminf(up ? h0 : l0, __shfl_xor_sync(0xffffffffu, up ? l0 : h0, 8));
        b[j] = fmaxf(up ? h1 : l1, __shfl_xor_sync(0xffffffffu, up ? l1 : h1, 8));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float r = __shfl_xor_sync(0xffffffffu, up ? v[j] : v[j + 8], 8);
        const float k = up ? v[j + 8] : v[j];
        a[j] = fminf(k, r);
        b[j] = fmaxf(k, r);
      }
    }
  }
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int j = 0; j < s; ++j) {
      const float sa = up ? a[j] : a[j + s], ka = up ? a[j + s] : a[j];
      const float sb = up ? b[j] : b[j + s], kb = up ? b[j + s] : b[j];
      a[j] = fminf(ka, __shfl_xor_sync(0xffffffffu, sa, s));
      b[j] = fmaxf(kb, __shfl_xor_sync(0xffffffffu, sb, s));
    }
  }
  mn = fminf(a[0], __shfl_xor_sync(0xffffffffu, a[0], 16));
  mx = fmaxf(b[0], __shfl_xor_sync(0xffffffffu, b[0], 16));
}

// Column extrema of a 32-column chunk over the warp's rows: lane j ends with column j.
// REDUX: one warp-wide min and max reduction per column (redux.sync .f32, sm_100a: CREDUX into a
// uniform register, NaN inputs ignored like fminf / fmaxf) and a select of column j by lane j --
// about 130 instructions per chunk instead of the transposing butterfly's ~250.  Measured: C4's
// one-tile v2 kernel 77.0 -> 82.3 TFLOP/s; C3's 256-wide tile 189.2 -> 188.4 (it keeps the
// butterfly); C5's v3 unchanged.
template <bool MASK, bool REDUX = true>
__device__ __forceinline__ void warp_col_extrema(const float (&v)[32], bool incl, float& mn, float& mx) {
  if constexpr (REDUX) {
    const int lane = threadIdx.x & 31;
    mn = INFINITY;
    mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float lo = MASK ? (incl ? v[j] : INFINITY) : v[j];
      const float hi = MASK ? (incl ? v[j] : -INFINITY) : v[j];
      float r0, r1;
      asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r0) : "f"(lo));
      asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r1) : "f"(hi));
      if (lane == j) {
        mn = r0;
        mx = r1;
      }
    }
  } else {
    float mn0, mx0, mn1, mx1;
    warp_col_extrema16<MASK>(v, incl, mn0, mx0);
    warp_col_extrema16<MASK>(v + 16, incl, mn1, mx1);
    const bool up = (threadIdx.x & 16) != 0;
    mn = up ? mn1 : mn0;
    mx = up ? mx1 : mx0;
  }
}

// Extrema of one scratch column over the tile's valid rows (v = col[r * stride])
// into the per-subdomain record at offset `off` within a subdomain's [H * SP] block:
// the unrolled two-subdomain form (rows [0, bnd) / [bnd, nvalid)) or, for tiles
// spanning more subdomains (parity-test sizes), a walk over segl.
__device__ __forceinline__ void scratch_column_extrema(const RolloutArgs& a, const float* col, int stride, bool two,
                                                       int bnd, int nvalid, const int* segl, long long seg0,
                                                       long long SPH, long long off) {
  if (two) {
    float mn0 = INFINITY, mx0 = -INFINITY, mn1 = INFINITY, mx1 = -INFINITY;
#pragma unroll 8
    for (int r = 0; r < bnd; ++r) {
      const float v = col[r * stride];
      mn0 = fminf(mn0, v);
      mx0 = fmaxf(mx0, v);
    }
#pragma unroll 8
    for (int r = bnd; r < nvalid; ++r) {
      const float v = col[r * stride];
      mn1 = fminf(mn1, v);
      mx1 = fmaxf(mx1, v);
    }
    if (bnd > 0) {
      atomicMin(a.stat_min + seg0 * SPH + off, enc_f(mn0));
      atomicMax(a.stat_max + seg0 * SPH + off, enc_f(mx0));
    }
    if (bnd < nvalid) {
      atomicMin(a.stat_min + (seg0 + 1) * SPH + off, enc_f(mn1));
      atomicMax(a.stat_max + (seg0 + 1) * SPH + off, enc_f(mx1));
    }
    return;
  }
  float mn = INFINITY, mx = -INFINITY;
  int sg = -1;
  for (int r = 0; r < nvalid; ++r) {
    const int s2 = segl[r];
    if (s2 != sg) {
      if (sg >= 0) {
        atomicMin(a.stat_min + (seg0 + sg) * SPH + off, enc_f(mn));
        atomicMax(a.stat_max + (seg0 + sg) * SPH + off, enc_f(mx));
      }
      sg = s2;
      mn = INFINITY;
      mx = -INFINITY;
    }
    const float v = col[r * stride];
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
  }
  if (sg >= 0) {
    atomicMin(a.stat_min + (seg0 + sg) * SPH + off, enc_f(mn));
    atomicMax(a.stat_max + (seg0 + sg) * SPH + off, enc_f(mx));
  }
}

// Column extrema of this warp's 32 rows (v: 32 columns of one row per lane) into the
// record: lane j handles column c0 + j (< ncols) at record offset off0 + j.
template <bool REDUX = true>
__device__ __forceinline__ void warp_chunk_extrema(const RolloutArgs& a, const float (&v)[32], bool simple, long long ws0,
                                                   long long ws1, bool row_ok, long long grow, long long rps,
                                                   long long SPH, long long off0, int col, int ncols) {
  if (simple) {
    float mn, mx;
    warp_col_extrema<false, REDUX>(v, true, mn, mx);
    if (col < ncols) {
      atomicMin(a.stat_min + ws0 * SPH + off0, enc_f(mn));
      atomicMax(a.stat_max + ws0 * SPH + off0, enc_f(mx));
    }
  } else {
    for (long long s = ws0; s <= ws1; ++s) {
      float mn, mx;
      warp_col_extrema<true, REDUX>(v, row_ok && grow / rps == s, mn, mx);
      if (col < ncols) {
        atomicMin(a.stat_min + s * SPH + off0, enc_f(mn));
        atomicMax(a.stat_max + s * SPH + off0, enc_f(mx));
      }
    }
  }
}

// hi / lo parts of one 32-column K-block of this thread's row: lo = lo_tf32(x) into the row's
// 128-byte line of the SW128 K-block in shared memory (four values at a time), then x itself as
// hi into TMEM (the tensor core truncates it).
__device__ __forceinline__ void store_operand(uint32_t t_hi, unsigned char* lo_blk, int row, float (&v)[32]) {
  float4* line = reinterpret_cast<float4*>(lo_blk + row * 128);
#pragma unroll
  for (int q = 0; q < 8; ++q)
    line[q ^ (row & 7)] = make_float4(lo_tf32(v[4 * q]), lo_tf32(v[4 * q + 1]), lo_tf32(v[4 * q + 2]), lo_tf32(v[4 * q + 3]));
  tmem_st32(t_hi, v);
}

// hi / lo parts of one 32-column K-block of this thread's row, both into TMEM (TS-only
// operands): hi = x (truncated by the tensor core), lo = lo_tf32(x).
__device__ __forceinline__ void store_operand_tt(uint32_t t_hi, uint32_t t_lo, float (&v)[32]) {
  tmem_st32(t_hi, v);
  float l[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) l[j] = lo_tf32(v[j]);
  tmem_st32(t_lo, l);
}

// Publish a written K-block: TMEM stores complete, shared stores visible to the
// async proxy, then one arrival per warp -- on rank 0's barrier for a CTA pair (rank 0
// issues the MMAs that read both CTAs' operands).
__device__ __forceinline__ void publish_chunk(uint64_t* bar, bool to_rank0 = false) {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  fence_proxy_async();
  fence_before();
  if (to_rank0) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive_cta(bar, 0);
  } else {
    mbar_arrive_warp(bar);
  }
}

}  // namespace tc
}  // namespace bp

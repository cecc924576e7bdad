// bp_common.cuh -- compiled device form of a bp_objective_desc and the
// helpers shared by the sm_100a kernels (rollout, bound, search).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bp {

constexpr int kMaxLayers = 8;
constexpr int kMaxOps = 32;
constexpr int kThreads = 256;  // every rollout / bound / search CTA

// One op of the per-step cost program, compiled (cf. bp_cost_op).
struct DevOp {
  int kind, src0, src1, dim, in_dim, begin;
  int is_term, weight_by_step;
  int col;       // column of this op's output inside the per-row scratch
  int c0, c1;    // scratch columns of src0 / src1 (c1 = -1 without a second argument)
  int stat;      // offset of its recorded extrema within one step's record, -1 if not recorded
  int stop;      // RELU op anchored as the last-ReLU stop at step H
  int folded;    // LINEAR on x_t computed by the v2 rollout's output-layer MMA (extra N columns)
  // float arena offsets (forward)
  int w, b, tgt, wt, ctr;
  // double arena offsets (bound)
  int wd, bd, tgtd, wtd, ctrd;
  float scale, offset, radius, penalty;
  double scaled, offsetd, radiusd, penaltyd;
};

// Compiled objective, passed by value to every kernel (~5 KB of params).
struct DevObjective {
  int ks, ka, kd, H, rel, L, d;
  int net;  // bare network (build_network_objective): the MLP reads u_t only, H = 1
  int widths[kMaxLayers + 1];
  int relu[kMaxLayers];
  // forward weights: layer l stored transposed [kpad][nstr] (k-major, zero padded)
  int kpad[kMaxLayers], nstr[kMaxLayers];
  int wt[kMaxLayers], bias[kMaxLayers];   // float arena offsets
  int w_smem_off[kMaxLayers];             // float offset of layer l inside the resident smem image
  int w_smem_total;                       // floats in the resident image (0 when streamed)
  int w_max_layer;                        // floats of the largest single layer image
  int red_w;                              // column stride of the fused-extrema scratch (4 x red_w ints)
  // backward weights: W [out][in] row-major and b, double arena offsets
  int wd[kMaxLayers], bd[kMaxLayers];
  // per-row scratch layout in the activation buffer
  int S;          // row stride (floats) of the activation buffer
  int bw;         // bound-kernel scratch width: max(widest layer, ks, end of the last op column)
  int ucol, pcol; // columns holding u_t and p_t during the cost program
  int n_ops;
  DevOp ops[kMaxOps];
  // watched-coordinate record of one step
  int SP;
  int pre_stat[kMaxLayers];  // preactivation of layer l (hidden, relu), -1 otherwise
  int x_stat, u_stat, p_stat;
  // stop set
  int stop_layer;   // hidden layer whose ReLU output at step H is the last-ReLU stop (-1)
  int stop_op;      // RELU cost op that is the last-ReLU stop at step H (-1)
  int xstop;        // int arena offset: H flags, x_t is a stop node
  // tcgen05 (3xTF32) rollout: per layer a K-block image [kb][hi|lo][npad rows x 32 tf32, 128B-swizzled]
  int tc;                    // eligible (all widths <= 128)
  int tc_w[kMaxLayers], tc_bias[kMaxLayers], tc_npad[kMaxLayers], tc_kb[kMaxLayers], tc_ksteps[kMaxLayers];
  int tc_kbmax, tc_npadmax, tc_S, tc_cols, tc_xs;
  // tcgen05 v2 (rollout_tc2.cu): tiles per CTA (2: widths <= 128, 1: widths <= 256; 0 ineligible) and the
  // weight ring bytes.  The tc_w images hold per K-block [hi: npad rows][lo: npad rows] x 32 (the B operand
  // of one N = npad MMA), each image starting on a 128-byte row of the arena.
  int tc2, tc2_rw, tc2_ring;  // tc2_rw: TMEM region width (128 or 256 columns)
  // v2 output-layer folding: the cost program's LINEAR ops on x_t become extra output columns
  // ks .. ks + fold_n - 1 of the last layer's MMA (W_op W_L, W_op b_L + b_op); int arena
  // fold_list: the scratch column of each extra output column
  int fold_n, fold_list;
  int tc2_pair;               // width 256 as a CTA pair (cta_group::2): every layer 256 wide or <= 128 in 32s
  // CTA pairs (v2, v3): TMA tensor maps over the float arena as [rows][32] fp32 rows, one per distinct
  // per-CTA block height (bp_load_objective encodes them): each CTA's half-block load completes on
  // rank 0's barrier (cp.async.bulk.tensor .cta_group::2), so rank 0 needs no relay of the peer's
  // arrivals
  int tmap_h[8], n_tmap;      // box height (rows) of each map
  const void* tmaps;          // device array of CUtensorMap (64-byte aligned), null when not encoded
  // tcgen05 v3 (rollout_tc3.cu): three layers [K0 <= 32, N0 <= 512, N1 <= 512, N2 <= 32], relu after
  // the hidden two; layer 1 in N chunks of <= 256 with layer 0 recomputed per chunk
  int tc3;                   // eligible
  int tc3_w[3];              // float arena: per layer the weight image (layer 0: [kb][hi|lo][32 x 32];
                             // layer 1: [chunk][kb][hi|lo][cw x 32]; layer 2: [kb][hi|lo][np2 x 32])
  int tc3_np[3];             // padded N of each layer (32, 32, 16 multiples)
  int tc3_bias;              // float arena: b0 [np0] | b1 [np1] | b2 [np2]
  int tc3_k0steps;           // k-steps of 8 of the features (layer-0 K)
  int tc3_ring;              // weight ring bytes
  int sc_list, n_sc;
  int cost_f0, cost_f1;  // float arena range holding every cost-op constant (copied to smem by the tcgen05 kernel)  // int arena: n_sc pairs (scratch column, offset in the step record) of recorded scratch values
  // constants
  int x0, p0, step_w;        // float arena offsets
  int x0d, p0d;              // double arena offsets
  const float* f;
  const double* dd;
  const int* iv;
};

// The tensor map (CTA pairs) whose box is `rows` arena rows tall.
__device__ __forceinline__ const void* tmap_rows(const DevObjective& o, int rows) {
  int i = 0;
  while (i + 1 < o.n_tmap && o.tmap_h[i] != rows) ++i;
  return static_cast<const unsigned char*>(o.tmaps) + 128 * i;
}

// Device-resident subdomain pool (pool.cu; SubdomainRecord payload, bab.hpp:18-28):
// per slot the box, the incumbent action and the top-sample list.  The head fields
// (id, lf, uf, depth, log_vol, samples) stay with the host planner, which replays
// pick_out / prune on them.  Slots live in fixed-size chunks (2^shift slots each, one
// allocation per chunk, never moved), found through a chunk table; within a chunk
// each field is a dense array at a fixed byte offset.
struct PoolArgs {
  int d, K;                       // dimension, top-list capacity
  int shift;                      // log2(slots per chunk)
  unsigned char* const* chunk;    // chunk table (device pointer in kernels, host array on the host)
  size_t o_lo, o_hi, o_best, o_val, o_act, o_n, o_has;  // byte offsets of the fields in a chunk
};
__host__ __device__ inline size_t pool_in_chunk(const PoolArgs& P, int s) {
  return static_cast<size_t>(s & ((1 << P.shift) - 1));
}
__host__ __device__ inline unsigned char* pool_chunk(const PoolArgs& P, int s) { return P.chunk[s >> P.shift]; }
__host__ __device__ inline double* pool_lo(const PoolArgs& P, int s) {  // [d]
  return reinterpret_cast<double*>(pool_chunk(P, s) + P.o_lo) + pool_in_chunk(P, s) * P.d;
}
__host__ __device__ inline double* pool_hi(const PoolArgs& P, int s) {  // [d]
  return reinterpret_cast<double*>(pool_chunk(P, s) + P.o_hi) + pool_in_chunk(P, s) * P.d;
}
__host__ __device__ inline float* pool_best(const PoolArgs& P, int s) {  // [d]
  return reinterpret_cast<float*>(pool_chunk(P, s) + P.o_best) + pool_in_chunk(P, s) * P.d;
}
__host__ __device__ inline float* pool_val(const PoolArgs& P, int s) {  // [K], ascending
  return reinterpret_cast<float*>(pool_chunk(P, s) + P.o_val) + pool_in_chunk(P, s) * P.K;
}
__host__ __device__ inline float* pool_act(const PoolArgs& P, int s) {  // [K][d]
  return reinterpret_cast<float*>(pool_chunk(P, s) + P.o_act) + pool_in_chunk(P, s) * P.K * P.d;
}
__host__ __device__ inline int* pool_n(const PoolArgs& P, int s) {
  return reinterpret_cast<int*>(pool_chunk(P, s) + P.o_n) + pool_in_chunk(P, s);
}
__host__ __device__ inline int* pool_has(const PoolArgs& P, int s) {
  return reinterpret_cast<int*>(pool_chunk(P, s) + P.o_has) + pool_in_chunk(P, s);
}
// One iteration's children by local index i: the search inputs the split writes and the
// top samples routed from the parent (merged with the search's list afterwards).
struct StageArgs {
  float* lo_f;       // [n][d]
  float* hi_f;
  float* warm_f;     // [n][d]; NaN first coordinate = no warm start
  double* lo_d;
  double* hi_d;
  float* val;        // [n][K]
  float* act;        // [n][K][d]
  int* n;            // [n]
};
// One parent split (bab.cpp:155-223).  k_round: -2 width rule (k = 0), -1 no samples
// yet (k = n_top), else llround(top_percent / 100 * samples) before the [1, n_top] clamp.
struct SplitTask {
  int parent;        // parent slot
  int slot[2];       // child slots of local children, else -1
  int dst[2];        // child local index, else -1
  int pack[2];       // shipped record index, else -1
  long long key[2];  // the children's global indices (shipped record header)
  long long k_round;
};
// Shipped child record: doubles {key, n, lo[d], hi[d]}, then floats {val[K], act[K][d]}.
__host__ __device__ inline size_t pool_record_bytes(int d, int K) {
  return sizeof(double) * (2 + 2 * static_cast<size_t>(d)) + sizeof(float) * static_cast<size_t>(K) * (1 + d);
}

// K7 launch arguments (bound.cu; built by host.cu).
struct BoundArgs {
  const double* lo;       // [n][d] boxes
  const double* hi;
  const int* stat_min;    // [n][H*SP] sample extrema (enc_f) or null
  const int* stat_max;
  const int* use_stats;   // [n]: 1 = empirical extrema valid for this subdomain
  double* ivl_lo;         // [n][H*SP] scratch for interval bounds
  double* ivl_hi;
  double* lf;             // [n]
  int mode;               // BP_BOUND_FULL_CROWN (0), BP_BOUND_EMPIRICAL (1) or BP_BOUND_INTERVAL (2)
  int alpha;              // 0 adaptive, 1 zero, 2 one
  // full CROWN (crown_node_bounds, crown.cpp:379-412): ivl_lo/ivl_hi already hold the
  // bounds of every node the pass reads, so no interval pass and no stop anchors.
  // start_kind >= 0: a node pass -- the backward sweep starts at row r of the slot's
  // node at step start_t (one CTA per (subdomain, row)) and writes the node's lower /
  // upper bound into ivl_lo / ivl_hi; -1: the pass from the objective's output into lf.
  int start_kind;         // -1 output, 0 pre-activation of layer start_index, 1 x_t, 2 u_t, 3 p_t, 4 cost op start_index
  int start_t, start_index, start_dim, start_slot;
};

// K3/K4/K5 launch arguments (search.cu; built by host.cu).
struct SearchArgs {
  int n, d, rows, n_samp;        // rows = n_samp + 1 (incumbent row); GD: rows = n_samp = starts
  int method;                    // 0 CEM, 1 MPPI, 2 GD
  int groups, per_group;         // CEM agents / MPPI instances, samples per group
  int elites;
  int top_cap;
  int iter;
  const unsigned long long* seeds;  // [n] derived per-box seeds
  const float* lo;               // [n][d]
  const float* hi;
  const float* warm;             // [n][d] or null; NaN first coordinate = none
  float* mu;                     // [n][groups][d]
  float* var;                    // [n][groups][d] (CEM)
  float* var_floor;              // [n][d] (CEM)
  float* best;                   // [n][d]
  float* uf;                     // [n]
  float* actions;                // [n][rows][d]
  const float* costs;            // [n][rows]
  int* failed;                   // [n]
  float* top_val[2];             // [n][top_cap]
  int* top_seq[2];
  float* top_act[2];             // [n][top_cap][d]
  int* top_cnt;                  // [n]
  int cur;                       // which top buffer holds the current list
  // CEM
  float jitter, init_sigma;
  // MPPI
  float noise_frac, temperature;
  const float* noise_ratios;     // [n_noise]
  const float* temp_ratios;      // [n_temp]
  int n_noise;
  // GD (search.cpp:214-245)
  float gd_base_step;
  const float* gd_ratios;        // [gd_n_ratios], assigned round-robin over the starts
  int gd_n_ratios;
  const float* grad;             // [n][rows][d]
  // search_update sort keys in global memory ([n][P] 12-byte keys) when P keys do not fit the
  // opt-in shared memory (large samples_per_iter + top_capacity); null = shared memory
  void* sort_keys;
};

// Order-preserving float <-> int encoding for atomicMin/atomicMax extrema.
__device__ __forceinline__ int enc_f(float f) {
  int i = __float_as_int(f);
  return i ^ ((i >> 31) & 0x7fffffff);
}
__device__ __forceinline__ float dec_f(int i) { return __int_as_float(i ^ ((i >> 31) & 0x7fffffff)); }
inline int enc_f_host(float f) {
  int i;
  static_assert(sizeof(int) == sizeof(float), "");
  __builtin_memcpy(&i, &f, 4);
  return i ^ ((i >> 31) & 0x7fffffff);
}
inline float dec_f_host(int i) {
  i = i ^ ((i >> 31) & 0x7fffffff);
  float f;
  __builtin_memcpy(&f, &i, 4);
  return f;
}

// Philox4x32-10 counter-based generator.
struct Philox {
  __device__ static uint4 gen(uint4 ctr, uint2 key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint32_t hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
      const uint32_t hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
      ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
      key.x += 0x9E3779B9u;
      key.y += 0xBB67AE85u;
    }
    return ctr;
  }
};
__device__ __forceinline__ float u01_open(uint32_t x) {  // (0, 1]
  return (static_cast<float>(x >> 8) + 1.0f) * (1.0f / 16777216.0f);
}

}  // namespace bp

// rollout_tc3.cu -- K1 v3 on the 5th-generation tensor cores for MLPs with two hidden
// layers up to 512 wide and narrow ends (C5: [20, 512, 512, 16]): the fused H-step
// rollout (reference evaluate / forward_chunk, proj/src/graph.cpp:252-401, on the
// build_objective graph, model.cpp:310-387) with every Linear layer done by
// tcgen05.mma (kind::tf32, 3xTF32) into TMEM.
//
// Why a third kernel: a 512-wide layer's accumulator is 512 TMEM columns -- all of
// TMEM -- and its 512-wide A operand would need as much again, so v2's "two in-place
// regions" scheme cannot hold it.  v3 never materialises either in full:
//  * layer 1 (K = N0, N = N1) is computed in N chunks of <= 256 columns (J = 2 at
//    C5), each accumulated in a 256-column TMEM region D1;
//  * its A operand -- relu(layer 0) -- is RECOMPUTED per chunk, one 32-column K-block
//    at a time: layer 0's input is the step's features (ks + ka <= 32: a single
//    K-block X kept in TMEM for the whole step), so N-block kb of
//    layer 0 is 9 small MMAs (N = 32) into one of NS TMEM slots, converted in place
//    by the L0 epilogue into A K-block kb of layer 1.  Layer 0 is ~4 % of the step's
//    FLOPs, so computing it J times costs ~4 % more MMA work;
//  * layer 2 (K = N1, N = N2 <= 32) consumes each D1 chunk as soon as the epilogue has
//    converted it in place (relu + hi/lo split) and accumulates into D2 across chunks.
// TMEM: D1 [0, 256), X hi [256, 288), L0 slots hi / lo [288, 480), D2 [480, 496): layer 1's A
// operand keeps both 3xTF32 parts in TMEM (TS-only MMAs, no shared-memory operand traffic), so
// shared memory is left to the weight ring; three slots let L0(kb + 2) queue behind L1(kb) in
// the (in-order) tensor pipe, so its epilogue runs under L1(kb + 1).
//
// Per step and chunk j the MMA warp issues
//   L0(j, 0 .. NS-2), then for kb: L1(j, kb) [12 MMAs, N = chunk width], L0(j, kb+NS-1)
//   [into the slot L1(j, kb-1) just freed -- L1(j, kb) keeps the pipe busy meanwhile],
// then L0(j+1, 0 .. NS-2) and L2(j, c) per K-block c the D1 epilogue publishes.
// Weight blocks stream through a byte ring in exactly that order (producer warp,
// cp.async.bulk); every ring entry has its own full / empty barrier pair, so the
// producer never waits on a barrier phase that could already have moved on.
//
// Precision: 3xTF32 as v1 / v2 (split_tf32: hi = rna(x), lo = rna(x - hi); weights split
// on the host): D += A_hi.B_hi + A_lo.B_hi + A_hi.B_lo, FP32 accumulation in TMEM; per
// row a fixed order of operations, so results are batch-decomposition invariant
// (graph.hpp:102-103).
//
// Warps (15, one 128-row tile per CTA; warp w reaches TMEM lanes 32 (w % 4) .. + 31):
//   0-3   L0 epilogue: layer-0 N-blocks -> layer-1 A K-blocks (+ layer-0 extrema)
//   4-11  D1 epilogue: two per quadrant, K-blocks c = h, h + 2, ... of each chunk (+ layer-1
//         extrema); warps 4-7 also turn D2 into x_t (cost scratch, x_t extrema) and the next
//         step's features X
//   12    MMA issuer (whole warp, elect.sync inside the asm)
//   13    producer (weight blocks)
//   14    cost warp: the cost program (4 rows per thread), states, scratch-column extrema
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "rollout_common.cuh"
#include "tc_common.cuh"
#include "tc_epilogue.cuh"

namespace bp {

namespace {

using namespace tc;

constexpr int kNS = 3;              // L0 output slots (layer-1 A K-blocks in flight)
constexpr int kRing = 16;           // ring entries in flight (full / empty barrier pairs)
constexpr int kWarps = 15;
constexpr int kThreads3 = 32 * kWarps;
constexpr int kMmaWarp = 12, kProducerWarp = 13, kCostWarp = 14;
// TMEM columns: D1 | X hi | L0 slot s hi, lo (s < kNS) | D2
constexpr uint32_t kColD1 = 0, kColXh = 256, kColL0 = 288, kColD2 = 480;
__device__ __forceinline__ uint32_t col_l0h(int s) { return kColL0 + 64u * s; }
__device__ __forceinline__ uint32_t col_l0l(int s) { return kColL0 + 64u * s + 32u; }
constexpr uint32_t kTmemCols = 512;
#ifndef BP_TC3_FEATURES_FIRST
#define BP_TC3_FEATURES_FIRST 1
#endif
#ifndef BP_TC3_SLEEP_EPI
#define BP_TC3_SLEEP_EPI 64
#endif
#ifndef BP_TC3_SLEEP_COST
#define BP_TC3_SLEEP_COST 128
#endif
constexpr uint32_t kSleepProducer = 0, kSleepCost = BP_TC3_SLEEP_COST, kSleepEpi = BP_TC3_SLEEP_EPI;  // producer: no __nanosleep (a 256 ns back-off delayed every ring refill by ~0.5k cycles)

// Debug timeline (compiled in with -DBP_TC_TIMELINE; tools/tc_timeline.py c5): clock64 marks of
// CTA 0 at step 3 -- MMA warp 0 (step start), 1000 + 64 j + 4 kb + {0 before / 1 after the A
// K-block wait, 2 / 3 weight hi / lo landed}, 1200 + j (D1 commit), 1300 + 16 j + 2 c + {0, 1}
// (layer-2 A wait); L0 epilogue 2000 + 64 j + 2 kb + {0 slot full, 1 published}; D1 epilogue
// 3000 + 32 j + 2 c + {0, 1}, 3100 + j (D1 full seen), 3200 / 3201 (D2 seen / X published).
#ifdef BP_TC_TIMELINE
__device__ __forceinline__ void mark3(const RolloutArgs& a, int t, int slot) {
  if (a.timeline != nullptr && blockIdx.x == 0 && t == 3 && (threadIdx.x & 31) == 0) a.timeline[slot] = clock64();
}
#else
__device__ __forceinline__ void mark3(const RolloutArgs&, int, int) {}
#endif

struct Tc3Smem {
  unsigned char* xlo;    // features lo K-block (128 rows x 128 B, SW128)
  unsigned char* a2lo;   // [2] layer-2 A lo K-blocks
  unsigned char* w;      // weight byte ring
  float* sc;             // [128][tc_S] per-row scratch of the cost warp (x_t written by the x epilogue)
  float* bias;           // b0 [np0], b1 [np1], b2 [np2]
  float* cconst;         // cost-op constants, arena range [cost_f0, cost_f1)
  FwdOp* ops;            // [n_ops]
  int* segl;             // [128] tile-local subdomain of each row (-1 past the last)
  int* pairs;            // [n_sc][2] recorded scratch columns (column, record offset)
  uint64_t* full;        // [kRing] ring entry landed
  uint64_t* peer_full;   // [kRing] CTA pair, rank 0: the peer's half of the entry landed (relayed)
  uint64_t* empty;       // [kRing] ring entry read by its MMAs (commit)
  uint64_t* l0_full;     // [kNS] layer-0 N-block in slot s complete
  uint64_t* a1_ready;    // [kNS] layer-1 A K-block in slot s written (4 quadrant warps)
  uint64_t* d1_full;     // D1 chunk complete
  uint64_t* a2_ready;    // [2] layer-2 A K-block written into slot h (4 quadrant warps)
  uint64_t* a2_free;     // [2] layer-2 MMAs of slot h retired (commit)
  uint64_t* d2_full;     // D2 (the step's output layer) complete
  uint64_t* x_ready;     // features X of the next step written (4 warps)
  uint64_t* x_full;      // x_t of every row in the scratch (4 warps)
  uint64_t* x_empty;     // the cost warp consumed the scratch of the step
  uint32_t* tmem_slot;
  uint32_t* ring;        // [kRing] x 8 B producer bookkeeping: virtual start of each in-flight entry
  size_t bytes;
};

__host__ __device__ inline Tc3Smem carve3(const DevObjective& o, unsigned char* base) {
  Tc3Smem m;
  size_t off = 0;
  auto take = [&](size_t n, size_t align) {
    off = (off + align - 1) & ~(align - 1);
    unsigned char* p = base + off;
    off += n;
    return p;
  };
  m.xlo = take(16384, 1024);
  m.a2lo = take(2 * 16384, 1024);
  m.w = take(static_cast<size_t>(o.tc3_ring), 1024);
  m.sc = reinterpret_cast<float*>(take(sizeof(float) * 128 * o.tc_S, 16));
  m.bias = reinterpret_cast<float*>(take(sizeof(float) * (o.tc3_np[0] + o.tc3_np[1] + o.tc3_np[2]), 16));
  m.cconst = reinterpret_cast<float*>(take(sizeof(float) * (o.cost_f1 - o.cost_f0), 16));
  m.ops = reinterpret_cast<FwdOp*>(take(sizeof(FwdOp) * o.n_ops, 16));
  m.segl = reinterpret_cast<int*>(take(sizeof(int) * 128, 16));
  m.pairs = reinterpret_cast<int*>(take(sizeof(int) * 2 * o.n_sc, 16));
  uint64_t* b = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * (3 * kRing + 2 * kNS + 2 * 2 + 6), 16));
  m.full = b;
  m.peer_full = m.full + kRing;
  m.empty = m.peer_full + kRing;
  m.l0_full = m.empty + kRing;
  m.a1_ready = m.l0_full + kNS;
  m.a2_ready = m.a1_ready + kNS;
  m.a2_free = m.a2_ready + 2;
  m.d1_full = m.a2_free + 2;
  m.d2_full = m.d1_full + 1;
  m.x_ready = m.d2_full + 1;
  m.x_full = m.x_ready + 1;
  m.x_empty = m.x_full + 1;
  m.tmem_slot = reinterpret_cast<uint32_t*>(take(16, 16));
  m.ring = reinterpret_cast<uint32_t*>(take(sizeof(unsigned long long) * kRing, 16));
  m.bytes = off;
  return m;
}

__host__ inline size_t tc3_fixed_bytes(DevObjective o) {
  o.tc3_ring = 0;
  return 1024 + carve3(o, nullptr).bytes + 1024;
}

// The weight stream, in the MMA warp's consumption order.  Entry kinds: layer-0 N-block
// (rows 32, the image's block kb), layer-1 block (chunk j, K-block kb: the chunk's rows),
// layer-2 K-block (np2 rows); each as a hi entry then a lo entry.
struct W3 {
  const float* src;
  uint32_t bytes;
};
// CTA pair (half = 1): each CTA streams rows [rank R/2, (rank + 1) R/2) of every block (the
// cta_group::2 B operand: N/2 rows in each CTA's shared memory at the same offset).
__device__ __forceinline__ W3 half_of(const float* part_base, int rows, int half, uint32_t rank) {
  const int r = rows >> half;
  return {part_base + static_cast<size_t>(rank) * r * 32, static_cast<uint32_t>(r) * 128u};
}
__device__ __forceinline__ W3 w0_entry(const DevObjective& o, int kb, int part, int half = 0, uint32_t rank = 0) {
  return half_of(o.f + o.tc3_w[0] + (static_cast<size_t>(kb) * 2 + part) * 32 * 32, 32, half, rank);
}
__device__ __forceinline__ int chunk_w(const DevObjective& o, int j) { return min(256, o.tc3_np[1] - 256 * j); }
__device__ __forceinline__ W3 w1_entry(const DevObjective& o, int j, int kb, int part, int half = 0, uint32_t rank = 0) {
  // image: per chunk j, per K-block kb: [hi: cw rows x 32][lo: cw rows x 32]
  const int cw = chunk_w(o, j);
  const size_t base = static_cast<size_t>(2 * 256) * j * o.tc3_np[0];  // earlier chunks: 256 rows x K, hi and lo
  return half_of(o.f + o.tc3_w[1] + base + (static_cast<size_t>(kb) * 2 + part) * cw * 32, cw, half, rank);
}
__device__ __forceinline__ W3 w2_entry(const DevObjective& o, int kb, int part, int half = 0, uint32_t rank = 0) {
  return half_of(o.f + o.tc3_w[2] + (static_cast<size_t>(kb) * 2 + part) * o.tc3_np[2] * 32, o.tc3_np[2], half, rank);
}

// Weight-stream groups of one step (the producer's sequence, counted by the pair's relay).
__device__ __forceinline__ int groups_per_step(const DevObjective& o, int KB1, int J) {
  int n = 0;
  for (int j = 0; j < J; ++j) {
    if (j == 0) n += min(kNS - 1, KB1);
    n += KB1;
    if (j + 1 < J) n += min(kNS - 1, KB1);
    n += chunk_w(o, j) / 32;
  }
  return n;
}

template <bool PAIR>  // PAIR: cluster of two CTAs (two 128-row tiles), rank 0 issues cta_group::2 MMAs (M = 256)
__global__ void __launch_bounds__(kThreads3, 1) rollout_tc3_kernel(const DevObjective o, const RolloutArgs a) {
  extern __shared__ unsigned char smraw[];
  const uint32_t s0 = smem_u32(smraw);
  const Tc3Smem m = carve3(o, smraw + (((s0 + 1023u) & ~1023u) - s0));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long row0 = static_cast<long long>(blockIdx.x) * 128;
  const int ks = o.ks, ka = o.ka, kd = o.kd, d = o.d, S = o.tc_S, H = o.H;
  const long long rps = a.rows_per_sub;
  const int np0 = o.tc3_np[0], np1 = o.tc3_np[1], np2 = o.tc3_np[2];
  const int KB1 = np0 / 32;               // layer-0 N-blocks = layer-1 K-blocks
  const int J = (np1 + 255) / 256;        // layer-1 N chunks
  const int k0q = o.tc3_k0steps;          // k-steps of 8 of the features
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  constexpr int kHalf = PAIR ? 1 : 0;     // each CTA of a pair streams half of every weight block's rows

  if (a.failed != nullptr) {  // skip tiles (pairs) whose subdomains all failed already
    const long long g0 = PAIR ? row0 - static_cast<long long>(rank) * 128 : row0;
    const long long last = min(a.n_rows, g0 + (PAIR ? 256 : 128)) - 1;
    bool all_failed = last >= g0;
    for (long long s = g0 / rps; s <= last / rps && all_failed; ++s) all_failed = a.failed[s] != 0;
    if (all_failed) return;
  }

  for (int i = tid; i < 128; i += kThreads3) {
    const long long r = row0 + i;
    m.segl[i] = r < a.n_rows ? static_cast<int>(r / rps - row0 / rps) : -1;
  }
  for (int i = tid; i < 128 * S; i += kThreads3) m.sc[i] = 0.f;
  for (int i = tid; i < np0 + np1 + np2; i += kThreads3) m.bias[i] = o.f[o.tc3_bias + i];
  for (int i = tid; i < o.n_ops; i += kThreads3) m.ops[i] = to_fwd(o.ops[i]);
  for (int i = tid; i < 2 * o.n_sc; i += kThreads3) m.pairs[i] = o.iv[o.sc_list + i];
  for (int i = tid; i < o.cost_f1 - o.cost_f0; i += kThreads3) m.cconst[i] = o.f[o.cost_f0 + i];
  if (tid == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(m.full + s, 1);
      mbar_init(m.peer_full + s, 1);
      mbar_init(m.empty + s, 1);
    }
    // operand-ready barriers count the quadrant warps of both CTAs of a pair (rank 0's MMA warp waits)
    constexpr uint32_t kQ = PAIR ? 8 : 4;
    for (int s = 0; s < kNS; ++s) {
      mbar_init(m.l0_full + s, 1);
      mbar_init(m.a1_ready + s, kQ);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(m.a2_ready + h, kQ);
      mbar_init(m.a2_free + h, 1);
    }
    mbar_init(m.d1_full, 1);
    mbar_init(m.d2_full, 1);
    mbar_init(m.x_ready, kQ);
    mbar_init(m.x_full, 4);
    mbar_init(m.x_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(m.tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(m.tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // both CTAs' barriers initialised before any remote arrive
  fence_after();
  const uint32_t tmem = *m.tmem_slot;
  const uint32_t ring_bytes = static_cast<uint32_t>(o.tc3_ring);

  // The weight stream is cut into GROUPS, one per MMA-warp step, each with one full / empty barrier
  // pair: a layer-1 K-block (W1 hi, lo) together with the layer-0 N-block issued after it (W0 hi,
  // lo), a layer-0 prologue, a layer-2 K-block.  One wait and one commit per group keep the MMA
  // warp's bookkeeping between its bursts short (per-entry barriers cost ~1k cycles per K-block).
  if (warp == kProducerWarp) {
    // ------------------------------------------------ producer: the weight stream
    if (lane == 0) {
      // Ring bookkeeping on a virtual byte counter: wrapping to 0 skips the tail (counted as
      // used), so virtual byte v lives at physical v mod ring and a group occupies the virtual
      // range [vstart, vpos).  A new group ending at vpos overwrites exactly the bytes of groups
      // that start before vpos - ring (the previous lap); groups retire in order, so the producer
      // waits for the oldest in-flight groups while they start in the previous lap (or hold the
      // barrier slot).  O(1) per group.
      uint32_t pos = 0;
      unsigned long long vpos = 0;
      unsigned long long* vstart_b = reinterpret_cast<unsigned long long*>(m.ring);  // [kRing]
      int g = 0, head = 0;
      int tcur = 0, gcur = 0;  // timeline: step and group index within the step
      W3 ent[4];
      uint32_t at[4];
      auto put_group = [&](int n) {
        if (gcur < 60) mark3(a, tcur, 3300 + 3 * gcur);
        unsigned long long vs = 0;  // virtual start of the group's first entry
        uint32_t bytes = 0;
        for (int i = 0; i < n; ++i) {
          if (pos + ent[i].bytes > ring_bytes) {
            vpos += ring_bytes - pos;
            pos = 0;
          }
          if (i == 0) vs = vpos;
          at[i] = pos;
          pos += ent[i].bytes;
          vpos += ent[i].bytes;
          bytes += ent[i].bytes;
        }
        while (head < g && (vstart_b[head % kRing] + ring_bytes < vpos || g - head >= kRing)) {
          mbar_wait(m.empty + head % kRing, static_cast<uint32_t>((head / kRing) & 1), kSleepProducer);
          ++head;
        }
        const int sl = g % kRing;
        vstart_b[sl] = vs;
        if (gcur < 60) mark3(a, tcur, 3301 + 3 * gcur);
#ifdef BP_TC3_WEIGHTS_ONCE  // timing-only experiment: no weight traffic after step 0 (wrong results)
        if (tcur > 0) {
          mbar_arrive(m.full + sl);
          ++gcur;
          ++g;
          return;
        }
#endif
        if (PAIR && o.tmaps != nullptr) {  // both CTAs' halves complete on rank 0's barrier
          if (rank == 0) mbar_expect_tx(m.full + sl, 2u * bytes);
          for (int i = 0; i < n; ++i)
            tma_rows_to_rank0(m.w + at[i], tmap_rows(o, static_cast<int>(ent[i].bytes / 128u)),
                              static_cast<int>((ent[i].src - o.f) / 32), m.full + sl);
        } else {
          mbar_expect_tx(m.full + sl, bytes);
          for (int i = 0; i < n; ++i) bulk_g2s(m.w + at[i], ent[i].src, ent[i].bytes, m.full + sl);
        }
        if (gcur < 60) mark3(a, tcur, 3302 + 3 * gcur);
        ++gcur;
        ++g;
      };
      for (int t = 0; t < H; ++t)
        for (int j = 0; j < J; ++j) {
          tcur = t;
          if (j == 0) gcur = 0;
          if (j == 0)
            for (int q = 0; q < kNS - 1 && q < KB1; ++q) {
              ent[0] = w0_entry(o, q, 0, kHalf, rank);
              ent[1] = w0_entry(o, q, 1, kHalf, rank);
              put_group(2);
            }
          for (int kb = 0; kb < KB1; ++kb) {
            ent[0] = w1_entry(o, j, kb, 0, kHalf, rank);
            ent[1] = w1_entry(o, j, kb, 1, kHalf, rank);
            const int nk = kb + kNS - 1;
            if (nk < KB1) {
              ent[2] = w0_entry(o, nk, 0, kHalf, rank);
              ent[3] = w0_entry(o, nk, 1, kHalf, rank);
            }
            put_group(nk < KB1 ? 4 : 2);
          }
          if (j + 1 < J)
            for (int q = 0; q < kNS - 1 && q < KB1; ++q) {
              ent[0] = w0_entry(o, q, 0, kHalf, rank);
              ent[1] = w0_entry(o, q, 1, kHalf, rank);
              put_group(2);
            }
          const int kb2 = chunk_w(o, j) / 32;
          for (int c = 0; c < kb2; ++c) {
            ent[0] = w2_entry(o, 8 * j + c, 0, kHalf, rank);
            ent[1] = w2_entry(o, 8 * j + c, 1, kHalf, rank);
            put_group(2);
          }
        }
    }
  } else if (warp == kMmaWarp && PAIR && rank == 1) {
    // ------------------------------------------------ CTA pair, rank 1: relay "my half of group g
    // landed" to rank 0, which issues the MMAs over both halves (nothing to relay when the halves
    // arrive by tensor-map TMA completing on rank 0's barriers)
    const int n_g = o.tmaps != nullptr ? 0 : H * groups_per_step(o, KB1, J);
    for (int gi = 0; gi < n_g; ++gi) {
      mbar_wait_warp(m.full + gi % kRing, static_cast<uint32_t>((gi / kRing) & 1));
      if (lane == 0) mbar_arrive_cta(m.peer_full + gi % kRing, 0);
      __syncwarp();
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------ MMA issuer (whole warp; elect.sync inside); a
    // CTA pair's rank 0 issues cta_group::2 MMAs over both CTAs' rows and both halves of B
    int g = 0;
    uint32_t pos = 0;
    const uint32_t wbase = smem_u32(m.w);
    int slot_grp[kNS];  // per L0 slot: the group whose commit follows the slot's last layer-1 use (-1 none)
    for (int q = 0; q < kNS; ++q) slot_grp[q] = -1;
    int l0_rdy[kNS] = {};  // per slot: a1_ready completions waited
    int a2_rdy[2] = {};
    int a2_last = -1;  // group committed after the last layer-2 K-block (D1 is free once it retired)
    auto idesc = [&](int n) { return PAIR ? tf32_idesc_mn(256, n) : tf32_idesc(n); };
    const uint32_t id0 = idesc(32), id2 = idesc(np2);
    // commits arrive in both CTAs of a pair; operand-ready barriers collect both CTAs' warps
    auto commit = [&](uint64_t* bar) {
      if constexpr (PAIR)
        commit_pair_elect(bar);
      else
        mma_commit_elect(bar);
    };
    auto wait_ready = [&](uint64_t* bar, uint32_t parity) {
      if constexpr (PAIR)
        mbar_wait_cluster(bar, parity);
      else
        mbar_wait_warp(bar, parity);
    };
    auto wait_group_retired = [&](int gi) {  // the MMAs issued before group gi's commit retired
      if (gi >= 0) mbar_wait_warp(m.empty + gi % kRing, static_cast<uint32_t>((gi / kRing) & 1));
    };
    // the next group of n entries of `rows` rows each (this CTA's half for a pair): wait until it
    // (and the peer's half) landed; descriptors in b[]; released by a commit after its MMAs
    uint64_t b[4];
    auto take_group = [&](int n, const uint32_t* rows) {
      for (int i = 0; i < n; ++i) b[i] = sw128_desc(wbase + ring_place(pos, (rows[i] >> kHalf) * 128u, ring_bytes));
      mbar_wait_warp(m.full + g % kRing, static_cast<uint32_t>((g / kRing) & 1));
      if constexpr (PAIR)
        if (o.tmaps == nullptr) mbar_wait_cluster(m.peer_full + g % kRing, static_cast<uint32_t>((g / kRing) & 1));
      fence_after();
    };
    auto release_group = [&]() {
      commit(m.empty + g % kRing);
      ++g;
    };
    auto tt_bhi = [&](uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint32_t id, uint32_t acc, int nq) {
      if constexpr (PAIR)
        mma_tt_bhi2(d, ah, al, bh, id, acc, nq);
      else
        mma_tt_bhi(d, ah, al, bh, id, acc, nq);
    };
    auto tt_blo = [&](uint32_t d, uint32_t ah, uint64_t bl, uint32_t id, int nq) {
      if constexpr (PAIR)
        mma_tt_blo2(d, ah, bl, id, nq);
      else
        mma_tt_blo(d, ah, bl, id, nq);
    };
    // A hi in TMEM, A lo in shared memory: TS/SS pairs on B_hi, then TS on B_lo
    auto ts_pair = [&](uint32_t d, uint32_t ah, uint64_t al, uint64_t bh, uint32_t id, uint32_t acc) {
      if constexpr (PAIR)
        mma_pair2_elect(d, ah, al, bh, id, acc);
      else
        mma_pair_elect(d, ah, al, bh, id, acc);
    };
    auto ts_one = [&](uint32_t d, uint32_t ah, uint64_t bl, uint32_t id) {
      if constexpr (PAIR)
        mma_ts2(d, ah, bl, id, 1u);
      else
        mma_ts(d, ah, bl, id, 1u);
    };
    // layer-0 N-block kb into slot kb % kNS with the W0 descriptors bh / bl (after the slot's
    // previous layer-1 MMAs retired)
    const uint64_t x_lo = sw128_desc(smem_u32(m.xlo));
    auto l0_mmas = [&](int kb, uint64_t bh, uint64_t bl) {
      const int s = kb % kNS;
      wait_group_retired(slot_grp[s]);
      const uint32_t d = tmem + col_l0h(s);
      for (int q = 0; q < k0q; ++q) ts_pair(d, tmem + kColXh + 8 * q, x_lo + 2 * q, bh + 2 * q, id0, q != 0 ? 1u : 0u);
      for (int q = 0; q < k0q; ++q) ts_one(d, tmem + kColXh + 8 * q, bl + 2 * q, id0);
      commit(m.l0_full + s);
    };
    const uint32_t rows_w0[2] = {32u, 32u};
    const uint32_t rows_w2[2] = {static_cast<uint32_t>(np2), static_cast<uint32_t>(np2)};
    auto l0_prologue = [&]() {
      for (int q = 0; q < kNS - 1 && q < KB1; ++q) {
        take_group(2, rows_w0);
        l0_mmas(q, b[0], b[1]);
        release_group();
      }
    };
    for (int t = 0; t < H; ++t) {
      wait_ready(m.x_ready, static_cast<uint32_t>(t & 1));  // the step's features X written
      fence_after();
      mark3(a, t, 0);
      for (int j = 0; j < J; ++j) {
        const int cw = chunk_w(o, j);
        const uint32_t id1 = idesc(cw);
        const uint32_t rows_g[4] = {static_cast<uint32_t>(cw), static_cast<uint32_t>(cw), 32u, 32u};
        if (j == 0) l0_prologue();
        for (int kb = 0; kb < KB1; ++kb) {
          const int s = kb % kNS;
          const int nk = kb + kNS - 1;
          if (kb == 0 && j > 0) wait_group_retired(a2_last);  // chunk j-1's layer-2 MMAs read D1 in place
          mark3(a, t, 1000 + 64 * j + 4 * kb);
          wait_ready(m.a1_ready + s, static_cast<uint32_t>(l0_rdy[s] & 1));
          ++l0_rdy[s];
          fence_after();
          mark3(a, t, 1001 + 64 * j + 4 * kb);
          take_group(nk < KB1 ? 4 : 2, rows_g);
          mark3(a, t, 1002 + 64 * j + 4 * kb);
          tt_bhi(tmem + kColD1, tmem + col_l0h(s), tmem + col_l0l(s), b[0], id1, kb > 0 ? 1u : 0u, 4);
          tt_blo(tmem + kColD1, tmem + col_l0h(s), b[1], id1, 4);
          if (nk < KB1) l0_mmas(nk, b[2], b[3]);
          slot_grp[s] = g;  // this group's commit follows L1(kb), the last use of slot s
          release_group();
          mark3(a, t, 1003 + 64 * j + 4 * kb);
        }
        commit(m.d1_full);
        mark3(a, t, 1200 + j);
        if (j + 1 < J) l0_prologue();
        const int kb2 = cw / 32;
        for (int c = 0; c < kb2; ++c) {
          const int h = c & 1;
          mark3(a, t, 1300 + 16 * j + 2 * c);
          wait_ready(m.a2_ready + h, static_cast<uint32_t>(a2_rdy[h] & 1));
          ++a2_rdy[h];
          fence_after();
          mark3(a, t, 1301 + 16 * j + 2 * c);
          // A2 hi in TMEM (D1 in place), lo in shared memory
          const uint32_t ah = tmem + kColD1 + 32 * c;
          const uint64_t al = sw128_desc(smem_u32(m.a2lo) + h * 16384u);
          take_group(2, rows_w2);
          for (int q = 0; q < 4; ++q)
            ts_pair(tmem + kColD2, ah + 8 * q, al + 2 * q, b[0] + 2 * q, id2, ((j | c) != 0 || q != 0) ? 1u : 0u);
          for (int q = 0; q < 4; ++q) ts_one(tmem + kColD2, ah + 8 * q, b[1] + 2 * q, id2);
          commit(m.a2_free + h);
          a2_last = g;
          release_group();
        }
      }
      commit(m.d2_full);
    }
  } else if (warp == kCostWarp) {
    // ------------------------------------------------ cost warp: 4 rows per thread
    constexpr int NR = 4;
    const long long rem = a.n_rows - row0;
    const int nvalid = static_cast<int>(rem < 0 ? 0 : rem < 128 ? rem : 128);
    const long long seg0 = row0 / rps;
    const long long SPH = static_cast<long long>(o.SP) * H;
    const bool rec_any = a.stat_min != nullptr;
    int rr[NR];
    float* rows[NR];
    float cost[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      rr[q] = 32 * q + lane;
      rows[q] = m.sc + rr[q] * S;
      cost[q] = 0.f;
      for (int e = 0; e < kd; ++e) rows[q][o.pcol + e] = o.f[o.p0 + e];
    }
    const int k_first = o.x_stat >= 0 ? ks : 0;  // the x_t columns' extrema come from the x epilogue
    const long long b1 = (seg0 + 1) * rps - row0;
    const int bnd = static_cast<int>(b1 < nvalid ? b1 : nvalid);
    const bool two = nvalid == 0 || (row0 + nvalid - 1) / rps - seg0 <= 1;
    for (int t = 0; t < H; ++t) {
      mbar_wait(m.x_full, static_cast<uint32_t>(t & 1), kSleepCost);
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int r = rr[q];
        const float* ur = a.actions + (row0 + r) * d + t * ka;
        for (int j = 0; j < ka; ++j) {
          const float u = r < nvalid ? __ldg(ur + j) : 0.f;
          rows[q][o.ucol + j] = u;
          if (j < kd) rows[q][o.pcol + j] += u;
        }
      }
      cost_program_n<NR>(o, m.ops, m.cconst - o.cost_f0, rows, t, cost);
      if (a.states != nullptr)
#pragma unroll
        for (int q = 0; q < NR; ++q)
          if (rr[q] < nvalid)
            for (int j = 0; j < ks; ++j) a.states[((row0 + rr[q]) * H + t) * ks + j] = rows[q][j];
      if (rec_any) {
        __syncwarp();
        for (int k = k_first + lane; k < o.n_sc; k += 32)
          scratch_column_extrema(a, m.sc + m.pairs[2 * k], S, two, bnd, nvalid, m.segl, seg0, SPH,
                                 t * o.SP + m.pairs[2 * k + 1]);
      }
      mbar_arrive_warp(m.x_empty);
    }
#pragma unroll
    for (int q = 0; q < NR; ++q)
      if (rr[q] < nvalid) {
        const long long r = row0 + rr[q];
        a.costs[r] = cost[q];
        if (a.failed != nullptr && !isfinite(cost[q])) atomicOr(a.failed + r / rps, 1);
      }
  } else if (warp < kMmaWarp) {
    // ------------------------------------------------ epilogue warps
    const int g = warp & 3;
    const int row = 32 * g + lane;
    const long long grow = row0 + row;
    const bool row_ok = grow < a.n_rows;
    const uint32_t tl = tmem + (static_cast<uint32_t>(32 * g) << 16);
    const long long wr0 = row0 + 32 * g;
    const long long wr1 = min(wr0 + 31, a.n_rows - 1);
    const long long ws0 = wr0 / rps, ws1 = wr1 >= wr0 ? wr1 / rps : ws0 - 1;
    const bool simple = ws0 == ws1 && wr0 + 31 < a.n_rows;
    const long long SPH = static_cast<long long>(o.SP) * H;
    if (warp < 4) {
      // -------------------------------------------- L0 epilogue: layer-0 N-block kb in slot s ->
      // layer-1 A K-block kb (relu, hi / lo), layer-0 pre-activation extrema on chunk 0
      const bool rec = o.relu[0] != 0 && o.pre_stat[0] >= 0 && a.stat_min != nullptr;
      const int N0 = o.widths[1];
      int l0_done[kNS] = {};
      for (int t = 0; t < H; ++t)
        for (int j = 0; j < J; ++j)
          for (int kb = 0; kb < KB1; ++kb) {
            const int s = kb % kNS;
            mbar_wait(m.l0_full + s, static_cast<uint32_t>(l0_done[s] & 1), kSleepEpi);
            ++l0_done[s];
            fence_after();
            if (warp == 0) mark3(a, t, 2000 + 64 * j + 2 * kb);
            float v[32];
            tmem_ld32(tl + col_l0h(s), v);
            const float4* b4 = reinterpret_cast<const float4*>(m.bias + kb * 32);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 bb = b4[q];
              v[4 * q] += bb.x;
              v[4 * q + 1] += bb.y;
              v[4 * q + 2] += bb.z;
              v[4 * q + 3] += bb.w;
            }
            {
              float w[32];
#pragma unroll
              for (int q = 0; q < 32; ++q) w[q] = fmaxf(v[q], 0.f);
              store_operand_tt(tl + col_l0h(s), tl + col_l0l(s), w);
              publish_chunk(m.a1_ready + s, PAIR);
              if (warp == 0) mark3(a, t, 2001 + 64 * j + 2 * kb);
            }
            if (rec && j == 0) {
              const int col = kb * 32 + lane;
              warp_chunk_extrema(a, v, simple, ws0, ws1, row_ok, grow, rps, SPH,
                                 static_cast<long long>(t) * o.SP + o.pre_stat[0] + col, col, N0);
            }
          }
    } else {
      // -------------------------------------------- D1 epilogue (K-blocks c = h, h + 2, ...) and, on
      // warps 4-7, the output layer: x_t and the next step's features
      const int h = (warp - 4) >> 2;
      const bool xw = h == 0;
      const bool rec = o.relu[1] != 0 && o.pre_stat[1] >= 0 && a.stat_min != nullptr;
      const bool x_rec = o.x_stat >= 0 && a.stat_min != nullptr;
      const int N1 = o.widths[2];
      const float* urow = row_ok ? a.actions + grow * d : nullptr;
      float* scrow = m.sc + row * S;
      float pe[8], u_nxt[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        pe[e] = e < kd ? o.f[o.p0 + e] : 0.f;
        u_nxt[e] = (row_ok && e < ka) ? __ldg(urow + e) : 0.f;  // u_0
      }
      // features concat(x [- tile(p)], u_{t+1}) of this row -> X (one K-block): v holds x
      // in the columns below ks and zeros above
      auto features_store = [&](float (&v)[32]) {
        if (o.rel) {
          int km = 0;
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            float pv = pe[0];
#pragma unroll
            for (int e = 1; e < 8; ++e) pv = km == e ? pe[e] : pv;
            if (q < ks) v[q] -= pv;
            km = km + 1 == kd ? 0 : km + 1;
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e)
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (e < ka && q == ks + e) v[q] = u_nxt[e];
        store_operand(tl + kColXh, m.xlo, row, v);
        publish_chunk(m.x_ready, PAIR);
      };
      if (xw) {  // features of step 0
        float v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = q < ks ? o.f[o.x0 + min(q, ks - 1)] : 0.f;
        features_store(v);
      }
      int a2_writes = 0;  // uses of A2 slot h so far
      for (int t = 0; t < H; ++t) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e < kd && e < ka) pe[e] += u_nxt[e];  // p_t = p_{t-1} + u_t
          u_nxt[e] = (row_ok && e < ka && t + 1 < H) ? __ldg(urow + (t + 1) * ka + e) : 0.f;  // u_{t+1}
        }
        for (int j = 0; j < J; ++j) {
          mbar_wait(m.d1_full, static_cast<uint32_t>((t * J + j) & 1), kSleepEpi);
          fence_after();
          if (warp == 4) mark3(a, t, 3100 + j);
          const int kb2 = chunk_w(o, j) / 32;
          for (int c = h; c < kb2; c += 2) {
            if (a2_writes > 0) mbar_wait(m.a2_free + h, static_cast<uint32_t>((a2_writes - 1) & 1), kSleepEpi);
            ++a2_writes;
            float v[32];
            tmem_ld32(tl + kColD1 + 32 * c, v);
            const float4* b4 = reinterpret_cast<const float4*>(m.bias + np0 + 256 * j + 32 * c);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 bb = b4[q];
              v[4 * q] += bb.x;
              v[4 * q + 1] += bb.y;
              v[4 * q + 2] += bb.z;
              v[4 * q + 3] += bb.w;
            }
            {
              float w[32];
#pragma unroll
              for (int q = 0; q < 32; ++q) w[q] = fmaxf(v[q], 0.f);
              store_operand(tl + kColD1 + 32 * c, m.a2lo + h * 16384, row, w);
              publish_chunk(m.a2_ready + h, PAIR);
              if (warp == 4 || warp == 8) mark3(a, t, 3001 + 32 * j + 2 * c);
            }
            if (rec) {
              const int col = 256 * j + 32 * c + lane;
              warp_chunk_extrema(a, v, simple, ws0, ws1, row_ok, grow, rps, SPH,
                                 static_cast<long long>(t) * o.SP + o.pre_stat[1] + col, col, N1);
            }
          }
        }
        mbar_wait(m.d2_full, static_cast<uint32_t>(t & 1), kSleepEpi);
        fence_after();
        if (warp == 4) mark3(a, t, 3200);
        if (xw) {
          float v[32];
          if (np2 > 16)
            tmem_ld32(tl + kColD2, v);
          else
            tmem_ld16(tl + kColD2, v);
          const float* b2 = m.bias + np0 + np1;
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = q < np2 ? v[q] + b2[q] : 0.f;
          if (BP_TC3_FEATURES_FIRST && t + 1 < H) {  // the next step's layer 0 waits on these first
            float f[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) f[q] = q < ks ? v[q] : 0.f;
            features_store(f);
          }
          if (t >= 1) mbar_wait(m.x_empty, static_cast<uint32_t>((t - 1) & 1), kSleepEpi);
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (q < ks) scrow[q] = v[q];
          if (x_rec)
            warp_chunk_extrema(a, v, simple, ws0, ws1, row_ok, grow, rps, SPH,
                               static_cast<long long>(t) * o.SP + o.x_stat + lane, lane, ks);
          mbar_arrive_warp(m.x_full);
          if (!BP_TC3_FEATURES_FIRST && t + 1 < H) {
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (q >= ks) v[q] = 0.f;
            features_store(v);
          }
        }
      }
    }
  }

  fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // both CTAs done with the pair's TMEM
  if (warp == 0) {
    fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

}  // namespace

size_t rollout_tc3_fixed_smem(const DevObjective& o) { return tc3_fixed_bytes(o); }
size_t rollout_tc3_smem(const DevObjective& o) { return 1024 + carve3(o, nullptr).bytes; }

cudaError_t launch_rollout_tc3(const DevObjective& o, const RolloutArgs& a, cudaStream_t st) {
  const size_t smem = rollout_tc3_smem(o);
  const long long grid = (a.n_rows + 127) / 128;
  if (grid <= 0) return cudaSuccess;
  // One CTA per tile by default; BP_TC3_PAIR=1 runs CTA pairs (clusters of two, cta_group::2:
  // each CTA streams half of every weight block -- the same results bit for bit).  Measured on
  // C5: pair 157 vs one CTA 164 TFLOP/s, with or without the relay of the peer's weight halves
  // (tensor-map TMA completing on rank 0's barriers): the cross-CTA operand hand-offs pace it.
  const char* env = std::getenv("BP_TC3_PAIR");
  const bool pair = env != nullptr && env[0] == '1';
  if (!pair) {
    cudaError_t e = cudaFuncSetAttribute(rollout_tc3_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    rollout_tc3_kernel<false><<<static_cast<unsigned>(grid), kThreads3, smem, st>>>(o, a);
    return cudaGetLastError();
  }
  cudaError_t e = cudaFuncSetAttribute(rollout_tc3_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((grid + 1) & ~1LL));
  cfg.blockDim = dim3(kThreads3);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, rollout_tc3_kernel<true>, o, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace bp

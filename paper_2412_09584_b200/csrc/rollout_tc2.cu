// rollout_tc2.cu -- K1 v2 on the 5th-generation tensor cores: the fused H-step
// rollout (reference evaluate / forward_chunk, proj/src/graph.cpp:252-401, on the
// build_objective graph, model.cpp:310-387) with every Linear layer done by
// tcgen05.mma (kind::tf32, 3xTF32) into TMEM, for layers up to 256 wide.
//
// What changes against rollout_tc.cu (v1, one 128-row tile per CTA, widths <= 128):
//  * TMEM holds, per 128-row tile, two regions of RW columns that swap roles every
//    layer: the epilogue converts the accumulator of layer l IN PLACE into the
//    hi part of layer l+1's A operand, while layer l+1 accumulates into the other
//    region (which held layer l's A, dead once layer l's MMAs retired).  The lo
//    part of A lives in shared memory (128B-swizzled K-major, SS MMAs).  That is
//    2*RW columns per tile instead of 4*128, so
//      RW = 128 (widths <= 128): TWO tiles per CTA ping-pong -- the MMAs of one
//           tile run while the epilogue of the other drains, so the tensor pipe
//           no longer idles through every epilogue (v1's serial chain);
//      RW = 256 (widths <= 256, C3): one tile, one N = 256 MMA per k-step.
//  * Sample extrema of the recorded pre-activations are reduced in the epilogue
//    registers by a transposing warp butterfly (lane j ends with column j over
//    the warp's 32 rows) and go straight to the global record with one atomic
//    pair per column and warp -- no staging buffer, no extrema warps.
//  * Weight blocks stream as separate hi and lo entries ([npad rows][128 B] each, placed
//    next to each other in the ring).  The MMA warp walks K-blocks: it waits for a
//    K-block's two blocks, issues its 12 MMAs (N = npad, up to 256) in one burst from one
//    elected asm, and commits one barrier per K-block (a_free) that frees both its ring
//    bytes and its A_lo slot.  A_lo keeps only ALO K-block slots (2 at width 256: K-block
//    c waits until K-block c-2's MMAs retired), which leaves the weight ring room for two
//    K-blocks' weights.  C3: 162.9 (N = 128 halves, per-block bursts) -> 178 (K-block
//    bursts) -> 193 TFLOP/s (N = 256: the SS MMAs read each A_lo k-step once instead of
//    once per half -- the MMA phases are bound by shared-memory reads).
//
// Precision (as v1): 3xTF32, D += A_hi.B_hi + A_lo.B_hi + A_hi.B_lo, hi read as the top
// 19 bits of the FP32 value, lo = x - trunc(x) exact; ~2^-21 relative per product.  The
// tests hold costs to 1e-5 and extrema / states to 2.5e-5 relative.
// Issue order (tools/mma_rate.cu): per K-block the A_hi.B_hi / A_lo.B_hi pairs strictly
// alternate TS/SS, then the A_hi.B_lo run; a 4xTF32 order with strict alternation runs
// each MMA faster but costs more in total (measured on C3: 142 vs 159 TFLOP/s).
//
// Warps (template <NT, RW, EPI, CW>; warp w can reach TMEM lanes 32*(w%4)..+31):
//   0..EPI-1  epilogue, EPI/NT per tile, chunks c = ((w % (EPI/NT)) / 4) mod WPQ.
//             Row = 32*(w%4) + lane of its tile.
//   EPI+1     MMA issuer (sub-partition 1), whole warp, elect.sync inside the asm.
//   EPI, EPI+2, ...  cost warps, CW per tile, 4/CW rows per thread: the cost program,
//             the states output and the extrema of the recorded scratch columns
//             (x_t, u_t, p_t, cost-op values).
//   last      producer: cp.async.bulk of the weight blocks into the byte ring.
// Instances: <2,128,16,1> two ping-pong tiles; <1,128,8,4> one tile whose cost program
// is heavy (C4: 4 cost warps, one row per thread); <1,256,16,1> one 256-wide tile (C3);
// <1,256,16,1,PAIR> the same tile as a CTA pair (opt-in, BP_TC2_PAIR=1): clusters of two
// CTAs, rank 0 issues cta_group::2 MMAs with M = 256 over both CTAs' rows, each CTA
// streams half of every weight block's N rows, commits multicast to both, the peer's
// epilogue arrives on rank 0's A barriers and its MMA warp relays its weight arrivals.
#include <cuda_runtime.h>

#include <cstdint>

#include "rollout_common.cuh"
#include "tc_common.cuh"
#include "tc_epilogue.cuh"

namespace bp {

namespace {

using namespace tc;


// Debug timeline (compiled in with -DBP_TC_TIMELINE, tools/tc_timeline.py): clock64 marks of
// CTA 0 at step 3.  Slots: 0 step start (epilogue warp 0); 100+20l+10i+{0,1,2} MMA layer l of
// tile i: A K-block 0 wait begins / ends, commit; 200+20l+10i+{0,1} epilogue of tile i (its
// first warp) wake / done; 400+10i+{0,1} cost warp of tile i start / done.
#ifdef BP_TC_TIMELINE
__device__ __forceinline__ void mark2(const RolloutArgs& a, int t, int slot) {
  if (a.timeline != nullptr && blockIdx.x == 0 && t == 3 && (threadIdx.x & 31) == 0) a.timeline[slot] = clock64();
}
__device__ __forceinline__ long long tl_clock() { return clock64(); }
__device__ __forceinline__ void put2(const RolloutArgs& a, int t, int slot, long long v) {
  if (a.timeline != nullptr && blockIdx.x == 0 && t == 3 && (threadIdx.x & 31) == 0) a.timeline[slot] = v;
}
#else
__device__ __forceinline__ void mark2(const RolloutArgs&, int, int) {}
__device__ __forceinline__ long long tl_clock() { return 0; }
__device__ __forceinline__ void put2(const RolloutArgs&, int, int, long long) {}
#endif
constexpr int kSlots = 8;  // weight blocks in flight at most (mbarrier pairs)
// __nanosleep backoff (ns) of the long waits: producer / cost warp / epilogue
#ifndef BP_TC2_SLEEP_PRODUCER
#define BP_TC2_SLEEP_PRODUCER 256
#endif
#ifndef BP_TC2_SLEEP_EPI
#define BP_TC2_SLEEP_EPI 64
#endif
constexpr uint32_t kSleepProducer = BP_TC2_SLEEP_PRODUCER, kSleepCost = 128, kSleepEpi = BP_TC2_SLEEP_EPI;

// A_lo K-block slots per tile: two at width 256 (the rest of shared memory goes to the
// weight ring, which then holds two K-blocks' weights), four for a CTA pair (its weight
// blocks are half as large; its epilogue, not the ring, is the constraint), else up to 4.
__host__ __device__ constexpr int tc2_alo_slots(int rw, bool pair) {
  return rw >= 256 ? (pair ? 4 : 2) : rw / 32 < 4 ? rw / 32 : 4;
}

template <int NT, int RW_, int EPI_, int CW_, bool PAIR_ = false>  // PAIR_: CTA pair (cluster of 2, cta_group::2, M = 256)
struct Tc2 {
  static constexpr int RW = RW_;                  // TMEM region width >= widest padded layer
  static constexpr int KBMAX = RW / 32;           // A operand K-blocks of 32 per tile
  static constexpr int ALO = tc2_alo_slots(RW, PAIR_);  // A_lo K-block slots per tile
  static constexpr int EPI = EPI_;                // epilogue warps (warps 0 .. EPI-1)
  static constexpr int WPQ = EPI / (4 * NT);      // epilogue warps per TMEM quadrant per tile
  static constexpr int CW = CW_;                  // cost warps per tile
  static constexpr int NR = 4 / CW;               // rows per cost-warp thread (128 rows per tile)
  static constexpr int kWarps = EPI + 2 + NT * CW;
  static constexpr int kThreads = 32 * kWarps;
  static constexpr int kMmaWarp = EPI + 1;        // sub-partition 1 (EPI is a multiple of 4)
  static constexpr int kProducerWarp = kWarps - 1;
  // index (0 .. NT*CW-1) of cost warp w: warps EPI, EPI+2, EPI+3, ...
  __device__ static int cost_index(int w) { return w == EPI ? 0 : w - EPI - 1; }
};

struct Tc2Smem {
  unsigned char* alo;  // [NT][ALO] slots of A lo K-blocks, 128 rows x 128 B (SW128 K-major); K-block c in slot c % ALO
  unsigned char* w;    // weight byte ring
  float* sc;           // [NT][128][tc_S] per-row scratch of the cost warps (x_t written by the epilogue)
  float* bias;         // [L][RW]
  float* cconst;       // cost-op constants, arena range [cost_f0, cost_f1)
  FwdOp* ops;          // [n_ops]
  int* segl;           // [NT][128] tile-local subdomain of each row (-1 past the last)
  int* pairs;          // [n_sc][2] recorded scratch columns (column, record offset)
  uint64_t* full;      // [kSlots] weight block landed
  uint64_t* peer_full; // [kSlots] CTA pair, rank 0: the peer's copy of the block landed (relayed)
  uint64_t* d_full;    // [NT][2] accumulator region ready for the epilogue
  uint64_t* a_chunk;   // [NT][KBMAX] A operand K-block written (4 quadrant warps)
  uint64_t* x_full;    // [NT] x_t of every row in the scratch (all epilogue warps of the tile)
  uint64_t* x_empty;   // [NT] step's scratch rows consumed (the tile's cost warp)
  uint64_t* a_free;    // [NT][KBMAX] A operand K-block read by its MMAs (commit): its A_lo slot is free
  uint32_t* tmem_slot;
  uint32_t* ring;      // [3][kSlots] producer bookkeeping
  size_t bytes;
};

__host__ __device__ inline Tc2Smem carve2(const DevObjective& o, unsigned char* base) {
  const int NT = o.tc2, RW = o.tc2_rw, KBMAX = RW / 32, ALO = tc2_alo_slots(RW, o.tc2_pair != 0);
  Tc2Smem m;
  size_t off = 0;
  auto take = [&](size_t n, size_t align) {
    off = (off + align - 1) & ~(align - 1);
    unsigned char* p = base + off;
    off += n;
    return p;
  };
  m.alo = take(static_cast<size_t>(NT) * ALO * 16384, 1024);
  m.w = take(static_cast<size_t>(o.tc2_ring), 1024);
  m.sc = reinterpret_cast<float*>(take(sizeof(float) * NT * 128 * o.tc_S, 16));
  m.bias = reinterpret_cast<float*>(take(sizeof(float) * o.L * RW, 16));
  m.cconst = reinterpret_cast<float*>(take(sizeof(float) * (o.cost_f1 - o.cost_f0), 16));
  m.ops = reinterpret_cast<FwdOp*>(take(sizeof(FwdOp) * o.n_ops, 16));
  m.segl = reinterpret_cast<int*>(take(sizeof(int) * NT * 128, 16));
  m.pairs = reinterpret_cast<int*>(take(sizeof(int) * 2 * o.n_sc, 16));
  uint64_t* bars = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * (2 * kSlots + NT * (2 + KBMAX + 2 + KBMAX)), 16));
  m.full = bars;
  m.peer_full = m.full + kSlots;
  m.d_full = m.peer_full + kSlots;
  m.a_chunk = m.d_full + 2 * NT;
  m.x_full = m.a_chunk + NT * KBMAX;
  m.x_empty = m.x_full + NT;
  m.a_free = m.x_empty + NT;
  m.tmem_slot = reinterpret_cast<uint32_t*>(take(16, 16));
  m.ring = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 3 * kSlots, 16));
  m.bytes = off;
  return m;
}

// Shared-memory bytes of everything but the weight ring (host planning).
__host__ inline size_t tc2_fixed_bytes(DevObjective o) {
  o.tc2_ring = 0;
  return 1024 + carve2(o, nullptr).bytes + 1024;  // base alignment + ring alignment slack
}


template <int NT, int RW_, int EPI_, int CW_, bool PAIR>
__global__ void __launch_bounds__(Tc2<NT, RW_, EPI_, CW_, PAIR>::kThreads, 1)
    rollout_tc2_kernel(const DevObjective o, const RolloutArgs a) {
  using C = Tc2<NT, RW_, EPI_, CW_, PAIR>;
  constexpr int RW = C::RW, KBMAX = C::KBMAX, ALO = C::ALO, WPQ = C::WPQ, CW = C::CW, NR = C::NR;
  constexpr bool kRedux = RW == 128;  // redux.sync column extrema (tc_epilogue.cuh): faster at width 128 only
  constexpr uint32_t kTmemCols = 2 * NT * RW;  // a power of two >= 32
  extern __shared__ unsigned char smraw[];
  const uint32_t s0 = smem_u32(smraw);
  const Tc2Smem m = carve2(o, smraw + (((s0 + 1023u) & ~1023u) - s0));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long cta_row0 = static_cast<long long>(blockIdx.x) * (128 * NT);
  const int ks = o.ks, ka = o.ka, kd = o.kd, d = o.d, S = o.tc_S, L = o.L, H = o.H;
  const long long rps = a.rows_per_sub;
  // CTA pair: rank 0 issues every MMA for both CTAs' rows (M = 256); both stream their
  // half of each weight block and run their own epilogue and cost warps
  const uint32_t rank = PAIR ? cluster_rank() : 0u;

  if (a.failed != nullptr) {  // skip CTAs (pairs) whose subdomains all failed already
    const long long g0 = PAIR ? cta_row0 - static_cast<long long>(rank) * 128 : cta_row0;
    const long long g1 = PAIR ? g0 + 256 : cta_row0 + 128 * NT;
    const long long last = min(a.n_rows, g1) - 1;
    bool all_failed = last >= g0;
    for (long long s = g0 / rps; s <= last / rps && all_failed; ++s) all_failed = a.failed[s] != 0;
    if (all_failed) return;
  }

  for (int i = tid; i < NT * 128; i += C::kThreads) {
    const long long r = cta_row0 + i;
    const long long tr0 = cta_row0 + (i / 128) * 128;
    m.segl[i] = r < a.n_rows ? static_cast<int>(r / rps - tr0 / rps) : -1;
  }
  for (int i = tid; i < NT * 128 * S; i += C::kThreads) m.sc[i] = 0.f;
  for (int i = tid; i < L * RW; i += C::kThreads) {
    const int l = i / RW, j = i % RW;
    m.bias[i] = j < o.tc_npad[l] ? o.f[o.tc_bias[l] + j] : 0.f;
  }
  for (int i = tid; i < o.n_ops; i += C::kThreads) {
    m.ops[i] = to_fwd(o.ops[i]);
    if (o.ops[i].folded) m.ops[i].kind = 7;  // values come from the output layer's extra columns
  }
  for (int i = tid; i < 2 * o.n_sc; i += C::kThreads) m.pairs[i] = o.iv[o.sc_list + i];
  for (int i = tid; i < o.cost_f1 - o.cost_f0; i += C::kThreads) m.cconst[i] = o.f[o.cost_f0 + i];
  if (tid == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(m.full + s, 1);
      mbar_init(m.peer_full + s, 1);
    }
    for (int i = 0; i < NT; ++i) {
      mbar_init(m.d_full + 2 * i, 1);
      mbar_init(m.d_full + 2 * i + 1, 1);
      for (int c = 0; c < KBMAX; ++c) mbar_init(m.a_chunk + i * KBMAX + c, PAIR ? 8 : 4);  // quadrant warps (of both CTAs)
      mbar_init(m.x_full + i, 4 * WPQ);
      mbar_init(m.x_empty + i, CW);
      for (int c = 0; c < KBMAX; ++c) mbar_init(m.a_free + i * KBMAX + c, 1);
    }
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
  const uint32_t ring_bytes = static_cast<uint32_t>(o.tc2_ring);

  if (warp == C::kProducerWarp) {
    // ------------------------------------------------ producer: weight blocks, hi then lo
    // A block's ring bytes are free once the MMAs of its K-block retired: the MMA warp
    // commits one barrier per K-block (a_free), so the producer waits on that, with the
    // completion's parity recorded when the block was placed.
    if (lane == 0) {
      uint32_t pos = 0;
      // virtual byte counter: advances by every block and by the tail a wrap skips, so block j
      // sits at virtual [vs_j, vs_j + bytes) and a new block ending at virtual ve overwrites
      // exactly the in-flight blocks with vs_j < ve - ring (a prefix of them, oldest first)
      uint32_t vpos = 0;
      uint32_t* vs_b = m.ring;  // virtual start of the in-flight blocks
      uint32_t* fr_b = m.ring + 2 * kSlots;  // a_free barrier index << 1 | parity of the completion
      uint32_t ppar = 0;  // bit i*KBMAX+kb: parity of a_free[i][kb]'s next completion
      int it = 0, head = 0;
      // two tiles (NT = 2) run each layer's K-blocks in lockstep on the same weight blocks:
      // streamed once per layer and freed by the last tile's release
      constexpr bool kLock = NT == 2;
      for (int t = 0; t < H; ++t)
        for (int l = 0; l < L; ++l)
          for (int i = kLock ? NT - 1 : 0; i < NT; ++i) {
            const int npad = o.tc_npad[l];
            for (int kb = 0; kb < o.tc_kb[l]; ++kb) {  // K-block outer: its A_lo slot is freed after it
              const int bit = i * KBMAX + kb;
              {
                // one block per part (hi, lo) holding all npad rows: the B operand of one N = npad
                // MMA per k-step; a CTA of a pair streams its half, rows [rank npad/2, (rank+1) npad/2)
                const int nr = PAIR ? npad / 2 : npad;
                const float* kbase = o.f + o.tc_w[l] + static_cast<size_t>(kb) * 2 * npad * 32;
                const uint32_t bytes = static_cast<uint32_t>(nr) * 128u;
                // the K-block's hi and lo blocks are placed contiguously (one wrap decision for
                // both), so a ring of two blocks' bytes never deadlocks on the pair the MMA waits for
                if (pos + 2u * bytes > ring_bytes) vpos += ring_bytes - pos;  // the tail the wrap skips
                const uint32_t at0 = ring_place(pos, 2u * bytes, ring_bytes);
                for (int part = 0; part < 2; ++part, ++it) {
                  const float* src = kbase + part * npad * 32 + (PAIR ? rank * nr * 32 : 0);
                  const uint32_t at = at0 + static_cast<uint32_t>(part) * bytes;
                  const uint32_t vs = vpos;
                  vpos += bytes;
                  // free the oldest blocks while they hold the barrier slot or the byte range
                  // (blocks are released strictly in order: per-K-block barriers shared between layers)
                  while (head < it) {
                    const int hs = head % kSlots;
                    if (it - head < kSlots && static_cast<int32_t>(vs_b[hs] - (vpos - ring_bytes)) >= 0) break;
                    mbar_wait(m.a_free + (fr_b[hs] >> 1), fr_b[hs] & 1u, kSleepProducer);
                    ++head;
                  }
                  const int s = it % kSlots;
                  vs_b[s] = vs;
                  fr_b[s] = (static_cast<uint32_t>(bit) << 1) | ((ppar >> bit) & 1u);
                  if (PAIR && o.tmaps != nullptr) {  // both halves complete on rank 0's barrier
                    if (rank == 0) mbar_expect_tx(m.full + s, 2u * bytes);
                    const int row = static_cast<int>((src - o.f) / 32);  // images start on arena rows
                    tma_rows_to_rank0(m.w + at, tmap_rows(o, nr), row, m.full + s);
                  } else {
                    mbar_expect_tx(m.full + s, bytes);
                    bulk_g2s(m.w + at, src, bytes, m.full + s);
                  }
                }
              }
            }
            ppar ^= ((1u << o.tc_kb[l]) - 1u) << (i * KBMAX);  // one completion per K-block of this operand
          }
    }
  } else if (warp == C::kMmaWarp && PAIR && rank == 1) {
    // (with the tensor maps the TMA completes on rank 0's barriers itself: nothing to relay)
    if (o.tmaps == nullptr) {
      // ---------------------------------------------- CTA pair, rank 1: relay "my half of
      // the block landed" to rank 0, which issues the MMAs over both halves
      int it = 0;
      for (int t = 0; t < H; ++t)
        for (int l = 0; l < L; ++l)
          for (int kb = 0; kb < o.tc_kb[l]; ++kb)
            for (int part = 0; part < 2; ++part, ++it) {
              mbar_wait(m.full + it % kSlots, static_cast<uint32_t>((it / kSlots) & 1));
              if (lane == 0) mbar_arrive_cta(m.peer_full + it % kSlots, 0);
              __syncwarp();
            }
    }
  } else if (warp == C::kMmaWarp && PAIR) {
    // ------------------------------------------------ CTA pair, rank 0: MMA issuer for both
    // CTAs (M = 256: each CTA's 128 rows of A from its TMEM / shared memory, B's N rows
    // half in each CTA); commits arrive in both CTAs
    int it = 0, li = 0;
    uint32_t pos = 0;
    uint32_t a_par = 0;
    const uint32_t wbase = smem_u32(m.w);
    const uint32_t abase = smem_u32(m.alo);
    for (int t = 0; t < H; ++t)
      for (int l = 0; l < L; ++l, ++li) {
        const int npad = o.tc_npad[l], ksteps = o.tc_ksteps[l];
        const uint32_t dreg = tmem + static_cast<uint32_t>((li & 1) * RW);
        const uint32_t areg = tmem + static_cast<uint32_t>(((li + 1) & 1) * RW);
        const uint32_t idesc = tf32_idesc_mn(256, npad);
        const uint32_t bytes = static_cast<uint32_t>(npad > 128 ? 128 : npad / 2) * 128u;
        long long wfull = 0, awt = 0;
        for (int kb = 0; kb < o.tc_kb[l]; ++kb) {
          if (kb == 0) mark2(a, t, 100 + 20 * l);
          const long long aw0 = tl_clock();
          mbar_wait_cluster(m.a_chunk + kb, (a_par >> kb) & 1u);  // both CTAs wrote this K-block of A
          awt += tl_clock() - aw0;
          if (kb == 0) mark2(a, t, 101 + 20 * l);
          a_par ^= 1u << kb;
          const uint64_t alo_d = sw128_desc(abase + static_cast<uint32_t>(kb % ALO) * 16384u);
          const int nq = min(4, ksteps - kb * 4);
          const uint32_t a0 = areg + 32 * kb;
          const uint32_t at_h = ring_place(pos, 2u * bytes, ring_bytes), at_l = at_h + bytes;  // hi, lo contiguous
          const long long w0 = tl_clock();
          for (int b = 0; b < 2; ++b) {
            mbar_wait_warp(m.full + (it + b) % kSlots, static_cast<uint32_t>(((it + b) / kSlots) & 1));
            if (o.tmaps == nullptr)
              mbar_wait_cluster(m.peer_full + (it + b) % kSlots, static_cast<uint32_t>(((it + b) / kSlots) & 1));
          }
          wfull += tl_clock() - w0;
          fence_after();
          if (l == 1) mark2(a, t, 600 + 2 * kb);
          const uint64_t bh = sw128_desc(wbase + at_h), bl = sw128_desc(wbase + at_l);
          if (nq == 4) {
            mma_kblock_pair_elect(dreg, a0, alo_d, bh, bl, idesc, kb != 0 ? 1u : 0u);
          } else {
            for (int q = 0; q < nq; ++q)
              mma_pair2_elect(dreg, a0 + 8 * q, alo_d + 2 * q, bh + 2 * q, idesc, (kb | q) != 0 ? 1u : 0u);
            for (int q = 0; q < nq; ++q) mma_ts2(dreg, a0 + 8 * q, bl + 2 * q, idesc, 1u);
          }
          if (l == 1) mark2(a, t, 601 + 2 * kb);
          it += 2;
          commit_pair_elect(m.a_free + kb);  // ring bytes and A_lo slot free in both CTAs
        }
        commit_pair_elect(m.d_full + (li & 1));  // accumulator complete in both CTAs
        mark2(a, t, 102 + 20 * l);
        put2(a, t, 300 + 20 * l, wfull + (1ll << 40));
        put2(a, t, 310 + 20 * l, awt + (1ll << 40));
      }
  } else if (warp == C::kMmaWarp && NT == 2) {
    // ------------------------------------------------ MMA issuer, two tiles in lockstep: per
    // K-block one wait for its weight blocks, then tile 0's burst and tile 1's burst on them
    // (each tile's A K-block waited just before its burst, its release committed after it)
    int it = 0, li = 0;
    uint32_t pos = 0;
    uint32_t a_par = 0;
    const uint32_t wbase = smem_u32(m.w);
    const uint32_t abase = smem_u32(m.alo);
    for (int t = 0; t < H; ++t)
      for (int l = 0; l < L; ++l, ++li) {
        const int npad = o.tc_npad[l], ksteps = o.tc_ksteps[l];
        const uint32_t idesc = tf32_idesc(npad);
        const uint32_t bytes = static_cast<uint32_t>(npad) * 128u;
        for (int kb = 0; kb < o.tc_kb[l]; ++kb) {
          const int nq = min(4, ksteps - kb * 4);
          const uint32_t at_h = ring_place(pos, 2u * bytes, ring_bytes), at_l = at_h + bytes;  // hi, lo contiguous
          bool weights = false;
          for (int i = 0; i < NT; ++i) {
            const int bit = i * KBMAX + kb;
            if (kb == 0) mark2(a, t, 100 + 20 * l + 10 * i);
            mbar_wait_warp(m.a_chunk + bit, (a_par >> bit) & 1u);
            if (kb == 0) mark2(a, t, 101 + 20 * l + 10 * i);
            a_par ^= 1u << bit;
            if (!weights) {
              mbar_wait_warp(m.full + it % kSlots, static_cast<uint32_t>((it / kSlots) & 1));
              mbar_wait_warp(m.full + (it + 1) % kSlots, static_cast<uint32_t>(((it + 1) / kSlots) & 1));
              weights = true;
            }
            fence_after();
            const uint32_t dreg = tmem + static_cast<uint32_t>(i * 2 * RW + (li & 1) * RW);
            const uint32_t areg = tmem + static_cast<uint32_t>(i * 2 * RW + ((li + 1) & 1) * RW);
            const uint64_t alo_d = sw128_desc(abase + static_cast<uint32_t>(i * ALO + kb % ALO) * 16384u);
            const uint32_t a0 = areg + 32 * kb;
            const uint64_t bh = sw128_desc(wbase + at_h), bl = sw128_desc(wbase + at_l);
            if (nq == 4) {
              mma_kblock_elect(dreg, a0, alo_d, bh, bl, idesc, kb != 0 ? 1u : 0u);
            } else {
              for (int q = 0; q < nq; ++q)
                mma_pair_elect(dreg, a0 + 8 * q, alo_d + 2 * q, bh + 2 * q, idesc, (kb | q) != 0 ? 1u : 0u);
              for (int q = 0; q < nq; ++q) mma_ts(dreg, a0 + 8 * q, bl + 2 * q, idesc, 1u);
            }
            mma_commit_elect(m.a_free + bit);  // tile 1's also frees the weight blocks
            if (kb + 1 == o.tc_kb[l]) {
              mma_commit_elect(m.d_full + 2 * i + (li & 1));  // this tile's accumulator complete
              mark2(a, t, 102 + 20 * l + 10 * i);
            }
          }
          it += 2;
        }
      }
  } else if (warp == C::kMmaWarp) {
    // ------------------------------------------------ MMA issuer: the whole warp runs the
    // uniform loop and waits; elect.sync inside the asm picks the issuing lane
    // (tools/mma_rate.cu: a diverged single issuing thread halves the tensor rate).
    int it = 0, li = 0;
    uint32_t pos = 0;
    uint32_t a_par = 0;  // bit i*KBMAX+kb: phase parity of a_chunk[i][kb]
    const uint32_t wbase = smem_u32(m.w);
    const uint32_t abase = smem_u32(m.alo);
    for (int t = 0; t < H; ++t)
      for (int l = 0; l < L; ++l, ++li)
        for (int i = 0; i < NT; ++i) {
          const int npad = o.tc_npad[l], ksteps = o.tc_ksteps[l];
          const uint32_t dreg = tmem + static_cast<uint32_t>(i * 2 * RW + (li & 1) * RW);
          const uint32_t areg = tmem + static_cast<uint32_t>(i * 2 * RW + ((li + 1) & 1) * RW);
          const uint32_t idesc = tf32_idesc(npad);  // one N = npad MMA per k-step (up to 256)
          const uint32_t bytes = static_cast<uint32_t>(npad) * 128u;
          long long wfull = 0, awt = 0;  // timeline: cycles waiting for weight blocks / A K-blocks
          for (int kb = 0; kb < o.tc_kb[l]; ++kb) {
            const int bit = i * KBMAX + kb;
            if (kb == 0) mark2(a, t, 100 + 20 * l + 10 * i);
            const long long aw0 = tl_clock();
            mbar_wait_warp(m.a_chunk + bit, (a_par >> bit) & 1u);  // this K-block of A written by the epilogue
            awt += tl_clock() - aw0;
            if (kb == 0) mark2(a, t, 101 + 20 * l + 10 * i);
            a_par ^= 1u << bit;
            fence_after();
            const uint64_t alo_d = sw128_desc(abase + static_cast<uint32_t>(i * ALO + kb % ALO) * 16384u);
            const int nq = min(4, ksteps - kb * 4);
            const uint32_t a0 = areg + 32 * kb;
            // the K-block's hi and lo weight blocks (consecutive ring entries), then all its MMAs
            // back to back: one burst per K-block keeps the tensor pipe fed (the waits and
            // commits between bursts are the issuer's overhead)
            if (l == 1 && i == 0) mark2(a, t, 600 + 2 * kb);
            {
              const uint32_t at_h = ring_place(pos, 2u * bytes, ring_bytes), at_l = at_h + bytes;  // hi, lo contiguous
              const long long w0 = tl_clock();
              mbar_wait_warp(m.full + it % kSlots, static_cast<uint32_t>((it / kSlots) & 1));
              mbar_wait_warp(m.full + (it + 1) % kSlots, static_cast<uint32_t>(((it + 1) / kSlots) & 1));
              wfull += tl_clock() - w0;
              const uint64_t bh = sw128_desc(wbase + at_h), bl = sw128_desc(wbase + at_l);
              if (nq == 4) {
                mma_kblock_elect(dreg, a0, alo_d, bh, bl, idesc, kb != 0 ? 1u : 0u);
              } else {
                // hi block: A_hi.B_hi and A_lo.B_hi as strictly alternating TS/SS pairs
                for (int q = 0; q < nq; ++q)
                  mma_pair_elect(dreg, a0 + 8 * q, alo_d + 2 * q, bh + 2 * q, idesc, (kb | q) != 0 ? 1u : 0u);
                // lo block: A_hi.B_lo
                for (int q = 0; q < nq; ++q) mma_ts(dreg, a0 + 8 * q, bl + 2 * q, idesc, 1u);
              }
            }
            if (l == 1 && i == 0) mark2(a, t, 601 + 2 * kb);
            it += 2;  // the blocks are free once these MMAs retire: the a_free commit below
            mma_commit_elect(m.a_free + bit);
          }
          mma_commit_elect(m.d_full + 2 * i + (li & 1));  // accumulator region complete
          mark2(a, t, 102 + 20 * l + 10 * i);
          put2(a, t, 300 + 20 * l + 10 * i, wfull + (1ll << 40));
          if (NT == 1) put2(a, t, 310 + 20 * l, awt + (1ll << 40));
        }
  } else if (warp >= C::EPI) {
    // ------------------------------------------------ cost warps: CW per tile, NR rows per
    // thread (rows 32 (cw NR + q) + lane); p_t lives in the scratch row (its pcol columns)
    const int ci = C::cost_index(warp);
    const int ti = ci / CW, cw = ci % CW;
    const long long row0 = cta_row0 + ti * 128;
    const long long rem = a.n_rows - row0;
    const int nvalid = static_cast<int>(rem < 0 ? 0 : rem < 128 ? rem : 128);
    const long long seg0 = row0 / rps;
    const long long SPH = static_cast<long long>(o.SP) * H;
    const bool rec_any = a.stat_min != nullptr;
    float* sct = m.sc + ti * 128 * S;
    int rr[NR];
    float* rows[NR];
    float cost[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      rr[q] = 32 * (cw * NR + q) + lane;
      rows[q] = sct + rr[q] * S;
      cost[q] = 0.f;
      for (int e = 0; e < kd; ++e) rows[q][o.pcol + e] = o.f[o.p0 + e];
    }
    const int* segl = m.segl + ti * 128;
    const int k_first = o.x_stat >= 0 ? ks : 0;  // the x_t columns' extrema come from the epilogue
    const long long b1 = (seg0 + 1) * rps - row0;
    const int bnd = static_cast<int>(b1 < nvalid ? b1 : nvalid);
    const bool two = nvalid == 0 || (row0 + nvalid - 1) / rps - seg0 <= 1;
    auto tile_sync = [&]() {  // the tile's cost warps (named barrier 1 + tile)
      if constexpr (CW == 1)
        __syncwarp();
      else
        asm volatile("bar.sync %0, %1;" ::"r"(1 + ti), "r"(32 * CW) : "memory");
    };
    for (int t = 0; t < H; ++t) {
      mbar_wait(m.x_full + ti, static_cast<uint32_t>(t & 1), kSleepCost);  // x_t of the tile's rows in the scratch
      mark2(a, t, 400 + 10 * ti);
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
      mark2(a, t, 403 + 10 * ti);
      if (a.states != nullptr)
#pragma unroll
        for (int q = 0; q < NR; ++q)
          if (rr[q] < nvalid)
            for (int j = 0; j < ks; ++j) a.states[((row0 + rr[q]) * H + t) * ks + j] = rows[q][j];
      if (rec_any) {
        tile_sync();  // every row of the tile written
        for (int k = k_first + 32 * cw + lane; k < o.n_sc; k += 32 * CW)
          scratch_column_extrema(a, sct + m.pairs[2 * k], S, two, bnd, nvalid, segl, seg0, SPH,
                                 t * o.SP + m.pairs[2 * k + 1]);
      }
      mark2(a, t, 401 + 10 * ti);
      mbar_arrive_warp(m.x_empty + ti);  // this warp's part of the scratch of step t consumed
    }
#pragma unroll
    for (int q = 0; q < NR; ++q)
      if (rr[q] < nvalid) {
        const long long r = row0 + rr[q];
        a.costs[r] = cost[q];
        if (a.failed != nullptr && !isfinite(cost[q])) atomicOr(a.failed + r / rps, 1);
      }
  } else {
    // ------------------------------------------------ epilogue warps: layer to layer
    constexpr int per_tile = C::EPI / NT;  // epilogue warps per tile
    const int ti = warp / per_tile;
    const int g = warp & 3;
    const int h = (warp % per_tile) >> 2;
    const int row = 32 * g + lane;
    const long long row0 = cta_row0 + ti * 128;
    const long long grow = row0 + row;
    const bool row_ok = grow < a.n_rows;
    const uint32_t tl = tmem + (static_cast<uint32_t>(32 * g) << 16) + static_cast<uint32_t>(ti * 2 * RW);
    unsigned char* alo = m.alo + ti * ALO * 16384;
    // A_lo slots: K-block c of an A operand goes to slot c % ALO.  K-block c >= ALO waits
    // until the MMAs read K-block c - ALO of the same operand (a_free, one completion per
    // operand; bit k of fpar = its parity); the slot's uses by earlier operands were read
    // before this operand's writer started (it waited for the accumulator).
    uint32_t fpar = 0;
    auto slot_wait = [&](int c) {
      if (c >= ALO) mbar_wait(m.a_free + ti * KBMAX + (c - ALO), (fpar >> (c - ALO)) & 1u, kSleepEpi);
    };
    auto a_done = [&](int kb) { fpar ^= (1u << kb) - 1u; };  // an operand of kb K-blocks was consumed
    float* scrow = m.sc + (ti * 128 + row) * S;
    const float* urow = row_ok ? a.actions + grow * d : nullptr;
    // warp's subdomain span (uniform): the common case is one subdomain, all rows valid
    const long long wr0 = row0 + 32 * g;
    const long long wr1 = min(wr0 + 31, a.n_rows - 1);
    const long long ws0 = wr0 / rps, ws1 = wr1 >= wr0 ? wr1 / rps : ws0 - 1;
    const bool simple = ws0 == ws1 && wr0 + 31 < a.n_rows;
    const long long SPH = static_cast<long long>(o.SP) * H;
    const bool x_rec = o.x_stat >= 0 && a.stat_min != nullptr;
    float pe[8], u_nxt[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      pe[e] = e < kd ? o.f[o.p0 + e] : 0.f;
      u_nxt[e] = (row_ok && e < ka) ? __ldg(urow + e) : 0.f;  // u_0
    }
    // A K-block c of the features concat(x [- tile(p)], u): v holds x in the columns
    // below ks and zeros above; x - tile(p) in relative mode, then the K-block is
    // stored with the u_{t+1} columns written by narrow stores over the zeros.
    auto features_store = [&](int c, float (&v)[32], uint32_t t_hi, unsigned char* lo_blk) {
      if (o.rel) {
        int km = (c * 32) % kd;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float pv = pe[0];
#pragma unroll
          for (int e = 1; e < 8; ++e) pv = km == e ? pe[e] : pv;
          if (c * 32 + j < ks) v[j] -= pv;
          km = km + 1 == kd ? 0 : km + 1;
        }
      }
      store_operand(t_hi, lo_blk, row, v);
      const int u0 = ks - c * 32;  // column of u_{t+1}[0] inside this K-block (warp-uniform)
      if (u0 + ka > 0 && u0 < 32) {
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");  // the zeros land first
        float* line = reinterpret_cast<float*>(lo_blk + row * 128);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = u0 + e;
          if (e < ka && j >= 0 && j < 32) {
            tmem_st1(t_hi + j, u_nxt[e]);
            line[(((j >> 2) ^ (row & 7)) << 2) + (j & 3)] = lo_tf32(u_nxt[e]);
          }
        }
      }
    };
    // features of step 0 -> A of layer 0 in region 1
    for (int c = h; c < o.tc_kb[0]; c += WPQ) {
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int k = c * 32 + j;
        v[j] = k < ks ? o.f[o.x0 + min(k, ks - 1)] : 0.f;
      }
      features_store(c, v, tl + RW + 32 * c, alo + (c % ALO) * 16384);  // no earlier use of the slots
      publish_chunk(m.a_chunk + ti * KBMAX + c, PAIR);
    }
    a_done(o.tc_kb[0]);
    int li = 0;
    const bool lead = warp % per_tile == 0;  // first epilogue warp of its tile (timeline)
    for (int t = 0; t < H; ++t) {
      if (warp == 0) mark2(a, t, 0);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (e < kd && e < ka) pe[e] += u_nxt[e];  // p_t = p_{t-1} + u_t (effector dims: the first kd)
        u_nxt[e] = (row_ok && e < ka && t + 1 < H) ? __ldg(urow + (t + 1) * ka + e) : 0.f;  // u_{t+1}
      }
      for (int l = 0; l < L; ++l, ++li) {
        const int npad = o.tc_npad[l];
        const uint32_t dcol = static_cast<uint32_t>((li & 1) * RW);
        const bool hidden = l + 1 < L;
        const float* bias = m.bias + l * RW;
        const int nch = (npad + 31) / 32;
        mbar_wait(m.d_full + 2 * ti + (li & 1), static_cast<uint32_t>((li >> 1) & 1), kSleepEpi);
        fence_after();
        if (lead) mark2(a, t, 200 + 20 * l + 10 * ti);
        if (hidden) {
          const int stat = o.pre_stat[l];
          const bool rec = o.relu[l] != 0 && stat >= 0 && a.stat_min != nullptr;
          const bool relu = o.relu[l] != 0;
          const int N = o.widths[l + 1];
          for (int c = h; c < nch; c += WPQ) {
            float v[32];
            if (npad - c * 32 >= 32)
              tmem_ld32(tl + dcol + 32 * c, v);
            else
              tmem_ld16(tl + dcol + 32 * c, v);
            const float4* b4 = reinterpret_cast<const float4*>(bias + c * 32);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 bb = b4[q];
              v[4 * q] += bb.x;
              v[4 * q + 1] += bb.y;
              v[4 * q + 2] += bb.z;
              v[4 * q + 3] += bb.w;
            }
            {  // A of layer l+1 first (in place), so its MMAs start before the extrema work
              float w[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) w[j] = relu ? fmaxf(v[j], 0.f) : v[j];
              slot_wait(c);
              store_operand(tl + dcol + 32 * c, alo + (c % ALO) * 16384, row, w);
              publish_chunk(m.a_chunk + ti * KBMAX + c, PAIR);
            }
            if (rec) {
              const int col = c * 32 + lane;
              warp_chunk_extrema<kRedux>(a, v, simple, ws0, ws1, row_ok, grow, rps, SPH,
                                 static_cast<long long>(t) * o.SP + stat + col, col, N);
            }
          }
          a_done(nch);
        } else {
          // output layer: x_t -> the cost warps' scratch; features of step t+1 -> A in place
          const int nf = t + 1 < H ? o.tc_kb[0] : 0;
          const int ncx = max(nch, nf);
          const int kx = ks + o.fold_n;  // x_t, then the folded cost-op columns (host.cu)
          if (h * 32 < kx && t >= 1) mbar_wait(m.x_empty + ti, static_cast<uint32_t>((t - 1) & 1), kSleepEpi);
          for (int c = h; c < ncx; c += WPQ) {
            float v[32];
            if (c < nch) {
              if (npad - c * 32 >= 32)
                tmem_ld32(tl + dcol + 32 * c, v);
              else
                tmem_ld16(tl + dcol + 32 * c, v);
              const float4* b4 = reinterpret_cast<const float4*>(bias + c * 32);
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 bb = b4[q];
                v[4 * q] += bb.x;
                v[4 * q + 1] += bb.y;
                v[4 * q + 2] += bb.z;
                v[4 * q + 3] += bb.w;
              }
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (c * 32 + j < ks) scrow[c * 32 + j] = v[j];
              if (c * 32 + 32 > ks && c * 32 < kx) {
                const int* fc = o.iv + o.fold_list - ks;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  const int k = c * 32 + j;
                  if (k >= ks && k < kx) scrow[__ldg(fc + k)] = v[j];
                }
              }
              if (x_rec && c * 32 < ks)  // x_t extrema here; the cost warp skips the x columns
                warp_chunk_extrema<kRedux>(a, v, simple, ws0, ws1, row_ok, grow, rps, SPH,
                                   static_cast<long long>(t) * o.SP + o.x_stat + c * 32 + lane, c * 32 + lane, ks);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = 0.f;
            }
            if (c < nf) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (c * 32 + j >= ks) v[j] = 0.f;
              slot_wait(c);
              features_store(c, v, tl + dcol + 32 * c, alo + (c % ALO) * 16384);
              publish_chunk(m.a_chunk + ti * KBMAX + c, PAIR);
            }
          }
          if (nf > 0) a_done(nf);
          mbar_arrive_warp(m.x_full + ti);  // this warp's x_t columns written
        }
        if (lead) mark2(a, t, 201 + 20 * l + 10 * ti);
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

size_t rollout_tc2_fixed_smem(const DevObjective& o) { return tc2_fixed_bytes(o); }
size_t rollout_tc2_smem(const DevObjective& o) { return 1024 + carve2(o, nullptr).bytes; }

cudaError_t launch_rollout_tc2(const DevObjective& o, const RolloutArgs& a, cudaStream_t st) {
  const size_t smem = rollout_tc2_smem(o);
  const int nt = o.tc2;
  const long long rows_per_cta = 128LL * nt;
  const long long grid = (a.n_rows + rows_per_cta - 1) / rows_per_cta;
  if (grid <= 0) return cudaSuccess;
  auto go = [&](auto kern, int threads) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(grid), threads, smem, st>>>(o, a);
    return cudaSuccess;
  };
  auto go_pair = [&](auto kern, int threads) {  // clusters of 2 CTAs (an even grid)
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>((grid + 1) & ~1LL));
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, o, a);
  };
  cudaError_t e;
  // (tiles, region width, epilogue warps, cost warps per tile[, CTA pair]): two ping-pong
  // tiles; one 128-wide tile with a heavy cost program (C4: 8 epilogue warps, 4 cost
  // warps); one 256-wide tile, as a CTA pair when every layer splits evenly (C3)
  if (nt == 2 && o.tc2_rw == 128)
    e = go(rollout_tc2_kernel<2, 128, 16, 1, false>, Tc2<2, 128, 16, 1>::kThreads);
  else if (nt == 1 && o.tc2_rw == 128)
    e = go(rollout_tc2_kernel<1, 128, 8, 4, false>, Tc2<1, 128, 8, 4>::kThreads);
  else if (nt == 1 && o.tc2_rw == 256 && o.tc2_pair)
    e = go_pair(rollout_tc2_kernel<1, 256, 16, 1, true>, Tc2<1, 256, 16, 1, true>::kThreads);
  else if (nt == 1 && o.tc2_rw == 256)
    e = go(rollout_tc2_kernel<1, 256, 16, 1, false>, Tc2<1, 256, 16, 1>::kThreads);
  else
    return cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace bp

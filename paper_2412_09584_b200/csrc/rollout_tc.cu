// rollout_tc.cu -- K1 on the 5th-generation tensor cores: the same fused
// H-step rollout as rollout.cu (reference evaluate / forward_chunk,
// proj/src/graph.cpp:252-401, on the build_objective graph, model.cpp:310-387),
// with every Linear layer done by tcgen05.mma (kind::tf32) into a TMEM
// accumulator.
//
// Precision: 3xTF32.  Weights are split on the host into hi = rna_tf32(w) and
// lo = rna_tf32(w - hi); activations into hi = x (the tensor core reads its top 19
// bits, i.e. truncates) and lo = rna_tf32(x - trunc_tf32(x)) -- an unbiased split;
// D += A_hi.B_hi + A_hi.B_lo + A_lo.B_hi keeps ~2^-21 relative per product (FP32 is
// 2^-24).  The pipe's FP32 accumulation truncates (tools/tc_rounding.cu).
// Measured against the FP64 oracle: <= 6e-6 relative on the parity cases; the
// tests hold costs to the FP32 bar (1e-5) and extrema / states to 2.5e-5.
//
// One CTA = 128 rows (the MMA M), 14 warps, warp-specialized:
//   warps 0-7   epilogue: warp w owns TMEM lanes 32(w%4).. = rows 32(w%4)..+31
//               and the 32-column chunks cb with cb%2 == w/4.  Per layer it
//               reads the accumulator (tcgen05.ld), adds the bias, stages the
//               recorded pre-activations for the extrema warps, applies ReLU and
//               writes the hi / lo split of the next layer's input straight back
//               into TMEM (tcgen05.st) as the next MMAs' A operand.  The output
//               layer's x_t goes to a shared-memory hand-off (double-buffered by
//               step) and the next step's features are built from it at once.
//   warps 8, 10 extrema: column extrema of staged chunks {0, 2} / {1, 3} of
//               every recorded pre-activation over the tile's rows (lane =
//               column), off the layer-to-layer path.
//   warps 11,12 cost: two rows per thread, the per-row cost program of step t
//               (rollout_common.cuh) from the x_t hand-off, the recorded scratch
//               extrema (redux.sync per column), the states output.
//   warp 9      producer: streams the weight K-blocks (hi and lo, host-side
//               pre-swizzled to the 128B K-major UMMA layout) into a ring of
//               shared-memory stages with cp.async.bulk + mbarrier tx counts,
//               running ahead across layers and steps.
//   warp 13     MMA issuer: one elected lane issues 3 tcgen05.mma (kind::tf32,
//               A from TMEM, B from shared memory) per K=8 step; tcgen05.commit
//               frees the weight stage and, at the end of a layer, hands the
//               accumulator to the epilogue.  Its sub-partition (warp % 4 == 1)
//               carries no extrema or cost warp: an issue-starved MMA thread
//               halves the tensor pipe's rate (tools/mma_rate.cu).
// TMEM: columns [0,128) and [128,256) two accumulators used by alternate
// layers, [256,384) A_hi, [384,512) A_lo.  The epilogue of layer l reads its
// accumulator 32 columns at a time and writes the matching 32-column K-block
// of layer l+1's A operand, arriving on that K-block's mbarrier; the MMAs of
// layer l+1 (into the other accumulator) start on each K-block as soon as it
// lands, so the tensor pipe and the epilogue overlap within one tile.
#include <cuda_runtime.h>

#include <cstdint>

#include "rollout_common.cuh"

namespace bp {

namespace {

#ifndef BP_V1_EPI
#define BP_V1_EPI 8
#endif
constexpr int kEpiWarps = BP_V1_EPI;              // epilogue warps: 4 TMEM quadrants x kEpiWarps/4 chunk groups
constexpr int kChunkGroups = kEpiWarps / 4;
constexpr int kTcThreads = 32 * (kEpiWarps + 6);  // + 4 aux warps + producer warp + MMA warp
constexpr int kProducerWarp = kEpiWarps + 1, kMmaWarp = kEpiWarps + 5;  // aux warps: E, E+2, E+3, E+4
__device__ __forceinline__ int aux_index(int warp) { return warp == kEpiWarps ? 0 : warp - kEpiWarps - 1; }
constexpr int kStgStride = 36;  // staging row stride (floats): 16B rows, conflict-free column reads
constexpr int kStages = 3;   // weight ring capacity, in K-blocks of the widest layer
constexpr int kSlots = 8;    // K-blocks in flight in the ring at most (mbarrier pairs)

// Weight ring: K-blocks of 2 * npad * 128 bytes (hi | lo) placed back to back in
// a byte ring of kStages widest blocks, wrapping to 0 when a block does not fit,
// so narrow layers keep more blocks in flight.  Producer and MMA issuer walk the
// same sequence and place block by block with this function.
__device__ __forceinline__ uint32_t ring_place(uint32_t& pos, uint32_t bytes, uint32_t ring) {
  if (pos + bytes > ring) pos = 0;
  const uint32_t at = pos;
  pos += bytes;
  return at;
}
// TMEM columns: two accumulators (layers alternate) and the hi / lo A operand
constexpr uint32_t kColD0 = 0, kColD1 = 128, kColAhi = 256, kColAlo = 384;
constexpr int kMaxChunks = 4;  // A operand K-blocks of 32 (widths <= 128)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Round to TF32, nearest with ties away (cvt.rna.tf32.f32 on finite values) in two
// integer ops.  Non-finite inputs stay non-finite through lo = x - hi.
__device__ __forceinline__ float rna_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
// 3xTF32 operand split: hi = rna_tf32(x), lo = rna_tf32(x - hi) (as tc_common.cuh split_tf32).
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = rna_tf32(x);
  lo = rna_tf32(x - hi);
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;                    // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>((1024u >> 4) & 0x3FFFu) << 32;  // SBO
  d |= static_cast<uint64_t>(1u) << 46;                    // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;                    // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M=128, N=n.
__device__ __forceinline__ uint32_t tf32_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  for (long long spin = 0; !done; ++spin) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(phase), "r"(0x989680u)  // suspend in hardware until the phase flips
        : "memory");
    if (spin > (1ll << 28)) asm volatile("trap;");  // never hang the device on a lost arrival
  }
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[32]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
#pragma unroll
  for (int j = 16; j < 32; ++j) v[j] = 0.f;
}

// The three 3xTF32 MMAs of one K-step (A_hi.B_hi, A_hi.B_lo, A_lo.B_hi), issued by one
// elected lane of a converged warp.
__device__ __forceinline__ void mma3_tf32_ts(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint64_t bl,
                                             uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e, one;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, one;\n\t}\n" ::"r"(d),
      "r"(ah), "r"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31])));
}

// Writes 32 consecutive K-values of this thread's row as the hi / lo A operand in TMEM.
__device__ __forceinline__ void store_operand_tmem(uint32_t tlane, int chunk, const float (&v)[32]) {
  // hi = v (the tensor core truncates it), lo = rna_tf32(v - trunc(v)): unbiased, within 2^-21 |v|.
  tmem_st32(tlane + kColAhi + 32 * chunk, v);
  float l[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) l[j] = rna_tf32(v[j] - __uint_as_float(__float_as_uint(v[j]) & 0xffffe000u));
  tmem_st32(tlane + kColAlo + 32 * chunk, l);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// One arrival per warp, after every lane's prior writes: __syncwarp orders the
// lanes' accesses before lane 0's release-arrive (barrier counts are in warps).
__device__ __forceinline__ void mbar_arrive_warp(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Debug timeline: compiled in with -DBP_TC_TIMELINE (_build.build_variant, used by
// tools/tc_timeline.py) and enabled by the BP_TC_TIMELINE environment variable;
// clock64 marks of CTA 0, step 3.  Slots: 0 step start, 100+10l+{0,1} MMA layer l
// first issue / commit, 200+10l+{0,1} epilogue layer l wake / chunks done (warp 0),
// 400/401 cost program start / done (warp 11), 403-407 features, 500+ MMA waits of
// the last layer, 520+ producer issues of the last layer, 600+ epilogue chunk phases.
#ifdef BP_TC_TIMELINE
__device__ __forceinline__ void mark(const RolloutArgs& a, int t, int slot) {
  if (a.timeline != nullptr && blockIdx.x == 0 && t == 3 && (threadIdx.x & 31) == 0) a.timeline[slot] = clock64();
}
#else
__device__ __forceinline__ void mark(const RolloutArgs&, int, int) {}  // timeline marks compiled out
#endif

// Bias rows padded to whole 32-column chunks (float4 reads of a full chunk).
__host__ __device__ __forceinline__ int bias_stride(const DevObjective& o) { return (o.tc_npadmax + 31) & ~31; }

struct TcSmem {
  unsigned char* w;    // weight ring: kStages x (hi | lo)[npadmax rows x 128 B] bytes
  float* stg;          // [kMaxChunks][128 rows][kStgStride] staged pre-activations
  float* sc;           // [128][tc_S] per-row scratch of the cost warps (x_t, u_t, p_t, op values)
  float* bias;         // [L][bias_stride]
  float* xbuf;         // [2][128][tc_xs] x_t hand-off rows, by step parity
  float* ubuf;         // [2][128][ustr] u_t rows for the features, by step parity (written by the cost warps)
  float* prow;         // [128][8] effector p_{t-1} of the epilogue
  float* cconst;       // cost-op constants, arena range [cost_f0, cost_f1)
  FwdOp* ops;          // [n_ops] forward op table
  int* segl;           // [128] tile-local subdomain of each row (-1 past the last)
  int* pairs;          // [n_sc][2] recorded scratch columns (column, record offset)
  uint64_t* full;      // [kSlots] weight K-block landed
  uint64_t* empty;     // [kSlots] weight K-block consumed by the MMAs
  uint64_t* d_full;    // [2] accumulator ready for the epilogue
  uint64_t* a_chunk;   // [kMaxChunks] A operand K-block written by its 4 epilogue warps
  uint64_t* stg_full;  // [kMaxChunks] chunk staged (4 epilogue warps)
  uint64_t* stg_empty; // [kMaxChunks] chunk consumed by its extrema warp
  uint64_t* x_full;    // [2] x_t rows written (8 epilogue warps)
  uint64_t* x_empty;   // [2] x_t rows copied by the 2 cost warps
  uint64_t* sc_full;   // [2] step's scratch rows complete (2 cost warps)
  uint64_t* sc_empty;  // [2] step's scratch extrema taken (2 extrema warps)
  uint64_t* u_full;    // [2] u rows of the slot written (2 cost warps)
  uint32_t* tmem_slot;
  uint32_t* ring;      // [2][kSlots] producer bookkeeping
  size_t bytes;        // total, from the 1024-aligned base
};

// Extrema of one column over the tile's valid rows (v = col[r * stride]) into the
// per-subdomain record at offset `off` within a subdomain's [H * SP] block: the
// two-subdomain form (rows [0, bnd) / [bnd, nvalid)) or, for tiles spanning more
// subdomains (parity-test sizes), a walk over segl.  `valid` gates the atomics.
__device__ __forceinline__ void column_extrema(const RolloutArgs& a, const float* col, int stride, bool valid, bool two,
                                               int bnd, int nvalid, const int* segl, long long seg0, long long SPH,
                                               long long off) {
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
    if (valid) {
      if (bnd > 0) {
        atomicMin(a.stat_min + seg0 * SPH + off, enc_f(mn0));
        atomicMax(a.stat_max + seg0 * SPH + off, enc_f(mx0));
      }
      if (bnd < nvalid) {
        atomicMin(a.stat_min + (seg0 + 1) * SPH + off, enc_f(mn1));
        atomicMax(a.stat_max + (seg0 + 1) * SPH + off, enc_f(mx1));
      }
    }
    return;
  }
  float mn = INFINITY, mx = -INFINITY;
  int sg = -1;
  for (int r = 0; r < nvalid; ++r) {
    const int s2 = segl[r];
    if (s2 != sg) {
      if (sg >= 0 && valid) {
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
  if (sg >= 0 && valid) {
    atomicMin(a.stat_min + (seg0 + sg) * SPH + off, enc_f(mn));
    atomicMax(a.stat_max + (seg0 + sg) * SPH + off, enc_f(mx));
  }
}

__host__ __device__ __forceinline__ int ustride(const DevObjective& o) { return o.ka | 1; }

// One carve for the kernel and the host-side size: 16-byte aligned regions.
__host__ __device__ inline TcSmem carve(const DevObjective& o, unsigned char* base) {
  TcSmem m;
  size_t off = 0;
  auto take = [&](size_t n) {
    unsigned char* p = base + off;
    off = (off + n + 15) & ~static_cast<size_t>(15);
    return p;
  };
  m.w = take(static_cast<size_t>(kStages) * 2 * o.tc_npadmax * 128);
  m.stg = reinterpret_cast<float*>(take(sizeof(float) * kMaxChunks * 128 * kStgStride));
  m.sc = reinterpret_cast<float*>(take(sizeof(float) * 128 * o.tc_S));
  m.bias = reinterpret_cast<float*>(take(sizeof(float) * o.L * bias_stride(o)));
  m.xbuf = reinterpret_cast<float*>(take(sizeof(float) * 2 * 128 * o.tc_xs));
  m.ubuf = reinterpret_cast<float*>(take(sizeof(float) * 2 * 128 * ustride(o)));
  m.prow = reinterpret_cast<float*>(take(sizeof(float) * 128 * 8));
  m.cconst = reinterpret_cast<float*>(take(sizeof(float) * (o.cost_f1 - o.cost_f0)));
  m.ops = reinterpret_cast<FwdOp*>(take(sizeof(FwdOp) * o.n_ops));
  m.segl = reinterpret_cast<int*>(take(sizeof(int) * 128));
  m.pairs = reinterpret_cast<int*>(take(sizeof(int) * 2 * o.n_sc));
  uint64_t* bars = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * (2 * kSlots + 2 + 3 * kMaxChunks + 10)));
  m.full = bars;
  m.empty = m.full + kSlots;
  m.d_full = m.empty + kSlots;
  m.a_chunk = m.d_full + 2;
  m.stg_full = m.a_chunk + kMaxChunks;
  m.stg_empty = m.stg_full + kMaxChunks;
  m.x_full = m.stg_empty + kMaxChunks;
  m.x_empty = m.x_full + 2;
  m.sc_full = m.x_empty + 2;
  m.sc_empty = m.sc_full + 2;
  m.u_full = m.sc_empty + 2;
  m.tmem_slot = reinterpret_cast<uint32_t*>(take(16));
  m.ring = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * 2 * kSlots));
  m.bytes = off;
  return m;
}

__global__ void __launch_bounds__(kTcThreads, 1) rollout_tc_kernel(const DevObjective o, const RolloutArgs a) {
  extern __shared__ unsigned char smraw[];
  const uint32_t s0 = smem_u32(smraw);
  const TcSmem m = carve(o, smraw + (((s0 + 1023u) & ~1023u) - s0));  // SW128 stages: 1024-aligned
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long row0 = static_cast<long long>(blockIdx.x) * 128;
  const long long rem_rows = a.n_rows - row0;
  const int nvalid = static_cast<int>(rem_rows < 128 ? rem_rows : 128);
  const int ks = o.ks, ka = o.ka, kd = o.kd, d = o.d, S = o.tc_S, L = o.L, H = o.H;

  if (a.failed != nullptr) {  // skip tiles whose subdomains already failed
    const long long s0 = row0 / a.rows_per_sub, s1 = (row0 + nvalid - 1) / a.rows_per_sub;
    bool all_failed = true;
    for (long long s = s0; s <= s1; ++s) all_failed = all_failed && a.failed[s] != 0;
    if (all_failed) return;
  }

  const long long seg0 = row0 / a.rows_per_sub;
  if (tid < 128) m.segl[tid] = tid < nvalid ? static_cast<int>((row0 + tid) / a.rows_per_sub - seg0) : -1;
  for (int i = tid; i < 128 * S; i += kTcThreads) m.sc[i] = 0.f;
  for (int i = tid; i < L * bias_stride(o); i += kTcThreads) {
    const int l = i / bias_stride(o), j = i % bias_stride(o);
    m.bias[i] = j < o.tc_npad[l] ? o.f[o.tc_bias[l] + j] : 0.f;
  }
  for (int i = tid; i < o.n_ops; i += kTcThreads) m.ops[i] = to_fwd(o.ops[i]);
  for (int i = tid; i < 2 * o.n_sc; i += kTcThreads) m.pairs[i] = o.iv[o.sc_list + i];
  for (int i = tid; i < o.cost_f1 - o.cost_f0; i += kTcThreads) m.cconst[i] = o.f[o.cost_f0 + i];
  if (tid == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(m.full + s, 1);
      mbar_init(m.empty + s, 1);
    }
    mbar_init(m.d_full + 0, 1);
    mbar_init(m.d_full + 1, 1);
    for (int c = 0; c < kMaxChunks; ++c) {
      mbar_init(m.a_chunk + c, 4);  // arrivals are per warp
      mbar_init(m.stg_full + c, 4);
      mbar_init(m.stg_empty + c, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(m.x_full + b, kEpiWarps);
      mbar_init(m.x_empty + b, 2);  // the two cost warps
      mbar_init(m.sc_full + b, 2);
      mbar_init(m.sc_empty + b, 2);  // the two extrema warps
      mbar_init(m.u_full + b, 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(m.tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *m.tmem_slot;
  const uint32_t ring_bytes = static_cast<uint32_t>(kStages) * 2u * o.tc_npadmax * 128u;

  if (warp == kProducerWarp) {
    // ------------------------------------------------ producer: weight K-blocks
    if (lane == 0) {
      // in-flight blocks [head, it): their byte ranges, oldest first (FIFO order of
      // the ring); block it waits for every older block whose bytes it overlaps
      uint32_t pos = 0;
      uint32_t* lo_b = m.ring;  // [kSlots] byte ranges of the in-flight blocks
      uint32_t* hi_b = m.ring + kSlots;
      int it = 0, head = 0;
      for (int t = 0; t < H; ++t)
        for (int l = 0; l < L; ++l) {
          const int npad = o.tc_npad[l];
          const uint32_t bytes = 2u * npad * 128u;
          for (int kb = 0; kb < o.tc_kb[l]; ++kb, ++it) {
            const uint32_t at = ring_place(pos, bytes, ring_bytes);
            // the slot's previous block and every in-flight block overlapping the byte range
            // must be free: wait in order up to the newest of them (a wrapped placement of
            // mixed-size blocks can overlap a newer block but not the oldest)
            int need = it - kSlots;
            for (int q = it - 1; q >= head && q > need; --q)
              if (!(hi_b[q % kSlots] <= at || lo_b[q % kSlots] >= at + bytes)) {
                need = q;
                break;
              }
            for (; head <= need; ++head)
              mbar_wait(m.empty + head % kSlots, static_cast<uint32_t>((head / kSlots) & 1));
            const int s = it % kSlots;
            lo_b[s] = at;
            hi_b[s] = at + bytes;
            if (l == L - 1) mark(a, t, 520 + kb);
            mbar_expect_tx(m.full + s, bytes);
            bulk_g2s(m.w + at, o.f + o.tc_w[l] + static_cast<size_t>(kb) * 2 * npad * 32, bytes, m.full + s);
          }
        }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------ MMA issuer: the whole warp runs the
    // (uniform) loop so descriptors stay in uniform registers; one elected lane issues.
    int it = 0, layer_it = 0;
    uint32_t pos = 0;
    uint32_t a_par = 0;  // bit kb: phase parity of a_chunk[kb] (registers, no local array)
    const uint64_t wdesc0 = sw128_desc(smem_u32(m.w));
    for (int t = 0; t < H; ++t)
      for (int l = 0; l < L; ++l, ++layer_it) {
        const int npad = o.tc_npad[l], ksteps = o.tc_ksteps[l];
        const uint32_t idesc = tf32_idesc(npad);
        const uint32_t dst = tmem + ((layer_it & 1) ? kColD1 : kColD0);
        const uint64_t lo_off = static_cast<uint64_t>(npad * 128) >> 4;
        for (int kb = 0; kb < o.tc_kb[l]; ++kb, ++it) {
          mbar_wait(m.a_chunk + kb, (a_par >> kb) & 1u);  // this K-block of A landed
          a_par ^= 1u << kb;
          if (kb == 0) mark(a, t, 100 + 10 * l);
          if (l == L - 1) mark(a, t, 500 + 2 * kb);
          const int s = it % kSlots;
          const uint32_t at = ring_place(pos, 2u * npad * 128u, ring_bytes);
          mbar_wait(m.full + s, static_cast<uint32_t>((it / kSlots) & 1));
          if (l == L - 1) mark(a, t, 501 + 2 * kb);
          fence_after();
          const uint64_t bh0 = wdesc0 + (static_cast<uint64_t>(at) >> 4);
          const int nq = min(4, ksteps - kb * 4);
          for (int q = 0; q < nq; ++q) {
            const int kstep = kb * 4 + q;
            const uint64_t bh = bh0 + 2 * q;  // +32 B along K inside the 128 B swizzle atom
            mma3_tf32_ts(dst, tmem + kColAhi + 8 * kstep, tmem + kColAlo + 8 * kstep, bh, bh + lo_off, idesc,
                         kstep > 0 ? 1u : 0u);
          }
          mma_commit_elect(m.empty + s);  // block's bytes free once these MMAs retire
        }
        mma_commit_elect(m.d_full + (layer_it & 1));  // accumulator complete
        mark(a, t, 101 + 10 * l);
      }
  } else if (warp >= kEpiWarps) {
    const int ai = aux_index(warp);
    const long long b1 = (seg0 + 1) * a.rows_per_sub - row0;
    const int bnd = static_cast<int>(b1 < nvalid ? b1 : nvalid);
    const bool two = (row0 + nvalid - 1) / a.rows_per_sub - seg0 <= 1;
    const long long SPH = static_cast<long long>(o.SP) * H;
    const bool rec_any = a.stat_min != nullptr;
    if (ai < 2) {
      // ---------------------------------------------- extrema warps: per step, chunks ai and
      // ai + 2 of every recorded hidden pre-activation (staged by the epilogue), then the
      // recorded scratch columns of the previous step (written by the cost warps);
      // lane = column, over the tile's rows
      uint32_t use_par = 0;  // bit u: phase parity of stg_full[ai + 2u]
      const int n_sc = rec_any ? o.n_sc : 0;
      auto scratch = [&](int ts) {
        mbar_wait(m.sc_full + (ts & 1), static_cast<uint32_t>((ts >> 1) & 1));
        for (int i = 32 * ai + lane; i < n_sc; i += 64)
          column_extrema(a, m.sc + m.pairs[2 * i], o.tc_S, true, two, bnd, nvalid, m.segl, seg0, SPH,
                         ts * o.SP + m.pairs[2 * i + 1]);
        mbar_arrive_warp(m.sc_empty + (ts & 1));
      };
      for (int t = 0; t < H; ++t) {
        for (int l = 0; l + 1 < L; ++l) {
          const int stat = o.pre_stat[l];
          if (o.relu[l] == 0 || stat < 0 || !rec_any) continue;
          const int nch = (o.tc_npad[l] + 31) / 32, N = o.widths[l + 1];
          for (int u = 0; u < 2; ++u) {
            const int c = ai + 2 * u;
            if (c >= nch) break;
            mbar_wait(m.stg_full + c, (use_par >> u) & 1u);
            use_par ^= 1u << u;
            const int col = c * 32 + lane;
            column_extrema(a, m.stg + c * 128 * kStgStride + lane, kStgStride, col < N, two, bnd, nvalid, m.segl, seg0, SPH,
                           t * o.SP + stat + col);
            __syncwarp();
            if (lane == 0) mbar_arrive(m.stg_empty + c);
          }
        }
        if (t >= 1) scratch(t - 1);
      }
      scratch(H - 1);
    } else {
      // ---------------------------------------------- cost warps: two rows per thread
      // (rows 64w + lane and 64w + 32 + lane), the step's cost program from the x_t hand-off
      const int cw = ai - 2;
      const int rA = 64 * cw + lane, rB = rA + 32;
      float* const rows[2] = {m.sc + rA * S, m.sc + rB * S};
      const bool ok[2] = {rA < nvalid, rB < nvalid};
      const float* ur[2] = {ok[0] ? a.actions + (row0 + rA) * d : nullptr, ok[1] ? a.actions + (row0 + rB) * d : nullptr};
      float p[2][8];
#pragma unroll
      for (int j = 0; j < 8; ++j) p[0][j] = p[1][j] = j < kd ? o.f[o.p0 + j] : 0.f;
      float cost[2] = {0.f, 0.f};
      const int us = ustride(o);
      for (int b = 0; b < 2; ++b) {  // u_0, u_1 for the epilogue's features
#pragma unroll
        for (int q = 0; q < 2; ++q)
          for (int j = 0; j < ka; ++j)
            m.ubuf[(b * 128 + (q ? rB : rA)) * us + j] = (ok[q] && b < H) ? __ldg(ur[q] + b * ka + j) : 0.f;
        mbar_arrive_warp(m.u_full + b);
      }
      for (int t = 0; t < H; ++t) {
        const int xb = t & 1;
        float un[2][8];  // u_t (this iteration) and u_{t+2} (the epilogue's features two steps on)
        float u2[2][8];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            un[q][j] = j < ka ? m.ubuf[(xb * 128 + (q ? rB : rA)) * us + j] : 0.f;
            u2[q][j] = (ok[q] && j < ka && t + 2 < H) ? __ldg(ur[q] + (t + 2) * ka + j) : 0.f;
          }
        if (t >= 1) mbar_wait(m.sc_empty + ((t - 1) & 1), static_cast<uint32_t>(((t - 1) >> 1) & 1));
        mbar_wait(m.x_full + xb, static_cast<uint32_t>((t >> 1) & 1));
        if (warp == 11) mark(a, t, 400);
        for (int j = 0; j < ks; ++j) {
          rows[0][j] = m.xbuf[(xb * 128 + rA) * o.tc_xs + j];
          rows[1][j] = m.xbuf[(xb * 128 + rB) * o.tc_xs + j];
        }
        mbar_arrive_warp(m.x_empty + xb);
        // x_full(t): the epilogue has read u_t (features, p update), so the slot takes u_{t+2}
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < ka) m.ubuf[(xb * 128 + (q ? rB : rA)) * us + j] = u2[q][j];
        mbar_arrive_warp(m.u_full + xb);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < ka) {
              rows[q][o.ucol + j] = un[q][j];
              p[q][j] += un[q][j];
            }
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (e < kd) rows[q][o.pcol + e] = p[q][e];
        }
        cost_program_n<2>(o, m.ops, m.cconst - o.cost_f0, rows, t, cost);
        if (warp == 11) mark(a, t, 401);
        if (a.states != nullptr)
#pragma unroll
          for (int q = 0; q < 2; ++q)
            if (ok[q])
              for (int j = 0; j < ks; ++j) a.states[((row0 + (q ? rB : rA)) * H + t) * ks + j] = rows[q][j];
        mbar_arrive_warp(m.sc_full + xb);  // scratch rows of step t complete: the extrema warps take them
      }
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (ok[q]) {
          const long long r = row0 + (q ? rB : rA);
          a.costs[r] = cost[q];
          if (a.failed != nullptr && !isfinite(cost[q])) atomicOr(a.failed + r / a.rows_per_sub, 1);
        }
    }
  } else {
    // ------------------------------------------------ epilogue warps: layer to layer
    const int g = warp & 3, h = warp >> 2;  // TMEM lane group, column-chunk group
    const int row = 32 * g + lane;
    const uint32_t tlane = tmem + (static_cast<uint32_t>(32 * g) << 16);
    const bool row_ok = row < nvalid;
    const float* urow = row_ok ? a.actions + (row0 + row) * d : nullptr;
    float* prow = m.prow + row * 8;      // effector p_{t-1} (h == 0 threads)
    // x_t goes to xbuf slot t&1; step t's features read x_{t-1} from slot (t+1)&1
    // (x_0 in slot 1) and u_t from ubuf slot t&1
    if (h == 0) {
      for (int j = 0; j < 8; ++j) prow[j] = j < kd ? o.f[o.p0 + j] : 0.f;
      for (int j = 0; j < ks; ++j) m.xbuf[(128 + row) * o.tc_xs + j] = o.f[o.x0 + j];
    }
    const int us = ustride(o);
    // early features: the input layer is one K-block and the output layer's x_t one chunk
    // (so the chunk-0 warps of the output epilogue hold all of x_t)
    const bool early = o.tc_kb[0] == 1 && o.tc_npad[L - 1] <= 32 && ks + ka <= 32;
    asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps) : "memory");
    int layer_it = 0;
    uint32_t stg_used = 0, stg_par = 0;  // bit cb: chunk staged before / parity of its last use
    for (int t = 0; t < H; ++t) {
      if (warp == 0) mark(a, t, 0);
      const float* xprev = m.xbuf + (((t + 1) & 1) * 128 + row) * o.tc_xs;  // x_{t-1}
      const float* ucur = m.ubuf + ((t & 1) * 128 + row) * us;               // u_t
      if (!early || t == 0) mbar_wait(m.u_full + (t & 1), static_cast<uint32_t>((t >> 1) & 1));  // written a step ago
      if (warp == 0) mark(a, t, 407);
      // features of layer 0 -> A: concat(x_{t-1} [- tile(p_{t-1})], u_t), zero padded (from
      // step 1 on, the early path wrote them in the previous step's output epilogue)
      for (int kb = h; kb < o.tc_kb[0] && (!early || t == 0); kb += kChunkGroups) {
        // every load is issued unconditionally from a clamped address (no predicated
        // loads, no branches), so they pipeline; the selects come after
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int k = kb * 32 + j;
          v[j] = k < ks ? xprev[min(k, ks - 1)] : ucur[min(max(k - ks, 0), ka - 1)];
        }
        if (o.rel) {  // x - tile(p_{t-1}): p index k mod kd, stepped with k, selected from registers
          float pa[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) pa[e] = prow[e];
          int km = (kb * 32) % kd;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float pv = pa[0];
#pragma unroll
            for (int e = 1; e < 8; ++e) pv = km == e ? pa[e] : pv;
            if (kb * 32 + j < ks) v[j] -= pv;
            km = km + 1 == kd ? 0 : km + 1;
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int k = kb * 32 + j;
          v[j] = k < ks + ka ? v[j] : 0.f;
        }
        if (warp == 0) mark(a, t, 404);
        store_operand_tmem(tlane, kb, v);
        if (warp == 0) mark(a, t, 405);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (warp == 0) mark(a, t, 406);
        fence_before();
        mbar_arrive_warp(m.a_chunk + kb);
      }
      if (warp == 0) mark(a, t, 403);
      // p_t and u_{t+1} for the next step's features
      asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps) : "memory");  // both groups read prow above
      if (h == 0)
        for (int j = 0; j < ka; ++j) prow[j] += ucur[j];
      for (int l = 0; l < L; ++l, ++layer_it) {
        const int npad = o.tc_npad[l];
        const uint32_t dcol = (layer_it & 1) ? kColD1 : kColD0;
        const bool hidden = l + 1 < L;
        if (!hidden) {  // x_t hand-off slot must be free (the aux warps consumed step t-2)
          if (t >= 2) mbar_wait(m.x_empty + (t & 1), static_cast<uint32_t>(((t >> 1) - 1) & 1));
        }
        mbar_wait(m.d_full + (layer_it & 1), static_cast<uint32_t>((layer_it >> 1) & 1));
        fence_after();
        if (warp == 0) mark(a, t, 200 + 10 * l);
        const bool relu = o.relu[l] != 0;
        const int stat = o.pre_stat[l];
        const bool rec = relu && stat >= 0 && a.stat_min != nullptr && hidden;
        const float* bias = m.bias + l * bias_stride(o);
        const int nchunk = (npad + 31) / 32;
        for (int cb = h; cb < nchunk; cb += kChunkGroups) {
          float v[32];
          float4 bb[8];  // bias loads issued first: their latency overlaps the TMEM load
          const float4* b4 = reinterpret_cast<const float4*>(bias + cb * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q) bb[q] = b4[q];
          if (npad - cb * 32 >= 32) {
            tmem_ld32(tlane + dcol + cb * 32, v);
          } else {
            tmem_ld16(tlane + dcol + cb * 32, v);
#pragma unroll
            for (int j = 16; j < 32; ++j) v[j] = 0.f;
          }
          const bool mk = warp == 0 && l == 1;
          if (mk) mark(a, t, 600 + 10 * (cb >> 1));
          // columns in [N, npad) are exact zeros: zero weight rows and zero bias padding
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            v[4 * q] += bb[q].x;
            v[4 * q + 1] += bb[q].y;
            v[4 * q + 2] += bb[q].z;
            v[4 * q + 3] += bb[q].w;
          }
          if (mk) mark(a, t, 604 + 10 * (cb >> 1));
          if (hidden) {
            // the next layer's A K-block first (its MMAs start on it), then the staging
            // of the pre-activations for the extrema warps, off the MMA's critical path
            float w[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) w[j] = relu ? fmaxf(v[j], 0.f) : v[j];
            store_operand_tmem(tlane, cb, w);
            if (mk) mark(a, t, 602 + 10 * (cb >> 1));
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            if (mk) mark(a, t, 603 + 10 * (cb >> 1));
            fence_before();
            mbar_arrive_warp(m.a_chunk + cb);  // the next layer's MMAs may start on this K-block
          }
          if (rec) {  // stage the pre-activations for this chunk's aux warp
            if ((stg_used >> cb) & 1u) mbar_wait(m.stg_empty + cb, ((stg_par >> cb) & 1u) ^ 1u);
            if (mk) mark(a, t, 605 + 10 * (cb >> 1));
            stg_used |= 1u << cb;
            stg_par ^= 1u << cb;
            float4* dst = reinterpret_cast<float4*>(m.stg + (cb * 128 + row) * kStgStride);
#pragma unroll
            for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            mbar_arrive_warp(m.stg_full + cb);
          }
          if (mk) mark(a, t, 601 + 10 * (cb >> 1));
          if (!hidden) {
            float* xo = m.xbuf + ((t & 1) * 128 + row) * o.tc_xs;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (relu) v[j] = fmaxf(v[j], 0.f);
              if (cb * 32 + j < ks) xo[cb * 32 + j] = v[j];
            }
            if (early && t + 1 < H) {
              // step t+1's features straight from x_t (this chunk holds all of it):
              // concat(x_t [- tile(p_t)], u_{t+1}) into A K-block 0, whose MMAs (this
              // output layer's) have retired
              mbar_wait(m.u_full + ((t + 1) & 1), static_cast<uint32_t>(((t + 1) >> 1) & 1));
              const float* unext = m.ubuf + (((t + 1) & 1) * 128 + row) * us;
              float f[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) f[j] = j < ks ? v[j] : unext[min(max(j - ks, 0), ka - 1)];
              if (o.rel) {
                float pa[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) pa[e] = prow[e];  // p_t
                int km = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  float pv = pa[0];
#pragma unroll
                  for (int e = 1; e < 8; ++e) pv = km == e ? pa[e] : pv;
                  if (j < ks) f[j] -= pv;
                  km = km + 1 == kd ? 0 : km + 1;
                }
              }
#pragma unroll
              for (int j = 0; j < 32; ++j) f[j] = j < ks + ka ? f[j] : 0.f;
              store_operand_tmem(tlane, 0, f);
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
              fence_before();
              mbar_arrive_warp(m.a_chunk + 0);
            }
          }
        }
        if (warp == 0) mark(a, t, 201 + 10 * l);
        if (!hidden) {  // x_t of every row written: hand it to the aux warps and to the next features
          fence_before();
          mbar_arrive_warp(m.x_full + (t & 1));
          asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps) : "memory");
        }
      }
    }
  }

  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace

size_t rollout_tc_smem(const DevObjective& o) { return 1024 + carve(o, nullptr).bytes; }

cudaError_t launch_rollout_tc(const DevObjective& o, const RolloutArgs& a, cudaStream_t st) {
  const size_t smem = rollout_tc_smem(o);
  cudaError_t e = cudaFuncSetAttribute(rollout_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const long long grid = (a.n_rows + 127) / 128;
  if (grid <= 0) return cudaSuccess;
  rollout_tc_kernel<<<static_cast<unsigned>(grid), kTcThreads, smem, st>>>(o, a);
  return cudaGetLastError();
}

}  // namespace bp

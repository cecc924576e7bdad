// tc_common.cuh -- sm_100a PTX helpers shared by the tcgen05 rollout kernels
// (rollout_tc.cu, rollout_tc2.cu): UMMA descriptors, tcgen05 MMA / load / store,
// mbarriers and bulk copies.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bp {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 3xTF32 operand split of an activation: hi = rna_tf32(x) and lo = rna_tf32(x - hi), both
// with their 13 low mantissa bits zero, so kind::tf32 (which reads the top 19 bits) sees
// them exactly.  x - hi is exact; hi + lo is within 2^-22 |x| of x and unbiased (a truncated
// lo instead biases every activation toward zero by ~2^-21, which expansive rollouts amplify
// step over step).
__device__ __forceinline__ float rna_tf32_dev(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = rna_tf32_dev(x);
  lo = rna_tf32_dev(x - hi);
}
// Cheaper epilogue form: hi is stored as x itself (kind::tf32 truncates it to its top 19 bits),
// lo = rna_tf32(x - trunc_tf32(x)) -- exact difference, rounded to nearest: within 2^-21 |x| of x
// and unbiased (only a truncated lo would bias the operand toward zero).
__device__ __forceinline__ float lo_tf32(float x) {
  return rna_tf32_dev(x - __uint_as_float(__float_as_uint(x) & 0xffffe000u));
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row groups 1024 B apart.
// Used for both operands: a [rows][32 x 32-bit] K-block, row r at r*128 B with its
// 16-byte chunks XOR-permuted by (r & 7); +2 in the encoded address = +32 B along K.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;                      // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>((1024u >> 4) & 0x3FFFu) << 32;  // SBO
  d |= static_cast<uint64_t>(1u) << 46;                      // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;                      // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M=128, N=n.
__device__ __forceinline__ uint32_t tf32_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t phase) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}\n"
      : "=r"(done)
      : "r"(a), "r"(phase), "r"(0x989680u)  // suspend in hardware until the phase flips (hint)
      : "memory");
  return done != 0;
}

// Wait for the phase with parity `phase` to complete.  Every try_wait a spinning warp
// issues takes an issue slot from the working warps of its sub-partition, so waits that
// are long by construction back off with __nanosleep (sleep_ns > 0) after a few tries;
// the MMA issuer (sleep_ns = 0) keeps polling.  A lost arrival traps instead of hanging.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase, uint32_t sleep_ns = 0) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try(a, phase)) return;
  for (long long spin = 0;; ++spin) {
    if (sleep_ns != 0 && spin >= 2) __nanosleep(sleep_ns);
    if (mbar_try(a, phase)) return;
    if (spin > (1ll << 26)) asm volatile("trap;");  // never hang the device on a lost arrival
  }
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (tcgen05.mma operands)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

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

__device__ __forceinline__ void tmem_st1(uint32_t taddr, float v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(__float_as_uint(v)));
}

// One tf32 MMA D (+)= A.B issued by one elected lane of a converged warp.
// TS: A from TMEM (column address), SS: A from shared memory (descriptor).
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

// Warp-converged forms for the MMA warp: every lane runs them, elect.sync picks the
// issuing lane inside the asm (tools/mma_rate.cu: MMAs issued from a diverged single
// thread lose ~half the tensor rate around any wait; from a converged warp none).
// A_hi.B (A in TMEM) then A_lo.B (A in shared memory), same B and accumulator.
__device__ __forceinline__ void mma_pair_elect(uint32_t d, uint32_t a_tmem, uint64_t a_lo, uint64_t b, uint32_t idesc,
                                               uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e, one;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %3, %4, one;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(a_lo), "l"(b), "r"(idesc), "r"(accum));
}
// One k-step of 4xTF32 in the only mixed order the tensor pipe runs at full rate
// (tools/mma_rate.cu: strict TS/SS alternation; 2 TS : 1 SS orders run at ~half rate):
// A_hi.B_hi (TS), A_lo.B_hi (SS), A_hi.B_lo (TS), A_lo.B_lo (SS).
__device__ __forceinline__ void mma_quad_elect(uint32_t d, uint32_t a_hi, uint64_t a_lo, uint64_t b_hi, uint64_t b_lo,
                                               uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e, one;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %3, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %4, %5, one;\n\t}\n" ::"r"(d),
      "r"(a_hi), "l"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(accum));
}
// One 32-wide K-block of 3xTF32 (4 k-steps, 12 MMAs) in one elected asm, in the order
// the pipe runs at full rate: the hi block as strict TS/SS pairs A_hi.B_hi, A_lo.B_hi
// over the 4 k-steps, then the lo block's 4 TS MMAs A_hi.B_lo (the order of the
// per-k-step form, so results are identical).  a_hi: TMEM column of k-step 0 (+8 per
// k-step); a_lo, b_hi, b_lo: descriptors of k-step 0 (+2 = 32 B per k-step inside the
// 128B swizzle atom).  accum = 0 starts the accumulator.
__device__ __forceinline__ void mma_kblock_elect(uint32_t d, uint32_t a_hi, uint64_t a_lo, uint64_t b_hi, uint64_t b_lo,
                                                 uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e, one;\n\t.reg .b32 r, a1, a2, a3;\n\t"
      ".reg .b64 l1, l2, l3, h1, h2, h3, o1, o2, o3;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "add.u64 l1, %2, 2;\n\tadd.u64 l2, %2, 4;\n\tadd.u64 l3, %2, 6;\n\t"
      "add.u64 h1, %3, 2;\n\tadd.u64 h2, %3, 4;\n\tadd.u64 h3, %3, 6;\n\t"
      "add.u64 o1, %4, 2;\n\tadd.u64 o2, %4, 4;\n\tadd.u64 o3, %4, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %3, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], h1, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], l1, h1, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a2], h2, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], l2, h2, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a3], h3, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], l3, h3, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], o1, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a2], o2, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a3], o3, %5, one;\n\t}\n" ::"r"(d),
      "r"(a_hi), "l"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(accum));
}
// 3xTF32 with both A parts in TMEM (TS only, the full-rate order), one 32-wide K-block
// split by weight part so each ring entry is released as soon as its MMAs are issued:
// the B_hi half (A_hi.B_hi, A_lo.B_hi per k-step, 2 nq MMAs) and the B_lo half (A_hi.B_lo).
__device__ __forceinline__ void mma_tt_bhi(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi, uint32_t idesc,
                                           uint32_t accum, int nq) {
  for (int q = 0; q < nq; ++q)
    asm volatile(
        "{\n\t.reg .pred p, e, one;\n\t.reg .b32 r;\n\t"
        "elect.sync r|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.b32 one, 0, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, one;\n\t}\n" ::"r"(d),
        "r"(a_hi + 8 * q), "r"(a_lo + 8 * q), "l"(b_hi + 2 * q), "r"((accum | q) != 0 ? 1u : 0u), "r"(idesc));
}
__device__ __forceinline__ void mma_tt_blo(uint32_t d, uint32_t a_hi, uint64_t b_lo, uint32_t idesc, int nq) {
  for (int q = 0; q < nq; ++q)
    asm volatile(
        "{\n\t.reg .pred e, one;\n\t.reg .b32 r;\n\t"
        "elect.sync r|e, 0xffffffff;\n\t"
        "setp.eq.b32 one, 0, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, one;\n\t}\n" ::"r"(d),
        "r"(a_hi + 8 * q), "l"(b_lo + 2 * q), "r"(idesc));
}

// The same two halves for a CTA pair (cta_group::2, idesc with M = 256): issued by rank 0.
__device__ __forceinline__ void mma_tt_bhi2(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi, uint32_t idesc,
                                            uint32_t accum, int nq) {
  for (int q = 0; q < nq; ++q)
    asm volatile(
        "{\n\t.reg .pred p, e, one;\n\t.reg .b32 r;\n\t"
        "elect.sync r|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.b32 one, 0, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %3, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%2], %3, %5, one;\n\t}\n" ::"r"(d),
        "r"(a_hi + 8 * q), "r"(a_lo + 8 * q), "l"(b_hi + 2 * q), "r"((accum | q) != 0 ? 1u : 0u), "r"(idesc));
}
__device__ __forceinline__ void mma_tt_blo2(uint32_t d, uint32_t a_hi, uint64_t b_lo, uint32_t idesc, int nq) {
  for (int q = 0; q < nq; ++q)
    asm volatile(
        "{\n\t.reg .pred e, one;\n\t.reg .b32 r;\n\t"
        "elect.sync r|e, 0xffffffff;\n\t"
        "setp.eq.b32 one, 0, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, one;\n\t}\n" ::"r"(d),
        "r"(a_hi + 8 * q), "l"(b_lo + 2 * q), "r"(idesc));
}

// ---- CTA pair (cta_group::2; tools/cta2_probe.cu checks the operand split): M = 256
// rows across the two CTAs of a cluster (128 in each CTA's TMEM / shared memory), B's N
// rows split between the CTAs' shared memory at the same offset (N/2 each), D = each
// CTA's 128 rows x N in its own TMEM.  Only rank 0 issues; commits multicast to both.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Arrive (release at cluster scope) on the mbarrier at the same offset in CTA `rank`.
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
// Whole-warp wait with cluster-scope acquire (arrivals from the peer CTA), trap on a
// lost arrival.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  for (long long spin = 0;; ++spin) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}\n"
        : "=r"(ok)
        : "r"(a), "r"(phase), "r"(0x989680u)
        : "memory");
    if (ok) return;
    if (spin > (1ll << 24)) asm volatile("trap;");
  }
}
// CTA pair: this CTA's half of a weight block by TMA (2-D tensor map over the float arena as
// [rows][32] fp32, box [h][32]) into its own shared memory, completing on rank 0's barrier at the
// same offset (.cta_group::2): rank 0's one expect_tx covers both halves, no relay.
__device__ __forceinline__ void tma_rows_to_rank0(void* dst, const void* tmap, int row, uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b32 rb;\n\tmapa.shared::cluster.u32 rb, %2, 0;\n\t"
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [rb];\n\t}\n"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(smem_u32(bar)), "r"(0), "r"(row)
      : "memory");
}
__device__ __forceinline__ void commit_pair_elect(uint64_t* bar) {  // arrive on `bar` in both CTAs
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
// mma_kblock_elect for the CTA pair (idesc with M = 256).
__device__ __forceinline__ void mma_kblock_pair_elect(uint32_t d, uint32_t a_hi, uint64_t a_lo, uint64_t b_hi,
                                                      uint64_t b_lo, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e, one;\n\t.reg .b32 r, a1, a2, a3;\n\t"
      ".reg .b64 l1, l2, l3, h1, h2, h3, o1, o2, o3;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "add.u64 l1, %2, 2;\n\tadd.u64 l2, %2, 4;\n\tadd.u64 l3, %2, 6;\n\t"
      "add.u64 h1, %3, 2;\n\tadd.u64 h2, %3, 4;\n\tadd.u64 h3, %3, 6;\n\t"
      "add.u64 o1, %4, 2;\n\tadd.u64 o2, %4, 4;\n\tadd.u64 o3, %4, 6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %3, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %2, %3, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [a1], h1, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], l1, h1, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [a2], h2, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], l2, h2, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [a3], h3, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], l3, h3, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %4, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [a1], o1, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [a2], o2, %5, one;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [a3], o3, %5, one;\n\t}\n" ::"r"(d),
      "r"(a_hi), "l"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(accum));
}
// Partial K-blocks of the pair: A_hi.B_hi (TS) + A_lo.B_hi (SS) pairs, then A_hi.B_lo (TS).
__device__ __forceinline__ void mma_pair2_elect(uint32_t d, uint32_t a_hi, uint64_t a_lo, uint64_t b, uint32_t idesc,
                                                uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e, one;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %3, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %2, %3, %4, one;\n\t}\n" ::"r"(d),
      "r"(a_hi), "l"(a_lo), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_ts2(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum));
}
// Instruction descriptor: D f32, A/B tf32, K-major, M, N.
__device__ __forceinline__ uint32_t tf32_idesc_mn(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
// Whole-warp wait in one asm loop (no per-iteration bookkeeping).
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(0x989680u)
      : "memory");
}

// Single-thread forms (the caller is the one issuing thread).
__device__ __forceinline__ void mma1_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma1_ts_acc(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.eq.b32 p, 0, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc));
}
__device__ __forceinline__ void mma1_ss_acc(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.eq.b32 p, 0, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc));
}
__device__ __forceinline__ void mma1_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
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

// Byte ring of weight blocks placed back to back, wrapping to 0 when a block does
// not fit.  Producer and MMA issuer walk the same sequence and place block by block.
__device__ __forceinline__ uint32_t ring_place(uint32_t& pos, uint32_t bytes, uint32_t ring) {
  if (pos + bytes > ring) pos = 0;
  const uint32_t at = pos;
  pos += bytes;
  return at;
}

}  // namespace tc
}  // namespace bp

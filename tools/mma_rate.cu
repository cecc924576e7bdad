// Microbenchmark (dev helper): cycles per tcgen05.mma dispatch on one SM for the
// shapes the rollout uses.  Operand contents are zeros; only the rate matters.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_mma_rate tools/mma_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t sw128(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= 1ull << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

__device__ __forceinline__ uint32_t idesc(int fmt, int n, int m = 128) {  // fmt 2: tf32 (kind::tf32), 1: bf16 (kind::f16)
  return (1u << 4) | (static_cast<uint32_t>(fmt) << 7) | (static_cast<uint32_t>(fmt) << 10) |
         (static_cast<uint32_t>(n >> 3) << 17) | ((static_cast<uint32_t>(m) >> 4) << 24);
}

template <int V>
__device__ __forceinline__ void issue(uint32_t d, uint32_t ta, uint64_t da, uint64_t db, uint32_t id) {
  if constexpr (V == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(d), "r"(ta), "l"(db), "r"(id));
  else if constexpr (V == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(da), "l"(db), "r"(id));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(da), "l"(db), "r"(id));
}

// V 3: TS and SS tf32 alternating (the 3xTF32 hi.hi / lo.hi pattern with lo in smem)
// V 4: TS, SS, TS per step (hi.hi, lo.hi, hi.lo)
template <int V>
__device__ __forceinline__ void issue_mix(int i, uint32_t d, uint32_t ta, uint64_t da, uint64_t db, uint32_t id) {
  if constexpr (V == 3) {
    if (i & 1) issue<1>(d, ta, da, db, id); else issue<0>(d, ta, da, db, id);
  } else {
    if (i % 3 == 1) issue<1>(d, ta, da, db, id); else issue<0>(d, ta, da, db, id);
  }
}

__device__ volatile int g_stop;

// V: 0 TS tf32, 1 SS tf32, 2 SS bf16.  N: MMA N.  I: interference from warps 1-3 while
// the MMAs run (0 none, 1 LDS.128 stream, 2 tcgen05.ld x32 stream, 3 STS.128 stream,
// 4 tcgen05.st x32 stream).
__device__ float g_src[65536];

template <int V, int N, int I = 0, int NI = 3>
__global__ void rate(int n_mma, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar, xbar, ybar;
  __shared__ int flag;
  if (threadIdx.x == 0) flag = 7;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024; i += blockDim.x) sm[i] = static_cast<unsigned char>((i * 2654435761u) >> 24) & 0x3f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(su32(&xbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&ybar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  __shared__ uint64_t cbar[2];
  if (I == 11 && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (I == 11) {
    if (threadIdx.x == 32) {
      uint32_t ph[2] = {0, 0};
      int k = 0;
      for (int it = 0; !stop && it < 100000; ++it, k ^= 1) {
        if (it >= 2) {
          uint32_t done = 0;
          while (!done)
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                         : "=r"(done) : "r"(su32(&cbar[k])), "r"(ph[k]));
          ph[k] ^= 1;
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&cbar[k])), "r"(16384));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sm + 65536 + 16384 * k)), "l"(g_src + 4096 * (it & 7)), "r"(16384), "r"(su32(&cbar[k])));
      }
    }
  }
  const bool only_sp0 = I >= 7;
  const int wq = threadIdx.x >> 5;
  const bool interferer = I != 0 && I != 11 && threadIdx.x >= 32 && !(I == 6 && wq % 4 == 0) &&
                          (!only_sp0 || (wq % 4 == 0 && wq / 4 <= NI));
  if (interferer) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float acc = 0.f;
    float4* region = reinterpret_cast<float4*>(sm + 65536);
    while (!stop) {
      for (int r = 0; r < 64; ++r) {
        if constexpr (I == 1) {
          const float4 v = region[(r * 32 + lane) & 1023];
          acc += v.x + v.y + v.z + v.w;
        } else if constexpr (I == 3) {
          region[(r * 32 + lane + w * 7) & 1023] = make_float4(acc, acc, acc, acc);
          acc += 1.f;
        } else if constexpr (I == 2) {
          uint32_t x[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
              "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
              : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]), "=r"(x[8]),
                "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15]), "=r"(x[16]),
                "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]), "=r"(x[21]), "=r"(x[22]), "=r"(x[23]), "=r"(x[24]),
                "=r"(x[25]), "=r"(x[26]), "=r"(x[27]), "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
              : "r"(tm + 384 + ((32u * w) << 16)));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          acc += __uint_as_float(x[r & 31]);
        } else if constexpr (I == 8) {  // FMNMX / FSEL chains
          float b0 = acc, b1 = acc + 1.f, b2 = acc + 2.f, b3 = acc + 3.f;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            b0 = fminf(b1, b0 + 0.5f);
            b1 = fmaxf(b2, b1 - 0.25f);
            b2 = (lane & q) ? b3 : b2 * 0.5f;
            b3 = fminf(b3, b0);
          }
          acc = b0 + b1 + b2 + b3;
        } else if constexpr (I == 9) {  // shuffle butterfly
          float b0 = acc;
#pragma unroll
          for (int q = 0; q < 16; ++q) b0 = fminf(b0, __shfl_xor_sync(0xffffffffu, b0, 1 << (q & 4)));
          acc += b0;
        } else if constexpr (I == 10) {  // integer ALU
          uint32_t x0 = __float_as_uint(acc), x1 = x0 + 7, x2 = x0 ^ 0x55, x3 = x0 * 3;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            x0 = (x0 ^ x1) + q;
            x1 = (x1 & x2) | x3;
            x2 = x2 + (x3 >> 1);
            x3 = x3 ^ (x0 << 2);
          }
          acc += __uint_as_float((x0 ^ x1 ^ x2 ^ x3) & 0x3fffffff);
        } else if constexpr (I == 5 || I == 6 || I == 7) {
          float b0 = acc, b1 = acc + 1.f, b2 = acc + 2.f, b3 = acc + 3.f;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            b0 = fmaf(b0, 1.0001f, 0.5f);
            b1 = fmaf(b1, 1.0001f, 0.5f);
            b2 = fmaf(b2, 1.0001f, 0.5f);
            b3 = fmaf(b3, 1.0001f, 0.5f);
          }
          acc = b0 + b1 + b2 + b3;
        } else {
          uint32_t x = __float_as_uint(acc);
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
              "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(tm + 384 + ((32u * w) << 16)),
              "r"(x));
          asm volatile("tcgen05.wait::st.sync.aligned;");
          acc += 1.f;
        }
      }
    }
    if (acc == 12345.f) out[1] = 1;
  }
  if (V >= 19 && threadIdx.x < 32) {
    const int ln = threadIdx.x;
    const uint32_t id = idesc(2, N);
    const uint64_t da = sw128(su32(sm)), db = sw128(su32(sm + 32768));
    const long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const uint64_t b = db + 2 * (i & 3) + 256 * ((i >> 2) & 7);
      const uint64_t aa = da + 2 * (i & 3) + 256 * ((i >> 2) & 3);
      if (V == 33) {  // 4xTF32 per k-step: TS(hi,Bhi) SS(lo,Bhi) TS(hi,Blo) SS(lo,Blo); commit every 16
        const int j = i % 16;
        const int q = j >> 2, p = j & 3;
        const uint64_t bq = db + 2 * q + 1024 * ((i / 16) & 1) + (p >= 2 ? 512 : 0);
        if (p & 1)
          asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da + 2 * q), "l"(bq), "r"(id));
        else
          asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm), "r"(tm + 256 + 8 * q), "l"(bq), "r"(id));
        if (j == 15) {
          asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                       "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&xbar)));
          asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t@!P1 bra WAIT_%=;\n\t}"
                       ::"r"(su32(&ybar)), "r"(1u), "r"(0x989680u) : "memory");
        }
        continue;
      }
      if (V == 29 || V == 30 || V == 31 || V == 32) {  // 29: pure TS, A walks 8q, B walks; 30: per k-step TS(hi.hi), SS(lo.hi), TS(hi.lo)
        const int j = i % 12;
        const int q = (V == 29 || V >= 31) ? (j & 3) : j / 3;
        const uint64_t bq = db + 2 * q + 1024 * ((i / 12) & 1) + (V >= 31 && (j >> 2) == 1 ? 512 : 0);
        const bool ss = (V == 30 && (j % 3) == 1) || (V == 31 && j >= 8) || (V == 32 && j < 4);
        if (ss)
          asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da + 2 * q), "l"(bq), "r"(id));
        else
          asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm), "r"(tm + 256 + 8 * q), "l"(bq), "r"(id));
        if (j == 11)
          asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                       "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&xbar)));
        continue;
      }
      if (V >= 23 && V <= 28) {  // the v2 kernel pattern: 12 MMAs = 4 x (TS, SS) + 4 x TS, commit+wait after 8 and 12
        const int j = i % 12;
        const int q = j < 8 ? (j >> 1) : j - 8;
        const uint64_t bq = db + 2 * q + 1024 * ((i / 12) & 1);
        if ((V == 28 ? true : j < 8) && (j & 1))
          asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da + 2 * q), "l"(bq), "r"(id));
        else
          asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                       "r"(tm + 256 + (V == 25 ? 0 : V == 26 ? 32 * q : 8 * q)), "l"(bq), "r"(id));
        if ((j == 7 || j == 11) && V != 27) {
          asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                       "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&xbar)));
          if (V == 23)
            asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t@!P1 bra WAIT_%=;\n\t}"
                         ::"r"(su32(&ybar)), "r"(1u), "r"(0x989680u) : "memory");
        }
        continue;
      }
      if (V >= 80 && V < 90) {
        // per 12-MMA group (issued at j == 0): 80 one asm block for all 12 (one elect);
        // 81 per k-step {TS hi.Bhi, SS lo.Bhi, TS hi.Blo} (mma3 style, 4 asm blocks);
        // 82/83 as 80/81 plus commit + wait after the group
        const int j = i % 12;
        if (j != 0) continue;
        if (V == 80 || V == 82) {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %3, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%6], %7, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %8, %7, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%9], %10, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %11, %10, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%12], %13, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %14, %13, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%6], %15, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%9], %16, %5, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%12], %17, %5, p;\n\t}"
              ::"r"(tm), "r"(tm + 256), "l"(da), "l"(db), "l"(db + 512), "r"(id),
              "r"(tm + 264), "l"(db + 2), "l"(da + 2), "r"(tm + 272), "l"(db + 4), "l"(da + 4),
              "r"(tm + 280), "l"(db + 6), "l"(da + 6), "l"(db + 514), "l"(db + 516), "l"(db + 518));
        } else {
          for (int q = 0; q < 4; ++q)
            asm volatile(
                "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, p;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %3, %5, p;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, p;\n\t}"
                ::"r"(tm), "r"(tm + 256 + 8 * q), "l"(da + 2 * q), "l"(db + 2 * q), "l"(db + 512 + 2 * q), "r"(id));
        }
        if (V >= 82) {
          asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                       "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&xbar)));
          asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t@!P1 bra WAIT_%=;\n\t}"
                       ::"r"(su32(&ybar)), "r"(1u), "r"(0x989680u) : "memory");
        }
        continue;
      }
      if (V >= 70 && V < 80) {  // v2 MMA warp: 4 elected pairs (TS,SS), [commit+wait], 4 elected TS, [commit+wait]
        // 70: commits + waits; 71: no commit/wait; 72: commit only; 73: wait only; 74: lo TS as elected pairs of 2
        const int j = i % 12;
        const int q = j < 8 ? (j >> 1) : j - 8;
        const uint64_t b = db + 2 * q + (j >= 8 ? 512 : 0);
        const bool ss = j < 8 && (j & 1);
        if (ss)
          asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da + 2 * q), "l"(b), "r"(id));
        else
          asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm), "r"(tm + 256 + 8 * q), "l"(b), "r"(id));
        if (j == 7 || j == 11) {
          if (V == 70 || V == 72)
            asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&xbar)));
          if (V == 70 || V == 73)
            asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t@!P1 bra WAIT_%=;\n\t}"
                         ::"r"(su32(&ybar)), "r"(1u), "r"(0x989680u) : "memory");
        }
        continue;
      }
      if (V >= 21) {  // elected lane inside the asm, the whole warp converged (v1 style)
        if (i & 1)
          asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(aa), "l"(b), "r"(id));
        else
          asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm), "r"(tm + 256), "l"(b), "r"(id));
        if (V >= 21 && i % 12 == 11) {
          uint32_t done = 0;
          if (V == 21)
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                         : "=r"(done) : "r"(su32(&ybar)), "r"(1u), "r"(0x989680u));
          else
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                         : "=r"(done) : "r"(su32(&ybar)), "r"(1u));
          if (!done) out[2] = 1;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                       "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&xbar)));
        }
        continue;
      }
      if (ln == 0) {
        if (i & 1) issue<1>(tm, tm + 256, aa, b, id); else issue<0>(tm, tm + 256, aa, b, id);
      }
      if (i % 12 == 11) {
        uint32_t done = 0;
        if (ln == 1) {
          if constexpr (V == 19)
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                         : "=r"(done) : "r"(su32(&ybar)), "r"(1u));
          else
            asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(done) : "r"(su32(&flag)));
        }
        done = __shfl_sync(0xffffffffu, done, 1);
        if (!done) out[2] = 1;
        if (ln == 0) {
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&xbar)));
        }
      }
    }
    if (ln == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
      uint32_t dn = 0;
      while (!dn)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                     : "=r"(dn) : "r"(su32(&bar)));
      const long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
      stop = 1;
    }
  } else if (V < 19 && threadIdx.x == 0) {
    const uint32_t id = (V >= 40 && V < 50) ? idesc(2, N, 64) : idesc(V == 2 ? 1 : 2, N);  // V 3..6: tf32
    const uint64_t da = sw128(su32(sm)), db = sw128(su32(sm + 32768));
    const long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      if constexpr (V >= 60 && V < 70) {
        // v2 kernel pattern per 12: q=0..3 {TS(Ahi_q,Bhi_q), SS(Alo_q,Bhi_q)}, q=0..3 TS(Ahi_q,Blo_q)
        // 61: lo-run reads other A columns; 62: SS uses another B than its TS partner; 63: lo-run reversed;
        // 64: pairs reordered SS first; 65: B blocks advance every 12 (fresh per group)
        const int j = i % 12, g = (i / 12) & 7;
        const uint64_t bbase = db + (V == 65 ? 512 * g : 0);
        int q;
        bool ss;
        uint64_t b;
        uint32_t acol;
        if (j < 8) {
          q = j >> 1;
          const bool second = (j & 1) != 0;
          ss = (V == 64) ? !second : second;
          b = bbase + 2 * q + ((V == 62 && ss) ? 256 : 0);
          acol = 8 * q;
        } else {
          q = V == 63 ? 11 - j : j - 8;
          ss = false;
          b = bbase + 256 * 2 + 2 * q;
          acol = (V == 61 ? 64 : 0) + 8 * q;
        }
        if (ss) issue<1>(tm, tm + 256, da + 2 * q, b, id); else issue<0>(tm, tm + 256 + acol, da, b, id);
      } else if constexpr (V >= 50 && V < 60) {  // runs: (2^(V-50)*8) TS then half as many SS
        const int run = 8 << (V - 50), per = run + run / 2;
        const int j = i % per;
        const uint64_t b = db + 2 * (i & 3) + 256 * ((i >> 2) & 7);
        if (j >= run) issue<1>(tm, tm + 256, da + 2 * (i & 3), b, id); else issue<0>(tm, tm + 256 + 8 * (i & 3), da, b, id);
      } else if constexpr (V >= 40) {
        const uint64_t b = db + 2 * (i & 3) + 256 * ((i >> 2) & 7);
        const uint32_t dl = (V == 42 && (i & 1)) ? (16u << 16) : 0u;  // second tile: lanes +16 per quadrant
        if (V == 41)
          issue<1>(tm + dl, tm + 256, da + 2 * (i & 3), b, id);
        else
          issue<0>(tm + dl, tm + 256 + dl, da, b, id);
      } else if constexpr (V >= 7) {
        const uint64_t b = db + 2 * (i & 3) + 256 * ((i >> 2) & 7);
        const uint64_t aa = da + 2 * (i & 3) + 256 * ((i >> 2) & 3);
        if (i & 1) issue<1>(tm, tm + 256, aa, b, id); else issue<0>(tm, tm + 256, aa, b, id);
        constexpr int P = (V == 13) ? 24 : 12;
        if (i % P == P - 1) {
          // V 7 commit, 8 fence, 9 try_wait, 10 test_wait, 11 commit+try_wait, 12 all three, 13 all three per 24
          if constexpr (V == 7 || V == 11 || V == 12 || V == 13)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&xbar)));
          if constexpr (V == 9 || V == 11 || V == 12 || V == 13) {
            uint32_t done = 0;
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                         : "=r"(done) : "r"(su32(&ybar)), "r"(1u));
            if (!done) out[2] = 1;
          }
          if constexpr (V == 14 || V == 15) {
            uint32_t done = 0;
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                         : "=r"(done) : "r"(su32(&ybar)), "r"(1u));
            if (!done) out[2] = 1;
          }
          if constexpr (V == 15) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&xbar)));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          if constexpr (V == 16) {
            int f;
            asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(f) : "r"(su32(&flag)));
            if (f != 7) out[2] = 1;
          }
          if constexpr (V == 17) {
            int f;
            asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(f) : "r"(su32(&flag)));
            if (f != 7) out[2] = 1;
          }
          if constexpr (V == 18) {
            int f;
            asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(f) : "r"(su32(&flag)));
            if (f != 7) out[2] = 1;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&xbar)));
          }
          if constexpr (V == 10) {
            uint32_t done = 0;
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                         : "=r"(done) : "r"(su32(&ybar)), "r"(1u));
            if (!done) out[2] = 1;
          }
          if constexpr (V == 8 || V == 12 || V == 13) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
      } else if constexpr (V >= 5) {  // fresh operands: B walks 8 K-blocks of 4 KB... (32 KB), A 4 blocks (16 KB)
        const uint64_t b = db + 2 * (i & 3) + 256 * ((i >> 2) & 7);
        const uint64_t aa = da + 2 * (i & 3) + 256 * ((i >> 2) & 3);
        if (V == 5 || (i & 1)) issue<1>(tm, tm + 256, aa, b, id); else issue<0>(tm, tm + 256, aa, b, id);
      } else if constexpr (V >= 3)
        issue_mix<V>(i, tm, tm + 256, da + 2 * (i & 3), db + 2 * (i & 3), id);
      else
        issue<V>(tm, tm + 256, da + 2 * (i & 3), db + 2 * (i & 3), id);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                   : "=r"(done) : "r"(su32(&bar)));
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int V, int N, int I = 0, int NI = 3>
void run(const char* name, int grid) {
  long long* d;
  cudaMalloc(&d, 16);
  auto k = rate<V, N, I, NI>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 97 * 1024);
  for (int n : {64, 1024}) {
    k<<<grid, I >= 5 ? 512 : 128, 97 * 1024>>>(n, d);
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * N * (V == 2 ? 16 : 8);
    std::printf("%-14s grid %3d n=%5d: %7.1f cyc/mma  (%6.0f flop/cyc/SM)\n", name, grid, n, double(c) / n,
                flops * n / double(c));
  }
  cudaFree(d);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
}

int main() {
#ifdef MMA_RATE_N256
  run<0, 128, 0>("TS n128", 148);
  run<0, 256, 0>("TS n256", 148);
  run<1, 256, 0>("SS n256", 148);
  run<3, 256, 0>("TS/SS n256", 148);
  run<6, 256, 0>("fresh TS/SS n256", 148);
  run<0, 256, 2>("TS n256 +ld", 148);
  run<0, 256, 4>("TS n256 +st", 148);
  run<0, 32, 0>("TS n32", 148);
  run<0, 16, 0>("TS n16", 148);
  return 0;
#endif
  run<71, 128, 0>("per-MMA elect", 148);
  run<80, 128, 0>("12 in one asm", 148);
  run<81, 128, 0>("mma3 per kstep", 148);
  run<82, 128, 0>("12 in one asm +c/w", 148);
  run<83, 128, 0>("mma3 per kstep +c/w", 148);
  return 0;
}

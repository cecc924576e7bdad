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

__device__ __forceinline__ uint32_t idesc(int fmt, int n) {  // fmt 2: tf32 (kind::tf32), 1: bf16 (kind::f16)
  return (1u << 4) | (static_cast<uint32_t>(fmt) << 7) | (static_cast<uint32_t>(fmt) << 10) |
         (static_cast<uint32_t>(n >> 3) << 17) | ((128u >> 4) << 24);
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
template <int V, int N, int I = 0>
__global__ void rate(int n_mma, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024; i += blockDim.x) sm[i] = static_cast<unsigned char>((i * 2654435761u) >> 24) & 0x3f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
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
  if (I != 0 && threadIdx.x >= 32 && !(I == 6 && (threadIdx.x >> 5) % 4 == 0)) {
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
        } else if constexpr (I == 5 || I == 6) {
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
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(V == 2 ? 1 : 2, N);  // V 3, 4: tf32
    const uint64_t da = sw128(su32(sm)), db = sw128(su32(sm + 32768));
    const long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      if constexpr (V >= 3)
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

template <int V, int N, int I = 0>
void run(const char* name, int grid) {
  long long* d;
  cudaMalloc(&d, 16);
  auto k = rate<V, N, I>;
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
  run<3, 128>("TS/SS alt N128", 148);
  run<4, 128>("TS,SS,TS N128", 148);
  run<3, 128, 3>("TS/SS alt +STS", 148);
  run<1, 128, 3>("SS N128 +STS", 148);
  run<0, 128, 5>("TS N128 +ALU15", 148);
  run<1, 128, 5>("SS N128 +ALU15", 148);
  run<0, 128, 6>("TS N128 +ALU12 other SPs", 148);
  run<0, 128, 1>("TS N128 +LDS", 148);
  run<0, 128, 2>("TS N128 +LDTM", 148);
  run<0, 128, 3>("TS N128 +STS", 148);
  run<0, 128, 4>("TS N128 +STTM", 148);
  run<1, 128, 1>("SS N128 +LDS", 148);
  run<1, 128, 3>("SS N128 +STS", 148);
  for (int grid : {148}) {
    run<0, 128>("TS tf32 N128", grid);
    run<1, 128>("SS tf32 N128", grid);
    run<0, 256>("TS tf32 N256", grid);
    run<1, 256>("SS tf32 N256", grid);
    run<0, 64>("TS tf32 N64", grid);
    run<2, 128>("SS bf16 N128", grid);
    run<2, 256>("SS bf16 N256", grid);
  }
  return 0;
}

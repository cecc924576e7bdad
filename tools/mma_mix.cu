// Microbenchmark (dev helper): cycles per "K-block group" of the tc3 MMA mix on every SM --
// 12 TS-only N=256 layer-1 MMAs (A hi / lo in TMEM) followed by 9 N=32 layer-0 MMAs (TS/SS
// pairs + TS), all operands resident, issued by one converged warp, commit + wait every G groups.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_mma_mix tools/mma_mix.cu
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
__device__ __forceinline__ uint32_t idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id));
}

template <int MODE>
__global__ void mix(int groups, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024; i += blockDim.x) sm[i] = 0;
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
  if (threadIdx.x < 32) {
    const uint64_t bw1 = sw128(su32(sm)), bw0 = sw128(su32(sm + 65536)), ax = sw128(su32(sm + 65536 + 8192));
    const uint32_t i256 = idesc(256), i32 = idesc(32);
    uint32_t ph = 0;
    const long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      // layer 1: 4 k-steps of (hi.Bhi, lo.Bhi) then 4 of hi.Blo, N = 256, A in TMEM cols 288.. / 320..
      for (int q = 0; q < 4; ++q) {
        ts(tm, tm + 288 + 8 * q, bw1 + 2 * q, i256);
        ts(tm, tm + 320 + 8 * q, bw1 + 2 * q, i256);
      }
      for (int q = 0; q < 4; ++q) ts(tm, tm + 288 + 8 * q, bw1 + 2048 + 2 * q, i256);
      if (MODE >= 1) {
        // layer 0: 3 k-steps (TS X hi, SS X lo) on W0 hi then TS on W0 lo, N = 32 into cols 352..
        for (int q = 0; q < 3; ++q) {
          ts(tm + 352, tm + 256 + 8 * q, bw0 + 2 * q, i32);
          ss(tm + 352, ax + 2 * q, bw0 + 2 * q, i32);
        }
        for (int q = 0; q < 3; ++q) ts(tm + 352, tm + 256 + 8 * q, bw0 + 256 + 2 * q, i32);
      }
      if (MODE == 2 || (MODE == 3 && (g & 3) == 3)) {  // commit + wait (drain) every group / every 4 groups
        asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar)));
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                       : "=r"(done) : "r"(su32(&bar)), "r"(ph));
        ph ^= 1;
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                   : "=r"(done) : "r"(su32(&bar)), "r"(ph));
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int MODE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mix<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 97 * 1024);
  for (int g : {16, 256}) {
    mix<MODE><<<148, 128, 97 * 1024>>>(g, d);
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    std::printf("%-28s groups %4d: %7.0f cycles/group\n", name, g, double(c) / g);
  }
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("L1 only (12 x N256)");
  run<1>("L1 + L0 (12 x N256 + 9 x N32)");
  run<2>("L1 + L0, drain every group");
  run<3>("L1 + L0, drain every 4");
  return 0;
}

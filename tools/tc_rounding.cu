// Microbenchmark (dev helper): how kind::tf32 tcgen05.mma rounds the FP32 accumulation.
// D starts at 1.0 (first MMA: A = [1, 0...], B = [1, 0...]); a second MMA adds a.b with
// a.b = +-0.75 ulp(1) (exactly representable): round-to-nearest gives 1 +- 2^-23, truncation
// (round toward zero) gives 1 (for +) / 1 - 2^-24 (for -).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_tc_rounding tools/tc_rounding.cu
#include <cstdint>
#include <cstdio>
#include <cstring>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sw128(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= 1ull << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}
__global__ void k(float add, float* out) {
  extern __shared__ __align__(1024) float sm[];  // A: 128 rows x 32, B: 16 rows x 32 (SW128: chunk q of row r at (q ^ (r & 7)))
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  float* A = sm;
  float* B = sm + 128 * 32;
  for (int i = threadIdx.x; i < 128 * 32 + 16 * 32; i += blockDim.x) sm[i] = 0.f;
  __syncthreads();
  if (threadIdx.x < 128) A[threadIdx.x * 32 + ((0 ^ (threadIdx.x & 7)) << 2)] = 1.0f;  // A[r][0] = 1
  if (threadIdx.x < 16) B[threadIdx.x * 32 + ((0 ^ (threadIdx.x & 7)) << 2)] = 1.0f;   // B[n][0] = 1 (k-step 0)
  // k-step 1 (k = 8): A[r][8] = 1, B[n][8] = add
  if (threadIdx.x < 128) A[threadIdx.x * 32 + ((2 ^ (threadIdx.x & 7)) << 2)] = 1.0f;
  if (threadIdx.x < 16) B[threadIdx.x * 32 + ((2 ^ (threadIdx.x & 7)) << 2)] = add;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint64_t da = sw128(su32(A)), db = sw128(su32(B));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da), "l"(db), "r"(id));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da + 2), "l"(db + 2), "r"(id));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(done) : "r"(su32(&bar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (threadIdx.x == 0) out[0] = __uint_as_float(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}
int main() {
  float* d;
  cudaMalloc(&d, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  const float ulp = 1.0f / 8388608.0f;  // 2^-23
  for (float f : {0.75f, 0.5f, 0.25f, -0.25f, -0.5f, -0.75f}) {
    k<<<1, 128, 32 * 1024>>>(f * ulp, d);
    float h = 0;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    const float rn = 1.0f + f * ulp;  // IEEE round-to-nearest of the exact sum
    std::printf("1 + %+.2f ulp: tcgen05 %.10g (%+.3f ulp)   RN %.10g\n", f, h, (h - 1.0) / ulp, rn);
  }
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
  return 0;
}

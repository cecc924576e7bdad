// cta2_probe.cu -- standalone probe of the CTA-pair MMA (tcgen05 cta_group::2) that a
// future rollout kernel would use: M = 256 rows across two CTAs of a cluster (128 rows
// of A in each CTA's TMEM), B = N rows split across the two CTAs' shared memory (N/2
// each, same offset), D = each CTA's 128 rows x N columns in its own TMEM.  Checks the
// operand split and the commit multicast against a host product.  Not part of the
// library.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o cta2_probe tools/cta2_probe.cu && ./cta2_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int K = 32, N = 64, NH = N / 2;  // B rows per CTA
constexpr uint32_t kColD = 0, kColA = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>((1024u >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}
// D f32, A/B tf32, K-major, M, N
__device__ __forceinline__ uint32_t idesc(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const float* A, const float* B, float* D, int m_field) {
  __shared__ __align__(1024) float bsm[NH * 32];  // NH rows x 128 B, SW128 K-major
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t done;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B rows of this CTA: global rows rank*NH .. +NH, K values 0..31 swizzled
  for (int i = tid; i < NH * 32; i += 128) {
    const int r = i / 32, k = i % 32;
    bsm[r * 32 + (((k >> 2) ^ (r & 7)) << 2) + (k & 3)] = B[(rank * NH + r) * K + k];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  // A: row = 32*warp + lane of this CTA (global row rank*128 + row), K columns at kColA
  {
    uint32_t v[32];
    for (int k = 0; k < K; ++k) v[k] = __float_as_uint(A[(rank * 128 + 32 * warp + lane) * K + k]);
    const uint32_t ta = tmem + (static_cast<uint32_t>(32 * warp) << 16) + kColA;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(ta),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (rank == 0 && warp == 0) {
    const uint64_t b0 = sw128_desc(smem_u32(bsm));
    const uint32_t id = idesc(m_field, N);
    for (int q = 0; q < K / 8; ++q) {
      asm volatile(
          "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
          "elect.sync r|e, 0xffffffff;\n\t"
          "setp.ne.b32 p, %4, 0;\n\t"
          "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem + kColD),
          "r"(tmem + kColA + 8 * q), "l"(b0 + 2 * q), "r"(id), "r"(q > 0 ? 1u : 0u));
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
            smem_u32(&done)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  }
  // both CTAs: wait for the product, read this CTA's 128 rows x N
  {
    uint32_t ok = 0;
    for (long long spin = 0; !ok; ++spin) {
      asm volatile(
          "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
          : "=r"(ok)
          : "r"(smem_u32(&done))
          : "memory");
      if (spin > (1ll << 26)) asm volatile("trap;");
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + (static_cast<uint32_t>(32 * warp) << 16) + kColD + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) D[(rank * 128 + 32 * warp + lane) * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

int main(int argc, char** argv) {
  const int m_field = argc > 1 ? atoi(argv[1]) : 256;
  std::vector<float> A(256 * K), B(N * K), D(256 * N, -1.f);
  for (int i = 0; i < 256 * K; ++i) A[i] = static_cast<float>((i * 7 + 3) % 9 - 4);
  for (int i = 0; i < N * K; ++i) B[i] = static_cast<float>((i * 5 + 1) % 7 - 3);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dD, D.data(), D.size() * 4, cudaMemcpyHostToDevice);
  probe<<<2, 128>>>(dA, dB, dD, m_field);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  // hypothesis: D[r][n] = sum_k A[r][k] B[n][k] over all 256 rows and N columns
  int bad = 0;
  double maxerr = 0;
  for (int r = 0; r < 256; ++r)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += static_cast<double>(A[r * K + k]) * B[n * K + k];
      const double err = std::abs(ref - D[r * N + n]);
      maxerr = err > maxerr ? err : maxerr;
      if (err > 1e-3 && bad++ < 5) printf("mismatch r=%d n=%d ref=%g got=%g\n", r, n, ref, D[r * N + n]);
    }
  printf("M field %d: %d mismatches of %d, max err %g\n", m_field, bad, 256 * N, maxerr);
  return bad ? 2 : 0;
}

// diag.cu -- peak microbenchmarks for the roofline denominators that
// MEASURED_PEAKS.json does not carry (it has copy bandwidth and bf16 tensor
// peaks only): FP32 FFMA (the SIMT rollout) and dense kind::tf32 tcgen05.mma
// (the tensor-core rollout; 3xTF32 issues three per FP32 product).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/babplan_cuda.h"

namespace {

__global__ void __launch_bounds__(256) ffma_kernel(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 123.456f) out[0] = s;  // keep the chains alive
}

// GEMM-shaped variant: every FFMA reads three distinct registers (acc += x * w).
__global__ void __launch_bounds__(256) ffma_reg_kernel(float* out, int iters, float a, float b) {
  float acc[16], x[4], w[4];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[i] = a + (threadIdx.x + i) * 1e-7f;
    w[i] = b - (threadIdx.x * 3 + i) * 1e-7f;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i * 4 + j] = fmaf(x[i], w[j], acc[i * 4 + j]);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 123.456f) out[0] = s;
}

// One CTA per SM: one elected thread issues back-to-back M=128 N=128 K=8
// kind::tf32 MMAs (A from TMEM, B from shared memory) -- the rollout's shape.
__global__ void __launch_bounds__(128, 1) tf32_mma_kernel(int n_mma, int* err) {
  __shared__ __align__(1024) unsigned char b_tile[16384];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(b_tile)[i] = 1e-3f * (i & 15);
  const uint32_t bar_a = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(&slot))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(b_tile));
    const uint64_t desc = static_cast<uint64_t>((sa >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    for (int i = 0; i < n_mma; ++i)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                   "r"(tm + 128 + 8 * (i & 7)), "l"(desc + 2 * (i & 3)), "r"(idesc), "r"(i));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_a));
    uint32_t done = 0;
    long long spin = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                   : "=r"(done)
                   : "r"(bar_a));
      if (++spin > (1ll << 30)) {
        atomicExch(err, 1);
        break;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

}  // namespace

extern "C" bp_status bp_measure_tf32_peak(int device, double* tflops, double* ms_out) {
  if (cudaSetDevice(device) != cudaSuccess) return BP_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int* err = nullptr;
  if (cudaMalloc(&err, 4) != cudaSuccess) return BP_CUDA;
  cudaMemset(err, 0, 4);
  const int n_mma = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    tf32_mma_kernel<<<sms, 128>>>(n_mma, err);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  int h_err = 0;
  cudaMemcpy(&h_err, err, 4, cudaMemcpyDeviceToHost);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(err);
  if (cudaGetLastError() != cudaSuccess || h_err) return BP_CUDA;
  const double flops = 2.0 * 128 * 128 * 8 * static_cast<double>(n_mma) * sms;
  *tflops = flops / (best * 1e-3) / 1e12;
  if (ms_out) *ms_out = best;
  return BP_OK;
}

extern "C" bp_status bp_measure_fp32_peak_reg(int device, double* tflops, double* ms_out) {
  if (cudaSetDevice(device) != cudaSuccess) return BP_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if (cudaMalloc(&out, 4) != cudaSuccess) return BP_CUDA;
  const int blocks = sms * 8, threads = 256, iters = 1 << 15;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    ffma_reg_kernel<<<blocks, threads>>>(out, iters, 0.9999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaFree(out);
  const double flops = 2.0 * 16 * static_cast<double>(iters) * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  if (ms_out) *ms_out = best;
  return BP_OK;
}

extern "C" bp_status bp_measure_fp32_peak(int device, double* tflops, double* ms_out) {
  if (cudaSetDevice(device) != cudaSuccess) return BP_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if (cudaMalloc(&out, 4) != cudaSuccess) return BP_CUDA;
  const int blocks = sms * 8, threads = 256, iters = 1 << 15;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    ffma_kernel<<<blocks, threads>>>(out, iters, 0.9999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return BP_CUDA;
  const double flops = 2.0 * 16 * static_cast<double>(iters) * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  if (ms_out) *ms_out = best;
  return BP_OK;
}

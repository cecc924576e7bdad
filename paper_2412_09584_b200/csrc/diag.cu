// diag.cu -- FP32 FMA peak microbenchmark (the SIMT roofline denominator;
// MEASURED_PEAKS.json has copy bandwidth and bf16 tensor peaks only).
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

}  // namespace

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

// FP64 roofline denominator: DFMA throughput of the device, measured with
// independent register-resident FMA chains (MEASURED_PEAKS.json has only HBM
// and bf16; SURVEY.md §8(d) asks for a measured fp64 peak).
#include <cuda_runtime.h>

#include "../../include/hdivred_b200.h"
#include "kernels.hpp"

namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) k_dfma(double* out, double seed) {
  double a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = seed + threadIdx.x * 1e-9 + c;
  const double m = 0.999999999, q = 1e-12;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = fma(a[c], m, q);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += a[c];
  if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains live
}

// fp64 tensor-core throughput: DMMA m8n8k4 (256 FMA per warp instruction), 8
// independent accumulator chains per warp, 16 warps per SM
__global__ void __launch_bounds__(512) k_dmma(double* out, int iters) {
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

}  // namespace

extern "C" hdr_status hdr_measure_dmma_peak(double* tflops, double* ms_out) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HDR_CUDA_ERROR;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, 512 * sizeof(double)) != cudaSuccess) return HDR_CUDA_ERROR;
  const int iters = 2048, reps = 10;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k_dmma<<<sms, 512>>>(out, iters);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k_dmma<<<sms, 512>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  hdr::count_launch(reps + 2);
  const double flops = 2.0 * 256.0 * 8.0 * iters * 16.0 * sms * reps;  // 16 warps per CTA, one CTA per SM
  if (tflops) *tflops = flops / (ms * 1e-3) / 1e12;
  if (ms_out) *ms_out = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? HDR_OK : HDR_CUDA_ERROR;
}

extern "C" hdr_status hdr_measure_fp64_peak(double* tflops, double* ms_out) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HDR_CUDA_ERROR;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, 256 * sizeof(double)) != cudaSuccess) return HDR_CUDA_ERROR;
  const int blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dfma<<<blocks, 256>>>(out, 1.0);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) k_dfma<<<blocks, 256>>>(out, 1.0 + r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  hdr::count_launch(reps + 3);
  const double flops = 2.0 * kChains * kIters * 256.0 * blocks * reps;
  if (tflops) *tflops = flops / (ms * 1e-3) / 1e12;
  if (ms_out) *ms_out = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? HDR_OK : HDR_CUDA_ERROR;
}

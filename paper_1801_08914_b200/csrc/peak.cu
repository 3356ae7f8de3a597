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

}  // namespace

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

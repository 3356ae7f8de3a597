// Microbenchmark: fp64 tensor-core (DMMA m8n8k4) vs DFMA throughput on one GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
  double d[8][2];
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x;
  const double a = 1.0000001, b = 0.9999999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096;
    k_dmma<<<sms, 32 * warps>>>(out, 16);
    cudaEventRecord(e0);
    k_dmma<<<sms, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 256 * 8 * iters * (double)warps * sms;  // 256 FMA per warp-MMA
    k_dfma<<<sms, 32 * warps>>>(out, 16);
    cudaEventRecord(e0);
    k_dfma<<<sms, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms2;
    cudaEventElapsedTime(&ms2, e0, e1);
    const double fl2 = 2.0 * 16 * iters * 32.0 * warps * sms;
    printf("warps/SM %2d: DMMA %.1f TFLOP/s, DFMA %.1f TFLOP/s\n", warps, fl / ms / 1e9, fl2 / ms2 / 1e9);
  }
  return 0;
}

// Legacy warp-level tensor-core throughput on this GPU (HMMA path): mma.sync
// m16n8k8 tf32 (1024 FMA per warp instruction) and, for comparison, DMMA
// m8n8k4 fp64 (256 FMA), 8 independent accumulator chains per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_tf32_peak tools/mma_tf32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_tf32(float* out, int iters) {
  float d[8][4];
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.f;
  const unsigned a0 = __float_as_uint(1.0f + threadIdx.x * 1e-6f), b0 = __float_as_uint(1.0f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
          : "r"(a0), "r"(a0), "r"(a0), "r"(a0), "r"(b0), "r"(b0));
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 12345.678f) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4096);
  const int iters = 4096;
  for (int w : {4, 8, 16}) {
    k_tf32<<<sms, 32 * w>>>(out, iters);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_tf32<<<sms, 32 * w>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 5.0 * sms * w * iters * 8.0 * 1024 * 2;
    printf("tf32 mma.sync m16n8k8: %d warps/SM: %.1f TFLOP/s (%.3f mma/clk/SM at 1.965 GHz)\n", w, fl / ms * 1e-9,
           fl / 2048 / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}

// Self-test of the tcgen05 TF32 path (umma.cuh): one CTA computes
// D (128 x N) = A (128 x K) * B^T (B: N x K) on the tensor core with the
// accumulator in TMEM, either in plain TF32 or as 3xTF32 (A_hi B_hi + A_hi B_lo
// + A_lo B_hi, hi = tf32(x), lo = tf32(x - hi)) — the split the correction
// GEMMs use to keep fp32 accuracy.  Exposed as hdr_umma_selftest for tests.
#include <cuda_runtime.h>

#include "capi_util.hpp"
#include "kernels.hpp"
#include "umma.cuh"

namespace hdr {
namespace {

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void __launch_bounds__(128) k_umma_selftest(int N, int K, const float* A, const float* B, float* D,
                                                       int split) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int M = 128;
  float* ahi = reinterpret_cast<float*>(sm);
  float* alo = ahi + M * K;
  float* bhi = alo + M * K;
  float* blo = bhi + N * K;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int t = tid; t < M * K; t += 128) {
    const int m = t / K, k = t % K;
    const float x = A[t], h = to_tf32(x);
    const uint32_t off = umma::kmajor_offset(m, k, M) >> 2;
    ahi[off] = h;
    alo[off] = to_tf32(x - h);
  }
  for (int t = tid; t < N * K; t += 128) {
    const int n = t / K, k = t % K;
    const float x = B[t], h = to_tf32(x);
    const uint32_t off = umma::kmajor_offset(n, k, N) >> 2;
    bhi[off] = h;
    blo[off] = to_tf32(x - h);
  }
  if (tid == 0) umma::mbar_init(&mbar, 1);
  umma::fence_proxy_async();
  __syncthreads();
  uint32_t ncols = 32;
  while (ncols < static_cast<uint32_t>(N)) ncols <<= 1;
  if (warp == 0) umma::tmem_alloc(&tslot, ncols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t idesc = umma::idesc_tf32(M, N);
    const uint32_t lbo_a = (M / 8) * 128, lbo_b = (N / 8) * 128;
    const int terms = split ? 3 : 1;
    for (int ks = 0; ks < K / 8; ++ks)
      for (int t = 0; t < terms; ++t) {
        const float* a = (t == 2) ? alo : ahi;
        const float* b = (t == 1) ? blo : bhi;
        const uint64_t ad = umma::smem_desc(umma::smem_u32(a) + ks * 2 * lbo_a, lbo_a, 128);
        const uint64_t bd = umma::smem_desc(umma::smem_u32(b) + ks * 2 * lbo_b, lbo_b, 128);
        umma::mma_tf32(tmem, ad, bd, idesc, ks > 0 || t > 0);
      }
    umma::commit(&mbar);
  }
  umma::mbar_wait(&mbar, 0);
  umma::fence_after();
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 8) {
    float v[8];
    umma::tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
    for (int j = 0; j < 8 && c0 + j < N; ++j) D[row * N + c0 + j] = v[j];
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, ncols);
}

}  // namespace
}  // namespace hdr

using namespace hdr;

extern "C" hdr_status hdr_umma_selftest(int n, int k, const float* a, const float* b, float* d, int split) {
  if (n < 16 || n > 256 || n % 16 || k < 8 || k % 8 || !a || !b || !d)
    return fail(HDR_INVALID_ARGUMENT, "umma selftest: N in 16..256 step 16, K multiple of 8");
  return catch_all([&]() -> hdr_status {
    const size_t smem = static_cast<size_t>(2 * 128 * k + 2 * n * k) * 4;
    if (smem > 220 * 1024) return fail(HDR_INVALID_ARGUMENT, "umma selftest: operands exceed shared memory");
    DBuf<float> da, db, dd;
    da.upload(a, static_cast<size_t>(128) * k);
    db.upload(b, static_cast<size_t>(n) * k);
    dd.alloc(static_cast<size_t>(128) * n);
    CK(cudaFuncSetAttribute(k_umma_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_umma_selftest<<<1, 128, smem>>>(n, k, da.p, db.p, dd.p, split);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(d, dd.p, static_cast<size_t>(128) * n * 4, cudaMemcpyDeviceToHost));
    count_launch();
    return HDR_OK;
  });
}

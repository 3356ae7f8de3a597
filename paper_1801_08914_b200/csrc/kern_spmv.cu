// spmv (src/csr.cpp:77-87): y_i = sum_k values[k] * x[col[k]], one sequential sum
// per row in storage order with separate multiply and add roundings (the
// reference's loop, as-shipped without FMA contraction), so for the same matrix
// and vector the result is bit-identical to the reference's spmv.
#include <cstdint>
#include <cstdlib>

#include "kernels.hpp"

namespace hdr {
namespace {

template <class Col>
__global__ void k_spmv_rows(int64_t nrows, const int64_t* __restrict__ ro, const Col* __restrict__ ci,
                            const double* __restrict__ v, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nrows) return;
  double s = 0.0;
  const int64_t end = ro[i + 1];
#ifdef HDR_SPMV_ROWS_PLAIN
  for (int64_t k = ro[i]; k < end; ++k) s = __dadd_rn(s, __dmul_rn(v[k], x[ci[k]]));
#else
  // four products in flight (independent loads), added in storage order
  int64_t k = ro[i];
  for (; k + 4 <= end; k += 4) {
    const double p0 = __dmul_rn(v[k], x[ci[k]]), p1 = __dmul_rn(v[k + 1], x[ci[k + 1]]);
    const double p2 = __dmul_rn(v[k + 2], x[ci[k + 2]]), p3 = __dmul_rn(v[k + 3], x[ci[k + 3]]);
    s = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(s, p0), p1), p2), p3);
  }
  for (; k < end; ++k) s = __dadd_rn(s, __dmul_rn(v[k], x[ci[k]]));
#endif
  y[i] = s;
}

// Coalesced form with the same bits: a warp owns 32 consecutive rows, i.e. one
// contiguous span of the CSR arrays.  The span goes through shared memory in
// tiles: the lanes form the products fl(v_k x_col) with coalesced loads of v and
// col (the rounding of a product does not depend on who computes it), then lane i
// adds the products of row i that fall in the tile, sequentially in storage order
// (the reference's sum, starting from 0.0).  HBM sees full sectors once instead of
// 32 strided streams; x is gathered through L1 / L2.
#ifndef HDR_SPMV_TILE
#define HDR_SPMV_TILE 256   // measured (cfg3 / cfg5 ms): 1024x4 0.229 / 1.194, 512x8 0.288 / 1.182, 256x8 0.206 / 1.171, 1024x8 0.212 / 1.166
#endif
#ifndef HDR_SPMV_UNROLL
#define HDR_SPMV_UNROLL 8
#endif
constexpr int kSpmvTile = HDR_SPMV_TILE;  // products per warp tile (8 bytes each; tile x unroll of the load loop)
constexpr int kSpmvUnroll = HDR_SPMV_UNROLL;

template <class Col>
__global__ void __launch_bounds__(128) k_spmv_tiled(int64_t nrows, const int64_t* __restrict__ ro,
                                                    const Col* __restrict__ ci, const double* __restrict__ v,
                                                    const double* __restrict__ x, double* __restrict__ y) {
  __shared__ double prod[4][kSpmvTile];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (static_cast<int64_t>(blockIdx.x) * 4 + warp) * 32;
  if (r0 >= nrows) return;
  const int64_t i = r0 + lane;
  const bool has = i < nrows;
  const int64_t gb = ro[r0], ge = ro[r0 + 32 < nrows ? r0 + 32 : nrows];
  // row bounds relative to the span start (32 rows: far below 2^31 entries)
  const int rb = has ? static_cast<int>(ro[i] - gb) : 0, re = has ? static_cast<int>(ro[i + 1] - gb) : 0;
  const int span = static_cast<int>(ge - gb);
  const double* __restrict__ vs = v + gb;
  const Col* __restrict__ cs = ci + gb;
  double* P = prod[warp];
  double s = 0.0;
  for (int t0 = 0; t0 < span; t0 += kSpmvTile) {
    const int t1 = min(t0 + kSpmvTile, span);
#pragma unroll kSpmvUnroll
    for (int q = t0 + lane; q < t1; q += 32) P[q - t0] = __dmul_rn(vs[q], x[cs[q]]);
    __syncwarp();
    const int a = max(rb, t0), b = min(re, t1);
    for (int k = a; k < b; ++k) s = __dadd_rn(s, P[k - t0]);
    __syncwarp();
  }
  if (has) y[i] = s;
}

}  // namespace

// measured on the B200 (10 steps, L2 flushed; tiles vs thread per row): 11 entries per row
// 64 vs 49 us, 44 per row 0.207 vs 0.244 ms, ~550 per row 1.17 vs 1.71 ms
static bool use_tiles(int64_t nrows, int64_t nnz) {
  if (getenv("HDR_SPMV_ROWS")) return false;
  if (getenv("HDR_SPMV_TILES")) return true;
  return nnz >= 32 * nrows;
}

void launch_spmv32(int64_t nrows, const int64_t* ro, const int32_t* ci, const double* v, const double* x, double* y,
                   cudaStream_t st, int64_t nnz) {
  if (nrows <= 0) return;
  if (!use_tiles(nrows, nnz)) k_spmv_rows<int32_t><<<static_cast<unsigned>((nrows + 127) / 128), 128, 0, st>>>(nrows, ro, ci, v, x, y);
  else k_spmv_tiled<int32_t><<<static_cast<unsigned>((nrows + 127) / 128), 128, 0, st>>>(nrows, ro, ci, v, x, y);
  count_launch();
}

void launch_spmv64(int64_t nrows, const int64_t* ro, const int64_t* ci, const double* v, const double* x, double* y,
                   cudaStream_t st, int64_t nnz) {
  if (nrows <= 0) return;
  if (!use_tiles(nrows, nnz)) k_spmv_rows<int64_t><<<static_cast<unsigned>((nrows + 127) / 128), 128, 0, st>>>(nrows, ro, ci, v, x, y);
  else k_spmv_tiled<int64_t><<<static_cast<unsigned>((nrows + 127) / 128), 128, 0, st>>>(nrows, ro, ci, v, x, y);
  count_launch();
}

}  // namespace hdr

// spmv (src/csr.cpp:77-87): y_i = sum_k values[k] * x[col[k]], one sequential sum
// per row in storage order with separate multiply and add roundings (the
// reference's loop, as-shipped without FMA contraction), so for the same matrix
// and vector the result is bit-identical to the reference's spmv.
#include <cstdint>

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
  for (int64_t k = ro[i]; k < end; ++k) s = __dadd_rn(s, __dmul_rn(v[k], x[ci[k]]));
  y[i] = s;
}

}  // namespace

void launch_spmv32(int64_t nrows, const int64_t* ro, const int32_t* ci, const double* v, const double* x, double* y,
                   cudaStream_t st) {
  if (nrows <= 0) return;
  k_spmv_rows<int32_t><<<static_cast<unsigned>((nrows + 127) / 128), 128, 0, st>>>(nrows, ro, ci, v, x, y);
  count_launch();
}

void launch_spmv64(int64_t nrows, const int64_t* ro, const int64_t* ci, const double* v, const double* x, double* y,
                   cudaStream_t st) {
  if (nrows <= 0) return;
  k_spmv_rows<int64_t><<<static_cast<unsigned>((nrows + 127) / 128), 128, 0, st>>>(nrows, ro, ci, v, x, y);
  count_launch();
}

}  // namespace hdr

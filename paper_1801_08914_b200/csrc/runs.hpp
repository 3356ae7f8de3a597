// Device from_triplets machinery shared by the algebraic and mapped-geometry
// paths: stable radix sort of (row, col) keys, run heads, CSR of the runs.
#pragma once

#include <cub/cub.cuh>

#include "capi_util.hpp"
#include "kernels.hpp"

namespace hdr {

template <class T>
inline void dev_scan(const T* in, T* out, int64_t count, cudaStream_t st) {
  size_t bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, static_cast<int>(count), st));
  DBuf<unsigned char> tmp;
  tmp.alloc(bytes);
  CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, static_cast<int>(count), st));
}

inline int key_bits(uint64_t maxkey) {
  int b = 1;
  while (b < 64 && (maxkey >> b) != 0) ++b;
  return b;
}

// Sorted runs of (key, src[, w]) triplets: the summation structure of
// from_triplets (stable radix sort keeps generation order within a run).
struct Runs {
  DBuf<uint64_t> keys;
  DBuf<int64_t> src;
  DBuf<double> w;
  DBuf<int64_t> start;  // nruns + 1
  DBuf<int64_t> index;  // vectors: row of each run; matrices: column of each run
  int64_t nruns = 0;
};

inline void sort_runs(int64_t n, DBuf<uint64_t>& keys_in, DBuf<int64_t>& src_in, DBuf<double>* w_in, uint64_t maxkey,
               int64_t ncols, DBuf<int64_t>* row_cnt, Runs& R, cudaStream_t st) {
  if (n >= (int64_t(1) << 31)) throw StatusError(HDR_UNSUPPORTED, "more than 2^31 triplets");
  R.keys.alloc(n);
  R.src.alloc(n);
  const int bits = key_bits(maxkey);
  if (w_in) {
    // sort (key, position) then gather src and w by position
    DBuf<int64_t> pos_in, pos_out;
    pos_in.alloc(n);
    pos_out.alloc(n);
    launch_iota(n, pos_in.p, st);
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in.p, R.keys.p, pos_in.p, pos_out.p, static_cast<int>(n), 0,
                                       bits, st));
    DBuf<unsigned char> tmp;
    tmp.alloc(bytes);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys_in.p, R.keys.p, pos_in.p, pos_out.p, static_cast<int>(n), 0,
                                       bits, st));
    R.w.alloc(n);
    launch_gather_i64(n, pos_out.p, src_in.p, R.src.p, st);
    launch_gather_f64(n, pos_out.p, w_in->p, R.w.p, st);
  } else {
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in.p, R.keys.p, src_in.p, R.src.p, static_cast<int>(n), 0,
                                       bits, st));
    DBuf<unsigned char> tmp;
    tmp.alloc(bytes);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys_in.p, R.keys.p, src_in.p, R.src.p, static_cast<int>(n), 0,
                                       bits, st));
  }
  DBuf<int> head, pos;
  head.alloc(n + 1);
  pos.alloc(n + 1);
  CK(cudaMemsetAsync(head.p, 0, static_cast<size_t>(n + 1) * sizeof(int), st));
  launch_run_heads(n, R.keys.p, head.p, st);
  dev_scan(head.p, pos.p, n + 1, st);
  int nr = 0;
  CK(cudaMemcpyAsync(&nr, pos.p + n, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  R.nruns = nr;
  R.start.alloc(static_cast<size_t>(nr) + 1);
  CK(cudaMemcpyAsync(R.start.p + nr, &n, 8, cudaMemcpyHostToDevice, st));
  if (row_cnt) {  // matrix: columns + per-row counts
    R.index.alloc(static_cast<size_t>(nr));
    launch_run_csr(n, R.keys.p, head.p, pos.p, ncols, R.start.p, R.index.p, row_cnt->p, st);
  } else {  // vector: the row of each run
    R.index.alloc(static_cast<size_t>(nr));
    launch_run_csr(n, R.keys.p, head.p, pos.p, ncols, R.start.p, nullptr, R.index.p, st);
  }
  CK(cudaStreamSynchronize(st));
}

}  // namespace hdr

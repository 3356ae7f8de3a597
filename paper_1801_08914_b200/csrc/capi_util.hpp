// Shared host-side helpers of the C ABI: error reporting, CUDA error checks,
// owning device buffers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <new>
#include <string>
#include <vector>

#include "../../include/hdivred_b200.h"

namespace hdr {

std::string& last_error_ref();

inline hdr_status fail(hdr_status s, const std::string& msg) {
  last_error_ref() = msg;
  return s;
}

struct CudaError : std::exception {
  cudaError_t e;
  std::string where;
  CudaError(cudaError_t err, const char* w) : e(err), where(w) {}
};

// A typed status raised from deep inside a host routine (mapped by catch_all).
struct StatusError : std::exception {
  hdr_status s;
  std::string msg;
  StatusError(hdr_status st, std::string m) : s(st), msg(std::move(m)) {}
};

#define CK(call)                                       \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) throw CudaError(_e, #call); \
  } while (0)

template <class T>
struct DBuf {  // owning device buffer
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    reset();
    if (count == 0) count = 1;
    CK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  // allocate and copy a host vector (synchronous upload)
  void upload(const std::vector<T>& v) {
    alloc(v.size());
    if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  void upload(const T* src, size_t count) {
    alloc(count);
    if (count) CK(cudaMemcpy(p, src, count * sizeof(T), cudaMemcpyHostToDevice));
  }
};

inline hdr_status catch_all(const std::function<hdr_status()>& fn) {
  try {
    return fn();
  } catch (const StatusError& e) {
    return fail(e.s, e.msg);
  } catch (const CudaError& e) {
    return fail(HDR_CUDA_ERROR, std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.e));
  } catch (const std::bad_alloc&) {
    return fail(HDR_CUDA_ERROR, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(HDR_UNSUPPORTED, e.what());
  }
}

}  // namespace hdr

// common.cuh -- shared helpers for libtcb200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cassert>

// TCB_DEBUG=1 builds device-side bounds asserts into the engine and the
// scatter kernels (tools/build_variant.sh debug -DTCB_DEBUG=1; the GPU pool
// has no compute-sanitizer).
#ifndef TCB_DEBUG
#define TCB_DEBUG 0
#endif

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tcb200.h"

namespace tcb {

// Error carried from the implementation to the C-ABI boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

void set_last_error(const std::string& msg);

#define TC_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e__ = (call);                                                      \
    if (e__ != cudaSuccess)                                                        \
      throw ::tcb::Error(TC_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
  } while (0)

#define TC_REQUIRE(cond, code, msg)                       \
  do {                                                    \
    if (!(cond)) throw ::tcb::Error((code), (msg));       \
  } while (0)

// Runs `body` and maps exceptions to C-ABI status codes.
template <class F>
int guarded(F&& body) {
  try {
    body();
    return TC_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return TC_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TC_ECUDA;
  }
}

// Library device memory (abi.cu): the caller's allocator if registered
// (tc_set_allocator), else the library's private stream-ordered pool.
struct DevBlock {
  void* p;
  tc_free_fn free_fn;  // NULL: the library pool
  void* ctx;
};
DevBlock dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(const DevBlock& b, cudaStream_t s);

// Stream-ordered scratch memory; everything is released on the same stream
// when the guard dies, so the library never holds device memory across calls.
class Scratch {
 public:
  explicit Scratch(cudaStream_t s) : s_(s) {}
  ~Scratch() {
    for (const DevBlock& b : ptrs_) dev_free(b, s_);
  }
  template <class T>
  T* alloc(size_t n) {
    ptrs_.push_back(dev_alloc((n ? n : 1) * sizeof(T), s_));
    return static_cast<T*>(ptrs_.back().p);
  }
  void* bytes(size_t n) { return alloc<unsigned char>(n); }

 private:
  cudaStream_t s_;
  std::vector<DevBlock> ptrs_;
};

inline int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

inline int grid_for(int64_t n, int block, int max_blocks = 148 * 32) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (int)g;
}

int sm_count();

inline void sync_stream(cudaStream_t s) { TC_CUDA(cudaStreamSynchronize(s)); }

// Counts launches of this library's own kernels (every launch site calls
// check_launch); CUB's kernels are not counted.  Read by tc_launch_count.
extern unsigned long long g_launches;

// Pairs per chunk of the host-input normalize pipeline (tc_set_tuning key 3).
extern int64_t g_host_chunk;

inline void check_launch() {
  ++g_launches;
  TC_CUDA(cudaGetLastError());
}

// Every row of a CSR sorted ascending, unsorted -> out (build.cu).
void sort_rows(Scratch& sc, const int64_t* indptr, int64_t n, int64_t m, const int32_t* unsorted, int32_t* out,
               cudaStream_t s);

// Row of forward edge e: the largest v with indptr[v] <= e (indptr[n] = m > e).
__device__ __forceinline__ int64_t row_of_edge(const int64_t* __restrict__ indptr, int64_t n, int64_t e) {
  int64_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(&indptr[mid]) <= e) lo = mid;
    else hi = mid;
  }
  return lo;
}

}  // namespace tcb

#define GRID_STRIDE(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)(n); i += (int64_t)gridDim.x * blockDim.x)

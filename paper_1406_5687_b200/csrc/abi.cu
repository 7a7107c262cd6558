// abi.cu -- error state, version and memory-pool plumbing of the C ABI.
#include <string>

#include "common.cuh"

namespace tcb {

static thread_local std::string g_last_error;
unsigned long long g_launches = 0;

void set_last_error(const std::string& msg) { g_last_error = msg; }

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, n = 0;
    TC_CUDA(cudaGetDevice(&dev));
    TC_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    // Keep the pool's freed blocks cached between calls (stream-ordered
    // scratch is re-used instead of returned to the driver every sync).
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = 64ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cached = n;
  }
  return cached;
}

}  // namespace tcb

extern "C" {

const char* tc_last_error(void) { return tcb::g_last_error.c_str(); }

int tc_abi_version(void) { return 1; }

unsigned long long tc_launch_count(void) { return tcb::g_launches; }

int tc_trim_pool(void) {
  return tcb::guarded([&] {
    int dev = 0;
    TC_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    TC_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    TC_CUDA(cudaDeviceSynchronize());
    TC_CUDA(cudaMemPoolTrimTo(pool, 0));
  });
}

}  // extern "C"

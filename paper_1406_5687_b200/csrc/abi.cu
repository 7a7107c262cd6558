// abi.cu -- error state, version and memory-pool plumbing of the C ABI.
#include <mutex>
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
    cached = n;
  }
  return cached;
}

// Library memory.  Scratch and plan memory come from the caller's allocator
// when one is registered (tc_set_allocator: e.g. torch's caching allocator,
// so torch owns every byte), else from a stream-ordered pool private to this
// library (one per device) that keeps freed blocks cached between calls.
// The device's default pool is left untouched.
static tc_alloc_fn g_alloc = nullptr;
static tc_free_fn g_free = nullptr;
static void* g_alloc_ctx = nullptr;

static cudaMemPool_t lib_pool() {
  static cudaMemPool_t pools[64] = {};
  static std::mutex mu;
  int dev = 0;
  TC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    TC_CUDA(cudaMemPoolCreate(&pools[dev], &props));
    uint64_t thr = UINT64_MAX;  // this pool only: keep freed blocks for re-use (tc_trim_pool releases them)
    TC_CUDA(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
  }
  return pools[dev];
}

DevBlock dev_alloc(size_t bytes, cudaStream_t s) {
  bytes = bytes ? bytes : 16;
  DevBlock b{nullptr, g_free, g_alloc_ctx};  // freed by the allocator that made it
  if (g_alloc) {
    b.p = g_alloc(bytes, (tc_stream_t)s, g_alloc_ctx);
    if (!b.p) throw Error(TC_ENOMEM, "caller allocator returned NULL for " + std::to_string(bytes) + " bytes");
    return b;
  }
  const cudaError_t e = cudaMallocFromPoolAsync(&b.p, bytes, lib_pool(), s);
  if (e != cudaSuccess)
    throw Error(TC_ENOMEM, "cudaMallocFromPoolAsync(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  return b;
}

void dev_free(const DevBlock& b, cudaStream_t s) {
  if (!b.p) return;
  if (b.free_fn) b.free_fn(b.p, (tc_stream_t)s, b.ctx);
  else cudaFreeAsync(b.p, s);
}

}  // namespace tcb

extern "C" {

const char* tc_last_error(void) { return tcb::g_last_error.c_str(); }

int tc_abi_version(void) { return 1; }

unsigned long long tc_launch_count(void) { return tcb::g_launches; }

int tc_trim_pool(void) {
  return tcb::guarded([&] {
    TC_CUDA(cudaDeviceSynchronize());
    TC_CUDA(cudaMemPoolTrimTo(tcb::lib_pool(), 0));
  });
}

int tc_set_allocator(tc_alloc_fn alloc, tc_free_fn free_fn, void* ctx) {
  return tcb::guarded([&] {
    TC_REQUIRE((alloc == nullptr) == (free_fn == nullptr), TC_EINVAL, "give both allocator functions or neither");
    tcb::g_alloc = alloc;
    tcb::g_free = free_fn;
    tcb::g_alloc_ctx = ctx;
  });
}

}  // extern "C"

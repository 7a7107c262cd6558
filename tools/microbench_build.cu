// microbench_build.cu -- dev tool: throughput of the primitives the graph
// build could be made of (atomics with/without return, counting scatters,
// CUB segmented sort, CUB radix passes) at cfg-2 sizes.  Not part of the
// product; numbers guide DESIGN.md §3.1.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 tools/microbench_build.cu -o /tmp/mb
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (uint32_t)(z ^ (z >> 31));
}

__global__ void k_keys(int32_t* k, int64_t m, int n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    k[i] = mix(i) % n;
}
__global__ void k_red(const int32_t* __restrict__ k, int64_t m, int* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[k[i]], 1);
}
__global__ void k_ret(const int32_t* __restrict__ k, int64_t m, int* cnt, int* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = atomicAdd(&cnt[k[i]], 1);
}
__global__ void k_scatter4(const int32_t* __restrict__ k, int64_t m, const int64_t* __restrict__ base, int* cnt,
                           int* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int r = k[i];
    out[base[r] + atomicAdd(&cnt[r], 1)] = (int)i;
  }
}
__global__ void k_scatter8(const int32_t* __restrict__ k, int64_t m, const int64_t* __restrict__ base, int* cnt,
                           int2* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int r = k[i];
    out[base[r] + atomicAdd(&cnt[r], 1)] = make_int2((int)i, r);
  }
}
__global__ void k_scatter4p(const int32_t* __restrict__ k, int64_t m, const int64_t* __restrict__ base, int* cnt,
                            int* out, int r0, int r1) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int r = k[i];
    if (r >= r0 && r < r1) out[base[r] + atomicAdd(&cnt[r], 1)] = (int)i;
  }
}
__global__ void k_scatter8p(const int32_t* __restrict__ k, int64_t m, const int64_t* __restrict__ base, int* cnt,
                            int2* out, int r0, int r1) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int r = k[i];
    if (r >= r0 && r < r1) out[base[r] + atomicAdd(&cnt[r], 1)] = make_int2((int)i, r);
  }
}
__global__ void k_copy8(const int2* __restrict__ a, int2* b, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

struct Timer {
  cudaEvent_t a, b;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); }
  float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
};

int main() {
  const int64_t m = 50000000;
  const int n = 1000000;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int32_t *keys, *cnt, *out;
  int64_t* base;
  int2* out8;
  CK(cudaMalloc(&keys, m * 4));
  CK(cudaMalloc(&cnt, n * 4));
  CK(cudaMalloc(&out, m * 4));
  CK(cudaMalloc(&out8, m * 8));
  CK(cudaMalloc(&base, (n + 1) * 8));
  k_keys<<<sms * 8, 256>>>(keys, m, n);
  // base = exclusive prefix of the histogram
  CK(cudaMemset(cnt, 0, n * 4));
  k_red<<<sms * 16, 256>>>(keys, m, cnt);
  std::vector<int> h(n);
  CK(cudaMemcpy(h.data(), cnt, n * 4, cudaMemcpyDeviceToHost));
  std::vector<int64_t> hb(n + 1, 0);
  for (int i = 0; i < n; ++i) hb[i + 1] = hb[i] + h[i];
  CK(cudaMemcpy(base, hb.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  Timer t;
  for (int grid : {sms * 8, sms * 16, sms * 32}) {
    float best[4] = {1e9, 1e9, 1e9, 1e9};
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(cnt, 0, n * 4); t.start(); k_red<<<grid, 256>>>(keys, m, cnt); best[0] = std::min(best[0], t.stop());
      cudaMemset(cnt, 0, n * 4); t.start(); k_ret<<<grid, 256>>>(keys, m, cnt, out); best[1] = std::min(best[1], t.stop());
      cudaMemset(cnt, 0, n * 4); t.start(); k_scatter4<<<grid, 256>>>(keys, m, base, cnt, out); best[2] = std::min(best[2], t.stop());
      cudaMemset(cnt, 0, n * 4); t.start(); k_scatter8<<<grid, 256>>>(keys, m, base, cnt, out8); best[3] = std::min(best[3], t.stop());
    }
    printf("grid %5d: RED %.3f ms | atomic+ret %.3f ms | scatter4 %.3f ms | scatter8 %.3f ms   (m=%lld, n=%d)\n", grid,
           best[0], best[1], best[2], best[3], (long long)m, n);
  }
  for (int P : {2, 4, 8, 16}) {
    float b4 = 1e9, b8 = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(cnt, 0, n * 4);
      t.start();
      for (int p = 0; p < P; ++p) k_scatter4p<<<sms * 16, 256>>>(keys, m, base, cnt, out, (int)((int64_t)n * p / P), (int)((int64_t)n * (p + 1) / P));
      b4 = std::min(b4, t.stop());
      cudaMemset(cnt, 0, n * 4);
      t.start();
      for (int p = 0; p < P; ++p) k_scatter8p<<<sms * 16, 256>>>(keys, m, base, cnt, out8, (int)((int64_t)n * p / P), (int)((int64_t)n * (p + 1) / P));
      b8 = std::min(b8, t.stop());
    }
    printf("phased scatter P=%d: scatter4 %.3f ms | scatter8 %.3f ms\n", P, b4, b8);
  }
  // copy bandwidth reference: 400 MB -> 400 MB
  {
    int2* tmp;
    CK(cudaMalloc(&tmp, m * 8));
    float b = 1e9;
    for (int r = 0; r < 3; ++r) { t.start(); k_copy8<<<sms * 16, 256>>>(out8, tmp, m); b = std::min(b, t.stop()); }
    printf("copy 400MB: %.3f ms (%.0f GB/s)\n", b, 2 * 8.0 * m / b / 1e6);
    cudaFree(tmp);
  }
  // CUB segmented sort: m int32 keys in n segments (sizes = histogram above)
  {
    int32_t* sorted;
    CK(cudaMalloc(&sorted, m * 4));
    k_keys<<<sms * 8, 256>>>(out, m, n);  // random values
    size_t tmp = 0;
    cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, out, sorted, (int)m, n, base, base + 1);
    void* ws;
    CK(cudaMalloc(&ws, tmp));
    float b = 1e9;
    for (int r = 0; r < 3; ++r) {
      t.start();
      cub::DeviceSegmentedSort::SortKeys(ws, tmp, out, sorted, (int)m, n, base, base + 1);
      b = std::min(b, t.stop());
    }
    printf("CUB segmented sort, %lld int32 keys in %d segments (avg %.0f): %.3f ms\n", (long long)m, n, (double)m / n, b);
    cudaFree(ws);
    cudaFree(sorted);
  }
  // CUB radix sort u64 keys: 20 and 40 bits; u32 20 bits
  {
    unsigned long long *a, *bb;
    CK(cudaMalloc(&a, m * 8));
    CK(cudaMalloc(&bb, m * 8));
    for (int bits : {20, 32, 40}) {
      size_t tmp = 0;
      cub::DoubleBuffer<unsigned long long> db(a, bb);
      cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, m, 0, bits);
      void* ws;
      CK(cudaMalloc(&ws, tmp));
      float b = 1e9;
      for (int r = 0; r < 3; ++r) {
        k_keys<<<sms * 8, 256>>>(reinterpret_cast<int32_t*>(a), 2 * m, 1 << 20);
        cub::DoubleBuffer<unsigned long long> d2(a, bb);
        t.start();
        cub::DeviceRadixSort::SortKeys(ws, tmp, d2, m, 0, bits);
        b = std::min(b, t.stop());
      }
      printf("CUB radix sort u64 x %lld, %d bits: %.3f ms\n", (long long)m, bits, b);
      cudaFree(ws);
    }
    cudaFree(a);
    cudaFree(bb);
  }
  return 0;
}

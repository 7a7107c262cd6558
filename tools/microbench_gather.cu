// microbench_gather.cu -- dev tool: what the B200 memory system delivers for the small tier's access pattern.
// Warps read "segments" of L consecutive 16-byte chunks at random 16-byte-aligned offsets of a pool, flattened
// over the lanes like the engine's windows (lane j of a window reads chunk (32 w + j) of the concatenated
// segments), kW windows in flight per warp, 42 warps per SM (7 x 6 blocks).  No probes, no tables: only the loads.
// Reports the requested bytes per second; the engine's figure to compare is its chunk-load request rate
// (l1tex global-load sectors x 32 B / time) and its DRAM rate.  Not part of the product.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 tools/microbench_gather.cu -o tools/microbench_gather.bin
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (uint32_t)(z ^ (z >> 31));
}

template <int kW>
__global__ void __launch_bounds__(224, 6) k_gather(const int4* __restrict__ pool, uint32_t nchunks, int L,
                                                   long long windows_per_warp, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t acc = 0;
  for (long long w = 0; w < windows_per_warp; w += kW) {
    int4 v[kW];
#pragma unroll
    for (int k = 0; k < kW; ++k) {
      const long long f = (warp * windows_per_warp + w + k) * 32 + lane;  // flat chunk index
      const long long seg = f / L;
      const uint32_t start = mix((uint64_t)seg) % (nchunks - (uint32_t)L);
      v[k] = __ldg(pool + start + (uint32_t)(f - seg * L));
    }
#pragma unroll
    for (int k = 0; k < kW; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

int main(int argc, char** argv) {
  const double pool_mb[] = {106, 212, 2048};
  const int Ls[] = {1, 2, 3, 4, 6, 8, 16, 32, 64};
  unsigned long long* out;
  CK(cudaMalloc(&out, 8));
  char* flush;
  CK(cudaMalloc(&flush, 1 << 30));
  for (double mb : pool_mb) {
    const uint32_t nchunks = (uint32_t)(mb * 1e6 / 16);
    int4* pool;
    CK(cudaMalloc(&pool, (size_t)nchunks * 16));
    CK(cudaMemset(pool, 1, (size_t)nchunks * 16));
    for (int L : Ls) {
      const int blocks = 148 * 6;
      const long long warps = (long long)blocks * 7;
      const long long wpw = 1536;  // windows per warp: 9.5 M windows = 4.9 GB requested
      cudaEvent_t a, b;
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      float best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        CK(cudaMemset(flush, rep, 1 << 30));
        CK(cudaEventRecord(a));
        k_gather<3><<<blocks, 224>>>(pool, nchunks, L, wpw, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (rep && ms < best) best = ms;
      }
      const double bytes = (double)warps * wpw * 32 * 16;
      printf("pool %6.0f MB  segment %3d chunks (%4d B): %.3f ms  %.2f TB/s requested\n", mb, L, L * 16, best,
             bytes / best / 1e9);
    }
    CK(cudaFree(pool));
  }
  return 0;
}

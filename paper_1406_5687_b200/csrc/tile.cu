// tile.cu -- L2-tiled regrouping of the middle-vertex engine's work.
//
// The pull engine streams, for every middle vertex u, the suffixes of its
// predecessors' lists N^_v.  In (u, v) order those reads hit the whole
// eff_indices array at random times, so once it exceeds L2 (126 MB) most
// reads go to DRAM.  Here the predecessor entries are regrouped tile-major:
// v is cut into tiles of at most `tile_ids` list entries (sized to stay L2
// resident), and entries are ordered by (tile(v), u, v).  Each (tile, u)
// with entries becomes one "virtual owner" whose table is N^_u; the engine
// then walks tiles one after another with the same kernel.  Extra cost: one
// table build per (tile, u) instead of per u.
#include <cub/cub.cuh>

#include "common.cuh"

namespace tcb {

static constexpr int64_t kSegCost = 2;  // must match build.cu / count.cu
static constexpr int64_t kTabCost = 16;

__global__ void k_tile_bounds(const int64_t* __restrict__ eff_indptr, int64_t n, int64_t tile_ids, int T,
                              int64_t* vt) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= T; k += gridDim.x * blockDim.x) {
    if (k == T) {
      vt[k] = n;
      continue;
    }
    int64_t want = (int64_t)k * tile_ids;  // first v with eff_indptr[v] >= want
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (eff_indptr[mid] < want) lo = mid + 1;
      else hi = mid;
    }
    vt[k] = lo;
  }
}

__global__ void k_entry_u(const int64_t* __restrict__ rev_indptr, int64_t u0, int64_t u1, int64_t r0,
                          int32_t* uarr) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = u0 + warp; u < u1; u += nwarps)
    for (int64_t j = rev_indptr[u] + lane; j < rev_indptr[u + 1]; j += 32) uarr[j - r0] = (int32_t)u;
}

__global__ void k_tile_keys(const int2* __restrict__ rev_seg, const int64_t* __restrict__ pool_indptr, int64_t n,
                            const int32_t* __restrict__ uarr, int64_t r0,
                            int64_t E, const int64_t* __restrict__ vt, int T, int64_t u0, int bu,
                            unsigned long long* keys, int32_t* vals) {
  GRID_STRIDE(i, E) {
    int64_t v = row_of_edge(pool_indptr, n, (int64_t)rev_seg[r0 + i].x - 1);
    int lo = 0, hi = T;  // largest t with vt[t] <= v
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (vt[mid] <= v) lo = mid;
      else hi = mid;
    }
    keys[i] = ((unsigned long long)lo << bu) | (unsigned long long)(uarr[i] - u0);
    vals[i] = (int32_t)i;
  }
}

__global__ void k_owner_flags(const unsigned long long* __restrict__ keys, int64_t E, int32_t* flag) {
  GRID_STRIDE(i, E) flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_owner_emit(const unsigned long long* __restrict__ keys, const int32_t* __restrict__ flag,
                             const int32_t* __restrict__ idx, int64_t E, int64_t u0, int bu,
                             int32_t* owner_u, int64_t* owner_ptr) {
  unsigned long long mask = (bu >= 64) ? ~0ull : ((1ull << bu) - 1);
  GRID_STRIDE(i, E) {
    if (flag[i]) {
      int32_t o = idx[i];
      owner_u[o] = (int32_t)((int64_t)(keys[i] & mask) + u0);
      owner_ptr[o] = i;
    }
  }
}

__global__ void k_gather_tseg(const int2* __restrict__ rev_seg, int64_t r0, const int32_t* __restrict__ vals,
                              int64_t E, int2* segs) {
  GRID_STRIDE(i, E) segs[i] = rev_seg[r0 + vals[i]];
}

__global__ void k_owner_cost(const int64_t* __restrict__ owner_ptr, const int32_t* __restrict__ owner_u,
                             const int2* __restrict__ segs, const int64_t* __restrict__ eff_indptr,
                             int64_t K, int64_t* cost) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = warp; x < K; x += nwarps) {
    int64_t u = owner_u[x];
    int64_t d = eff_indptr[u + 1] - eff_indptr[u];
    long long s = 0;
    if (d > 0)
      for (int64_t r = owner_ptr[x] + lane; r < owner_ptr[x + 1]; r += 32) s += (segs[r].y - segs[r].x) + kSegCost;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) cost[x] = d > 0 ? (int64_t)s + d + kTabCost : 0;
  }
}

template <class In, class Out>
static void excl_sum(Scratch& sc, In in, Out out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  void* t = sc.bytes(tmp);
  TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, s));
}

static void tile_pull(const int64_t* eff_indptr, const int64_t* pool_indptr, int64_t n, const int64_t* rev_indptr,
                      const int32_t* rev_seg, int64_t u0, int64_t u1, int64_t tile_ids, int32_t* owner_u,
                      int64_t* owner_ptr, int32_t* segs, int64_t* cost_prefix, int64_t* k_host,
                      int64_t* ntiles_host, cudaStream_t s) {
  TC_REQUIRE(0 <= u0 && u0 <= u1 && u1 <= n, TC_EINVAL, "bad owner range");
  TC_REQUIRE(tile_ids >= 1, TC_EINVAL, "tile_ids must be >= 1");
  Scratch sc(s);
  int64_t h[3];
  TC_CUDA(cudaMemcpyAsync(&h[0], rev_indptr + u0, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaMemcpyAsync(&h[1], rev_indptr + u1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaMemcpyAsync(&h[2], eff_indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  sync_stream(s);
  const int64_t r0 = h[0], E = h[1] - h[0], mids = h[2];
  TC_REQUIRE(E < (1ll << 31) - 1, TC_EINVAL, "too many entries");
  int T = (int)std::max<int64_t>(1, (mids + tile_ids - 1) / tile_ids);
  *ntiles_host = T;
  *k_host = 0;
  if (E == 0) {
    TC_CUDA(cudaMemsetAsync(owner_ptr, 0, sizeof(int64_t), s));
    TC_CUDA(cudaMemsetAsync(cost_prefix, 0, sizeof(int64_t), s));
    return;
  }
  int sms = sm_count();
  int64_t* vt = sc.alloc<int64_t>(T + 1);
  k_tile_bounds<<<grid_for(T + 1, 128), 128, 0, s>>>(eff_indptr, n, tile_ids, T, vt);
  check_launch();
  int32_t* uarr = sc.alloc<int32_t>(E);
  k_entry_u<<<grid_for((u1 - u0) * 32, 256, sms * 16), 256, 0, s>>>(rev_indptr, u0, u1, r0, uarr);
  check_launch();
  int bu = std::max(1, bits_for((uint64_t)(u1 - u0)));
  int eb = bu + std::max(1, bits_for((uint64_t)T));
  auto* ka = sc.alloc<unsigned long long>(E);
  auto* kb = sc.alloc<unsigned long long>(E);
  int32_t* va = sc.alloc<int32_t>(E);
  int32_t* vb = sc.alloc<int32_t>(E);
  k_tile_keys<<<grid_for(E, 256, sms * 16), 256, 0, s>>>(reinterpret_cast<const int2*>(rev_seg), pool_indptr, n, uarr, r0, E, vt, T, u0, bu, ka, va);
  check_launch();
  {
    cub::DoubleBuffer<unsigned long long> dk(ka, kb);
    cub::DoubleBuffer<int32_t> dv(va, vb);
    size_t tmp = 0;
    TC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, E, 0, eb, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, E, 0, eb, s));
    ka = dk.Current();
    va = dv.Current();
  }
  int32_t* flag = uarr;  // reuse
  int32_t* idx = sc.alloc<int32_t>(E + 1);
  k_owner_flags<<<grid_for(E, 256, sms * 16), 256, 0, s>>>(ka, E, flag);
  check_launch();
  excl_sum(sc, flag, idx, E, s);
  int32_t hk[2];
  TC_CUDA(cudaMemcpyAsync(&hk[0], idx + E - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaMemcpyAsync(&hk[1], flag + E - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  sync_stream(s);
  const int64_t K = (int64_t)hk[0] + hk[1];
  k_owner_emit<<<grid_for(E, 256, sms * 16), 256, 0, s>>>(ka, flag, idx, E, u0, bu, owner_u, owner_ptr);
  check_launch();
  TC_CUDA(cudaMemcpyAsync(owner_ptr + K, &E, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  k_gather_tseg<<<grid_for(E, 256, sms * 16), 256, 0, s>>>(reinterpret_cast<const int2*>(rev_seg), r0, va, E,
                                                           reinterpret_cast<int2*>(segs));
  check_launch();
  int64_t* cost = sc.alloc<int64_t>(K + 1);
  TC_CUDA(cudaMemsetAsync(cost + K, 0, sizeof(int64_t), s));
  k_owner_cost<<<grid_for(K * 32, 256, sms * 16), 256, 0, s>>>(owner_ptr, owner_u,
                                                               reinterpret_cast<const int2*>(segs),
                                                               eff_indptr, K, cost);
  check_launch();
  excl_sum(sc, cost, cost_prefix, K + 1, s);
  sync_stream(s);  // the host-to-device copy of E reads a stack variable
  *k_host = K;
}

}  // namespace tcb

extern "C" int tc_tile_pull(const int64_t* eff_indptr, const int64_t* pool_indptr, int64_t n, const int64_t* rev_indptr,
                            const int32_t* rev_seg, int64_t u0, int64_t u1,
                            int64_t tile_ids, int32_t* owner_u, int64_t* owner_ptr, int32_t* segs,
                            int64_t* cost_prefix, int64_t* k_host, int64_t* ntiles_host, tc_stream_t stream) {
  return tcb::guarded([&] {
    tcb::tile_pull(eff_indptr, pool_indptr, n, rev_indptr, rev_seg, u0, u1, tile_ids, owner_u, owner_ptr, segs,
                   cost_prefix, k_host, ntiles_host, (cudaStream_t)stream);
  });
}

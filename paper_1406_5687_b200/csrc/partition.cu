// partition.cu -- cost-balanced ranges, the task plan, and the surrogate
// (non-overlapping partition) exchange on the device.
//
// balanced_ranges  partitioning.py:95-122   (prefix scan + k-1 lower_bounds)
// plan_tasks       dynamic_lb.py:68-109     (one warp, 32-ary searches)
// census/records   _kernels.py:94-126 scan_for_surrogate (LastProc runs)
// owner segments   _kernels.py:70-91 surrogate_count_list, re-expressed as
//                  pull-engine segments so received lists feed count.cu.
#include <cub/cub.cuh>

#include "common.cuh"

namespace tcb {

static constexpr int kSegCost = 2;  // must match build.cu / count.cu
static constexpr int kTabCost = 16;

template <class T>
static T read_scalar(const T* d, cudaStream_t s) {
  T h;
  TC_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  sync_stream(s);
  return h;
}

template <class In, class Out>
static void inclusive_sum(Scratch& sc, In in, Out out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  TC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out, n, s));
  void* t = sc.bytes(tmp);
  TC_CUDA(cub::DeviceScan::InclusiveSum(t, tmp, in, out, n, s));
}

template <class In, class Out>
static void exclusive_sum(Scratch& sc, In in, Out out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  void* t = sc.bytes(tmp);
  TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, s));
}

// first i in [0, n) with pref[i] >= want (n if none) -- searchsorted 'left'
__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* pref, int64_t n, int64_t want) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (pref[mid] < want) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// bounds[j] for j in [0, k]; pref = inclusive prefix of costs[start, stop)
__global__ void k_bounds(const int64_t* __restrict__ pref, int64_t start, int64_t count, int64_t k,
                         int64_t* bounds) {
  int64_t total = count ? pref[count - 1] : 0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= k;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t b;
    if (j == 0) b = start;
    else if (j == k) b = start + count;
    else if (total == 0) b = start + (j * count) / k;
    else {
      __int128 num = (__int128)j * total;
      int64_t thr = (int64_t)((num + k - 1) / k);  // ceil(j*total/k)
      b = start + lower_bound_i64(pref, count, thr) + 1;
      if (b > start + count) b = start + count;
    }
    bounds[j] = b;
  }
}

static void balanced_bounds(const int64_t* costs, int64_t start, int64_t count, int64_t k,
                            int64_t* bounds, cudaStream_t s) {
  TC_REQUIRE(k >= 1, TC_EINVAL, "k must be >= 1");  // partitioning.py:104-105
  TC_REQUIRE(start >= 0 && count >= 0, TC_EINVAL, "bad node range");
  Scratch sc(s);
  int64_t* pref = sc.alloc<int64_t>(count);
  if (count) inclusive_sum(sc, costs + start, pref, count, s);
  k_bounds<<<grid_for(k + 1, 256), 256, 0, s>>>(pref, start, count, k, bounds);
  check_launch();
}

// ------------------------------------------------------------------ plan

// first i in [lo, hi) with pref[i] >= want, one warp, 32-ary steps
__device__ int64_t warp_lower_bound(const int64_t* pref, int64_t lo, int64_t hi, int64_t want) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    int64_t step = (hi - lo + 31) / 32;
    int64_t idx = lo + (int64_t)(lane + 1) * step - 1;
    bool less = (idx < hi) && (pref[idx] < want);
    int c = __popc(__ballot_sync(0xffffffffu, less));
    lo += (int64_t)c * step;
    hi = min(hi, lo + step);
  }
  bool less = (lo + lane < hi) && (pref[lo + lane] < want);
  return lo + __popc(__ballot_sync(0xffffffffu, less));
}

__global__ void k_plan_tasks(const int64_t* __restrict__ pref, int64_t n, int64_t workers,
                             int64_t* queue_v, int64_t* queue_t, double* targets,
                             int64_t* scal /* [0] split [1] nqueue [2] total */) {
  const int lane = threadIdx.x & 31;
  int64_t total = n ? pref[n - 1] : 0;
  int64_t split = 0;
  if (total != 0) split = warp_lower_bound(pref, 0, n, (total + 1) / 2) + 1;  // :83-88
  int64_t pos = split;
  int64_t remaining = total - (split ? pref[split - 1] : 0);
  int64_t nq = 0;
  while (pos < n) {  // dynamic_lb.py:94-102
    int64_t threshold = remaining > 0 ? (remaining + workers - 1) / workers : 0;
    int64_t base = pos ? pref[pos - 1] : 0;
    int64_t q = warp_lower_bound(pref, 0, n, base + threshold);
    if (q < pos) q = pos;
    if (q > n - 1) q = n - 1;
    if (lane == 0) {
      queue_v[nq] = pos;
      queue_t[nq] = q - pos + 1;
      targets[nq] = (double)remaining / (double)workers;
    }
    ++nq;
    remaining -= pref[q] - base;
    pos = q + 1;
  }
  if (lane == 0) {
    scal[0] = split;
    scal[1] = nq;
    scal[2] = total;
  }
}

__global__ void k_check_nonneg(const int64_t* __restrict__ c, int64_t n, int* bad) {
  GRID_STRIDE(i, n) if (c[i] < 0) atomicOr(bad, 1);
}

static void plan_tasks(const int64_t* costs, int64_t n, int64_t nranks, int64_t* initial_bounds,
                       int64_t* queue_v, int64_t* queue_t, double* targets, int64_t* split_host,
                       int64_t* nqueue_host, int64_t* total_host, cudaStream_t s) {
  TC_REQUIRE(nranks >= 2, TC_EINVAL, "dynamic scheme needs a coordinator plus at least one worker");
  Scratch sc(s);
  if (n) {
    int* bad = sc.alloc<int>(1);
    TC_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    k_check_nonneg<<<grid_for(n, 256), 256, 0, s>>>(costs, n, bad);
    check_launch();
    TC_REQUIRE(read_scalar(bad, s) == 0, TC_EINVAL, "costs must be non-negative");
  }
  int64_t* pref = sc.alloc<int64_t>(n);
  if (n) inclusive_sum(sc, costs, pref, n, s);
  int64_t* scal = sc.alloc<int64_t>(3);
  k_plan_tasks<<<1, 32, 0, s>>>(pref, n, nranks - 1, queue_v, queue_t, targets, scal);
  check_launch();
  int64_t h[3];
  TC_CUDA(cudaMemcpyAsync(h, scal, sizeof(h), cudaMemcpyDeviceToHost, s));
  sync_stream(s);
  // initial = balanced_ranges(costs, [0, split), P-1)   (dynamic_lb.py:89)
  k_bounds<<<grid_for(nranks, 256), 256, 0, s>>>(pref, 0, h[0], nranks - 1, initial_bounds);
  check_launch();
  sync_stream(s);
  *split_host = h[0];
  *nqueue_host = h[1];
  *total_host = h[2];
}

// ------------------------------------------------------------- surrogate

__device__ __forceinline__ int owner_of(const int64_t* bounds, int P, int64_t v) {
  int lo = 0, hi = P;  // largest j with bounds[j] <= v
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (bounds[mid] <= v) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Thread per v: LastProc records (one per remote owner run of N^_v).
__global__ void k_census(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                         int64_t n, const int64_t* __restrict__ bounds, int P,
                         unsigned long long* census, unsigned long long* words) {
  GRID_STRIDE(v, n) {
    int64_t e0 = indptr[v], e1 = indptr[v + 1];
    if (e0 == e1) continue;
    int i = owner_of(bounds, P, v);
    int seg = i, last = -1;
    for (int64_t e = e0; e < e1; ++e) {
      int64_t u = indices[e];
      while (bounds[seg + 1] <= u) ++seg;
      if (seg != i && seg != last) {
        atomicAdd(&census[(int64_t)i * P + seg], 1ull);
        atomicAdd(&words[i], (unsigned long long)(2 + (e1 - e0)));
        last = seg;
      }
    }
  }
}

// number of records of each owned v (for the two-pass emit)
__global__ void k_rec_count(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const int64_t* __restrict__ bounds, int P, int rank, int64_t row_base, int32_t* cnt) {
  const int64_t lo = bounds[rank], hi = bounds[rank + 1];
  GRID_STRIDE(i, hi - lo) {
    int64_t v = lo + i;
    int64_t e0 = indptr[v - row_base], e1 = indptr[v - row_base + 1];
    int seg = rank, last = -1, c = 0;
    for (int64_t e = e0; e < e1; ++e) {
      int64_t u = indices[e];
      while (bounds[seg + 1] <= u) ++seg;
      if (seg != rank && seg != last) {
        ++c;
        last = seg;
      }
    }
    cnt[i] = c;
  }
}

__global__ void k_rec_emit(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const int64_t* __restrict__ bounds, int P, int rank, int64_t row_base,
                           const int32_t* __restrict__ off, uint32_t* dest, int32_t* vv) {
  const int64_t lo = bounds[rank], hi = bounds[rank + 1];
  GRID_STRIDE(i, hi - lo) {
    int64_t v = lo + i;
    int64_t e0 = indptr[v - row_base], e1 = indptr[v - row_base + 1];
    int seg = rank, last = -1;
    int64_t o = off[i];
    for (int64_t e = e0; e < e1; ++e) {
      int64_t u = indices[e];
      while (bounds[seg + 1] <= u) ++seg;
      if (seg != rank && seg != last) {
        dest[o] = (uint32_t)seg;
        vv[o] = (int32_t)v;
        ++o;
        last = seg;
      }
    }
  }
}

// records are sorted by destination: count per dest by binary search
__global__ void k_dest_counts(const uint32_t* __restrict__ dest, int64_t nrec, int P, long long* counts) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) {
    auto lb = [&](uint32_t x) {
      int64_t lo = 0, hi = nrec;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (dest[mid] < x) lo = mid + 1;
        else hi = mid;
      }
      return lo;
    };
    counts[j] = lb((uint32_t)j + 1) - lb((uint32_t)j);
  }
}

__global__ void k_pack_len(const int64_t* __restrict__ indptr, const int32_t* __restrict__ rec_v,
                           int64_t nrec, int64_t* len) {
  GRID_STRIDE(i, nrec) {
    int32_t v = rec_v[i];
    len[i] = indptr[v + 1] - indptr[v];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) len[nrec] = 0;
}

__global__ void k_pack(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                       const int32_t* __restrict__ rec_v, int64_t nrec, const int64_t* __restrict__ off,
                       int32_t* out) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < nrec; r += nwarps) {
    int32_t v = rec_v[r];
    int64_t e0 = indptr[v], e1 = indptr[v + 1], o = off[r];
    for (int64_t e = e0 + lane; e < e1; e += 32) out[o + (e - e0)] = indices[e];
  }
}

// For list l (ids[off[l], off[l+1])) and each position k holding an owned
// id u in [lo, hi) with a non-empty suffix: segment (pool_base + k + 1,
// pool_base + off[l+1]) for owner u - lo.  Warp per list; pass 1 counts per
// list, a scan gives every list its output offset, pass 2 writes in list
// order (no global atomics).
__device__ __forceinline__ bool owned_pos(const int32_t* __restrict__ ids, int64_t k, int64_t b, int64_t lo,
                                          int64_t hi, int32_t* u) {
  if (k >= b) return false;
  *u = ids[k];
  return *u >= lo && *u < hi && k + 1 < b;  // empty suffixes carry no work
}

__global__ void k_owner_seg_count(const int64_t* __restrict__ off, const int32_t* __restrict__ ids, int64_t nl,
                                  int64_t lo, int64_t hi, int64_t* cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t l = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; l < nl; l += nwarps) {
    const int64_t a = off[l], b = off[l + 1];
    int c = 0;
    for (int64_t k = a + lane; k < b; k += 32) {
      int32_t u;
      c += owned_pos(ids, k, b, lo, hi, &u);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) cnt[l] = c;
  }
}

__global__ void k_owner_seg_emit(const int64_t* __restrict__ off, const int32_t* __restrict__ ids, int64_t nl,
                                 int64_t lo, int64_t hi, int64_t pool_base, const int64_t* __restrict__ out_off,
                                 int32_t* owner, int2* segs) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t l = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; l < nl; l += nwarps) {
    const int64_t a = off[l], b = off[l + 1];
    int64_t o = out_off[l];
    for (int64_t k0 = a; k0 < b; k0 += 32) {
      const int64_t k = k0 + lane;
      int32_t u = 0;
      const bool own = owned_pos(ids, k, b, lo, hi, &u);
      const unsigned msk = __ballot_sync(0xffffffffu, own);
      if (own) {
        const int64_t slot = o + __popc(msk & ((1u << lane) - 1u));
        owner[slot] = u - (int32_t)lo;
        segs[slot] = make_int2((int)(pool_base + k + 1), (int)(pool_base + b));
      }
      o += __popc(msk);
    }
  }
}

__global__ void k_seg_cost_rows(const int64_t* __restrict__ row, const int2* __restrict__ segs,
                                const int64_t* __restrict__ tab_indptr, int64_t n, int64_t* cost) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = warp; x < n; x += nwarps) {
    int64_t d = tab_indptr[x + 1] - tab_indptr[x];
    int64_t r0 = row[x], r1 = row[x + 1];
    long long s = 0;
    if (d > 0)
      for (int64_t r = r0 + lane; r < r1; r += 32) s += (segs[r].y - segs[r].x) + kSegCost;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) cost[x] = (d > 0 && r1 > r0) ? (int64_t)s + d + kTabCost : 0;
  }
}

template <class RowOf>
__global__ void k_row_counts2(RowOf row_of, int64_t m, long long* cnt) {
  GRID_STRIDE(i, m) {
    int64_t r = row_of(i);
    if (i == 0 || row_of(i - 1) != r) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[r]), (unsigned long long)(-(long long)i));
    if (i == m - 1 || row_of(i + 1) != r) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[r]), (unsigned long long)(i + 1));
  }
}
struct RowI32 {
  const int32_t* k;
  __device__ int64_t operator()(int64_t i) const { return (int64_t)k[i]; }
};

__global__ void k_iota64(int64_t* a, int64_t n) {
  GRID_STRIDE(i, n) a[i] = i;
}
__global__ void k_gather_segs(const int2* __restrict__ in, const int64_t* __restrict__ idx,
                              int64_t n, int2* out) {
  GRID_STRIDE(i, n) out[i] = in[idx[i]];
}

}  // namespace tcb

extern "C" {

int tc_balanced_bounds(const int64_t* costs, int64_t start, int64_t count, int64_t k,
                       int64_t* bounds, tc_stream_t stream) {
  return tcb::guarded([&] { tcb::balanced_bounds(costs, start, count, k, bounds, (cudaStream_t)stream); });
}

int tc_plan_tasks(const int64_t* costs, int64_t n, int64_t nranks, int64_t* initial_bounds,
                  int64_t* queue_v, int64_t* queue_t, double* targets, int64_t* split_host,
                  int64_t* nqueue_host, int64_t* total_host, tc_stream_t stream) {
  return tcb::guarded([&] {
    tcb::plan_tasks(costs, n, nranks, initial_bounds, queue_v, queue_t, targets, split_host,
                    nqueue_host, total_host, (cudaStream_t)stream);
  });
}

int tc_surrogate_census(const int64_t* eff_indptr, const int32_t* eff_indices, int64_t n,
                        const int64_t* bounds, int32_t P, long long* census, long long* words,
                        tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(P >= 1, TC_EINVAL, "P must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    TC_CUDA(cudaMemsetAsync(census, 0, (size_t)P * P * sizeof(long long), s));
    TC_CUDA(cudaMemsetAsync(words, 0, (size_t)P * sizeof(long long), s));
    if (n == 0 || P == 1) return;
    tcb::k_census<<<tcb::grid_for(n, 256), 256, 0, s>>>(
        eff_indptr, eff_indices, n, bounds, P, reinterpret_cast<unsigned long long*>(census),
        reinterpret_cast<unsigned long long*>(words));
    tcb::check_launch();
  });
}

int tc_surrogate_records(const int64_t* eff_indptr, const int32_t* eff_indices, int64_t n,
                         const int64_t* bounds, int32_t P, int32_t rank, int64_t row_base, int32_t* rec_v,
                         int32_t* rec_dest, int64_t cap, long long* counts, int64_t* nrec_host,
                         tc_stream_t stream) {
  return tcb::guarded([&] {
    (void)n;
    TC_REQUIRE(P >= 1 && rank >= 0 && rank < P, TC_EINVAL, "bad rank");
    cudaStream_t s = (cudaStream_t)stream;
    tcb::Scratch sc(s);
    int64_t hb[2];
    TC_CUDA(cudaMemcpyAsync(hb, bounds + rank, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    tcb::sync_stream(s);
    int64_t nv = hb[1] - hb[0];
    TC_CUDA(cudaMemsetAsync(counts, 0, (size_t)P * sizeof(long long), s));
    *nrec_host = 0;
    if (nv <= 0) return;
    int32_t* cnt = sc.alloc<int32_t>(nv + 1);
    int32_t* off = sc.alloc<int32_t>(nv + 1);
    TC_CUDA(cudaMemsetAsync(cnt + nv, 0, sizeof(int32_t), s));
    tcb::k_rec_count<<<tcb::grid_for(nv, 256), 256, 0, s>>>(eff_indptr, eff_indices, bounds, P, rank, row_base, cnt);
    tcb::check_launch();
    tcb::exclusive_sum(sc, cnt, off, nv + 1, s);
    int32_t nrec = tcb::read_scalar(off + nv, s);
    *nrec_host = nrec;
    TC_REQUIRE(nrec <= cap, TC_EINVAL, "record buffer too small");
    if (nrec == 0) return;
    uint32_t* dk = sc.alloc<uint32_t>(nrec);
    uint32_t* dk2 = sc.alloc<uint32_t>(nrec);
    int32_t* vv = sc.alloc<int32_t>(nrec);
    int32_t* vv2 = sc.alloc<int32_t>(nrec);
    tcb::k_rec_emit<<<tcb::grid_for(nv, 256), 256, 0, s>>>(eff_indptr, eff_indices, bounds, P, rank, row_base, off, dk, vv);
    tcb::check_launch();
    {  // stable sort by destination: grouped by dest, v ascending within
      cub::DoubleBuffer<uint32_t> k(dk, dk2);
      cub::DoubleBuffer<int32_t> v(vv, vv2);
      size_t tmp = 0;
      int eb = std::max(1, tcb::bits_for((uint64_t)P));
      TC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k, v, (int64_t)nrec, 0, eb, s));
      void* t = sc.bytes(tmp);
      TC_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, k, v, (int64_t)nrec, 0, eb, s));
      dk = k.Current();
      vv = v.Current();
    }
    TC_CUDA(cudaMemcpyAsync(rec_v, vv, nrec * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    TC_CUDA(cudaMemcpyAsync(rec_dest, dk, nrec * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    tcb::k_dest_counts<<<tcb::grid_for(P, 128), 128, 0, s>>>(dk, nrec, P, counts);
    tcb::check_launch();
    tcb::sync_stream(s);
  });
}

int tc_surrogate_pack_sizes(const int64_t* eff_indptr, const int32_t* rec_v, int64_t nrec,
                            int64_t* out_offsets, int64_t* total_host, tc_stream_t stream) {
  return tcb::guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    tcb::Scratch sc(s);
    int64_t* len = sc.alloc<int64_t>(nrec + 1);
    tcb::k_pack_len<<<tcb::grid_for(nrec + 1, 256), 256, 0, s>>>(eff_indptr, rec_v, nrec, len);
    tcb::check_launch();
    tcb::exclusive_sum(sc, len, out_offsets, nrec + 1, s);
    *total_host = tcb::read_scalar(out_offsets + nrec, s);
  });
}

int tc_surrogate_pack(const int64_t* eff_indptr, const int32_t* eff_indices, const int32_t* rec_v,
                      int64_t nrec, const int64_t* offsets, int32_t* out_ids, tc_stream_t stream) {
  return tcb::guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    if (nrec <= 0) return;
    tcb::k_pack<<<tcb::grid_for(nrec * 32, 256, tcb::sm_count() * 16), 256, 0, s>>>(
        eff_indptr, eff_indices, rec_v, nrec, offsets, out_ids);
    tcb::check_launch();
  });
}

int tc_owner_segments(const int64_t* list_offsets, const int32_t* list_ids, int64_t nl, int64_t lo,
                      int64_t hi, int64_t pool_base, int32_t* owner, int32_t* segs, int64_t cap,
                      int64_t* nseg_host, tc_stream_t stream) {
  return tcb::guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    *nseg_host = 0;
    if (nl <= 0) return;
    tcb::Scratch sc(s);
    int64_t last = 0;
    TC_CUDA(cudaMemcpyAsync(&last, list_offsets + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    tcb::sync_stream(s);
    TC_REQUIRE(pool_base >= 0 && pool_base + last < (1ll << 31), TC_EINVAL, "segment pool must stay below 2^31 ids");
    int64_t* cnt = sc.alloc<int64_t>(nl + 1);
    int64_t* out_off = sc.alloc<int64_t>(nl + 1);
    TC_CUDA(cudaMemsetAsync(cnt + nl, 0, sizeof(int64_t), s));
    const int grid = tcb::grid_for(nl * 32, 256, tcb::sm_count() * 16);
    tcb::k_owner_seg_count<<<grid, 256, 0, s>>>(list_offsets, list_ids, nl, lo, hi, cnt);
    tcb::check_launch();
    tcb::exclusive_sum(sc, cnt, out_off, nl + 1, s);
    const int64_t c = tcb::read_scalar(out_off + nl, s);
    *nseg_host = c;
    if (owner == nullptr || c == 0) return;
    TC_REQUIRE(c <= cap, TC_EINVAL, "segment buffer too small");
    tcb::k_owner_seg_emit<<<grid, 256, 0, s>>>(list_offsets, list_ids, nl, lo, hi, pool_base, out_off, owner,
                                               reinterpret_cast<int2*>(segs));
    tcb::check_launch();
  });
}

int tc_segments_csr(const int32_t* owner, const int32_t* segs, int64_t nseg, int64_t n_owner,
                    const int64_t* tab_indptr, int64_t* row_indptr, int32_t* row_segs,
                    int64_t* cost_prefix, tc_stream_t stream) {
  return tcb::guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    tcb::Scratch sc(s);
    int32_t* k1 = sc.alloc<int32_t>(nseg);
    int32_t* k2 = sc.alloc<int32_t>(nseg);
    int64_t* i1 = sc.alloc<int64_t>(nseg);
    int64_t* i2 = sc.alloc<int64_t>(nseg);
    if (nseg) {
      TC_CUDA(cudaMemcpyAsync(k1, owner, nseg * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      tcb::k_iota64<<<tcb::grid_for(nseg, 256), 256, 0, s>>>(i1, nseg);
      tcb::check_launch();
      cub::DoubleBuffer<int32_t> k(k1, k2);
      cub::DoubleBuffer<int64_t> v(i1, i2);
      size_t tmp = 0;
      int eb = std::max(1, tcb::bits_for((uint64_t)n_owner));
      TC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k, v, nseg, 0, eb, s));
      void* t = sc.bytes(tmp);
      TC_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, k, v, nseg, 0, eb, s));
      k1 = k.Current();
      i1 = v.Current();
      tcb::k_gather_segs<<<tcb::grid_for(nseg, 256), 256, 0, s>>>(
          reinterpret_cast<const int2*>(segs), i1, nseg, reinterpret_cast<int2*>(row_segs));
      tcb::check_launch();
    }
    long long* cnt = sc.alloc<long long>(n_owner + 1);
    TC_CUDA(cudaMemsetAsync(cnt, 0, (n_owner + 1) * sizeof(long long), s));
    if (nseg) {
      tcb::k_row_counts2<<<tcb::grid_for(nseg, 256), 256, 0, s>>>(tcb::RowI32{k1}, nseg, cnt);
      tcb::check_launch();
    }
    tcb::exclusive_sum(sc, cnt, reinterpret_cast<long long*>(row_indptr), n_owner + 1, s);
    int64_t* cost = sc.alloc<int64_t>(n_owner + 1);
    TC_CUDA(cudaMemsetAsync(cost + n_owner, 0, sizeof(int64_t), s));
    if (n_owner) {
      tcb::k_seg_cost_rows<<<tcb::grid_for(n_owner * 32, 256, tcb::sm_count() * 16), 256, 0, s>>>(
          row_indptr, reinterpret_cast<const int2*>(row_segs), tab_indptr, n_owner, cost);
      tcb::check_launch();
    }
    tcb::exclusive_sum(sc, cost, cost_prefix, n_owner + 1, s);
  });
}

}  // extern "C"

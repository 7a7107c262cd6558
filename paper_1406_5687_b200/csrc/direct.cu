// direct.cu -- the direct (request/response) scheme over non-overlapping
// partitions (space_efficient.py:179-262), B200 form.
//
// The reference owner of v asks u's owner for N^_u once per cross pair
// (v, u) and counts |N^_v ∩ N^_u| itself, so a rank's partial is
// count_node_range(lo, hi) (lowest-vertex attribution).  On the GPU the
// requests of one rank are deduplicated ("rank-level pull"):
//
//   tc_direct_census    the reference's per-pair counters for all ranks at
//                       once (requests_to, reply words), one warp per v.
//   tc_direct_requests  one rank: the distinct remote ids its lists name,
//                       sorted (= grouped by owner), with multiplicities
//                       (= the reference's per-pair request count).
//   tc_direct_table     the rank's lookup CSR over ids [0, n_rows): own rows
//                       from the shard, fetched rows from the replies, every
//                       other row empty -- the push engine then runs
//                       unchanged over [lo, hi).
#include <cub/cub.cuh>

#include "common.cuh"

namespace tcb {

__device__ __forceinline__ int direct_owner(const int64_t* __restrict__ bounds, int P, int64_t v) {
  int lo = 0, hi = P;  // largest j with bounds[j] <= v
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(&bounds[mid]) <= v) lo = mid;
    else hi = mid;
  }
  return lo;
}

static constexpr int kCensusThreads = 256;
static constexpr int kCensusSmemP = 32;  // P <= 32: per-block shared accumulators

// Warp per v.  Lists are ascending and ranges consecutive, so the remote
// ids of N^_v are exactly those >= bounds[owner(v)+1] and their owners are
// non-decreasing along the list: each 32-id window aggregates per owner run
// with a ballot loop before touching the accumulators.
template <bool kShared>
__global__ void __launch_bounds__(kCensusThreads) k_direct_census(
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t n,
    const int64_t* __restrict__ bounds, int P, unsigned long long* req, unsigned long long* words) {
  __shared__ unsigned long long s_req[kShared ? kCensusSmemP * kCensusSmemP : 1];
  __shared__ unsigned long long s_words[kShared ? kCensusSmemP : 1];
  if (kShared) {
    for (int i = threadIdx.x; i < P * P; i += blockDim.x) s_req[i] = 0;
    for (int i = threadIdx.x; i < P; i += blockDim.x) s_words[i] = 0;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += nw) {
    const int64_t e0 = __ldg(&indptr[v]), e1 = __ldg(&indptr[v + 1]);
    if (e0 == e1) continue;
    const int i = direct_owner(bounds, P, v);
    const int64_t bhi = __ldg(&bounds[i + 1]);
    if (__ldg(&indices[e1 - 1]) < bhi) continue;  // no remote id
    for (int64_t b = e0; b < e1; b += 32) {
      const int64_t e = b + lane;
      int j = -1;
      unsigned long long w = 0;
      if (e < e1) {
        const int64_t u = __ldg(&indices[e]);
        if (u >= bhi) {
          j = direct_owner(bounds, P, u);
          w = 2ull + (unsigned long long)(__ldg(&indptr[u + 1]) - __ldg(&indptr[u]));
        }
      }
      unsigned rem = __ballot_sync(0xffffffffu, j >= 0);
      while (rem) {
        const int jl = __shfl_sync(0xffffffffu, j, __ffs(rem) - 1);
        const unsigned peers = __ballot_sync(0xffffffffu, j == jl);
        unsigned long long sw = (j == jl) ? w : 0ull;
        for (int o = 16; o; o >>= 1) sw += __shfl_xor_sync(0xffffffffu, sw, o);
        if (lane == 0) {
          if (kShared) {
            atomicAdd(&s_req[i * P + jl], (unsigned long long)__popc(peers));
            atomicAdd(&s_words[jl], sw);
          } else {
            atomicAdd(&req[(int64_t)i * P + jl], (unsigned long long)__popc(peers));
            atomicAdd(&words[jl], sw);
          }
        }
        rem &= ~peers;
      }
    }
  }
  if (kShared) {
    __syncthreads();
    for (int k = threadIdx.x; k < P * P; k += blockDim.x)
      if (s_req[k]) atomicAdd(&req[k], s_req[k]);
    for (int k = threadIdx.x; k < P; k += blockDim.x)
      if (s_words[k]) atomicAdd(&words[k], s_words[k]);
  }
}

struct AtLeast {
  int32_t hi;
  __host__ __device__ bool operator()(const int32_t& u) const { return u >= hi; }
};

// per destination j: number of distinct ids and sum of multiplicities
__global__ void k_request_split(const int32_t* __restrict__ ids, const int64_t* __restrict__ mult_incl,
                                int64_t k, const int64_t* __restrict__ bounds, int P, long long* counts,
                                long long* ref_counts) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) {
    auto lb = [&](int64_t x) {  // first position with ids[pos] >= x
      int64_t lo = 0, hi = k;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)ids[mid] < x) lo = mid + 1;
        else hi = mid;
      }
      return lo;
    };
    const int64_t a = lb(bounds[j]), b = lb(bounds[j + 1]);
    counts[j] = b - a;
    ref_counts[j] = (b > a) ? mult_incl[b - 1] - (a ? mult_incl[a - 1] : 0) : 0;
  }
}

__global__ void k_table_lens(const int64_t* __restrict__ shard_indptr, int64_t nloc, int64_t lo,
                             const int32_t* __restrict__ req_ids, const int64_t* __restrict__ req_lens,
                             int64_t nreq, int64_t* lens) {
  GRID_STRIDE(i, nloc) lens[lo + i] = shard_indptr[i + 1] - shard_indptr[i];
  GRID_STRIDE(k, nreq) lens[req_ids[k]] = req_lens[k];
}

}  // namespace tcb

extern "C" {

int tc_direct_census(const int64_t* eff_indptr, const int32_t* eff_indices, int64_t n, const int64_t* bounds,
                     int32_t P, long long* requests, long long* reply_words, tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(P >= 1, TC_EINVAL, "P must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    TC_CUDA(cudaMemsetAsync(requests, 0, (size_t)P * P * sizeof(long long), s));
    TC_CUDA(cudaMemsetAsync(reply_words, 0, (size_t)P * sizeof(long long), s));
    if (n == 0 || P == 1) return;
    const int grid = tcb::grid_for(n * 32, tcb::kCensusThreads, tcb::sm_count() * 8);
    auto* rq = reinterpret_cast<unsigned long long*>(requests);
    auto* rw = reinterpret_cast<unsigned long long*>(reply_words);
    if (P <= tcb::kCensusSmemP)
      tcb::k_direct_census<true><<<grid, tcb::kCensusThreads, 0, s>>>(eff_indptr, eff_indices, n, bounds, P, rq, rw);
    else
      tcb::k_direct_census<false><<<grid, tcb::kCensusThreads, 0, s>>>(eff_indptr, eff_indices, n, bounds, P, rq, rw);
    tcb::check_launch();
  });
}

int tc_direct_requests(const int64_t* shard_indptr, const int32_t* shard_indices, int64_t nloc, int64_t hi,
                       const int64_t* bounds, int32_t P, int32_t* req_ids, int64_t* req_mult, int64_t cap,
                       long long* counts, long long* ref_counts, int64_t* nreq_host, tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(P >= 1 && nloc >= 0, TC_EINVAL, "bad sizes");
    cudaStream_t s = (cudaStream_t)stream;
    *nreq_host = 0;
    TC_CUDA(cudaMemsetAsync(counts, 0, (size_t)P * sizeof(long long), s));
    TC_CUDA(cudaMemsetAsync(ref_counts, 0, (size_t)P * sizeof(long long), s));
    if (nloc == 0) {
      tcb::sync_stream(s);
      return;
    }
    int64_t m = 0;
    TC_CUDA(cudaMemcpyAsync(&m, shard_indptr + nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    tcb::sync_stream(s);
    if (m == 0) return;
    tcb::Scratch sc(s);
    // remote ids (>= hi), sorted, run-length encoded
    int32_t* rem = sc.alloc<int32_t>(m);
    int32_t* rem2 = sc.alloc<int32_t>(m);
    long long* nsel = sc.alloc<long long>(1);
    {
      size_t tmp = 0;
      tcb::AtLeast pred{(int32_t)hi};
      TC_CUDA(cub::DeviceSelect::If(nullptr, tmp, shard_indices, rem, nsel, m, pred, s));
      void* t = sc.bytes(tmp);
      TC_CUDA(cub::DeviceSelect::If(t, tmp, shard_indices, rem, nsel, m, pred, s));
    }
    long long k = 0;
    TC_CUDA(cudaMemcpyAsync(&k, nsel, sizeof(k), cudaMemcpyDeviceToHost, s));
    tcb::sync_stream(s);
    if (k == 0) return;
    {
      cub::DoubleBuffer<int32_t> db(rem, rem2);
      size_t tmp = 0;
      TC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, k, 0, 31, s));
      void* t = sc.bytes(tmp);
      TC_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, db, k, 0, 31, s));
      rem = db.Current();
    }
    int32_t* uniq = sc.alloc<int32_t>(k);
    int64_t* mult = sc.alloc<int64_t>(k);
    long long* nruns = sc.alloc<long long>(1);
    {
      size_t tmp = 0;
      TC_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tmp, rem, uniq, mult, nruns, k, s));
      void* t = sc.bytes(tmp);
      TC_CUDA(cub::DeviceRunLengthEncode::Encode(t, tmp, rem, uniq, mult, nruns, k, s));
    }
    long long r = 0;
    TC_CUDA(cudaMemcpyAsync(&r, nruns, sizeof(r), cudaMemcpyDeviceToHost, s));
    tcb::sync_stream(s);
    TC_REQUIRE(r <= cap, TC_EINVAL, "request buffer too small");
    TC_CUDA(cudaMemcpyAsync(req_ids, uniq, r * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    TC_CUDA(cudaMemcpyAsync(req_mult, mult, r * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    int64_t* incl = sc.alloc<int64_t>(r);
    {
      size_t tmp = 0;
      TC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, mult, incl, r, s));
      void* t = sc.bytes(tmp);
      TC_CUDA(cub::DeviceScan::InclusiveSum(t, tmp, mult, incl, r, s));
    }
    tcb::k_request_split<<<tcb::grid_for(P, 128), 128, 0, s>>>(uniq, incl, r, bounds, P, counts, ref_counts);
    tcb::check_launch();
    tcb::sync_stream(s);
    *nreq_host = r;
  });
}

int tc_direct_table(const int64_t* shard_indptr, int64_t nloc, int64_t lo, const int32_t* req_ids,
                    const int64_t* req_lens, int64_t nreq, int64_t n_rows, int64_t* out_indptr,
                    tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(nloc >= 0 && nreq >= 0 && lo >= 0 && lo + nloc <= n_rows, TC_EINVAL, "bad table sizes");
    cudaStream_t s = (cudaStream_t)stream;
    tcb::Scratch sc(s);
    int64_t* lens = sc.alloc<int64_t>(n_rows + 1);
    TC_CUDA(cudaMemsetAsync(lens, 0, (n_rows + 1) * sizeof(int64_t), s));
    const int64_t work = nloc > nreq ? nloc : nreq;
    if (work) {
      tcb::k_table_lens<<<tcb::grid_for(work, 256, tcb::sm_count() * 8), 256, 0, s>>>(shard_indptr, nloc, lo, req_ids,
                                                                                     req_lens, nreq, lens);
      tcb::check_launch();
    }
    size_t tmp = 0;
    TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, lens, out_indptr, n_rows + 1, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, lens, out_indptr, n_rows + 1, s));
  });
}

}  // extern "C"

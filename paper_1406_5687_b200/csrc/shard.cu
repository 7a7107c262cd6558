// shard.cu -- the per-rank device steps of the sharded multi-GPU pipeline
// (paper_1406_5687_b200/sharded.py): a distributed normalize + build_graph
// in which no rank ever holds more than its share of the raw pairs, its
// share of the deduplicated edges and, at the end, the forward lists of its
// own node range (the non-overlapping partition of PAPER.md:314-323), and
// the surrogate exchange of the count (space_efficient.py:81-144) as padded
// suffix lists fed to the middle-vertex engine.
//
// Between these steps the ranks exchange small replicated arrays (label
// presence, first positions, degrees, PRED_SUM costs: all_reduce) and edge
// or list buffers (all_to_all); the collectives run in sharded.py over
// torch.distributed (NCCL).  Every kernel here works on one rank's data.
//
// Semantics followed (reference graph.py:76-153, partitioning.py:79-141):
//   * self-loops are dropped before anything else (graph.py:89);
//   * labels are kept when the distinct labels are exactly 0..K-1
//     (graph.py:94), else compacted in order of first occurrence in the
//     raveled (u0, v0, u1, v1, ...) list (graph.py:92-99) -- a rank's pair i
//     has raveled positions 2 (base + i) and 2 (base + i) + 1;
//   * canonical order = ascending (degree, id), stable (graph.py:152);
//   * PRED_SUM cost of v = sum over w with v in N^_w of d^_w + d^_v
//     (partitioning.py:91).
#include <cub/cub.cuh>

#include "common.cuh"

namespace tcb {

static constexpr int kSegCostS = 2;  // must match count.cu / build.cu
static constexpr int kTabCostS = 16;
static constexpr int kBlk = 256;

__device__ __forceinline__ long long add64(long long* p, long long v) {
  return (long long)atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

template <class T>
static T scalar_of(const T* d, cudaStream_t s) {
  T h;
  TC_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  sync_stream(s);
  return h;
}

template <class In, class Out>
static void ex_sum(Scratch& sc, In in, Out out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  void* t = sc.bytes(tmp);
  TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, s));
}

// ------------------------------------------------------------ labels

__global__ void k_sh_minmax(const int32_t* __restrict__ p, int64_t n2, int* mm) {
  int lo = INT_MAX, hi = INT_MIN;
  GRID_STRIDE(i, n2) {
    lo = min(lo, p[i]);
    hi = max(hi, p[i]);
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
}

// presence (uint8) and first raveled position (int32) of every label that
// occurs in a non-self-loop pair
__global__ void k_sh_scan(const int2* __restrict__ pairs, int64_t m, int64_t pos_base, uint8_t* present,
                          int32_t* first) {
  GRID_STRIDE(i, m) {
    const int2 e = pairs[i];
    if (e.x == e.y) continue;
    present[e.x] = 1;
    present[e.y] = 1;
    const int32_t q = (int32_t)(2 * (pos_base + i));
    atomicMin(&first[e.x], q);
    atomicMin(&first[e.y], q + 1);
  }
}

__global__ void k_sh_identity(int32_t* map, int64_t k) {
  GRID_STRIDE(i, k) map[i] = (int32_t)i;
}

__global__ void k_sh_present_keys(const uint8_t* __restrict__ present, const int32_t* __restrict__ first, int64_t k,
                                  uint32_t* key, int32_t* val, int32_t* map) {
  GRID_STRIDE(i, k) {
    key[i] = present[i] ? (uint32_t)first[i] : 0xFFFFFFFFu;  // absent labels sort last
    val[i] = (int32_t)i;
    map[i] = -1;
  }
}

__global__ void k_sh_rank_scatter(const int32_t* __restrict__ lab, int64_t cnt, int32_t* map) {
  GRID_STRIDE(r, cnt) map[lab[r]] = (int32_t)r;
}

// ------------------------------------------------------------ dedup routing

__device__ __forceinline__ int dest_of_key(unsigned long long key, int P) {
  return (int)(((key * 0x9E3779B97F4A7C15ull) >> 33) % (unsigned long long)P);
}

__global__ void k_sh_keys(const int2* __restrict__ pairs, int64_t m, const int32_t* __restrict__ map, int P,
                          unsigned long long* key, int32_t* dest, long long* counts) {
  GRID_STRIDE(i, m) {
    const int2 e = pairs[i];
    int d = -1;
    unsigned long long k = 0;
    if (e.x != e.y) {
      const uint32_t a = (uint32_t)(map ? map[e.x] : e.x), b = (uint32_t)(map ? map[e.y] : e.y);
      k = ((unsigned long long)min(a, b) << 32) | max(a, b);
      d = dest_of_key(k, P);
      add64(&counts[d], 1ll);
    }
    key[i] = k;
    dest[i] = d;
  }
}

// scatter into groups by destination (order inside a group unspecified)
template <class T>
__global__ void k_sh_group(const T* __restrict__ in, const int32_t* __restrict__ dest, int64_t m,
                           const long long* __restrict__ counts, const long long* __restrict__ off, long long* cursor,
                           T* out) {
  GRID_STRIDE(i, m) {
    const int d = dest[i];
    if (d < 0) continue;
    const long long c = add64(&cursor[d], 1ll);
#if TCB_DEBUG
    assert(c < counts[d]);
#else
    (void)counts;
#endif
    out[off[d] + c] = in[i];
  }
}

__global__ void k_sh_unique_flags(const unsigned long long* __restrict__ k, int64_t n, uint8_t* f) {
  GRID_STRIDE(i, n) f[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

// ------------------------------------------------------------ build

__global__ void k_sh_degrees(const unsigned long long* __restrict__ key, int64_t k, int32_t* deg) {
  GRID_STRIDE(i, k) {
    atomicAdd(&deg[(int32_t)(key[i] >> 32)], 1);
    atomicAdd(&deg[(int32_t)(key[i] & 0xFFFFFFFFu)], 1);
  }
}

__global__ void k_sh_iota(int32_t* a, int64_t n) {
  GRID_STRIDE(i, n) a[i] = (int32_t)i;
}
__global__ void k_sh_relabel(const int32_t* __restrict__ orig, int64_t n, int32_t* relabel) {
  GRID_STRIDE(i, n) relabel[orig[i]] = (int32_t)i;
}

__global__ void k_sh_orient(const unsigned long long* __restrict__ key, int64_t k, const int32_t* __restrict__ relabel,
                            int2* lohi, int32_t* effdeg) {
  GRID_STRIDE(i, k) {
    const int32_t a = relabel[(int32_t)(key[i] >> 32)], b = relabel[(int32_t)(key[i] & 0xFFFFFFFFu)];
    const int32_t lo = min(a, b), hi = max(a, b);
    lohi[i] = make_int2(lo, hi);
    atomicAdd(&effdeg[lo], 1);
  }
}

__global__ void k_sh_predsum(const int2* __restrict__ lohi, int64_t k, const int32_t* __restrict__ effdeg,
                             unsigned long long* cost) {
  GRID_STRIDE(i, k) {
    const int2 e = lohi[i];
    atomicAdd(&cost[e.y], (unsigned long long)(effdeg[e.x] + effdeg[e.y]));
  }
}

__device__ __forceinline__ int owner_of_id(const int64_t* __restrict__ bounds, int P, int64_t v) {
  int lo = 0, hi = P;  // largest j with bounds[j] <= v
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (bounds[mid] <= v) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void k_sh_route_dest(const int2* __restrict__ lohi, int64_t k, const int64_t* __restrict__ bounds, int P,
                                int32_t* dest, long long* counts) {
  GRID_STRIDE(i, k) {
    const int d = owner_of_id(bounds, P, lohi[i].x);
    dest[i] = d;
    add64(&counts[d], 1ll);
  }
}

__global__ void k_sh_row_count(const int2* __restrict__ lohi, int64_t k, int64_t lo, long long* cnt) {
  GRID_STRIDE(i, k) add64(&cnt[lohi[i].x - lo], 1ll);
}

__global__ void k_sh_row_scatter(const int2* __restrict__ lohi, int64_t k, int64_t lo,
                                 const int64_t* __restrict__ indptr, int32_t* cursor, int32_t* out) {
  GRID_STRIDE(i, k) {
    const int64_t r = lohi[i].x - lo;
    out[indptr[r] + atomicAdd(&cursor[r], 1)] = lohi[i].y;
  }
}

// padded pool (rows at multiples of 4 ids, INT32_MAX padding); warp per row
__global__ void k_sh_pool_sizes(const int64_t* __restrict__ indptr, int64_t nrow, int64_t* sz) {
  GRID_STRIDE(v, nrow + 1) sz[v] = (v < nrow) ? ((indptr[v + 1] - indptr[v] + 3) & ~(int64_t)3) : 0;
}

__global__ void k_sh_pool_fill(const int64_t* __restrict__ indptr, const int32_t* __restrict__ ids, int64_t nrow,
                               const int64_t* __restrict__ pptr, int32_t* pool) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < nrow; v += nw) {
    const int64_t a = indptr[v], d = indptr[v + 1] - a, p = pptr[v], pd = pptr[v + 1] - p;
    for (int64_t i = lane; i < pd; i += 32) pool[p + i] = i < d ? ids[a + i] : INT32_MAX;
  }
}

__global__ void k_sh_len_sizes(const int32_t* __restrict__ len, int64_t nrow, int64_t* sz) {
  GRID_STRIDE(r, nrow + 1) sz[r] = (r < nrow) ? (((int64_t)len[r] + 3) & ~(int64_t)3) : 0;
}

__global__ void k_sh_fill(int32_t* p, int64_t k, int32_t v) {
  GRID_STRIDE(i, k) p[i] = v;
}

// engine cost contributions of local rows (global owner ids): every
// predecessor entry (v, u) adds the suffix length + kSegCost to u
__global__ void k_sh_engine_cost(const int64_t* __restrict__ indptr, const int32_t* __restrict__ ids, int64_t nrow,
                                 int64_t seg_weight, unsigned long long* acc) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < nrow; v += nw) {
    const int64_t a = indptr[v], d = indptr[v + 1] - a;
    for (int64_t i = lane; i < d; i += 32)
      atomicAdd(&acc[ids[a + i]], (unsigned long long)(d - i - 1 + seg_weight));
  }
}

__global__ void k_sh_engine_cost_fin(const unsigned long long* __restrict__ acc, const int32_t* __restrict__ effdeg,
                                     int64_t n, int64_t tab_weight, int64_t send_weight, int64_t* cost) {
  GRID_STRIDE(u, n) {
    const int64_t d = effdeg[u];
    cost[u] = ((d > 0 && acc[u] > 0) ? (int64_t)acc[u] + tab_weight * d + kTabCostS : 0) + send_weight * d;
  }
}

// ------------------------------------------------------------ surrogate send

// first position in row [a, a + d) with ids[pos] >= x
__device__ __forceinline__ int64_t row_lb(const int32_t* __restrict__ ids, int64_t a, int64_t d, int64_t x) {
  int64_t lo = 0, hi = d;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ids[a + mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Per row v and destination j > rank that owns an id of N^_v (LastProc,
// _kernels.py:94-126): one list message.  The receiver only ever reads the
// part of N^_v at or above bounds[j] (a triangle's middle vertex owned by j
// and its third vertex come after u >= bounds[j]), so the message is the
// row of the padded pool from the 16-byte chunk holding the first id >=
// bounds[j] to the row's padded end (the few leading ids of that chunk are
// < bounds[j]: they never own a segment and never lie in a suffix).
// Per destination: lists, padded ids, whole-list words (the reference's
// bytes_sent accounting).  Lane = destination.
__global__ void k_sh_send_count(const int64_t* __restrict__ indptr, const int32_t* __restrict__ ids, int64_t nrow,
                                const int64_t* __restrict__ pptr, const int64_t* __restrict__ bounds, int P,
                                int rank, long long* lists, long long* words, long long* full) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  long long cl = 0, cw = 0, cf = 0;
  const int j = lane;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < nrow; v += nw) {
    const int64_t a = indptr[v], d = indptr[v + 1] - a;
    if (j > rank && j < P && d > 0) {
      const int64_t s = row_lb(ids, a, d, bounds[j]), e = row_lb(ids, a, d, bounds[j + 1]);
      if (s < e) {
        ++cl;
        cw += (pptr[v + 1] - pptr[v]) - (s & ~3ll);
        cf += d;
      }
    }
  }
  if (j < P) {
    add64(&lists[j], cl);
    add64(&words[j], cw);
    add64(&full[j], cf);
  }
}

// Emit pass.  A block takes a contiguous run of rows; its warps (one row at
// a time, lanes = destinations) first total the block's messages per
// destination in shared memory, one thread claims the block's ranges with
// one global atomic per destination, and the warps then claim slots inside
// them and copy each message as 16-byte chunks of the padded pool.  A slot
// claim is one 64-bit atomic holding the message count (high 26 bits) and
// its words (low 38), so the lengths and the lists agree in order (which is
// otherwise unspecified; the receiver's count does not depend on it).
static constexpr int kEmitMaxP = 32;
__device__ __forceinline__ bool send_dest(const int32_t* __restrict__ ids, int64_t a, int64_t d,
                                          const int64_t* __restrict__ bounds, int lane, int P, int rank, int64_t& s) {
  s = 0;
  if (lane <= rank || lane >= P) return false;
  s = row_lb(ids, a, d, bounds[lane]);
  return s < row_lb(ids, a, d, bounds[lane + 1]);
}

__global__ void k_sh_send_emit(const int64_t* __restrict__ indptr, const int32_t* __restrict__ ids, int64_t nrow,
                               const int64_t* __restrict__ pptr, const int4* __restrict__ pool4,
                               const int64_t* __restrict__ bounds, int P, int rank,
                               const long long* __restrict__ list_off, const long long* __restrict__ word_off,
                               unsigned long long* cur, int32_t* out_len, int4* out4) {
  __shared__ unsigned long long btot[kEmitMaxP], bcur[kEmitMaxP];
  __shared__ long long bl[kEmitMaxP], bw[kEmitMaxP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int64_t per = (nrow + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(nrow, r0 + per);
  if (threadIdx.x < kEmitMaxP) {
    btot[threadIdx.x] = 0;
    bcur[threadIdx.x] = 0;
  }
  __syncthreads();
  for (int64_t v = r0 + warp; v < r1; v += nwarp) {  // block totals
    const int64_t a = indptr[v], d = indptr[v + 1] - a;
    if (d == 0) continue;
    int64_t s;
    if (send_dest(ids, a, d, bounds, lane, P, rank, s)) {
      const int64_t nch = ((pptr[v + 1] - pptr[v]) >> 2) - (s >> 2);
      atomicAdd(&btot[lane], (1ull << 38) + (unsigned long long)(4 * nch));
    }
  }
  __syncthreads();
  if (threadIdx.x < P && btot[threadIdx.x]) {  // the block's ranges
    const unsigned long long old = atomicAdd(&cur[threadIdx.x], btot[threadIdx.x]);
    bl[threadIdx.x] = list_off[threadIdx.x] + (long long)(old >> 38);
    bw[threadIdx.x] = word_off[threadIdx.x] + (long long)(old & ((1ull << 38) - 1));
  }
  __syncthreads();
  for (int64_t v = r0 + warp; v < r1; v += nwarp) {
    const int64_t a = indptr[v], d = indptr[v + 1] - a;
    if (d == 0) continue;
    int64_t s;
    const bool hit = send_dest(ids, a, d, bounds, lane, P, rank, s);
    unsigned todo = __ballot_sync(0xffffffffu, hit);
    const int64_t p0 = pptr[v] >> 2, pd = (pptr[v + 1] - pptr[v]) >> 2;  // in chunks
    long long li = 0, wi = 0;
    if (hit) {  // lane j claims this row's slot in destination j's block range
      const int64_t nch = pd - (s >> 2);
      const unsigned long long old = atomicAdd(&bcur[lane], (1ull << 38) + (unsigned long long)(4 * nch));
      li = bl[lane] + (long long)(old >> 38);
      wi = bw[lane] + (long long)(old & ((1ull << 38) - 1));
      out_len[li] = (int32_t)(d - 4 * (s >> 2));
    }
    while (todo) {
      const int jj = __ffs(todo) - 1;
      todo &= todo - 1;
      const int64_t c0 = __shfl_sync(0xffffffffu, s, jj) >> 2;  // first chunk of the message
      const int64_t w0 = __shfl_sync(0xffffffffu, wi, jj) >> 2;
      for (int64_t c = lane; c < pd - c0; c += 32) out4[w0 + c] = __ldg(&pool4[p0 + c0 + c]);
    }
  }
}

// ------------------------------------------------------------ receive index

// Rows of a padded pool (row r at pptr[r], length len[r]); owners u in
// [lo, hi).  Pass 1 accumulates, per owner, its non-empty suffix segments
// and their total length in one 64-bit atomic (count << 40 | length sum);
// pass 2 scatters the segments with a 32-bit cursor.
static constexpr int kCntShift = 40;
__global__ void k_sh_idx_count(const int64_t* __restrict__ pptr, const int32_t* __restrict__ len, int64_t nrow,
                               const int32_t* __restrict__ pool, int64_t lo, int64_t hi, unsigned long long* acc) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrow; r += nw) {
    const int64_t p = pptr[r], d = len[r];
    for (int64_t i = lane; i + 1 < d; i += 32) {
      const int32_t u = pool[p + i];
      if (u >= lo && u < hi)
        atomicAdd(&acc[u - lo], (1ull << kCntShift) + (unsigned long long)(d - i - 1));
    }
  }
}

__global__ void k_sh_idx_rows(const unsigned long long* __restrict__ acc, const int64_t* __restrict__ tab_indptr,
                              int64_t nx, int64_t* cnt, int64_t* cost) {
  GRID_STRIDE(x, nx + 1) {
    if (x == nx) {
      cnt[x] = 0;
      cost[x] = 0;
      continue;
    }
    const unsigned long long a = acc[x];
    const int64_t k = (int64_t)(a >> kCntShift), sum = (int64_t)(a & ((1ull << kCntShift) - 1));
    const int64_t d = tab_indptr[x + 1] - tab_indptr[x];
    cnt[x] = k;
    // the pull-engine cost of build_graph's rev_cost (suffix lengths + 2 per
    // segment, table d + 16)
    cost[x] = (d > 0 && k > 0) ? sum + kSegCostS * k + d + kTabCostS : 0;
  }
}

__global__ void k_sh_idx_emit(const int64_t* __restrict__ pptr, const int32_t* __restrict__ len, int64_t nrow,
                              const int32_t* __restrict__ pool, int64_t lo, int64_t hi,
                              const int64_t* __restrict__ rev_indptr, int32_t* cursor, int2* rev_seg) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrow; r += nw) {
    const int64_t p = pptr[r], d = len[r];
    for (int64_t i = lane; i + 1 < d; i += 32) {
      const int32_t u = pool[p + i];
      if (u >= lo && u < hi) {
        const int64_t x = u - lo;
        const int64_t slot = rev_indptr[x] + atomicAdd(&cursor[x], 1);
#if TCB_DEBUG
        assert(slot < rev_indptr[x + 1]);
#endif
        rev_seg[slot] = make_int2((int)(p + i + 1), (int)(p + d));
      }
    }
  }
}

}  // namespace tcb

using namespace tcb;

extern "C" {

int tc_shard_minmax(const int32_t* pairs, int64_t m, int32_t* min_host, int32_t* max_host, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    *min_host = INT_MAX;
    *max_host = -1;
    if (m <= 0) return;
    Scratch sc(s);
    int* mm = sc.alloc<int>(2);
    const int init[2] = {INT_MAX, INT_MIN};
    TC_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_sh_minmax<<<grid_for(2 * m, kBlk), kBlk, 0, s>>>(pairs, 2 * m, mm);
    check_launch();
    int h[2];
    TC_CUDA(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, s));
    sync_stream(s);
    *min_host = h[0];
    *max_host = h[1];
  });
}

int tc_shard_label_scan(const int32_t* pairs, int64_t m, int64_t pos_base, int64_t k, uint8_t* present,
                        int32_t* first, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(k >= 0 && m >= 0 && pos_base >= 0, TC_EINVAL, "bad sizes");
    TC_REQUIRE(2 * (pos_base + m) < INT32_MAX, TC_EINVAL, "raveled positions must fit int32");
    if (k == 0) return;
    TC_CUDA(cudaMemsetAsync(present, 0, k, s));
    TC_CUDA(cudaMemsetAsync(first, 0x7F, k * sizeof(int32_t), s));  // 0x7F7F7F7F > every position
    if (m == 0) return;
    k_sh_scan<<<grid_for(m, kBlk), kBlk, 0, s>>>(reinterpret_cast<const int2*>(pairs), m, pos_base, present, first);
    check_launch();
  });
}

int tc_shard_relabel_map(const uint8_t* present, const int32_t* first, int64_t k, int32_t* map, int64_t* n_host,
                         int32_t* dense_host, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    *n_host = 0;
    *dense_host = 1;
    if (k == 0) return;
    Scratch sc(s);
    long long* cnt = sc.alloc<long long>(1);
    {
      size_t tmp = 0;
      TC_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, present, cnt, k, s));
      void* t = sc.bytes(tmp);
      TC_CUDA(cub::DeviceReduce::Sum(t, tmp, present, cnt, k, s));
    }
    const long long c = scalar_of(cnt, s);
    *n_host = c;
    if (c == k) {  // dense labels are kept (graph.py:94)
      k_sh_identity<<<grid_for(k, kBlk), kBlk, 0, s>>>(map, k);
      check_launch();
      return;
    }
    *dense_host = 0;
    // first-seen compaction (graph.py:95-99): present labels ranked by first position
    uint32_t* k1 = sc.alloc<uint32_t>(k);
    uint32_t* k2 = sc.alloc<uint32_t>(k);
    int32_t* v1 = sc.alloc<int32_t>(k);
    int32_t* v2 = sc.alloc<int32_t>(k);
    k_sh_present_keys<<<grid_for(k, kBlk), kBlk, 0, s>>>(present, first, k, k1, v1, map);
    check_launch();
    cub::DoubleBuffer<uint32_t> kb(k1, k2);
    cub::DoubleBuffer<int32_t> vb(v1, v2);
    size_t tmp = 0;
    TC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, k, 0, 32, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, k, 0, 32, s));
    k_sh_rank_scatter<<<grid_for(c, kBlk), kBlk, 0, s>>>(vb.Current(), c, map);
    check_launch();
  });
}

int tc_shard_keys(const int32_t* pairs, int64_t m, const int32_t* map, int32_t P, uint64_t* keys_out,
                  int64_t* counts_host, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(P >= 1 && P <= 1024, TC_EINVAL, "P must be in [1, 1024]");
    for (int j = 0; j < P; ++j) counts_host[j] = 0;
    if (m <= 0) return;
    Scratch sc(s);
    auto* key = sc.alloc<unsigned long long>(m);
    int32_t* dest = sc.alloc<int32_t>(m);
    long long* cnt = sc.alloc<long long>(3 * P);
    TC_CUDA(cudaMemsetAsync(cnt, 0, 3 * P * sizeof(long long), s));
    k_sh_keys<<<grid_for(m, kBlk), kBlk, 0, s>>>(reinterpret_cast<const int2*>(pairs), m, map, P, key, dest, cnt);
    check_launch();
    ex_sum(sc, cnt, cnt + P, P, s);
    k_sh_group<<<grid_for(m, kBlk), kBlk, 0, s>>>(key, dest, m, cnt, cnt + P, cnt + 2 * P,
                                                 reinterpret_cast<unsigned long long*>(keys_out));
    check_launch();
    TC_CUDA(cudaMemcpyAsync(counts_host, cnt, P * sizeof(long long), cudaMemcpyDeviceToHost, s));
    sync_stream(s);
  });
}

int tc_shard_dedup(const uint64_t* keys, int64_t k, int32_t key_bits, uint64_t* out, int64_t* k_host,
                   tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    *k_host = 0;
    if (k <= 0) return;
    Scratch sc(s);
    auto* a = sc.alloc<unsigned long long>(k);
    auto* b = sc.alloc<unsigned long long>(k);
    TC_CUDA(cudaMemcpyAsync(a, keys, k * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
    cub::DoubleBuffer<unsigned long long> db(a, b);
    size_t tmp = 0;
    const int bits = std::max(1, std::min(64, (int)key_bits));
    // keys are (lo << 32 | hi): sort the hi bits and the lo bits
    TC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, k, 0, 64, s));
    void* t = sc.bytes(tmp);
    if (bits >= 32) {
      TC_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, db, k, 0, 64, s));
    } else {
      // labels < 2^bits: sort bits [0, bits) then [32, 32 + bits)
      TC_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, db, k, 0, bits, s));
      TC_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, db, k, 32, 32 + bits, s));
    }
    uint8_t* f = sc.alloc<uint8_t>(k);
    k_sh_unique_flags<<<grid_for(k, kBlk), kBlk, 0, s>>>(db.Current(), k, f);
    check_launch();
    long long* nsel = sc.alloc<long long>(1);
    size_t tmp2 = 0;
    TC_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp2, db.Current(), f, reinterpret_cast<unsigned long long*>(out), nsel,
                                       k, s));
    void* t2 = sc.bytes(tmp2);
    TC_CUDA(cub::DeviceSelect::Flagged(t2, tmp2, db.Current(), f, reinterpret_cast<unsigned long long*>(out), nsel, k,
                                       s));
    *k_host = scalar_of(nsel, s);
  });
}

int tc_shard_degrees(const uint64_t* keys, int64_t k, int32_t* deg, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    if (k <= 0) return;
    k_sh_degrees<<<grid_for(k, kBlk), kBlk, 0, s>>>(reinterpret_cast<const unsigned long long*>(keys), k, deg);
    check_launch();
  });
}

int tc_shard_order(const int32_t* deg, int64_t n, int32_t* orig_ids, int32_t* relabel, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    if (n <= 0) return;
    Scratch sc(s);
    int32_t* k1 = sc.alloc<int32_t>(n);
    int32_t* k2 = sc.alloc<int32_t>(n);
    int32_t* v1 = sc.alloc<int32_t>(n);
    int32_t* v2 = sc.alloc<int32_t>(n);
    TC_CUDA(cudaMemcpyAsync(k1, deg, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    k_sh_iota<<<grid_for(n, kBlk), kBlk, 0, s>>>(v1, n);
    check_launch();
    cub::DoubleBuffer<int32_t> kb(k1, k2), vb(v1, v2);
    size_t tmp = 0;
    TC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, n, 0, 31, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, n, 0, 31, s));  // stable: (degree, id)
    TC_CUDA(cudaMemcpyAsync(orig_ids, vb.Current(), n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    k_sh_relabel<<<grid_for(n, kBlk), kBlk, 0, s>>>(orig_ids, n, relabel);
    check_launch();
  });
}

int tc_shard_orient(const uint64_t* keys, int64_t k, const int32_t* relabel, int32_t* lohi, int32_t* effdeg,
                    tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    if (k <= 0) return;
    k_sh_orient<<<grid_for(k, kBlk), kBlk, 0, s>>>(reinterpret_cast<const unsigned long long*>(keys), k, relabel,
                                                  reinterpret_cast<int2*>(lohi), effdeg);
    check_launch();
  });
}

int tc_shard_predsum(const int32_t* lohi, int64_t k, const int32_t* effdeg, int64_t* cost, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    if (k <= 0) return;
    k_sh_predsum<<<grid_for(k, kBlk), kBlk, 0, s>>>(reinterpret_cast<const int2*>(lohi), k, effdeg,
                                                   reinterpret_cast<unsigned long long*>(cost));
    check_launch();
  });
}

int tc_shard_route(const int32_t* lohi, int64_t k, const int64_t* bounds, int32_t P, int32_t* out,
                   int64_t* counts_host, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(P >= 1 && P <= 1024, TC_EINVAL, "P must be in [1, 1024]");
    for (int j = 0; j < P; ++j) counts_host[j] = 0;
    if (k <= 0) return;
    Scratch sc(s);
    int32_t* dest = sc.alloc<int32_t>(k);
    long long* cnt = sc.alloc<long long>(3 * P);
    TC_CUDA(cudaMemsetAsync(cnt, 0, 3 * P * sizeof(long long), s));
    k_sh_route_dest<<<grid_for(k, kBlk), kBlk, 0, s>>>(reinterpret_cast<const int2*>(lohi), k, bounds, P, dest, cnt);
    check_launch();
    ex_sum(sc, cnt, cnt + P, P, s);
    k_sh_group<<<grid_for(k, kBlk), kBlk, 0, s>>>(reinterpret_cast<const int2*>(lohi), dest, k, cnt, cnt + P, cnt + 2 * P,
                                                 reinterpret_cast<int2*>(out));
    check_launch();
    TC_CUDA(cudaMemcpyAsync(counts_host, cnt, P * sizeof(long long), cudaMemcpyDeviceToHost, s));
    sync_stream(s);
  });
}

int tc_shard_csr(const int32_t* lohi, int64_t k, int64_t lo, int64_t nrow, int64_t* indptr, int32_t* indices,
                 tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(k < (1ll << 31), TC_EINVAL, "shard too large (>= 2^31 edges)");
    Scratch sc(s);
    long long* cnt = sc.alloc<long long>(nrow + 1);
    TC_CUDA(cudaMemsetAsync(cnt, 0, (nrow + 1) * sizeof(long long), s));
    if (k > 0) {
      k_sh_row_count<<<grid_for(k, kBlk), kBlk, 0, s>>>(reinterpret_cast<const int2*>(lohi), k, lo, cnt);
      check_launch();
    }
    ex_sum(sc, cnt, reinterpret_cast<long long*>(indptr), nrow + 1, s);
    if (k == 0) return;
    int32_t* cur = sc.alloc<int32_t>(nrow);
    int32_t* unsorted = sc.alloc<int32_t>(k);
    TC_CUDA(cudaMemsetAsync(cur, 0, nrow * sizeof(int32_t), s));
    k_sh_row_scatter<<<grid_for(k, kBlk), kBlk, 0, s>>>(reinterpret_cast<const int2*>(lohi), k, lo, indptr, cur,
                                                       unsorted);
    check_launch();
    size_t tmp = 0;
    TC_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, unsorted, indices, (int)k, (int)nrow, indptr, indptr + 1,
                                               s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceSegmentedSort::SortKeys(t, tmp, unsorted, indices, (int)k, (int)nrow, indptr, indptr + 1, s));
  });
}

int tc_shard_pool(const int64_t* indptr, const int32_t* indices, int64_t nrow, int64_t* pool_indptr, int32_t* pool,
                  tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    Scratch sc(s);
    k_sh_fill<<<1, kBlk, 0, s>>>(pool - TC_POOL_HEAD, TC_POOL_HEAD, INT32_MAX);
    check_launch();
    int64_t* sz = sc.alloc<int64_t>(nrow + 1);
    k_sh_pool_sizes<<<grid_for(nrow + 1, kBlk), kBlk, 0, s>>>(indptr, nrow, sz);
    check_launch();
    ex_sum(sc, sz, pool_indptr, nrow + 1, s);
    if (nrow > 0) {
      k_sh_pool_fill<<<grid_for(nrow * 32, kBlk, sm_count() * 16), kBlk, 0, s>>>(indptr, indices, nrow, pool_indptr,
                                                                                pool);
      check_launch();
    }
  });
}

int tc_shard_engine_cost(const int64_t* indptr, const int32_t* indices, int64_t nrow, int64_t seg_weight,
                         uint64_t* acc, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(seg_weight >= 0, TC_EINVAL, "negative segment weight");
    if (nrow <= 0) return;
    k_sh_engine_cost<<<grid_for(nrow * 32, kBlk, sm_count() * 16), kBlk, 0, s>>>(
        indptr, indices, nrow, seg_weight, reinterpret_cast<unsigned long long*>(acc));
    check_launch();
  });
}

int tc_shard_engine_cost_fin(const uint64_t* acc, const int32_t* effdeg, int64_t n, int64_t tab_weight,
                             int64_t send_weight, int64_t* cost, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    if (n <= 0) return;
    TC_REQUIRE(tab_weight >= 0 && send_weight >= 0, TC_EINVAL, "negative weight");
    k_sh_engine_cost_fin<<<grid_for(n, kBlk), kBlk, 0, s>>>(reinterpret_cast<const unsigned long long*>(acc), effdeg, n,
                                                          tab_weight, send_weight, cost);
    check_launch();
  });
}

int tc_shard_send_sizes(const int64_t* indptr, const int32_t* indices, int64_t nrow, const int64_t* pool_indptr,
                        const int64_t* bounds, int32_t P, int32_t rank, int64_t* sizes_dev, int64_t* sizes_host,
                        tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(P >= 1 && P <= 32, TC_EINVAL, "the surrogate send supports P <= 32 ranks");
    TC_REQUIRE(rank >= 0 && rank < P, TC_EINVAL, "rank out of range");
    TC_CUDA(cudaMemsetAsync(sizes_dev, 0, 3 * P * sizeof(int64_t), s));
    if (nrow > 0) {
      k_sh_send_count<<<grid_for(nrow * 32, kBlk, sm_count() * 8), kBlk, 0, s>>>(
          indptr, indices, nrow, pool_indptr, bounds, P, rank, reinterpret_cast<long long*>(sizes_dev),
          reinterpret_cast<long long*>(sizes_dev) + P, reinterpret_cast<long long*>(sizes_dev) + 2 * P);
      check_launch();
    }
    if (sizes_host) {
      TC_CUDA(cudaMemcpyAsync(sizes_host, sizes_dev, 3 * P * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      sync_stream(s);
    }
  });
}

int tc_shard_send_pack(const int64_t* indptr, const int32_t* indices, int64_t nrow, const int64_t* pool_indptr,
                       const int32_t* pool, const int64_t* bounds, int32_t P, int32_t rank, const int64_t* sizes_dev,
                       int32_t* out_len, int32_t* out_ids, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(P >= 1 && P <= 32, TC_EINVAL, "the surrogate send supports P <= 32 ranks");
    TC_REQUIRE(((uintptr_t)pool & 15) == 0 && ((uintptr_t)out_ids & 15) == 0, TC_EINVAL,
               "pool and out_ids must be 16-byte aligned");
    if (nrow <= 0) return;
    Scratch sc(s);
    long long* off = sc.alloc<long long>(4 * P);
    ex_sum(sc, reinterpret_cast<const long long*>(sizes_dev), off, P, s);
    ex_sum(sc, reinterpret_cast<const long long*>(sizes_dev) + P, off + P, P, s);
    TC_CUDA(cudaMemsetAsync(off + 2 * P, 0, 2 * P * sizeof(long long), s));
    k_sh_send_emit<<<grid_for(nrow * 32, kBlk, sm_count() * 8), kBlk, 0, s>>>(
        indptr, indices, nrow, pool_indptr, reinterpret_cast<const int4*>(pool), bounds, P, rank, off, off + P,
        reinterpret_cast<unsigned long long*>(off + 2 * P), out_len, reinterpret_cast<int4*>(out_ids));
    check_launch();
  });
}

int tc_shard_index(const int32_t* row_len, int64_t nrow, const int32_t* pool, int64_t lo, int64_t hi,
                   const int64_t* tab_indptr, int64_t* pool_indptr, int64_t* rev_indptr, int32_t* rev_seg,
                   int64_t* rev_cost, int64_t* nseg_host, tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(lo >= 0 && lo <= hi, TC_EINVAL, "bad owner range");
    const int64_t nx = hi - lo;
    Scratch sc(s);
    // padded row offsets from the lengths
    int64_t* sz = sc.alloc<int64_t>(nrow + 1);
    k_sh_len_sizes<<<grid_for(nrow + 1, kBlk), kBlk, 0, s>>>(row_len, nrow, sz);
    check_launch();
    ex_sum(sc, sz, pool_indptr, nrow + 1, s);
    auto* acc = sc.alloc<unsigned long long>(nx + 1);
    TC_CUDA(cudaMemsetAsync(acc, 0, (nx + 1) * sizeof(unsigned long long), s));
    const int grid = grid_for(std::max<int64_t>(nrow, 1) * 32, kBlk, sm_count() * 16);
    if (nrow > 0) {
      k_sh_idx_count<<<grid, kBlk, 0, s>>>(pool_indptr, row_len, nrow, pool, lo, hi, acc);
      check_launch();
    }
    int64_t* cnt = sc.alloc<int64_t>(nx + 1);
    int64_t* cost = sc.alloc<int64_t>(nx + 1);
    k_sh_idx_rows<<<grid_for(nx + 1, kBlk), kBlk, 0, s>>>(acc, tab_indptr, nx, cnt, cost);
    check_launch();
    ex_sum(sc, cnt, rev_indptr, nx + 1, s);
    ex_sum(sc, cost, rev_cost, nx + 1, s);
    int32_t* cur = sc.alloc<int32_t>(nx + 1);
    TC_CUDA(cudaMemsetAsync(cur, 0, (nx + 1) * sizeof(int32_t), s));
    if (nrow > 0) {
      k_sh_idx_emit<<<grid, kBlk, 0, s>>>(pool_indptr, row_len, nrow, pool, lo, hi, rev_indptr, cur,
                                          reinterpret_cast<int2*>(rev_seg));
      check_launch();
    }
    if (nseg_host) *nseg_host = scalar_of(rev_indptr + nx, s);
  });
}

}  // extern "C"

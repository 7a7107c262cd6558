// build.cu -- device graph construction: normalize, degree ordering,
// orientation, forward / reverse / full CSR, node costs.
//
// Restates graph.py:76-153 and partitioning.py:79-92 of the reference with
// device radix sorts (CUB onesweep), atomic histograms and boundary-search
// CSR builds.  Every sort is stable, which is what makes the outputs
// bit-identical to numpy's stable lexsort / unique.
#include <cub/cub.cuh>
#include <cub/device/device_merge.cuh>
#include <thrust/iterator/transform_output_iterator.h>

#include <mutex>

#include "common.cuh"

namespace tcb {

static constexpr uint32_t kInf32 = 0xFFFFFFFFu;

int64_t g_host_chunk = 1 << 22;  // pairs (32 MB)
static constexpr int kBlock = 256;

// Pull-engine cost model (count.cu reads it through rev_cost): per
// predecessor segment its length plus kSegCost, per table build d^_u plus
// kTabCost; zero for u without successors (the engine skips them).
static constexpr int64_t kSegCost = 2;
static constexpr int64_t kTabCost = 16;

// ---------------------------------------------------------------- kernels

__global__ void k_minmax(const int32_t* __restrict__ a, int64_t cnt, int* mn, int* mx) {
  int lo = INT_MAX, hi = INT_MIN;
  GRID_STRIDE(i, cnt) {
    int x = a[i];
    lo = min(lo, x);
    hi = max(hi, x);
  }
  typedef cub::BlockReduce<int, kBlock> R;
  __shared__ typename R::TempStorage t1, t2;
  int blo = R(t1).Reduce(lo, cub::Min());
  int bhi = R(t2).Reduce(hi, cub::Max());
  if (threadIdx.x == 0) {
    atomicMin(mn, blo);
    atomicMax(mx, bhi);
  }
}


// Run aggregation for scattered atomics: lanes of a warp that hold equal
// keys in consecutive lanes form a run; the run's last lane gets its length
// and the lane index where it starts (other lanes get 0).  Sorted or
// grouped inputs (normalized edge lists, generator output) turn up to 32
// atomics into one; arbitrary inputs stay correct.
__device__ __forceinline__ int warp_run_end(int32_t key, bool valid, int lane, int* start) {
  const int32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
  const int32_t next = __shfl_down_sync(0xffffffffu, key, 1);
  const bool vprev = __shfl_up_sync(0xffffffffu, valid, 1);
  const bool vnext = __shfl_down_sync(0xffffffffu, valid, 1);
  const bool head = lane == 0 || !vprev || prev != key;
  const bool tail = lane == 31 || !vnext || next != key;
  const unsigned heads = __ballot_sync(0xffffffffu, valid && head);
  if (!valid || !tail) return 0;
  *start = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
  return lane - *start + 1;
}

// First position of every label in the raveled pair list, self-loops
// excluded (thread per pair; the two endpoint columns are aggregated
// separately).  Positions count the raw list, self-loops included: the
// relative order of the remaining pairs -- all the first-seen ranks depend
// on -- is the same as after graph.py:89 drops them.
// Chunked form (host-input pipeline): pairs [pos0, pos0 + npairs) of the
// list, labels >= cap (the speculative table size) set *over and are
// skipped; deg (nullable) also gets the chunk's degree histogram.
__global__ void k_first_pos(const int32_t* __restrict__ ids, int64_t npairs, uint32_t* fp, int64_t pos0 = 0,
                            int64_t cap = INT64_MAX, int* over = nullptr, int32_t* deg = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool ov = false;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < npairs; base += stride) {
    const int64_t i = base + threadIdx.x;
    const int2 p = i < npairs ? reinterpret_cast<const int2*>(ids)[i] : make_int2(-1, -1);
    const bool in = i < npairs && (int64_t)p.x < cap && (int64_t)p.y < cap;
    ov |= i < npairs && !in;
    const bool valid = in && p.x != p.y;
    const int64_t pos = 2 * (pos0 + i - lane);
    int st = 0, c;
    if ((c = warp_run_end(p.x, valid, lane, &st))) {
      atomicMin(&fp[p.x], (uint32_t)(pos + 2 * st));
      if (deg) atomicAdd(&deg[p.x], c);
    }
    if ((c = warp_run_end(p.y, valid, lane, &st))) {
      atomicMin(&fp[p.y], (uint32_t)(pos + 2 * st + 1));
      if (deg) atomicAdd(&deg[p.y], c);
    }
  }
  if (over && __any_sync(0xffffffffu, ov) && lane == 0) atomicOr(over, 1);
}

// K = number of present labels, Lf = largest present label.
__global__ void k_present(const uint32_t* __restrict__ fp, int64_t L1,
                          unsigned long long* count, int* maxid) {
  unsigned long long c = 0;
  int mx = -1;
  GRID_STRIDE(i, L1) {
    if (fp[i] != kInf32) {
      ++c;
      mx = max(mx, (int)i);
    }
  }
  typedef cub::BlockReduce<unsigned long long, kBlock> R1;
  typedef cub::BlockReduce<int, kBlock> R2;
  __shared__ typename R1::TempStorage t1;
  __shared__ typename R2::TempStorage t2;
  unsigned long long bc = R1(t1).Sum(c);
  int bm = R2(t2).Reduce(mx, cub::Max());
  if (threadIdx.x == 0) {
    atomicAdd(count, bc);
    atomicMax(maxid, bm);
  }
}

struct IsPresent {
  const uint32_t* fp;
  __host__ __device__ bool operator()(const int& i) const { return fp[i] != 0xFFFFFFFFu; }
};

__global__ void k_gather_u32(const int32_t* __restrict__ idx, const uint32_t* __restrict__ src,
                             int64_t cnt, uint32_t* out) {
  GRID_STRIDE(i, cnt) out[i] = src[idx[i]];
}

__global__ void k_rank_scatter(const int32_t* __restrict__ ids, int64_t cnt, int32_t* new_id) {
  GRID_STRIDE(i, cnt) new_id[ids[i]] = (int32_t)i;
}

// (min, max) of each pair packed as lo << b | hi; optional relabel map.  A
// self-loop packs as the sentinel (mask, mask), above every real pair
// (min < max), so it sorts last and is dropped after the unique pass.
__device__ __forceinline__ unsigned long long pair_key(const int32_t* __restrict__ e, int64_t i,
                                                     const int32_t* __restrict__ relabel, int b) {
  int32_t x = e[2 * i], y = e[2 * i + 1];
  if (x == y) return (2ull << (2 * b - 1)) - 1;
  if (relabel) {
    x = relabel[x];
    y = relabel[y];
  }
  return ((unsigned long long)(uint32_t)min(x, y) << b) | (uint32_t)max(x, y);
}

// Packs (min, max) keys and records how far the list is from sorted:
// flags bit 0 = some key decreases, bit 1 = some low half (max endpoint)
// decreases.  With bit 1 clear the low-half radix passes would be identity
// permutations, so the sort only needs the high half (e.g. generator output
// grouped by the newer endpoint); with bit 0 clear it needs nothing.
__global__ void k_pack_pairs(const int32_t* __restrict__ e, int64_t m,
                             const int32_t* __restrict__ relabel, int b,
                             unsigned long long* keys, unsigned* order_flags) {
  const unsigned long long mask = (1ull << b) - 1;
  unsigned f = 0;
  GRID_STRIDE(i, m) {
    const unsigned long long k = pair_key(e, i, relabel, b);
    keys[i] = k;
    if (order_flags && e[2 * i] == e[2 * i + 1]) f |= 4u;  // self-loop: one sentinel survives unique
    if (order_flags && i > 0) {
      const unsigned long long p = pair_key(e, i - 1, relabel, b);
      f |= (k < p ? 1u : 0u) | ((k & mask) < (p & mask) ? 2u : 0u);
    }
  }
  if (!order_flags) return;
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(order_flags, f);
}

// Publishes a chunk's order flags and the running largest label to mapped
// pinned host memory (two words over PCIe; no copy-engine round trip).
__global__ void k_publish_flags(const unsigned* __restrict__ flags, const int* __restrict__ mx,
                                volatile unsigned* host) {
  host[0] = *flags;
  host[1] = (unsigned)*mx;
  __threadfence_system();
}

// (lo << b | hi) key -> (lo, hi) pair, written by the unique pass itself.
struct UnpackKey {
  int b;
  __host__ __device__ int2 operator()(unsigned long long k) const {
    return make_int2((int32_t)(k >> b), (int32_t)(k & ((1ull << b) - 1)));
  }
};


// Degree histogram over the pair list (thread per pair, run-aggregated),
// fused with the endpoint range check: out-of-range ids set `bad` (bit 0
// negative, bit 1 >= n) and are not counted.
__global__ void k_histogram(const int32_t* __restrict__ ids, int64_t npairs, int64_t n, int32_t* h, int* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int flags = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < npairs; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < npairs;
    int2 p = valid ? reinterpret_cast<const int2*>(ids)[i] : make_int2(0, 0);
    const bool okx = p.x >= 0 && (int64_t)p.x < n, oky = p.y >= 0 && (int64_t)p.y < n;
    flags |= (p.x < 0 || p.y < 0 ? 1 : 0) | ((int64_t)p.x >= n || (int64_t)p.y >= n ? 2 : 0);
    int st = 0, c;
    if ((c = warp_run_end(p.x, valid && okx, lane, &st))) atomicAdd(&h[p.x], c);
    if ((c = warp_run_end(p.y, valid && oky, lane, &st))) atomicAdd(&h[p.y], c);
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (lane == 0 && flags) atomicOr(bad, flags);
}

__global__ void k_iota(int32_t* a, int64_t n) {
  GRID_STRIDE(i, n) a[i] = (int32_t)i;
}

__global__ void k_copy_i32(const int32_t* __restrict__ a, int32_t* b, int64_t n) {
  GRID_STRIDE(i, n) b[i] = a[i];
}


// Orientation (graph.py:113-125), counting-sort form.  Pass 1: every pair
// becomes (lo, hi) in canonical labels (kept for pass 2) and counts one
// predecessor of hi.  Row lo's size is then deg - predecessors (k_eff_counts):
// every pair gives one endpoint slot to its lo row and one to hi, so this
// holds with duplicates and self-loops too.  Counting hi rather than lo lets
// the atomics aggregate over runs: a normalized list is sorted by its
// smaller original label, which is usually the higher-degree endpoint, so
// consecutive pairs share hi (cfg 2: 50 M L2 atomics became a few M).
__global__ void k_orient_count(const int32_t* __restrict__ e, int64_t m, const int32_t* __restrict__ relabel,
                               int2* __restrict__ lohi, int32_t* hicnt) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < m;
    int2 k = make_int2(0, 0);
    if (valid) {
      const int2 p = reinterpret_cast<const int2*>(e)[i];
      const int32_t x = relabel[p.x], y = relabel[p.y];
      k = make_int2(min(x, y), max(x, y));
      lohi[i] = k;
    }
    int st = 0, c;
    if ((c = warp_run_end(k.y, valid, lane, &st))) atomicAdd(&hicnt[k.y], c);
  }
}

// Forward row sizes (int64, for the offsets scan): deg - predecessors.
__global__ void k_eff_counts(const int32_t* __restrict__ deg_orig, const int32_t* __restrict__ orig_ids,
                             const int32_t* __restrict__ hicnt, int64_t n, long long* cnt) {
  GRID_STRIDE(v, n + 1) cnt[v] = v < n ? (long long)(deg_orig[orig_ids[v]] - hicnt[v]) : 0;
}

// Pass 2: hi goes to a slot of row lo claimed with an atomic cursor.  The
// scatter runs in phases over row ranges [bounds[ph], bounds[ph+1]) whose
// slots span about the same number of entries, so each phase's writes land
// in an L2-resident window of the output instead of random DRAM sectors.
// cursor[v] starts at row v's first slot (k_cursor_init; m < 2^31), so a
// slot costs one atomic and no read of indptr.
__global__ void k_orient_scatter(const int2* __restrict__ lohi, int64_t m, const int64_t* __restrict__ bounds,
                                 int ph, int32_t* cursor, int32_t* out) {
  const int64_t r0 = bounds[ph], r1 = bounds[ph + 1];
  GRID_STRIDE(i, m) {
    const int2 k = lohi[i];
    if (k.x >= r0 && k.x < r1) out[atomicAdd(&cursor[k.x], 1)] = k.y;
  }
}

// front[v] = indptr[v]; back[v] (nullable) = indptr[v + 1] - 1: the slot
// cursors of the counting scatters as absolute positions.
__global__ void k_cursor_init(const int64_t* __restrict__ indptr, int64_t n, int32_t* front, int32_t* back) {
  GRID_STRIDE(v, n) {
    front[v] = (int32_t)indptr[v];
    if (back) back[v] = (int32_t)(indptr[v + 1] - 1);
  }
}

// Row boundaries of `nph` phases holding about equal shares of the
// indptr[n] entries (thread per boundary, binary search).
__global__ void k_phase_bounds(const int64_t* __restrict__ indptr, int64_t n, int nph, int64_t* bounds) {
  const int p = threadIdx.x;
  if (p > nph) return;
  if (p == 0 || p == nph) {
    bounds[p] = p == 0 ? 0 : n;
    return;
  }
  const int64_t target = (int64_t)((__int128)indptr[n] * p / nph);
  int64_t lo = 0, hi = n;  // first row whose start is >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (indptr[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  bounds[p] = lo;
}

// deg / eff_deg of the canonical nodes, and the in-degree (number of
// predecessors, = deg - eff_deg) that sizes the reverse CSR rows.
__global__ void k_degrees(const int64_t* __restrict__ indptr, const int32_t* __restrict__ deg_orig,
                          const int32_t* __restrict__ orig_ids, int64_t n, int32_t* deg,
                          int32_t* eff_deg, int64_t* in_deg) {
  GRID_STRIDE(v, n) {
    const int32_t ed = (int32_t)(indptr[v + 1] - indptr[v]);
    const int32_t d = deg_orig[orig_ids[v]];
    eff_deg[v] = ed;
    deg[v] = d;
    in_deg[v] = d - ed;
  }
}

// Reverse CSR by counting scatter: forward edge e = (v, u) goes to a slot
// of row u claimed with an atomic cursor -- non-empty suffixes from the
// front of the row, empty ones (u is the last id of N^_v) from the back, so
// the engine's segment groups are prefix-dense and need no compaction.
// Order within those two parts is unspecified (the pull engine only sums
// over a row); the full CSR sorts its rows when it is assembled.  A warp
// takes kRevSpan consecutive forward edges (coalesced reads whatever the
// row lengths); each lane walks from the chunk's first row to its own.
// Phased over destination rows like k_orient_scatter.
static constexpr int kRevSpan = 1024;
#ifndef TCB_REV_COST_STREAM
#define TCB_REV_COST_STREAM 1
#endif
__global__ void k_rev_scatter(const int64_t* __restrict__ eff_indptr, const int32_t* __restrict__ eff_indices,
                              int64_t n, int64_t m, const int64_t* __restrict__ rev_indptr,
                              const int64_t* __restrict__ bounds, int ph, int32_t* cursor, int32_t* back,
                              int2* rev_seg, const int64_t* __restrict__ pool_indptr, int32_t* pool) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t u0 = bounds[ph], u1 = bounds[ph + 1];
  for (int64_t e0 = warp * kRevSpan; e0 < m; e0 += nwarps * kRevSpan) {
    const int64_t e1 = min(m, e0 + kRevSpan);
    int64_t v = row_of_edge(eff_indptr, n, e0);
    int64_t vbeg = eff_indptr[v], vend = eff_indptr[v + 1];
    for (int64_t c = e0; c < e1; c += 32) {
      const int64_t e = min(c + lane, e1 - 1);
      int64_t w = v, wbeg = vbeg, wend = vend;
      while (wend <= e) {
        wbeg = wend;
        wend = eff_indptr[++w + 1];
      }
      v = __shfl_sync(0xffffffffu, w, 31);
      vbeg = __shfl_sync(0xffffffffu, wbeg, 31);
      vend = __shfl_sync(0xffffffffu, wend, 31);
      if (c + lane >= e1) continue;
      const int64_t u = eff_indices[e];
      const int64_t p0 = pool_indptr[w];  // row w of the padded pool
      if (ph == 0) {  // the padded pool: row w's ids, then INT32_MAX up to a multiple of 4
        pool[p0 + (e - wbeg)] = (int32_t)u;
        if (e + 1 == wend)
          for (int64_t q = p0 + (wend - wbeg); q < pool_indptr[w + 1]; ++q) pool[q] = INT32_MAX;
      }
      if (u < u0 || u >= u1) continue;
      // front / back cursors hold absolute slots (k_cursor_init)
      const int64_t slot = (e + 1 < wend) ? atomicAdd(&cursor[u], 1) : atomicSub(&back[u], 1);
#if TCB_DEBUG
      assert(slot >= rev_indptr[u] && slot < rev_indptr[u + 1]);
#endif
      // the suffix of N^_w after u, in pool coordinates
      rev_seg[slot] = make_int2((int)(p0 + (e + 1 - wbeg)), (int)(p0 + (wend - wbeg)));
    }
  }
}

// Padded pool row sizes (multiples of 4 ids: a 16-byte chunk never holds
// ids of two rows) and the INT32_MAX head before the pool.
__global__ void k_pool_sizes(const int64_t* __restrict__ eff_indptr, int64_t n, int64_t* sz) {
  GRID_STRIDE(v, n + 1) sz[v] = (v < n) ? ((eff_indptr[v + 1] - eff_indptr[v] + 3) & ~(int64_t)3) : 0;
}

__global__ void k_fill_i32(int32_t* p, int64_t k, int32_t val) {
  GRID_STRIDE(i, k) p[i] = val;
}

// Row sorts after the counting scatter.  CUB's segmented sort handles rows
// of at most kCubRowMax ids with sub-warp merge sorts (fast) and larger
// ones with one block-wide radix sort per row (slow when there are many,
// e.g. dense ER rows of 100-400: 68 ms at cfg 5).  Rows in (kCubRowMax,
// kBlockRowMax] are sorted here instead -- a warp per row up to 1 024 ids
// (merge sorts of 8 / 16 / 32 keys per lane), a block per row above (256 x 8
// or 512 x 16 keys) -- and
// are handed to CUB as empty segments.
static constexpr int kCubRowMax = 112;  // CUB's sm_100 (Policy860) medium tile: 16 threads x 7 keys
static constexpr int kBlockRowMax = 8192;

__global__ void k_row_classes(const int64_t* __restrict__ indptr, int64_t n, int64_t* seg_end, int32_t* rows,
                              int64_t cap, int* counts) {
  GRID_STRIDE(v, n) {
    const int64_t b = indptr[v], e = indptr[v + 1], L = e - b;
    const int cls = L <= kCubRowMax ? -1
                    : L <= 256 ? 0 : L <= 512 ? 1 : L <= 1024 ? 2 : L <= 2048 ? 3 : L <= kBlockRowMax ? 4 : -1;
    seg_end[v] = cls < 0 ? e : b;
    if (cls >= 0) rows[cls * cap + atomicAdd(&counts[cls], 1)] = (int32_t)v;
  }
}

struct LessI32 {
  __device__ bool operator()(const int32_t& a, const int32_t& b) const { return a < b; }
};

template <int kIpt>
__global__ void __launch_bounds__(256) k_sort_rows_warp(const int64_t* __restrict__ indptr,
                                                        const int32_t* __restrict__ in, int32_t* out,
                                                        const int32_t* __restrict__ rows, const int* count) {
  using WS = cub::WarpMergeSort<int32_t, kIpt, 32>;
  __shared__ typename WS::TempStorage tmp[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int cnt = *count;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < cnt; r += nwarps) {
    const int32_t v = rows[r];
    const int64_t b = indptr[v];
    const int L = (int)(indptr[v + 1] - b);
    int32_t k[kIpt];
#pragma unroll
    for (int i = 0; i < kIpt; ++i) {
      const int idx = i * 32 + lane;  // striped load (coalesced) ...
      k[i] = idx < L ? in[b + idx] : INT_MAX;
    }
    WS(tmp[wid]).Sort(k, LessI32());  // ... blocked result: lane holds ranks lane*kIpt + i
#pragma unroll
    for (int i = 0; i < kIpt; ++i) {
      const int idx = lane * kIpt + i;
      if (idx < L) out[b + idx] = k[i];
    }
    __syncwarp();
  }
}

template <int kThreads, int kIpt>
__global__ void __launch_bounds__(kThreads) k_sort_rows_block(const int64_t* __restrict__ indptr,
                                                              const int32_t* __restrict__ in, int32_t* out,
                                                              const int32_t* __restrict__ rows, const int* count) {
  using BS = cub::BlockMergeSort<int32_t, kThreads, kIpt>;
  __shared__ typename BS::TempStorage tmp;
  const int cnt = *count;
  for (int r = blockIdx.x; r < cnt; r += gridDim.x) {
    const int32_t v = rows[r];
    const int64_t b = indptr[v];
    const int L = (int)(indptr[v + 1] - b);
    int32_t k[kIpt];
#pragma unroll
    for (int i = 0; i < kIpt; ++i) {
      const int idx = i * kThreads + threadIdx.x;
      k[i] = idx < L ? in[b + idx] : INT_MAX;
    }
    BS(tmp).Sort(k, LessI32());
#pragma unroll
    for (int i = 0; i < kIpt; ++i) {
      const int idx = threadIdx.x * kIpt + i;
      if (idx < L) out[b + idx] = k[i];
    }
    __syncthreads();
  }
}

// Phase count for a scatter of `bytes` of output: enough phases that each
// window fits comfortably in L2 (64 MB), when at most 4 do (every phase
// re-reads the source); otherwise one.
#ifndef TCB_REV_WINDOW_MB
#define TCB_REV_WINDOW_MB 200
#endif
#ifndef TCB_SCATTER_WINDOW_MB
#define TCB_SCATTER_WINDOW_MB 64
#endif
inline int scatter_phases(int64_t bytes, int64_t window = (int64_t)TCB_SCATTER_WINDOW_MB << 20) {
  const int64_t p = (bytes + window - 1) / window;
  return p <= 4 ? (int)std::max<int64_t>(1, p) : 1;
}

// Warp per u: pull-engine cost of u (see kSegCost / kTabCost).
__global__ void k_rev_cost(const int64_t* __restrict__ rev_indptr, const int2* __restrict__ rev_seg,
                           const int64_t* __restrict__ eff_indptr, int64_t n, int64_t* cost) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = warp; u < n; u += nwarps) {
    int64_t d = eff_indptr[u + 1] - eff_indptr[u];
    int64_t r0 = rev_indptr[u], r1 = rev_indptr[u + 1];
    long long s = 0;
    if (d > 0)
      for (int64_t r = r0 + lane; r < r1; r += 32) {
        const int2 sg = rev_seg[r];
        s += (sg.y - sg.x) + kSegCost;
      }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) cost[u] = (d > 0 && r1 > r0) ? (int64_t)s + d + kTabCost : 0;
  }
}

// Streaming form of k_rev_cost: thread t sums the suffix lengths of
// kCostRun consecutive reverse entries (coalesced reads of the flat rev_seg
// array), finding the row of its first entry by binary search and walking
// row boundaries from there; each row's partial sum goes out with one
// fire-and-forget atomic.  k_rev_cost_fin adds the per-row terms.
static constexpr int kCostRun = 8;
__global__ void k_rev_len_sum(const int64_t* __restrict__ rev_indptr, const int2* __restrict__ rev_seg, int64_t n,
                              int64_t m, unsigned long long* acc) {
  const int64_t nt = (m + kCostRun - 1) / kCostRun;
  GRID_STRIDE(t, nt) {
    const int64_t r0 = t * kCostRun, r1 = min(m, r0 + kCostRun);
    int64_t u = row_of_edge(rev_indptr, n, r0);
    int64_t uend = rev_indptr[u + 1];
    unsigned long long s = 0;
    for (int64_t r = r0; r < r1; ++r) {
      int walked = 0;
      while (r >= uend) {  // row change: flush (rows may be empty)
        if (s) atomicAdd(&acc[u], s);
        s = 0;
        if (++walked > 4) {
          // a long run of empty rows (R-MAT: up to ~10^5 nodes without
          // predecessors between two that have one): search instead of
          // walking them one dependent load at a time (14 ms at cfg 4)
          u = row_of_edge(rev_indptr, n, r);
          uend = rev_indptr[u + 1];
        } else {
          uend = rev_indptr[++u + 1];
        }
      }
      const int2 sg = rev_seg[r];
      s += (unsigned long long)(sg.y - sg.x);
    }
    // Consecutive threads end in the same row when it is a hub's (millions of
    // entries at R-MAT scale 24: one atomic per thread serialised on a few
    // thousand addresses, 14 ms at cfg 4): the lanes of a warp that end in
    // one row add their sums with one reduction and one atomic.  A thread's
    // run is at most kCostRun suffixes, so a warp's sum fits 32 bits.
    const unsigned active = __activemask();
    const unsigned grp = __match_any_sync(active, (unsigned)u);
    const unsigned tot = __reduce_add_sync(grp, (unsigned)s);
    if (tot && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&acc[u], (unsigned long long)tot);
  }
}

__global__ void k_rev_cost_fin(const int64_t* __restrict__ rev_indptr, const int64_t* __restrict__ eff_indptr,
                               const unsigned long long* __restrict__ acc, int64_t n, int64_t* cost) {
  GRID_STRIDE(u, n) {
    const int64_t d = eff_indptr[u + 1] - eff_indptr[u], k = rev_indptr[u + 1] - rev_indptr[u];
    cost[u] = (d > 0 && k > 0) ? (int64_t)acc[u] + kSegCost * k + d + kTabCost : 0;
  }
}

// full CSR row u = predecessors (the row of each rev_seg's edge) then N^_u;
// rows are sorted afterwards.
__global__ void k_full(const int64_t* __restrict__ eff_indptr, const int32_t* __restrict__ eff_indices,
                       const int64_t* __restrict__ rev_indptr, const int2* __restrict__ rev_seg,
                       const int64_t* __restrict__ pool_indptr, int64_t n, int64_t* full_indptr,
                       int32_t* full_indices) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = warp; u <= n; u += nwarps) {
    int64_t base = rev_indptr[u] + eff_indptr[u];
    if (lane == 0) full_indptr[u] = base;
    if (u == n) continue;
    int64_t r0 = rev_indptr[u], r1 = rev_indptr[u + 1];
    for (int64_t r = r0 + lane; r < r1; r += 32)
      full_indices[base + (r - r0)] = (int32_t)row_of_edge(pool_indptr, n, (int64_t)rev_seg[r].x - 1);
    int64_t e0 = eff_indptr[u], e1 = eff_indptr[u + 1];
    int64_t off = base + (r1 - r0);
    for (int64_t e = e0 + lane; e < e1; e += 32) full_indices[off + (e - e0)] = eff_indices[e];
  }
}

// ---------------------------------------------------------------- sorting

template <class K>
K* sort_keys(Scratch& sc, K* a, K* b, int64_t n, int end_bit, cudaStream_t s, int begin_bit = 0) {
  if (n <= 1 || end_bit <= begin_bit) return a;
  cub::DoubleBuffer<K> db(a, b);
  size_t tmp = 0;
  TC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, n, begin_bit, end_bit, s));
  void* t = sc.bytes(tmp);
  TC_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, db, n, begin_bit, end_bit, s));
  return db.Current();
}

// Radix sort of packed (lo << b | hi) keys using the order flags of
// k_pack_pairs: skip the sort, or sort the high half only (stable LSD
// passes over an already non-decreasing low half change nothing).
template <class K>
K* sort_packed(Scratch& sc, K* a, K* bb, int64_t n, int b, const unsigned* order_flags, cudaStream_t s,
               unsigned* flags_out = nullptr) {
  unsigned f = 0;
  TC_CUDA(cudaMemcpyAsync(&f, order_flags, sizeof(f), cudaMemcpyDeviceToHost, s));
  sync_stream(s);
  if (flags_out) *flags_out = f;
  if (!(f & 1u)) return a;
  return sort_keys(sc, a, bb, n, 2 * b, s, (f & 2u) ? 0 : b);
}

template <class K, class V>
void sort_pairs(Scratch& sc, K*& ka, K* kb, V*& va, V* vb, int64_t n, int end_bit,
                cudaStream_t s) {
  if (n <= 1 || end_bit <= 0) return;
  cub::DoubleBuffer<K> dk(ka, kb);
  cub::DoubleBuffer<V> dv(va, vb);
  size_t tmp = 0;
  TC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, n, 0, end_bit, s));
  void* t = sc.bytes(tmp);
  TC_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, n, 0, end_bit, s));
  ka = dk.Current();
  va = dv.Current();
}


template <class T>
T read_scalar(const T* d, cudaStream_t s) {
  T h;
  TC_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  sync_stream(s);
  return h;
}

// ---------------------------------------------------------------- normalize

void present_labels(Scratch& sc, const uint32_t* fp, int64_t L1, int64_t* K, int64_t* Lf, cudaStream_t s);
void normalize_tail(Scratch& sc, const int32_t* edges, int64_t m_raw, uint32_t* fp, int64_t L1, int64_t K,
                    int64_t Lf, int32_t* out_edges, int64_t* m_host, int64_t* n_host, cudaStream_t s,
                    const unsigned long long* sorted32 = nullptr, bool sentinel = false);

void normalize(const int32_t* edges, int64_t m_raw, int32_t* out_edges, int64_t* m_host,
               int64_t* n_host, cudaStream_t s) {
  *m_host = 0;
  *n_host = 0;
  TC_REQUIRE(m_raw >= 0, TC_EINVAL, "negative edge count");
  TC_REQUIRE(m_raw < (1ll << 30), TC_EINVAL, "edge list too long for int32 positions (m_raw >= 2^30)");
  if (m_raw == 0) return;
  TC_REQUIRE(((uintptr_t)edges & 7) == 0, TC_EINVAL, "edges must be 8-byte aligned");
  Scratch sc(s);
  int sms = sm_count();
  int* mm = sc.alloc<int>(2);
  int init[2] = {INT_MAX, INT_MIN};
  TC_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
  k_minmax<<<grid_for(2 * m_raw, kBlock, sms * 8), kBlock, 0, s>>>(edges, 2 * m_raw, mm, mm + 1);
  check_launch();
  int hmm[2];
  TC_CUDA(cudaMemcpyAsync(hmm, mm, sizeof(hmm), cudaMemcpyDeviceToHost, s));
  sync_stream(s);
  TC_REQUIRE(hmm[0] >= 0, TC_EINVAL, "negative node id in edge list");  // graph.py:87-88

  // first occurrence of each label in the raveled order, self-loops
  // excluded (graph.py:89-93)
  const int64_t L1 = (int64_t)hmm[1] + 1;
  uint32_t* fp = sc.alloc<uint32_t>(L1);
  TC_CUDA(cudaMemsetAsync(fp, 0xFF, L1 * sizeof(uint32_t), s));
  k_first_pos<<<grid_for(m_raw, kBlock, sms * 16), kBlock, 0, s>>>(edges, m_raw, fp);
  check_launch();
  int64_t K = 0, Lf = 0;
  present_labels(sc, fp, L1, &K, &Lf, s);
  normalize_tail(sc, edges, m_raw, fp, L1, K, Lf, out_edges, m_host, n_host, s);
}

// K = labels present outside self-loops, Lf = the largest (graph.py:92-94).
void present_labels(Scratch& sc, const uint32_t* fp, int64_t L1, int64_t* K, int64_t* Lf, cudaStream_t s) {
  const int sms = sm_count();
  auto* cnt = sc.alloc<unsigned long long>(1);
  int* lf = sc.alloc<int>(1);
  TC_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
  int minus1 = -1;
  TC_CUDA(cudaMemcpyAsync(lf, &minus1, sizeof(int), cudaMemcpyHostToDevice, s));
  k_present<<<grid_for(L1, kBlock, sms * 8), kBlock, 0, s>>>(fp, L1, cnt, lf);
  check_launch();
  unsigned long long hk[2] = {0, 0};  // one transfer for K and Lf
  TC_CUDA(cudaMemcpyAsync(&hk[0], cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaMemcpyAsync(&hk[1], lf, sizeof(int), cudaMemcpyDeviceToHost, s));
  sync_stream(s);
  *K = (int64_t)hk[0];
  *Lf = (int64_t)(int32_t)(uint32_t)hk[1];
}

// Census of a sorted pair list (8-byte pairs read as one word): [0] pairs
// equal to their successor, self-loop sentinels (-1, -1) excluded; [1]
// sentinels.
__global__ void k_dup_census(const long long* __restrict__ e, int64_t m, unsigned long long* cnt) {
  constexpr int U = 4;  // independent loads in flight per thread
  unsigned long long d = 0, z = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < m; i0 += U * stride) {
    long long a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      a[u] = i < m ? __ldg(&e[i]) : 0;
      b[u] = i + 1 < m ? __ldg(&e[i + 1]) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < m) {
        if (a[u] == -1ll) ++z;
        else if (i + 1 < m && b[u] == a[u]) ++d;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, o);
    z += __shfl_xor_sync(0xffffffffu, z, o);
  }
  if ((threadIdx.x & 31) == 0 && (d | z)) {
    atomicAdd(&cnt[0], d);
    atomicAdd(&cnt[1], z);
  }
}

// normalize from the label census on: the first-seen map, packing, sort
// and unique (graph.py:95-103).  sorted32 (nullable): the list's keys
// (min << 32 | max, raw labels; a self-loop as ~0, flagged by `sentinel`)
// already sorted -- used when the labels are dense, so only the unique
// pass remains.
void normalize_tail(Scratch& sc, const int32_t* edges, int64_t m_raw, uint32_t* fp, int64_t L1, int64_t K,
                    int64_t Lf, int32_t* out_edges, int64_t* m_host, int64_t* n_host, cudaStream_t s,
                    const unsigned long long* sorted32, bool sentinel) {
  const int sms = sm_count();
  if (K == 0) return;  // only self-loops (graph.py:90-91)
  auto* nsel = sc.alloc<long long>(1);
  const int32_t* relabel = nullptr;
  if (sorted32 && K == Lf + 1) {  // dense labels kept: unique (writing pairs) of the presorted keys
    auto out = thrust::make_transform_output_iterator(reinterpret_cast<int2*>(out_edges), UnpackKey{32});
    size_t tmp = 0;
    TC_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, sorted32, out, nsel, m_raw, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceSelect::Unique(t, tmp, sorted32, out, nsel, m_raw, s));
    const int64_t m2 = read_scalar(nsel, s) - (sentinel ? 1 : 0);  // the self-loop key sorts last
    *m_host = m2;
    *n_host = K;
    return;
  }

  if (K != Lf + 1) {
    // first-seen compaction (graph.py:96-98): new id = rank of first position
    int32_t* pid = sc.alloc<int32_t>(K);
    int32_t* pid2 = sc.alloc<int32_t>(K);
    {
      size_t tmp = 0;
      cub::CountingInputIterator<int> it(0);
      IsPresent pred{fp};
      TC_CUDA(cub::DeviceSelect::If(nullptr, tmp, it, pid, nsel, L1, pred, s));
      void* t = sc.bytes(tmp);
      TC_CUDA(cub::DeviceSelect::If(t, tmp, it, pid, nsel, L1, pred, s));
    }
    uint32_t* fk = sc.alloc<uint32_t>(K);
    uint32_t* fk2 = sc.alloc<uint32_t>(K);
    k_gather_u32<<<grid_for(K, kBlock), kBlock, 0, s>>>(pid, fp, K, fk);
    check_launch();
    sort_pairs(sc, fk, fk2, pid, pid2, K, bits_for((uint64_t)(2 * m_raw)), s);
    int32_t* new_id = reinterpret_cast<int32_t*>(fp);  // fp no longer needed
    k_rank_scatter<<<grid_for(K, kBlock), kBlock, 0, s>>>(pid, K, new_id);
    check_launch();
    relabel = new_id;
  }

  // (lo, hi) + unique rows (graph.py:99-102)
  int b = std::max(1, bits_for((uint64_t)(K - 1)));
  auto* ka = sc.alloc<unsigned long long>(m_raw);
  auto* kb = sc.alloc<unsigned long long>(m_raw);
  unsigned* oflags = sc.alloc<unsigned>(1);
  TC_CUDA(cudaMemsetAsync(oflags, 0, sizeof(unsigned), s));
  k_pack_pairs<<<grid_for(m_raw, kBlock, sms * 16), kBlock, 0, s>>>(edges, m_raw, relabel, b, ka, oflags);
  check_launch();
  unsigned hflags = 0;
  unsigned long long* sorted = sort_packed(sc, ka, kb, m_raw, b, oflags, s, &hflags);
  {
    auto out = thrust::make_transform_output_iterator(reinterpret_cast<int2*>(out_edges), UnpackKey{b});
    size_t tmp = 0;
    TC_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, sorted, out, nsel, m_raw, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceSelect::Unique(t, tmp, sorted, out, nsel, m_raw, s));
  }
  int64_t m2 = read_scalar(nsel, s);
  if (hflags & 4u) --m2;  // drop the self-loop sentinel (sorted last, once after unique)
  *m_host = m2;
  *n_host = K;  // graph.py:103
}


// Host-input normalize: the raw list is copied from (pinned) host memory in
// chunks on a copy stream, and each chunk's min/max, first occurrences and
// degree histogram run on the compute stream as soon as it has landed, so
// those passes hide under the PCIe transfer.  The first-occurrence and
// degree tables are sized speculatively for labels < 2 m_raw + 1 (every
// dense labelling fits: n <= 2m); a larger label sends the call down the
// device path once the copy is done.  deg (nullable, int32[2 m_raw + 1]) is
// the degree of every label; *deg_valid says whether it is the normalized
// graph's degree array (dense labels kept, nothing dropped), which
// build_graph can then take instead of its own histogram.
struct KeyLess {
  __device__ bool operator()(unsigned long long a, unsigned long long b) const { return a < b; }
};

static cudaStream_t copy_stream() {
  static cudaStream_t cs[64] = {};
  int dev = 0;
  TC_CUDA(cudaGetDevice(&dev));
  if (!cs[dev]) TC_CUDA(cudaStreamCreateWithFlags(&cs[dev], cudaStreamNonBlocking));
  return cs[dev];
}

void normalize_host(const int32_t* host, int64_t m_raw, int32_t* dev, int32_t* out_edges, int64_t* m_host,
                    int64_t* n_host, int32_t* deg, int32_t* deg_valid, cudaStream_t s) {
  *m_host = 0;
  *n_host = 0;
  if (deg_valid) *deg_valid = 0;
  TC_REQUIRE(m_raw >= 0, TC_EINVAL, "negative edge count");
  TC_REQUIRE(m_raw < (1ll << 30), TC_EINVAL, "edge list too long for int32 positions (m_raw >= 2^30)");
  if (m_raw == 0) return;
  TC_REQUIRE(((uintptr_t)dev & 7) == 0, TC_EINVAL, "edges must be 8-byte aligned");
  Scratch sc(s);
  const int sms = sm_count();
  cudaStream_t cs = copy_stream();
  constexpr int kMaxChunks = 16;
  static cudaEvent_t ev[64][kMaxChunks + 1] = {};
  int d = 0;
  TC_CUDA(cudaGetDevice(&d));
  // The copy stream, the chunk events and the mapped flag slots below are
  // per device and shared by every call: one call per device at a time (the
  // host waits on every chunk's flags before returning, so nothing of a
  // call's flag traffic outlives it).
  static std::mutex call_mu[64];
  std::lock_guard<std::mutex> call_lock(call_mu[d]);
  if (!ev[d][0])
    for (auto& e : ev[d]) TC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // the copy waits only for the caller's prior work on s (dev is the
  // caller's), not for the table initialisation below
  TC_CUDA(cudaEventRecord(ev[d][kMaxChunks], s));
  TC_CUDA(cudaStreamWaitEvent(cs, ev[d][kMaxChunks], 0));
  const int64_t cap = std::min<int64_t>(2 * m_raw + 1, INT32_MAX);
  uint32_t* fp = sc.alloc<uint32_t>(cap);
  int* mm = sc.alloc<int>(3);  // min, max, label >= cap seen
  static const int init[3] = {INT_MAX, INT_MIN, 0};
  TC_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
  TC_CUDA(cudaMemsetAsync(fp, 0xFF, cap * sizeof(uint32_t), s));
  if (deg) TC_CUDA(cudaMemsetAsync(deg, 0, cap * sizeof(int32_t), s));
  const int nch = (int)std::max<int64_t>(1, std::min<int64_t>(kMaxChunks, m_raw / g_host_chunk));
  const int64_t per = (m_raw + nch - 1) / nch;
  for (int c = 0; c < nch; ++c) {
    const int64_t o = c * per, mc = std::min(per, m_raw - o);
    if (mc <= 0) break;
    TC_CUDA(cudaMemcpyAsync(dev + 2 * o, host + 2 * o, mc * 2 * sizeof(int32_t), cudaMemcpyHostToDevice, cs));
    TC_CUDA(cudaEventRecord(ev[d][c], cs));
  }
  // Behind the copy, each chunk's keys (min << 32 | max, raw labels) are
  // packed and sorted -- by the smaller endpoint only (stable) when the
  // chunk is already ordered by its larger one, as a generator emitting
  // edges per new node is -- so the chunks become sorted runs that a merge
  // tree joins, mostly while the copy is still running, instead of a full
  // radix sort after it.
  unsigned long long* ka = sc.alloc<unsigned long long>(m_raw);
  unsigned long long* kb = sc.alloc<unsigned long long>(m_raw);
  unsigned long long* kc = sc.alloc<unsigned long long>(m_raw);
  unsigned* cflags = sc.alloc<unsigned>(kMaxChunks);
  TC_CUDA(cudaMemsetAsync(cflags, 0, kMaxChunks * sizeof(unsigned), s));
  size_t sort_tmp = 0;
  TC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, sort_tmp, ka, kb, per, 0, 64, s));
  void* sort_ws = sc.bytes(sort_tmp);
  bool runs = true, any_loop = false;
  // Sorted runs as a binary counter: a run of level l holds 2^l chunks; two
  // runs of equal level merge while later chunks are still being copied.
  // A merge writes a third buffer (its region is free in every buffer but
  // the two it reads), so runs may live in any of ka / kb / kc.
  struct Run {
    int64_t o, len;
    unsigned long long* buf;
    int level;
  };
  std::vector<Run> stack;
  size_t mcap = 0;
  void* mws = nullptr;
  auto merge_top = [&]() {
    const Run r2 = stack.back();
    stack.pop_back();
    const Run r1 = stack.back();
    stack.pop_back();
    unsigned long long* z = (r1.buf != ka && r2.buf != ka) ? ka : (r1.buf != kb && r2.buf != kb) ? kb : kc;
    size_t need = 0;
    TC_CUDA(cub::DeviceMerge::MergeKeys(nullptr, need, r1.buf + r1.o, (int)r1.len, r2.buf + r2.o, (int)r2.len,
                                        z + r1.o, KeyLess(), s));
    if (need > mcap) {
      mws = sc.bytes(need);
      mcap = need;
    }
    TC_CUDA(cub::DeviceMerge::MergeKeys(mws, need, r1.buf + r1.o, (int)r1.len, r2.buf + r2.o, (int)r2.len, z + r1.o,
                                        KeyLess(), s));
    stack.push_back(Run{r1.o, r1.len + r2.len, z, std::max(r1.level, r2.level) + 1});
  };
  // Chunk c's flags (sortedness, largest label so far) travel to pinned host
  // memory behind its pack kernel and the host waits on one event for both
  // (one short round trip per chunk; the copy stream runs on meanwhile).  The
  // sort must follow chunk c's passes before the stream waits for chunk c+1's
  // copy, or it would queue behind that copy.
  static unsigned* hflags[64] = {};
  static unsigned* dflags[64] = {};  // device view of the mapped hflags
  static cudaEvent_t fev[64][kMaxChunks] = {};
  if (!hflags[d]) {
    TC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hflags[d]), 2 * kMaxChunks * sizeof(unsigned),
                          cudaHostAllocMapped));
    TC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dflags[d]), hflags[d], 0));
    for (auto& e : fev[d]) TC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  auto sort_chunk = [&](int c) {
    const int64_t o = c * per, mc = std::min(per, m_raw - o);
    TC_CUDA(cudaEventSynchronize(fev[d][c]));
    const unsigned f = hflags[d][2 * c], hmax = hflags[d][2 * c + 1];
    if ((int)hmax < 0) {  // a negative label: no runs (the device path reports it)
      runs = false;
      return;
    }
    any_loop |= (f & 4u) != 0;  // a self-loop packs as ~0: sorts last, one survives unique
    const int hi_bits = 32 + std::max(1, bits_for((uint64_t)hmax));
    size_t tb = sort_tmp;
    if (!(f & 1u))  // already sorted
      TC_CUDA(cudaMemcpyAsync(kb + o, ka + o, mc * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
    else if (!(f & 2u))  // larger endpoints non-decreasing: a stable sort by the smaller one suffices
      TC_CUDA(cub::DeviceRadixSort::SortKeys(sort_ws, tb, ka + o, kb + o, mc, 32, hi_bits, s));
    else  // (e.g. a generator's seed clique) the whole key
      TC_CUDA(cub::DeviceRadixSort::SortKeys(sort_ws, tb, ka + o, kb + o, mc, 0, hi_bits, s));
    stack.push_back(Run{o, mc, kb, 0});
    while (stack.size() >= 2 && stack[stack.size() - 1].level == stack[stack.size() - 2].level) merge_top();
  };
  for (int c = 0; c < nch; ++c) {
    const int64_t o = c * per, mc = std::min(per, m_raw - o);
    if (mc <= 0) break;
    TC_CUDA(cudaStreamWaitEvent(s, ev[d][c], 0));
    k_minmax<<<grid_for(2 * mc, kBlock, sms * 8), kBlock, 0, s>>>(dev + 2 * o, 2 * mc, mm, mm + 1);
    check_launch();
    k_first_pos<<<grid_for(mc, kBlock, sms * 16), kBlock, 0, s>>>(dev + 2 * o, mc, fp, o, cap, mm + 2, deg);
    check_launch();
    if (runs) {
      k_pack_pairs<<<grid_for(mc, kBlock, sms * 16), kBlock, 0, s>>>(dev + 2 * o, mc, nullptr, 32, ka + o,
                                                                       cflags + c);
      check_launch();
      k_publish_flags<<<1, 1, 0, s>>>(cflags + c, mm + 1, dflags[d] + 2 * c);
      check_launch();
      TC_CUDA(cudaEventRecord(fev[d][c], s));
      sort_chunk(c);
    }
  }
  int hmm[3];
  TC_CUDA(cudaMemcpyAsync(hmm, mm, sizeof(hmm), cudaMemcpyDeviceToHost, s));
  sync_stream(s);
  TC_REQUIRE(hmm[0] >= 0, TC_EINVAL, "negative node id in edge list");  // graph.py:87-88
  if (hmm[2]) {  // a label beyond the speculative tables: the device path on the copied list
    normalize(dev, m_raw, out_edges, m_host, n_host, s);
    return;
  }
  const int64_t L1 = (int64_t)hmm[1] + 1;
  int64_t K = 0, Lf = 0;
  present_labels(sc, fp, L1, &K, &Lf, s);
  const unsigned long long* sorted32 = nullptr;
  if (runs && K == Lf + 1) {  // join the remaining runs, smallest first
    while (stack.size() > 2) merge_top();
    if (stack.size() == 2) {
      // Last level straight into the output pairs; when the census finds no
      // duplicate edge (self-loop sentinels sort last and are cut off) this
      // is the unique list and the select pass is skipped.  Otherwise the
      // level is merged again into keys for the unique pass.
      const Run r1 = stack[0], r2 = stack[1];
      auto out = thrust::make_transform_output_iterator(reinterpret_cast<int2*>(out_edges), UnpackKey{32});
      size_t need = 0;
      TC_CUDA(cub::DeviceMerge::MergeKeys(nullptr, need, r1.buf + r1.o, (int)r1.len, r2.buf + r2.o, (int)r2.len,
                                          out, KeyLess(), s));
      if (need > mcap) {
        mws = sc.bytes(need);
        mcap = need;
      }
      TC_CUDA(cub::DeviceMerge::MergeKeys(mws, need, r1.buf + r1.o, (int)r1.len, r2.buf + r2.o, (int)r2.len, out,
                                          KeyLess(), s));
      auto* cnt = sc.alloc<unsigned long long>(2);
      TC_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), s));
      k_dup_census<<<grid_for(m_raw, kBlock, sms * 16), kBlock, 0, s>>>(reinterpret_cast<const long long*>(out_edges),
                                                                        m_raw, cnt);
      check_launch();
      unsigned long long hc[2];
      TC_CUDA(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
      sync_stream(s);
      if (hc[0] == 0) {
        *m_host = m_raw - (int64_t)hc[1];
        *n_host = K;
        if (deg_valid) *deg_valid = (*m_host == m_raw && *n_host == L1) ? 1 : 0;
        return;
      }
      merge_top();
    }
    sorted32 = stack[0].buf;
  }
  normalize_tail(sc, dev, m_raw, fp, L1, K, Lf, out_edges, m_host, n_host, s, sorted32, any_loop);
  if (deg_valid) *deg_valid = (*m_host == m_raw && *n_host == L1) ? 1 : 0;
}

// Sorts every CSR row (ascending ids) from `unsorted` into `out`, by row
// length class: CUB's segmented sort for the shortest rows, warp / block
// sorting networks for the rest (k_row_classes empties the segments the
// class kernels own).  Shared by tc_build_graph and the sharded build
// (tc_shard_csr).
void sort_rows(Scratch& sc, const int64_t* indptr, int64_t n, int64_t m, const int32_t* unsorted, int32_t* out,
               cudaStream_t s) {
  if (n <= 0 || m <= 0) return;
  const int sms = sm_count();
  int64_t* seg_end = sc.alloc<int64_t>(n);
  int32_t* rows = sc.alloc<int32_t>(5 * n);
  int* counts = sc.alloc<int>(5);
  TC_CUDA(cudaMemsetAsync(counts, 0, 5 * sizeof(int), s));
  k_row_classes<<<grid_for(n, kBlock), kBlock, 0, s>>>(indptr, n, seg_end, rows, n, counts);
  check_launch();
  size_t tmp2 = 0;
  TC_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp2, unsorted, out, (int)m, (int)n, indptr, seg_end, s));
  void* t2 = sc.bytes(tmp2);
  TC_CUDA(cub::DeviceSegmentedSort::SortKeys(t2, tmp2, unsorted, out, (int)m, (int)n, indptr, seg_end, s));
  k_sort_rows_warp<8><<<sms * 8, 256, 0, s>>>(indptr, unsorted, out, rows, counts);
  check_launch();
  k_sort_rows_warp<16><<<sms * 8, 256, 0, s>>>(indptr, unsorted, out, rows + n, counts + 1);
  check_launch();
  k_sort_rows_warp<32><<<sms * 4, 256, 0, s>>>(indptr, unsorted, out, rows + 2 * n, counts + 2);
  check_launch();
  k_sort_rows_block<256, 8><<<sms * 4, 256, 0, s>>>(indptr, unsorted, out, rows + 3 * n, counts + 3);
  check_launch();
  k_sort_rows_block<512, kBlockRowMax / 512><<<sms * 2, 512, 0, s>>>(indptr, unsorted, out, rows + 4 * n, counts + 4);
  check_launch();
}

// ---------------------------------------------------------------- build

void build_graph(const int32_t* edges, int64_t m, int64_t n, const int32_t* order,
                 int64_t* eff_indptr, int32_t* eff_indices, int32_t* relabel, int32_t* orig_ids,
                 int32_t* deg, int32_t* eff_deg, int64_t* rev_indptr, int32_t* rev_seg,
                 int64_t* rev_cost, int64_t* pool_indptr, int32_t* pool, cudaStream_t s,
                 const int32_t* deg_hint = nullptr) {
  TC_REQUIRE(n >= 0 && m >= 0, TC_EINVAL, "negative size");
  TC_REQUIRE(n < (1ll << 31) - 1, TC_EINVAL, "n must fit int32 ids");
  TC_REQUIRE(m < (1ll << 31) - 1, TC_EINVAL, "m must be < 2^31");
  Scratch sc(s);
  int sms = sm_count();
  // degrees (graph.py:149-151), with the endpoint range check -- or the
  // degrees normalize_host computed while the list was arriving (its
  // output is in range by construction)
  const int32_t* deg_orig = deg_hint;
  if (!deg_hint) {
    int32_t* h = sc.alloc<int32_t>(n);
    if (n) TC_CUDA(cudaMemsetAsync(h, 0, n * sizeof(int32_t), s));
    if (m > 0) {
      TC_REQUIRE(((uintptr_t)edges & 7) == 0, TC_EINVAL, "edges must be 8-byte aligned");
      int* bad = sc.alloc<int>(1);
      TC_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
      k_histogram<<<grid_for(m, kBlock, sms * 16), kBlock, 0, s>>>(edges, m, n, h, bad);
      check_launch();
      int hb = read_scalar(bad, s);
      TC_REQUIRE(!(hb & 1), TC_EINVAL, "negative node id in edge list");
      TC_REQUIRE(!(hb & 2), TC_EINDEX, "edge endpoint >= n");
    }
    deg_orig = h;
  }
  // the pool's INT32_MAX head (TC_POOL_HEAD ids before pool[0])
  k_fill_i32<<<1, 256, 0, s>>>(pool - TC_POOL_HEAD, TC_POOL_HEAD, INT32_MAX);
  check_launch();
  if (n == 0) {
    TC_CUDA(cudaMemsetAsync(eff_indptr, 0, sizeof(int64_t), s));
    TC_CUDA(cudaMemsetAsync(rev_indptr, 0, sizeof(int64_t), s));
    TC_CUDA(cudaMemsetAsync(rev_cost, 0, sizeof(int64_t), s));
    TC_CUDA(cudaMemsetAsync(pool_indptr, 0, sizeof(int64_t), s));
    return;
  }
  // canonical order: ascending (degree, id) via a stable radix sort (graph.py:152)
  if (order) {
    k_copy_i32<<<grid_for(n, kBlock), kBlock, 0, s>>>(order, orig_ids, n);
    check_launch();
  } else {
    uint32_t* dk = sc.alloc<uint32_t>(n);
    uint32_t* dk2 = sc.alloc<uint32_t>(n);
    int32_t* ov = sc.alloc<int32_t>(n);
    int32_t* ov2 = sc.alloc<int32_t>(n);
    TC_CUDA(cudaMemcpyAsync(dk, deg_orig, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    k_iota<<<grid_for(n, kBlock), kBlock, 0, s>>>(ov, n);
    check_launch();
    sort_pairs(sc, dk, dk2, ov, ov2, n, std::max(1, bits_for((uint64_t)(2 * m))), s);
    TC_CUDA(cudaMemcpyAsync(orig_ids, ov, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  }
  k_rank_scatter<<<grid_for(n, kBlock), kBlock, 0, s>>>(orig_ids, n, relabel);  // graph.py:111-112
  check_launch();

  // orientation + forward CSR (graph.py:113-124): row sizes, offsets,
  // phased counting scatter, then every row sorted (segmented sort)
  int64_t* bounds = sc.alloc<int64_t>(8);
  {
    long long* cnt = sc.alloc<long long>(n + 1);
    int32_t* hicnt = sc.alloc<int32_t>(n);
    TC_CUDA(cudaMemsetAsync(hicnt, 0, n * sizeof(int32_t), s));
    int2* lohi = sc.alloc<int2>(m);
    if (m) {
      k_orient_count<<<grid_for(m, kBlock, sms * 16), kBlock, 0, s>>>(edges, m, relabel, lohi, hicnt);
      check_launch();
    }
    k_eff_counts<<<grid_for(n + 1, kBlock), kBlock, 0, s>>>(deg_orig, orig_ids, hicnt, n, cnt);
    check_launch();
    size_t tmp = 0;
    auto* cin = cnt;
    auto* cout = reinterpret_cast<long long*>(eff_indptr);
    TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cin, cout, n + 1, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, cin, cout, n + 1, s));
    if (m) {
      int32_t* unsorted = sc.alloc<int32_t>(m);
      TC_REQUIRE(m < (1ll << 31), TC_EINVAL, "m must be < 2^31");
      int32_t* cursor = sc.alloc<int32_t>(n);
      k_cursor_init<<<grid_for(n, kBlock), kBlock, 0, s>>>(eff_indptr, n, cursor, nullptr);
      check_launch();
      const int nph = scatter_phases(m * 4);
      k_phase_bounds<<<1, 32, 0, s>>>(eff_indptr, n, nph, bounds);
      check_launch();
      for (int ph = 0; ph < nph; ++ph) {
        k_orient_scatter<<<grid_for(m, kBlock, sms * 16), kBlock, 0, s>>>(lohi, m, bounds, ph, cursor, unsorted);
        check_launch();
      }
      sort_rows(sc, eff_indptr, n, m, unsorted, eff_indices, s);
    }
  }
  int64_t* in_deg = sc.alloc<int64_t>(n + 1);
  TC_CUDA(cudaMemsetAsync(in_deg + n, 0, sizeof(int64_t), s));
  k_degrees<<<grid_for(n, kBlock), kBlock, 0, s>>>(eff_indptr, deg_orig, orig_ids, n, deg, eff_deg, in_deg);
  check_launch();

  // reverse CSR: predecessors of u, each with the suffix of N^_v after u
  {
    size_t tmp = 0;
    TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in_deg, rev_indptr, n + 1, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in_deg, rev_indptr, n + 1, s));
  }
  // padded pool row offsets (rows filled by the reverse scatter's first phase)
  {
    int64_t* psz = sc.alloc<int64_t>(n + 1);
    k_pool_sizes<<<grid_for(n + 1, kBlock), kBlock, 0, s>>>(eff_indptr, n, psz);
    check_launch();
    size_t tmp = 0;
    TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, psz, pool_indptr, n + 1, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, psz, pool_indptr, n + 1, s));
  }
  if (m) {
    int32_t* cursor = sc.alloc<int32_t>(2 * n);
    k_cursor_init<<<grid_for(n, kBlock), kBlock, 0, s>>>(rev_indptr, n, cursor, cursor + n);
    check_launch();
    const int nph = scatter_phases(m * 8, (int64_t)TCB_REV_WINDOW_MB << 20);
    k_phase_bounds<<<1, 32, 0, s>>>(rev_indptr, n, nph, bounds);
    check_launch();
    for (int ph = 0; ph < nph; ++ph) {
      k_rev_scatter<<<grid_for((m + kRevSpan - 1) / kRevSpan * 32, kBlock, sms * 16), kBlock, 0, s>>>(
          eff_indptr, eff_indices, n, m, rev_indptr, bounds, ph, cursor, cursor + n, reinterpret_cast<int2*>(rev_seg),
          pool_indptr, pool);
      check_launch();
    }
  }
  // pull-engine cost prefix over u
  int64_t* cu = sc.alloc<int64_t>(n + 1);
#if TCB_REV_COST_STREAM
  {
    auto* acc = sc.alloc<unsigned long long>(n);
    TC_CUDA(cudaMemsetAsync(acc, 0, n * sizeof(unsigned long long), s));
    if (m) {
      k_rev_len_sum<<<grid_for((m + kCostRun - 1) / kCostRun, kBlock, sms * 16), kBlock, 0, s>>>(
          rev_indptr, reinterpret_cast<const int2*>(rev_seg), n, m, acc);
      check_launch();
    }
    k_rev_cost_fin<<<grid_for(n, kBlock, sms * 8), kBlock, 0, s>>>(rev_indptr, eff_indptr, acc, n, cu);
    check_launch();
  }
#else
  k_rev_cost<<<grid_for(n * 32, kBlock, sms * 16), kBlock, 0, s>>>(
      rev_indptr, reinterpret_cast<const int2*>(rev_seg), eff_indptr, n, cu);
  check_launch();
#endif
  TC_CUDA(cudaMemsetAsync(cu + n, 0, sizeof(int64_t), s));
  {
    size_t tmp = 0;
    TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cu, rev_cost, n + 1, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, cu, rev_cost, n + 1, s));
  }
}

// ---------------------------------------------------------------- costs

__global__ void k_cost_simple(int kind, const int32_t* __restrict__ deg, int64_t n, int64_t* out) {
  GRID_STRIDE(v, n) out[v] = (kind == TC_COST_UNIT) ? 1 : (kind == TC_COST_DEGREE ? (int64_t)deg[v] : 0);
}

// SUCC_SUM (partitioning.py:89): warp per v, sum over N^_v of d^_v + d^_u.
__global__ void k_cost_succ(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const int32_t* __restrict__ eff_deg, int64_t n, int64_t* out) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps) {
    int64_t e0 = indptr[v], e1 = indptr[v + 1];
    long long s = 0;
    for (int64_t e = e0 + lane; e < e1; e += 32) s += eff_deg[indices[e]];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[v] = (int64_t)s + (e1 - e0) * (e1 - e0);
  }
}

// PRED_SUM (partitioning.py:91): each edge (v,u) adds d^_v + d^_u to u.
__global__ void k_cost_pred(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const int32_t* __restrict__ eff_deg, int64_t n, int64_t* out) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps) {
    int64_t e0 = indptr[v], e1 = indptr[v + 1];
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      int32_t u = indices[e];
      atomicAdd(reinterpret_cast<unsigned long long*>(&out[u]),
                (unsigned long long)((e1 - e0) + eff_deg[u]));
    }
  }
}

void node_costs(int kind, const int64_t* eff_indptr, const int32_t* eff_indices, const int32_t* deg,
                const int32_t* eff_deg, int64_t n, int64_t* out, cudaStream_t s) {
  TC_REQUIRE(kind >= 0 && kind <= 3, TC_EINVAL, "unknown cost kind");
  if (n == 0) return;
  int sms = sm_count();
  k_cost_simple<<<grid_for(n, kBlock), kBlock, 0, s>>>(kind, deg, n, out);
  check_launch();
  if (kind == TC_COST_SUCC_SUM) {
    k_cost_succ<<<grid_for(n * 32, kBlock, sms * 16), kBlock, 0, s>>>(eff_indptr, eff_indices, eff_deg, n, out);
  } else if (kind == TC_COST_PRED_SUM) {
    k_cost_pred<<<grid_for(n * 32, kBlock, sms * 16), kBlock, 0, s>>>(eff_indptr, eff_indices, eff_deg, n, out);
  }
  check_launch();
}

}  // namespace tcb

extern "C" {

int tc_normalize(const int32_t* edges, int64_t m_raw, int32_t* out_edges, int64_t* m_host,
                 int64_t* n_host, tc_stream_t stream) {
  return tcb::guarded([&] {
    tcb::normalize(edges, m_raw, out_edges, m_host, n_host, (cudaStream_t)stream);
  });
}

int tc_build_graph(const int32_t* edges, int64_t m, int64_t n, const int32_t* order,
                   int64_t* eff_indptr, int32_t* eff_indices, int32_t* relabel,
                   int32_t* orig_ids, int32_t* deg, int32_t* eff_deg, int64_t* rev_indptr,
                   int32_t* rev_seg, int64_t* rev_cost, int64_t* pool_indptr, int32_t* pool,
                   tc_stream_t stream) {
  return tcb::guarded([&] {
    tcb::build_graph(edges, m, n, order, eff_indptr, eff_indices, relabel, orig_ids, deg, eff_deg,
                     rev_indptr, rev_seg, rev_cost, pool_indptr, pool, (cudaStream_t)stream);
  });
}

int tc_build_graph_deg(const int32_t* edges, int64_t m, int64_t n, const int32_t* deg_hint,
                       int64_t* eff_indptr, int32_t* eff_indices, int32_t* relabel,
                       int32_t* orig_ids, int32_t* deg, int32_t* eff_deg, int64_t* rev_indptr,
                       int32_t* rev_seg, int64_t* rev_cost, int64_t* pool_indptr, int32_t* pool,
                       tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(deg_hint != nullptr, TC_EINVAL, "NULL deg_hint");
    tcb::build_graph(edges, m, n, nullptr, eff_indptr, eff_indices, relabel, orig_ids, deg, eff_deg,
                     rev_indptr, rev_seg, rev_cost, pool_indptr, pool, (cudaStream_t)stream, deg_hint);
  });
}

int tc_normalize_host(const int32_t* host_edges, int64_t m_raw, int32_t* dev_edges, int32_t* out_edges,
                      int64_t* m_host, int64_t* n_host, int32_t* deg, int32_t* deg_valid, tc_stream_t stream) {
  return tcb::guarded([&] {
    tcb::normalize_host(host_edges, m_raw, dev_edges, out_edges, m_host, n_host, deg, deg_valid,
                        (cudaStream_t)stream);
  });
}

int tc_build_full(const int64_t* eff_indptr, const int32_t* eff_indices,
                  const int64_t* rev_indptr, const int32_t* rev_seg, const int64_t* pool_indptr, int64_t n,
                  int64_t* full_indptr, int32_t* full_indices, tc_stream_t stream) {
  return tcb::guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    int sms = tcb::sm_count();
    int64_t m2 = 0;
    {
      int64_t a = 0, b = 0;
      TC_CUDA(cudaMemcpyAsync(&a, eff_indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      TC_CUDA(cudaMemcpyAsync(&b, rev_indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      tcb::sync_stream(s);
      m2 = a + b;
    }
    tcb::Scratch sc(s);
    int32_t* unsorted = sc.alloc<int32_t>(m2 > 0 ? m2 : 1);
    tcb::k_full<<<tcb::grid_for((n + 1) * 32, 256, sms * 16), 256, 0, s>>>(
        eff_indptr, eff_indices, rev_indptr, reinterpret_cast<const int2*>(rev_seg), pool_indptr, n, full_indptr,
        unsorted);
    tcb::check_launch();
    if (m2 > 0) {  // predecessor rows are unordered (k_rev_scatter): sort every row
      TC_REQUIRE(m2 < (1ll << 31), TC_EINVAL, "full CSR too large");
      size_t tmp = 0;
      TC_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, unsorted, full_indices, (int)m2, (int)n,
                                                 full_indptr, full_indptr + 1, s));
      void* t = sc.bytes(tmp);
      TC_CUDA(cub::DeviceSegmentedSort::SortKeys(t, tmp, unsorted, full_indices, (int)m2, (int)n, full_indptr,
                                                 full_indptr + 1, s));
    }
  });
}

int tc_node_costs(int32_t kind, const int64_t* eff_indptr, const int32_t* eff_indices,
                  const int32_t* deg, const int32_t* eff_deg, int64_t n, int64_t* out,
                  tc_stream_t stream) {
  return tcb::guarded([&] {
    tcb::node_costs(kind, eff_indptr, eff_indices, deg, eff_deg, n, out, (cudaStream_t)stream);
  });
}

}  // extern "C"

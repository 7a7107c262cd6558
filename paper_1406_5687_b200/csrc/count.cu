// count.cu -- the intersection engine (sm_100a).
//
// Work model.  Every triangle v < u < w (canonical degree order) is found by
// probing list elements into a shared-memory table:
//
//   pull ("middle vertex", tc_count_middle): owner = u.  Table = N^_u;
//        segments = for each predecessor v of u, the suffix of N^_v after u
//        (rev_seg).  Probes per graph = sum_v C(d^_v, 2), 2-5x fewer than the
//        merge model's W -- the headline path.
//   push ("lowest vertex", tc_count_lowest): owner = v.  Table = N^_v;
//        segments = N^_u for every u in N^_v.  This is exactly
//        count_node_range(v0, v1) (_kernels.py:40-52) with per-bucket
//        partials, used for count_task / count_dynamic.
//
// A warp owns one owner at a time: it stages the owner's list in its
// shared-memory slice (sorted copy + hashed bitmap filter), then streams the
// owner's segments 32 probes per step: segments are compacted across lanes,
// flattened with a warp scan, and each lane resolves its segment with one
// ballot + one redux.or + popc (no per-probe search).  A probe is a range
// check, one bitmap LDS, and -- only for bitmap hits -- a binary search in
// the sorted copy.  Lists longer than the shared slice fall back to binary
// search in global memory (L1/L2 resident).
//
// Load balance (the paper's dynamic load balancing, PAPER.md:788-822,
// dynamic_lb.py:68-109, restated for warps): the owner-cost prefix is split
// in cost space -- the first half into one equal chunk per warp, then
// geometrically shrinking chunks of (remaining / warps), then fixed minimum
// chunks -- and chunk boundaries fall INSIDE an owner's segment list, so a
// hub never pins a warp.  Warps pull chunk indices from one global atomic
// counter (the coordinator's queue).
#include <cub/cub.cuh>

#include "common.cuh"

namespace tcb {

#ifndef TCB_MINBLOCKS
#define TCB_MINBLOCKS 6
#endif
#ifndef TCB_WINDOWS
#define TCB_WINDOWS 2
#endif
static constexpr int kWarps = 8;          // warps per block
static constexpr int kWin = TCB_WINDOWS;  // 32-chunk windows in flight per warp
static constexpr int kThreads = kWarps * 32;
static constexpr int kTabCap = 256;       // sorted-table capacity per warp (elements)
static constexpr int kBmWords = 512;      // filter words per warp (16384 bits)
static constexpr int kSegCost = 2;        // must match build.cu
static constexpr int kTabCost = 16;

struct WarpSlice {
  int32_t tab[kTabCap];
  uint32_t bm[kBmWords];
};

// --------------------------------------------------------------- segments

struct PullSegs {  // rev_seg pairs (start, end) into the pool
  const longlong2* seg;
  __device__ __forceinline__ void get(int64_t r, int64_t& s, int64_t& e) const {
    longlong2 x = __ldg(&seg[r]);
    s = x.x;
    e = x.y;
  }
};

struct PushSegs {  // forward edge e of v -> N^_u, u = indices[e]
  const int64_t* indptr;
  const int32_t* indices;
  __device__ __forceinline__ void get(int64_t r, int64_t& s, int64_t& e) const {
    int32_t u = __ldg(&indices[r]);
    s = __ldg(&indptr[u]);
    e = __ldg(&indptr[u + 1]);
  }
};

__device__ __forceinline__ uint32_t hash32(uint32_t w) { return w * 0x9E3779B1u; }

__device__ __forceinline__ bool bsearch_smem(const int32_t* t, int d, int32_t w) {
  int lo = 0, hi = d;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (t[mid] < w) lo = mid + 1;
    else hi = mid;
  }
  return lo < d && t[lo] == w;
}

__device__ __forceinline__ bool bsearch_gmem(const int32_t* __restrict__ t, int64_t d, int32_t w) {
  int64_t lo = 0, hi = d;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(&t[mid]) < w) lo = mid + 1;
    else hi = mid;
  }
  return lo < d && __ldg(&t[lo]) == w;
}

struct EngineArgs {
  const int64_t* row_indptr;  // owner -> segment index range
  const int64_t* tab_indptr;  // owner -> table list
  const int32_t* tab_indices;
  const int32_t* pool;        // segment coordinates index this array
  const int64_t* chunk_r;     // [nmax+1] segment-index chunk boundaries
  const int32_t* chunk_x;     // [nmax] owner at chunk start
  const int* nchunks;
  int* queue;
  const int64_t* bucket_bounds;  // nullable; bins owners
  int nbuckets;
  unsigned long long* out;
  int64_t n_owner;            // row_indptr has n_owner + 1 entries
  const int32_t* owner_map;   // nullable: owner x -> table/bucket node id
};

__device__ __forceinline__ int bucket_of(const int64_t* bb, int nb, int64_t x) {
  if (!bb) return 0;
  int lo = 0, hi = nb;  // largest b with bb[b] <= x
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (__ldg(&bb[mid]) <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Hashed one-bit filter over one owner's list: bit (h >> 18) of the 16K-bit
// word array (word h >> 23, bit (h >> 18) & 31), h = w * golden.  A probe is
// one LDS and three ALU ops; the false-positive rate is d / 16384 per probe,
// and positives are verified by binary search in the sorted copy.
__device__ __forceinline__ uint32_t filt_hash(uint32_t w) { return w * 0x9E3779B1u; }

__device__ __forceinline__ void filt_insert(uint32_t* bm, int32_t w) {
  uint32_t h = filt_hash((uint32_t)w);
  atomicOr(&bm[h >> 23], 1u << ((h >> 18) & 31));
}

// 4-bit mask of the elements of v (valid ones per vmask) that pass the
// range check and hit the filter.  Branch-free.
__device__ __forceinline__ uint32_t filt_probe4(const uint32_t* bm, int4 v, uint32_t vmask, int32_t tmin,
                                                int32_t tmax) {
  uint32_t m = 0;
  int32_t xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t h = filt_hash((uint32_t)xs[k]);
    uint32_t wd = bm[h >> 23];
    uint32_t bit = (wd >> ((h >> 18) & 31)) & 1u;
    bool in = ((vmask >> k) & 1u) && xs[k] >= tmin && xs[k] <= tmax;
    m |= (in ? bit : 0u) << k;
  }
  return m;
}

// Resolve the probes of one group of <= 32 compacted segments.  The group is
// flattened over the 16-byte chunks its segments touch: lane j of window k
// loads chunk base+32k+j as one int4 (4 list elements) and probes the
// elements of it that lie inside its segment.  Two windows are in flight.
// Segment s covers chunks [excl_s, endx_s) of the flat space; chunk f of it
// is pool4[delta_s + f]; `edge_s` packs (first-chunk offset | last-chunk
// count << 2).
template <bool kSmall>
__device__ __forceinline__ void probe_group(const int4* __restrict__ pool4, const WarpSlice& sl,
                                            const int32_t* __restrict__ gtab, int64_t d, int32_t tmin,
                                            int32_t tmax, int nseg, int excl, int endx, int edge,
                                            int64_t delta, int total, int lane, uint32_t& cnt) {
  const unsigned FULL = 0xffffffffu;
  const bool lane_seg = lane < nseg;
  for (int base = 0; base < total; base += 32 * kWin) {
    int4 v[kWin];
    uint32_t vm[kWin];
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
      const int b = base + 32 * k;
      vm[k] = 0;
      v[k] = make_int4(0, 0, 0, 0);
      if (b < total) {
        unsigned cov = __ballot_sync(FULL, lane_seg && excl <= b);
        int c0 = __popc(cov) - 1;
        unsigned bit = (lane_seg && excl > b && excl < b + 32) ? (1u << (excl - b)) : 0u;
        unsigned starts = __reduce_or_sync(FULL, bit);
        int sj = c0 + __popc(starts & ((2u << lane) - 1u));
        int64_t dl = __shfl_sync(FULL, delta, sj);
        int ex = __shfl_sync(FULL, excl, sj);
        int en = __shfl_sync(FULL, endx, sj);
        int eg = __shfl_sync(FULL, edge, sj);
        int f = b + lane;
        if (f < total) {
          v[k] = __ldg(&pool4[dl + f]);
          uint32_t lo = (f == ex) ? (uint32_t)(eg & 3) : 0u;
          uint32_t hi = (f == en - 1) ? (uint32_t)(eg >> 2) : 4u;
          vm[k] = (0xFu >> (4 - hi)) & (0xFu << lo);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
      if (kSmall) {
        uint32_t m = filt_probe4(sl.bm, v[k], vm[k], tmin, tmax);
        if (m) {
          int32_t xs[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if ((m >> e) & 1u) cnt += bsearch_smem(sl.tab, (int)d, xs[e]);
        }
      } else {
        int32_t xs[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (((vm[k] >> e) & 1u) && xs[e] >= tmin && xs[e] <= tmax) cnt += bsearch_gmem(gtab, d, xs[e]);
      }
    }
  }
}

template <class Segs>
__global__ void __launch_bounds__(kThreads, TCB_MINBLOCKS) k_engine(EngineArgs a, Segs segs) {
  __shared__ WarpSlice slices[kWarps];
  const int lane = threadIdx.x & 31;
  WarpSlice& sl = slices[threadIdx.x >> 5];
  const unsigned FULL = 0xffffffffu;
  const int nch = *a.nchunks;
  for (int i = lane; i < kBmWords; i += 32) sl.bm[i] = 0;
  __syncwarp();

  unsigned long long acc = 0;  // warp total for the current bucket (same on all lanes)
  int cur_bucket = -1;
  uint32_t cnt = 0;            // per-lane hits since the last fold
  auto fold = [&]() {
    unsigned long long t = cnt;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
    acc += t;
    cnt = 0;
  };

  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(a.queue, 1);
    c = __shfl_sync(FULL, c, 0);
    if (c >= nch) break;
    int64_t r = a.chunk_r[c];
    const int64_t r1 = a.chunk_r[c + 1];
    int64_t x = a.chunk_x[c];

    while (r < r1) {
      // advance to the owner whose segment row contains r (skips empty rows)
      for (;;) {
        int64_t idx = x + 1 + lane;
        int64_t nx = (idx <= a.n_owner) ? __ldg(&a.row_indptr[idx]) : INT64_MAX;
        unsigned past = __ballot_sync(FULL, nx > r);
        if (past) {
          x += __ffs(past) - 1;
          break;
        }
        x += 32;
      }
      const int64_t xe_row = __ldg(&a.row_indptr[x + 1]);
      const int64_t rb = min(xe_row, r1);
      const int64_t ra = r;

      if (a.bucket_bounds) {
        int b = bucket_of(a.bucket_bounds, a.nbuckets, a.owner_map ? (int64_t)__ldg(&a.owner_map[x]) : x);
        if (b != cur_bucket) {
          fold();
          if (lane == 0 && cur_bucket >= 0 && acc) atomicAdd(&a.out[cur_bucket], acc);
          acc = 0;
          cur_bucket = b;
        }
      } else {
        cur_bucket = 0;
      }

      const int64_t u = a.owner_map ? (int64_t)__ldg(&a.owner_map[x]) : x;
      const int64_t t0 = __ldg(&a.tab_indptr[u]);
      const int64_t d = __ldg(&a.tab_indptr[u + 1]) - t0;
      if (d > 0) {
        const bool small = d <= kTabCap;
        int32_t tmin, tmax;
        const int32_t* gtab = a.tab_indices + t0;
        if (small) {
          for (int i = lane; i < d; i += 32) {
            int32_t w = __ldg(&gtab[i]);
            sl.tab[i] = w;
            filt_insert(sl.bm, w);
          }
          __syncwarp();
          tmin = sl.tab[0];
          tmax = sl.tab[d - 1];
        } else {
          tmin = __ldg(&gtab[0]);
          tmax = __ldg(&gtab[d - 1]);
        }

        for (int64_t g = ra; g < rb; g += 32) {
          int64_t s = 0, e = 0;
          if (g + lane < rb) segs.get(g + lane, s, e);
          int len = (int)(e - s);
          // compact non-empty segments to the low lanes
          unsigned nz = __ballot_sync(FULL, len > 0);
          int nseg = __popc(nz);
          int src = (lane < nseg) ? (int)__fns(nz, 0, lane + 1) : 0;
          int64_t cs = __shfl_sync(FULL, s, src);
          int clen = __shfl_sync(FULL, len, src);
          if (lane >= nseg) clen = 0;
          // chunk span of each segment: [cs >> 2, (cs + clen + 3) >> 2)
          const int64_t c0s = cs >> 2;
          const int nch = (lane < nseg) ? (int)(((cs + clen + 3) >> 2) - c0s) : 0;
          const int edge = (int)(cs & 3) | ((int)(((cs + clen - 1) & 3) + 1) << 2);
          int incl = nch;  // inclusive prefix of chunk counts
          for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
          }
          const int total = __shfl_sync(FULL, incl, 31);
          const int excl = incl - nch;
          const int64_t delta = c0s - excl;  // flat chunk f of this segment: pool4[delta + f]
          const int4* pool4 = reinterpret_cast<const int4*>(a.pool);
          if (small)
            probe_group<true>(pool4, sl, gtab, d, tmin, tmax, nseg, excl, incl, edge, delta, total, lane, cnt);
          else
            probe_group<false>(pool4, sl, gtab, d, tmin, tmax, nseg, excl, incl, edge, delta, total, lane, cnt);
        }
        if (small) {  // clear the words this owner set
          __syncwarp();
          for (int i = lane; i < d; i += 32) sl.bm[filt_hash((uint32_t)sl.tab[i]) >> 23] = 0;
          __syncwarp();
        }
      }
      r = rb;
    }
    fold();
  }
  if (lane == 0 && cur_bucket >= 0 && acc) atomicAdd(&a.out[cur_bucket], acc);
}

// --------------------------------------------------------------- planning

// Chunk schedule in cost space (see file header).  Thread i computes the
// i-th boundary; thread 0 also publishes the chunk count.
// mode 0 (paper): first half of the cost in one chunk per warp (Eq. 1),
// then geometric chunks.  mode 1 (L2-tiled owners): the first 3/4 in
// uniform chunks of 1/8 per-warp share, consumed in owner order so the
// active window stays inside one or two tiles, then the geometric tail.
__global__ void k_plan(const int64_t* __restrict__ cp, const int64_t* __restrict__ row_indptr,
                       int64_t x0, int64_t x1, int nW, int nmax, int64_t* chunk_r,
                       int32_t* chunk_x, int* nchunks, int mode) {
  const int64_t base = cp[x0];
  const int64_t C = cp[x1] - base;
  const double Cd = (double)C;
  const int nfirst = mode == 0 ? nW : 6 * nW;
  const double half = mode == 0 ? floor(Cd / 2.0) : floor(Cd * 0.75);
  const double R0 = Cd - half;
  const double q = 1.0 - 1.0 / (double)nW;
  const double minc = fmax(Cd / (32.0 * nW), 64.0);
  int64_t J = 0;
  if (nW > 1 && R0 / nW > minc) J = (int64_t)ceil(log(minc * nW / R0) / log(q));
  if (J < 0) J = 0;
  const double RJ = R0 * pow(q, (double)J);
  const int64_t ntail = (int64_t)ceil(RJ / minc);
  int64_t total = (C == 0) ? 0 : (int64_t)nfirst + J + ntail;
  if (total > nmax) total = nmax;
  if (blockIdx.x == 0 && threadIdx.x == 0) *nchunks = (int)total;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nmax;
       i += (int64_t)gridDim.x * blockDim.x) {
    double t;
    if (i >= total) t = Cd;
    else if (i <= nfirst) t = floor((double)i * half / (double)nfirst);
    else {
      int64_t j = i - nfirst;
      if (j <= J) t = half + R0 * (1.0 - pow(q, (double)j));
      else t = half + (R0 - RJ) + (double)(j - J) * minc;
    }
    int64_t T = (int64_t)t;
    if (T > C) T = C;
    if (T < 0) T = 0;
    int64_t r, x;
    if (T >= C) {
      x = x1;
      r = row_indptr[x1];
    } else {
      // largest x in [x0, x1) with cp[x] - base <= T
      int64_t lo = x0, hi = x1;
      while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (cp[mid] - base <= T) lo = mid;
        else hi = mid;
      }
      x = lo;
      int64_t cx = cp[x + 1] - cp[x];
      int64_t rows = row_indptr[x + 1] - row_indptr[x];
      int64_t off = 0;
      if (cx > 0) off = (int64_t)((double)(T - (cp[x] - base)) / (double)cx * (double)rows);
      if (off > rows) off = rows;
      r = row_indptr[x] + off;
    }
    chunk_r[i] = r;
    if (i < nmax) chunk_x[i] = (int32_t)x;
  }
}

// push-engine owner cost: sum over u in N^_v of (d^_u + kSegCost) + d^_v + kTabCost
__global__ void k_push_cost(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            int64_t v0, int64_t v1, int64_t* cost) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = v0 + warp; v < v1; v += nwarps) {
    int64_t e0 = indptr[v], e1 = indptr[v + 1];
    long long s = 0;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      int32_t u = indices[e];
      s += (indptr[u + 1] - indptr[u]) + kSegCost;
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) cost[v - v0] = (e1 > e0) ? (int64_t)s + (e1 - e0) + kTabCost : 0;
  }
}

// --------------------------------------------------------------- drivers

// Optional CUDA-event bracket around every engine launch (bench.py reads
// the dominant kernel's device time through tc_engine_time_ms).
static bool g_time_engine = false;
static cudaEvent_t g_ev[2] = {nullptr, nullptr};
static double g_engine_ms = 0.0;
static long long g_engine_launches = 0;

static int engine_blocks() {
  static int blocks = 0;
  if (!blocks) {
    int per_sm = 0;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_engine<PullSegs>, kThreads, 0));
    if (per_sm < 1) per_sm = 1;
    blocks = per_sm * sm_count();
  }
  return blocks;
}

template <class Segs>
void run_engine(Scratch& sc, int64_t n_owner, const int64_t* cp, const int64_t* row_indptr, const int64_t* tab_indptr,
                const int32_t* tab_indices, const int32_t* pool, int64_t x0, int64_t x1,
                const int64_t* bucket_bounds, int nbuckets, unsigned long long* out, Segs segs,
                cudaStream_t s, const int32_t* owner_map = nullptr, int mode = 0) {
  int blocks = engine_blocks();
  int nW = blocks * kWarps;
  int nmax = 10 * nW + 8;
  int64_t* chunk_r = sc.alloc<int64_t>(nmax + 1);
  int32_t* chunk_x = sc.alloc<int32_t>(nmax);
  int* ctl = sc.alloc<int>(2);  // [0] nchunks, [1] queue
  TC_CUDA(cudaMemsetAsync(ctl, 0, 2 * sizeof(int), s));
  k_plan<<<grid_for(nmax + 1, 256), 256, 0, s>>>(cp, row_indptr, x0, x1, nW, nmax, chunk_r, chunk_x, ctl, mode);
  check_launch();
  EngineArgs a{row_indptr, tab_indptr, tab_indices, pool, chunk_r, chunk_x, ctl, ctl + 1,
               bucket_bounds, nbuckets, out, n_owner, owner_map};
  if (g_time_engine) {
    if (!g_ev[0]) {
      TC_CUDA(cudaEventCreate(&g_ev[0]));
      TC_CUDA(cudaEventCreate(&g_ev[1]));
    }
    TC_CUDA(cudaEventRecord(g_ev[0], s));
  }
  k_engine<Segs><<<blocks, kThreads, 0, s>>>(a, segs);
  check_launch();
  if (g_time_engine) {
    TC_CUDA(cudaEventRecord(g_ev[1], s));
    TC_CUDA(cudaEventSynchronize(g_ev[1]));
    float ms = 0.f;
    TC_CUDA(cudaEventElapsedTime(&ms, g_ev[0], g_ev[1]));
    g_engine_ms += ms;
    ++g_engine_launches;
  }
}

void count_middle(const int64_t* tab_indptr, const int32_t* tab_indices, const int64_t* rev_indptr,
                  const int64_t* rev_seg, const int64_t* rev_cost, const int32_t* pool, int64_t n,
                  int64_t u0, int64_t u1, const int64_t* bucket_bounds, int nbuckets,
                  unsigned long long* out, cudaStream_t s) {
  TC_REQUIRE(0 <= u0 && u0 <= u1 && u1 <= n, TC_EINVAL, "bad owner range");
  TC_REQUIRE(nbuckets >= 1, TC_EINVAL, "nbuckets must be >= 1");
  TC_REQUIRE(bucket_bounds || nbuckets == 1, TC_EINVAL, "bucket_bounds required for nbuckets > 1");
  TC_REQUIRE(((uintptr_t)pool & 15) == 0, TC_EINVAL, "pool must be 16-byte aligned (and padded to a multiple of 4 ids)");
  TC_CUDA(cudaMemsetAsync(out, 0, nbuckets * sizeof(unsigned long long), s));
  if (u1 <= u0) return;
  Scratch sc(s);
  run_engine(sc, n, rev_cost, rev_indptr, tab_indptr, tab_indices, pool, u0, u1, bucket_bounds,
             nbuckets, out, PullSegs{reinterpret_cast<const longlong2*>(rev_seg)}, s, nullptr, 1);
}

void count_owners(const int64_t* tab_indptr, const int32_t* tab_indices, const int32_t* owner_map,
                  const int64_t* row_indptr, const int64_t* segs, const int64_t* cost_prefix,
                  const int32_t* pool, int64_t k, const int64_t* bucket_bounds, int nbuckets,
                  unsigned long long* out, int mode, cudaStream_t s) {
  TC_REQUIRE(k >= 0 && nbuckets >= 1, TC_EINVAL, "bad owner count / nbuckets");
  TC_REQUIRE(bucket_bounds || nbuckets == 1, TC_EINVAL, "bucket_bounds required for nbuckets > 1");
  TC_REQUIRE(((uintptr_t)pool & 15) == 0, TC_EINVAL, "pool must be 16-byte aligned (and padded to a multiple of 4 ids)");
  TC_CUDA(cudaMemsetAsync(out, 0, nbuckets * sizeof(unsigned long long), s));
  if (k == 0) return;
  Scratch sc(s);
  run_engine(sc, k, cost_prefix, row_indptr, tab_indptr, tab_indices, pool, 0, k, bucket_bounds,
             nbuckets, out, PullSegs{reinterpret_cast<const longlong2*>(segs)}, s, owner_map, mode);
}

void count_lowest(const int64_t* indptr, const int32_t* indices, int64_t n, int64_t v0, int64_t v1,
                  const int64_t* bucket_bounds, int nbuckets, unsigned long long* out,
                  cudaStream_t s) {
  TC_REQUIRE(0 <= v0 && v0 <= v1 && v1 <= n, TC_EINVAL, "bad node range");
  TC_REQUIRE(nbuckets >= 1, TC_EINVAL, "nbuckets must be >= 1");
  TC_REQUIRE(bucket_bounds || nbuckets == 1, TC_EINVAL, "bucket_bounds required for nbuckets > 1");
  TC_REQUIRE(((uintptr_t)indices & 15) == 0, TC_EINVAL, "indices must be 16-byte aligned (and padded to a multiple of 4 ids)");
  TC_CUDA(cudaMemsetAsync(out, 0, nbuckets * sizeof(unsigned long long), s));
  if (v1 <= v0) return;
  Scratch sc(s);
  int64_t nv = v1 - v0;
  // cost prefix over owners [v0, v1], stored relative (index x - v0)
  int64_t* cost = sc.alloc<int64_t>(nv + 1);
  int64_t* cp = sc.alloc<int64_t>(nv + 1);
  TC_CUDA(cudaMemsetAsync(cost + nv, 0, sizeof(int64_t), s));
  k_push_cost<<<grid_for(nv * 32, 256, sm_count() * 16), 256, 0, s>>>(indptr, indices, v0, v1, cost);
  check_launch();
  {
    size_t tmp = 0;
    TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cost, cp, nv + 1, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, cost, cp, nv + 1, s));
  }
  // the planner indexes cp by absolute owner id: shift the pointer
  run_engine(sc, n, cp - v0, indptr, indptr, indices, indices, v0, v1, bucket_bounds, nbuckets, out,
             PushSegs{indptr, indices}, s);
}

// --------------------------------------------------------------- small kernels

__global__ void k_intersect(const int32_t* __restrict__ a, int64_t na, const int32_t* __restrict__ b,
                            int64_t nb, unsigned long long* out) {
  unsigned long long c = 0;
  GRID_STRIDE(i, na) c += bsearch_gmem(b, nb, a[i]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void k_brute_bits(const int64_t* __restrict__ ip, const int32_t* __restrict__ ix, int64_t n,
                             int64_t words, uint32_t* adj) {
  GRID_STRIDE(v, n) {
    for (int64_t k = ip[v]; k < ip[v + 1]; ++k) {
      int32_t u = ix[k];
      atomicOr(&adj[v * words + (u >> 5)], 1u << (u & 31));
    }
  }
}

// Sum over edges u < v of |N(u) ∩ N(v) ∩ (v, n)| from the dense bitmap.
__global__ void k_brute_count(const uint32_t* __restrict__ adj, int64_t n, int64_t words,
                              unsigned long long* out) {
  unsigned long long c = 0;
  GRID_STRIDE(p, n * n) {
    int64_t u = p / n, v = p % n;
    if (u < v && ((adj[u * words + (v >> 5)] >> (v & 31)) & 1u)) {
      for (int64_t wd = (v + 1) >> 5; wd < words; ++wd) {
        uint32_t m = adj[u * words + wd] & adj[v * words + wd];
        if (wd == ((v + 1) >> 5)) m &= ~0u << ((v + 1) & 31);
        c += __popc(m);
      }
    }
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

}  // namespace tcb

extern "C" {

int tc_count_middle(const int64_t* tab_indptr, const int32_t* tab_indices,
                    const int64_t* rev_indptr, const int64_t* rev_seg, const int64_t* rev_cost,
                    const int32_t* pool, int64_t n, int64_t u0, int64_t u1,
                    const int64_t* bucket_bounds, int32_t nbuckets, unsigned long long* out,
                    tc_stream_t stream) {
  return tcb::guarded([&] {
    tcb::count_middle(tab_indptr, tab_indices, rev_indptr, rev_seg, rev_cost, pool, n, u0, u1,
                      bucket_bounds, nbuckets, out, (cudaStream_t)stream);
  });
}

int tc_count_owners(const int64_t* tab_indptr, const int32_t* tab_indices, const int32_t* owner_map,
                    const int64_t* row_indptr, const int64_t* segs, const int64_t* cost_prefix,
                    const int32_t* pool, int64_t k, const int64_t* bucket_bounds, int32_t nbuckets,
                    unsigned long long* out, int32_t mode, tc_stream_t stream) {
  return tcb::guarded([&] {
    tcb::count_owners(tab_indptr, tab_indices, owner_map, row_indptr, segs, cost_prefix, pool, k,
                      bucket_bounds, nbuckets, out, mode, (cudaStream_t)stream);
  });
}

int tc_count_lowest(const int64_t* eff_indptr, const int32_t* eff_indices, int64_t n, int64_t v0,
                    int64_t v1, const int64_t* bucket_bounds, int32_t nbuckets,
                    unsigned long long* out, tc_stream_t stream) {
  return tcb::guarded([&] {
    tcb::count_lowest(eff_indptr, eff_indices, n, v0, v1, bucket_bounds, nbuckets, out,
                      (cudaStream_t)stream);
  });
}

int tc_engine_timing(int32_t enable, double* total_ms_host, long long* launches_host) {
  return tcb::guarded([&] {
    if (total_ms_host) *total_ms_host = tcb::g_engine_ms;
    if (launches_host) *launches_host = tcb::g_engine_launches;
    if (enable >= 0) {
      tcb::g_time_engine = enable != 0;
      tcb::g_engine_ms = 0.0;
      tcb::g_engine_launches = 0;
    }
  });
}

int tc_intersect_count(const int32_t* a, int64_t na, const int32_t* b, int64_t nb,
                       unsigned long long* out, tc_stream_t stream) {
  return tcb::guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), s));
    if (na <= 0 || nb <= 0) return;
    tcb::k_intersect<<<tcb::grid_for(na, 256), 256, 0, s>>>(a, na, b, nb, out);
    tcb::check_launch();
  });
}

int tc_count_brute(const int64_t* full_indptr, const int32_t* full_indices, int64_t n,
                   unsigned long long* out, tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(n <= 2000, TC_EINVAL, "brute-force counter limited to n <= 2000");
    cudaStream_t s = (cudaStream_t)stream;
    TC_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), s));
    if (n < 3) return;
    tcb::Scratch sc(s);
    int64_t words = (n + 31) / 32;
    uint32_t* adj = sc.alloc<uint32_t>(n * words);
    TC_CUDA(cudaMemsetAsync(adj, 0, n * words * sizeof(uint32_t), s));
    tcb::k_brute_bits<<<tcb::grid_for(n, 256), 256, 0, s>>>(full_indptr, full_indices, n, words, adj);
    tcb::check_launch();
    tcb::k_brute_count<<<tcb::grid_for(n * n, 256), 256, 0, s>>>(adj, n, words, out);
    tcb::check_launch();
  });
}

}  // extern "C"

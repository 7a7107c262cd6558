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

// Per-destination counters of a block (P <= kMaxDest): elements are counted
// in shared memory and every block adds its totals once -- one global atomic
// per element on P addresses serialised the whole grid (35 ms per 64 M pairs).
static constexpr int kMaxDest = 1024;

__device__ __forceinline__ void flush_counts(const unsigned int* sc, int P, long long* counts) {
  __syncthreads();
  for (int j = threadIdx.x; j < P; j += blockDim.x)
    if (sc[j]) add64(&counts[j], (long long)sc[j]);
}

__global__ void k_sh_keys(const int2* __restrict__ pairs, int64_t m, const int32_t* __restrict__ map, int P,
                          unsigned long long* key, int32_t* dest, long long* counts) {
  __shared__ unsigned int sc[kMaxDest];
  for (int j = threadIdx.x; j < P; j += blockDim.x) sc[j] = 0;
  __syncthreads();
  GRID_STRIDE(i, m) {
    const int2 e = pairs[i];
    int d = -1;
    unsigned long long k = 0;
    if (e.x != e.y) {
      const uint32_t a = (uint32_t)(map ? map[e.x] : e.x), b = (uint32_t)(map ? map[e.y] : e.y);
      k = ((unsigned long long)min(a, b) << 32) | max(a, b);
      d = dest_of_key(k, P);
      atomicAdd(&sc[d], 1u);
    }
    key[i] = k;
    dest[i] = d;
  }
  flush_counts(sc, P, counts);
}

// scatter into groups by destination (order inside a group unspecified):
// per tile of blockDim elements the block counts its destinations in shared
// memory (the atomic's return value is the element's rank in the tile),
// reserves one range per destination with one global atomic, and writes.
template <class T>
__global__ void k_sh_group(const T* __restrict__ in, const int32_t* __restrict__ dest, int64_t m,
                           const long long* __restrict__ counts, const long long* __restrict__ off, long long* cursor,
                           T* out, int P) {
  __shared__ unsigned int sc[kMaxDest];
  __shared__ long long sbase[kMaxDest];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m; base += stride) {  // block-uniform trip count
    for (int j = threadIdx.x; j < P; j += blockDim.x) sc[j] = 0;
    __syncthreads();
    const int64_t i = base + threadIdx.x;
    const int d = i < m ? dest[i] : -1;
    unsigned int r = 0;
    if (d >= 0) r = atomicAdd(&sc[d], 1u);
    __syncthreads();
    for (int j = threadIdx.x; j < P; j += blockDim.x)
      if (sc[j]) {
        const long long c = add64(&cursor[j], (long long)sc[j]);
#if TCB_DEBUG
        assert(c + sc[j] <= counts[j]);
#endif
        sbase[j] = off[j] + c;
      }
    __syncthreads();
    if (d >= 0) out[sbase[d] + r] = in[i];
    __syncthreads();
  }
  (void)counts;
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
  __shared__ unsigned int sc[kMaxDest];
  for (int j = threadIdx.x; j < P; j += blockDim.x) sc[j] = 0;
  __syncthreads();
  GRID_STRIDE(i, k) {
    const int d = owner_of_id(bounds, P, lohi[i].x);
    dest[i] = d;
    atomicAdd(&sc[d], 1u);
  }
  flush_counts(sc, P, counts);
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
//
// Work layout of both send kernels: a warp handles 32 / G rows at a time
// (steps interleaved over all the grid's warps), G = max(8, pow2 >= P - 1 - rank)
// lanes per row, lane jl of a row's group standing for destination
// rank + 1 + jl; the rows of a warp and their order are fixed by (block,
// warp, nrow) alone.  The count kernel leaves, per (warp, destination), the
// warp's lists and padded words; a prefix over the warps turns them into
// each warp's first list / word slot inside each destination's part of the
// send buffers (the "send plan": static for a partitioned graph, kept with
// the sizes).  The pack kernel then needs no atomics and no counting pass,
// and its output is deterministic: a warp walks its rows with running
// offsets per destination (a prefix over the row slots of each step by
// shuffles) and the group's lanes copy each message as 16-byte chunks of
// the padded pool.
static constexpr int kEmitMaxP = 32;
static constexpr int kSendWarps = kBlk / 32;

static int send_group(int P, int rank) {  // lanes per row
  int g = 8;
  while (g < P - 1 - rank) g <<= 1;
  return g;
}

static int send_blocks(int64_t nrow) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((nrow + 255) / 256, (int64_t)sm_count() * 8));
}

// first id >= bj of row [a, a + d); true when it is owned by the destination
__device__ __forceinline__ bool send_msg(const int32_t* __restrict__ ids, int64_t a, int64_t d, int64_t bj,
                                         int64_t bj1, int64_t& s) {
  s = row_lb(ids, a, d, bj);
  return s < d && ids[a + s] < bj1;
}

__global__ void __launch_bounds__(kBlk) k_sh_send_count(const int64_t* __restrict__ indptr,
                                                        const int32_t* __restrict__ ids, int64_t nrow,
                                                        const int64_t* __restrict__ pptr,
                                                        const int64_t* __restrict__ bounds, int P, int rank, int G,
                                                        long long* tot, long long* unit_l, long long* unit_w) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rpw = 32 / G, g = lane / G, jl = lane % G, j = rank + 1 + jl;
  const int64_t unit = (int64_t)blockIdx.x * kSendWarps + warp, nunit = (int64_t)gridDim.x * kSendWarps;
  const bool dest = j < P;
  const int64_t bj = dest ? bounds[j] : 0, bj1 = dest ? bounds[j + 1] : 0;
  long long cl = 0, cw = 0, cf = 0;
  if (dest)
    // warp step q covers rows [q rpw, (q + 1) rpw); a warp takes the steps
    // q = unit (mod nunit): rows ascend in degree, so contiguous runs per
    // block would leave the last blocks with most of the ids
    for (int64_t v = unit * rpw + g; v < nrow; v += nunit * rpw) {
      const int64_t a = indptr[v], d = indptr[v + 1] - a;
      int64_t s;
      if (d > 0 && send_msg(ids, a, d, bj, bj1, s)) {
        ++cl;
        cw += (pptr[v + 1] - pptr[v]) - (s & ~3ll);
        cf += d;
      }
    }
  for (int o = G; o < 32; o <<= 1) {  // over the row slots of each destination
    cl += __shfl_xor_sync(FULL, cl, o);
    cw += __shfl_xor_sync(FULL, cw, o);
    cf += __shfl_xor_sync(FULL, cf, o);
  }
  if (g == 0 && dest) {
    unit_l[unit * P + j] = cl;
    unit_w[unit * P + j] = cw;
    if (cl) {
      add64(&tot[j], cl);
      add64(&tot[P + j], cw);
      add64(&tot[2 * P + j], cf);
    }
  }
}

// Per destination (one warp each): the warps' counts become their first
// slots, offset by the destinations before it.
__global__ void k_sh_send_prefix(const long long* __restrict__ tot, int P, int64_t nunit, long long* unit_l,
                                 long long* unit_w) {
  const int lane = threadIdx.x & 31, j = threadIdx.x >> 5;
  if (j >= P) return;
  long long run_l = 0, run_w = 0;
  for (int i = 0; i < j; ++i) {
    run_l += tot[i];
    run_w += tot[P + i];
  }
  for (int64_t b0 = 0; b0 < nunit; b0 += 32) {
    const int64_t b = b0 + lane;
    const long long vl = b < nunit ? unit_l[b * P + j] : 0, vw = b < nunit ? unit_w[b * P + j] : 0;
    long long il = vl, iw = vw;
    for (int o = 1; o < 32; o <<= 1) {
      const long long yl = __shfl_up_sync(0xffffffffu, il, o), yw = __shfl_up_sync(0xffffffffu, iw, o);
      if (lane >= o) {
        il += yl;
        iw += yw;
      }
    }
    if (b < nunit) {
      unit_l[b * P + j] = run_l + il - vl;
      unit_w[b * P + j] = run_w + iw - vw;
    }
    run_l += __shfl_sync(0xffffffffu, il, 31);
    run_w += __shfl_sync(0xffffffffu, iw, 31);
  }
}

// lower bound of x in a shared-memory row of d ascending ids
__device__ __forceinline__ int smem_lb(const int32_t* ids, int d, int64_t x) {
  int lo = 0, hi = d;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ids[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

static constexpr int kStageChunks = 32;  // rows of <= 128 ids are staged in shared memory

__global__ void __launch_bounds__(kBlk) k_sh_send_emit(const int64_t* __restrict__ indptr,
                                                       const int32_t* __restrict__ ids, int64_t nrow,
                                                       const int64_t* __restrict__ pptr,
                                                       const int4* __restrict__ pool4,
                                                       const int64_t* __restrict__ bounds, int P, int rank, int G,
                                                       const long long* __restrict__ base_l,
                                                       const long long* __restrict__ base_w, int32_t* out_len,
                                                       int4* out4) {
  // Rows of <= 32 chunks (almost all of them) are read once: the row's G
  // lanes stage its padded chunks in shared memory with up to 32 / G
  // independent 16-byte loads each, the destinations' lanes search the staged
  // ids, and the messages are written from shared memory -- two dependent
  // global round trips per step (offsets, row) instead of one per search
  // step and per message.  Longer rows search and copy from global memory.
  __shared__ int4 s_row[kSendWarps][4][kStageChunks];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rpw = 32 / G, g = lane / G, jl = lane % G, j = rank + 1 + jl, ndest = P - 1 - rank;
  const bool dest = j < P;
  const int64_t bj = dest ? bounds[j] : 0, bj1 = dest ? bounds[j + 1] : 0;
  const int64_t unit = (int64_t)blockIdx.x * kSendWarps + warp, nunit = (int64_t)gridDim.x * kSendWarps;
  long long run_l = dest ? base_l[unit * P + j] : 0;        // next list slot of destination j (this warp)
  long long run_c = dest ? base_w[unit * P + j] >> 2 : 0;   // next 16-byte chunk slot
  const int last = (rpw - 1) * G + jl;                       // the last row slot's lane for this destination
  const int32_t* pool = reinterpret_cast<const int32_t*>(pool4);
  int4* row = s_row[warp][g];  // rpw <= 4 rows per warp step
  (void)ids;
  for (int64_t vb = unit * rpw; vb < nrow; vb += nunit * rpw) {  // warp-uniform trip count (steps as in the count)
    const int64_t v = vb + g;
    int64_t d = 0, p = 0;
    if (v < nrow) {
      d = indptr[v + 1] - indptr[v];
      p = pptr[v];
    }
    const int pd = (int)((d + 3) >> 2);
    const bool staged = pd <= kStageChunks;
    __syncwarp();  // the previous step's reads of the staged rows are done
    if (staged)
      for (int c = jl; c < pd; c += G) row[c] = __ldg(&pool4[(p >> 2) + c]);
    __syncwarp();
    int s = 0, nch = 0;
    if (dest && d > 0) {
      bool hit;
      if (staged) {
        const int32_t* rid = reinterpret_cast<const int32_t*>(row);
        s = smem_lb(rid, (int)d, bj);
        hit = s < d && rid[s] < bj1;
      } else {
        int64_t s64;
        hit = send_msg(pool, p, d, bj, bj1, s64);
        s = (int)s64;
      }
      if (hit) nch = pd - (s >> 2);
    }
    // slots of this step's messages: prefix over the row slots of each destination
    int il = nch > 0, ic = nch;
    for (int o = G; o < 32; o <<= 1) {
      const int yl = __shfl_up_sync(FULL, il, o), yc = __shfl_up_sync(FULL, ic, o);
      if (lane >= o) {
        il += yl;
        ic += yc;
      }
    }
    if (nch > 0) out_len[run_l + (il - 1)] = (int32_t)(d - 4 * (s >> 2));
    const long long dst0 = run_c + (ic - nch);
    run_l += __shfl_sync(FULL, il, last);
    run_c += __shfl_sync(FULL, ic, last);
    const int c00 = s >> 2;  // first chunk of this lane's message inside its row
    for (int jj = 0; jj < ndest; ++jj) {  // the group's lanes copy one message at a time
      const int from = g * G + jj;
      const int n = __shfl_sync(FULL, nch, from);
      if (!__any_sync(FULL, n > 0)) continue;
      const int c0 = __shfl_sync(FULL, c00, from);
      const long long dc = __shfl_sync(FULL, dst0, from);
      if (staged) {
        for (int c = jl; c < n; c += G) out4[dc + c] = row[c0 + c];
      } else {
        const int4* src = pool4 + (p >> 2) + c0;
        for (int c = jl; c < n; c += G) out4[dc + c] = __ldg(&src[c]);
      }
    }
  }
}

// ------------------------------------------------------------ receive index

// Rows of a padded pool (row r at pptr[r], length len[r]); owners u in
// [lo, hi).  Pass 1 accumulates, per owner, its non-empty suffix segments
// and their total length in one 64-bit atomic (count << 40 | length sum);
// pass 2 scatters the segments with a 32-bit cursor.
static constexpr int kCntShift = 40;
// kG lanes per row (8 for short lists, 32 otherwise): a lane walks ids
// jl, jl + kG, ... of its row and stops at the first id >= hi (rows ascend,
// so its later ids are not owned either).
template <int kG>
__global__ void k_sh_idx_count(const int64_t* __restrict__ pptr, const int32_t* __restrict__ len, int64_t nrow,
                               const int32_t* __restrict__ pool, int64_t lo, int64_t hi, unsigned long long* acc) {
  const int jl = threadIdx.x % kG;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / kG;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG; r < nrow; r += ng) {
    const int64_t p = pptr[r], d = len[r];
    for (int64_t i = jl; i + 1 < d; i += kG) {
      const int32_t u = pool[p + i];
      if (u >= hi) break;
      if (u >= lo) atomicAdd(&acc[u - lo], (1ull << kCntShift) + (unsigned long long)(d - i - 1));
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

// cursor[x] = rev_indptr[x]: the emit pass then takes a segment's slot with
// one atomic (segments < 2^31: they index an int32 pool)
__global__ void k_sh_idx_cursor(const int64_t* __restrict__ rev_indptr, int64_t nx, int32_t* cursor) {
  GRID_STRIDE(x, nx) cursor[x] = (int32_t)rev_indptr[x];
}

template <int kG>
__global__ void k_sh_idx_emit(const int64_t* __restrict__ pptr, const int32_t* __restrict__ len, int64_t nrow,
                              const int32_t* __restrict__ pool, int64_t lo, int64_t hi,
                              const int64_t* __restrict__ rev_indptr, int32_t* cursor, int2* rev_seg) {
  const int jl = threadIdx.x % kG;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / kG;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG; r < nrow; r += ng) {
    const int64_t p = pptr[r], d = len[r];
    for (int64_t i = jl; i + 1 < d; i += kG) {
      const int32_t u = pool[p + i];
      if (u >= hi) break;
      if (u >= lo) {
        const int64_t x = u - lo;
        const int64_t slot = atomicAdd(&cursor[x], 1);
#if TCB_DEBUG
        assert(slot >= rev_indptr[x] && slot < rev_indptr[x + 1]);
#endif
        rev_seg[slot] = make_int2((int)(p + i + 1), (int)(p + d));
      }
    }
  }
}

// lanes per row of the receive-index kernels for rows of this mean padded
// length (pool_words 0: unknown)
static int idx_group(int64_t nrow, int64_t pool_words) {
  return (nrow > 0 && pool_words > 0 && pool_words / nrow < 96) ? 8 : 32;
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
                                                 reinterpret_cast<unsigned long long*>(keys_out), P);
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
                                                 reinterpret_cast<int2*>(out), P);
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
    sort_rows(sc, indptr, nrow, k, unsorted, indices, s);  // the length-classed row sorts of tc_build_graph
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

int tc_shard_send_plan_len(int64_t nrow, int32_t P, int64_t* len_host) {
  return guarded([&] {
    TC_REQUIRE(len_host != nullptr && P >= 1 && nrow >= 0, TC_EINVAL, "bad send plan query");
    *len_host = 3 * (int64_t)P + 2 * (int64_t)P * send_blocks(nrow) * kSendWarps;
  });
}

int tc_shard_send_sizes(const int64_t* indptr, const int32_t* indices, int64_t nrow, const int64_t* pool_indptr,
                        const int64_t* bounds, int32_t P, int32_t rank, int64_t* sizes_dev, int64_t* sizes_host,
                        tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(P >= 1 && P <= kEmitMaxP, TC_EINVAL, "the surrogate send supports P <= 32 ranks");
    TC_REQUIRE(rank >= 0 && rank < P, TC_EINVAL, "rank out of range");
    const int nblk = send_blocks(nrow);
    const int64_t nunit = (int64_t)nblk * kSendWarps;
    TC_CUDA(cudaMemsetAsync(sizes_dev, 0, (3 * (size_t)P + 2 * (size_t)P * nunit) * sizeof(int64_t), s));
    if (nrow > 0 && rank + 1 < P) {
      long long* tot = reinterpret_cast<long long*>(sizes_dev);
      long long* unit_l = tot + 3 * P;
      long long* unit_w = unit_l + (int64_t)P * nunit;
      k_sh_send_count<<<nblk, kBlk, 0, s>>>(indptr, indices, nrow, pool_indptr, bounds, P, rank,
                                             send_group(P, rank), tot, unit_l, unit_w);
      check_launch();
      k_sh_send_prefix<<<1, 32 * P, 0, s>>>(tot, P, nunit, unit_l, unit_w);
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
    TC_REQUIRE(P >= 1 && P <= kEmitMaxP, TC_EINVAL, "the surrogate send supports P <= 32 ranks");
    TC_REQUIRE(((uintptr_t)pool & 15) == 0 && ((uintptr_t)out_ids & 15) == 0, TC_EINVAL,
               "pool and out_ids must be 16-byte aligned");
    if (nrow <= 0 || rank + 1 >= P) return;
    const int nblk = send_blocks(nrow);
    const long long* base_l = reinterpret_cast<const long long*>(sizes_dev) + 3 * P;
    const long long* base_w = base_l + (int64_t)P * nblk * kSendWarps;
    k_sh_send_emit<<<nblk, kBlk, 0, s>>>(indptr, indices, nrow, pool_indptr, reinterpret_cast<const int4*>(pool),
                                          bounds, P, rank, send_group(P, rank), base_l, base_w, out_len,
                                          reinterpret_cast<int4*>(out_ids));
    check_launch();
  });
}

int tc_shard_index(const int32_t* row_len, int64_t nrow, const int32_t* pool, int64_t pool_words, int64_t lo,
                   int64_t hi, const int64_t* tab_indptr, int64_t* pool_indptr, int64_t* rev_indptr,
                   int32_t* rev_seg, int64_t* rev_cost, int64_t* nseg_host, tc_stream_t stream) {
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
    const int G = idx_group(nrow, pool_words);
    const int grid = grid_for(std::max<int64_t>(nrow, 1) * G, kBlk, sm_count() * 16);
    if (nrow > 0) {
      if (G == 8) k_sh_idx_count<8><<<grid, kBlk, 0, s>>>(pool_indptr, row_len, nrow, pool, lo, hi, acc);
      else k_sh_idx_count<32><<<grid, kBlk, 0, s>>>(pool_indptr, row_len, nrow, pool, lo, hi, acc);
      check_launch();
    }
    int64_t* cnt = sc.alloc<int64_t>(nx + 1);
    int64_t* cost = sc.alloc<int64_t>(nx + 1);
    k_sh_idx_rows<<<grid_for(nx + 1, kBlk), kBlk, 0, s>>>(acc, tab_indptr, nx, cnt, cost);
    check_launch();
    ex_sum(sc, cnt, rev_indptr, nx + 1, s);
    ex_sum(sc, cost, rev_cost, nx + 1, s);
    int32_t* cur = sc.alloc<int32_t>(nx + 1);
    k_sh_idx_cursor<<<grid_for(nx + 1, kBlk), kBlk, 0, s>>>(rev_indptr, nx, cur);
    check_launch();
    if (nrow > 0) {
      if (G == 8)
        k_sh_idx_emit<8><<<grid, kBlk, 0, s>>>(pool_indptr, row_len, nrow, pool, lo, hi, rev_indptr, cur,
                                               reinterpret_cast<int2*>(rev_seg));
      else
        k_sh_idx_emit<32><<<grid, kBlk, 0, s>>>(pool_indptr, row_len, nrow, pool, lo, hi, rev_indptr, cur,
                                                reinterpret_cast<int2*>(rev_seg));
      check_launch();
    }
    if (nseg_host) *nseg_host = scalar_of(rev_indptr + nx, s);
  });
}

// The scatter pass of tc_shard_index alone, for rows whose owner offsets
// (rev_indptr) are already known: a round of the exchange delivers the same
// lists at every count of a partitioned graph, so the per-owner counts, the
// cost prefix and the engine plan built from them are kept and only the
// segments are scattered again.
int tc_shard_index_emit(const int32_t* row_len, int64_t nrow, const int32_t* pool, int64_t pool_words, int64_t lo,
                        int64_t hi, const int64_t* rev_indptr, int64_t* pool_indptr, int32_t* rev_seg,
                        tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(lo >= 0 && lo <= hi, TC_EINVAL, "bad owner range");
    const int64_t nx = hi - lo;
    Scratch sc(s);
    int64_t* sz = sc.alloc<int64_t>(nrow + 1);
    k_sh_len_sizes<<<grid_for(nrow + 1, kBlk), kBlk, 0, s>>>(row_len, nrow, sz);
    check_launch();
    ex_sum(sc, sz, pool_indptr, nrow + 1, s);
    int32_t* cur = sc.alloc<int32_t>(nx + 1);
    k_sh_idx_cursor<<<grid_for(nx + 1, kBlk), kBlk, 0, s>>>(rev_indptr, nx, cur);
    check_launch();
    if (nrow > 0) {
      const int G = idx_group(nrow, pool_words);
      const int grid = grid_for(nrow * G, kBlk, sm_count() * 16);
      if (G == 8)
        k_sh_idx_emit<8><<<grid, kBlk, 0, s>>>(pool_indptr, row_len, nrow, pool, lo, hi, rev_indptr, cur,
                                               reinterpret_cast<int2*>(rev_seg));
      else
        k_sh_idx_emit<32><<<grid, kBlk, 0, s>>>(pool_indptr, row_len, nrow, pool, lo, hi, rev_indptr, cur,
                                                reinterpret_cast<int2*>(rev_seg));
      check_launch();
    }
  });
}

}  // extern "C"

// count.cu -- the intersection engine (sm_100a).
//
// Work model.  Every triangle v < u < w (canonical degree order) is found by
// probing list elements into a shared-memory table:
//
//   pull ("middle vertex", tc_count_middle / tc_count_owners): owner = u.
//        Table = N^_u; segments = for each predecessor v of u, the suffix of
//        N^_v after u (rev_seg).  Probes = sum_v C(d^_v, 2), 2-5x fewer than
//        the merge model's W -- the headline path.
//   push ("lowest vertex", tc_count_lowest): owner = v.  Table = N^_v;
//        segments = N^_u for every u in N^_v.  This is exactly
//        count_node_range(v0, v1) (_kernels.py:40-52) with per-bucket
//        partials, used for count_task / count_dynamic.
//
// Three tiers by table size d (the shape bucketing of SURVEY.md §7 step 6);
// each tier runs over a compacted list of its own owners:
//   small  (d <= 128, k_small): a warp owns a 4 KB one-bit hashed filter
//          and holds the owner's list in registers (4 ids per lane): the
//          rare filter hits are verified with one shuffle + one ballot, no
//          bucket table is built; three windows per step are loaded
//          straight into registers.  Wide form (k_small<.., 8>: d <= 256,
//          8 ids per lane, two filter bits per id): the plan cuts the tiers
//          at 256 instead of 128 when the owners with 128 < d <= 256 carry a
//          third of the engine's cost (dense graphs: cfg 5 50.6 -> 45.6 ms);
//   mid    (d <= 512): 8 KB slices (32K-bit two-bit filter + 2^8 buckets),
//          4 warps per block, windows software-pipelined in registers;
//   block  (d  > 512): a 512-thread block stages up to 4096 ids (256K-bit
//          filter + 2^11 buckets) and all 16 warps stream the owner's
//          segments -- the hubs of Chung-Lu / R-MAT; beyond 4096 ids the
//          probes use binary search in global memory (L1/L2 resident).
// Tables whose ids span less than the slice's bit count become exact
// direct-mapped bitmaps (no hashing, no verification): every block-tier
// owner of the benchmark graphs.
// Segment streaming: a warp takes up to 32 segments, compacts the non-empty
// ones, and flattens the 16-byte chunks they touch with a warp scan; lane j
// of a window loads chunk base+j as one int4 (4 list ids), resolving its
// segment from a shared bitmap of segment starts (popc) or, for groups
// wider than the bitmap, one ballot + one redux.or + popc; the block tier
// on padded pools carries each lane's segment from window to window instead
// (stream_group_inc).  A probe is one filter LDS and a few ALU ops,
// branch-free over the 4 ids; only filter hits are verified (inline in the
// warp tiers, queued and verified in bulk in the block tier).  On the
// row-padded pool (tc_build_graph, the sharded ranks' pools) no tier masks
// ids: whatever a chunk holds outside its segment is <= u or INT32_MAX and
// cannot be in N^_u.
//
// Load balance (the paper's dynamic load balancing, PAPER.md:788-822,
// dynamic_lb.py:68-109, restated for warps): each tier splits its owners'
// cost prefix into chunks whose boundaries fall INSIDE an owner's segment
// list (so a hub never pins a warp), ending with the paper's geometrically
// shrinking tasks of (remaining / workers); workers pull chunk indices from
// one global atomic counter (the coordinator's queue).
#include <cub/cub.cuh>
#include <mutex>

#include "common.cuh"

namespace tcb {

#ifndef TCB_MID_PAD_MODE
#define TCB_MID_PAD_MODE 2  // padded pools in the mid tier: 0 id masks as for any pool, 2 no masks
#endif
#ifndef TCB_BIG_INC_PIPE
#define TCB_BIG_INC_PIPE 0
#endif
// chunk schedule of the warp tiers (k_plan, mode 1): uniform chunks per worker
// over the first TCB_PLAN_HALF of the cost, smallest chunk = cost / (MINDIV * workers)
#ifndef TCB_PLAN_FIRST
#define TCB_PLAN_FIRST 6
#endif
#ifndef TCB_PLAN_HALF
#define TCB_PLAN_HALF 0.75
#endif
#ifndef TCB_PLAN_MINDIV
#define TCB_PLAN_MINDIV 256.0  // 32 -> 256: finer tail chunks, cfg 2 1.68 -> 1.61 ms, cfg 5 small tier 11.95 -> 11.47
#endif
#ifndef TCB_PLAN_SEG_MINDIV
#define TCB_PLAN_SEG_MINDIV 32.0  // the block tier's plan (k_plan_seg)
#endif
#ifndef TCB_PLAN_NMAX
#define TCB_PLAN_NMAX 16  // chunk slots per worker (first + geometric + tail chunks must fit)
#endif
#ifndef TCB_MINBLOCKS
#define TCB_MINBLOCKS 5
#endif
#ifndef TCB_PF_NEXT
#define TCB_PF_NEXT 0
#endif
#ifndef TCB_BIG_CLAIM
#define TCB_BIG_CLAIM 16
#endif
static constexpr int kBigClaim = TCB_BIG_CLAIM;  // block tier: segments per dynamic claim (<= 32)
#ifndef TCB_BIG_STAGES
#define TCB_BIG_STAGES 0
#endif
static constexpr int kBigStages = TCB_BIG_STAGES;  // block tier, exact tables: cp.async ring stages per warp
#ifndef TCB_BIG_FB
#define TCB_BIG_FB 1
#endif
#ifndef TCB_BIG_SB
#define TCB_BIG_SB false
#endif
#ifndef TCB_BIG_PIPE
#define TCB_BIG_PIPE 0
#endif
#ifndef TCB_MID_PIPE
#define TCB_MID_PIPE 1
#endif
#ifndef TCB_SEGPTR
#define TCB_SEGPTR 1
#endif
#ifndef TCB_WIPE
#define TCB_WIPE 1
#endif
#ifndef TCB_WINDOWS
#define TCB_WINDOWS 2
#endif
#ifndef TCB_SMALL_WARPS
#define TCB_SMALL_WARPS 7  // x 6 blocks = 42 warps per SM at 40 registers (8 x 5 = 40 warps at 48: cfg 2 1.63 -> 1.60 ms)
#endif
static constexpr int kWarps = TCB_SMALL_WARPS;  // warps per block (small tier)
static constexpr int kWin = TCB_WINDOWS;  // 32-chunk windows in flight per warp
static constexpr int kThreads = kWarps * 32;
#ifndef TCB_SMALL_CAP
#define TCB_SMALL_CAP 128
#define TCB_SMALL_LW 8
#define TCB_SMALL_LB 6
#endif
static constexpr int kTabCap = TCB_SMALL_CAP;  // small tier: ids per table
static constexpr int kLwWarp = TCB_SMALL_LW;   // small tier filter: 2^8 words = 8K bits (1 KB)
static constexpr int kLbWarp = TCB_SMALL_LB;   // small tier buckets: 2^6 x 4 ids (1 KB), load <= 1/2
static constexpr int kMidCap = 512;       // mid tier: ids per table
static constexpr int kLwMid = 10;         // mid tier filter: 2^10 words = 32K bits (4 KB)
static constexpr int kLbMid = 8;          // mid tier buckets: 2^8 x 4 ids (4 KB), load <= 1/2
static constexpr int kMidWarps = 4;       // mid tier: warps per block (8 KB private slices)
static constexpr int kBigThreads = 512;   // block tier
static constexpr int kBigWarps = kBigThreads / 32;
#ifndef TCB_BIG_CAP
#define TCB_BIG_CAP 4096
#endif
#ifndef TCB_BIG_LB
#define TCB_BIG_LB 11
#endif
#ifndef TCB_POS_CAP
#define TCB_POS_CAP 512
#endif
#ifndef TCB_BIG_MINB
#define TCB_BIG_MINB 2
#endif
static constexpr int kBigCap = TCB_BIG_CAP;  // block tier: ids per staged table
static constexpr int kLwBig = 13;         // block tier filter: 2^13 words = 256K bits (32 KB)
static constexpr int kLbBig = TCB_BIG_LB;  // block tier buckets: 2^11 x 4 ids (32 KB), load <= 1/2
static constexpr int kPosCap = TCB_POS_CAP;  // block tier: per-warp queue of filter hits
#ifndef TCB_BIG_WINDOWS
#define TCB_BIG_WINDOWS 3  // block tier: windows in flight per warp (2 -> 3: cfg 4 block tier 114.0 -> 106.4 ms)
#endif
static constexpr int kBigWin = TCB_BIG_WINDOWS;
#ifndef TCB_BIG_WINDOWS_EXACT
#define TCB_BIG_WINDOWS_EXACT 4  // the exact-only form (no hit queue)
#endif
#ifndef TCB_BIG_EXACT_PIPE
#define TCB_BIG_EXACT_PIPE true
#endif
static constexpr int kBigWinExact = TCB_BIG_WINDOWS_EXACT;
static constexpr int kPosDrain = kPosCap - 128 * kBigWin;  // drain before a step could overflow
static_assert(kPosDrain > 0, "the block tier's hit queue must hold one step of hits");
#ifndef TCB_SBWORDS
#define TCB_SBWORDS 64
#endif
static constexpr int kSbWords = TCB_SBWORDS;  // per-warp bitmap of segment starts: groups of <= 32 kSbWords chunks
static constexpr int kSegTab = 32 + kSbWords / 4;  // int4 per warp: 32 segment entries + the start bitmap

static_assert(kBigStages == 0 || (1 << kLbBig) >= kBigWarps * kBigStages * 32,
              "block-tier rings live in the bucket area");
// Block-tier shared memory: filter / exact bitmap, bucket table, per-warp hit
// queues, per-warp segment tables.  When every owner of the tier has an
// exact bitmap (all of them on the benchmark graphs) the kernel is launched
// in its exact-only form without buckets and queues: 44 KB instead of 108 KB
// per block leaves the SM 168 KB of L1 instead of 40 KB (cfg 4 block tier
// 107.8 -> 102.5 ms).
static constexpr size_t kBigTabBytesFull = (sizeof(uint32_t) << kLwBig) + (sizeof(int4) << kLbBig) +
                                           sizeof(int32_t) * kPosCap * kBigWarps;
static constexpr size_t kBigTabBytesExact = sizeof(uint32_t) << kLwBig;
static constexpr size_t kBigSegBytes = sizeof(int4) * kSegTab * kBigWarps;
static constexpr size_t kBigSmem = kBigTabBytesFull + kBigSegBytes;
static constexpr size_t kBigSmemExact = kBigTabBytesExact + kBigSegBytes;
static constexpr int kSegCost = 2;        // must match build.cu
static constexpr int kTabCost = 16;
static constexpr int32_t kEmpty = -1;

// Verification kinds of a staged table (see probe4).
enum : int { kGlobal = 0, kInline = 1, kBuckets = 2, kExact = 3 };

template <int kLb, int kLw>
struct WarpSliceT {
  uint32_t bm[1 << kLw];
  int4 bkt[1 << kLb];
};

// --------------------------------------------------------------- segments

// Segment coordinates are int32: pools hold fewer than 2^31 ids (m < 2^31,
// enforced at build; owner_segments checks its pool).
struct PullSegs {  // rev_seg int32 pairs (start, end) into the pool
  const int2* seg;
  __device__ __forceinline__ void get(int r, int& s, int& e) const {
    const int2 x = __ldg(&seg[r]);
    s = x.x;
    e = x.y;
  }
};

struct PushSegs {  // forward edge e of v -> N^_u, u = indices[e]
  const int64_t* indptr;
  const int32_t* indices;
  __device__ __forceinline__ void get(int r, int& s, int& e) const {
    int32_t u = __ldg(&indices[r]);
    s = (int)__ldg(&indptr[u]);
    e = (int)__ldg(&indptr[u + 1]);
  }
};

// Per-owner tables.  Every staged table has a hashed filter in front (2^lw
// words, h = id * golden, word = h >> (32 - lw), bit h & 31, and in the warp
// tiers a second bit (h >> 5) & 31 in the same word): a probe is one LDS.32
// and a few ALU ops, and only filter hits (true hits plus the false
// positives: ~d/2^(lw+5) with one bit, ~20x fewer with two) are verified:
//   kInline  (warp tiers): inline lookup in a bucketized hash table whose
//            maximum displacement is recorded at build time, so a lookup is a
//            warp-uniform handful of LDS.128 (usually one), no search loop;
//   kBuckets (block tier): hits are queued per warp and verified in bulk
//            against a bucketized hash table (2^lb buckets of 4 ids,
//            bucket = h >> (32 - lb), overflow to the next bucket, load
//            <= 1/2): one LDS.128 per hit -- for hubs, where hit rates
//            reach ~40% (R-MAT) and a 12-step binary search per hit would
//            dominate;
//   kGlobal  (beyond the block cap): binary search in global memory.
__device__ __forceinline__ uint32_t tab_hash(uint32_t w) { return w * 0x9E3779B1u; }

__device__ __forceinline__ int tab_lb(int64_t d) {  // log2 buckets: smallest 2^lb >= d/2, >= 8
  int64_t want = (d + 1) / 2;
  int lb = 32 - __clz((int)(want > 2 ? want - 1 : 1));
  return max(lb, 3);
}

// One bit per id: word = top lw hash bits, bit = the low 5 (id * odd keeps
// the id's low 5 bits a permutation, independent enough of the top bits for
// a filter); a probe then takes the bit with one funnel shift by h itself.
// (A blocked Bloom variant with two bits per id in the same word was
// measured: -4% on cfg 2, +3% on cfg 5 -- not worth the extra ALU.)
template <int kLw>
__device__ __forceinline__ uint32_t filt_mask(uint32_t h) {
  return 1u << (h & 31);
}

// kFb = 2: a second bit per id in the same word (hash bits 5..9): a blocked
// Bloom filter with ~20x fewer false positives at mid-tier loads.
template <int kLw, int kFb = 1>
__device__ __forceinline__ void filt_insert(uint32_t* bm, int32_t w) {
  const uint32_t h = tab_hash((uint32_t)w);
  atomicOr(&bm[h >> (32 - kLw)], filt_mask<kLw>(h) | (kFb == 2 ? 1u << ((h >> 5) & 31) : 0u));
}

template <int kLw>
__device__ __forceinline__ void filt_clear(uint32_t* bm, int32_t w) {
  bm[tab_hash((uint32_t)w) >> (32 - kLw)] = 0;
}

__device__ __forceinline__ bool bkt_has(int4 q, int32_t x) { return (q.x == x) | (q.y == x) | (q.z == x) | (q.w == x); }

// Inserts w; returns its displacement (buckets past its home bucket).
__device__ __forceinline__ int bkt_insert(int4* bkt, int lb, int32_t w) {
  int32_t* slots = reinterpret_cast<int32_t*>(bkt);
  const uint32_t mask = (1u << lb) - 1;
  uint32_t b = tab_hash((uint32_t)w) >> (32 - lb);
  for (int i = 0;; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (atomicCAS(&slots[b * 4 + k], kEmpty, w) == kEmpty) return i;
    b = (b + 1) & mask;
  }
}

// Membership with a known maximum displacement (warp-uniform per table):
// a fixed number of bucket reads, no data-dependent loop.
__device__ __forceinline__ bool bkt_find(const int4* bkt, int lb, int dmax, int32_t x) {
  const uint32_t mask = (1u << lb) - 1;
  const uint32_t b = tab_hash((uint32_t)x) >> (32 - lb);
  bool f = bkt_has(bkt[b], x);
  for (int i = 1; i <= dmax; ++i) f |= bkt_has(bkt[(b + i) & mask], x);
  return f;
}


__device__ __forceinline__ bool bkt_lookup(const int4* bkt, int lb, int32_t x) {
  const uint32_t mask = (1u << lb) - 1;
  uint32_t b = tab_hash((uint32_t)x) >> (32 - lb);
  for (;;) {
    int4 q = bkt[b];
    if (bkt_has(q, x)) return true;
    if (q.w == kEmpty) return false;
    b = (b + 1) & mask;
  }
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

struct Table {
  const uint32_t* bm;   // filter (kInline, kBuckets)
  const int32_t* tab;   // global list (kGlobal)
  const int4* bkt;      // buckets (kInline, kBuckets)
  int32_t* pos;         // per-warp hit queue (kBuckets)
  int64_t d;
  int lb;
  int32_t tmin, tmax;
  int dmax;             // max bucket displacement (kInline)
  uint32_t span;        // kExact: bit (id - tmin) of bm, ids in [tmin, tmin + span)
};

// Verify the queued filter hits of this warp (kBuckets) and empty the queue.
__device__ __forceinline__ void drain(const Table& t, int& npos, int lane, uint32_t& cnt) {
  __syncwarp();
  for (int i = lane; i < npos; i += 32) cnt += bkt_lookup(t.bkt, t.lb, t.pos[i]);
  __syncwarp();
  npos = 0;
}

// Filter the 4 ids of v; `vmask` marks the ids inside the chunk's segment
// (ids outside it belong to neighbouring lists and must not be counted).
// Only filter hits are verified; no range check is needed for exactness.
template <int kKind, int kLw, int kCap = 1>  // kCap: filter bits per id (kFb)
__device__ __forceinline__ void probe4(const Table& t, int4 v, uint32_t vmask, int lane, int& npos, uint32_t& cnt) {
  int32_t xs[4] = {v.x, v.y, v.z, v.w};
  if (kKind == kGlobal) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((vmask >> k) & 1u) && xs[k] >= t.tmin && xs[k] <= t.tmax) cnt += bsearch_gmem(t.tab, t.d, xs[k]);
    return;
  }
  if (kKind == kExact) {  // direct-mapped exact bitmap: no hashing, no verification
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // ids outside [tmin, tmin + span) clamp to offset span, whose bit is
      // never set (span < 32 << lw keeps that word inside the bitmap)
      const uint32_t off = min((uint32_t)(xs[k] - t.tmin), t.span);
      const uint32_t wd = t.bm[off >> 5];
      m |= __funnelshift_r(wd, wd, off - k) & (1u << k);  // bit (off mod 32) rotated to position k
    }
    cnt += __popc(m & vmask);
    return;
  }
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t h = tab_hash((uint32_t)xs[k]);
    const uint32_t wd = t.bm[h >> (32 - kLw)];
    // rotate bit (h mod 32) of the word to position k (amount taken mod 32)
    uint32_t b = __funnelshift_r(wd, wd, h - k);
    if (kCap == 2) b &= __funnelshift_r(wd, wd, (h >> 5) - k);
    m |= b & (1u << k);
  }
  m &= vmask;
  if (kKind == kInline) {
    if (m) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((m >> k) & 1u) cnt += bkt_find(t.bkt, t.lb, t.dmax, xs[k]);
    }
    return;
  }
  const unsigned FULL = 0xffffffffu;  // kBuckets: warp-aggregated append
  if (__any_sync(FULL, m != 0)) {
    const int c = __popc(m);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    int at = npos + incl - c;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if ((m >> k) & 1u) t.pos[at++] = xs[k];
    npos += __shfl_sync(FULL, incl, 31);
  }
}

// Probes of one group of <= 32 compacted segments.  The group is flattened
// over the 16-byte chunks its segments touch: lane j of window k loads
// chunk base+32k+j as one int4 and probes the ids of it inside its segment.
// Segment s covers chunks [excl_s, endx_s) of the flat space; chunk f of it
// is pool4[delta_s + f]; `edge_s` packs (first-chunk offset | last-chunk
// count << 2).
// Resolves and loads the kW windows starting at chunk `base` (see
// probe_group).
template <int kW, bool kMayFast, bool kNoMask = false>
__device__ __forceinline__ void load_windows(const int4* __restrict__ pool4, bool lane_seg, int excl,
                                             const int4* __restrict__ segtab, const uint32_t* __restrict__ sbits,
                                             int total, int lane, bool fast_rt, int base, int& cbase, int4 (&v)[kW],
                                             uint32_t (&vm)[kW]) {
  const bool fast = kMayFast && fast_rt;
  const unsigned FULL = 0xffffffffu;
#pragma unroll
  for (int k = 0; k < kW; ++k) {
    const int b = base + 32 * k;
    vm[k] = 0;
    v[k] = make_int4(0, 0, 0, 0);
    if (b < total) {
      int sj;  // segment of chunk b + lane = (segments starting at or before it) - 1
      if (fast) {
        const unsigned starts = sbits[b >> 5];
        sj = cbase + __popc(starts & ((2u << lane) - 1u)) - 1;
        cbase += __popc(starts);
      } else {
        const unsigned cov = __ballot_sync(FULL, lane_seg && excl <= b);
        const unsigned bit = (lane_seg && excl > b && excl < b + 32) ? (1u << (excl - b)) : 0u;
        const unsigned starts = __reduce_or_sync(FULL, bit);
        sj = __popc(cov) - 1 + __popc(starts & ((2u << lane) - 1u));
      }
      const int f = b + lane;
      if (f < total) {
#if TCB_DEBUG
        assert(sj >= 0 && sj < 32 && f >= segtab[sj].z && f <= (segtab[sj].w >> 8));
#endif
#if TCB_SEGPTR
        const int4 q = segtab[sj];  // (&pool4[delta] lo, hi, excl, (endx - 1) << 8 | last mask << 4 | first mask)
        const int4* p = reinterpret_cast<const int4*>(((unsigned long long)(unsigned)q.y << 32) | (unsigned)q.x);
        v[k] = __ldg(p + f);
#else
        const int4 q = segtab[sj];  // (delta, -, excl, (endx - 1) << 8 | last mask << 4 | first mask)
        v[k] = __ldg(&pool4[q.x + f]);
#endif
        uint32_t mk = 0xFu;
        if (!kNoMask) {  // row-padded pools need no id masks (see stream_group_inc)
          if (f == q.z) mk &= (uint32_t)q.w & 0xFu;
          if (f == (q.w >> 8)) mk &= ((uint32_t)q.w >> 4) & 0xFu;
        }
        vm[k] = mk;
      }
    }
  }
}

// Probes of one group of <= 32 compacted segments.  The group is flattened
// over the 16-byte chunks its segments touch: lane j of window k loads
// chunk base+32k+j as one int4 and probes the ids of it inside its segment.
// Segment s covers chunks [excl_s, endx_s) of the flat space; chunk f of it
// is pool4[delta_s + f]; `edge_s` packs (first-chunk offset | last-chunk
// count << 2).  Software-pipelined: the next kW windows are resolved and
// their loads issued before the current ones are probed (kPipe), so up to
// 2 kW loads per warp are in flight across the probe work.  Measured: the
// mid tier gains (cfg 5 24.2 -> 20.6 ms), the small tier loses (cfg 2 2.49 ->
// 2.61 ms: registers), so only the mid tier pipelines.
template <int kKind, int kLw, int kCap, int kW, bool kFast, bool kPipe, bool kNoMask = false>
__device__ __forceinline__ void probe_loop(const int4* __restrict__ pool4, const Table& t, int nseg, int excl,
                                           const int4* __restrict__ segtab, const uint32_t* __restrict__ sbits,
                                           int total, int lane, int& npos, uint32_t& cnt, bool fast = kFast) {
  const bool lane_seg = lane < nseg;
  int cbase = 0;  // fast path: segments starting before the window
  int4 v[kW];
  uint32_t vm[kW];
  load_windows<kW, kFast, kNoMask>(pool4, lane_seg, excl, segtab, sbits, total, lane, fast, 0, cbase, v, vm);
  for (int base = 0; base < total; base += 32 * kW) {
    if (kPipe) {
      int4 nv[kW];
      uint32_t nvm[kW];
      const int nb = base + 32 * kW;
      if (nb < total) {
        load_windows<kW, kFast, kNoMask>(pool4, lane_seg, excl, segtab, sbits, total, lane, fast, nb, cbase, nv, nvm);
      } else {
#pragma unroll
        for (int k = 0; k < kW; ++k) {
          nvm[k] = 0;
          nv[k] = make_int4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int k = 0; k < kW; ++k) probe4<kKind, kLw, kCap>(t, v[k], vm[k], lane, npos, cnt);
      if (kKind == kBuckets && npos > kPosDrain) drain(t, npos, lane, cnt);
#pragma unroll
      for (int k = 0; k < kW; ++k) {
        v[k] = nv[k];
        vm[k] = nvm[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < kW; ++k) probe4<kKind, kLw, kCap>(t, v[k], vm[k], lane, npos, cnt);
      if (kKind == kBuckets && npos > kPosDrain) drain(t, npos, lane, cnt);
      if (base + 32 * kW < total)
        load_windows<kW, kFast, kNoMask>(pool4, lane_seg, excl, segtab, sbits, total, lane, fast, base + 32 * kW, cbase, v,
                                 vm);
    }
  }
}

// Asynchronous window staging (tiny tier): lane j of window b copies chunk
// b + j into a shared-memory ring slot with cp.async (16 B, L1 bypassed)
// and later probes it from there, so kS - 1 windows per warp are in flight
// without holding their data in registers.  Each lane reads back only what
// it copied itself, so the per-thread cp.async.wait_group is the only
// synchronisation.  Returns the window's id mask for this lane (the 4-bit
// masks of the in-flight windows ride in one register).
template <bool kMayFast>
__device__ __forceinline__ uint32_t issue_window(bool lane_seg, int excl, const int4* __restrict__ segtab,
                                                 const uint32_t* __restrict__ sbits, int total, int lane,
                                                 bool fast_rt, int b, int& cbase, int4* dst) {
  const unsigned FULL = 0xffffffffu;
  const bool fast = kMayFast && fast_rt;
  int sj;
  if (fast) {
    const unsigned starts = sbits[b >> 5];
    sj = cbase + __popc(starts & ((2u << lane) - 1u)) - 1;
    cbase += __popc(starts);
  } else {
    const unsigned cov = __ballot_sync(FULL, lane_seg && excl <= b);
    const unsigned bit = (lane_seg && excl > b && excl < b + 32) ? (1u << (excl - b)) : 0u;
    const unsigned starts = __reduce_or_sync(FULL, bit);
    sj = __popc(cov) - 1 + __popc(starts & ((2u << lane) - 1u));
  }
  const int f = b + lane;
  if (f >= total) return 0u;
  const int4 q = segtab[sj];
  const int4* p = reinterpret_cast<const int4*>(((unsigned long long)(unsigned)q.y << 32) | (unsigned)q.x);
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(p + f) : "memory");
  uint32_t mk = 0xFu;
  if (f == q.z) mk &= (uint32_t)q.w & 0xFu;
  if (f == (q.w >> 8)) mk &= ((uint32_t)q.w >> 4) & 0xFu;
  return mk;
}

template <int kN>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(kN) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int kKind, int kLw, int kCap, int kS, bool kMayFast>
__device__ __forceinline__ void probe_loop_async(const Table& t, int nseg, int excl, const int4* __restrict__ segtab,
                                                 const uint32_t* __restrict__ sbits, int total, int lane, int& npos,
                                                 uint32_t& cnt, bool fast, int4* ring) {
  static_assert(kS >= 2 && kS <= 8 && (kS & (kS - 1)) == 0, "ring stages: 2, 4 or 8");
  const bool lane_seg = lane < nseg;
  const int nwin = (total + 31) >> 5;
  int cbase = 0;
  uint32_t mring = 0;
#pragma unroll
  for (int i = 0; i < kS - 1; ++i) {
    if (i < nwin) {
      const uint32_t m = issue_window<kMayFast>(lane_seg, excl, segtab, sbits, total, lane, fast, 32 * i, cbase,
                                                ring + i * 32 + lane);
      mring |= m << (4 * i);
    }
    cp_async_commit();
  }
  for (int w = 0; w < nwin; ++w) {
    const int wi = w + kS - 1;
    if (wi < nwin) {
      const int sl = wi & (kS - 1);
      const uint32_t m = issue_window<kMayFast>(lane_seg, excl, segtab, sbits, total, lane, fast, 32 * wi, cbase,
                                                ring + sl * 32 + lane);
      mring = (mring & ~(0xFu << (4 * sl))) | (m << (4 * sl));
    }
    cp_async_commit();
    cp_async_wait<kS - 1>();
    const int sl = w & (kS - 1);
    const int4 v = ring[sl * 32 + lane];
    probe4<kKind, kLw, kCap>(t, v, (mring >> (4 * sl)) & 0xFu, lane, npos, cnt);
    if (kKind == kBuckets && npos > kPosDrain) drain(t, npos, lane, cnt);
  }
}

// kSbW: words of the warp's start bitmap (groups of <= 32 kSbW chunks take
// the bitmap path).
template <int kKind, int kLw, int kCap = 1, int kW = kWin, bool kSb = true, bool kPipe = false, int kS = 0,
          int kSbW = kSbWords, bool kNoMask = false>
__device__ __forceinline__ void probe_group(const int4* __restrict__ pool4, const Table& t, int nseg, int excl,
                                            const int4* __restrict__ segtab, const uint32_t* __restrict__ sbits,
                                            int total, int lane, int& npos, uint32_t& cnt, int4* ring = nullptr) {
  const bool fast = kSb && total <= 32 * kSbW;  // warp-uniform
  if (kS > 0) {
    probe_loop_async<kKind, kLw, kCap, (kS > 0 ? kS : 2), kSb>(t, nseg, excl, segtab, sbits, total, lane, npos, cnt,
                                                              fast, ring);
    return;
  }
  probe_loop<kKind, kLw, kCap, kW, kSb, kPipe, kNoMask>(pool4, t, nseg, excl, segtab, sbits, total, lane, npos, cnt,
                                                       fast);
}

// One warp streams segments [g0, g1) (g1 - g0 <= 32) of the current owner;
// segtab is the warp's shared-memory table (kSegTab int4): 32 segment
// entries followed by the bitmap of segment starts over the group's chunks.
// kSb: use the start bitmap (warp tiers; hub groups of the block tier are
// mostly longer than 1024 chunks and keep the ballot/redux resolution).
template <int kKind, int kLw, class Segs, int kCap = 1, int kW = kWin, bool kSb = true, bool kPipe = false,
          int kS = 0, int kSbW = kSbWords, bool kNoMask = false>
__device__ __forceinline__ void stream_group(const Segs& segs, const int32_t* __restrict__ pool, const Table& t,
                                             int g0, int g1, int lane, int& npos, uint32_t& cnt,
                                             int4* segtab, int pf_end = 0, int4* ring = nullptr) {
  const unsigned FULL = 0xffffffffu;
  int s = 0, e = 0;
  if (g0 + lane < g1) segs.get(g0 + lane, s, e);
#if TCB_PF_NEXT
  // the next group of this owner: fetch its coordinates now, prefetch its
  // suffixes into L2 once the setup below has hidden that load
  int s2 = 0, e2 = 0;
  if (g1 + lane < pf_end) segs.get(g1 + lane, s2, e2);
#endif
  int len = e - s;
  unsigned nz = __ballot_sync(FULL, len > 0);  // compact non-empty segments to the low lanes
  int nseg = __popc(nz);
  // rows keep non-empty segments first (build.cu k_rev_scatter; owner
  // segments never emit empty ones), so nz is almost always a low-lane
  // prefix and the compaction is the identity
  int src = lane;
  if (nz & (nz + 1u)) src = (lane < nseg) ? (int)__fns(nz, 0, lane + 1) : 0;
  int cs = __shfl_sync(FULL, s, src);
  int clen = __shfl_sync(FULL, len, src);
  if (lane >= nseg) clen = 0;
  // chunk span of each segment: [cs >> 2, (cs + clen + 3) >> 2)
  const int c0s = cs >> 2;
  const int nch = (lane < nseg) ? ((cs + clen + 3) >> 2) - c0s : 0;
  const int fm = (int)((0xFu << (cs & 3)) & 0xFu);            // ids of the first chunk inside the segment
  const int lm = (int)(0xFu >> (3 - ((cs + clen - 1) & 3)));  // ids of the last chunk inside it
  int incl = nch;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(FULL, incl, 31);
  const int excl = incl - nch;
  const int delta = c0s - excl;  // chunk f of the segment is pool4[delta + f]
  uint32_t* sbits = reinterpret_cast<uint32_t*>(segtab + 32);
  const bool fast = kSb && total <= 32 * kSbW;
  __syncwarp();  // the previous group's reads of segtab are done
  if (lane < nseg) {
#if TCB_SEGPTR
    const unsigned long long p = (unsigned long long)pool + 16ll * (long long)delta;  // chunk 0 of the flat space
    segtab[lane] = make_int4((int)(unsigned)p, (int)(unsigned)(p >> 32), excl, ((incl - 1) << 8) | (lm << 4) | fm);
#else
    segtab[lane] = make_int4(delta, 0, excl, ((incl - 1) << 8) | (lm << 4) | fm);
#endif
    if (fast) atomicOr(&sbits[excl >> 5], 1u << (excl & 31));  // starts are distinct (nch >= 1)
  }
  __syncwarp();
#if TCB_PF_NEXT
  for (int c = s2 & ~31; c < e2; c += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(pool + c));
#endif
  probe_group<kKind, kLw, kCap, kW, kSb, kPipe, kS, kSbW, kNoMask>(reinterpret_cast<const int4*>(pool), t, nseg, excl,
                                                             segtab, sbits, total, lane, npos, cnt, ring);
  if (fast) {
    __syncwarp();
    if (lane < nseg) sbits[excl >> 5] = 0;
  }
}

// Block-tier streaming over a row-padded pool (EngineArgs::padded).  Two
// things the general path pays per window are not needed here:
//   * id masks: ids of a chunk outside its segment are either <= u (before
//     the suffix start; every table id is > u) or the row's INT32_MAX
//     padding, so probing them can never count -- and window lanes past the
//     group's end read the pool's INT32_MAX head instead of being masked;
//   * per-window segment resolution (ballot + OR-reduction + two popc + a
//     16-byte table read): hub suffixes are many chunks long, so each lane
//     carries its current segment (its end and the address of its flat
//     chunk 0) from window to window and only steps to the next table entry
//     when its chunk index passes that end.
// ncu (cfg 3, profiles/r18_*): resolution + masks were 24 of the 49 warp
// instructions per window, the probes themselves 20.
template <int kKind, int kLw, int kCap, class Segs, int kW, bool kPipe = TCB_BIG_INC_PIPE>
__device__ __forceinline__ void stream_group_inc(const Segs& segs, const int32_t* __restrict__ pool, const Table& t,
                                                 int g0, int g1, int lane, int& npos, uint32_t& cnt, int4* segtab) {
  const unsigned FULL = 0xffffffffu;
  int s = 0, e = 0;
  if (g0 + lane < g1) segs.get(g0 + lane, s, e);
  const int len = e - s;
  const unsigned nz = __ballot_sync(FULL, len > 0);
  const int nseg = __popc(nz);
  int src = lane;
  if (nz & (nz + 1u)) src = (lane < nseg) ? (int)__fns(nz, 0, lane + 1) : 0;
  const int cs = __shfl_sync(FULL, s, src);
  int clen = __shfl_sync(FULL, len, src);
  if (lane >= nseg) clen = 0;
  const int c0s = cs >> 2;
  const int nch = (lane < nseg) ? ((cs + clen + 3) >> 2) - c0s : 0;
  int incl = nch;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(FULL, incl, 31);
  if (total == 0) return;
  const int excl = incl - nch;
  __syncwarp();  // the previous group's reads of segtab are done
  if (lane < nseg) {
    const unsigned long long p = (unsigned long long)pool + 16ll * (long long)(c0s - excl);  // flat chunk 0
    segtab[lane] = make_int4((int)(unsigned)p, (int)(unsigned)(p >> 32), incl, 0);
  }
  __syncwarp();
  const int4* const head = reinterpret_cast<const int4*>(pool) - 1;  // INT32_MAX ids
  int sj = 0;
  int4 q = segtab[0];
  int sEnd = q.z;
  const int4* sPtr = reinterpret_cast<const int4*>(((unsigned long long)(unsigned)q.y << 32) | (unsigned)q.x);
  int4 v[kW];
  auto load = [&](int base) {
#pragma unroll
    for (int k = 0; k < kW; ++k) {
      const int f = base + 32 * k + lane;
      const int4* p = head;
      if (f < total) {
        while (f >= sEnd) {  // segments are non-empty: at most nseg - 1 steps in all
          q = segtab[++sj];
          sEnd = q.z;
          sPtr = reinterpret_cast<const int4*>(((unsigned long long)(unsigned)q.y << 32) | (unsigned)q.x);
        }
#if TCB_DEBUG
        assert(sj < nseg && f < sEnd && (sj == 0 || f >= segtab[sj - 1].z));
#endif
        p = sPtr + f;
      }
      v[k] = __ldg(p);
    }
  };
  load(0);
  for (int base = 0; base < total; base += 32 * kW) {
    if (kPipe) {  // the next windows' loads are issued before the current ones are probed
      int4 cur[kW];
#pragma unroll
      for (int k = 0; k < kW; ++k) cur[k] = v[k];
      if (base + 32 * kW < total) load(base + 32 * kW);
#pragma unroll
      for (int k = 0; k < kW; ++k) probe4<kKind, kLw, kCap>(t, cur[k], 0xFu, lane, npos, cnt);
      if (kKind == kBuckets && npos > kPosDrain) drain(t, npos, lane, cnt);
    } else {
#pragma unroll
      for (int k = 0; k < kW; ++k) probe4<kKind, kLw, kCap>(t, v[k], 0xFu, lane, npos, cnt);
      if (kKind == kBuckets && npos > kPosDrain) drain(t, npos, lane, cnt);
      if (base + 32 * kW < total) load(base + 32 * kW);
    }
  }
}

struct EngineArgs {
  const int64_t* row_indptr;  // owner -> segment index range
  const int64_t* tab_indptr;  // node -> table list
  const int32_t* tab_indices;
  const int32_t* pool;        // segment coordinates index this array
  const int64_t* chunk_r;     // [nmax+1] segment-index chunk boundaries
  const int32_t* chunk_x;     // [nmax] owner at chunk start
  const int* nchunks;
  int* queue;
  const int64_t* bucket_bounds;  // nullable; bins owner_map(x)
  int nbuckets;
  unsigned long long* out;
  int64_t n_owner;            // row_indptr has n_owner + 1 entries
  const int32_t* owner_map;   // nullable: owner -> table/bucket node id
  int64_t d_lo, d_hi;         // this launch handles owners with d_lo < d <= d_hi
  int big_cap;                // block tier stages d <= big_cap, else global search
  // Tier compaction: the launch walks a compacted list of its own owners.
  // x is a tier-local index; tier_owner[x] is the owner and its segments
  // [row_indptr[x], row_indptr[x+1]) are physical [phys_row[o], ...).
  const int32_t* tier_owner;
  const int64_t* phys_row;
  // Owner descriptors, built with the plan: everything the engine needs to
  // stage an owner's table in two independent 16-byte loads instead of a
  // chain of dependent ones (tier_owner -> phys_row / owner_map ->
  // tab_indptr -> first / last table id).
  const int4* desc_a;       // (u, d, first id, id span)
  const longlong2* desc_b;  // (table offset t0, physical - tier-local segment index)
  // Chunk interleave: queue ticket q claims chunk q * stride + part, so
  // `stride` devices holding the same plan split every tier's chunks
  // between them (replicated multi-GPU count); 1 / 0 runs them all.
  int stride = 1;
  int part = 0;
  // The pool is row-padded (tc_build_graph's padded pool: every row starts
  // at a multiple of 4 ids, is padded with INT32_MAX, and TC_POOL_HEAD
  // INT32_MAX ids precede pool[0]): the small tier streams without id masks.
  int padded = 0;
};

struct OwnerRef {
  int64_t u;        // table / bucket node id
  int64_t seg_off;  // physical segment index - tier-local segment index
  int64_t t0;       // table list offset in tab_indices
  int d;            // table size
  int32_t tlo;      // first (smallest) table id
  uint32_t span;    // last - first + 1
};

__device__ __forceinline__ OwnerRef resolve_owner(const EngineArgs& a, int64_t x) {
  const int4 da = __ldg(&a.desc_a[x]);
  const longlong2 db = __ldg(&a.desc_b[x]);
  return OwnerRef{da.x, db.y, db.x, da.y, da.z, (uint32_t)da.w};
}

// Descriptor of tier-local owner x (see EngineArgs::desc_a).
__global__ void k_owner_desc(const int32_t* __restrict__ own, const int64_t* __restrict__ vrow,
                             const int64_t* __restrict__ phys_row, const int32_t* __restrict__ owner_map,
                             const int64_t* __restrict__ tab_indptr, const int32_t* __restrict__ tab_indices,
                             int64_t cnt, int4* desc_a, longlong2* desc_b) {
  GRID_STRIDE(x, cnt) {
    const int64_t o = own[x];
    const int64_t u = owner_map ? (int64_t)owner_map[o] : o;
    const int64_t t0 = tab_indptr[u], d = tab_indptr[u + 1] - t0;
    const int32_t tlo = d ? tab_indices[t0] : 0;
    const uint32_t span = d ? (uint32_t)(tab_indices[t0 + d - 1] - tlo) + 1u : 0u;
    desc_a[x] = make_int4((int)u, (int)d, tlo, (int)span);
    desc_b[x] = make_longlong2(t0, phys_row[o] - vrow[x]);
  }
}

// Runtime tier caps (tc_set_tuning; tests lower them to force every tier).
static constexpr int kWideCap = 2 * kTabCap;  // the small tier's wide form (8 ids per lane)
static int g_warp_cap = kTabCap;
static int g_mid_cap = kMidCap;
static int g_big_cap = kBigCap;

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

// First owner >= x whose segment row ends after r (warp-cooperative skip).
__device__ __forceinline__ int64_t advance_owner(const EngineArgs& a, int64_t x, int64_t r, int lane) {
  for (;;) {
    int64_t idx = x + 1 + lane;
    int64_t nx = (idx <= a.n_owner) ? __ldg(&a.row_indptr[idx]) : INT64_MAX;
    unsigned past = __ballot_sync(0xffffffffu, nx > r);
    if (past) return x + __ffs(past) - 1;
    x += 32;
  }
}

// advance_owner in 32-bit indices (tier-local owners and segment rows are
// < 2^31): the warp tiers' loop state then fits fewer registers.
__device__ __forceinline__ int advance_owner32(const EngineArgs& a, int x, int r, int lane) {
  for (;;) {
    const int idx = x + 1 + lane;
    const int nx = (idx <= a.n_owner) ? (int)__ldg(&a.row_indptr[idx]) : INT_MAX;
    const unsigned past = __ballot_sync(0xffffffffu, nx > r);
    if (past) return x + __ffs(past) - 1;
    x += 32;
  }
}

// Clears a warp's filter slice: when the slice is at most 4 words per id
// of the table, a 16-byte store per lane per 512 bytes beats re-reading and
// re-hashing the table's ids.
template <int kLw>
__device__ __forceinline__ void wipe_filter(uint32_t* bm, int lane, int words = 1 << kLw) {
  int4* b4 = reinterpret_cast<int4*>(bm);
  for (int i = lane; i < words / 4; i += 32) b4[i] = make_int4(0, 0, 0, 0);
}

// Per-warp accumulation, flushed per bucket.
struct Acc {
  unsigned long long acc = 0;  // same on all lanes
  int cur = -1;
  uint32_t cnt = 0;            // per-lane hits since the last fold
  __device__ __forceinline__ void fold() {
    unsigned long long t = cnt;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    acc += t;
    cnt = 0;
  }
  __device__ __forceinline__ void flush(unsigned long long* out, int lane) {
    if (lane == 0 && cur >= 0 && acc) atomicAdd(&out[cur], acc);
    acc = 0;
  }
  __device__ __forceinline__ void to_bucket(const EngineArgs& a, int64_t u, int lane) {
    int b = a.bucket_bounds ? bucket_of(a.bucket_bounds, a.nbuckets, u) : 0;
    if (b != cur) {
      fold();
      flush(a.out, lane);
      cur = b;
    }
  }
};

// Warp tiers (small: d <= 256 in 3 KB slices, 8 warps/block; mid:
// d <= 1024 in 8 KB slices, 4 warps/block): each warp owns a private slice.
template <class Segs, int kLb, int kLw, int kWPB, int kMinB, int kW, bool kPipe, int kS = 0, int kSbW = kSbWords,
          int kFb = 1, bool kPadded = false>
__global__ void __launch_bounds__(kWPB * 32, kMinB) k_engine(EngineArgs a, Segs segs) {
  __shared__ WarpSliceT<kLb, kLw> slices[kWPB];
  __shared__ int4 segtabs[kWPB][32 + kSbW / 4];
  __shared__ int4 rings[kWPB][kS > 0 ? kS * 32 : 1];  // cp.async window ring (kS > 0)
  const int lane = threadIdx.x & 31;
  WarpSliceT<kLb, kLw>& sl = slices[threadIdx.x >> 5];
  int4* segtab = segtabs[threadIdx.x >> 5];
  int4* ring = rings[threadIdx.x >> 5];
  for (int i = lane; i < kSbW; i += 32) reinterpret_cast<uint32_t*>(segtab + 32)[i] = 0;  // start bitmap
  const unsigned FULL = 0xffffffffu;
  const int nch = *a.nchunks;
  for (int i = lane; i < (1 << kLw); i += 32) sl.bm[i] = 0;
  __syncwarp();
  Acc acc;

  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(a.queue, 1) * a.stride + a.part;
    c = __shfl_sync(FULL, c, 0);
    if (c >= nch) break;
    int r = (int)a.chunk_r[c];  // 32-bit loop state (segment rows and owners < 2^31)
    const int r1 = (int)a.chunk_r[c + 1];
    int x = a.chunk_x[c];
    while (r < r1) {
      x = advance_owner32(a, x, r, lane);
      const int xe_row = (int)__ldg(&a.row_indptr[x + 1]);
      const int rb = min(xe_row, r1);
      const int ra = r;
      r = rb;
      const OwnerRef ow = resolve_owner(a, x);
      const int u = (int)ow.u;
      const int so = (int)ow.seg_off;
      const int d = ow.d;  // in (d_lo, d_hi]: the list holds this tier's owners only
      acc.to_bucket(a, u, lane);
      const int32_t* gtab = a.tab_indices + ow.t0;
      const int32_t tlo = ow.tlo;
      const uint32_t span = ow.span;
      // exact tables use the whole slice (filter and bucket words) as the bitmap
      constexpr int kExactWords = (1 << kLw) + 4 * (1 << kLb);
      if (span < 32u * kExactWords) {
        // Narrow id span (hub owners at the top of the degree order): the
        // slice becomes an exact direct-mapped bitmap over [tlo, tlo+span).
        // The filter words are zero between owners; the bucket words hold
        // the last hashed owner's table and are zeroed here.
        if (span >= 32u << kLw) {
          for (int i = lane; i < (1 << kLb); i += 32) sl.bkt[i] = make_int4(0, 0, 0, 0);
          __syncwarp();
        }
        for (int i = lane; i < d; i += 32) {
          const uint32_t off = (uint32_t)(__ldg(&gtab[i]) - tlo);
          atomicOr(&sl.bm[off >> 5], 1u << (off & 31));
        }
        __syncwarp();
        Table t{sl.bm, nullptr, nullptr, nullptr, d, 0, tlo, 0, 0, span};
        int npos = 0;
        for (int g = ra; g < rb; g += 32)
          if (kPadded && TCB_MID_PAD_MODE == 2)
            stream_group<kExact, kLw, Segs, kFb, kW, true, kPipe, kS, kSbW, true>(segs, a.pool, t, g + so,
                                                                                min(g + 32, rb) + so, lane, npos,
                                                                                acc.cnt, segtab, rb + so, ring);
          else
            stream_group<kExact, kLw, Segs, kFb, kW, true, kPipe, kS, kSbW>(segs, a.pool, t, g + so,
                                                                          min(g + 32, rb) + so, lane, npos, acc.cnt,
                                                                          segtab, rb + so, ring);
        __syncwarp();
#if TCB_WIPE
        wipe_filter<kLw + 0>(sl.bm, lane, kExactWords);
#else
        for (int i = lane; i < d; i += 32) sl.bm[(uint32_t)(__ldg(&gtab[i]) - tlo) >> 5] = 0;
#endif
        __syncwarp();
        continue;
      }
      const int lb = min(tab_lb(d), kLb);
      for (int i = lane; i < (1 << lb); i += 32) sl.bkt[i] = make_int4(kEmpty, kEmpty, kEmpty, kEmpty);
      __syncwarp();
      int disp = 0;
      for (int i = lane; i < d; i += 32) {
        const int32_t w = __ldg(&gtab[i]);
        filt_insert<kLw, kFb>(sl.bm, w);
        disp = max(disp, bkt_insert(sl.bkt, lb, w));
      }
      disp = __reduce_max_sync(FULL, disp);
      Table t{sl.bm, nullptr, sl.bkt, nullptr, d, lb, 0, 0, disp, 0};
      __syncwarp();
      int npos = 0;
      for (int g = ra; g < rb; g += 32)
        if (kPadded && TCB_MID_PAD_MODE == 2)
          stream_group<kInline, kLw, Segs, kFb, kW, true, kPipe, kS, kSbW, true>(segs, a.pool, t, g + so,
                                                                               min(g + 32, rb) + so, lane, npos,
                                                                               acc.cnt, segtab, rb + so, ring);
        else
          stream_group<kInline, kLw, Segs, kFb, kW, true, kPipe, kS, kSbW>(segs, a.pool, t, g + so,
                                                                         min(g + 32, rb) + so, lane, npos, acc.cnt,
                                                                         segtab, rb + so, ring);
      __syncwarp();
#if TCB_WIPE
      wipe_filter<kLw>(sl.bm, lane);
#else
      for (int i = lane; i < d; i += 32) filt_clear<kLw>(sl.bm, __ldg(&gtab[i]));
#endif
      __syncwarp();
    }
    acc.fold();
  }
  acc.flush(a.out, lane);
}

// ------------------------------------------------------------ small tier (v20)
//
// Owners with d <= 128 (cfg 2: every owner).  The v19 form of this tier was
// bound by the SM's shared-memory data pipe (ncu, profiles/r13_*: 81% of
// peak LSU wavefronts, 410 M shared wavefronts per launch at cfg 2): 19% went
// to the cp.async window ring (write + read back), 14% to building a
// bucketized hash table per owner with atomicCAS, 9% to 16-byte segment-table
// reads.  v20 keeps only the hashed two-bit filter in shared memory and
//   * holds the owner's list N^_u in registers (4 ids per lane, d <= 128) and
//     verifies the rare filter hits against it with one shuffle + one ballot
//     per hit (no bucket table to build or read);
//   * loads the windows straight into registers with 16-byte streaming loads
//     (ld.global.nc.L1::no_allocate), no shared-memory staging;
//   * keeps 8-byte segment-table entries (chunk offset, last chunk | masks);
//     whether a chunk is its segment's first comes from the start bitmap.
#ifndef TCB_SMALL_V20
#define TCB_SMALL_V20 1
#endif
#ifndef TCB_SBITS_MATCH
#define TCB_SBITS_MATCH 0  // 1: match_any + reduce_or (measured: spills, cfg2 1.70 -> 1.98 ms)
#endif
#ifndef TCB_SMALL_W
#define TCB_SMALL_W 3  // windows per step
#endif
#ifndef TCB_SMALL_PIPE2
#define TCB_SMALL_PIPE2 0  // issue the next step's loads before probing the current one
#endif
#ifndef TCB_SMALL_MINB
#define TCB_SMALL_MINB 6
#endif
#ifndef TCB_SMALL_LWS
#define TCB_SMALL_LWS 10  // filter words = 2^10 (32K bits, 4 KB per warp); exact spans < 32 * 2^10 ids
#endif
#ifndef TCB_SMALL_FB2
#define TCB_SMALL_FB2 1  // filter bits per id
#endif
static constexpr int kLwS = TCB_SMALL_LWS;
static constexpr int kSmallFb = TCB_SMALL_FB2;
static constexpr int kSmallCap = 128;  // 4 ids per lane
static constexpr int kSmallSbW = kSbWords;

// 16-byte streaming load: every chunk is read once per owner, so it should
// not displace the L1 lines of the tables and descriptors.
#ifndef TCB_LDMODE
#define TCB_LDMODE 0
#endif
__device__ __forceinline__ int4 ld_stream(const int4* p) {
#if TCB_LDMODE == 0
  return __ldg(p);
#else
  int4 r;
#if TCB_LDMODE == 1
  asm("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#else
  asm("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
#endif
  return r;
#endif
}

// Resolves chunk b + lane of the warp's flat chunk space (its segment, the
// ids of the chunk inside that segment) and issues its load.  `fast`: the
// group's start bitmap covers it (total <= 32 kSmallSbW); otherwise the
// starts come from a ballot and a warp OR-reduction over the lanes' segment
// starts.  Segment table entry: (chunk f of the segment is pool4[x + f],
// (last chunk) << 8 | last-chunk id mask << 4 | first-chunk id mask).
template <bool kPadded>
__device__ __forceinline__ void small_window(const int4* __restrict__ pool4, const int2* __restrict__ segtab,
                                             const uint32_t* __restrict__ sbits, bool fast, bool lane_seg,
                                             int excl, int total, int lane, int b, int& cbase, int4& v,
                                             uint32_t& vm) {
  const unsigned FULL = 0xffffffffu;
  vm = 0;
  v = make_int4(0, 0, 0, 0);
  if (b >= total) return;  // warp-uniform
  unsigned starts;
  int sj;
  if (fast) {
    starts = sbits[b >> 5];
    sj = cbase + __popc(starts & ((2u << lane) - 1u)) - 1;
    cbase += __popc(starts);
  } else {
    const unsigned before = __ballot_sync(FULL, lane_seg && excl < b);
    const unsigned bit = (lane_seg && excl >= b && excl < b + 32) ? (1u << (excl - b)) : 0u;
    starts = __reduce_or_sync(FULL, bit);
    if (kPadded && (unsigned)(total - b) < 32u) starts |= 1u << (total - b);  // the tail segment
    sj = __popc(before) - 1 + __popc(starts & ((2u << lane) - 1u));
  }
  const int f = b + lane;
#if TCB_DEBUG
  {  // the resolved segment covers chunk f (the tail segment: f >= total)
    assert(sj >= 0 && sj <= 32);
    const int last = segtab[sj].y >> 8, prev = sj ? (segtab[sj - 1].y >> 8) : -1;
    assert(f > prev && (f <= last || f >= total));
    if (kPadded && f >= total) assert(segtab[sj].x + f >= -32 && segtab[sj].x + f < 0);
  }
#endif
  if (kPadded) {
    // chunks past `total` resolve to the tail segment (INT32_MAX head of the
    // pool); ids before a suffix's start in its first chunk are <= u and ids
    // after a row's end are INT32_MAX padding: neither is in N^_u, so no mask
    v = __ldg(pool4 + (reinterpret_cast<const int*>(segtab)[2 * sj] + f));
    vm = 0xFu;
  } else if (f < total) {
    const int2 q = segtab[sj];
    v = ld_stream(pool4 + (q.x + f));
    uint32_t mk = 0xFu;
    if ((starts >> lane) & 1u) mk &= (uint32_t)q.y & 0xFu;
    if (f == (q.y >> 8)) mk &= ((uint32_t)q.y >> 4) & 0xFu;
    vm = mk;
  }
}

// Filter (kExactT false: two bits per id in one hashed word) or exact bitmap
// (ids in [tlo, tlo + span)) test of the 4 ids of v; returns the hit mask.
template <bool kExactT, bool kPadded, int kFb = kSmallFb>
__device__ __forceinline__ uint32_t small_probe(const uint32_t* __restrict__ bm, int32_t tlo, uint32_t span, int4 v,
                                                uint32_t vm) {
  const int32_t xs[4] = {v.x, v.y, v.z, v.w};
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (kExactT) {
      const uint32_t off = min((uint32_t)(xs[k] - tlo), span);
      const uint32_t wd = bm[off >> 5];
      m |= __funnelshift_r(wd, wd, off - k) & (1u << k);
    } else {
      const uint32_t h = tab_hash((uint32_t)xs[k]);
      const uint32_t wd = bm[h >> (32 - kLwS)];
      if (kFb == 2)
        m |= __funnelshift_r(wd, wd, h - k) & __funnelshift_r(wd, wd, (h >> 5) - k) & (1u << k);
      else
        m |= __funnelshift_r(wd, wd, h - k) & (1u << k);
    }
  }
  return kPadded ? m : (m & vm);
}

// Exact membership of the filter hits: the owner's list is held in
// registers (lane l has ids l, l + 32, l + 64, l + 96; -1 pads), so each hit
// (lane, id) is one shuffle, four compares and one ballot for the whole
// warp.  Returns the number of true hits (warp-uniform).  kIds = 8 (the wide
// form, d <= 256): lane l also holds ids l + 128 .. l + 224 in t2.
template <int kIds>
__device__ __forceinline__ uint32_t small_verify(uint32_t m, int4 v, int4 t, int4 t2, int lane) {
  const unsigned FULL = 0xffffffffu;
  uint32_t c = 0;
  unsigned any = __ballot_sync(FULL, m != 0);
  while (any) {
    const int src = __ffs(any) - 1;
    const int k = __ffs(m) - 1;
    int x = (k == 0) ? v.x : (k == 1) ? v.y : (k == 2) ? v.z : v.w;
    x = __shfl_sync(FULL, x, src);
    bool eq = (t.x == x) | (t.y == x) | (t.z == x) | (t.w == x);
    if (kIds == 8) eq |= (t2.x == x) | (t2.y == x) | (t2.z == x) | (t2.w == x);
    c += __ballot_sync(FULL, eq) != 0u;
    if (lane == src) m &= m - 1u;
    any = __ballot_sync(FULL, m != 0);
  }
  return c;
}

template <bool kExactT, bool kPadded, int kIds>
__device__ __forceinline__ void small_step(const uint32_t* bm, int32_t tlo, uint32_t span, int4 t, int4 t2, int4 v,
                                           uint32_t vm, int lane, uint32_t& cnt) {
  const uint32_t m = small_probe<kExactT, kPadded, (kIds == 8 ? 2 : kSmallFb)>(bm, tlo, span, v, vm);
  if (kExactT) {
    cnt += __popc(m);
  } else {
    const uint32_t c = small_verify<kIds>(m, v, t, t2, lane);
    if (lane == 0) cnt += c;
  }
}

// One warp streams segments [g0, g1) (<= 32) of the current owner.
// kPadded: a tail segment (index nseg, starting at chunk `total`) maps the
// chunks past the group's end onto the pool's INT32_MAX head, so window
// lanes need no bounds check.
template <bool kExactT, bool kPadded, int kIds, class Segs>
__device__ __forceinline__ void small_group(const Segs& segs, const int32_t* __restrict__ pool,
                                            const uint32_t* bm, int32_t tlo, uint32_t span, int4 t, int4 t2, int g0,
                                            int g1, int lane, uint32_t& cnt, int2* segtab, uint32_t* sbits) {
  const unsigned FULL = 0xffffffffu;
  constexpr int kW = TCB_SMALL_W;
  int s = 0, e = 0;
  if (g0 + lane < g1) segs.get(g0 + lane, s, e);
  const int len = e - s;
  const unsigned nz = __ballot_sync(FULL, len > 0);  // compact non-empty segments to the low lanes
  const int nseg = __popc(nz);
  int src = lane;
  if (nz & (nz + 1u)) src = (lane < nseg) ? (int)__fns(nz, 0, lane + 1) : 0;
  const int cs = __shfl_sync(FULL, s, src);
  int clen = __shfl_sync(FULL, len, src);
  if (lane >= nseg) clen = 0;
  const int c0s = cs >> 2;
  const int nch = (lane < nseg) ? ((cs + clen + 3) >> 2) - c0s : 0;
  const int fm = (int)((0xFu << (cs & 3)) & 0xFu);
  const int lm = (int)(0xFu >> (3 - ((cs + clen - 1) & 3)));
  int incl = nch;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(FULL, incl, 31);
  const int excl = incl - nch;
  const bool fast = kPadded ? total < 32 * kSmallSbW : total <= 32 * kSmallSbW;
  const bool lane_seg = lane < nseg;
  __syncwarp();  // the previous group's reads of segtab / sbits are done
  if (lane_seg)
    // chunk f of this segment is pool4[c0s - excl + f]; last chunk incl - 1 (< 2^23:
    // oriented lists hold at most sqrt(2m) ids)
    segtab[lane] = make_int2(c0s - excl, ((incl - 1) << 8) | (lm << 4) | fm);
#if TCB_SBITS_MATCH
  if (fast) {
    // starts are distinct and ascending: the lanes sharing a bitmap word OR
    // their bits with one reduction and its lowest lane stores the word (no
    // shared atomics on the same word)
    const unsigned w = lane_seg ? (unsigned)(excl >> 5) : 0xFFFFFFFFu;
    const unsigned grp = __match_any_sync(FULL, w);
    const unsigned bits = __reduce_or_sync(grp, lane_seg ? 1u << (excl & 31) : 0u);
    if (lane_seg && lane == __ffs(grp) - 1) sbits[w] = bits;
  }
#else
  if (lane_seg && fast) atomicOr(&sbits[excl >> 5], 1u << (excl & 31));  // starts are distinct (nch >= 1)
#endif
  if (kPadded && lane == 0) {
    // tail segment: chunk f >= total reads pool4[f - total - 32], in the head
    segtab[nseg] = make_int2(-total - 32, 0x7FFFFF << 8);
    if (fast) atomicOr(&sbits[total >> 5], 1u << (total & 31));
  }
  __syncwarp();
  const int4* pool4 = reinterpret_cast<const int4*>(pool);
  int cbase = 0;
  int4 v[kW];
  uint32_t vm[kW];
#pragma unroll
  for (int k = 0; k < kW; ++k)
    small_window<kPadded>(pool4, segtab, sbits, fast, lane_seg, excl, total, lane, 32 * k, cbase, v[k], vm[k]);
  for (int base = 0; base < total; base += 32 * kW) {
#if TCB_SMALL_PIPE2
    int4 nv[kW];
    uint32_t nvm[kW];
#pragma unroll
    for (int k = 0; k < kW; ++k)
      small_window<kPadded>(pool4, segtab, sbits, fast, lane_seg, excl, total, lane, base + 32 * (kW + k), cbase,
                            nv[k], nvm[k]);
#pragma unroll
    for (int k = 0; k < kW; ++k) small_step<kExactT, kPadded, kIds>(bm, tlo, span, t, t2, v[k], vm[k], lane, cnt);
#pragma unroll
    for (int k = 0; k < kW; ++k) {
      v[k] = nv[k];
      vm[k] = nvm[k];
    }
#else
#pragma unroll
    for (int k = 0; k < kW; ++k) small_step<kExactT, kPadded, kIds>(bm, tlo, span, t, t2, v[k], vm[k], lane, cnt);
    if (base + 32 * kW < total) {
#pragma unroll
      for (int k = 0; k < kW; ++k)
        small_window<kPadded>(pool4, segtab, sbits, fast, lane_seg, excl, total, lane, base + 32 * (kW + k), cbase,
                              v[k], vm[k]);
    }
#endif
  }
  if (fast) {
    __syncwarp();
    if (lane_seg) sbits[excl >> 5] = 0;
    if (kPadded && lane == 0) sbits[total >> 5] = 0;
  }
}

template <class Segs, bool kPadded, int kIds = 4>
__global__ void __launch_bounds__(kThreads, TCB_SMALL_MINB) k_small(EngineArgs a, Segs segs) {
  constexpr int kFb = kIds == 8 ? 2 : kSmallFb;  // the wide form holds up to 256 ids: two filter bits per id
  __shared__ uint32_t filts[kWarps][1 << kLwS];
  __shared__ int2 segtabs[kWarps][33];
  __shared__ uint32_t sbitss[kWarps][kSmallSbW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* bm = filts[warp];
  int2* segtab = segtabs[warp];
  uint32_t* sbits = sbitss[warp];
  const unsigned FULL = 0xffffffffu;
  for (int i = lane; i < kSmallSbW; i += 32) sbits[i] = 0;
  for (int i = lane; i < (1 << kLwS); i += 32) bm[i] = 0;
  __syncwarp();
  const int nch = *a.nchunks;
  Acc acc;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(a.queue, 1) * a.stride + a.part;
    c = __shfl_sync(FULL, c, 0);
    if (c >= nch) break;
    int r = (int)a.chunk_r[c];
    const int r1 = (int)a.chunk_r[c + 1];
    int x = a.chunk_x[c];
    while (r < r1) {
      x = advance_owner32(a, x, r, lane);
      const int rb = min((int)__ldg(&a.row_indptr[x + 1]), r1);
      const int ra = r;
      r = rb;
      const OwnerRef ow = resolve_owner(a, x);
      const int so = (int)ow.seg_off;
      const int d = ow.d;  // <= 32 kIds
      acc.to_bucket(a, ow.u, lane);
      const int32_t* gtab = a.tab_indices + ow.t0;
      int4 t = make_int4(-1, -1, -1, -1);
      t.x = lane < d ? __ldg(&gtab[lane]) : -1;
      if (d > 32) t.y = lane + 32 < d ? __ldg(&gtab[lane + 32]) : -1;
      if (d > 64) t.z = lane + 64 < d ? __ldg(&gtab[lane + 64]) : -1;
      if (d > 96) t.w = lane + 96 < d ? __ldg(&gtab[lane + 96]) : -1;
      int4 t2 = make_int4(-1, -1, -1, -1);
      if (kIds == 8 && d > 128) {
        t2.x = lane + 128 < d ? __ldg(&gtab[lane + 128]) : -1;
        if (d > 160) t2.y = lane + 160 < d ? __ldg(&gtab[lane + 160]) : -1;
        if (d > 192) t2.z = lane + 192 < d ? __ldg(&gtab[lane + 192]) : -1;
        if (d > 224) t2.w = lane + 224 < d ? __ldg(&gtab[lane + 224]) : -1;
      }
      const int32_t tlo = ow.tlo;
      const uint32_t span = ow.span;
      const int32_t tv[8] = {t.x, t.y, t.z, t.w, t2.x, t2.y, t2.z, t2.w};
      if (span < (32u << kLwS)) {
        // narrow id span: exact direct-mapped bitmap over [tlo, tlo + span)
#pragma unroll
        for (int k = 0; k < kIds; ++k)
          if (tv[k] >= 0) {
            const uint32_t off = (uint32_t)(tv[k] - tlo);
            atomicOr(&bm[off >> 5], 1u << (off & 31));
          }
        __syncwarp();
        for (int g = ra; g < rb; g += 32)
          small_group<true, kPadded, kIds>(segs, a.pool, bm, tlo, span, t, t2, g + so, min(g + 32, rb) + so, lane,
                                           acc.cnt, segtab, sbits);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < kIds; ++k)
          if (tv[k] >= 0) bm[(uint32_t)(tv[k] - tlo) >> 5] = 0;
      } else {
#pragma unroll
        for (int k = 0; k < kIds; ++k)
          if (tv[k] >= 0) filt_insert<kLwS, kFb>(bm, tv[k]);
        __syncwarp();
        for (int g = ra; g < rb; g += 32)
          small_group<false, kPadded, kIds>(segs, a.pool, bm, tlo, span, t, t2, g + so, min(g + 32, rb) + so, lane,
                                            acc.cnt, segtab, sbits);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < kIds; ++k)
          if (tv[k] >= 0) filt_clear<kLwS>(bm, tv[k]);
      }
      __syncwarp();
    }
    acc.fold();
  }
  acc.flush(a.out, lane);
}

// Block tier: owners with d > d_lo (the mid tier's cap).  The block stages the owner's table
// once per chunk-owner and its 16 warps stream groups of 32 segments.
// kExactOnly: every owner of the launch has an exact bitmap (checked when the
// plan is built); no bucket table and no hit queues exist.
template <class Segs, bool kPadded, bool kExactOnly = false>
__global__ void __launch_bounds__(kBigThreads, TCB_BIG_MINB) k_engine_big(EngineArgs a, Segs segs) {
  extern __shared__ __align__(16) unsigned char big_smem[];
  uint32_t* bm = reinterpret_cast<uint32_t*>(big_smem);
  int4* bkt = reinterpret_cast<int4*>(big_smem + (sizeof(uint32_t) << kLwBig));
  int32_t* pos = reinterpret_cast<int32_t*>(big_smem + (sizeof(uint32_t) << kLwBig) + (sizeof(int4) << kLbBig)) +
                 (threadIdx.x >> 5) * kPosCap;
  int4* segtab = reinterpret_cast<int4*>(big_smem + (kExactOnly ? kBigTabBytesExact : kBigTabBytesFull)) +
                 (threadIdx.x >> 5) * kSegTab;
  __shared__ int s_chunk;
  __shared__ int s_next;  // next segment group of the current staged owner (dynamic claiming)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = kBigWarps;
  const int nch = *a.nchunks;
  for (int i = threadIdx.x; i < (1 << kLwBig); i += kBigThreads) bm[i] = 0;
  for (int i = lane; i < kSbWords; i += 32) reinterpret_cast<uint32_t*>(segtab + 32)[i] = 0;  // start bitmap
  Acc acc;
  int64_t staged = -1;  // node whose table is staged
  const int32_t* staged_list = nullptr;
  int64_t staged_d = 0;
  bool staged_exact = false;
  int32_t staged_lo = 0;
  uint32_t staged_span = 0;

  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_chunk = atomicAdd(a.queue, 1) * a.stride + a.part;
      s_next = 0;
    }
    __syncthreads();
    const int c = s_chunk;
    if (c >= nch) break;
    int r = (int)a.chunk_r[c];  // 32-bit loop state, as in k_engine
    const int r1 = (int)a.chunk_r[c + 1];
    int x = a.chunk_x[c];
    while (r < r1) {
      x = advance_owner32(a, x, r, lane);  // same result in every warp
      const int xe_row = (int)__ldg(&a.row_indptr[x + 1]);
      const int rb = min(xe_row, r1);
      const int ra = r;
      r = rb;
      const OwnerRef ow = resolve_owner(a, x);
      const int64_t u = ow.u;
      const int so = (int)ow.seg_off;
      const int64_t d = ow.d;
      acc.to_bucket(a, u, lane);
      const int32_t* gtab = a.tab_indices + ow.t0;
      const int lb = tab_lb(d);
      if (d <= a.big_cap) {
        if (staged != u) {
          __syncthreads();
          if (threadIdx.x == 0) s_next = 0;
          if (staged_exact) {
            for (int i = threadIdx.x; i < staged_d; i += kBigThreads)
              bm[(uint32_t)(__ldg(&staged_list[i]) - staged_lo) >> 5] = 0;
          } else {
            for (int i = threadIdx.x; i < staged_d; i += kBigThreads) filt_clear<kLwBig>(bm, __ldg(&staged_list[i]));
          }
          const int32_t tlo = ow.tlo;
          const uint32_t span = ow.span;
          const bool exact = kExactOnly || span < (32u << kLwBig);
#if TCB_DEBUG
          assert(span < (32u << kLwBig) || !kExactOnly);
#endif
          if (!exact)
            for (int i = threadIdx.x; i < (1 << lb); i += kBigThreads) bkt[i] = make_int4(kEmpty, kEmpty, kEmpty, kEmpty);
          __syncthreads();
          for (int i = threadIdx.x; i < d; i += kBigThreads) {
            const int32_t w = __ldg(&gtab[i]);
            if (exact) {
              const uint32_t off = (uint32_t)(w - tlo);
              atomicOr(&bm[off >> 5], 1u << (off & 31));
            } else {
              filt_insert<kLwBig, TCB_BIG_FB>(bm, w);
              bkt_insert(bkt, lb, w);
            }
          }
          __syncthreads();
          staged = u;
          staged_list = gtab;
          staged_d = d;
          staged_exact = exact;
          staged_lo = tlo;
          staged_span = span;
        }
        Table t{bm, nullptr, bkt, pos, d, lb, staged_lo, 0, 0, staged_span};
        int npos = 0;
        // Groups are claimed dynamically: every owner change passes a block
        // barrier (restage or chunk fetch) that reset s_next, and the wait at
        // the next barrier is at most one group long.
        for (;;) {
          int gi = 0;
          if (lane == 0) gi = atomicAdd(&s_next, 1);
          gi = __shfl_sync(0xffffffffu, gi, 0);
          // kBigClaim segments per claim: hub suffixes are long (R-MAT: ~50
          // chunks each), so a claim of a few segments is still many windows,
          // and the wait at the next block barrier is at most one claim long
          const int g = ra + kBigClaim * gi;
          if (g >= rb) break;
          if (kPadded && kExactOnly)  // no hit queue to bound the step: more windows in flight, pipelined
            stream_group_inc<kExact, kLwBig, 1, Segs, kBigWinExact, TCB_BIG_EXACT_PIPE>(
                segs, a.pool, t, g + so, min(g + kBigClaim, rb) + so, lane, npos, acc.cnt, segtab);
          else if (kPadded && staged_exact)
            stream_group_inc<kExact, kLwBig, 1, Segs, kBigWin>(segs, a.pool, t, g + so, min(g + kBigClaim, rb) + so, lane,
                                                            npos, acc.cnt, segtab);
          else if (kPadded && !kExactOnly)
            stream_group_inc<kBuckets, kLwBig, TCB_BIG_FB, Segs, kBigWin>(segs, a.pool, t, g + so,
                                                                      min(g + kBigClaim, rb) + so, lane, npos, acc.cnt,
                                                                      segtab);
          else if (staged_exact)
            // exact tables leave the bucket area free: it holds the warps'
            // cp.async window rings (kBigStages stages of 32 chunks each)
            stream_group<kExact, kLwBig, Segs, 1, kBigWin, TCB_BIG_SB, TCB_BIG_PIPE, kBigStages>(
                segs, a.pool, t, g + so, min(g + kBigClaim, rb) + so, lane, npos, acc.cnt, segtab, 0,
                bkt + warp * (kBigStages > 0 ? kBigStages * 32 : 0));
          else if (!kExactOnly)
            stream_group<kBuckets, kLwBig, Segs, TCB_BIG_FB, kBigWin, TCB_BIG_SB, TCB_BIG_PIPE>(
                segs, a.pool, t, g + so, min(g + kBigClaim, rb) + so, lane, npos, acc.cnt, segtab);
        }
        if (!kExactOnly && !staged_exact) drain(t, npos, lane, acc.cnt);
      } else {
        Table t{nullptr, gtab, nullptr, nullptr, d, 0, __ldg(&gtab[0]), __ldg(&gtab[d - 1]), 0, 0};
        int npos = 0;
        for (int g = ra + 32 * warp; g < rb; g += 32 * nwarps)
          stream_group<kGlobal, 0, Segs, 1, kBigWin, false, TCB_BIG_PIPE>(segs, a.pool, t, g + so, min(g + 32, rb) + so, lane, npos,
                                   acc.cnt, segtab);
      }
    }
    acc.fold();
  }
  acc.flush(a.out, lane);
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
  const int nfirst = mode == 0 ? nW : TCB_PLAN_FIRST * nW;
  const double half = mode == 0 ? floor(Cd / 2.0) : floor(Cd * TCB_PLAN_HALF);
  const double R0 = Cd - half;
  const double q = 1.0 - 1.0 / (double)nW;
  const double minc = fmax(Cd / (TCB_PLAN_MINDIV * nW), 64.0);
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
static double g_tier_ms[3] = {0.0, 0.0, 0.0};
static cudaEvent_t g_tev[4] = {nullptr, nullptr, nullptr, nullptr};
static long long g_engine_launches = 0;

// Engine tiers (same order as the cost split): small / mid warp tiers, block tier.
#ifndef TCB_MID_WINDOWS
#define TCB_MID_WINDOWS 2
#endif
#ifndef TCB_SMALL_PIPE
#define TCB_SMALL_PIPE 0
#endif
#ifndef TCB_SMALL_STAGES
#define TCB_SMALL_STAGES 4
#endif
// small tier: 1.5 KB table slices + a 4-stage cp.async window ring per warp
#ifndef TCB_SMALL_FB
#define TCB_SMALL_FB 2
#endif
#define K_SMALL(S) k_engine<S, kLbWarp, kLwWarp, kWarps, TCB_MINBLOCKS, kWin, TCB_SMALL_PIPE, TCB_SMALL_STAGES, \
                            kSbWords, TCB_SMALL_FB>
#ifndef TCB_MID_MINB
#define TCB_MID_MINB 6
#endif
#ifndef TCB_MID_STAGES
#define TCB_MID_STAGES 0
#endif
#ifndef TCB_MID_SBW
#define TCB_MID_SBW 96
#endif
#ifndef TCB_MID_FB
#define TCB_MID_FB 2
#endif
#define K_MID(S) k_engine<S, kLbMid, kLwMid, kMidWarps, TCB_MID_MINB, TCB_MID_WINDOWS, TCB_MID_PIPE, TCB_MID_STAGES, \
                          TCB_MID_SBW, TCB_MID_FB>
#define K_MID_PAD(S) k_engine<S, kLbMid, kLwMid, kMidWarps, TCB_MID_MINB, TCB_MID_WINDOWS, TCB_MID_PIPE, \
                              TCB_MID_STAGES, TCB_MID_SBW, TCB_MID_FB, true>

struct TierShape {
  int blocks[3];   // persistent grid per tier
  int workers[3];  // chunk-queue workers per tier (warps / warps / blocks)
};

static const TierShape& tier_shape() {
  static TierShape ts;
  static bool init = false;
  if (!init) {
    int per_sm = 0;
#if TCB_SMALL_V20
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_small<PullSegs, true>, kThreads, 0));
#else
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K_SMALL(PullSegs), kThreads, 0));
#endif
    ts.blocks[0] = std::max(per_sm, 1) * sm_count();
    ts.workers[0] = ts.blocks[0] * kWarps;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K_MID_PAD(PullSegs), kMidWarps * 32, 0));
    ts.blocks[1] = std::max(per_sm, 1) * sm_count();
    ts.workers[1] = ts.blocks[1] * kMidWarps;
    TC_CUDA(cudaFuncSetAttribute(k_engine_big<PullSegs, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kBigSmem));
    TC_CUDA(cudaFuncSetAttribute(k_engine_big<PullSegs, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kBigSmemExact));
    TC_CUDA(cudaFuncSetAttribute(k_engine_big<PushSegs, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kBigSmemExact));
    TC_CUDA(cudaFuncSetAttribute(k_engine_big<PushSegs, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kBigSmem));
    TC_CUDA(cudaFuncSetAttribute(k_engine_big<PullSegs, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kBigSmem));
    TC_CUDA(cudaFuncSetAttribute(k_engine_big<PushSegs, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kBigSmem));
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_engine_big<PullSegs, true>, kBigThreads, kBigSmem));
    ts.blocks[2] = std::max(per_sm, 1) * sm_count();
#ifndef TCB_BIG_WORKERS_X4
#define TCB_BIG_WORKERS_X4 8
#endif
    ts.workers[2] = std::max(1, ts.blocks[2] * TCB_BIG_WORKERS_X4 / 4);
    init = true;
  }
  return ts;
}

// Exact per-segment cost of a tier (warp per tier owner): segment length +
// kSegCost, plus the owner's table build (d + kTabCost) on its first segment.
template <class Segs>
__global__ void k_seg_cost(const int32_t* __restrict__ own, const int64_t* __restrict__ vrow,
                           const int64_t* __restrict__ phys_row, const int32_t* __restrict__ owner_map,
                           const int64_t* __restrict__ tab_indptr, int64_t k, Segs segs, int64_t* cost) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = warp; x < k; x += nwarps) {
    const int64_t o = own[x];
    const int64_t u = owner_map ? (int64_t)owner_map[o] : o;
    const int64_t d = tab_indptr[u + 1] - tab_indptr[u];
    const int64_t r0 = vrow[x], r1 = vrow[x + 1], p0 = phys_row[o];
    for (int64_t r = r0 + lane; r < r1; r += 32) {
      int s = 0, e = 0;
      segs.get(p0 + (r - r0), s, e);
      cost[r] = (e - s) + kSegCost + (r == r0 ? d + kTabCost : 0);
    }
  }
}

// Chunk boundaries from an exact per-segment cost prefix (sp, nseg + 1):
// the same schedule as k_plan, but a threshold maps to a segment index by
// binary search instead of a proportional split inside the owner.
__global__ void k_plan_seg(const int64_t* __restrict__ sp, int64_t nseg, const int64_t* __restrict__ vrow,
                           int64_t nx, int nW, int nmax, int64_t* chunk_r, int32_t* chunk_x, int* nchunks) {
  const int64_t C = sp[nseg];
  const double Cd = (double)C;
  const int nfirst = 6 * nW;
  const double half = floor(Cd * 0.75);
  const double R0 = Cd - half;
  const double q = 1.0 - 1.0 / (double)nW;
  const double minc = fmax(Cd / (TCB_PLAN_SEG_MINDIV * nW), 64.0);
  int64_t J = 0;
  if (nW > 1 && R0 / nW > minc) J = (int64_t)ceil(log(minc * nW / R0) / log(q));
  if (J < 0) J = 0;
  const double RJ = R0 * pow(q, (double)J);
  const int64_t ntail = (int64_t)ceil(RJ / minc);
  int64_t total = (C == 0) ? 0 : (int64_t)nfirst + J + ntail;
  if (total > nmax) total = nmax;
  if (blockIdx.x == 0 && threadIdx.x == 0) *nchunks = (int)total;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nmax; i += (int64_t)gridDim.x * blockDim.x) {
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
    int64_t lo = 0, hi = nseg;  // first segment r with sp[r] >= T
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (sp[mid] < T) lo = mid + 1;
      else hi = mid;
    }
    const int64_t r = (T >= C) ? nseg : lo;
    int64_t a = 0, b = nx;  // owner: largest x with vrow[x] <= r
    while (b - a > 1) {
      int64_t mid = (a + b) >> 1;
      if (vrow[mid] <= r) a = mid;
      else b = mid;
    }
    chunk_r[i] = r;
    if (i < nmax) chunk_x[i] = (int32_t)a;
  }
}

// Tier of each owner in [x0, x1) (flags; owners without cost join no tier).
__global__ void k_tier_flags(const int64_t* __restrict__ cp, int64_t x0, int64_t x1,
                             const int32_t* __restrict__ owner_map, const int64_t* __restrict__ tab_indptr,
                             int c0, int c1, int32_t* f0, int32_t* f1, int32_t* f2, unsigned long long* sizes) {
  // sizes[0..2]: owners per tier; sizes[3]: engine cost of the owners with c0 < d <= 2 c0 (the candidates of
  // the small tier's wide form), sizes[4]: cost of all owners
  unsigned long long c[5] = {0, 0, 0, 0, 0};
  GRID_STRIDE(i, x1 - x0 + 1) {
    int64_t x = x0 + i;
    int t = -1;
    if (x < x1 && cp[x + 1] > cp[x]) {
      int64_t u = owner_map ? (int64_t)owner_map[x] : x;
      int64_t d = tab_indptr[u + 1] - tab_indptr[u];
      t = (d <= c0) ? 0 : (d <= c1 ? 1 : 2);
      const unsigned long long w = (unsigned long long)(cp[x + 1] - cp[x]);
      c[4] += w;
      if (d > c0 && d <= 2 * (int64_t)c0) c[3] += w;
    }
    f0[i] = t == 0;
    f1[i] = t == 1;
    f2[i] = t == 2;
    if (t >= 0) ++c[t];
  }
  for (int k = 0; k < 5; ++k) {
    unsigned long long v = c[k];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sizes[k], v);
  }
}

// Compacts one tier: own[p] = owner, len[p] = its segment count, cost[p];
// entries past the tier's size stay zero (caller memsets), so exclusive
// scans over the full length give tier-local rows / cost prefixes.
__global__ void k_tier_scatter(const int32_t* __restrict__ flag, const int32_t* __restrict__ pos, int64_t x0,
                               int64_t nx, const int64_t* __restrict__ row_indptr, const int64_t* __restrict__ cp,
                               int32_t* own, int64_t* len, int64_t* cost) {
  GRID_STRIDE(i, nx) {
    if (flag[i]) {
      const int64_t x = x0 + i;
      const int p = pos[i];
      own[p] = (int32_t)x;
      len[p] = row_indptr[x + 1] - row_indptr[x];
      cost[p] = cp[x + 1] - cp[x];
    }
  }
}

// Device memory that outlives one call (engine plans): same interface as
// Scratch, freed when the plan is destroyed.
class Persist {
 public:
  Persist() = default;
  Persist(const Persist&) = delete;
  Persist& operator=(const Persist&) = delete;
  ~Persist() { release(); }
  void set_stream(cudaStream_t s) { s_ = s; }
  void release() {
    // on the legacy default stream (ordered after work on blocking streams,
    // e.g. runs of the plan issued elsewhere)
    for (const DevBlock& b : ptrs_) dev_free(b, 0);
    ptrs_.clear();
  }
  void* bytes(size_t n) {  // pool allocation, valid on every stream once s_ has synchronised
    ptrs_.push_back(dev_alloc(n ? n : 16, s_));
    return ptrs_.back().p;
  }
  template <class T>
  T* alloc(int64_t n) {
    return static_cast<T*>(bytes(sizeof(T) * (size_t)(n > 0 ? n : 1)));
  }

 private:
  std::vector<DevBlock> ptrs_;
  cudaStream_t s_ = 0;
};

// Largest id span and table size among a tier's owners (exact-only dispatch).
__global__ void k_max_span(const int4* __restrict__ desc_a, int64_t cnt, unsigned int* out) {
  unsigned int ms = 0, md = 0;
  GRID_STRIDE(x, cnt) {
    const int4 a = desc_a[x];
    ms = max(ms, (unsigned int)a.w);
    md = max(md, (unsigned int)a.y);
  }
  ms = __reduce_max_sync(0xffffffffu, ms);
  md = __reduce_max_sync(0xffffffffu, md);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out[0], ms);
    atomicMax(&out[1], md);
  }
}

// Everything one engine run needs beyond the graph: per tier the compacted
// owner list, rows, chunk plan and queue counter (EngineArgs.out is set per
// run).  Built by prepare_engine, consumed by launch_engine.
struct EngineLaunch {
  bool big_exact = false;  // every block-tier owner has an exact bitmap: launch the exact-only kernel
  bool small_wide = false;  // the small tier takes d <= 256 (8 ids per lane, two filter bits)
  unsigned long long hsz[3] = {0, 0, 0};
  EngineArgs args[3];
  int* queue[3] = {nullptr, nullptr, nullptr};
};

template <class Segs, class Alloc>
EngineLaunch prepare_engine(Alloc& al, Scratch& tmp_sc, const int64_t* cp, const int64_t* row_indptr,
                            const int64_t* tab_indptr, const int32_t* tab_indices, const int32_t* pool, int64_t x0,
                            int64_t x1, const int64_t* bucket_bounds, int nbuckets, Segs segs, cudaStream_t s,
                            const int32_t* owner_map = nullptr, int mode = 0, int parts = 1, int padded = 0) {
  const TierShape& ts = tier_shape();
  const int64_t nx = x1 - x0;
  int c0 = g_warp_cap, c1 = std::max(g_mid_cap, g_warp_cap);
  const int grid = grid_for(nx + 1, 256, sm_count() * 16);
  EngineLaunch L;
  L.small_wide = c0 > kTabCap;  // forced by tc_set_tuning(0, 129..256)
  int32_t* flag[3];
  for (int k = 0; k < 3; ++k) flag[k] = tmp_sc.alloc<int32_t>(nx + 1);
  auto* sizes = tmp_sc.alloc<unsigned long long>(5);
  unsigned long long hs[5] = {0, 0, 0, 0, 0};
  TC_CUDA(cudaMemsetAsync(sizes, 0, 5 * sizeof(unsigned long long), s));
  k_tier_flags<<<grid, 256, 0, s>>>(cp, x0, x1, owner_map, tab_indptr, c0, c1, flag[0], flag[1], flag[2], sizes);
  check_launch();
  TC_CUDA(cudaMemcpyAsync(hs, sizes, sizeof(hs), cudaMemcpyDeviceToHost, s));
  sync_stream(s);  // empty tiers are skipped entirely
  if (TCB_SMALL_V20 && c0 == kTabCap && c1 >= kWideCap && 3 * hs[3] >= hs[4] && hs[3] > 0) {
    // Dense graphs: when the owners with 128 < d <= 256 carry a third or more of the engine's cost, they run
    // faster in the small tier's wide form than in the mid tier (cfg 5: 51.0 -> 47.5 ms; below that share the
    // wide form's two-bit filter and longer verification cost the d <= 128 owners more than the move gains:
    // cfg 3 14.1 -> 14.6 ms, cfg 2 1.60 -> 1.77 ms), so the tiers are cut again at 256.
    c0 = kWideCap;
    L.small_wide = true;
    TC_CUDA(cudaMemsetAsync(sizes, 0, 5 * sizeof(unsigned long long), s));
    k_tier_flags<<<grid, 256, 0, s>>>(cp, x0, x1, owner_map, tab_indptr, c0, c1, flag[0], flag[1], flag[2], sizes);
    check_launch();
    TC_CUDA(cudaMemcpyAsync(hs, sizes, sizeof(hs), cudaMemcpyDeviceToHost, s));
    sync_stream(s);
  }
  for (int k = 0; k < 3; ++k) L.hsz[k] = hs[k];
  size_t tmp = 0, tmp2 = 0;
  TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag[0], flag[0], nx + 1, s));
  TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, (int64_t*)nullptr, (int64_t*)nullptr, nx + 1, s));
  void* t = tmp_sc.bytes(std::max(tmp, tmp2));
  for (int k = 0; k < 3; ++k) {
    if (L.hsz[k] == 0) continue;
    int32_t* pos = tmp_sc.alloc<int32_t>(nx + 1);
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, flag[k], pos, nx + 1, s));
    int32_t* own = al.template alloc<int32_t>(nx + 1);
    int64_t* len = tmp_sc.alloc<int64_t>(nx + 1);
    int64_t* cst = tmp_sc.alloc<int64_t>(nx + 1);
    int64_t* vrow = al.template alloc<int64_t>(nx + 1);
    int64_t* vcost = tmp_sc.alloc<int64_t>(nx + 1);
    TC_CUDA(cudaMemsetAsync(len, 0, (nx + 1) * sizeof(int64_t), s));
    TC_CUDA(cudaMemsetAsync(cst, 0, (nx + 1) * sizeof(int64_t), s));
    k_tier_scatter<<<grid, 256, 0, s>>>(flag[k], pos, x0, nx, row_indptr, cp, own, len, cst);
    check_launch();
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp2, len, vrow, nx + 1, s));
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp2, cst, vcost, nx + 1, s));
    // planned for the workers of all `parts` devices that split the chunks
    const int nW = ts.workers[k] * parts;
    const int nmax = TCB_PLAN_NMAX * nW + 8;
    int64_t* chunk_r = al.template alloc<int64_t>(nmax + 1);
    int32_t* chunk_x = al.template alloc<int32_t>(nmax);
    int* ctl = al.template alloc<int>(2);  // [0] nchunks, [1] queue
    TC_CUDA(cudaMemsetAsync(ctl, 0, 2 * sizeof(int), s));
    if (k == 2) {  // block tier: hub segments vary wildly in cost -> plan on an exact per-segment prefix
      int64_t nseg = 0;
      TC_CUDA(cudaMemcpyAsync(&nseg, vrow + nx, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      sync_stream(s);
      int64_t* scost = tmp_sc.alloc<int64_t>(nseg + 1);
      int64_t* sp = tmp_sc.alloc<int64_t>(nseg + 1);
      TC_CUDA(cudaMemsetAsync(scost + nseg, 0, sizeof(int64_t), s));
      k_seg_cost<<<grid_for((int64_t)L.hsz[k] * 32, 256, sm_count() * 16), 256, 0, s>>>(
          own, vrow, row_indptr, owner_map, tab_indptr, (int64_t)L.hsz[k], segs, scost);
      check_launch();
      size_t tmp3 = 0;
      TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp3, scost, sp, nseg + 1, s));
      void* t3 = tmp_sc.bytes(tmp3);
      TC_CUDA(cub::DeviceScan::ExclusiveSum(t3, tmp3, scost, sp, nseg + 1, s));
      k_plan_seg<<<grid_for(nmax + 1, 256), 256, 0, s>>>(sp, nseg, vrow, nx, nW, nmax, chunk_r, chunk_x, ctl);
    } else {
      k_plan<<<grid_for(nmax + 1, 256), 256, 0, s>>>(vcost, vrow, 0, nx, nW, nmax, chunk_r, chunk_x, ctl, mode);
    }
    check_launch();
    const int64_t lo = k == 0 ? 0 : (k == 1 ? c0 : c1);
    const int64_t hi = k == 0 ? c0 : (k == 1 ? c1 : INT64_MAX);
    int4* desc_a = al.template alloc<int4>((int64_t)L.hsz[k]);
    longlong2* desc_b = al.template alloc<longlong2>((int64_t)L.hsz[k]);
    k_owner_desc<<<grid_for((int64_t)L.hsz[k], 256, sm_count() * 8), 256, 0, s>>>(
        own, vrow, row_indptr, owner_map, tab_indptr, tab_indices, (int64_t)L.hsz[k], desc_a, desc_b);
    check_launch();
    if (k == 2) {  // all tables exact bitmaps and staged (d <= block cap)?
      unsigned int* mx = tmp_sc.alloc<unsigned int>(2);
      TC_CUDA(cudaMemsetAsync(mx, 0, 2 * sizeof(unsigned int), s));
      k_max_span<<<grid_for((int64_t)L.hsz[k], 256, sm_count() * 8), 256, 0, s>>>(desc_a, (int64_t)L.hsz[k], mx);
      check_launch();
      unsigned int hmx[2] = {0, 0};
      TC_CUDA(cudaMemcpyAsync(hmx, mx, sizeof(hmx), cudaMemcpyDeviceToHost, s));
      sync_stream(s);
      L.big_exact = hmx[0] < (32u << kLwBig) && (int64_t)hmx[1] <= (int64_t)g_big_cap;
    }
    L.args[k] = EngineArgs{vrow, tab_indptr, tab_indices, pool, chunk_r, chunk_x, ctl, ctl + 1,
                           bucket_bounds, nbuckets, nullptr, nx, owner_map, lo, hi, g_big_cap, own, row_indptr,
                           desc_a, desc_b};
    L.args[k].padded = padded;
    L.queue[k] = ctl + 1;
  }
  return L;
}

// Concurrent tier launches (one stream per tier, the block tier first):
// measured cfg 4 -0.8 %, cfg 5 +5.8 % (the first kernel holds every SM until
// its tail, and the small tier's blocks then compete with the mid tier's) --
// off by default.
#ifndef TCB_TIER_STREAMS
#define TCB_TIER_STREAMS 0
#endif

template <class Segs>
static void launch_tier(EngineLaunch& L, int k, Segs segs, cudaStream_t s, const TierShape& ts) {
  if (k == 0) {
#if TCB_SMALL_V20
    if (L.small_wide) {
      if (L.args[0].padded) k_small<Segs, true, 8><<<ts.blocks[0], kThreads, 0, s>>>(L.args[0], segs);
      else k_small<Segs, false, 8><<<ts.blocks[0], kThreads, 0, s>>>(L.args[0], segs);
    } else if (L.args[0].padded) {
      k_small<Segs, true><<<ts.blocks[0], kThreads, 0, s>>>(L.args[0], segs);
    } else {
      k_small<Segs, false><<<ts.blocks[0], kThreads, 0, s>>>(L.args[0], segs);
    }
#else
    K_SMALL(Segs)<<<ts.blocks[0], kThreads, 0, s>>>(L.args[0], segs);
#endif
  } else if (k == 1) {
    if (L.args[1].padded) K_MID_PAD(Segs)<<<ts.blocks[1], kMidWarps * 32, 0, s>>>(L.args[1], segs);
    else K_MID(Segs)<<<ts.blocks[1], kMidWarps * 32, 0, s>>>(L.args[1], segs);
  } else {
    if (L.args[2].padded && L.big_exact)
      k_engine_big<Segs, true, true><<<ts.blocks[2], kBigThreads, kBigSmemExact, s>>>(L.args[2], segs);
    else if (L.args[2].padded)
      k_engine_big<Segs, true><<<ts.blocks[2], kBigThreads, kBigSmem, s>>>(L.args[2], segs);
    else
      k_engine_big<Segs, false><<<ts.blocks[2], kBigThreads, kBigSmem, s>>>(L.args[2], segs);
  }
  check_launch();
}

struct TierStreams {
  cudaStream_t st[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t fork = nullptr, join[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t t0[3] = {nullptr, nullptr, nullptr}, t1[3] = {nullptr, nullptr, nullptr};
  std::mutex mu;
};

static TierStreams& tier_streams() {
  static TierStreams ts[64];
  int dev = 0;
  TC_CUDA(cudaGetDevice(&dev));
  TierStreams& t = ts[dev];
  if (!t.fork) {
    std::lock_guard<std::mutex> lk(t.mu);
    if (!t.fork) {
      for (int k = 0; k < 3; ++k) {
        TC_CUDA(cudaStreamCreateWithFlags(&t.st[k], cudaStreamNonBlocking));
        TC_CUDA(cudaEventCreateWithFlags(&t.join[k], cudaEventDisableTiming));
        TC_CUDA(cudaEventCreate(&t.t0[k]));
        TC_CUDA(cudaEventCreate(&t.t1[k]));
      }
      cudaEvent_t f;
      TC_CUDA(cudaEventCreateWithFlags(&f, cudaEventDisableTiming));
      t.fork = f;
    }
  }
  return t;
}

template <class Segs>
static void launch_tiers_concurrent(EngineLaunch& L, Segs segs, cudaStream_t s, const TierShape& ts) {
  TierStreams& T = tier_streams();
  std::lock_guard<std::mutex> lk(T.mu);  // the fork/join events are shared per device
  if (g_time_engine) {
    if (!g_ev[0]) {
      TC_CUDA(cudaEventCreate(&g_ev[0]));
      TC_CUDA(cudaEventCreate(&g_ev[1]));
    }
    TC_CUDA(cudaEventRecord(g_ev[0], s));
  }
  TC_CUDA(cudaEventRecord(T.fork, s));  // after the queue resets and the caller's prior work
  for (int k = 2; k >= 0; --k) {
    if (!L.hsz[k]) continue;
    TC_CUDA(cudaStreamWaitEvent(T.st[k], T.fork, 0));
    if (g_time_engine) TC_CUDA(cudaEventRecord(T.t0[k], T.st[k]));
    launch_tier<Segs>(L, k, segs, T.st[k], ts);
    if (g_time_engine) TC_CUDA(cudaEventRecord(T.t1[k], T.st[k]));
    TC_CUDA(cudaEventRecord(T.join[k], T.st[k]));
  }
  for (int k = 0; k < 3; ++k)
    if (L.hsz[k]) TC_CUDA(cudaStreamWaitEvent(s, T.join[k], 0));
  if (g_time_engine) {
    TC_CUDA(cudaEventRecord(g_ev[1], s));
    TC_CUDA(cudaEventSynchronize(g_ev[1]));
    float ms = 0.f;
    TC_CUDA(cudaEventElapsedTime(&ms, g_ev[0], g_ev[1]));
    g_engine_ms += ms;
    for (int k = 0; k < 3; ++k)
      if (L.hsz[k]) {
        TC_CUDA(cudaEventElapsedTime(&ms, T.t0[k], T.t1[k]));
        g_tier_ms[k] += ms;
      }
    ++g_engine_launches;
  }
}

// Launches the non-empty tiers (queue counters reset first); `out` must be
// zeroed by the caller.
template <class Segs>
void launch_engine(EngineLaunch& L, unsigned long long* out, Segs segs, cudaStream_t s, int part = 0,
                   int stride = 1) {
  const TierShape& ts = tier_shape();
  for (int k = 0; k < 3; ++k) {
    L.args[k].out = out;
    L.args[k].part = part;
    L.args[k].stride = stride;
    if (L.hsz[k]) TC_CUDA(cudaMemsetAsync(L.queue[k], 0, sizeof(int), s));
  }
  int nonempty = (L.hsz[0] > 0) + (L.hsz[1] > 0) + (L.hsz[2] > 0);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  TC_CUDA(cudaStreamIsCapturing(s, &cap));
  if (TCB_TIER_STREAMS && nonempty > 1 && cap == cudaStreamCaptureStatusNone) {
    // Concurrent tiers: each tier on its own stream, the longest (block)
    // first, so a tier's tail overlaps the next tier's work instead of
    // idling the SMs that finished early.
    launch_tiers_concurrent(L, segs, s, ts);
    return;
  }
  if (g_time_engine) {
    if (!g_ev[0]) {
      TC_CUDA(cudaEventCreate(&g_ev[0]));
      TC_CUDA(cudaEventCreate(&g_ev[1]));
    }
    TC_CUDA(cudaEventRecord(g_ev[0], s));
    if (!g_tev[0])
      for (auto& e : g_tev) TC_CUDA(cudaEventCreate(&e));
    TC_CUDA(cudaEventRecord(g_tev[0], s));
  }
  if (L.hsz[0]) {
    launch_tier<Segs>(L, 0, segs, s, ts);
  }
  if (g_time_engine) TC_CUDA(cudaEventRecord(g_tev[1], s));
  if (L.hsz[1]) {
    launch_tier<Segs>(L, 1, segs, s, ts);
  }
  if (g_time_engine) TC_CUDA(cudaEventRecord(g_tev[2], s));
  if (L.hsz[2]) {
    launch_tier<Segs>(L, 2, segs, s, ts);
  }
  if (g_time_engine) {
    TC_CUDA(cudaEventRecord(g_tev[3], s));
    TC_CUDA(cudaEventRecord(g_ev[1], s));
    TC_CUDA(cudaEventSynchronize(g_ev[1]));
    float ms = 0.f;
    TC_CUDA(cudaEventElapsedTime(&ms, g_ev[0], g_ev[1]));
    g_engine_ms += ms;
    for (int k = 0; k < 3; ++k) {
      TC_CUDA(cudaEventElapsedTime(&ms, g_tev[k], g_tev[k + 1]));
      g_tier_ms[k] += ms;
    }
    ++g_engine_launches;
  }
}

template <class Segs>
void run_engine(Scratch& sc, int64_t n_owner, const int64_t* cp, const int64_t* row_indptr, const int64_t* tab_indptr,
                const int32_t* tab_indices, const int32_t* pool, int64_t x0, int64_t x1,
                const int64_t* bucket_bounds, int nbuckets, unsigned long long* out, Segs segs,
                cudaStream_t s, const int32_t* owner_map = nullptr, int mode = 0, int padded = 0) {
  (void)n_owner;
  EngineLaunch L = prepare_engine(sc, sc, cp, row_indptr, tab_indptr, tab_indices, pool, x0, x1, bucket_bounds,
                                  nbuckets, segs, s, owner_map, mode, 1, padded);
  launch_engine(L, out, segs, s);
}

// A reusable middle-vertex engine run over a fixed (graph, owner range):
// the tier lists and chunk plan are computed once; every run is the memsets
// plus the engine launches, with no host synchronisation.  The plan keeps
// the caller's array pointers and re-plans itself if the tier caps changed.
struct MiddlePlan {
  const int64_t *tab_indptr, *rev_indptr, *rev_cost, *bucket_bounds;
  const int32_t *tab_indices, *rev_seg, *pool;
  int64_t n, u0, u1;
  int nbuckets;
  int caps[3];
  Persist mem;
  EngineLaunch L;
  int parts = 1;  // devices the chunk plan is cut for (tc_plan_middle_parts)
  int padded = 0;  // pool is tc_build_graph's row-padded pool
  cudaEvent_t ready = nullptr;  // recorded after the planning kernels; runs on any stream wait on it
  cudaEvent_t done = nullptr;   // recorded behind each run: the next run (any stream) waits on it
  ~MiddlePlan() {
    if (ready) cudaEventDestroy(ready);
    if (done) cudaEventDestroy(done);
  }
};

static void plan_build(MiddlePlan& P, cudaStream_t s) {
  P.mem.release();
  P.mem.set_stream(s);
  P.L = EngineLaunch{};
  P.caps[0] = g_warp_cap;
  P.caps[1] = g_mid_cap;
  P.caps[2] = g_big_cap;
  if (P.u1 <= P.u0) return;
  Scratch sc(s);
  P.L = prepare_engine(P.mem, sc, P.rev_cost, P.rev_indptr, P.tab_indptr, P.tab_indices, P.pool, P.u0, P.u1,
                       P.bucket_bounds, P.nbuckets, PullSegs{reinterpret_cast<const int2*>(P.rev_seg)}, s,
                       nullptr, 1, P.parts, P.padded);
  // no host synchronisation: a run waits on this event (pool memory of the
  // plan becomes valid on the run's stream through it)
  if (!P.ready) TC_CUDA(cudaEventCreateWithFlags(&P.ready, cudaEventDisableTiming));
  TC_CUDA(cudaEventRecord(P.ready, s));
}

void count_middle(const int64_t* tab_indptr, const int32_t* tab_indices, const int64_t* rev_indptr,
                  const int32_t* rev_seg, const int64_t* rev_cost, const int32_t* pool, int pool_padded, int64_t n,
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
             nbuckets, out, PullSegs{reinterpret_cast<const int2*>(rev_seg)}, s, nullptr, 1, pool_padded);
}

void count_owners(const int64_t* tab_indptr, const int32_t* tab_indices, const int32_t* owner_map,
                  const int64_t* row_indptr, const int32_t* segs, const int64_t* cost_prefix,
                  const int32_t* pool, int64_t k, const int64_t* bucket_bounds, int nbuckets,
                  unsigned long long* out, int mode, cudaStream_t s) {
  TC_REQUIRE(k >= 0 && nbuckets >= 1, TC_EINVAL, "bad owner count / nbuckets");
  TC_REQUIRE(bucket_bounds || nbuckets == 1, TC_EINVAL, "bucket_bounds required for nbuckets > 1");
  TC_REQUIRE(((uintptr_t)pool & 15) == 0, TC_EINVAL, "pool must be 16-byte aligned (and padded to a multiple of 4 ids)");
  TC_CUDA(cudaMemsetAsync(out, 0, nbuckets * sizeof(unsigned long long), s));
  if (k == 0) return;
  Scratch sc(s);
  run_engine(sc, k, cost_prefix, row_indptr, tab_indptr, tab_indices, pool, 0, k, bucket_bounds,
             nbuckets, out, PullSegs{reinterpret_cast<const int2*>(segs)}, s, owner_map, mode);
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
                    const int64_t* rev_indptr, const int32_t* rev_seg, const int64_t* rev_cost,
                    const int32_t* pool, int32_t pool_padded, int64_t n, int64_t u0, int64_t u1,
                    const int64_t* bucket_bounds, int32_t nbuckets, unsigned long long* out,
                    tc_stream_t stream) {
  return tcb::guarded([&] {
    tcb::count_middle(tab_indptr, tab_indices, rev_indptr, rev_seg, rev_cost, pool, pool_padded, n, u0, u1,
                      bucket_bounds, nbuckets, out, (cudaStream_t)stream);
  });
}

int tc_plan_middle_parts(const int64_t* tab_indptr, const int32_t* tab_indices, const int64_t* rev_indptr,
                         const int32_t* rev_seg, const int64_t* rev_cost, const int32_t* pool, int32_t pool_padded,
                         int64_t n, int64_t u0, int64_t u1, const int64_t* bucket_bounds, int32_t nbuckets,
                         int32_t nparts, tc_plan_t* plan, tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(plan != nullptr, TC_EINVAL, "plan out-pointer is NULL");
    *plan = nullptr;
    TC_REQUIRE(0 <= u0 && u0 <= u1 && u1 <= n, TC_EINVAL, "bad owner range");
    TC_REQUIRE(nbuckets >= 1, TC_EINVAL, "nbuckets must be >= 1");
    TC_REQUIRE(nparts >= 1 && nparts <= 1024, TC_EINVAL, "nparts must be in [1, 1024]");
    TC_REQUIRE(bucket_bounds || nbuckets == 1, TC_EINVAL, "bucket_bounds required for nbuckets > 1");
    TC_REQUIRE(((uintptr_t)pool & 15) == 0, TC_EINVAL, "pool must be 16-byte aligned");
    auto* P = new tcb::MiddlePlan{tab_indptr, rev_indptr, rev_cost, bucket_bounds, tab_indices, rev_seg, pool,
                                  n, u0, u1, nbuckets, {0, 0, 0}, {}, {}, nparts, pool_padded != 0};
    try {
      tcb::plan_build(*P, (cudaStream_t)stream);
    } catch (...) {
      delete P;
      throw;
    }
    *plan = reinterpret_cast<tc_plan_t>(P);
  });
}

int tc_plan_middle(const int64_t* tab_indptr, const int32_t* tab_indices, const int64_t* rev_indptr,
                   const int32_t* rev_seg, const int64_t* rev_cost, const int32_t* pool, int32_t pool_padded,
                   int64_t n, int64_t u0, int64_t u1, const int64_t* bucket_bounds, int32_t nbuckets,
                   tc_plan_t* plan, tc_stream_t stream) {
  return tc_plan_middle_parts(tab_indptr, tab_indices, rev_indptr, rev_seg, rev_cost, pool, pool_padded, n, u0, u1,
                              bucket_bounds, nbuckets, 1, plan, stream);
}

int tc_plan_run_part(tc_plan_t plan, int32_t part, unsigned long long* out, tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(plan != nullptr, TC_EINVAL, "NULL plan");
    auto* P = reinterpret_cast<tcb::MiddlePlan*>(plan);
    TC_REQUIRE(part >= -1 && part < P->parts, TC_EINVAL, "part out of range");
    cudaStream_t s = (cudaStream_t)stream;
    if (P->caps[0] != tcb::g_warp_cap || P->caps[1] != tcb::g_mid_cap || P->caps[2] != tcb::g_big_cap)
      tcb::plan_build(*P, s);
    TC_CUDA(cudaMemsetAsync(out, 0, P->nbuckets * sizeof(unsigned long long), s));
    if (P->u1 <= P->u0) return;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    TC_CUDA(cudaStreamIsCapturing(s, &cap));
    if (cap == cudaStreamCaptureStatusNone) {
      TC_CUDA(cudaStreamWaitEvent(s, P->ready, 0));
      // the plan's queue counters are shared: a run on another stream must
      // not reset them while an earlier run still claims chunks
      if (!P->done) TC_CUDA(cudaEventCreateWithFlags(&P->done, cudaEventDisableTiming));
      else TC_CUDA(cudaStreamWaitEvent(s, P->done, 0));
    }
    const tcb::PullSegs segs{reinterpret_cast<const int2*>(P->rev_seg)};
    if (part < 0) tcb::launch_engine(P->L, out, segs, s);  // every chunk
    else tcb::launch_engine(P->L, out, segs, s, part, P->parts);
    if (cap == cudaStreamCaptureStatusNone) TC_CUDA(cudaEventRecord(P->done, s));
  });
}

int tc_plan_run(tc_plan_t plan, unsigned long long* out, tc_stream_t stream) {
  return tc_plan_run_part(plan, -1, out, stream);
}

int tc_plan_rebind(tc_plan_t plan, const int32_t* rev_seg, const int32_t* pool) {
  return tcb::guarded([&] {
    TC_REQUIRE(plan != nullptr && rev_seg != nullptr && pool != nullptr, TC_EINVAL, "NULL plan or array");
    TC_REQUIRE(((uintptr_t)pool & 15) == 0, TC_EINVAL, "pool must be 16-byte aligned");
    auto* P = reinterpret_cast<tcb::MiddlePlan*>(plan);
    P->rev_seg = rev_seg;
    P->pool = pool;
    for (int k = 0; k < 3; ++k) P->L.args[k].pool = pool;  // launch arguments are copied at each run
  });
}

int tc_plan_free(tc_plan_t plan) {
  return tcb::guarded([&] { delete reinterpret_cast<tcb::MiddlePlan*>(plan); });
}

int tc_count_owners(const int64_t* tab_indptr, const int32_t* tab_indices, const int32_t* owner_map,
                    const int64_t* row_indptr, const int32_t* segs, const int64_t* cost_prefix,
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

int tc_engine_timing(int32_t enable, double* total_ms_host, long long* launches_host, double* tier_ms_host) {
  return tcb::guarded([&] {
    if (total_ms_host) *total_ms_host = tcb::g_engine_ms;
    if (launches_host) *launches_host = tcb::g_engine_launches;
    if (tier_ms_host)
      for (int k = 0; k < 3; ++k) tier_ms_host[k] = tcb::g_tier_ms[k];
    if (enable >= 0) {
      tcb::g_time_engine = enable != 0;
      tcb::g_engine_ms = 0.0;
      tcb::g_engine_launches = 0;
      for (int k = 0; k < 3; ++k) tcb::g_tier_ms[k] = 0.0;
    }
  });
}

int tc_set_tuning(int32_t key, int64_t value) {
  return tcb::guarded([&] {
    // value -1 restores a cap's default
    if (key == 0) {
      if (value == -1) value = tcb::kTabCap;
      // 129..256 force the small tier's wide form (8 ids per lane)
      TC_REQUIRE(value >= 0 && value <= tcb::kWideCap, TC_EINVAL, "warp cap out of range");
      tcb::g_warp_cap = (int)value;
    } else if (key == 2) {
      if (value == -1) value = tcb::kMidCap;
      TC_REQUIRE(value >= 0 && value <= tcb::kMidCap, TC_EINVAL, "mid cap out of range");
      tcb::g_mid_cap = (int)value;
    } else if (key == 1) {
      if (value == -1) value = tcb::kBigCap;
      TC_REQUIRE(value >= 0 && value <= tcb::kBigCap, TC_EINVAL, "block cap out of range");
      tcb::g_big_cap = (int)value;
    } else if (key == 3) {
      TC_REQUIRE(value >= 1, TC_EINVAL, "host chunk size out of range");
      tcb::g_host_chunk = value;
    } else {
      throw tcb::Error(TC_EINVAL, "unknown tuning key");
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

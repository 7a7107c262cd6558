/*
 * tcb200.h -- C ABI of libtcb200.so, the B200-native (sm_100a) exact triangle
 * counter.  Drop-in replacement for the native boundary of the reference
 * `tricount` package (/root/reference/pkg/src/tricount): the numba kernels
 * of _kernels.py and the numpy construction of graph.py / partitioning.py.
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer unless its name ends in
 *     `_host`.  The library never frees caller memory; scratch is
 *     stream-ordered (cudaMallocAsync) and released before return.
 *   - Node ids are int32, CSR offsets int64, counts uint64 (the reference
 *     uses int64 everywhere, graph.py:85,111,120).
 *   - `stream` is a cudaStream_t (0 = legacy default stream).  Calls are
 *     stream-ordered; a call that returns host scalars (`*_host`)
 *     synchronises the stream before returning.
 *   - Return 0 (TC_OK) or a negative status; tc_last_error() describes the
 *     last failure on the calling thread.  The Python layer maps
 *     TC_EINVAL -> ValueError, TC_EINDEX -> IndexError, others ->
 *     RuntimeError, mirroring the reference's exceptions.
 *   - Thread-safe across host threads using distinct streams (the reference's
 *     kernels are nogil and called concurrently from rank threads,
 *     _kernels.py:12, runtime.py:420-454).
 */
#ifndef TCB200_H
#define TCB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* tc_stream_t; /* cudaStream_t */

enum {
  TC_OK = 0,
  TC_EINVAL = -1, /* ValueError in the reference */
  TC_EINDEX = -2, /* IndexError */
  TC_ECUDA = -3,  /* CUDA runtime failure */
  TC_ENOMEM = -4  /* device allocation failure */
};

/* Cost kinds, CostKind order (partitioning.py:32-35). */
enum { TC_COST_UNIT = 0, TC_COST_DEGREE = 1, TC_COST_SUCC_SUM = 2, TC_COST_PRED_SUM = 3 };

const char* tc_last_error(void);
int tc_abi_version(void);
/* Number of this library's kernels launched so far in the process (CUB's
 * sort/scan kernels excluded).  Measurement only. */
unsigned long long tc_launch_count(void);
/* Device memory.  Every scratch / plan allocation of the library goes to the
 * caller's allocator when one is registered (e.g. torch's caching allocator,
 * so the caller owns every byte; register before the first call), else to a
 * stream-ordered pool private to the library (the device's default pool is
 * never modified).  alloc returns NULL on failure (-> TC_ENOMEM); frees are
 * stream-ordered on the given stream.  NULL, NULL restores the pool. */
typedef void* (*tc_alloc_fn)(size_t bytes, tc_stream_t stream, void* ctx);
typedef void (*tc_free_fn)(void* ptr, tc_stream_t stream, void* ctx);
int tc_set_allocator(tc_alloc_fn alloc, tc_free_fn free_fn, void* ctx);
/* Releases the private pool's cached blocks back to the driver. */
int tc_trim_pool(void);

/* ---------------------------------------------------------------- build */

/* normalize (graph.py:76-103): drop self-loops, first-seen compaction of
 * non-dense labels, dedup undirected pairs; output sorted (lo, hi) pairs.
 * edges: int32[2*m_raw] (u0,v0,u1,v1,...), labels >= 0 else TC_EINVAL.
 * out_edges: int32[2*m_raw] capacity.  Synchronises (returns m, n). */
int tc_normalize(const int32_t* edges, int64_t m_raw, int32_t* out_edges,
                 int64_t* m_host, int64_t* n_host, tc_stream_t stream);

/* normalize from a host edge list (same result as tc_normalize): host_edges
 * (int32[2*m_raw], pinned for an asynchronous copy) is copied into
 * dev_edges (int32[2*m_raw] device staging) in chunks on a copy stream while
 * each landed chunk's min/max, first occurrences and degree histogram run on
 * `stream`.  deg (nullable, int32[2*m_raw+1]) receives every label's degree;
 * *deg_valid = 1 when it is the normalized graph's degree array (dense
 * labels kept, no self-loop or duplicate dropped), for tc_build_graph_deg.
 * Replaces the H2D copy + graph.normalize of a host list (graph.py:76-103).
 * Synchronises (returns m, n).  Calls for one device are serialised by a
 * per-device lock (they share that device's copy stream, chunk events and
 * mapped flag slots); calls for different devices run concurrently. */
int tc_normalize_host(const int32_t* host_edges, int64_t m_raw, int32_t* dev_edges, int32_t* out_edges,
                      int64_t* m_host, int64_t* n_host, int32_t* deg, int32_t* deg_valid,
                      tc_stream_t stream);

/* build_graph + _assemble (graph.py:106-153): degree order (ascending
 * (deg, id), graph.py:152) unless `order` (int32[n], order[i] = original id
 * at canonical position i) is given (the _build_graph_input_order hook,
 * graph.py:156-160).  Edge ids must lie in [0, n) (else TC_EINDEX).
 * Outputs (all caller-allocated):
 *   eff_indptr int64[n+1], eff_indices int32[m]      forward CSR N^_v
 *   relabel, orig_ids, deg, eff_deg  int32[n]
 *   rev_indptr int64[n+1]   predecessor rows: one entry per v with u in N^_v,
 *                           in unspecified order (the engine sums over a row)
 *   rev_seg    int32[2*m]   the suffix of N^_v after u of the edge e = (v, u),
 *                           as [start, end) in pool coordinates
 *   rev_cost   int64[n+1]   exclusive prefix over u of the pull-engine cost
 *   pool_indptr int64[n+1]  row offsets of the padded pool (multiples of 4)
 *   pool       int32[TC_POOL_HEAD + m + 3n + 4] buffer; pass the pointer
 *                           TC_POOL_HEAD ids past its start: pool[-TC_POOL_HEAD..-1]
 *                           = INT32_MAX, row v = N^_v at pool[pool_indptr[v]..]
 *                           padded with INT32_MAX to a multiple of 4 ids, so a
 *                           16-byte chunk never mixes two rows (the engine's
 *                           mask-free streaming, tc_count_middle pool_padded)
 * Asynchronous. */
#define TC_POOL_HEAD 512
int tc_build_graph(const int32_t* edges, int64_t m, int64_t n, const int32_t* order,
                   int64_t* eff_indptr, int32_t* eff_indices, int32_t* relabel,
                   int32_t* orig_ids, int32_t* deg, int32_t* eff_deg, int64_t* rev_indptr,
                   int32_t* rev_seg, int64_t* rev_cost, int64_t* pool_indptr, int32_t* pool,
                   tc_stream_t stream);

/* tc_build_graph in degree order with the degree array given (deg_hint
 * int32[n], e.g. from tc_normalize_host with *deg_valid): skips the degree
 * histogram (graph.py:149-151) and its range check -- the edges must be a
 * normalized list in [0, n). */
int tc_build_graph_deg(const int32_t* edges, int64_t m, int64_t n, const int32_t* deg_hint,
                       int64_t* eff_indptr, int32_t* eff_indices, int32_t* relabel,
                       int32_t* orig_ids, int32_t* deg, int32_t* eff_deg, int64_t* rev_indptr,
                       int32_t* rev_seg, int64_t* rev_cost, int64_t* pool_indptr, int32_t* pool,
                       tc_stream_t stream);

/* Full CSR (graph.py:125-127) assembled from the forward and reverse CSRs:
 * row u = its neighbours ascending (predecessors, then N^_u).  pool_indptr:
 * the row offsets rev_seg's coordinates refer to (tc_build_graph's).
 * full_indptr int64[n+1], full_indices int32[2m].  Synchronises. */
int tc_build_full(const int64_t* eff_indptr, const int32_t* eff_indices,
                  const int64_t* rev_indptr, const int32_t* rev_seg, const int64_t* pool_indptr, int64_t n,
                  int64_t* full_indptr, int32_t* full_indices, tc_stream_t stream);

/* ---------------------------------------------------------------- count */

/* Middle-vertex ("pull") engine: triangles v < u < w whose middle vertex u
 * lies in [u0, u1), written to out[bucket(u)] (uint64).  bucket_bounds
 * (int64[nbuckets+1], ascending) bins u; NULL with nbuckets==1 sums all.
 * Table lists N^_u come from (tab_indptr, tab_indices) indexed by u;
 * predecessor suffixes are rev_seg int32 pairs indexing `pool` (int32).
 * pool_padded = 1: `pool` is tc_build_graph's row-padded pool (rows at
 * multiples of 4 ids, INT32_MAX padding and TC_POOL_HEAD INT32_MAX ids before
 * pool[0]) and the engine streams it without per-chunk id masks; 0: any
 * 16-byte aligned pool padded by >= 4 ids at its end (e.g. received lists).
 * out is overwritten (not accumulated).
 * This is count_node_range(0, n) (_kernels.py:40-52) for the whole range,
 * and the per-rank partials of count_space_surrogate for rank buckets. */
int tc_count_middle(const int64_t* tab_indptr, const int32_t* tab_indices,
                    const int64_t* rev_indptr, const int32_t* rev_seg,
                    const int64_t* rev_cost, const int32_t* pool, int32_t pool_padded, int64_t n,
                    int64_t u0, int64_t u1, const int64_t* bucket_bounds, int32_t nbuckets,
                    unsigned long long* out, tc_stream_t stream);

/* The same total by the formulation BASELINE.json's north_star names: one
 * warp per oriented edge (v, u), |N^_v ∩ N^_u| by warp merge-path over both
 * lists staged in shared memory (comparable lengths) or a binary-search
 * probe of the long list (skewed pairs) -- merge_count summed over the
 * edges, _kernels.py:15-52, with the merge model's W list steps.  The
 * measured comparator of the middle-vertex engine, not the
 * headline path.  out: one uint64. */
int tc_count_merge_path(const int64_t* eff_indptr, const int32_t* eff_indices, int64_t n, unsigned long long* out,
                        tc_stream_t stream);

/* Reusable form of tc_count_middle for repeated counts of one graph: the
 * plan (tier lists and chunk boundaries for owners [u0, u1)) is computed
 * once (synchronises); tc_plan_run then only zeroes `out` and launches the
 * engine (no host synchronisation, graph-capturable).  The plan keeps the
 * argument pointers -- the caller keeps those arrays alive and unchanged --
 * and re-plans itself if tc_set_tuning changed the tier caps.  Planning does
 * not synchronise at its end: runs wait on the plan's event (a run captured
 * into a CUDA graph must be captured after the planning stream has
 * synchronised).  Runs of one plan share its chunk-queue counters, so runs
 * issued on different streams are serialised: each run waits on the event
 * the previous run recorded behind its engine launches. */
typedef struct tc_plan_s* tc_plan_t;
int tc_plan_middle(const int64_t* tab_indptr, const int32_t* tab_indices, const int64_t* rev_indptr,
                   const int32_t* rev_seg, const int64_t* rev_cost, const int32_t* pool, int32_t pool_padded,
                   int64_t n, int64_t u0, int64_t u1, const int64_t* bucket_bounds, int32_t nbuckets,
                   tc_plan_t* plan, tc_stream_t stream);
int tc_plan_run(tc_plan_t plan, unsigned long long* out, tc_stream_t stream);
/* Points the plan at another copy of the segment array and the pool with the
 * same structure (same owners, same segments per owner, same segment
 * lengths per owner up to their order): the sharded count's received lists
 * arrive in fresh buffers at every count (tc_shard_index_emit).  Host-side
 * only; runs issued afterwards use the new arrays. */
int tc_plan_rebind(tc_plan_t plan, const int32_t* rev_seg, const int32_t* pool);
int tc_plan_free(tc_plan_t plan);

/* Interleaved split of one plan across `nparts` devices that each hold the
 * whole graph (the replicated multi-GPU count; the work split of
 * dynamic_lb.py:68-109 across ranks instead of one rank's workers): the
 * chunk plan is cut for the workers of all parts, and tc_plan_run_part runs
 * the chunks c with c mod nparts == part (part -1: every chunk, i.e.
 * tc_plan_run).  Every tier is split, so the parts stay balanced whatever
 * the cost model's error between tiers; the part counts sum to the total. */
int tc_plan_middle_parts(const int64_t* tab_indptr, const int32_t* tab_indices, const int64_t* rev_indptr,
                         const int32_t* rev_seg, const int64_t* rev_cost, const int32_t* pool, int32_t pool_padded,
                         int64_t n, int64_t u0, int64_t u1, const int64_t* bucket_bounds, int32_t nbuckets,
                         int32_t nparts, tc_plan_t* plan, tc_stream_t stream);
int tc_plan_run_part(tc_plan_t plan, int32_t part, unsigned long long* out, tc_stream_t stream);

/* Generic engine over k "virtual owners": owner x probes the table list
 * N^_{owner_map[x]} (owner_map NULL: identity) with segments
 * segs[row_indptr[x] .. row_indptr[x+1]) (int32 pairs into `pool`); cost_prefix
 * int64[k+1] drives the chunk plan.  mode 0 = the paper's schedule (half
 * the cost in one chunk per warp, then geometric), mode 1 = owner-ordered
 * uniform chunks then a geometric tail (for L2-tiled owners).  Buckets bin
 * owner_map[x].  out is overwritten. */
int tc_count_owners(const int64_t* tab_indptr, const int32_t* tab_indices, const int32_t* owner_map,
                    const int64_t* row_indptr, const int32_t* segs, const int64_t* cost_prefix,
                    const int32_t* pool, int64_t k, const int64_t* bucket_bounds, int32_t nbuckets,
                    unsigned long long* out, int32_t mode, tc_stream_t stream);

/* L2-tiled regrouping of the predecessor entries of u in [u0, u1): v is cut
 * into tiles of <= tile_ids list entries and entries are ordered
 * (tile(v), u, v); each (tile, u) with entries is one virtual owner.
 * Outputs (capacity E = rev_indptr[u1] - rev_indptr[u0]): owner_u int32[E],
 * owner_ptr int64[E+1], segs int32[2E], cost_prefix int64[E+1]; returns the
 * owner count k and the tile count.  pool_indptr: the row offsets rev_seg's
 * coordinates refer to.  Feed to tc_count_owners (mode 1).
 * Synchronises. */
int tc_tile_pull(const int64_t* eff_indptr, const int64_t* pool_indptr, int64_t n, const int64_t* rev_indptr,
                 const int32_t* rev_seg, int64_t u0, int64_t u1,
                 int64_t tile_ids, int32_t* owner_u, int64_t* owner_ptr, int32_t* segs,
                 int64_t* cost_prefix, int64_t* k_host, int64_t* ntiles_host, tc_stream_t stream);

/* Lowest-vertex ("push") engine: count_node_range(v0, v1)
 * (_kernels.py:40-52) with per-bucket partials: out[b] = triangles whose
 * lowest vertex lies in [bucket_bounds[b], bucket_bounds[b+1]).
 * bucket_bounds NULL with nbuckets==1 means the single range [v0, v1). */
int tc_count_lowest(const int64_t* eff_indptr, const int32_t* eff_indices, int64_t n,
                    int64_t v0, int64_t v1, const int64_t* bucket_bounds, int32_t nbuckets,
                    unsigned long long* out, tc_stream_t stream);

/* Engine timing (measurement only): reports the accumulated device time and
 * launch count of engine kernels since the last reset (tier_ms_host, if not
 * NULL, gets the time of the small / mid / block tiers), then, if
 * enable >= 0, resets the counters and turns CUDA-event bracketing of every
 * engine launch on (1) or off (0).  Bracketing synchronises after each
 * launch. */
int tc_engine_timing(int32_t enable, double* total_ms_host, long long* launches_host, double* tier_ms_host);

/* Engine tier caps (testing / tuning): key 0 = small warp-tier table cap
 * (0..256, default 128; 129..256 force the tier's wide form -- 8 ids of the
 * owner's list per lane -- which the plan otherwise picks itself when the
 * owners with 128 < d^ <= 256 carry a third of the engine's cost),
 * key 2 = mid warp-tier cap (0..512, default 512),
 * key 1 = block-tier staged-table cap (0..4096, default 4096; larger tables
 * use binary search in global memory); value -1 restores a cap's default.
 * key 3 = pairs per chunk of tc_normalize_host's copy pipeline (>= 1,
 * default 2^22; at most 16 chunks). */
int tc_set_tuning(int32_t key, int64_t value);

/* |a ∩ b| of two strictly ascending int32 lists (_kernels.py:15-37). */
int tc_intersect_count(const int32_t* a, int64_t na, const int32_t* b, int64_t nb,
                       unsigned long long* out, tc_stream_t stream);

/* Dense-bitmap brute-force count over the full CSR, n <= 2000
 * (sequential.py:37-51); independent of the engines above. */
int tc_count_brute(const int64_t* full_indptr, const int32_t* full_indices, int64_t n,
                   unsigned long long* out, tc_stream_t stream);

/* ---------------------------------------------------------- partitioning */

/* node_costs (partitioning.py:79-92) -> int64[n]. */
int tc_node_costs(int32_t kind, const int64_t* eff_indptr, const int32_t* eff_indices,
                  const int32_t* deg, const int32_t* eff_deg, int64_t n, int64_t* out,
                  tc_stream_t stream);

/* balanced_ranges (partitioning.py:95-122): bounds int64[k+1] (device)
 * for `costs` restricted to [start, start+count). */
int tc_balanced_bounds(const int64_t* costs, int64_t start, int64_t count, int64_t k,
                       int64_t* bounds, tc_stream_t stream);

/* plan_tasks (dynamic_lb.py:68-109).  initial_bounds int64[nranks]
 * (P-1 ranges), queue_v/queue_t int64[n] capacity, targets f64[n].
 * Synchronises (returns split, nqueue, total). */
int tc_plan_tasks(const int64_t* costs, int64_t n, int64_t nranks, int64_t* initial_bounds,
                  int64_t* queue_v, int64_t* queue_t, double* targets, int64_t* split_host,
                  int64_t* nqueue_host, int64_t* total_host, tc_stream_t stream);

/* Surrogate census (scan_for_surrogate's LastProc records,
 * _kernels.py:94-126): census int64[P*P], census[i*P+j] = number of owned
 * v of rank i whose N^_v has an id owned by j != i.  words int64[P] =
 * sum over those records of (2 + d^_v) (runtime.py:80-86 wire model). */
int tc_surrogate_census(const int64_t* eff_indptr, const int32_t* eff_indices, int64_t n,
                        const int64_t* bounds, int32_t P, long long* census, long long* words,
                        tc_stream_t stream);

/* Owner-change records of one rank (the send list of the surrogate push):
 * for owned v in [bounds[rank], bounds[rank+1]) emits one (v, dest) per
 * remote rank dest > rank touched by N^_v, grouped by dest ascending then v
 * ascending.  The CSR row of global node v is eff_indptr[v - row_base]
 * (row_base = 0 for a whole graph, = bounds[rank] for a rank's shard).
 * rec_v/rec_dest int32[cap]; counts int64[P] per dest.
 * Synchronises (returns the record count). */
int tc_surrogate_records(const int64_t* eff_indptr, const int32_t* eff_indices, int64_t n,
                         const int64_t* bounds, int32_t P, int32_t rank, int64_t row_base, int32_t* rec_v,
                         int32_t* rec_dest, int64_t cap, long long* counts,
                         int64_t* nrec_host, tc_stream_t stream);

/* Packs the N^_v lists of records [r0, r1) into one send buffer:
 * out_len int64[r1-r0] list lengths, out_ids int32[...] concatenated lists,
 * out_v int32[r1-r0] node ids.  out_offsets int64[r1-r0+1] (device) must
 * hold the exclusive prefix of lengths (see tc_surrogate_pack_sizes). */
int tc_surrogate_pack_sizes(const int64_t* eff_indptr, const int32_t* rec_v, int64_t nrec,
                            int64_t* out_offsets, int64_t* total_host, tc_stream_t stream);
int tc_surrogate_pack(const int64_t* eff_indptr, const int32_t* eff_indices,
                      const int32_t* rec_v, int64_t nrec, const int64_t* offsets,
                      int32_t* out_ids, tc_stream_t stream);

/* Pull-engine segments from neighbour lists (surrogate_count_list,
 * _kernels.py:70-80, re-expressed): for list l = ids[off[l], off[l+1]) and
 * every position k holding an owned id u in [lo, hi) with a non-empty
 * suffix, emits owner[i] = u - lo and segs[2i..2i+1] =
 * (pool_base + k + 1, pool_base + off[l+1]) as int32 (the pool must stay
 * below 2^31 ids).  Works for the local shard's own rows and for received
 * lists alike.  owner == NULL only counts; otherwise cap >= the number of
 * ids always suffices.  Segments come in list order, positions ascending.
 * Synchronises (returns the segment count). */
int tc_owner_segments(const int64_t* list_offsets, const int32_t* list_ids, int64_t nl,
                      int64_t lo, int64_t hi, int64_t pool_base, int32_t* owner, int32_t* segs,
                      int64_t cap, int64_t* nseg_host, tc_stream_t stream);

/* Groups segments by owner into a CSR usable by tc_count_middle:
 * row_indptr int64[n_owner+1], row_segs int32[2*nseg], cost_prefix
 * int64[n_owner+1] (pull-engine cost, needs the table CSR tab_indptr). */
int tc_segments_csr(const int32_t* owner, const int32_t* segs, int64_t nseg, int64_t n_owner,
                    const int64_t* tab_indptr, int64_t* row_indptr, int32_t* row_segs,
                    int64_t* cost_prefix, tc_stream_t stream);

/* ------------------------------------------------------------ direct scheme */

/* Direct-scheme census (the per-pair counters of _direct_rank,
 * space_efficient.py:188-231 with runtime.py:139-149 accounting) for all
 * ranks: requests int64[P*P], requests[i*P+j] = number of oriented edges
 * (v, u) with owner(v) = i != owner(u) = j (one TASK_REQUEST each);
 * reply_words int64[P], reply_words[j] = sum over those pairs of
 * (2 + d^_u) (the DATA replies j serves, runtime.py:80-81). */
int tc_direct_census(const int64_t* eff_indptr, const int32_t* eff_indices, int64_t n, const int64_t* bounds,
                     int32_t P, long long* requests, long long* reply_words, tc_stream_t stream);

/* One rank of the deduplicated pull: the distinct ids >= hi named by the
 * shard's lists (shard_indptr int64[nloc+1] local offsets, shard_indices
 * global ids), ascending -- hence grouped by owner -- into req_ids
 * int32[cap], their multiplicities (the reference's per-pair request
 * count) into req_mult int64[cap]; counts int64[P] = distinct ids per owner,
 * ref_counts int64[P] = requests per owner as the reference counts them.
 * cap >= shard_indptr[nloc] always suffices.  Synchronises. */
int tc_direct_requests(const int64_t* shard_indptr, const int32_t* shard_indices, int64_t nloc, int64_t hi,
                       const int64_t* bounds, int32_t P, int32_t* req_ids, int64_t* req_mult, int64_t cap,
                       long long* counts, long long* ref_counts, int64_t* nreq_host, tc_stream_t stream);

/* Lookup CSR of one rank over ids [0, n_rows): row lo+i = the shard's row
 * i, row req_ids[k] has length req_lens[k] (the fetched lists, ascending
 * ids all >= lo + nloc), every other row empty.  out_indptr int64[n_rows+1];
 * the matching indices are the shard's ids followed by the fetched ids. */
int tc_direct_table(const int64_t* shard_indptr, int64_t nloc, int64_t lo, const int32_t* req_ids,
                    const int64_t* req_lens, int64_t nreq, int64_t n_rows, int64_t* out_indptr,
                    tc_stream_t stream);

/* ------------------------------------------------------------ ingestion */

/* load_edge_list (graph_io.py:42-71) on the device: buf = the file's bytes
 * (device).  Lines split on '\n'; blank lines and lines whose first token
 * starts with '#' are skipped; every other line must hold exactly two
 * Python-int() tokens (sign, ASCII digits, single underscores between
 * digits) with non-negative values < 2^31.  On success out_pairs int32
 * [2*cap] (cap >= nbytes/4 + 1 always suffices) gets the pairs in file
 * order and n = max id + 1.  On the first malformed line *err_line_host =
 * its 1-based number, *err_code_host = 2 (token count, *err_tokens_host
 * holds it), 3 (non-integer), 4 (negative) or 5 (exceeds int32).
 * Synchronises. */
int tc_parse_edge_list(const unsigned char* buf, int64_t nbytes, int32_t* out_pairs, int64_t cap,
                       int64_t* m_host, int64_t* n_host, int64_t* err_line_host, int32_t* err_code_host,
                       int32_t* err_tokens_host, tc_stream_t stream);

/* ---------------------------------------------------- sharded multi-GPU */

/* The per-rank steps of the sharded pipeline (sharded.py): rank r holds
 * only its slice of the raw pairs, then its hash share of the deduplicated
 * edges, then the forward lists of its node range -- a distributed
 * graph.normalize + build_graph (graph.py:76-153) with partition_ranges
 * (partitioning.py:139-141) and the surrogate exchange of
 * space_efficient.py:81-144.  The collectives between the steps (all_reduce
 * of the replicated per-label arrays, all_to_all of edges and lists) are
 * the caller's (NCCL).  `pairs` are int32 (u, v) pairs. */

/* Smallest / largest label of the rank's raw slice (negative labels are the
 * caller's ValueError, graph.py:87-88).  Synchronises. */
int tc_shard_minmax(const int32_t* pairs, int64_t m, int32_t* min_host, int32_t* max_host, tc_stream_t stream);
/* present uint8[k] (label occurs in a non-self-loop pair) and first int32[k]
 * (first raveled position 2(pos_base+i)+j, 0x7F7F7F7F if absent) of the
 * slice; the caller all-reduces them (MAX / MIN) across ranks. */
int tc_shard_label_scan(const int32_t* pairs, int64_t m, int64_t pos_base, int64_t k, uint8_t* present,
                        int32_t* first, tc_stream_t stream);
/* From the global present / first arrays: map int32[k] = the label's
 * normalized id (identity when the labels are dense, else first-seen
 * compaction, graph.py:92-99; -1 for absent labels), n = distinct labels.
 * Synchronises. */
int tc_shard_relabel_map(const uint8_t* present, const int32_t* first, int64_t k, int32_t* map, int64_t* n_host,
                         int32_t* dense_host, tc_stream_t stream);
/* Canonical keys (min << 32 | max) of the mapped non-self-loop pairs
 * grouped by destination rank hash(key) mod P (the dedup exchange):
 * keys_out uint64[m], counts_host int64[P].  map NULL = identity.
 * Synchronises. */
int tc_shard_keys(const int32_t* pairs, int64_t m, const int32_t* map, int32_t P, uint64_t* keys_out,
                  int64_t* counts_host, tc_stream_t stream);
/* Sorted distinct keys (np.unique(axis=0), graph.py:100-102); labels <
 * 2^key_bits.  out uint64[k].  Synchronises (returns the count). */
int tc_shard_dedup(const uint64_t* keys, int64_t k, int32_t key_bits, uint64_t* out, int64_t* k_host,
                   tc_stream_t stream);
/* deg int32[n] += both endpoints' counts (graph.py:149-151; caller zeroes
 * and all-reduces). */
int tc_shard_degrees(const uint64_t* keys, int64_t k, int32_t* deg, tc_stream_t stream);
/* Canonical order from the global degrees: orig_ids = ids by ascending
 * (degree, id) (stable, graph.py:152), relabel = its inverse (graph.py:111-112). */
int tc_shard_order(const int32_t* deg, int64_t n, int32_t* orig_ids, int32_t* relabel, tc_stream_t stream);
/* Oriented pairs lohi int32[2k] = (min, max) of the relabelled keys
 * (graph.py:113-116); effdeg int32[n] += out-degree (caller all-reduces). */
int tc_shard_orient(const uint64_t* keys, int64_t k, const int32_t* relabel, int32_t* lohi, int32_t* effdeg,
                    tc_stream_t stream);
/* PRED_SUM contributions (partitioning.py:91): cost[hi] += d^_lo + d^_hi
 * (int64[n], caller zeroes and all-reduces). */
int tc_shard_predsum(const int32_t* lohi, int64_t k, const int32_t* effdeg, int64_t* cost, tc_stream_t stream);
/* Oriented pairs grouped by the owner of lo under bounds int64[P+1]
 * (owner_of, partitioning.py:134-136): out int32[2k], counts_host int64[P].
 * Synchronises. */
int tc_shard_route(const int32_t* lohi, int64_t k, const int64_t* bounds, int32_t P, int32_t* out,
                   int64_t* counts_host, tc_stream_t stream);
/* The rank's forward CSR from its routed pairs (lo in [lo, lo + nrow)):
 * indptr int64[nrow+1] (local offsets), indices int32[k] rows ascending. */
int tc_shard_csr(const int32_t* lohi, int64_t k, int64_t lo, int64_t nrow, int64_t* indptr, int32_t* indices,
                 tc_stream_t stream);
/* Row-padded copy of a CSR for the engine (see tc_build_graph's pool):
 * pool_indptr int64[nrow+1]; pool int32[TC_POOL_HEAD + indptr[nrow] + 3 nrow + 4]
 * passed TC_POOL_HEAD ids past its start. */
int tc_shard_pool(const int64_t* indptr, const int32_t* indices, int64_t nrow, int64_t* pool_indptr, int32_t* pool,
                  tc_stream_t stream);
/* Engine cost of the middle-vertex owners (the pull cost of build_graph's
 * rev_cost): acc uint64[n] += suffix length + seg_weight per predecessor
 * entry of the local rows (caller zeroes, all-reduces); _fin adds the table term
 * tab_weight * d^_u + 16 for owners with work, and send_weight * d^_v for
 * every node (its list's share of the surrogate send) (build_graph's
 * rev_cost is seg_weight 2, tab_weight 1, send_weight 0; the partition
 * weights are sharded.py's). */
int tc_shard_engine_cost(const int64_t* indptr, const int32_t* indices, int64_t nrow, int64_t seg_weight,
                         uint64_t* acc, tc_stream_t stream);
int tc_shard_engine_cost_fin(const uint64_t* acc, const int32_t* effdeg, int64_t n, int64_t tab_weight,
                             int64_t send_weight, int64_t* cost, tc_stream_t stream);
/* Surrogate send plan (_kernels.py:94-126 LastProc records, one message per
 * (v, dest > rank) with an id of N^_v owned by dest; the message is row v of
 * the shard's padded pool from the 16-byte chunk holding its first id >=
 * bounds[dest] on): sizes_dev int64[tc_shard_send_plan_len] = lists, padded
 * words, whole-list words per destination (3P entries; the last is the
 * reference's bytes_sent accounting; copied to sizes_host if not NULL, which
 * synchronises), followed by the pack kernel's per-block first list / word
 * slots (static for a partitioned graph: the pack then runs without a
 * counting pass and without global atomics).  P <= 32. */
int tc_shard_send_plan_len(int64_t nrow, int32_t P, int64_t* len_host);
int tc_shard_send_sizes(const int64_t* indptr, const int32_t* indices, int64_t nrow, const int64_t* pool_indptr,
                        const int64_t* bounds, int32_t P, int32_t rank, int64_t* sizes_dev, int64_t* sizes_host,
                        tc_stream_t stream);
/* The messages, grouped by destination: out_len int32[lists] (ids per
 * message), out_ids int32[words] (padded rows; 16-byte aligned). */
int tc_shard_send_pack(const int64_t* indptr, const int32_t* indices, int64_t nrow, const int64_t* pool_indptr,
                       const int32_t* pool, const int64_t* bounds, int32_t P, int32_t rank, const int64_t* sizes_dev,
                       int32_t* out_len, int32_t* out_ids, tc_stream_t stream);
/* Middle-vertex segments of a set of padded rows (row r: row_len[r] ids at
 * pool_indptr[r], computed here) for owners u in [lo, hi): the suffix of the
 * row after each u (surrogate_count_list, _kernels.py:70-80), grouped by
 * owner -- rev_indptr int64[hi-lo+1], rev_seg int32[2*cap], rev_cost
 * int64[hi-lo+1] (tables tab_indptr indexed u - lo) for tc_plan_middle with
 * pool_padded = 1.  cap >= the number of row entries; pool_words = the ids
 * the rows occupy (a launch-shape hint: short rows get 8 lanes each; 0 =
 * unknown).  nseg_host (nullable) synchronises. */
int tc_shard_index(const int32_t* row_len, int64_t nrow, const int32_t* pool, int64_t pool_words, int64_t lo,
                   int64_t hi, const int64_t* tab_indptr, int64_t* pool_indptr, int64_t* rev_indptr,
                   int32_t* rev_seg, int64_t* rev_cost, int64_t* nseg_host, tc_stream_t stream);

/* The scatter pass of tc_shard_index for rows whose per-owner offsets
 * rev_indptr are kept from an earlier call on lists of the same structure
 * (the same exchange round of the same partitioned graph): fills
 * pool_indptr and rev_seg only. */
int tc_shard_index_emit(const int32_t* row_len, int64_t nrow, const int32_t* pool, int64_t pool_words, int64_t lo,
                        int64_t hi, const int64_t* rev_indptr, int64_t* pool_indptr, int32_t* rev_seg,
                        tc_stream_t stream);

/* ------------------------------------------------------------ NCCL layer */

/* The collectives of the multi-GPU schemes for a caller that binds this
 * library directly: communicator setup, the
 * all-reduce of the per-rank partials (reduce_sum, runtime.py:255-259) and
 * the list exchange of the surrogate scheme (space_efficient.py:116-144) as
 * grouped ncclSend/ncclRecv.  libnccl is loaded at the first call (dlopen of
 * $TCB_NCCL_LIB, else libnccl.so.2); every call is stream-ordered. */
typedef struct tc_nccl_s* tc_nccl_t;
enum { TC_DT_U8 = 0, TC_DT_I32 = 1, TC_DT_I64 = 2, TC_DT_U64 = 3 };
enum { TC_OP_SUM = 0, TC_OP_MAX = 1, TC_OP_MIN = 2 };
/* 128-byte unique id for tc_nccl_init_rank (rank 0 creates, all share). */
int tc_nccl_unique_id(void* id_out);
int tc_nccl_init_rank(const void* id, int32_t nranks, int32_t rank, tc_nccl_t* comm);
/* One process driving ndev GPUs (ncclCommInitAll). */
int tc_nccl_init_all(int32_t ndev, const int32_t* devices, tc_nccl_t* comms);
int tc_nccl_free(tc_nccl_t comm);
/* In-place all-reduce of count elements (TC_DT_*, TC_OP_*). */
int tc_allreduce(void* buf, int64_t count, int32_t dtype, int32_t op, tc_nccl_t comm, tc_stream_t stream);
/* In-place SUM of uint64 counts (the per-rank triangle partials). */
int tc_allreduce_u64(unsigned long long* buf, int64_t count, tc_nccl_t comm, tc_stream_t stream);
/* All-to-all-v: send_counts[p] elements to rank p from consecutive send
 * offsets, recv_counts[p] from rank p into consecutive recv offsets (host
 * count arrays of nranks entries). */
int tc_exchange(const void* send, const int64_t* send_counts, void* recv, const int64_t* recv_counts, int32_t dtype,
                int32_t nranks, tc_nccl_t comm, tc_stream_t stream);
/* tc_exchange of int32 list ids (the surrogate's packed N^_v lists). */
int tc_exchange_lists(const int32_t* send, const int64_t* send_counts, int32_t* recv, const int64_t* recv_counts,
                      int32_t nranks, tc_nccl_t comm, tc_stream_t stream);

/* ------------------------------------------------------------ generators */

/* ER G(n,m) raw pairs (configs 1, 5): out int32[2m]. */
int tc_gen_er(int64_t n, int64_t m, uint64_t seed, int32_t* out, tc_stream_t stream);
/* R-MAT raw pairs (config 4): 2^scale*edge_factor samples, (.57,.19,.19,.05). */
int tc_gen_rmat(int32_t scale, int64_t edge_factor, uint64_t seed, int32_t* out,
                tc_stream_t stream);
/* Chung-Lu raw pairs (config 3), exact model: w_i = c (i+1)^(-1/(gamma-1))
 * capped at w_max and scaled to mean degree `mean`; every pair u < v is an
 * edge independently with p_uv = min(1, w_u w_v / sum w) (geometric-skip
 * sampling per row).  out == NULL returns the edge count only; otherwise
 * out int32[2*cap].  Synchronises (returns m). */
int tc_gen_chung_lu(int64_t n, double mean, double gamma, double w_max, uint64_t seed, int32_t* out,
                    int64_t cap, int64_t* m_host, tc_stream_t stream);
/* Preferential attachment, bit-identical to the reference's pa_edge_list
 * (_kernels.py:129-178; sequential by construction, runs on the host).
 * out_host int32[2*tc_pa_num_edges(n,k)] as (src, dst) pairs. */
int64_t tc_pa_num_edges(int64_t n, int64_t k);
int tc_gen_pa_host(int64_t n, int64_t k, uint64_t seed, int32_t* out_host);

#ifdef __cplusplus
}
#endif

#endif /* TCB200_H */

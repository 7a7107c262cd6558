/*
 * oracle.c -- CPU restatement of the reference `tricount` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") of bench.py.  Nothing in the product package
 * (paper_1406_5687_b200/) links, loads or calls it; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * do.  Parity is pinned: tests/test_oracle_golden.py checks every function
 * here against vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/tricount).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/pkg/src/tricount).  Ids and offsets are int64 like the
 * reference (graph.py:85,111,120).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* LSD radix sort of (uint64 key, int64 payload), stable.  numpy's     */
/* lexsort / unique(axis=0) / argsort(kind="stable") are all stable     */
/* orderings by key, which is what this gives.                          */
/* ------------------------------------------------------------------ */
static void rsort_pairs(uint64_t *key, int64_t *val, int64_t n, int bits) {
    if (n <= 1 || bits <= 0) return;
    uint64_t *k2 = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    int64_t *v2 = val ? (int64_t *)malloc(sizeof(int64_t) * (size_t)n) : NULL;
    uint64_t *ka = key, *kb = k2;
    int64_t *va = val, *vb = v2;
    int passes = (bits + 10) / 11;
    for (int p = 0; p < passes; ++p) {
        int shift = p * 11;
        int64_t cnt[2048];
        memset(cnt, 0, sizeof(cnt));
        for (int64_t i = 0; i < n; ++i) cnt[(ka[i] >> shift) & 2047]++;
        int64_t s = 0;
        for (int b = 0; b < 2048; ++b) { int64_t c = cnt[b]; cnt[b] = s; s += c; }
        for (int64_t i = 0; i < n; ++i) {
            int64_t d = cnt[(ka[i] >> shift) & 2047]++;
            kb[d] = ka[i];
            if (va) vb[d] = va[i];
        }
        uint64_t *tk = ka; ka = kb; kb = tk;
        int64_t *tv = va; va = vb; vb = tv;
    }
    if (ka != key) {
        memcpy(key, ka, sizeof(uint64_t) * (size_t)n);
        if (val) memcpy(val, va, sizeof(int64_t) * (size_t)n);
    }
    free(k2);
    free(v2);
}

static int bits_for(uint64_t maxval) {
    int b = 0;
    while (b < 64 && (maxval >> b)) ++b;
    return b;
}

/* ------------------------------------------------------------------ */
/* normalize: graph.py:76-103                                          */
/* edges: (m_raw, 2) int64.  out_edges must hold m_raw pairs.          */
/* returns 0, or -1 for a negative id (graph.py:87-88 ValueError).     */
/* ------------------------------------------------------------------ */
int or_normalize(const int64_t *edges, int64_t m_raw, int64_t *out_edges,
                 int64_t *out_m, int64_t *out_n) {
    *out_m = 0;
    *out_n = 0;
    for (int64_t i = 0; i < 2 * m_raw; ++i)
        if (edges[i] < 0) return -1;                       /* graph.py:87-88 */
    /* drop self-loops (graph.py:89) */
    int64_t m = 0;
    int64_t *e = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * m_raw + 2));
    for (int64_t i = 0; i < m_raw; ++i) {
        if (edges[2 * i] != edges[2 * i + 1]) {
            e[2 * m] = edges[2 * i];
            e[2 * m + 1] = edges[2 * i + 1];
            ++m;
        }
    }
    if (m == 0) { free(e); return 0; }                      /* graph.py:90-91 */
    /* uniq, first_pos = np.unique(ids, return_index=True)  (graph.py:92-93) */
    int64_t nid = 2 * m;
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)nid);
    int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)nid);
    uint64_t mx = 0;
    for (int64_t i = 0; i < nid; ++i) {
        key[i] = (uint64_t)e[i];
        pos[i] = i;
        if (key[i] > mx) mx = key[i];
    }
    rsort_pairs(key, pos, nid, bits_for(mx));   /* stable: first occurrence first */
    int64_t K = 0;
    int64_t *uniq = (int64_t *)malloc(sizeof(int64_t) * (size_t)nid);
    int64_t *first = (int64_t *)malloc(sizeof(int64_t) * (size_t)nid);
    for (int64_t i = 0; i < nid; ++i) {
        if (i == 0 || key[i] != key[i - 1]) {
            uniq[K] = (int64_t)key[i];
            first[K] = pos[i];
            ++K;
        }
    }
    free(key);
    free(pos);
    if (K > 0 && K != uniq[K - 1] + 1) {
        /* new_id[argsort(first_pos, stable)] = arange(K)   (graph.py:96-97) */
        uint64_t *fk = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)K);
        int64_t *fi = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);
        for (int64_t j = 0; j < K; ++j) { fk[j] = (uint64_t)first[j]; fi[j] = j; }
        rsort_pairs(fk, fi, K, bits_for((uint64_t)nid));
        int64_t *new_id = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);
        for (int64_t r = 0; r < K; ++r) new_id[fi[r]] = r;
        /* compact = new_id[searchsorted(uniq, ids)]  (graph.py:98) */
        for (int64_t i = 0; i < nid; ++i) {
            int64_t lo = 0, hi = K;
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                if (uniq[mid] < e[i]) lo = mid + 1; else hi = mid;
            }
            e[i] = new_id[lo];
        }
        free(fk); free(fi); free(new_id);
    }
    free(uniq);
    free(first);
    /* lo/hi + np.unique(axis=0)  (graph.py:99-102) */
    uint64_t *pk = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)m);
    int b = bits_for((uint64_t)(K - 1));
    if (b == 0) b = 1;
    for (int64_t i = 0; i < m; ++i) {
        int64_t a = e[2 * i], c = e[2 * i + 1];
        int64_t lo = a < c ? a : c, hi = a < c ? c : a;
        pk[i] = ((uint64_t)lo << b) | (uint64_t)hi;
    }
    rsort_pairs(pk, NULL, m, 2 * b);
    int64_t mo = 0;
    uint64_t mask = (b >= 64) ? ~0ULL : ((1ULL << b) - 1);
    for (int64_t i = 0; i < m; ++i) {
        if (i == 0 || pk[i] != pk[i - 1]) {
            out_edges[2 * mo] = (int64_t)(pk[i] >> b);
            out_edges[2 * mo + 1] = (int64_t)(pk[i] & mask);
            ++mo;
        }
    }
    free(pk);
    free(e);
    *out_m = mo;
    *out_n = K;                                             /* graph.py:103 */
    return 0;
}

/* ------------------------------------------------------------------ */
/* build_graph + _assemble + csr: graph.py:106-153                      */
/* order == NULL -> degree order lexsort((arange, deg)) (graph.py:152);  */
/* otherwise the given order (the _build_graph_input_order hook, 156).   */
/* full_* may be NULL to skip the full CSR.                              */
/* ------------------------------------------------------------------ */
int or_build_graph(int64_t n, const int64_t *edges, int64_t m, const int64_t *order_in,
                   int64_t *eff_indptr, int64_t *eff_indices, int64_t *full_indptr,
                   int64_t *full_indices, int64_t *relabel, int64_t *orig_ids,
                   int64_t *deg, int64_t *eff_deg) {
    for (int64_t i = 0; i < 2 * m; ++i)
        if (edges[i] < 0 || edges[i] >= n) return -1;
    int64_t *dg = (int64_t *)calloc((size_t)(n + 1), sizeof(int64_t));
    for (int64_t i = 0; i < 2 * m; ++i) dg[edges[i]]++;    /* graph.py:149-151 */
    if (order_in) {
        for (int64_t i = 0; i < n; ++i) orig_ids[i] = order_in[i];
    } else {
        uint64_t *k = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(n + 1));
        uint64_t mx = 0;
        for (int64_t i = 0; i < n; ++i) {
            k[i] = (uint64_t)dg[i];
            orig_ids[i] = i;
            if (k[i] > mx) mx = k[i];
        }
        rsort_pairs(k, orig_ids, n, bits_for(mx));        /* graph.py:152 */
        free(k);
    }
    for (int64_t i = 0; i < n; ++i) relabel[orig_ids[i]] = i;   /* graph.py:111-112 */
    int b = bits_for((uint64_t)(n > 0 ? n - 1 : 0));
    if (b == 0) b = 1;
    uint64_t mask = (1ULL << b) - 1;
    uint64_t *pk = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(2 * m + 1));
    /* eff CSR (graph.py:113-124): rows=lo, cols=hi, lexsort((cols, rows)) */
    for (int64_t i = 0; i < m; ++i) {
        int64_t a = relabel[edges[2 * i]], c = relabel[edges[2 * i + 1]];
        int64_t lo = a < c ? a : c, hi = a < c ? c : a;
        pk[i] = ((uint64_t)lo << b) | (uint64_t)hi;
    }
    rsort_pairs(pk, NULL, m, 2 * b);
    memset(eff_indptr, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < m; ++i) {
        eff_indptr[(pk[i] >> b) + 1]++;
        eff_indices[i] = (int64_t)(pk[i] & mask);
    }
    for (int64_t v = 0; v < n; ++v) eff_indptr[v + 1] += eff_indptr[v];
    if (full_indptr) {
        /* full CSR (graph.py:125-127): rows = lo||hi, cols = hi||lo */
        for (int64_t i = 0; i < m; ++i) {
            uint64_t lo = pk[i] >> b, hi = pk[i] & mask;
            pk[m + i] = (hi << b) | lo;
        }
        rsort_pairs(pk, NULL, 2 * m, 2 * b);
        memset(full_indptr, 0, sizeof(int64_t) * (size_t)(n + 1));
        for (int64_t i = 0; i < 2 * m; ++i) {
            full_indptr[(pk[i] >> b) + 1]++;
            full_indices[i] = (int64_t)(pk[i] & mask);
        }
        for (int64_t v = 0; v < n; ++v) full_indptr[v + 1] += full_indptr[v];
    }
    for (int64_t v = 0; v < n; ++v) {                      /* graph.py:137-138 */
        deg[v] = dg[orig_ids[v]];
        eff_deg[v] = eff_indptr[v + 1] - eff_indptr[v];
    }
    free(pk);
    free(dg);
    return 0;
}

/* ------------------------------------------------------------------ */
/* merge_count: _kernels.py:15-32                                       */
/* ------------------------------------------------------------------ */
static inline int64_t merge_count(const int64_t *a, int64_t a0, int64_t a1,
                                  const int64_t *b, int64_t b0, int64_t b1) {
    int64_t c = 0, i = a0, j = b0;
    while (i < a1 && j < b1) {
        int64_t x = a[i], y = b[j];
        if (x == y) { ++c; ++i; ++j; }
        else if (x < y) ++i;
        else ++j;
    }
    return c;
}

int64_t or_intersect_size(const int64_t *a, int64_t na, const int64_t *b, int64_t nb) {
    return merge_count(a, 0, na, b, 0, nb);                /* _kernels.py:35-37 */
}

/* count_node_range: _kernels.py:40-52 */
int64_t or_count_node_range(const int64_t *indptr, const int64_t *indices,
                            int64_t start, int64_t stop) {
    int64_t total = 0;
    for (int64_t v = start; v < stop; ++v) {
        int64_t s0 = indptr[v], s1 = indptr[v + 1];
        for (int64_t k = s0; k < s1; ++k) {
            int64_t u = indices[k];
            total += merge_count(indices, s0, s1, indices, indptr[u], indptr[u + 1]);
        }
    }
    return total;
}

/* ------------------------------------------------------------------ */
/* node_costs: partitioning.py:79-92.  kind 0 UNIT, 1 DEGREE,           */
/* 2 SUCC_SUM, 3 PRED_SUM (CostKind order, partitioning.py:32-35).      */
/* ------------------------------------------------------------------ */
int or_node_costs(int kind, int64_t n, const int64_t *eff_indptr, const int64_t *eff_indices,
                  const int64_t *deg, int64_t *out) {
    if (kind < 0 || kind > 3) return -1;
    for (int64_t v = 0; v < n; ++v) out[v] = kind == 0 ? 1 : kind == 1 ? deg[v] : 0;
    if (kind < 2) return 0;
    for (int64_t v = 0; v < n; ++v) {
        int64_t dv = eff_indptr[v + 1] - eff_indptr[v];
        for (int64_t k = eff_indptr[v]; k < eff_indptr[v + 1]; ++k) {
            int64_t u = eff_indices[k];
            int64_t w = dv + (eff_indptr[u + 1] - eff_indptr[u]);   /* partitioning.py:87 */
            out[kind == 2 ? v : u] += w;                             /* :89 / :91 */
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* balanced_ranges: partitioning.py:95-122.  Writes k+1 bounds.         */
/* ------------------------------------------------------------------ */
int or_balanced_bounds(const int64_t *costs, int64_t start, int64_t count, int64_t k,
                       int64_t *bounds) {
    if (k < 1) return -1;                                   /* partitioning.py:104-105 */
    int64_t stop = start + count;
    bounds[0] = start;
    bounds[k] = stop;
    if (k == 1) return 0;
    int64_t total = 0;
    for (int64_t i = start; i < stop; ++i) total += costs[i];
    if (total == 0) {                                       /* :111-112 */
        for (int64_t j = 1; j < k; ++j) bounds[j] = start + (j * count) / k;
        return 0;
    }
    /* cut_j = start + searchsorted(pref, ceil(j*total/k), 'left') + 1 (:113-118) */
    int64_t j = 1;
    int64_t pref = 0;
    for (int64_t i = start; i < stop && j < k; ++i) {
        pref += costs[i];
        while (j < k) {
            __int128 num = (__int128)j * total;
            int64_t thr = (int64_t)((num + k - 1) / k);
            if (pref >= thr) { bounds[j] = i + 1; ++j; } else break;
        }
    }
    for (; j < k; ++j) bounds[j] = stop;
    for (int64_t q = 1; q < k; ++q) if (bounds[q] > stop) bounds[q] = stop;
    return 0;
}

/* ------------------------------------------------------------------ */
/* plan_tasks: dynamic_lb.py:68-109.  queue_v/queue_t must hold n       */
/* entries; initial_bounds nranks entries (P-1 ranges + 1).             */
/* ------------------------------------------------------------------ */
int or_plan_tasks(const int64_t *costs, int64_t n, int64_t nranks, int64_t *split_out,
                  int64_t *initial_bounds, int64_t *queue_v, int64_t *queue_t,
                  double *targets, int64_t *nqueue, int64_t *total_out) {
    if (nranks < 2) return -1;                              /* :76-77 */
    for (int64_t i = 0; i < n; ++i) if (costs[i] < 0) return -2;   /* :79-80 */
    int64_t workers = nranks - 1;
    int64_t *pref = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t acc = 0;
    for (int64_t i = 0; i < n; ++i) { acc += costs[i]; pref[i] = acc; }
    int64_t total = n ? pref[n - 1] : 0;
    int64_t split = 0;
    if (total != 0) {                                       /* :83-88 */
        int64_t half = (total + 1) / 2;
        int64_t lo = 0, hi = n;
        while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (pref[mid] < half) lo = mid + 1; else hi = mid; }
        split = lo + 1;
    }
    or_balanced_bounds(costs, 0, split, workers, initial_bounds);   /* :89 */
    int64_t q_n = 0;
    int64_t pos = split;
    int64_t remaining = total - (split ? pref[split - 1] : 0);
    while (pos < n) {                                       /* :94-102 */
        int64_t threshold = remaining > 0 ? (remaining + workers - 1) / workers : 0;
        int64_t base = pos ? pref[pos - 1] : 0;
        int64_t want = base + threshold;
        int64_t lo = 0, hi = n;
        while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (pref[mid] < want) lo = mid + 1; else hi = mid; }
        int64_t q = lo;
        if (q < pos) q = pos;
        if (q > n - 1) q = n - 1;
        queue_v[q_n] = pos;
        queue_t[q_n] = q - pos + 1;
        targets[q_n] = (double)remaining / (double)workers;
        ++q_n;
        remaining -= pref[q] - base;
        pos = q + 1;
    }
    *split_out = split;
    *nqueue = q_n;
    *total_out = total;
    free(pref);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Surrogate scheme (space_efficient.py:81-144, _kernels.py:70-126).    */
/* Per-rank partials: rank r counts local pairs from scan_for_surrogate */
/* plus surrogate_count_list over every list it receives.  Census       */
/* data_msgs_to[i*P+j] = LastProc records i->j.                         */
/* ------------------------------------------------------------------ */
static int64_t surrogate_count_list(const int64_t *indptr, const int64_t *indices,
                                    int64_t lo, int64_t hi, const int64_t *x, int64_t nx) {
    /* _kernels.py:70-80 */
    int64_t total = 0;
    int64_t a = 0, b = nx;
    while (a < b) { int64_t mid = (a + b) >> 1; if (x[mid] < lo) a = mid + 1; else b = mid; }
    for (int64_t k = a; k < nx && x[k] < hi; ++k) {
        int64_t u = x[k];
        total += merge_count(indices, indptr[u], indptr[u + 1], x, 0, nx);
    }
    return total;
}

int64_t or_surrogate_count_list(const int64_t *indptr, const int64_t *indices, int64_t lo,
                                int64_t hi, const int64_t *x, int64_t nx) {
    return surrogate_count_list(indptr, indices, lo, hi, x, nx);
}

int or_surrogate(const int64_t *indptr, const int64_t *indices, int64_t n,
                 const int64_t *bounds, int64_t P, int64_t *partials, int64_t *census) {
    (void)n;
    for (int64_t i = 0; i < P; ++i) partials[i] = 0;
    for (int64_t i = 0; i < P * P; ++i) census[i] = 0;
    for (int64_t r = 0; r < P; ++r) {
        int64_t lo = bounds[r], hi = bounds[r + 1];
        for (int64_t v = lo; v < hi; ++v) {               /* scan_for_surrogate :94-126 */
            int64_t s0 = indptr[v], s1 = indptr[v + 1];
            int64_t last = -1, seg = 0;
            for (int64_t k = s0; k < s1; ++k) {
                int64_t u = indices[k];
                if (lo <= u && u < hi) {
                    partials[r] += merge_count(indices, s0, s1, indices, indptr[u], indptr[u + 1]);
                } else {
                    while (bounds[seg + 1] <= u) ++seg;
                    if (seg != last) {
                        census[r * P + seg]++;
                        /* receiver: surrogate_count_list (space_efficient.py:93-97) */
                        partials[seg] += surrogate_count_list(indptr, indices, bounds[seg],
                                                              bounds[seg + 1], indices + s0, s1 - s0);
                        last = seg;
                    }
                }
            }
        }
    }
    return 0;
}

/* Direct scheme (space_efficient.py:188-231): rank r counts
 * count_node_range(lo, hi) itself (count_local_pairs + intersect_size with
 * each fetched N^_u); one TASK_REQUEST per cross pair (v, u) to owner(u)
 * (207-209), answered by one data_msg of 2 + d^_u words (runtime.py:80-81,
 * space_efficient.py:195-197). */
int or_direct(const int64_t *indptr, const int64_t *indices, int64_t n, const int64_t *bounds,
              int64_t P, int64_t *partials, int64_t *requests, int64_t *reply_words) {
    (void)n;
    for (int64_t i = 0; i < P; ++i) partials[i] = reply_words[i] = 0;
    for (int64_t i = 0; i < P * P; ++i) requests[i] = 0;
    for (int64_t r = 0; r < P; ++r) {
        int64_t lo = bounds[r], hi = bounds[r + 1];
        for (int64_t v = lo; v < hi; ++v) {
            int64_t s0 = indptr[v], s1 = indptr[v + 1], seg = r;
            for (int64_t k = s0; k < s1; ++k) {
                int64_t u = indices[k];
                partials[r] += merge_count(indices, s0, s1, indices, indptr[u], indptr[u + 1]);
                if (u >= hi) {
                    while (bounds[seg + 1] <= u) ++seg;
                    requests[r * P + seg]++;
                    reply_words[seg] += 2 + (indptr[u + 1] - indptr[u]);
                }
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* pa_edge_list: _kernels.py:129-178 (splitmix64, resample duplicates) */
/* ------------------------------------------------------------------ */
int64_t or_pa_num_edges(int64_t n, int64_t k) { return k * (k + 1) / 2 + (n - k - 1) * k; }

int or_pa_edge_list(int64_t n, int64_t k, uint64_t seed, int64_t *src, int64_t *dst) {
    int64_t m = or_pa_num_edges(n, k);
    int64_t *rep = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * m + 2));
    int64_t *picks = (int64_t *)malloc(sizeof(int64_t) * (size_t)(k + 1));
    int64_t e = 0, r = 0;
    for (int64_t a = 0; a < k + 1; ++a)
        for (int64_t b = a + 1; b < k + 1; ++b) {
            src[e] = a; dst[e] = b; ++e;
            rep[r] = a; rep[r + 1] = b; r += 2;
        }
    uint64_t state = seed;
    for (int64_t v = k + 1; v < n; ++v) {
        for (int64_t t = 0; t < k; ++t) {
            int64_t cand;
            for (;;) {
                state += 0x9E3779B97F4A7C15ULL;
                uint64_t z = state;
                z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
                z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
                z = z ^ (z >> 31);
                cand = rep[z % (uint64_t)r];
                int fresh = 1;
                for (int64_t q = 0; q < t; ++q) if (picks[q] == cand) { fresh = 0; break; }
                if (fresh) break;
            }
            picks[t] = cand;
        }
        for (int64_t t = 0; t < k; ++t) {
            src[e] = picks[t]; dst[e] = v; ++e;
            rep[r] = v; rep[r + 1] = picks[t]; r += 2;
        }
    }
    free(rep);
    free(picks);
    return 0;
}

/* ------------------------------------------------------------------ */
/* count_dynamic's CPU execution (dynamic_lb.py:121-209) on host        */
/* threads: the coordinator's queue becomes an atomic task index, the   */
/* P-1 workers are pthreads running count_node_range (GIL-free numba    */
/* kernels in the reference, _kernels.py:12).  This is the CPU          */
/* baseline timed by bench.py.  Tasks: [tv[i], tv[i]+tt[i]).            */
/* ------------------------------------------------------------------ */
typedef struct {
    const int64_t *indptr, *indices, *tv, *tt;
    int64_t ntask;
    volatile int64_t *next;
    int64_t result;
} or_worker_t;

static void *or_worker(void *arg) {
    or_worker_t *w = (or_worker_t *)arg;
    int64_t total = 0;
    for (;;) {
        int64_t i = __atomic_fetch_add(w->next, 1, __ATOMIC_RELAXED);
        if (i >= w->ntask) break;
        total += or_count_node_range(w->indptr, w->indices, w->tv[i], w->tv[i] + w->tt[i]);
    }
    w->result = total;
    return NULL;
}

int64_t or_count_tasks_threaded(const int64_t *indptr, const int64_t *indices,
                                const int64_t *tv, const int64_t *tt, int64_t ntask,
                                int nthreads) {
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    or_worker_t *ws = (or_worker_t *)malloc(sizeof(or_worker_t) * (size_t)nthreads);
    volatile int64_t next = 0;
    for (int t = 0; t < nthreads; ++t) {
        ws[t].indptr = indptr; ws[t].indices = indices; ws[t].tv = tv; ws[t].tt = tt;
        ws[t].ntask = ntask; ws[t].next = &next; ws[t].result = 0;
        pthread_create(&th[t], NULL, or_worker, &ws[t]);
    }
    int64_t total = 0;
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        total += ws[t].result;
    }
    free(th);
    free(ws);
    return total;
}

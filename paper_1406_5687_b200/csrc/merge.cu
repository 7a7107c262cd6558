// merge.cu -- the list-intersection engine in the form BASELINE.json's
// north_star spells out: one warp per oriented edge (v, u), |N^_v ∩ N^_u| by
//   * warp merge-path for lists of comparable length: both lists are staged
//     in shared memory with coalesced 4-byte loads, the merge path of their
//     a + b steps is cut into 32 equal diagonals (one binary search per lane)
//     and every lane merges its piece;
//   * a shared-memory-staged binary-search probe for skewed pairs: the lanes
//     take the ids of the short list and search the long one.
// This is merge_count per oriented edge summed over the graph, i.e.
// count_node_range(0, n) (_kernels.py:15-52), with the work of SURVEY.md
// §8(d)'s merge model: W = sum over edges of (d^_v + d^_u) list steps.
//
// It is the measured comparator of DESIGN.md §3.2, not the headline path:
// the middle-vertex engine (count.cu) probes sum_v C(d^_v, 2) ids, 4x fewer
// than W at cfg 2, and never re-reads N^_u per edge.  Both give the same
// count on every test (tests/test_gpu_parity.py::test_merge_path_engine).
#include "common.cuh"

namespace tcb {

static constexpr int kMpWarps = 8;      // warps per block
static constexpr int kMpStage = 512;    // ids staged per warp (both lists)
static constexpr int kMpRows = 4;       // rows per queue ticket
static constexpr int kMpSkew = 8;       // binary-search probe when one list is 8x the other

// |A ∩ B| of two ascending shared-memory lists by warp merge-path: lane l
// owns steps [l * per, (l + 1) * per) of the a + b merge steps, A first on
// ties; an equal pair is counted at the step that takes its A element.
__device__ __forceinline__ uint32_t mp_merge(const int32_t* A, int a, const int32_t* B, int b, int lane) {
  const int total = a + b, per = (total + 31) >> 5;
  const int d0 = min(lane * per, total), d1 = min(d0 + per, total);
  int lo = max(0, d0 - b), hi = min(d0, a);  // A elements among the first d0 steps
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A[mid] <= B[d0 - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  int i = lo, j = d0 - lo;
  uint32_t c = 0;
  for (int s = d0; s < d1; ++s) {
    const bool takeA = i < a && (j >= b || A[i] <= B[j]);
    if (takeA) {
      c += (j < b && A[i] == B[j]);
      ++i;
    } else {
      ++j;
    }
  }
  return c;
}

// |S ∩ L| for a short list S and a long list L: lanes probe L by binary search.
__device__ __forceinline__ uint32_t mp_search(const int32_t* S, int s, const int32_t* L, int l, int lane) {
  uint32_t c = 0;
  for (int k = lane; k < s; k += 32) {
    const int32_t x = S[k];
    int lo = 0, hi = l;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (L[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    c += (lo < l && L[lo] == x);
  }
  return c;
}

__global__ void __launch_bounds__(kMpWarps * 32) k_merge_path(const int64_t* __restrict__ indptr,
                                                               const int32_t* __restrict__ indices, int64_t n,
                                                               int* queue, unsigned long long* out) {
  __shared__ int32_t stage[kMpWarps][kMpStage];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* buf = stage[warp];
  unsigned long long acc = 0;
  for (;;) {
    int64_t v0 = 0;
    if (lane == 0) v0 = (int64_t)atomicAdd(queue, 1) * kMpRows;
    v0 = __shfl_sync(0xffffffffu, v0, 0);
    if (v0 >= n) break;
    const int64_t v1 = min(n, v0 + kMpRows);
    for (int64_t v = v0; v < v1; ++v) {
      const int64_t r0 = __ldg(&indptr[v]), r1 = __ldg(&indptr[v + 1]);
      uint32_t c = 0;
      for (int64_t e = r0; e + 1 < r1; ++e) {  // the last id of a row has an empty suffix
        // A = the part of N^_v after u (ids <= u cannot be in N^_u), B = N^_u
        const int32_t u = __ldg(&indices[e]);
        const int64_t b0 = __ldg(&indptr[u]);
        const int a = (int)(r1 - e - 1), b = (int)(__ldg(&indptr[u + 1]) - b0);
        if (b == 0) continue;
        const int32_t* A = indices + e + 1;
        const int32_t* B = indices + b0;
        const bool staged = a + b <= kMpStage;
        __syncwarp();
        if (staged) {  // coalesced loads of both lists
          for (int k = lane; k < a; k += 32) buf[k] = __ldg(&A[k]);
          for (int k = lane; k < b; k += 32) buf[a + k] = __ldg(&B[k]);
          __syncwarp();
          A = buf;
          B = buf + a;
        }
        if (a * kMpSkew < b) c += mp_search(A, a, B, b, lane);
        else if (b * kMpSkew < a) c += mp_search(B, b, A, a, lane);
        else c += mp_merge(A, a, B, b, lane);
      }
      acc += c;
    }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc) atomicAdd(out, acc);
}

}  // namespace tcb

using namespace tcb;

extern "C" {

int tc_count_merge_path(const int64_t* eff_indptr, const int32_t* eff_indices, int64_t n, unsigned long long* out,
                        tc_stream_t stream) {
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    TC_REQUIRE(n >= 0, TC_EINVAL, "negative node count");
    TC_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), s));
    if (n < 3) return;
    Scratch sc(s);
    int* queue = sc.alloc<int>(1);
    TC_CUDA(cudaMemsetAsync(queue, 0, sizeof(int), s));
    int per_sm = 0;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_merge_path, kMpWarps * 32, 0));
    k_merge_path<<<std::max(per_sm, 1) * sm_count(), kMpWarps * 32, 0, s>>>(eff_indptr, eff_indices, n, queue, out);
    check_launch();
  });
}

}  // extern "C"

// gen.cu -- seeded synthetic inputs for the five BASELINE configs.
//
// Device generators (configs 1, 4, 5) are counter-based: draw i of stream s
// is mix(key(seed, s) + (i+1) * GAMMA) with the splitmix64 finaliser, so any
// thread can produce any edge independently.  oracle/gen_twin.py is the
// bit-identical numpy statement of the same streams (tests compare them).
//
// Preferential attachment (config 2) is the reference's own generator
// (_kernels.py:129-178): sequential by construction (each pick reads the
// endpoint multiset built by earlier picks, duplicates are re-drawn), so it
// runs on the host and is bit-identical to pa_edge_list.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"

namespace tcb {

static constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
static constexpr uint64_t kSeedMul = 0xD1B54A32D192ED03ull;
static constexpr uint64_t kStreamEr = 1, kStreamRmat = 2, kStreamCl = 3;
// (a, a+b, a+b+c) = (0.57, 0.76, 0.95) as fractions of 2^64
static constexpr uint64_t kRmatT0 = 0x91eb851eb851e800ull;
static constexpr uint64_t kRmatT1 = 0xc28f5c28f5c29000ull;
static constexpr uint64_t kRmatT2 = 0xf333333333333000ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t s) {
  return mix64(seed * kSeedMul + s);
}
__device__ __forceinline__ uint64_t rnd(uint64_t key, uint64_t i) { return mix64(key + (i + 1) * kGamma); }
__device__ __forceinline__ uint32_t mulhi_n(uint64_t r, uint64_t n) { return (uint32_t)__umul64hi(r, n); }

__global__ void k_gen_er(int64_t n, int64_t m, uint64_t key, int32_t* out) {
  GRID_STRIDE(i, m) {
    uint64_t u = mulhi_n(rnd(key, 2 * (uint64_t)i), (uint64_t)n);
    uint64_t v = mulhi_n(rnd(key, 2 * (uint64_t)i + 1), (uint64_t)n);
    reinterpret_cast<int2*>(out)[i] = make_int2((int)u, (int)v);
  }
}

__global__ void k_gen_rmat(int scale, int64_t ns, uint64_t key, int32_t* out) {
  GRID_STRIDE(i, ns) {
    uint32_t src = 0, dst = 0;
    for (int l = 0; l < scale; ++l) {
      uint64_t r = rnd(key, (uint64_t)i * scale + l);
      uint32_t sb = r >= kRmatT1;
      uint32_t db = (r >= kRmatT0 && r < kRmatT1) || r >= kRmatT2;
      src |= sb << (scale - 1 - l);
      dst |= db << (scale - 1 - l);
    }
    reinterpret_cast<int2*>(out)[i] = make_int2((int)src, (int)dst);
  }
}

// Chung-Lu, exact model: row u draws every v > u independently with
// p_uv = min(1, w_u w_v / S) by geometric skips under the current bound p
// (weights are non-increasing in the id), accepting a landing v with
// probability p_uv / p (Miller & Hagberg 2011).  Row u uses draws
// (u << 32) + j of stream kStreamCl, so the count pass and the write pass
// see the same sequence.  Uniforms are (r >> 11 + 1) * 2^-53 in (0, 1].
__device__ __forceinline__ double unif(uint64_t key, uint64_t i) {
  return (double)((rnd(key, i) >> 11) + 1) * 0x1.0p-53;
}

template <bool kWrite>
__global__ void k_gen_cl(const double* __restrict__ w, int64_t n, double S, uint64_t key,
                         const long long* __restrict__ off, int32_t* out, long long* cnt) {
  GRID_STRIDE(u, n) {
    const double wu = w[u];
    uint64_t j = (uint64_t)u << 32;
    long long k = kWrite ? off[u] : 0;
    int64_t v = u + 1;
    double p = 1.0;
    while (v < n) {
      p = fmin(1.0, __dmul_rn(wu, w[v]) / S);
      if (p <= 0.0) break;
      if (p < 1.0) {
        double r = unif(key, j++);
        double skip = floor(log(r) / log1p(-p));
        if (skip >= (double)(n - v)) break;
        v += (int64_t)skip;
        double q = fmin(1.0, __dmul_rn(wu, w[v]) / S);
        if (unif(key, j++) >= q / p) {
          ++v;
          continue;
        }
      }
      if (kWrite) reinterpret_cast<int2*>(out)[k] = make_int2((int)u, (int)v);
      ++k;
      ++v;
    }
    if (!kWrite) cnt[u] = k;
  }
}

}  // namespace tcb

extern "C" {

int tc_gen_er(int64_t n, int64_t m, uint64_t seed, int32_t* out, tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(n > 0 && n < (1ll << 31), TC_EINVAL, "n must be in [1, 2^31)");
    TC_REQUIRE(m >= 0, TC_EINVAL, "m must be >= 0");
    if (m == 0) return;
    cudaStream_t s = (cudaStream_t)stream;
    tcb::k_gen_er<<<tcb::grid_for(m, 256, tcb::sm_count() * 16), 256, 0, s>>>(
        n, m, tcb::stream_key(seed, tcb::kStreamEr), out);
    tcb::check_launch();
  });
}

int tc_gen_rmat(int32_t scale, int64_t edge_factor, uint64_t seed, int32_t* out, tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(scale >= 1 && scale <= 30, TC_EINVAL, "scale must be in [1, 30]");
    TC_REQUIRE(edge_factor >= 1, TC_EINVAL, "edge_factor must be >= 1");
    int64_t ns = (1ll << scale) * edge_factor;
    cudaStream_t s = (cudaStream_t)stream;
    tcb::k_gen_rmat<<<tcb::grid_for(ns, 256, tcb::sm_count() * 16), 256, 0, s>>>(
        scale, ns, tcb::stream_key(seed, tcb::kStreamRmat), out);
    tcb::check_launch();
  });
}

// Chung-Lu weights: w_i = c (i+1)^(-1/(gamma-1)) capped at w_max, with c
// chosen so that sum_i w_i = mean * n (the cap is solved exactly: the k
// capped entries contribute k * w_max).
static void chung_lu_weights(int64_t n, double mean, double gamma, double w_max, std::vector<double>& w) {
  const double a = 1.0 / (gamma - 1.0);
  w.resize((size_t)n);
  for (int64_t i = 0; i < n; ++i) w[i] = std::pow((double)(i + 1), -a);
  std::vector<double> suffix((size_t)n + 1, 0.0);
  for (int64_t i = n - 1; i >= 0; --i) suffix[i] = suffix[i + 1] + w[i];
  const double target = mean * (double)n;
  double c = target / suffix[0];
  for (int64_t k = 0; k < n; ++k) {  // k = number of capped entries
    c = (target - (double)k * w_max) / suffix[k];
    if (c * w[k] <= w_max) break;
  }
  for (int64_t i = 0; i < n; ++i) w[i] = std::min(c * w[i], w_max);
}

int tc_gen_chung_lu(int64_t n, double mean, double gamma, double w_max, uint64_t seed, int32_t* out,
                    int64_t cap, int64_t* m_host, tc_stream_t stream) {
  return tcb::guarded([&] {
    TC_REQUIRE(n > 1 && n < (1ll << 31), TC_EINVAL, "n must be in [2, 2^31)");
    TC_REQUIRE(gamma > 1.0 && mean > 0.0 && w_max > 0.0, TC_EINVAL, "bad Chung-Lu parameters");
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<double> w;
    chung_lu_weights(n, mean, gamma, w_max, w);
    double S = 0.0;
    for (double x : w) S += x;
    tcb::Scratch sc(s);
    double* dw = sc.alloc<double>(n);
    TC_CUDA(cudaMemcpyAsync(dw, w.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    long long* cnt = sc.alloc<long long>(n + 1);
    long long* off = sc.alloc<long long>(n + 1);
    TC_CUDA(cudaMemsetAsync(cnt + n, 0, sizeof(long long), s));
    const uint64_t key = tcb::stream_key(seed, tcb::kStreamCl);
    const int grid = tcb::grid_for(n, 128, tcb::sm_count() * 32);
    tcb::k_gen_cl<false><<<grid, 128, 0, s>>>(dw, n, S, key, nullptr, nullptr, cnt);
    tcb::check_launch();
    size_t tmp = 0;
    TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, off, n + 1, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, cnt, off, n + 1, s));
    long long m = 0;
    TC_CUDA(cudaMemcpyAsync(&m, off + n, sizeof(long long), cudaMemcpyDeviceToHost, s));
    tcb::sync_stream(s);
    *m_host = m;
    if (!out) return;  // size query
    TC_REQUIRE(m <= cap, TC_EINVAL, "output buffer too small");
    tcb::k_gen_cl<true><<<grid, 128, 0, s>>>(dw, n, S, key, off, out, nullptr);
    tcb::check_launch();
    tcb::sync_stream(s);
  });
}

int64_t tc_pa_num_edges(int64_t n, int64_t k) { return k * (k + 1) / 2 + (n - k - 1) * k; }

// _kernels.py:129-178, restated on int32 ids (the endpoint multiset `rep`
// needs 2m entries; picks are compared against earlier picks of the node).
int tc_gen_pa_host(int64_t n, int64_t k, uint64_t seed, int32_t* out_host) {
  return tcb::guarded([&] {
    TC_REQUIRE(k >= 1 && n > k, TC_EINVAL, "need n > k >= 1");
    TC_REQUIRE(n < (1ll << 31), TC_EINVAL, "n must fit int32 ids");
    int64_t m = tc_pa_num_edges(n, k);
    std::vector<int32_t> rep((size_t)(2 * m));
    std::vector<int32_t> picks((size_t)k);
    int64_t e = 0, r = 0;
    for (int64_t a = 0; a < k + 1; ++a)
      for (int64_t b = a + 1; b < k + 1; ++b) {
        out_host[2 * e] = (int32_t)a;
        out_host[2 * e + 1] = (int32_t)b;
        ++e;
        rep[r] = (int32_t)a;
        rep[r + 1] = (int32_t)b;
        r += 2;
      }
    uint64_t state = seed;
    for (int64_t v = k + 1; v < n; ++v) {
      for (int64_t t = 0; t < k; ++t) {
        int32_t cand;
        for (;;) {
          state += tcb::kGamma;
          uint64_t z = tcb::mix64(state);
          cand = rep[z % (uint64_t)r];
          bool fresh = true;
          for (int64_t q = 0; q < t; ++q)
            if (picks[q] == cand) {
              fresh = false;
              break;
            }
          if (fresh) break;
        }
        picks[t] = cand;
      }
      for (int64_t t = 0; t < k; ++t) {
        out_host[2 * e] = picks[t];
        out_host[2 * e + 1] = (int32_t)v;
        ++e;
        rep[r] = (int32_t)v;
        rep[r + 1] = picks[t];
        r += 2;
      }
    }
  });
}

}  // extern "C"

// parse.cu -- edge-list text ingestion on the device (graph_io.py:42-71).
//
// The reference parses line by line in Python: lines split on b'\n',
// `line.strip()`, skip blank lines and lines starting with '#', exactly two
// whitespace-separated tokens, each parsed with int() (optional sign, ASCII
// digits, single underscores between digits), negative ids rejected, and the
// FIRST malformed line raises EdgeListParseError(lineno).  Here: one pass
// marks line starts, a scan numbers them, one thread parses each line, the
// first error is an atomicMin over line numbers, and valid pairs are
// compacted in line order.  Byte-level, HBM-bound work (no tensor cores).
#include <cub/cub.cuh>

#include "common.cuh"

namespace tcb {

enum : int { kLineOk = 0, kLineSkip = 1, kLineTokens = 2, kLineNonInt = 3, kLineNegative = 4, kLineTooBig = 5 };

// Python str.isspace() over ASCII: \t \n \v \f \r \x1c-\x1f and ' '.
__device__ __forceinline__ bool py_space(unsigned char c) {
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}

// int() of one token [p, q); returns status, value in *v (int64, saturating).
__device__ int parse_int(const unsigned char* __restrict__ b, int64_t p, int64_t q, int64_t* v) {
  bool neg = false;
  if (p < q && (b[p] == '+' || b[p] == '-')) {
    neg = b[p] == '-';
    ++p;
  }
  if (p >= q) return kLineNonInt;
  int64_t x = 0;
  bool big = false, prev_digit = false;
  for (int64_t i = p; i < q; ++i) {
    const unsigned char c = b[i];
    if (c >= '0' && c <= '9') {
      if (x > (INT64_MAX - 9) / 10) big = true;
      else x = x * 10 + (c - '0');
      prev_digit = true;
    } else if (c == '_' && prev_digit && i + 1 < q && b[i + 1] >= '0' && b[i + 1] <= '9') {
      prev_digit = false;
    } else {
      return kLineNonInt;
    }
  }
  if (neg && (x != 0 || big)) return kLineNegative;
  if (big || x > 0x7FFFFFFFll) return kLineTooBig;
  *v = x;
  return kLineOk;
}

__global__ void k_line_flags(const unsigned char* __restrict__ b, int64_t nb, int32_t* flag) {
  GRID_STRIDE(i, nb) flag[i] = (i == 0) || (b[i - 1] == '\n');
}

__global__ void k_line_starts(const int32_t* __restrict__ flag, const int64_t* __restrict__ pos, int64_t nb,
                              int64_t* starts) {
  GRID_STRIDE(i, nb) if (flag[i]) starts[pos[i]] = i;
}

// Thread per line: status, token count and the pair.
__global__ void k_parse_lines(const unsigned char* __restrict__ b, int64_t nb, const int64_t* __restrict__ starts,
                              int64_t nlines, int32_t* status, int32_t* ntok, int2* pair,
                              unsigned long long* first_err, int* maxid) {
  int mx = -1;
  GRID_STRIDE(l, nlines) {
    const int64_t s = starts[l];
    const int64_t e = (l + 1 < nlines) ? starts[l + 1] : nb;  // [s, e) includes the '\n'
    int64_t tb[3], te[3];
    int k = 0;
    int64_t i = s;
    while (i < e) {
      while (i < e && py_space(b[i])) ++i;
      if (i >= e) break;
      const int64_t t0 = i;
      while (i < e && !py_space(b[i])) ++i;
      if (k < 3) {
        tb[k] = t0;
        te[k] = i;
      }
      ++k;
    }
    int st;
    int64_t u = 0, v = 0;
    if (k == 0 || b[tb[0]] == '#') st = kLineSkip;
    else if (k != 2) st = kLineTokens;
    else {
      int s0 = parse_int(b, tb[0], te[0], &u);
      int s1 = parse_int(b, tb[1], te[1], &v);
      // Python evaluates both int() before the sign check: a non-integer
      // token anywhere wins over a negative one.
      if (s0 == kLineNonInt || s1 == kLineNonInt) st = kLineNonInt;
      else if (s0 == kLineNegative || s1 == kLineNegative) st = kLineNegative;
      else if (s0 == kLineTooBig || s1 == kLineTooBig) st = kLineTooBig;
      else st = kLineOk;
    }
    status[l] = st;
    ntok[l] = k;
    pair[l] = make_int2((int)u, (int)v);
    if (st >= kLineTokens) atomicMin(first_err, (unsigned long long)l);
    if (st == kLineOk) mx = max(mx, (int)max(u, v));
  }
  typedef cub::BlockReduce<int, 256> R;
  __shared__ typename R::TempStorage tmp;
  int bm = R(tmp).Reduce(mx, cub::Max());
  if (threadIdx.x == 0) atomicMax(maxid, bm);
}

struct LineOk {
  const int32_t* status;
  __host__ __device__ bool operator()(const int64_t& l) const { return status[l] == kLineOk; }
};

__global__ void k_gather_pairs(const int2* __restrict__ pair, const int64_t* __restrict__ idx, int64_t m,
                               int2* out) {
  GRID_STRIDE(i, m) out[i] = pair[idx[i]];
}

}  // namespace tcb

extern "C" int tc_parse_edge_list(const unsigned char* buf, int64_t nbytes, int32_t* out_pairs, int64_t cap,
                                  int64_t* m_host, int64_t* n_host, int64_t* err_line_host, int32_t* err_code_host,
                                  int32_t* err_tokens_host, tc_stream_t stream) {
  return tcb::guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    *m_host = 0;
    *n_host = 0;
    *err_line_host = 0;
    *err_code_host = 0;
    *err_tokens_host = 0;
    if (nbytes <= 0) return;
    tcb::Scratch sc(s);
    const int sms = tcb::sm_count();
    int32_t* flag = sc.alloc<int32_t>(nbytes);
    int64_t* pos = sc.alloc<int64_t>(nbytes + 1);
    tcb::k_line_flags<<<tcb::grid_for(nbytes, 256, sms * 16), 256, 0, s>>>(buf, nbytes, flag);
    tcb::check_launch();
    size_t tmp = 0;
    TC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag, pos, nbytes, s));
    void* t = sc.bytes(tmp);
    TC_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, flag, pos, nbytes, s));
    int64_t hl[2];
    int32_t hf = 0;
    TC_CUDA(cudaMemcpyAsync(&hl[0], pos + nbytes - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaMemcpyAsync(&hf, flag + nbytes - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    tcb::sync_stream(s);
    const int64_t nlines = hl[0] + hf;
    int64_t* starts = sc.alloc<int64_t>(nlines);
    tcb::k_line_starts<<<tcb::grid_for(nbytes, 256, sms * 16), 256, 0, s>>>(flag, pos, nbytes, starts);
    tcb::check_launch();
    int32_t* status = sc.alloc<int32_t>(nlines);
    int32_t* ntok = sc.alloc<int32_t>(nlines);
    int2* pair = sc.alloc<int2>(nlines);
    auto* ctl = sc.alloc<unsigned long long>(1);
    int* mx = sc.alloc<int>(1);
    const unsigned long long none = ~0ull;
    const int minus1 = -1;
    TC_CUDA(cudaMemcpyAsync(ctl, &none, sizeof(none), cudaMemcpyHostToDevice, s));
    TC_CUDA(cudaMemcpyAsync(mx, &minus1, sizeof(int), cudaMemcpyHostToDevice, s));
    tcb::k_parse_lines<<<tcb::grid_for(nlines, 256, sms * 16), 256, 0, s>>>(buf, nbytes, starts, nlines, status, ntok,
                                                                           pair, ctl, mx);
    tcb::check_launch();
    unsigned long long herr = 0;
    int hmx = -1;
    TC_CUDA(cudaMemcpyAsync(&herr, ctl, sizeof(herr), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaMemcpyAsync(&hmx, mx, sizeof(int), cudaMemcpyDeviceToHost, s));
    tcb::sync_stream(s);
    if (herr != none) {
      int32_t st = 0, nt = 0;
      TC_CUDA(cudaMemcpyAsync(&st, status + herr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      TC_CUDA(cudaMemcpyAsync(&nt, ntok + herr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      tcb::sync_stream(s);
      *err_line_host = (int64_t)herr + 1;  // 1-based, like enumerate(stream, start=1)
      *err_code_host = st;
      *err_tokens_host = nt;
      return;
    }
    // compact the valid pairs in line order
    int64_t* idx = sc.alloc<int64_t>(nlines);
    int64_t* nsel = sc.alloc<int64_t>(1);
    {
      size_t tmp2 = 0;
      cub::CountingInputIterator<int64_t> it(0);
      tcb::LineOk pred{status};
      TC_CUDA(cub::DeviceSelect::If(nullptr, tmp2, it, idx, nsel, nlines, pred, s));
      void* t2 = sc.bytes(tmp2);
      TC_CUDA(cub::DeviceSelect::If(t2, tmp2, it, idx, nsel, nlines, pred, s));
    }
    int64_t m = 0;
    TC_CUDA(cudaMemcpyAsync(&m, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    tcb::sync_stream(s);
    TC_REQUIRE(m <= cap, TC_EINVAL, "output buffer too small");
    if (m) {
      tcb::k_gather_pairs<<<tcb::grid_for(m, 256, sms * 16), 256, 0, s>>>(pair, idx, m,
                                                                         reinterpret_cast<int2*>(out_pairs));
      tcb::check_launch();
    }
    tcb::sync_stream(s);
    *m_host = m;
    *n_host = m ? (int64_t)hmx + 1 : 0;
  });
}

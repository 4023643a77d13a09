// Edge-list text -> canonical graph, parsed on the device.
//
// Restates reference graph.py:132-180 (parse_edge_list) for a byte buffer:
//   * lines end at '\n'; each line is stripped of ASCII whitespace
//     (" \t\n\r\v\f", what str.strip()/split() remove);
//   * blank lines are skipped; "%%MatrixMarket..." switches to MatrixMarket
//     mode -- ids become 1-based and the next data line (the size line) is
//     skipped; other lines starting with '#' or '%' are comments;
//   * a data line needs exactly two integer tokens (MatrixMarket: at least
//     two; a value column may follow);
//   * ids are compacted to [0, n) in ascending order (np.unique), then the
//     graph goes through mce_graph_from_edges (loops dropped, duplicates
//     merged, symmetric).
// The sequential rules (the header applies to the lines after it, the size
// line is the first data line after a header) become two max-scans over the
// line classes.  Errors report the FIRST offending line, as the reference's
// sequential loop does: atomicMin over (line number, error code).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "mce_common.cuh"
#include "mce_b200.h"

namespace {

enum LineKind : int8_t { BLANK = 0, COMMENT = 1, HEADER = 2, DATA = 3 };

__device__ __forceinline__ bool is_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

template <typename T>
int dalloc(T** p, size_t count, cudaStream_t s) {
  *p = nullptr;
  if (count == 0) count = 1;
  MCE_CHECK(cudaMallocAsync((void**)p, count * sizeof(T), s));
  return 0;
}

int grid_for(int64_t work, int threads = 256) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

__global__ void k_line_flags(const unsigned char* __restrict__ text, int64_t len,
                             uint8_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0) || text[i - 1] == '\n';
}

// kind of every line; hdr[i] = i for headers else -1; dat[i] = i for data lines else -1
__global__ void k_classify(const unsigned char* __restrict__ text, int64_t len,
                           const int64_t* __restrict__ start, int64_t nlines,
                           int8_t* __restrict__ kind, int64_t* __restrict__ hdr,
                           int64_t* __restrict__ dat) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nlines;
       l += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = start[l];
    const int64_t e = l + 1 < nlines ? start[l + 1] : len;
    while (p < e && is_space(text[p])) ++p;
    int8_t k = DATA;
    if (p >= e) {
      k = BLANK;
    } else if (text[p] == '#' || text[p] == '%') {
      k = COMMENT;
      const char* tag = "%%MatrixMarket";
      int j = 0;
      while (tag[j] && p + j < e && text[p + j] == (unsigned char)tag[j]) ++j;
      if (!tag[j]) k = HEADER;
    }
    kind[l] = k;
    hdr[l] = k == HEADER ? l : -1;
    dat[l] = k == DATA ? l : -1;
  }
}

// Python int() on one token: [+-]digits with single '_' between digits.
// Returns false on a malformed token or an id that does not fit 62 bits.
__device__ bool parse_int(const unsigned char* t, int64_t n, int64_t* out) {
  int64_t i = 0;
  bool neg = false;
  if (i < n && (t[i] == '+' || t[i] == '-')) {
    neg = t[i] == '-';
    ++i;
  }
  if (i >= n) return false;
  int64_t v = 0;
  bool prev_digit = false;
  for (; i < n; ++i) {
    const unsigned char c = t[i];
    if (c >= '0' && c <= '9') {
      if (v > (((int64_t)1 << 62) - 10) / 10) return false;
      v = v * 10 + (c - '0');
      prev_digit = true;
    } else if (c == '_' && prev_digit && i + 1 < n && t[i + 1] >= '0' && t[i + 1] <= '9') {
      prev_digit = false;
    } else {
      return false;
    }
  }
  *out = neg ? -v : v;
  return true;
}

// parse data lines: pairs (u, v) per line, ok flag; first error -> err
__global__ void k_parse(const unsigned char* __restrict__ text, int64_t len,
                        const int64_t* __restrict__ start, int64_t nlines,
                        const int8_t* __restrict__ kind, const int64_t* __restrict__ last_hdr,
                        const int64_t* __restrict__ last_dat_before, int base,
                        int64_t* __restrict__ pairs, uint8_t* __restrict__ ok,
                        unsigned long long* __restrict__ err) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nlines;
       l += (int64_t)gridDim.x * blockDim.x) {
    ok[l] = 0;
    if (kind[l] != DATA) continue;
    const int64_t h = last_hdr[l];
    const bool mm = h >= 0;
    if (mm && last_dat_before[l] < h) continue;  // the size line after a header
    const int b = mm ? 1 : base;
    int64_t p = start[l];
    const int64_t e = l + 1 < nlines ? start[l + 1] : len;
    int64_t ts[3], te[3];
    int nt = 0;
    while (p < e && nt < 3) {
      while (p < e && is_space(text[p])) ++p;
      if (p >= e) break;
      ts[nt] = p;
      while (p < e && !is_space(text[p])) ++p;
      te[nt] = p;
      ++nt;
    }
    unsigned code = 0;
    if (nt < 2 || (nt > 2 && !mm)) {
      code = 1;  // "expected two integer tokens"
    } else {
      int64_t u = 0, v = 0;
      if (!parse_int(text + ts[0], te[0] - ts[0], &u) || !parse_int(text + ts[1], te[1] - ts[1], &v)) {
        code = 2;  // "non-integer token"
      } else {
        u -= b;
        v -= b;
        if (u < 0 || v < 0) {
          code = 3;  // "vertex id below base"
        } else {
          pairs[2 * l] = u;
          pairs[2 * l + 1] = v;
          ok[l] = 1;
        }
      }
    }
    if (code) atomicMin(err, ((unsigned long long)(l + 1) << 4) | code);
  }
}

__global__ void k_compact_ids(int64_t* __restrict__ e, int64_t count,
                              const int64_t* __restrict__ ids, int64_t nid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = e[i];
    int64_t lo = 0, hi = nid;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ids[mid] < x) lo = mid + 1; else hi = mid;
    }
    e[i] = lo;
  }
}

struct MaxOp {
  __device__ __forceinline__ int64_t operator()(const int64_t& a, const int64_t& b) const {
    return a > b ? a : b;
  }
};

}  // namespace

extern "C" int mce_graph_from_text(const char* text, int64_t len, int base, int text_on_device,
                                   void* stream, mce_graph** out, int64_t* err_line,
                                   int* err_code, int64_t* num_vertices) {
  mce_prepare_device();
  cudaStream_t s = (cudaStream_t)stream;
  *out = nullptr;
  *err_line = 0;
  *err_code = 0;
  *num_vertices = 0;
  if (len < 0 || (base != 0 && base != 1)) {
    mce_set_error("from_text: bad length or base");
    return -2;
  }
  std::vector<void*> owned;
  auto get = [&](auto** p, size_t count) -> int {
    if (dalloc(p, count, s)) return -1;
    owned.push_back((void*)*p);
    return 0;
  };
  auto cleanup = [&]() {
    for (void* p : owned) cudaFreeAsync(p, s);
    owned.clear();
  };
  const unsigned char* d_text = (const unsigned char*)text;
  if (!text_on_device && len > 0) {
    unsigned char* t = nullptr;
    if (get(&t, len)) return -1;
    MCE_CHECK(cudaMemcpyAsync(t, text, len, cudaMemcpyHostToDevice, s));
    d_text = t;
  }
  int64_t nlines = 0;
  int64_t *start = nullptr, *d_n = nullptr;
  uint8_t* flag = nullptr;
  if (len > 0) {
    if (get(&flag, len) || get(&start, len) || get(&d_n, 1)) { cleanup(); return -1; }
    k_line_flags<<<grid_for(len), 256, 0, s>>>(d_text, len, flag);
    mce_count_launch();
    cub::CountingInputIterator<int64_t> it(0);
    size_t tb = 0;
    MCE_CHECK(cub::DeviceSelect::Flagged(nullptr, tb, it, flag, start, d_n, len, s));
    void* tmp = nullptr;
    MCE_CHECK(cudaMallocAsync(&tmp, tb, s));
    MCE_CHECK(cub::DeviceSelect::Flagged(tmp, tb, it, flag, start, d_n, len, s));
    cudaFreeAsync(tmp, s);
    MCE_CHECK(cudaMemcpyAsync(&nlines, d_n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
  }
  int64_t* edges = nullptr;
  int64_t m = 0, n = 0;
  if (nlines > 0) {
    int8_t* kind = nullptr;
    int64_t *hdr = nullptr, *dat = nullptr, *last_hdr = nullptr, *last_dat = nullptr;
    int64_t *pairs = nullptr, *d_m = nullptr;
    uint8_t* ok = nullptr;
    unsigned long long* d_err = nullptr;
    if (get(&kind, nlines) || get(&hdr, nlines) || get(&dat, nlines) ||
        get(&last_hdr, nlines) || get(&last_dat, nlines) || get(&pairs, 2 * nlines) ||
        get(&ok, nlines) || get(&d_err, 1) || get(&edges, 2 * nlines) || get(&d_m, 1)) {
      cleanup();
      return -1;
    }
    k_classify<<<grid_for(nlines), 256, 0, s>>>(d_text, len, start, nlines, kind, hdr, dat);
    mce_count_launch();
    // last header at or before each line; last data line strictly before it
    size_t tb = 0, tb2 = 0;
    MCE_CHECK(cub::DeviceScan::InclusiveScan(nullptr, tb, hdr, last_hdr, MaxOp(), nlines, s));
    MCE_CHECK(cub::DeviceScan::ExclusiveScan(nullptr, tb2, dat, last_dat, MaxOp(), (int64_t)-1,
                                             nlines, s));
    void* tmp = nullptr;
    MCE_CHECK(cudaMallocAsync(&tmp, std::max(tb, tb2), s));
    MCE_CHECK(cub::DeviceScan::InclusiveScan(tmp, tb, hdr, last_hdr, MaxOp(), nlines, s));
    MCE_CHECK(cub::DeviceScan::ExclusiveScan(tmp, tb2, dat, last_dat, MaxOp(), (int64_t)-1,
                                             nlines, s));
    cudaFreeAsync(tmp, s);
    MCE_CHECK(cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), s));
    k_parse<<<grid_for(nlines), 256, 0, s>>>(d_text, len, start, nlines, kind, last_hdr, last_dat,
                                             base, pairs, ok, d_err);
    mce_count_launch();
    unsigned long long h_err = 0;
    MCE_CHECK(cudaMemcpyAsync(&h_err, d_err, sizeof(h_err), cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
    if (h_err != ~0ull) {
      *err_line = (int64_t)(h_err >> 4);
      *err_code = (int)(h_err & 15);
      mce_set_error("parse error at line %lld", (long long)*err_line);
      cleanup();
      return -2;
    }
    // compact the pairs of the parsed lines, in line order
    tb = 0;
    const longlong2* pv = reinterpret_cast<const longlong2*>(pairs);
    longlong2* ev = reinterpret_cast<longlong2*>(edges);
    MCE_CHECK(cub::DeviceSelect::Flagged(nullptr, tb, pv, ok, ev, d_m, nlines, s));
    MCE_CHECK(cudaMallocAsync(&tmp, tb, s));
    MCE_CHECK(cub::DeviceSelect::Flagged(tmp, tb, pv, ok, ev, d_m, nlines, s));
    cudaFreeAsync(tmp, s);
    MCE_CHECK(cudaMemcpyAsync(&m, d_m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
    if (m > 0) {
      // ids = np.unique(all endpoints); endpoints -> their rank
      int64_t *vals = nullptr, *sorted = nullptr, *ids = nullptr, *d_k = nullptr;
      if (get(&vals, 2 * m) || get(&sorted, 2 * m) || get(&ids, 2 * m) || get(&d_k, 1)) {
        cleanup();
        return -1;
      }
      MCE_CHECK(cudaMemcpyAsync(vals, edges, sizeof(int64_t) * 2 * m, cudaMemcpyDeviceToDevice, s));
      tb = 0;
      MCE_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tb, vals, sorted, 2 * m, 0, 63, s));
      MCE_CHECK(cudaMallocAsync(&tmp, tb, s));
      MCE_CHECK(cub::DeviceRadixSort::SortKeys(tmp, tb, vals, sorted, 2 * m, 0, 63, s));
      cudaFreeAsync(tmp, s);
      tb = 0;
      MCE_CHECK(cub::DeviceSelect::Unique(nullptr, tb, sorted, ids, d_k, 2 * m, s));
      MCE_CHECK(cudaMallocAsync(&tmp, tb, s));
      MCE_CHECK(cub::DeviceSelect::Unique(tmp, tb, sorted, ids, d_k, 2 * m, s));
      cudaFreeAsync(tmp, s);
      MCE_CHECK(cudaMemcpyAsync(&n, d_k, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      MCE_CHECK(cudaStreamSynchronize(s));
      if (n >= (int64_t(1) << 31)) {
        mce_set_error("from_text: %lld distinct vertex ids exceed the int32 CSR", (long long)n);
        cleanup();
        return -2;
      }
      k_compact_ids<<<grid_for(2 * m), 256, 0, s>>>(edges, 2 * m, ids, n);
      mce_count_launch();
      MCE_CHECK(cudaGetLastError());
    }
  }
  *num_vertices = n;
  int rc = mce_graph_from_edges(edges, m, n, 1, stream, out);
  cleanup();
  return rc;
}

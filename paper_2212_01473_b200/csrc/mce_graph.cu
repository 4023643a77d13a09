// Graph ingestion on the device: canonical CSR construction, degeneracy
// ordering by parallel peeling, reordering and CSR orientation.
//
// Reference behaviour restated (file:line in /root/reference/pkg/src/mce):
//   from_edges ......... graph.py:103-129  (drop loops, merge duplicates, both directions,
//                                          rows strictly ascending)
//   degeneracy_order ... graph.py:183-210 (method 1 = the reference's exact
//                                          min-degree/smallest-id order; method 0 = parallel
//                                          bucket peel, a valid degeneracy order with the
//                                          same degeneracy)
//   reorder ............ graph.py:213-224
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <vector>

#include "mce_common.cuh"
#include "mce_b200.h"

static thread_local char g_err[1024];

void mce_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* mce_last_error(void) { return g_err; }

static std::atomic<int64_t> g_launches{0};
void mce_count_launch(int64_t k) { g_launches += k; }
extern "C" int64_t mce_launch_count(void) { return g_launches.load(); }

void mce_prepare_device() {
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

namespace {

template <typename T>
int dev_alloc(T** p, size_t count, cudaStream_t s) {
  *p = nullptr;
  if (count == 0) count = 1;
  MCE_CHECK(cudaMallocAsync((void**)p, count * sizeof(T), s));
  return 0;
}

template <typename T>
void dev_free(T* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

int bits_for(int64_t n) {
  int b = 1;
  while ((int64_t(1) << b) < n) ++b;
  return b;
}

// ---------------------------------------------------------------- kernels

__global__ void k_edge_keys(const int64_t* __restrict__ edges, int64_t m, int b,
                            uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = edges[2 * i], c = edges[2 * i + 1];
    int64_t lo = a < c ? a : c, hi = a < c ? c : a;
    keys[i] = (lo == hi) ? ~0ull : (((uint64_t)lo << b) | (uint64_t)hi);
  }
}

struct NotAllOnes {
  __host__ __device__ bool operator()(const uint64_t& k) const { return k != ~0ull; }
};

__global__ void k_expand_directed(const uint64_t* __restrict__ und, int64_t m, int b,
                                  uint64_t* __restrict__ out) {
  const uint64_t mask = (1ull << b) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = und[i];
    uint64_t lo = k >> b, hi = k & mask;
    out[2 * i] = k;
    out[2 * i + 1] = (hi << b) | lo;
  }
}

// keys sorted by (src, dst): emit col and row offsets
__global__ void k_keys_to_csr(const uint64_t* __restrict__ keys, int64_t nnz, int b, int64_t n,
                              int64_t* __restrict__ ro, int32_t* __restrict__ col) {
  const uint64_t mask = (1ull << b) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    int64_t s = (int64_t)(k >> b);
    col[i] = (int32_t)(k & mask);
    int64_t prev = (i == 0) ? -1 : (int64_t)(keys[i - 1] >> b);
    for (int64_t v = prev + 1; v <= s; ++v) ro[v] = i;
    if (i == nnz - 1)
      for (int64_t v = s + 1; v <= n; ++v) ro[v] = nnz;
  }
}

__global__ void k_narrow(const int64_t* __restrict__ src, int64_t count, int32_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (int32_t)src[i];
}

__global__ void k_widen(const int32_t* __restrict__ src, int64_t count, int64_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_fill_i64(int64_t* p, int64_t count, int64_t value) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = value;
}

__global__ void k_split(const int64_t* __restrict__ ro, const int32_t* __restrict__ col,
                        int64_t n, int64_t* __restrict__ split,
                        unsigned long long* __restrict__ stats /* maxdeg, maxlater, maxearlier */) {
  unsigned long long md = 0, ml = 0, me = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = ro[v], hi = ro[v + 1];
    int64_t a = lo, c = hi;
    while (a < c) {
      int64_t mid = (a + c) >> 1;
      if (col[mid] < v) a = mid + 1; else c = mid;
    }
    split[v] = a;
    md = max(md, (unsigned long long)(hi - lo));
    ml = max(ml, (unsigned long long)(hi - a));
    me = max(me, (unsigned long long)(a - lo));
  }
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage t0, t1, t2;
  md = BR(t0).Reduce(md, cub::Max());
  ml = BR(t1).Reduce(ml, cub::Max());
  me = BR(t2).Reduce(me, cub::Max());
  if (threadIdx.x == 0) {
    atomicMax(&stats[0], md);
    atomicMax(&stats[1], ml);
    atomicMax(&stats[2], me);
  }
}

// ---- parallel peel

__global__ void k_init_peel(const int64_t* __restrict__ ro, int64_t n, int32_t* __restrict__ deg,
                            int32_t* __restrict__ alive, uint8_t* __restrict__ removed) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    deg[v] = (int32_t)(ro[v + 1] - ro[v]);
    alive[v] = (int32_t)v;
    removed[v] = 0;
  }
}

__global__ void k_peel_flags(const int32_t* __restrict__ alive, int64_t na,
                             const int32_t* __restrict__ deg, int32_t k,
                             uint8_t* __restrict__ take, uint8_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool t = deg[alive[i]] <= k;
    take[i] = t;
    keep[i] = !t;
  }
}

__global__ void k_peel_assign(const int32_t* __restrict__ frontier, int64_t nf, int64_t base,
                              int64_t* __restrict__ position, uint8_t* __restrict__ removed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nf;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = frontier[i];
    position[v] = base + i;
    removed[v] = 1;
  }
}

// one warp per frontier vertex: decrement the live neighbours' degrees
__global__ void k_peel_decrement(const int32_t* __restrict__ frontier, int64_t nf,
                                 const int64_t* __restrict__ ro, const int32_t* __restrict__ col,
                                 const uint8_t* __restrict__ removed, int32_t* __restrict__ deg) {
  const int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nf; i += nwarps) {
    int32_t v = frontier[i];
    for (int64_t e = ro[v] + lane; e < ro[v + 1]; e += 32) {
      int32_t u = col[e];
      if (!removed[u]) atomicSub(&deg[u], 1);
    }
  }
}

struct DegOf {
  const int32_t* deg;
  __host__ __device__ int32_t operator()(const int32_t& v) const { return deg[v]; }
};

// ---- exact order (reference tie-break): single CTA, min-segment-tree over
// keys (deg << 32 | id).  Sequential by nature; used for reference-identical
// orderings, the parallel peel is the throughput path.
constexpr int EXACT_THREADS = 1024;

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__global__ void __launch_bounds__(EXACT_THREADS)
k_exact_order(const int64_t* __restrict__ ro, const int32_t* __restrict__ col, int64_t n,
              int64_t leaves, uint64_t* __restrict__ tree, int64_t* __restrict__ position,
              int64_t* __restrict__ out_degeneracy) {
  // tree: 2*leaves nodes, node 1 = root, leaves at [leaves, 2*leaves)
  __shared__ uint64_t s_root;
  __shared__ int s_levels;
  const int tid = threadIdx.x;
  for (int64_t i = tid; i < leaves; i += blockDim.x) {
    tree[leaves + i] = (i < n) ? (((uint64_t)(ro[i + 1] - ro[i]) << 32) | (uint64_t)i) : ~0ull;
  }
  __syncthreads();
  int levels = 0;
  for (int64_t w = leaves; w > 1; w >>= 1) ++levels;
  for (int64_t w = leaves >> 1; w >= 1; w >>= 1) {
    for (int64_t i = tid; i < w; i += blockDim.x)
      tree[w + i] = umin64(tree[2 * (w + i)], tree[2 * (w + i) + 1]);
    __syncthreads();
  }
  if (tid == 0) s_levels = levels;
  int64_t degeneracy = 0;
  for (int64_t rank = 0; rank < n; ++rank) {
    if (tid == 0) s_root = tree[1];
    __syncthreads();
    uint64_t key = s_root;
    int64_t v = (int64_t)(key & 0xffffffffull);
    int64_t dv = (int64_t)(key >> 32);
    if (dv > degeneracy) degeneracy = dv;
    if (tid == 0) {
      position[v] = rank;
      tree[leaves + v] = ~0ull;
    }
    // decrement live neighbours (their leaves hold their current key)
    for (int64_t e = ro[v] + tid; e < ro[v + 1]; e += blockDim.x) {
      int64_t u = col[e];
      uint64_t k = tree[leaves + u];
      if (k != ~0ull) tree[leaves + u] = k - (1ull << 32);
    }
    __syncthreads();
    // refresh ancestors of every touched leaf, level by level
    int64_t deg_v = ro[v + 1] - ro[v];
    for (int l = 1; l <= s_levels; ++l) {
      for (int64_t j = tid; j <= deg_v; j += blockDim.x) {
        int64_t leaf = (j == deg_v) ? v : (int64_t)col[ro[v] + j];
        int64_t node = (leaves + leaf) >> l;
        tree[node] = umin64(tree[2 * node], tree[2 * node + 1]);
      }
      __syncthreads();
    }
  }
  if (tid == 0) *out_degeneracy = degeneracy;
}

// ---- reorder

__global__ void k_reorder_keys(const int64_t* __restrict__ ro, const int32_t* __restrict__ col,
                               int64_t n, const int64_t* __restrict__ pos, int b,
                               uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps) {
    uint64_t pv = (uint64_t)pos[v] << b;
    for (int64_t e = ro[v] + lane; e < ro[v + 1]; e += 32) keys[e] = pv | (uint64_t)pos[col[e]];
  }
}

__global__ void k_relabel(const int64_t* __restrict__ pos, int64_t n,
                          const int64_t* __restrict__ old_labels, int64_t* __restrict__ labels) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    labels[pos[v]] = old_labels ? old_labels[v] : v;
}

int grid_for(int64_t work, int threads = 256) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

// sort `count` keys in place (via an alternate buffer) over [0, end_bit)
int sort_keys(uint64_t** keys, int64_t count, int end_bit, cudaStream_t s) {
  if (count <= 1) return 0;
  uint64_t* alt = nullptr;
  if (dev_alloc(&alt, count, s)) return -1;
  cub::DoubleBuffer<uint64_t> db(*keys, alt);
  size_t tmp_bytes = 0;
  MCE_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, count, 0, end_bit, s));
  void* tmp = nullptr;
  MCE_CHECK(cudaMallocAsync(&tmp, tmp_bytes, s));
  MCE_CHECK(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, db, count, 0, end_bit, s));
  cudaFreeAsync(tmp, s);
  if (db.Current() != *keys) {
    dev_free(*keys, s);
    *keys = db.Current();
  } else {
    dev_free(alt, s);
  }
  return 0;
}

int csr_from_sorted_keys(mce_graph* g, uint64_t* keys, int64_t nnz, int b, cudaStream_t s) {
  g->nnz = nnz;
  if (dev_alloc(&g->ro, g->n + 1, s)) return -1;
  if (dev_alloc(&g->col, nnz, s)) return -1;
  if (nnz == 0) {
    k_fill_i64<<<grid_for(g->n + 1), 256, 0, s>>>(g->ro, g->n + 1, 0);
    mce_count_launch();
  } else {
    k_keys_to_csr<<<grid_for(nnz), 256, 0, s>>>(keys, nnz, b, g->n, g->ro, g->col);
    mce_count_launch();
  }
  MCE_CHECK(cudaGetLastError());
  return mce_graph_build_split(g, s);
}

}  // namespace

int mce_graph_build_split(mce_graph* g, cudaStream_t s) {
  if (!g->split && dev_alloc(&g->split, g->n, s)) return -1;
  unsigned long long* st = nullptr;
  if (dev_alloc(&st, 3, s)) return -1;
  MCE_CHECK(cudaMemsetAsync(st, 0, 3 * sizeof(unsigned long long), s));
  if (g->n > 0) k_split<<<grid_for(g->n), 256, 0, s>>>(g->ro, g->col, g->n, g->split, st);
  mce_count_launch();
  MCE_CHECK(cudaGetLastError());
  unsigned long long h[3];
  MCE_CHECK(cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
  MCE_CHECK(cudaStreamSynchronize(s));
  dev_free(st, s);
  g->max_degree = (int64_t)h[0];
  g->max_later = (int64_t)h[1];
  g->max_earlier = (int64_t)h[2];
  return 0;
}

extern "C" {

int mce_graph_from_edges(const int64_t* edges, int64_t num_edges, int64_t num_vertices,
                         int edges_on_device, void* stream, mce_graph** out) {
  mce_prepare_device();
  cudaStream_t s = (cudaStream_t)stream;
  *out = nullptr;
  if (num_vertices < 0 || num_vertices >= (int64_t(1) << 31) || num_edges < 0) {
    mce_set_error("from_edges: vertex count %lld out of range", (long long)num_vertices);
    return -2;
  }
  mce_graph* g = new mce_graph();
  cudaGetDevice(&g->device);
  g->n = num_vertices;
  const int b = bits_for(std::max<int64_t>(num_vertices, 2));
  const int64_t* d_edges = edges;
  int64_t* owned = nullptr;
  if (!edges_on_device && num_edges > 0) {
    if (dev_alloc(&owned, 2 * num_edges, s)) { delete g; return -1; }
    MCE_CHECK(cudaMemcpyAsync(owned, edges, sizeof(int64_t) * 2 * num_edges,
                              cudaMemcpyHostToDevice, s));
    d_edges = owned;
  }
  uint64_t* keys = nullptr;
  int64_t m = 0;
  if (num_edges > 0) {
    uint64_t* raw = nullptr;
    if (dev_alloc(&raw, num_edges, s)) return -1;
    k_edge_keys<<<grid_for(num_edges), 256, 0, s>>>(d_edges, num_edges, b, raw);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    dev_free(owned, s);
    // drop self-loops
    if (dev_alloc(&keys, num_edges, s)) return -1;
    int64_t* d_cnt = nullptr;
    if (dev_alloc(&d_cnt, 1, s)) return -1;
    size_t tb = 0;
    MCE_CHECK(cub::DeviceSelect::If(nullptr, tb, raw, keys, d_cnt, num_edges, NotAllOnes(), s));
    void* tmp = nullptr;
    MCE_CHECK(cudaMallocAsync(&tmp, tb, s));
    MCE_CHECK(cub::DeviceSelect::If(tmp, tb, raw, keys, d_cnt, num_edges, NotAllOnes(), s));
    cudaFreeAsync(tmp, s);
    int64_t kept = 0;
    MCE_CHECK(cudaMemcpyAsync(&kept, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
    dev_free(raw, s);
    if (sort_keys(&keys, kept, 2 * b, s)) return -1;
    // merge duplicates
    uint64_t* uniq = nullptr;
    if (dev_alloc(&uniq, kept, s)) return -1;
    tb = 0;
    MCE_CHECK(cub::DeviceSelect::Unique(nullptr, tb, keys, uniq, d_cnt, kept, s));
    MCE_CHECK(cudaMallocAsync(&tmp, tb, s));
    MCE_CHECK(cub::DeviceSelect::Unique(tmp, tb, keys, uniq, d_cnt, kept, s));
    cudaFreeAsync(tmp, s);
    MCE_CHECK(cudaMemcpyAsync(&m, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
    dev_free(keys, s);
    dev_free(d_cnt, s);
    // both directions, sorted by (src, dst)
    if (dev_alloc(&keys, 2 * m, s)) return -1;
    if (m > 0) k_expand_directed<<<grid_for(m), 256, 0, s>>>(uniq, m, b, keys);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    dev_free(uniq, s);
    if (sort_keys(&keys, 2 * m, 2 * b, s)) return -1;
  } else {
    dev_free(owned, s);
  }
  int rc = csr_from_sorted_keys(g, keys, 2 * m, b, s);
  dev_free(keys, s);
  if (rc) { delete g; return rc; }
  *out = g;
  return 0;
}

int mce_graph_from_csr(const int64_t* row_offsets, const int64_t* col_indices, int64_t n,
                       int64_t nnz, int on_device, void* stream, mce_graph** out) {
  mce_prepare_device();
  cudaStream_t s = (cudaStream_t)stream;
  *out = nullptr;
  if (n < 0 || n >= (int64_t(1) << 31)) {
    mce_set_error("from_csr: vertex count %lld out of range", (long long)n);
    return -2;
  }
  mce_graph* g = new mce_graph();
  cudaGetDevice(&g->device);
  g->n = n;
  g->nnz = nnz;
  if (dev_alloc(&g->ro, n + 1, s)) return -1;
  if (dev_alloc(&g->col, nnz, s)) return -1;
  MCE_CHECK(cudaMemcpyAsync(g->ro, row_offsets, sizeof(int64_t) * (n + 1),
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  if (nnz > 0) {
    // narrow to int32 on the device
    int64_t* tmp = nullptr;
    if (on_device) {
      tmp = (int64_t*)col_indices;
    } else {
      if (dev_alloc(&tmp, nnz, s)) return -1;
      MCE_CHECK(cudaMemcpyAsync(tmp, col_indices, sizeof(int64_t) * nnz,
                                cudaMemcpyHostToDevice, s));
    }
    k_narrow<<<grid_for(nnz), 256, 0, s>>>(tmp, nnz, g->col);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    if (!on_device) dev_free(tmp, s);
  }
  int rc = mce_graph_build_split(g, s);
  if (rc) { delete g; return rc; }
  *out = g;
  return 0;
}

}  // extern "C"

extern "C" {

int mce_graph_info(const mce_graph* g, int64_t* n, int64_t* nnz, int64_t* max_degree,
                   int64_t* max_later, int64_t* max_earlier) {
  if (!g) { mce_set_error("null graph"); return -2; }
  if (n) *n = g->n;
  if (nnz) *nnz = g->nnz;
  if (max_degree) *max_degree = g->max_degree;
  if (max_later) *max_later = g->max_later;
  if (max_earlier) *max_earlier = g->max_earlier;
  return 0;
}

int mce_graph_copy_csr(const mce_graph* g, int64_t* row_offsets, int64_t* col_indices,
                       int64_t* labels, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (row_offsets)
    MCE_CHECK(cudaMemcpyAsync(row_offsets, g->ro, sizeof(int64_t) * (g->n + 1),
                              cudaMemcpyDeviceToHost, s));
  if (col_indices && g->nnz > 0) {
    int64_t* wide = nullptr;
    if (dev_alloc(&wide, g->nnz, s)) return -1;
    auto n = g->nnz;
    k_widen<<<grid_for(n), 256, 0, s>>>(g->col, n, wide);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    MCE_CHECK(cudaMemcpyAsync(col_indices, wide, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    dev_free(wide, s);
  }
  if (labels && g->labels)
    MCE_CHECK(cudaMemcpyAsync(labels, g->labels, sizeof(int64_t) * g->n,
                              cudaMemcpyDeviceToHost, s));
  MCE_CHECK(cudaStreamSynchronize(s));
  return 0;
}

void mce_graph_free(mce_graph* g) {
  if (!g) return;
  cudaFree(g->ro);
  cudaFree(g->col);
  cudaFree(g->split);
  cudaFree(g->labels);
  delete g;
}

// position: out, n entries (host or device per position_on_device)
int mce_degeneracy_order(const mce_graph* g, int method, int64_t* position,
                         int position_on_device, int64_t* degeneracy, void* stream) {
  mce_prepare_device();
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = g->n;
  *degeneracy = 0;
  if (n == 0) return 0;
  int64_t* d_pos = position_on_device ? position : nullptr;
  if (!d_pos && dev_alloc(&d_pos, n, s)) return -1;
  if (method == 1) {
    int64_t leaves = 2;
    while (leaves < n) leaves <<= 1;
    uint64_t* tree = nullptr;
    int64_t* d_deg = nullptr;
    if (dev_alloc(&tree, 2 * leaves, s) || dev_alloc(&d_deg, 1, s)) return -1;
    k_exact_order<<<1, EXACT_THREADS, 0, s>>>(g->ro, g->col, n, leaves, tree, d_pos, d_deg);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    MCE_CHECK(cudaMemcpyAsync(degeneracy, d_deg, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
    dev_free(tree, s);
    dev_free(d_deg, s);
  } else {
    int32_t *deg = nullptr, *alive = nullptr, *alive2 = nullptr, *frontier = nullptr;
    uint8_t *removed = nullptr, *take = nullptr, *keep = nullptr;
    int64_t* d_cnt = nullptr;
    int32_t* d_min = nullptr;
    if (dev_alloc(&deg, n, s) || dev_alloc(&alive, n, s) || dev_alloc(&alive2, n, s) ||
        dev_alloc(&frontier, n, s) || dev_alloc(&removed, n, s) || dev_alloc(&take, n, s) ||
        dev_alloc(&keep, n, s) || dev_alloc(&d_cnt, 2, s) || dev_alloc(&d_min, 1, s))
      return -1;
    k_init_peel<<<grid_for(n), 256, 0, s>>>(g->ro, n, deg, alive, removed);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    size_t tb_sel = 0, tb_min = 0;
    MCE_CHECK(cub::DeviceSelect::Flagged(nullptr, tb_sel, alive, take, frontier, d_cnt, n, s));
    cub::TransformInputIterator<int32_t, DegOf, const int32_t*> degs(alive, DegOf{deg});
    MCE_CHECK(cub::DeviceReduce::Min(nullptr, tb_min, degs, d_min, n, s));
    void* tmp = nullptr;
    size_t tb = std::max(tb_sel, tb_min);
    MCE_CHECK(cudaMallocAsync(&tmp, tb, s));
    int64_t na = n, base = 0;
    int32_t k = 0;
    int64_t deg_max = 0;
    while (na > 0) {
      k_peel_flags<<<grid_for(na), 256, 0, s>>>(alive, na, deg, k, take, keep);
      mce_count_launch();
      size_t t1 = tb;
      MCE_CHECK(cub::DeviceSelect::Flagged(tmp, t1, alive, take, frontier, d_cnt, na, s));
      int64_t nf = 0;
      MCE_CHECK(cudaMemcpyAsync(&nf, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      MCE_CHECK(cudaStreamSynchronize(s));
      if (nf == 0) {
        cub::TransformInputIterator<int32_t, DegOf, const int32_t*> dg(alive, DegOf{deg});
        size_t t2 = tb;
        MCE_CHECK(cub::DeviceReduce::Min(tmp, t2, dg, d_min, na, s));
        int32_t mn = 0;
        MCE_CHECK(cudaMemcpyAsync(&mn, d_min, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        MCE_CHECK(cudaStreamSynchronize(s));
        k = std::max(k + 1, mn);
        continue;
      }
      if (k > deg_max) deg_max = k;
      k_peel_assign<<<grid_for(nf), 256, 0, s>>>(frontier, nf, base, d_pos, removed);
      mce_count_launch();
      k_peel_decrement<<<grid_for(nf * 32), 256, 0, s>>>(frontier, nf, g->ro, g->col, removed, deg);
      mce_count_launch();
      size_t t3 = tb;
      MCE_CHECK(cub::DeviceSelect::Flagged(tmp, t3, alive, keep, alive2, d_cnt + 1, na, s));
      MCE_CHECK(cudaGetLastError());
      std::swap(alive, alive2);
      base += nf;
      na -= nf;
    }
    // the degeneracy is the largest peel level at which a vertex left, but a
    // level may be reached only because k jumped to the minimum degree: the
    // real degree at removal is what the reference reports (graph.py:198-205)
    *degeneracy = deg_max;
    cudaFreeAsync(tmp, s);
    dev_free(deg, s); dev_free(alive, s); dev_free(alive2, s); dev_free(frontier, s);
    dev_free(removed, s); dev_free(take, s); dev_free(keep, s); dev_free(d_cnt, s);
    dev_free(d_min, s);
  }
  if (!position_on_device) {
    MCE_CHECK(cudaMemcpyAsync(position, d_pos, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
    dev_free(d_pos, s);
  }
  return 0;
}

int mce_reorder(const mce_graph* g, const int64_t* position, int position_on_device,
                void* stream, mce_graph** out) {
  mce_prepare_device();
  cudaStream_t s = (cudaStream_t)stream;
  *out = nullptr;
  mce_graph* h = new mce_graph();
  h->device = g->device;
  h->n = g->n;
  const int64_t n = g->n;
  const int b = bits_for(std::max<int64_t>(n, 2));
  const int64_t* d_pos = position;
  int64_t* owned = nullptr;
  if (!position_on_device && n > 0) {
    if (dev_alloc(&owned, n, s)) return -1;
    MCE_CHECK(cudaMemcpyAsync(owned, position, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    d_pos = owned;
  }
  uint64_t* keys = nullptr;
  if (dev_alloc(&keys, g->nnz, s)) return -1;
  if (g->nnz > 0) {
    k_reorder_keys<<<grid_for(n * 32), 256, 0, s>>>(g->ro, g->col, n, d_pos, b, keys);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    if (sort_keys(&keys, g->nnz, 2 * b, s)) return -1;
  }
  if (dev_alloc(&h->labels, n, s)) return -1;
  if (n > 0) k_relabel<<<grid_for(n), 256, 0, s>>>(d_pos, n, g->labels, h->labels);
  mce_count_launch();
  MCE_CHECK(cudaGetLastError());
  int rc = csr_from_sorted_keys(h, keys, g->nnz, b, s);
  dev_free(keys, s);
  dev_free(owned, s);
  if (rc) { mce_graph_free(h); return rc; }
  *out = h;
  return 0;
}

}  // extern "C"

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
#include <cub/device/device_segmented_sort.cuh>
#include <cooperative_groups.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
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
struct ArenaState {
  std::mutex mu;
  bool busy = false;
  char* base = nullptr;
  size_t cap = 0, want = 0;
  cudaEvent_t last = nullptr;   // recorded at the end of the last call's work
  cudaStream_t last_stream = nullptr;
  bool used = false;
};
ArenaState g_arena[64];
constexpr size_t ARENA_ALIGN = 256;
bool g_free_stale[64];  // set when the scratch arena re-sizes itself
}  // namespace

void mce_trace_mark(const char* what) {
  static const bool on = getenv("MCE_TRACE") != nullptr;
  if (!on) return;
  static thread_local std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  const auto now = std::chrono::steady_clock::now();
  fprintf(stderr, "[mce_trace] %-22s +%8.3f ms\n", what,
          std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

size_t mce_free_memory() {
  static std::mutex mu;
  static size_t cached[64];
  static std::chrono::steady_clock::time_point at[64];
  static bool have[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lk(mu);
  const auto now = std::chrono::steady_clock::now();
  if (!have[dev] || g_free_stale[dev] || now - at[dev] > std::chrono::seconds(1)) {
    g_free_stale[dev] = false;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    cached[dev] = free_b;
    at[dev] = now;
    have[dev] = true;
  }
  return cached[dev];
}

Scratch::Scratch(cudaStream_t s) : s_(s) {
  if (cudaGetDevice(&dev_) != cudaSuccess || dev_ < 0 || dev_ >= 64) return;
  ArenaState& a = g_arena[dev_];
  std::lock_guard<std::mutex> lk(a.mu);
  if (a.busy) return;
  a.busy = true;
  owner_ = true;
  if (!a.last && cudaEventCreateWithFlags(&a.last, cudaEventDisableTiming) != cudaSuccess) {
    a.busy = false;
    owner_ = false;
    return;
  }
  // stream order: this call's work starts after the previous call's work on
  // the arena (same stream: already ordered; another stream: wait on the device)
  if (a.used && a.last_stream != s) cudaStreamWaitEvent(s, a.last, 0);
  if (a.want > a.cap) {  // grow, stream-ordered (no host wait)
    if (a.base) cudaFreeAsync(a.base, s);
    a.base = nullptr;
    a.cap = 0;
    if (cudaMallocAsync((void**)&a.base, a.want, s) == cudaSuccess) a.cap = a.want;
    else a.base = nullptr;
    g_free_stale[dev_] = true;
  }
}

size_t Scratch::reserved() const { return owner_ ? g_arena[dev_].cap : 0; }

int Scratch::raw(void** p, size_t bytes) {
  bytes = (bytes + ARENA_ALIGN - 1) / ARENA_ALIGN * ARENA_ALIGN;
  demand_ += bytes;
  if (owner_) {
    ArenaState& a = g_arena[dev_];
    if (a.base && used_ + bytes <= a.cap) {
      *p = a.base + used_;
      used_ += bytes;
      return 0;
    }
  }
  MCE_CHECK(cudaMallocAsync(p, bytes, s_));
  extra_.push_back(*p);
  return 0;
}

Scratch::~Scratch() {
  for (void* q : extra_) cudaFreeAsync(q, s_);
  if (owner_) {
    ArenaState& a = g_arena[dev_];
    std::lock_guard<std::mutex> lk(a.mu);
    cudaEventRecord(a.last, s_);
    a.last_stream = s_;
    a.used = true;
    if (demand_ > a.cap) a.want = demand_ + demand_ / 8;
    a.busy = false;
  }
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

// ids outside [0, n) raise `bad` (reference: ValueError, graph.py:103-129)
// both directed keys of every input pair; loops -> all-ones (dropped later).
// T = int64_t (the reference's edge array) or int32_t (half the ingress bytes)
template <typename T>
__global__ void k_edge_keys_both(const T* __restrict__ edges, int64_t m, int b, int64_t n,
                                 uint64_t* __restrict__ keys, int* __restrict__ bad) {
  bool oob = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = edges[2 * i], c = edges[2 * i + 1];
    oob |= (a < 0) | (c < 0) | (a >= n) | (c >= n);
    const bool loop = a == c;
    keys[2 * i] = loop ? ~0ull : (((uint64_t)a << b) | (uint64_t)c);
    keys[2 * i + 1] = loop ? ~0ull : (((uint64_t)c << b) | (uint64_t)a);
  }
  if (__syncthreads_or(oob) && threadIdx.x == 0) atomicExch(bad, 1);
}

// cnt[2] = 1 when the last unique key is the (sorted-last) loop sentinel
__global__ void k_last_is_loop(const uint64_t* __restrict__ uniq, int64_t* cnt, int bits) {
  const int64_t u = cnt[0];
  const uint64_t mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
  cnt[2] = (u > 0 && (uniq[u - 1] & mask) == mask) ? 1 : 0;
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

// ---- persistent parallel peel: the whole bucket-peeling loop in ONE
// launch (software grid barrier; every CTA co-resident), no host round trip
// per round.  Peel level k removes, round by round, every live vertex whose
// current degree is <= k; the position of a vertex is its (round, id) rank,
// so the order is deterministic -- identical to a round-synchronous bucket
// peel that ranks each round by id -- although nothing inside a round is
// ordered: the kernel only records each vertex's round, and one radix sort of
// (round, id) keys afterwards yields the positions.
//
//  * FULL round (a level's first round): the CTAs scan the alive list; live
//    vertices with deg <= k join the frontier, the rest are compacted into the
//    other alive buffer and give the minimum live degree (an empty frontier
//    raises k to max(k + 1, that minimum)).
//  * INCREMENTAL round: the frontier is exactly the vertices whose degree
//    crossed k+1 -> k during the previous decrement; they were claimed right
//    there (the unique atomicSub that returned k+1), so the round is just the
//    decrement phase plus ONE grid barrier.
//  * decrement work list: a frontier vertex enters as ceil(deg/32) chunk
//    descriptors (vertex, chunk); warps take descriptors grid-wide, one lane
//    per edge, so a hub's adjacency is spread over many warps.
constexpr int PEEL_THREADS = 512;

struct PeelShared {
  unsigned int bar_count;
  unsigned int bar_gen;
  // per round parity: (frontier vertices << 32) | chunk descriptors, one
  // 64-bit atomic claims both
  unsigned long long fc[2];
  unsigned int acount;      // survivors of the current full scan
  int mindeg;               // their minimum degree
};

// Grid barrier; the last CTA to arrive runs `reset` (all others are waiting).
template <typename F>
__device__ __forceinline__ void grid_barrier(PeelShared* sh, unsigned int nblocks, F reset) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = &sh->bar_gen;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(&sh->bar_count, 1u) == nblocks - 1) {
      reset();
      sh->bar_count = 0;
      __threadfence();
      atomicAdd(&sh->bar_gen, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// frontier vertex v of the round with parity p: ceil(deg/32) descriptors,
// each an edge range (start << 6 | length <= 32) -- the decrement needs no
// further offset loads
__device__ __forceinline__ void peel_enqueue(const int64_t* __restrict__ ro, int32_t v, int p,
                                             uint64_t* __restrict__ chunks, int64_t cap,
                                             PeelShared* sh) {
  const int64_t e0 = ro[v], e1 = ro[v + 1];
  const unsigned nch = (unsigned)((e1 - e0 + 31) >> 5);
  const unsigned long long old = atomicAdd(&sh->fc[p], (1ull << 32) | nch);
  uint64_t* out = chunks + (size_t)p * cap + (uint32_t)old;
  for (unsigned j = 0; j < nch; ++j) {
    const int64_t st = e0 + 32 * (int64_t)j;
    const int64_t len = e1 - st < 32 ? e1 - st : 32;
    out[j] = ((uint64_t)st << 6) | (uint64_t)len;
  }
}

__global__ void __launch_bounds__(PEEL_THREADS)
k_peel_persistent(const int64_t* __restrict__ ro, const int32_t* __restrict__ col, int64_t n,
                  int32_t* __restrict__ deg, int32_t* alive_a, int32_t* alive_b,
                  uint64_t* __restrict__ chunks, int64_t chunk_cap,
                  uint8_t* __restrict__ removed, uint32_t* __restrict__ key, PeelShared* sh,
                  int64_t* __restrict__ out_degeneracy) {
  const unsigned int G = gridDim.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int64_t gtid = (int64_t)blockIdx.x * PEEL_THREADS + tid;
  const int64_t gstride = (int64_t)G * PEEL_THREADS;
  const int64_t gwarp = gtid >> 5;
  const int64_t nwarps = gstride >> 5;
  auto nothing = [] {};

  for (int64_t v = gtid; v < n; v += gstride) {
    deg[v] = (int32_t)(ro[v + 1] - ro[v]);
    alive_a[v] = (int32_t)v;
    removed[v] = 0;
  }
  grid_barrier(sh, G, nothing);

  int32_t* alive = alive_a;
  int32_t* alive2 = alive_b;
  int64_t na = n, left = n;
  int32_t k = 0, deg_max = 0;
  int64_t r = 0;  // round
  bool full = true;
  while (left > 0) {
    const int p = (int)(r & 1);
    int64_t nf;
    if (full) {
      for (int64_t i = gtid; i < na; i += gstride) {
        const int32_t v = __ldcg(&alive[i]);
        if (__ldcg(&removed[v])) continue;  // claimed as a crosser earlier
        const int32_t d = __ldcg(&deg[v]);
        if (d <= k) {
          removed[v] = 1;
          key[v] = (uint32_t)r;
          peel_enqueue(ro, v, p, chunks, chunk_cap, sh);
        } else {
          alive2[atomicAdd(&sh->acount, 1u)] = v;
          atomicMin(&sh->mindeg, d);
        }
      }
      grid_barrier(sh, G, nothing);
      nf = (int64_t)(*(volatile unsigned long long*)&sh->fc[p] >> 32);
      na = *(volatile unsigned int*)&sh->acount;
      const int32_t mn = *(volatile int*)&sh->mindeg;
      int32_t* t = alive;
      alive = alive2;
      alive2 = t;
      if (nf == 0) {  // nothing at this level: jump to the next populated one
        k = max(k + 1, mn);
        grid_barrier(sh, G, [sh] {
          sh->acount = 0;
          sh->mindeg = 0x7fffffff;
        });
        continue;
      }
    } else {
      nf = (int64_t)(*(volatile unsigned long long*)&sh->fc[p] >> 32);
      if (nf == 0) {  // the level is exhausted
        k += 1;
        full = true;
        // nobody may start the full scan (which appends to this round's
        // counters) before every CTA has read them
        grid_barrier(sh, G, nothing);
        continue;
      }
    }
    if (k > deg_max) deg_max = k;
    // decrement the live neighbours of the frontier; the unique k+1 -> k
    // crossing claims the vertex for round r + 1
    const int64_t nc = (int64_t)(uint32_t)*(volatile unsigned long long*)&sh->fc[p];
    const uint64_t* cl = chunks + (size_t)p * chunk_cap;
    const uint32_t next_round = (uint32_t)(r + 1);
    for (int64_t c = gwarp; c < nc; c += nwarps) {
      const uint64_t dsc = __ldcg(&cl[c]);
      if (lane < (int)(dsc & 63)) {
        const int32_t u = col[(int64_t)(dsc >> 6) + lane];
        // no removed[] test needed: a peeled vertex has deg <= the level it
        // left at <= k, so its decrement never returns k + 1
        if (atomicSub(&deg[u], 1) == k + 1) {
          removed[u] = 1;
          key[u] = next_round;
          peel_enqueue(ro, u, p ^ 1, chunks, chunk_cap, sh);
        }
      }
    }
    // every CTA has read this round's counters: they become round r + 2's
    grid_barrier(sh, G, [sh, p] {
      sh->fc[p] = 0;
      sh->acount = 0;
      sh->mindeg = 0x7fffffff;
    });
    left -= nf;
    r += 1;
    full = false;
  }
  if (blockIdx.x == 0 && tid == 0) *out_degeneracy = deg_max;
}

// ---- asynchronous peel (method 2): no rounds inside a level.  A level k
// starts with a scan of the alive list that claims every live vertex with
// degree <= k; from then on the claimed vertices' adjacency is consumed as a
// task queue of 32-edge chunks by every warp of the grid, and a decrement
// that takes a neighbour from k+1 to k claims it on the spot (its chunks are
// appended to the queue).  The level ends at quiescence -- every claimed
// chunk processed -- detected on two monotonic counters (chunks claimed,
// chunks done; done is read first).  Positions are handed out at claim time, so a vertex's later
// neighbours are exactly those that had not decremented it yet: at most k,
// a valid degeneracy order (graph.py:183-210's invariant) with the same
// degeneracy, in a data-dependent order (tie-breaks differ from run to run).
// Per level: two grid barriers instead of one per peel round.
constexpr int APEEL_THREADS = 256;
#ifndef MCE_APEEL_BATCH
#define MCE_APEEL_BATCH 8
#endif
constexpr int APEEL_BATCH = MCE_APEEL_BATCH;  // queue slots a warp reserves at once
constexpr unsigned long long TASK_EMPTY = ~0ull;
constexpr int APEEL_TRACE_LEVELS = 4096;
constexpr unsigned APEEL_MIN_PART = 256;

struct APeelShared {
  alignas(128) unsigned int bar_count;
  unsigned int bar_gen;
  alignas(128) unsigned long long tclaim;  // chunks claimed (producers need the old value)
  alignas(128) unsigned long long tdone;   // chunks processed (no-return adds)
  alignas(128) unsigned long long head;    // queue slots reserved by consumers
  alignas(128) unsigned int vclaim;        // positions handed out
  alignas(128) unsigned int acount;        // scan survivors
  int mindeg;
  unsigned int scan_claims;
  int mindeg0;  // INT_MAX - minimum initial degree (max-reduced from the host's zero)
  unsigned int part;              // warps consuming chunks in this level's async phase
  unsigned long long head0;       // first queue slot of this level (static reservations)
  // hand-over to the cluster tail (k_peel_tail): set by the grid kernel when
  // at most `tail_max` vertices remain at a level boundary
  int tail;
  int tail_k, tail_degmax, tail_sel;
  unsigned int tail_na;
  alignas(128) unsigned int scans_done;  // k_peel_async1: warps past this level's scan
  alignas(128) int cert;                  // k_peel_async1: best degeneracy certificate
  int cert_maxdeg;                        // max degree of the residual it was taken on
  int cert_k0, cert_k1;                   // diagnostics: threshold before / after the jump
  unsigned long long cert_t[3];           // diagnostics: globaltimer at start / cert / end
  unsigned long long lvl[64][3];          // diagnostics: per level (k, end time, positions)
  unsigned int nlvl;
};

// ---- degeneracy certificate (k_peel_async1's residual jump).  The
// degeneracy of any subgraph is a lower bound on the graph's degeneracy d,
// so a level threshold may jump to it: every vertex still leaves with at
// most threshold <= d later neighbours.  For a sampled live vertex v one CTA
// computes the degeneracy of G[{v} + live N(v)] (|N(v)| < CERT_M): warp 0
// lists the members (ascending) and their row offsets in shared memory, all
// warps build the members' rows as CERT_M-bit bitsets in one flattened walk
// of their adjacency lists, and warp 0 runs a sequential min-degree peel
// with warp reductions.  -1 when the neighbourhood is too big.
constexpr int CERT_M = 128;               // members (v last)
constexpr int CERT_W = CERT_M / 32;       // bitset words per row
constexpr int64_t CERT_EMAX = 8192;       // adjacency entries walked per sample
constexpr int CERT_U = 8;                 // entry loads in flight per thread
struct CertCta {
  int32_t mem[CERT_M];      // live neighbours of v, ascending
  int32_t pre[CERT_M + 1];  // exclusive prefix of the members' row lengths
  int64_t start[CERT_M];    // row starts
  unsigned rows[CERT_M * CERT_W];
  int m, E;                 // members, entries (m < 0: too big)
};

__device__ __forceinline__ bool cert_live(const unsigned* __restrict__ rbits, int32_t w) {
  return !((__ldcg(&rbits[w >> 5]) >> (w & 31)) & 1u);
}

// Called by every thread of the CTA (v uniform); the result is valid in warp 0.
__device__ int peel_certificate(const int64_t* __restrict__ ro, const int32_t* __restrict__ col,
                                const unsigned* __restrict__ rbits, int32_t v, CertCta& cw) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  if (threadIdx.x < 32) {
    // members: the live neighbours (the row is ascending), v gets index m
    const int64_t r0 = ro[v], r1 = ro[v + 1];
    int m = r1 - r0 > CERT_EMAX ? -1 : 0;
    for (int64_t b = r0; m >= 0 && b < r1; b += 32) {
      const int64_t e = b + lane;
      const int32_t w = e < r1 ? col[e] : -1;
      const bool live = w >= 0 && cert_live(rbits, w);
      const unsigned bl = __ballot_sync(0xffffffffu, live);
      if (m + __popc(bl) > CERT_M - 1) {
        m = -1;
        break;
      }
      if (live) cw.mem[m + __popc(bl & lt)] = w;
      m += __popc(bl);
    }
    __syncwarp();
    // row lengths and starts, exclusive prefix over the members
    int carry = 0;
    int64_t qa[CERT_W], ql[CERT_W];  // every slot's offsets loaded before any scan
#pragma unroll
    for (int q = 0; q < CERT_W; ++q) {
      const int i = lane + 32 * q;
      qa[q] = i < m ? ro[cw.mem[i]] : 0;
      ql[q] = i < m ? ro[cw.mem[i] + 1] : 0;
    }
#pragma unroll
    for (int q = 0; q < CERT_W; ++q) {
      if (m <= 0) break;
      const int i = lane + 32 * q;
      const int64_t a = qa[q], len = i < m ? ql[q] - a : 0;
      if (i < m) cw.start[i] = a;
      const int l32 = (int)(len < CERT_EMAX ? len : CERT_EMAX);
      int inc = l32;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
      }
      if (i < m) cw.pre[i] = carry + inc - l32;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (carry > CERT_EMAX) m = -1;
    if (lane == 0) {
      cw.m = m;
      cw.E = carry;
      if (m > 0) cw.pre[m] = carry;
    }
  }
  for (int i = threadIdx.x; i < CERT_M * CERT_W; i += blockDim.x) cw.rows[i] = 0u;
  __syncthreads();
  const int m = cw.m, E = cw.E;
  if (m <= 0) {
    __syncthreads();
    return m < 0 ? -1 : 0;
  }
  // flattened walk over the CTA: entry e of the concatenated member rows
  for (int e0 = 0; e0 < E; e0 += (int)blockDim.x * CERT_U) {
    int32_t w[CERT_U];
    int own[CERT_U];
#pragma unroll
    for (int u = 0; u < CERT_U; ++u) {
      const int e = e0 + u * (int)blockDim.x + (int)threadIdx.x;
      w[u] = -1;
      own[u] = 0;
      if (e < E) {
        int lo = 0, hi = m;  // owner: last i with pre[i] <= e
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (cw.pre[mid] <= e) lo = mid; else hi = mid;
        }
        own[u] = lo;
        w[u] = col[cw.start[lo] + (e - cw.pre[lo])];
      }
    }
#pragma unroll
    for (int u = 0; u < CERT_U; ++u) {
      if (w[u] < 0 || w[u] == v) continue;
      int lo = 0, hi = m;  // w among the members (ascending)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cw.mem[mid] < w[u]) lo = mid + 1; else hi = mid;
      }
      if (lo < m && cw.mem[lo] == w[u])
        atomicOr(&cw.rows[own[u] * CERT_W + (lo >> 5)], 1u << (lo & 31));
    }
  }
  __syncthreads();
  int cert = 0;
  if (threadIdx.x < 32) {
    // v (index m) is adjacent to every member
    const int tot = m + 1;
    int dg[CERT_W];
    unsigned alive = 0;
#pragma unroll
    for (int q = 0; q < CERT_W; ++q) {
      const int i = lane + 32 * q;
      dg[q] = 0x7fff;
      if (i < m) {
        int c = 1;
#pragma unroll
        for (int x = 0; x < CERT_W; ++x) c += __popc(cw.rows[i * CERT_W + x]);
        dg[q] = c;
        alive |= 1u << q;
      } else if (i == m) {
        dg[q] = m;
        alive |= 1u << q;
      }
    }
    // min-degree peel: the certificate is the largest minimum degree seen
    for (int left = tot; left - 1 > cert; --left) {
      int key = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < CERT_W; ++q)
        if ((alive >> q) & 1u) key = min(key, (dg[q] << 8) | (lane + 32 * q));
      key = __reduce_min_sync(0xffffffffu, key);
      const int md = key >> 8, j = key & 255;
      cert = max(cert, md);
      if ((j & 31) == lane) alive &= ~(1u << (j >> 5));
#pragma unroll
      for (int q = 0; q < CERT_W; ++q) {
        const int i = lane + 32 * q;
        bool adj;
        if (j == m) adj = i < m;
        else if (i == m) adj = true;
        else adj = (cw.rows[j * CERT_W + q] >> lane) & 1u;
        if (((alive >> q) & 1u) && adj) dg[q]--;
      }
    }
  }
  __syncthreads();
  return cert;
}

// The tail kernel's own counters (zeroed by the host).
struct PeelTailState {
  alignas(128) unsigned int nloc;          // remaining vertices (local indices handed out)
  alignas(128) unsigned long long qtail;   // claimed vertices queued (monotonic)
  alignas(128) unsigned long long qhead;   // queue slots reserved by consumers
  alignas(128) unsigned long long qdone;   // queued vertices processed
  alignas(128) unsigned int claims[2];     // scan claims, by level parity
  int mindeg[2];                           // INT_MAX - min unclaimed degree, by level parity
};

template <typename F>
__device__ __forceinline__ void agrid_barrier(APeelShared* sh, unsigned int nblocks, F reset) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = &sh->bar_gen;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(&sh->bar_count, 1u) == nblocks - 1) {
      reset();
      sh->bar_count = 0;
      __threadfence();
      atomicAdd(&sh->bar_gen, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Claim the lanes' vertices (cnt[lane] of them in cand[0..cnt)): positions
// from vclaim, chunk descriptors appended to the queue; `done` processed
// chunks are retired in the same atomic as the new chunks are claimed (same
// word: the claims are counted before the work that found them is retired).
// cand[t]'s adjacency is col[e0[t], e1[t]) (the caller loads the offsets --
// the consumer ahead of its decrements, off the dependent chain)
template <int MAXC>
__device__ __forceinline__ void apeel_claim(const int32_t (&cand)[MAXC], const int64_t (&e0)[MAXC],
                                            const int64_t (&e1)[MAXC],
                                            unsigned cmask, unsigned done, APeelShared* sh,
                                            uint64_t* __restrict__ tasks, int32_t* __restrict__ order,
                                            uint8_t* __restrict__ removed, int lane) {
  // slot t holds a claim iff bit t of cmask (static indices: no local memory)
  const int cnt = __popc(cmask);
  int nch = 0;
#pragma unroll
  for (int t = 0; t < MAXC; ++t)
    if ((cmask >> t) & 1u) nch += (int)((e1[t] - e0[t] + 31) >> 5);
  int ic = cnt, in = nch;  // inclusive warp scans of vertices and chunks
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, ic, d);
    const int b = __shfl_up_sync(0xffffffffu, in, d);
    if (lane >= d) {
      ic += a;
      in += b;
    }
  }
  const int tv = __shfl_sync(0xffffffffu, ic, 31);
  const int tc = __shfl_sync(0xffffffffu, in, 31);
  if (tv == 0 && done == 0) return;
  unsigned vpos = 0;
  unsigned long long old = 0;
  if (lane == 0 && tv) {
    vpos = atomicAdd(&sh->vclaim, (unsigned)tv);
    old = atomicAdd(&sh->tclaim, (unsigned long long)tc);
  }
  // the processed chunks are retired only after the chunks they produced are
  // counted (tclaim's returned value is consumed first), so done <= claimed
  // holds at every instant
  if (tv == 0) {
    if (lane == 0 && done) atomicAdd(&sh->tdone, (unsigned long long)done);
    return;
  }
  vpos = __shfl_sync(0xffffffffu, vpos, 0);
  const unsigned long long tpos = __shfl_sync(0xffffffffu, old, 0);
  unsigned vp = vpos + (unsigned)(ic - cnt);
  unsigned long long tp = tpos + (unsigned)(in - nch);
#pragma unroll
  for (int t = 0; t < MAXC; ++t) {
    if ((cmask >> t) & 1u) {
      const int32_t v = cand[t];
      order[vp++] = v;
      removed[v] = 1;
      const int64_t end = e1[t];
      for (int64_t st = e0[t]; st < end; st += 32) {
        const int64_t len = end - st < 32 ? end - st : 32;
        tasks[tp++] = ((uint64_t)st << 6) | (uint64_t)len;
      }
    }
  }
  if (lane == 0 && done) atomicAdd(&sh->tdone, (unsigned long long)done);
}

__global__ void __launch_bounds__(APEEL_THREADS)
k_peel_async(const int64_t* __restrict__ ro, const int32_t* __restrict__ col, int64_t n,
             int32_t* __restrict__ deg, int32_t* alive_a, int32_t* alive_b,
             uint64_t* __restrict__ tasks, uint8_t* __restrict__ removed,
             int32_t* __restrict__ order, APeelShared* sh, int64_t* __restrict__ out_degeneracy,
             unsigned poll_mask, unsigned sleep_ns, unsigned long long* trace, int64_t tail_max,
             int k_floor) {
  const unsigned int G = gridDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * APEEL_THREADS + threadIdx.x;
  const int64_t gstride = (int64_t)G * APEEL_THREADS;
  auto nothing = [] {};
  int dmin = 0x7fffffff;
  for (int64_t v = gtid; v < n; v += gstride) {
    const int32_t d0 = (int32_t)(ro[v + 1] - ro[v]);
    deg[v] = d0;
    dmin = min(dmin, (int)d0);
    alive_a[v] = (int32_t)v;
    removed[v] = 0;
  }
  // the first level is the minimum degree (no empty scans below it)
  dmin = __reduce_min_sync(0xffffffffu, dmin);
  if (lane == 0 && dmin != 0x7fffffff) atomicMax(&sh->mindeg0, 0x7fffffff - dmin);
  if (gtid == 0) sh->mindeg = 0x7fffffff;  // the rest of *sh is zeroed by the host
  if (trace && gtid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trace[8 * APEEL_TRACE_LEVELS]));
  agrid_barrier(sh, G, nothing);
  int32_t* alive = alive_a;
  int32_t* alive2 = alive_b;
  int64_t na = n;
  // the first level: the minimum degree, or the density floor when higher
  // (k_floor = ceil(m / n) <= degeneracy, see peel_async)
  int32_t k = max(0x7fffffff - *(volatile int*)&sh->mindeg0, k_floor), deg_max = 0;
  for (;;) {
    // few vertices left: the remaining levels go to one thread-block cluster
    // (k_peel_tail) -- here every level pays two grid-wide barriers
    if (tail_max > 0 && n - (int64_t)*(volatile unsigned*)&sh->vclaim <= tail_max) {
      if (gtid == 0) {
        sh->tail_k = k;
        sh->tail_degmax = deg_max;
        sh->tail_sel = alive == alive_a ? 0 : 1;
        sh->tail_na = (unsigned)na;
        sh->tail = 1;
      }
      break;
    }
    // ---- scan: claim every live vertex with deg <= k (degrees are stable
    // here).  A warp covers 32 * SCAN_U consecutive entries with every load
    // issued before any is used (the scan is one dependent chain, not one
    // per 32 entries), and makes one atomic per counter.
    constexpr int SCAN_U = 8;
    for (int64_t base = (gtid - lane) * SCAN_U; base < na; base += gstride * SCAN_U) {
      int32_t v[SCAN_U], d[SCAN_U];
      uint8_t rm[SCAN_U];
#pragma unroll
      for (int u = 0; u < SCAN_U; ++u) {
        const int64_t i = base + u * 32 + lane;
        v[u] = i < na ? __ldcg(&alive[i]) : -1;
      }
#pragma unroll
      for (int u = 0; u < SCAN_U; ++u) {
        rm[u] = v[u] >= 0 ? __ldcg(&removed[v[u]]) : (uint8_t)1;
        d[u] = v[u] >= 0 ? __ldcg(&deg[v[u]]) : 0x7fffffff;
      }
      int64_t e0[SCAN_U], e1[SCAN_U];
      int nkeep = 0, md = 0x7fffffff;
      unsigned km[SCAN_U], tmask = 0;
#pragma unroll
      for (int u = 0; u < SCAN_U; ++u) {
        const bool live = !rm[u];
        const bool take = live && d[u] <= k;
        const bool keep = live && !take;
        km[u] = __ballot_sync(0xffffffffu, keep);
        nkeep += __popc(km[u]);
        if (keep) md = min(md, (int)d[u]);
        if (take) tmask |= 1u << u;
      }
#pragma unroll
      for (int u = 0; u < SCAN_U; ++u) {
        const bool t = (tmask >> u) & 1u;
        e0[u] = t ? ro[v[u]] : 0;
        e1[u] = t ? ro[v[u] + 1] : 0;
      }
      if (nkeep) {
        unsigned o = 0;
        if (lane == 0) o = atomicAdd(&sh->acount, (unsigned)nkeep);
        o = __shfl_sync(0xffffffffu, o, 0);
        const unsigned lt = (1u << lane) - 1;
#pragma unroll
        for (int u = 0; u < SCAN_U; ++u) {
          if ((km[u] >> lane) & 1u) alive2[o + __popc(km[u] & lt)] = v[u];
          o += __popc(km[u]);
        }
        md = __reduce_min_sync(0xffffffffu, md);
        if (lane == 0) atomicMin(&sh->mindeg, md);
      }
      const int ntake = __reduce_add_sync(0xffffffffu, __popc(tmask));
      if (ntake) {
        if (lane == 0) atomicAdd(&sh->scan_claims, (unsigned)ntake);
        apeel_claim<SCAN_U>(v, e0, e1, tmask, 0u, sh, tasks, order, removed, lane);
      }
    }
    // the async phase's consumers: about one warp per 4 queued chunks (at
    // least APEEL_MIN_PART), each starting on its own statically assigned
    // reservation -- a small level does not send every warp of the grid
    // through one contended head counter
    const unsigned total_warps = G * (APEEL_THREADS / 32);
    agrid_barrier(sh, G, [sh, total_warps] {
      const unsigned long long h0 = sh->head;
      const unsigned long long t0 = sh->tclaim;
      unsigned long long part = (t0 - h0 + 3) / 4;
      part = part < APEEL_MIN_PART ? APEEL_MIN_PART : part;
      part = part > total_warps ? total_warps : part;
      sh->part = (unsigned)part;
      sh->head0 = h0;
      sh->head = h0 + part * APEEL_BATCH;
    });
    const unsigned claims = *(volatile unsigned*)&sh->scan_claims;
    if (trace && gtid == 0 && k < APEEL_TRACE_LEVELS) {  // diagnostics (MCE_PEEL_TRACE)
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[8 * k + 0] = t;
      trace[8 * k + 1] = claims;
      trace[8 * k + 2] = ~0ull;  // first chunk taken (atomicMin below)
    }
    const unsigned vc = *(volatile unsigned*)&sh->vclaim;
    const int32_t mn = *(volatile int*)&sh->mindeg;
    na = *(volatile unsigned*)&sh->acount;
    {
      int32_t* t = alive;
      alive = alive2;
      alive2 = t;
    }
    if (claims) deg_max = max(deg_max, k);
    if ((int64_t)vc >= n) break;  // every position handed out
    if (claims == 0) {
      k = max(k + 1, mn);
      agrid_barrier(sh, G, [sh] {
        sh->head = sh->tclaim;  // undo the (empty) level's static reservations
        sh->acount = 0;
        sh->mindeg = 0x7fffffff;
      });
      continue;
    }
    // ---- asynchronous phase: consume chunks until quiescence
    const int32_t kp1 = k + 1;
    const unsigned gw = (unsigned)(gtid >> 5);
    bool over = gw >= *(volatile unsigned*)&sh->part;
    bool first = true;
    while (!over) {
      unsigned long long h = 0;
      if (first) {
        h = *(volatile unsigned long long*)&sh->head0 + (unsigned long long)gw * APEEL_BATCH;
        first = false;
      } else {
        if (lane == 0) h = atomicAdd(&sh->head, (unsigned long long)APEEL_BATCH);
        h = __shfl_sync(0xffffffffu, h, 0);
      }
      int got = 0;
      while (got < APEEL_BATCH) {
        uint64_t dsc = TASK_EMPTY;
        int c = 0;
        for (unsigned polls = 0;; ++polls) {
          dsc = lane < APEEL_BATCH - got ? __ldcv(&tasks[h + got + lane]) : TASK_EMPTY;
          const unsigned av = __ballot_sync(0xffffffffu, dsc != TASK_EMPTY);
          c = __ffs(~av) - 1;  // available prefix of the reservation
          if (c > 0) break;
          if ((polls & poll_mask) == poll_mask) {
            // done first, then claimed: equal values mean nothing was in
            // flight at the second read (done <= claimed, both monotonic)
            const unsigned long long dn = __ldcv(&sh->tdone);
            const unsigned long long cl = __ldcv(&sh->tclaim);
            if ((cl == dn && h + got >= cl) || __ldcv(&sh->vclaim) >= (unsigned)n) {
              over = true;
              if (trace && lane == 0 && k < APEEL_TRACE_LEVELS) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                atomicMin(&trace[8 * k + 4], t);
                atomicMax(&trace[8 * k + 5], t);
              }
              break;
            }
          }
          if (sleep_ns) __nanosleep(sleep_ns);
        }
        if (over) break;
        if (trace && lane == 0 && got == 0 && k < APEEL_TRACE_LEVELS) {
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          atomicMin(&trace[8 * k + 2], t);
        }
        // c chunks: lane l takes edge l of each; c decrements in flight per lane
        int32_t u[APEEL_BATCH];
#pragma unroll
        for (int t = 0; t < APEEL_BATCH; ++t) {
          const uint64_t dt = __shfl_sync(0xffffffffu, dsc, t);
          u[t] = -1;
          if (t < c && lane < (int)(dt & 63)) u[t] = col[(int64_t)(dt >> 6) + lane];
        }
        // every neighbour's adjacency range, loaded alongside its decrement
        // (a crosser's chunks are enqueued without another round trip)
        int64_t r0[APEEL_BATCH], r1[APEEL_BATCH];
        int old_deg[APEEL_BATCH];
#pragma unroll
        for (int t = 0; t < APEEL_BATCH; ++t) {
          r0[t] = u[t] >= 0 ? __ldg(&ro[u[t]]) : 0;
          r1[t] = u[t] >= 0 ? __ldg(&ro[u[t] + 1]) : 0;
          old_deg[t] = u[t] >= 0 ? atomicSub(&deg[u[t]], 1) : 0;
        }
        unsigned cm = 0;
#pragma unroll
        for (int t = 0; t < APEEL_BATCH; ++t)
          if (u[t] >= 0 && old_deg[t] == kp1) cm |= 1u << t;
        apeel_claim<APEEL_BATCH>(u, r0, r1, cm, (unsigned)c, sh, tasks, order, removed, lane);
        got += c;
        if (trace && lane == 0 && k < APEEL_TRACE_LEVELS) {
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          atomicMax(&trace[8 * k + 6], t);
          atomicAdd(&trace[8 * k + 7], (unsigned long long)c);
        }
      }
    }
    // the next scan runs on quiescent degrees; consumers restart at the queue end
    agrid_barrier(sh, G, [sh] {
      sh->head = sh->tclaim;
      sh->scan_claims = 0;
      sh->acount = 0;
      sh->mindeg = 0x7fffffff;
    });
    if (trace && gtid == 0 && k < APEEL_TRACE_LEVELS) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[8 * k + 3] = t;
    }
    k += 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out_degeneracy = deg_max;
}

// ---- one grid barrier per level (k_peel_async1, the default): the level's
// scan runs concurrently with the consumers of the chunks it produces, and
// quiescence additionally waits for every warp's scan (a counter bumped
// after its claims are counted).  A scan and a decrement may then want the
// same vertex (its degree dropped to k while the scan looked at it): a
// claim is a test-and-set on the `rbits` bitmap, so exactly one wins.  The
// rules are k_peel_async's otherwise -- the same valid degeneracy order
// family and degeneracy -- with one barrier and no scan -> consumer hand-off
// per level instead of two barriers.
__global__ void __launch_bounds__(APEEL_THREADS)
k_peel_async1(const int64_t* __restrict__ ro, const int32_t* __restrict__ col, int64_t n,
              int32_t* __restrict__ deg, int32_t* alive_a, int32_t* alive_b,
              uint64_t* __restrict__ tasks, uint8_t* __restrict__ removed,
              unsigned* __restrict__ rbits, int32_t* __restrict__ order, APeelShared* sh,
              int64_t* __restrict__ out_degeneracy, unsigned poll_mask, unsigned sleep_ns,
              int64_t tail_max, int k_floor, int64_t cert_n, int slack) {
  __shared__ CertCta s_cert;
  const unsigned int G = gridDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * APEEL_THREADS + threadIdx.x;
  const int64_t gstride = (int64_t)G * APEEL_THREADS;
  const unsigned total_warps = G * (APEEL_THREADS / 32);
  auto nothing = [] {};
  int dmin = 0x7fffffff;
  for (int64_t v = gtid; v < n; v += gstride) {
    const int32_t d0 = (int32_t)(ro[v + 1] - ro[v]);
    deg[v] = d0;
    dmin = min(dmin, (int)d0);
    alive_a[v] = (int32_t)v;
    removed[v] = 0;
  }
  for (int64_t w = gtid; w < (n + 31) / 32; w += gstride) rbits[w] = 0;
  if (gtid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(sh->cert_t[2]));
  dmin = __reduce_min_sync(0xffffffffu, dmin);
  if (lane == 0 && dmin != 0x7fffffff) atomicMax(&sh->mindeg0, 0x7fffffff - dmin);
  if (gtid == 0) sh->mindeg = 0x7fffffff;  // the rest of *sh is zeroed by the host
  agrid_barrier(sh, G, nothing);
  int32_t* alive = alive_a;
  int32_t* alive2 = alive_b;
  int64_t na = n;
  // the first level: the minimum degree, or the density floor when higher
  // (k_floor = ceil(m / n) <= degeneracy, see peel_async)
  int32_t k = max(0x7fffffff - *(volatile int*)&sh->mindeg0, k_floor), deg_max = 0;
  // test-and-set claim of v: true for exactly one caller
  auto claim = [&](int32_t v) {
    const unsigned bit = 1u << (v & 31);
    return !(atomicOr(&rbits[v >> 5], bit) & bit);
  };
  bool cert_done = cert_n <= 0;
  // one sampled live vertex per CTA: its closed neighbourhood's degeneracy
  // max-reduced into sh->cert (a lower bound on d); with `maxdeg`, also the
  // residual's maximum degree into sh->cert_maxdeg.  Callers barrier after.
  auto certify = [&](const int32_t* al, int64_t cnt, bool maxdeg) {
    const int64_t stride = (cnt + G - 1) / G;
    if (maxdeg) {
      int mx = 0;
      for (int64_t i = gtid; i < cnt; i += gstride) {
        const int32_t v = __ldcg(&al[i]);
        if (cert_live(rbits, v)) mx = max(mx, (int)__ldcg(&deg[v]));
      }
      mx = __reduce_max_sync(0xffffffffu, mx);
      if (lane == 0 && mx) atomicMax(&sh->cert_maxdeg, mx);
    }
    const int64_t i = (int64_t)blockIdx.x * stride;
    if (i < cnt) {
      const int32_t v = __ldcg(&al[i]);
      if (cert_live(rbits, v)) {  // uniform over the CTA
        const int c = peel_certificate(ro, col, rbits, v, s_cert);
        if (threadIdx.x == 0 && c > 0) atomicMax(&sh->cert, c);
      }
    }
  };
  // Level slack: a level may claim up to `slack` above its level number k
  // while that stays <= a certified lower bound `dlb` of d (the density
  // floor, then a certificate sampled over the residual after the first
  // level -- a graph peeled in one level pays nothing).  A vertex then
  // leaves with at most core + slack later neighbours (never above d), and
  // consecutive levels whose cascades are long merge into one (planted1m:
  // 13, the bulk level 14 and 15 become one level).  Taking the certificate
  // before the first level too (merging 12 as well) measured 35 us faster on
  // planted1m but costs a graph peeled in one level (ba200k) 25 us.
  int dlb = k_floor;
  bool slack_cert = slack > 0;
  int levels = 0;
  for (;;) {
    const unsigned vc0 = *(volatile unsigned*)&sh->vclaim;
    if (tail_max > 0 && n - (int64_t)vc0 <= tail_max) {  // see k_peel_async
      if (gtid == 0) {
        sh->tail_k = k;
        sh->tail_degmax = deg_max;
        sh->tail_sel = alive == alive_a ? 0 : 1;
        sh->tail_na = (unsigned)na;
        sh->tail = 1;
      }
      break;
    }
    // ---- residual jump (once, when at most cert_n vertices and n / 16 are
    // left).  The remaining levels of a small residual cost a barrier and a
    // scan each for little work (planted1m: 31 levels of planted cliques).
    // A certificate c <= d (the best degeneracy of a sampled vertex's live
    // closed neighbourhood) lets the threshold jump to c at once.  A vertex
    // still leaves with at most min(its degree, c) <= d later neighbours, so
    // the widest root class is unchanged; a vertex of core number k' < c may
    // get up to c instead of k'.  The jump is taken only when no residual
    // vertex has degree above 4c: a residual dominated by hubs (an R-MAT
    // core) keeps the level-by-level peel.
    if (!cert_done && na <= cert_n && na * 16 <= n) {
      cert_done = true;
      if (gtid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(sh->cert_t[0]));
      certify(alive, na, true);
      agrid_barrier(sh, G, nothing);
      const int c = *(volatile int*)&sh->cert;
      dlb = max(dlb, c);
      if (gtid == 0) {
        sh->cert_k0 = k;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(sh->cert_t[1]));
      }
      if (*(volatile int*)&sh->cert_maxdeg <= 4 * c) k = max(k, c);
      if (gtid == 0) sh->cert_k1 = k;
    }
    if (slack_cert && levels > 0 && k + slack > dlb) {
      slack_cert = false;
      certify(alive, na, false);
      agrid_barrier(sh, G, nothing);
      dlb = max(dlb, *(volatile int*)&sh->cert);
    }
    // this level's threshold: k plus the slack, within the certified bound
    const int32_t t = max(k, min(k + slack, dlb));
    // ---- scan (consumers may already be decrementing)
    constexpr int SCAN_U = 8;
    for (int64_t base = (gtid - lane) * SCAN_U; base < na; base += gstride * SCAN_U) {
      int32_t v[SCAN_U], d[SCAN_U];
      unsigned rb[SCAN_U];
#pragma unroll
      for (int u = 0; u < SCAN_U; ++u) {
        const int64_t i = base + u * 32 + lane;
        v[u] = i < na ? __ldcg(&alive[i]) : -1;
      }
#pragma unroll
      for (int u = 0; u < SCAN_U; ++u) {
        rb[u] = v[u] >= 0 ? __ldcg(&rbits[v[u] >> 5]) : ~0u;
        d[u] = v[u] >= 0 ? __ldcg(&deg[v[u]]) : 0x7fffffff;
      }
      int64_t e0[SCAN_U], e1[SCAN_U];
      int nkeep = 0, md = 0x7fffffff;
      unsigned km[SCAN_U], tmask = 0;
#pragma unroll
      for (int u = 0; u < SCAN_U; ++u) {
        const bool live = v[u] >= 0 && !((rb[u] >> (v[u] & 31)) & 1u);
        const bool take = live && d[u] <= t && claim(v[u]);
        const bool keep = live && d[u] > t;
        km[u] = __ballot_sync(0xffffffffu, keep);
        nkeep += __popc(km[u]);
        if (keep) md = min(md, (int)d[u]);
        if (take) tmask |= 1u << u;
      }
#pragma unroll
      for (int u = 0; u < SCAN_U; ++u) {
        const bool t = (tmask >> u) & 1u;
        e0[u] = t ? ro[v[u]] : 0;
        e1[u] = t ? ro[v[u] + 1] : 0;
      }
      if (nkeep) {
        unsigned o = 0;
        if (lane == 0) o = atomicAdd(&sh->acount, (unsigned)nkeep);
        o = __shfl_sync(0xffffffffu, o, 0);
        const unsigned lt = (1u << lane) - 1;
#pragma unroll
        for (int u = 0; u < SCAN_U; ++u) {
          if ((km[u] >> lane) & 1u) alive2[o + __popc(km[u] & lt)] = v[u];
          o += __popc(km[u]);
        }
        md = __reduce_min_sync(0xffffffffu, md);
        if (lane == 0) atomicMin(&sh->mindeg, md);
      }
      if (__any_sync(0xffffffffu, tmask != 0))
        apeel_claim<SCAN_U>(v, e0, e1, tmask, 0u, sh, tasks, order, removed, lane);
    }
    __threadfence();  // this warp's claims are counted before its scan is
    if (lane == 0) atomicAdd(&sh->scans_done, 1u);
    // ---- consume chunks until every scan is done and nothing is in flight
    const int32_t kp1 = t + 1;
    bool over = false;
    while (!over) {
      unsigned long long h = 0;
      if (lane == 0) h = atomicAdd(&sh->head, (unsigned long long)APEEL_BATCH);
      h = __shfl_sync(0xffffffffu, h, 0);
      int got = 0;
      while (got < APEEL_BATCH) {
        uint64_t dsc = TASK_EMPTY;
        int c = 0;
        for (unsigned polls = 0;; ++polls) {
          dsc = lane < APEEL_BATCH - got ? __ldcv(&tasks[h + got + lane]) : TASK_EMPTY;
          const unsigned av = __ballot_sync(0xffffffffu, dsc != TASK_EMPTY);
          c = __ffs(~av) - 1;
          if (c > 0) break;
          if ((polls & poll_mask) == poll_mask) {
            // scans first, then done, then claimed (all monotonic in a level)
            const unsigned sd = __ldcv(&sh->scans_done);
            const unsigned long long dn = __ldcv(&sh->tdone);
            const unsigned long long cl = __ldcv(&sh->tclaim);
            if ((sd == total_warps && cl == dn && h + got >= cl) ||
                __ldcv(&sh->vclaim) >= (unsigned)n) {
              over = true;
              break;
            }
          }
          if (sleep_ns) __nanosleep(sleep_ns);
        }
        if (over) break;
        int32_t u[APEEL_BATCH];
#pragma unroll
        for (int t = 0; t < APEEL_BATCH; ++t) {
          const uint64_t dt = __shfl_sync(0xffffffffu, dsc, t);
          u[t] = -1;
          if (t < c && lane < (int)(dt & 63)) u[t] = col[(int64_t)(dt >> 6) + lane];
        }
        int64_t r0[APEEL_BATCH], r1[APEEL_BATCH];
        int old_deg[APEEL_BATCH];
#pragma unroll
        for (int t = 0; t < APEEL_BATCH; ++t) {
          r0[t] = u[t] >= 0 ? __ldg(&ro[u[t]]) : 0;
          r1[t] = u[t] >= 0 ? __ldg(&ro[u[t] + 1]) : 0;
          old_deg[t] = u[t] >= 0 ? atomicSub(&deg[u[t]], 1) : 0;
        }
        unsigned cm = 0;
#pragma unroll
        for (int t = 0; t < APEEL_BATCH; ++t)
          if (u[t] >= 0 && old_deg[t] == kp1 && claim(u[t])) cm |= 1u << t;
        apeel_claim<APEEL_BATCH>(u, r0, r1, cm, (unsigned)c, sh, tasks, order, removed, lane);
        got += c;
      }
    }
    // the level's results are final here (every scan done, nothing in flight)
    const unsigned vc = *(volatile unsigned*)&sh->vclaim;
    const int32_t mn = *(volatile int*)&sh->mindeg;
    na = *(volatile unsigned*)&sh->acount;
    {
      int32_t* t = alive;
      alive = alive2;
      alive2 = t;
    }
    const bool claimed = vc > vc0;
    if (claimed) deg_max = max(deg_max, t);
    agrid_barrier(sh, G, [sh, t, vc] {
      sh->head = sh->tclaim;
      sh->scans_done = 0;
      sh->acount = 0;
      sh->mindeg = 0x7fffffff;
      if (sh->nlvl < 64) {  // diagnostics (MCE_PEEL_CERT_TRACE prints them)
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        sh->lvl[sh->nlvl][0] = (unsigned long long)t;
        sh->lvl[sh->nlvl][1] = now;
        sh->lvl[sh->nlvl][2] = vc;
        sh->nlvl++;
      }
    });
    if ((int64_t)vc >= n) break;
    k = claimed ? t + 1 : max(t + 1, mn);
    ++levels;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *out_degeneracy = deg_max;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(sh->cert_t[2]));
  }
}

// ---- the asynchronous peel on ONE thread-block cluster, for the last levels
// (at most PEEL_TAIL_MAX vertices left) -- by default only small graphs
// (n <= PEEL_TAIL_SMALL_N), which it peels whole: a level costs the grid
// kernel two grid-wide barriers and a few dependent L2 round trips across
// 148 SMs for very little work.  Here
// the remaining vertices' degrees live in the cluster's distributed shared
// memory (vertex j in CTA j / PEEL_TAIL_SLICE), decrements are DSMEM
// atomics, and levels are separated by hardware cluster barriers.  Same
// rules as k_peel_async (claim deg <= k at the level's scan, claim a vertex
// the moment a decrement takes it from k + 1 to k, level over at quiescence,
// k += 1 or jump to the minimum degree): a valid degeneracy order with the
// same degeneracy.
constexpr int PEEL_TAIL_CLUSTER = 8;
constexpr int PEEL_TAIL_THREADS = 1024;
#ifndef MCE_PEEL_TAIL_MAX
#define MCE_PEEL_TAIL_MAX 65536
#endif
constexpr int PEEL_TAIL_MAX = MCE_PEEL_TAIL_MAX;
constexpr int PEEL_TAIL_SLICE = PEEL_TAIL_MAX / PEEL_TAIL_CLUSTER;
constexpr int PEEL_TAIL_BIG = 1 << 29;  // added to a claimed vertex's degree
constexpr int64_t PEEL_TAIL_SMALL_N = 8192;  // graphs this small peel on the cluster only

__global__ void __cluster_dims__(PEEL_TAIL_CLUSTER, 1, 1) __launch_bounds__(PEEL_TAIL_THREADS)
k_peel_tail(const int64_t* __restrict__ ro, const int32_t* __restrict__ col, int64_t n,
            const int32_t* __restrict__ deg, const int32_t* alive_a, const int32_t* alive_b,
            const uint8_t* __restrict__ removed, int32_t* __restrict__ order, APeelShared* sh,
            PeelTailState* ts, int32_t* __restrict__ lidx, int32_t* __restrict__ gid,
            int32_t* __restrict__ queue, int64_t* __restrict__ out_degeneracy) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  if (!*(volatile int*)&sh->tail) return;  // the grid kernel finished the peel itself
  __shared__ int sdeg[PEEL_TAIL_SLICE];
  const int rank = (int)cl.block_rank();
  const int lane = threadIdx.x & 31;
  constexpr int WPB = PEEL_TAIL_THREADS / 32;
  constexpr int NW = PEEL_TAIL_CLUSTER * WPB;
  const int gw = rank * WPB + (threadIdx.x >> 5);
  const unsigned lt = (1u << lane) - 1u;
  const int32_t* alive = sh->tail_sel ? alive_b : alive_a;
  const unsigned na = sh->tail_na;
  // local ids of the remaining vertices, their degrees into the owner CTA's slice
  for (unsigned base = (unsigned)gw * 32; base < na; base += NW * 32) {
    const unsigned i = base + lane;
    const int32_t v = i < na ? alive[i] : -1;
    const bool live = v >= 0 && !removed[v];
    const unsigned m = __ballot_sync(0xffffffffu, live);
    unsigned o = 0;
    if (lane == 0 && m) o = atomicAdd(&ts->nloc, (unsigned)__popc(m));
    o = __shfl_sync(0xffffffffu, o, 0);
    if (live) {
      const int j = (int)(o + __popc(m & lt));
      lidx[v] = j;
      gid[j] = v;
      int* rd = cl.map_shared_rank(sdeg, j / PEEL_TAIL_SLICE);
      rd[j % PEEL_TAIL_SLICE] = deg[v];
    }
  }
  cl.sync();
  const int nloc = (int)*(volatile unsigned*)&ts->nloc;
  const int s0 = rank * PEEL_TAIL_SLICE;
  const int s1 = min(nloc, s0 + PEEL_TAIL_SLICE);
  int k = sh->tail_k, deg_max = sh->tail_degmax;
  for (int level = 0;; ++level) {
    const int p = level & 1;
    if (rank == 0 && threadIdx.x == 0) {  // the other parity's counters, for the next level
      ts->claims[p ^ 1] = 0;
      ts->mindeg[p ^ 1] = 0;
    }
    // ---- scan of this CTA's slice (no decrements run now)
    int md = 0x7fffffff;
    for (int base = s0 + (threadIdx.x & ~31); base < s1; base += PEEL_TAIL_THREADS) {
      const int j = base + lane;
      const int d = j < s1 ? sdeg[j - s0] : PEEL_TAIL_BIG;
      const bool take = d <= k;
      if (d < PEEL_TAIL_BIG && !take) md = min(md, d);
      const unsigned tm = __ballot_sync(0xffffffffu, take);
      if (tm) {
        unsigned pos = 0;
        unsigned long long q = 0;
        if (lane == 0) {
          pos = atomicAdd(&sh->vclaim, (unsigned)__popc(tm));
          q = atomicAdd(&ts->qtail, (unsigned long long)__popc(tm));
          atomicAdd(&ts->claims[p], (unsigned)__popc(tm));
        }
        pos = __shfl_sync(0xffffffffu, pos, 0);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (take) {
          const int r = __popc(tm & lt);
          sdeg[j - s0] = d + PEEL_TAIL_BIG;
          order[pos + r] = gid[j];
          queue[q + r] = j;
        }
      }
    }
    md = __reduce_min_sync(0xffffffffu, md);
    if (lane == 0 && md != 0x7fffffff) atomicMax(&ts->mindeg[p], 0x7fffffff - md);
    cl.sync();
    const unsigned claims = *(volatile unsigned*)&ts->claims[p];
    if (claims) deg_max = max(deg_max, k);
    if ((int64_t)*(volatile unsigned*)&sh->vclaim >= n) break;
    if (claims == 0) {
      k = max(k + 1, 0x7fffffff - *(volatile int*)&ts->mindeg[p]);
      cl.sync();  // everyone has read this parity's counters
      continue;
    }
    // ---- consume the queue until quiescence: a decrement taking a vertex
    // from k + 1 to k claims it (one DSMEM atomic decides)
    const int kp1 = k + 1;
    for (;;) {
      unsigned long long h = 0;
      if (lane == 0) h = atomicAdd(&ts->qhead, 1ull);
      h = __shfl_sync(0xffffffffu, h, 0);
      bool over = false;
      int32_t item = -1;
      for (;;) {  // slot h is written just after its producer's qtail add (-1 until then)
        item = *(volatile int32_t*)&queue[h];
        if (item >= 0) break;
        // processed first, then queued: equal values mean nothing in flight
        const unsigned long long dn = *(volatile unsigned long long*)&ts->qdone;
        const unsigned long long qt = *(volatile unsigned long long*)&ts->qtail;
        if (dn == qt && h >= qt) {
          over = true;
          break;
        }
        __nanosleep(32);
      }
      if (over) break;
      const int32_t v = gid[item];
      const int64_t e0 = ro[v], e1 = ro[v + 1];
      for (int64_t base = e0; base < e1; base += 32) {
        const int64_t e = base + lane;
        bool claim = false;
        int l = 0;
        if (e < e1) {
          const int32_t u = col[e];
          if (!removed[u]) {
            l = lidx[u];
            int* rd = cl.map_shared_rank(sdeg, l / PEEL_TAIL_SLICE);
            const int old = atomicSub(&rd[l % PEEL_TAIL_SLICE], 1);
            if (old == kp1) {
              atomicAdd(&rd[l % PEEL_TAIL_SLICE], PEEL_TAIL_BIG);
              claim = true;
            }
          }
        }
        const unsigned cm = __ballot_sync(0xffffffffu, claim);
        if (cm) {
          unsigned pos = 0;
          unsigned long long q = 0;
          if (lane == 0) {
            pos = atomicAdd(&sh->vclaim, (unsigned)__popc(cm));
            q = atomicAdd(&ts->qtail, (unsigned long long)__popc(cm));
          }
          pos = __shfl_sync(0xffffffffu, pos, 0);
          q = __shfl_sync(0xffffffffu, q, 0);
          if (claim) {
            const int r = __popc(cm & lt);
            order[pos + r] = gid[l];
            queue[q + r] = l;
          }
        }
      }
      __threadfence();  // the vertices it queued are counted before it is done
      __syncwarp();
      if (lane == 0) atomicAdd(&ts->qdone, 1ull);
    }
    cl.sync();
    if (rank == 0 && threadIdx.x == 0) ts->qhead = *(volatile unsigned long long*)&ts->qtail;
    k += 1;
    cl.sync();
  }
  if (rank == 0 && threadIdx.x == 0) *out_degeneracy = deg_max;
}

// ids 0..n-1 (the values of the stable round sort)
__global__ void k_iota32(int32_t* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

// position of the i-th vertex of the (round, id) order
__global__ void k_peel_positions(const int32_t* __restrict__ ids, int64_t n,
                                 int64_t* __restrict__ pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    pos[ids[i]] = i;
}

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

// ndeg[pos[v]] = deg(v); ndeg[n] = 0 (so an exclusive scan gives n + 1 offsets)
__global__ void k_permuted_degrees(const int64_t* __restrict__ ro, const int64_t* __restrict__ pos,
                                   int64_t n, int64_t* __restrict__ ndeg) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x)
    ndeg[v < n ? pos[v] : n] = v < n ? ro[v + 1] - ro[v] : 0;
}

// Bitonic sort of 32*E values held E per lane (element lane*E + e),
// ascending: exchanges between lanes by shuffles, within a lane in registers.
template <int E>
__device__ __forceinline__ void warp_bitonic(int32_t (&x)[E], int lane) {
  constexpr int N = 32 * E;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= E) {
        const int lj = j / E;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int idx = lane * E + e;
          const int32_t y = __shfl_xor_sync(0xffffffffu, x[e], lj);
          const bool up = (idx & k) == 0, lower = (lane & lj) == 0;
          x[e] = (lower == up) ? min(x[e], y) : max(x[e], y);
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int q = e ^ j;
          if (q > e) {
            const bool up = ((lane * E + e) & k) == 0;
            const int32_t a = x[e], b = x[q];
            const bool sw = (a > b) == up;
            x[e] = sw ? b : a;
            x[q] = sw ? a : b;
          }
        }
      }
    }
  }
}

// one row of d <= 32*E entries: map through pos, sort, store
template <int E>
__device__ __forceinline__ void reorder_row(const int32_t* __restrict__ col,
                                            const int64_t* __restrict__ pos, int64_t src, int d,
                                            int32_t* __restrict__ out, int64_t dst, int lane) {
  int32_t x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int idx = lane * E + e;
    x[e] = idx < d ? (int32_t)pos[col[src + idx]] : 0x7fffffff;
  }
  warp_bitonic<E>(x, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int idx = lane * E + e;
    if (idx < d) out[dst + idx] = x[e];
  }
}

// Relabel and sort each row in one pass, one warp per source row: rows of up
// to REORDER_REG entries are sorted in registers (a warp bitonic network over
// E = ceil(d/32) <= 8 values per lane); longer rows are written unsorted to
// `tmp` and listed as segments (begin/end) for k_sort_long_rows.
constexpr int REORDER_THREADS = 256;
constexpr int REORDER_REG = 256;
__global__ void __launch_bounds__(REORDER_THREADS)
k_reorder_rows(const int64_t* __restrict__ ro, const int32_t* __restrict__ col, int64_t n,
               const int64_t* __restrict__ pos, const int64_t* __restrict__ nro,
               int32_t* __restrict__ out, int32_t* __restrict__ tmp, int64_t* __restrict__ seg_b,
               int64_t* __restrict__ seg_e, unsigned long long* __restrict__ nlong) {
  const int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps) {
    const int64_t src = ro[v];
    const int d = (int)(ro[v + 1] - src);
    const int64_t dst = nro[pos[v]];
    if (d <= 32) reorder_row<1>(col, pos, src, d, out, dst, lane);
    else if (d <= 64) reorder_row<2>(col, pos, src, d, out, dst, lane);
    else if (d <= 128) reorder_row<4>(col, pos, src, d, out, dst, lane);
    else if (d <= REORDER_REG) reorder_row<8>(col, pos, src, d, out, dst, lane);
    else {
      for (int i = lane; i < d; i += 32) tmp[dst + i] = (int32_t)pos[col[src + i]];
      if (lane == 0) {
        const unsigned long long idx = atomicAdd(nlong, 1ull);
        seg_b[idx] = dst;
        seg_e[idx] = dst + d;
      }
    }
  }
}

// The rows k_reorder_rows listed as long (REORDER_REG < len <= LONGROW_MAX):
// one CTA per row at a time, bitonic sort in shared memory, written in place
// of the unsorted copy.  (Longer rows -- only the largest R-MAT hubs -- go
// through a segmented sort instead.)
constexpr int LONGROW_THREADS = 1024;
constexpr int LONGROW_MAX = 16384;
__global__ void __launch_bounds__(LONGROW_THREADS)
k_sort_long_rows(const int32_t* __restrict__ tmp, int32_t* __restrict__ out,
                 const int64_t* __restrict__ seg_b, const int64_t* __restrict__ seg_e,
                 const unsigned long long* __restrict__ nlong) {
  extern __shared__ int32_t sb[];
  const unsigned long long cnt = *nlong;
  for (unsigned long long r = blockIdx.x; r < cnt; r += gridDim.x) {
    const int64_t b = seg_b[r];
    const int len = (int)(seg_e[r] - b);
    int p2 = 256;
    while (p2 < len) p2 <<= 1;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) sb[i] = i < len ? tmp[b + i] : 0x7fffffff;
    __syncthreads();
    for (int k = 2; k <= p2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < p2; i += blockDim.x) {
          const int ij = i ^ j;
          if (ij > i) {
            const int32_t x = sb[i], y = sb[ij];
            if ((x > y) == ((i & k) == 0)) {
              sb[i] = y;
              sb[ij] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int i = threadIdx.x; i < len; i += blockDim.x) out[b + i] = sb[i];
    __syncthreads();
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

// ---- row-wise canonicalisation (from_edges, graph.py:103-129): count each
// vertex's endpoints, scatter the directed entries into their rows, then
// sort + deduplicate every row where it lies (registers for rows <= 256,
// one CTA in shared memory up to LONGROW_MAX) and compact.  Instead of one
// radix sort of 2E 64-bit (u, v) keys over 2 log n bits (5 full passes on
// planted1m), each entry moves about twice.
template <typename T>
__global__ void k_count_endpoints(const T* __restrict__ edges, int64_t m, int64_t n,
                                  int32_t* __restrict__ cnt, int* __restrict__ bad) {
  bool oob = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = edges[2 * i], c = edges[2 * i + 1];
    const bool o = (a < 0) | (c < 0) | (a >= n) | (c >= n);
    oob |= o;
    if (!o && a != c) {
      atomicAdd(&cnt[a], 1);
      atomicAdd(&cnt[c], 1);
    }
  }
  if (__syncthreads_or(oob) && threadIdx.x == 0) atomicExch(bad, 1);
}

template <typename T>
__global__ void k_scatter_endpoints(const T* __restrict__ edges, int64_t m,
                                    const int64_t* __restrict__ rs, int32_t* __restrict__ cur,
                                    int32_t* __restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = (int32_t)edges[2 * i], c = (int32_t)edges[2 * i + 1];
    if (a == c) continue;
    buf[rs[a] + atomicAdd(&cur[a], 1)] = c;
    buf[rs[c] + atomicAdd(&cur[c], 1)] = a;
  }
}

// Sort 32*E entries of one row in registers, keep the first of each run of
// equal values, write them compacted to the row's start; returns the count.
template <int E>
__device__ __forceinline__ int canon_row(int32_t* __restrict__ buf, int64_t b, int d, int lane) {
  int32_t x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int idx = lane * E + e;
    x[e] = idx < d ? buf[b + idx] : 0x7fffffff;
  }
  warp_bitonic<E>(x, lane);
  const int32_t prev_last = __shfl_up_sync(0xffffffffu, x[E - 1], 1);
  unsigned keep = 0;
  int c = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int idx = lane * E + e;
    const int32_t p = e ? x[e - 1] : (lane ? prev_last : (int32_t)0x80000000);
    const bool k = idx < d && x[e] != p;
    keep |= (unsigned)k << e;
    c += k;
  }
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  int pos = incl - c;
  __syncwarp();  // every lane has read the row before any writes it back
#pragma unroll
  for (int e = 0; e < E; ++e)
    if ((keep >> e) & 1u) buf[b + pos++] = x[e];
  return __shfl_sync(0xffffffffu, incl, 31);
}

// one warp per row; rows longer than REORDER_REG listed for k_canon_long_rows
__global__ void __launch_bounds__(256)
k_canon_rows(const int64_t* __restrict__ rs, int64_t n, int32_t* __restrict__ buf,
             int32_t* __restrict__ ucnt, int64_t* __restrict__ seg_v,
             unsigned long long* __restrict__ nlong) {
  const int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps) {
    const int64_t b = rs[v];
    const int d = (int)(rs[v + 1] - b);
    int u;
    if (d == 0) u = 0;
    else if (d <= 32) u = canon_row<1>(buf, b, d, lane);
    else if (d <= 64) u = canon_row<2>(buf, b, d, lane);
    else if (d <= 128) u = canon_row<4>(buf, b, d, lane);
    else if (d <= REORDER_REG) u = canon_row<8>(buf, b, d, lane);
    else {
      if (lane == 0) seg_v[atomicAdd(nlong, 1ull)] = v;
      continue;
    }
    if (lane == 0) ucnt[v] = u;
  }
}

// the long rows: one CTA each, bitonic sort in shared memory, deduplicated
__global__ void __launch_bounds__(LONGROW_THREADS)
k_canon_long_rows(const int64_t* __restrict__ rs, int32_t* __restrict__ buf,
                  int32_t* __restrict__ ucnt, const int64_t* __restrict__ seg_v,
                  const unsigned long long* __restrict__ nlong) {
  extern __shared__ int32_t sb[];
  __shared__ int wsum[LONGROW_THREADS / 32];
  const unsigned long long cnt = *nlong;
  for (unsigned long long r = blockIdx.x; r < cnt; r += gridDim.x) {
    const int64_t v = seg_v[r];
    const int64_t b = rs[v];
    const int len = (int)(rs[v + 1] - b);
    int p2 = 256;
    while (p2 < len) p2 <<= 1;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) sb[i] = i < len ? buf[b + i] : 0x7fffffff;
    __syncthreads();
    for (int k = 2; k <= p2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < p2; i += blockDim.x) {
          const int ij = i ^ j;
          if (ij > i) {
            const int32_t x = sb[i], y = sb[ij];
            if ((x > y) == ((i & k) == 0)) {
              sb[i] = y;
              sb[ij] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    // compact the first of each run: block-wide prefix over chunks of blockDim
    int base = 0;
    for (int i0 = 0; i0 < len; i0 += blockDim.x) {
      const int i = i0 + threadIdx.x;
      const bool k = i < len && (i == 0 || sb[i] != sb[i - 1]);
      const int32_t val = k ? sb[i] : 0;
      const unsigned bm = __ballot_sync(0xffffffffu, k);
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
      if (lane == 0) wsum[w] = __popc(bm);
      __syncthreads();
      int before = 0, tot = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
        if (q < w) before += wsum[q];
        tot += wsum[q];
      }
      if (k) buf[b + base + before + __popc(bm & ((1u << lane) - 1))] = val;
      base += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) ucnt[v] = base;
    __syncthreads();
  }
}

// row v's ucnt[v] deduplicated entries from buf[rs[v] ..) to col[ro[v] ..)
// Deduplicated rows into the final CSR.  A warp moves 32 consecutive rows:
// their destinations are one contiguous range, written coalesced, each
// entry's source row found by a 5-step shuffle search over the rows' offsets
// (a warp per row waited on two offset loads for every ~20-entry row).
__global__ void k_compact_rows(const int64_t* __restrict__ rs, const int64_t* __restrict__ ro,
                               const int32_t* __restrict__ buf, int64_t n,
                               int32_t* __restrict__ col) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 32; v0 < n;
       v0 += nw * 32) {
    const int64_t v = v0 + lane;
    const int64_t src = v < n ? rs[v] : 0;
    const int64_t o = v < n ? ro[v] : INT64_MAX;
    const int64_t obeg = __shfl_sync(0xffffffffu, o, 0);
    const int64_t oend = ro[v0 + 32 < n ? v0 + 32 : n];
    constexpr int U = 4;  // loads in flight per lane
    for (int64_t base = obeg; base < oend; base += 32 * U) {
      int32_t val[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = base + 32 * u + lane;
        int r = 0;  // last row whose range starts at or before j
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int64_t t = __shfl_sync(0xffffffffu, o, r + step);
          if (t <= j) r += step;
        }
        const int64_t sr = __shfl_sync(0xffffffffu, src, r);
        const int64_t orr = __shfl_sync(0xffffffffu, o, r);
        val[u] = j < oend ? buf[sr + (j - orr)] : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (base + 32 * u + lane < oend) col[base + 32 * u + lane] = val[u];
    }
  }
}

__global__ void k_widen32(const int32_t* __restrict__ src, int64_t count, int64_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_max_i32(const int32_t* __restrict__ x, int64_t count, int* __restrict__ out) {
  int mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, x[i]);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// Row-wise canonical CSR of g from device edges (two host waits: the
// counts' maximum, then the deduplicated total).  Returns 1 -- nothing
// changed -- when a vertex has more than CANON_ROWS_MAX_DEG endpoints: the
// key sort handles hubs better (ba200k's 7.6 k-entry rows: 0.57 ms by key
// sort, 0.70 ms by rows; planted1m, all rows <= 256: 3.09 -> 2.78 ms and
// steadier).  -2 for an id outside [0, n).
constexpr int CANON_ROWS_MAX_DEG = 2048;
static_assert(CANON_ROWS_MAX_DEG <= LONGROW_MAX, "long canonical rows are sorted by one CTA");
template <typename T>
int canon_rows(mce_graph* g, const T* d_edges, int64_t num_edges, cudaStream_t s) {
  const int64_t n = g->n;
  int32_t *cnt = nullptr, *cur = nullptr, *buf = nullptr, *ucnt = nullptr;
  int64_t *rs = nullptr, *seg = nullptr;
  int* flags = nullptr;  // [0] out of range, [1] max endpoints per vertex
  unsigned long long* nlong = nullptr;
  if (dev_alloc(&cnt, n, s) || dev_alloc(&flags, 2, s)) return -1;
  MCE_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * n, s));
  MCE_CHECK(cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
  k_count_endpoints<T><<<grid_for(num_edges), 256, 0, s>>>(d_edges, num_edges, n, cnt, flags);
  mce_count_launch();
  k_max_i32<<<grid_for(n), 256, 0, s>>>(cnt, n, flags + 1);
  mce_count_launch();
  int hf[2] = {0, 0};
  MCE_CHECK(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, s));
  MCE_CHECK(cudaStreamSynchronize(s));
  dev_free(flags, s);
  if (hf[0]) {
    dev_free(cnt, s);
    mce_set_error("vertex id outside [0, num_vertices)");
    return -2;
  }
  if (hf[1] > CANON_ROWS_MAX_DEG) {
    dev_free(cnt, s);
    return 1;
  }
  // row starts of the raw (duplicate-carrying) rows
  if (dev_alloc(&rs, n + 1, s)) return -1;
  MCE_CHECK(cudaMemsetAsync(rs + n, 0, sizeof(int64_t), s));
  k_widen32<<<grid_for(n), 256, 0, s>>>(cnt, n, rs);
  mce_count_launch();
  size_t tb = 0;
  MCE_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, rs, rs, n + 1, s));
  void* tmp = nullptr;
  MCE_CHECK(cudaMallocAsync(&tmp, tb, s));
  MCE_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tb, rs, rs, n + 1, s));
  cur = cnt;  // reused as the scatter cursors
  MCE_CHECK(cudaMemsetAsync(cur, 0, sizeof(int32_t) * n, s));
  if (dev_alloc(&buf, 2 * num_edges, s) || dev_alloc(&ucnt, n, s) || dev_alloc(&seg, n + 1, s))
    return -1;
  nlong = reinterpret_cast<unsigned long long*>(seg + n);
  MCE_CHECK(cudaMemsetAsync(nlong, 0, sizeof(unsigned long long), s));
  k_scatter_endpoints<T><<<grid_for(num_edges), 256, 0, s>>>(d_edges, num_edges, rs, cur, buf);
  mce_count_launch();
  k_canon_rows<<<grid_for(n * 32), 256, 0, s>>>(rs, n, buf, ucnt, seg, nlong);
  mce_count_launch();
  static bool attr = false;
  if (!attr) {
    MCE_CHECK(cudaFuncSetAttribute(k_canon_long_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(LONGROW_MAX * sizeof(int32_t))));
    attr = true;
  }
  k_canon_long_rows<<<296, LONGROW_THREADS, LONGROW_MAX * sizeof(int32_t), s>>>(rs, buf, ucnt, seg,
                                                                                nlong);
  mce_count_launch();
  // final row offsets (the deduplicated counts' exclusive sum)
  if (dev_alloc(&g->ro, n + 1, s)) return -1;
  MCE_CHECK(cudaMemsetAsync(g->ro + n, 0, sizeof(int64_t), s));
  k_widen32<<<grid_for(n), 256, 0, s>>>(ucnt, n, g->ro);
  mce_count_launch();
  MCE_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tb, g->ro, g->ro, n + 1, s));
  int64_t nnz = 0;
  MCE_CHECK(cudaMemcpyAsync(&nnz, g->ro + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  MCE_CHECK(cudaStreamSynchronize(s));
  g->nnz = nnz;
  if (dev_alloc(&g->col, std::max<int64_t>(nnz, 1), s)) return -1;
  if (nnz > 0) {
    k_compact_rows<<<grid_for(n), 256, 0, s>>>(rs, g->ro, buf, n, g->col);
    mce_count_launch();
  }
  MCE_CHECK(cudaGetLastError());
  cudaFreeAsync(tmp, s);
  dev_free(cnt, s);
  dev_free(rs, s);
  dev_free(buf, s);
  dev_free(ucnt, s);
  dev_free(seg, s);
  return mce_graph_build_split(g, s);
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

// Bucket peeling in one persistent launch + one (round, id) sort; positions
// to d_pos (device).
int peel_parallel(const mce_graph* g, int64_t* d_pos, int64_t* d_degeneracy, cudaStream_t s) {
  const int64_t n = g->n;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  MCE_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_peel_persistent,
                                                          PEEL_THREADS, 0));
  if (per_sm < 1) {
    mce_set_error("peel kernel does not fit on an SM");
    return -3;
  }
  // every CTA must be co-resident (software grid barrier)
  int64_t grid = std::min<int64_t>((int64_t)per_sm * sms, std::max<int64_t>(1, (n + 2047) / 2048));
  int32_t *deg = nullptr, *alive = nullptr, *alive2 = nullptr;
  uint64_t* chunks = nullptr;
  uint8_t* removed = nullptr;
  uint32_t* key = nullptr;  // round of every vertex
  PeelShared* sh = nullptr;
  // one round's descriptors: sum over its vertices of ceil(deg/32) <= n + 2m/32
  const int64_t chunk_cap = n + g->nnz / 32 + 1;
  if (dev_alloc(&deg, n, s) || dev_alloc(&alive, n, s) || dev_alloc(&alive2, n, s) ||
      dev_alloc(&chunks, 2 * chunk_cap, s) || dev_alloc(&removed, n, s) ||
      dev_alloc(&key, n, s) || dev_alloc(&sh, 1, s))
    return -1;
  PeelShared init{};
  init.mindeg = 0x7fffffff;
  MCE_CHECK(cudaMemcpyAsync(sh, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  k_peel_persistent<<<(int)grid, PEEL_THREADS, 0, s>>>(g->ro, g->col, n, deg, alive, alive2,
                                                      chunks, chunk_cap, removed, key, sh,
                                                      d_degeneracy);
  mce_count_launch();
  MCE_CHECK(cudaGetLastError());
  // rounds < n, ids < 2^31: sort the (round, id) keys over the bits they use
  // stable sort of the vertex ids by round (ids enter ascending, so ties stay
  // in id order); rounds < n bound the key bits
  {
    const int rb = bits_for(std::max<int64_t>(n, 2));
    uint32_t* key2 = nullptr;
    int32_t *ids = nullptr, *ids2 = nullptr;
    if (dev_alloc(&key2, n, s) || dev_alloc(&ids, n, s) || dev_alloc(&ids2, n, s)) return -1;
    k_iota32<<<grid_for(n), 256, 0, s>>>(ids, n);
    mce_count_launch();
    cub::DoubleBuffer<uint32_t> dk(key, key2);
    cub::DoubleBuffer<int32_t> dv(ids, ids2);
    size_t tb = 0;
    MCE_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, 0, rb, s));
    void* tmp = nullptr;
    MCE_CHECK(cudaMallocAsync(&tmp, tb, s));
    MCE_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, n, 0, rb, s));
    cudaFreeAsync(tmp, s);
    k_peel_positions<<<grid_for(n), 256, 0, s>>>(dv.Current(), n, d_pos);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    dev_free(key2, s); dev_free(ids, s); dev_free(ids2, s);
  }
  dev_free(deg, s); dev_free(alive, s); dev_free(alive2, s); dev_free(chunks, s);
  dev_free(removed, s); dev_free(key, s); dev_free(sh, s);
  return 0;
}

unsigned apeel_env(const char* name, unsigned dflt) {  // diagnostics knobs
  const char* e = getenv(name);
  return e ? (unsigned)atoi(e) : dflt;
}

// Asynchronous peel (method 2); positions to d_pos straight from the claim order.
int peel_async(const mce_graph* g, int64_t* d_pos, int64_t* d_degeneracy, cudaStream_t s,
               Scratch& scr) {
  const int64_t n = g->n;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static int per_sm = -1;
  if (per_sm < 0) {  // (both variants: the smaller residency bounds the grid)
    int a = 0, b = 0;
    MCE_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_peel_async, APEEL_THREADS, 0));
    MCE_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_peel_async1, APEEL_THREADS, 0));
    per_sm = std::min(a, b);
  }
  if (per_sm < 1) {
    mce_set_error("async peel kernel does not fit on an SM");
    return -3;
  }
  const char* e = getenv("MCE_APEEL_CTAS_PER_SM");  // diagnostics
  const int want = e ? atoi(e) : 2;
  int64_t grid = std::min<int64_t>((int64_t)std::min(per_sm, std::max(want, 1)) * sms,
                                   std::max<int64_t>(1, (n + 127) / 128));
  int32_t *deg = nullptr, *alive = nullptr, *alive2 = nullptr, *order = nullptr;
  uint64_t* tasks = nullptr;
  uint8_t* removed = nullptr;
  APeelShared* sh = nullptr;
  const int64_t task_cap = n + g->nnz / 32 + 2 * APEEL_BATCH * grid * (APEEL_THREADS / 32) + 64;
  if (scr.get(&deg, n) || scr.get(&alive, n) || scr.get(&alive2, n) || scr.get(&order, n) ||
      scr.get(&tasks, task_cap) || scr.get(&removed, n) || scr.get(&sh, 1))
    return -1;
  MCE_CHECK(cudaMemsetAsync(tasks, 0xff, sizeof(uint64_t) * task_cap, s));
  MCE_CHECK(cudaMemsetAsync(sh, 0, sizeof(APeelShared), s));  // mindeg: set by the kernel
  mce_trace_mark("peel setup");
  // diagnostics: MCE_PEEL_TRACE=<file> writes per level (k, scan end ns, scan claims,
  // alive scanned, level end ns) relative to the kernel start
  const char* trace_path = getenv("MCE_PEEL_TRACE");
  unsigned long long* trace = nullptr;
  const size_t trace_words = 8 * APEEL_TRACE_LEVELS + 1;
  if (trace_path) {
    if (scr.get(&trace, trace_words)) return -1;
    MCE_CHECK(cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * trace_words, s));
    for (int k = 0; k < APEEL_TRACE_LEVELS; ++k)  // first-quiescence slots start at ~0 (atomicMin)
      MCE_CHECK(cudaMemsetAsync(trace + 8 * k + 4, 0xff, sizeof(unsigned long long), s));
  }
  // Small graphs peel entirely on one cluster (k_peel_tail).  A larger graph's
  // last levels could too (MCE_PEEL_TAIL=<remaining vertices>), but measured
  // slower there: one warp per claimed vertex serialises the hubs of an
  // R-MAT core (rmat20 8.8 -> 11.9 ms at 4096) and 8 SMs cannot absorb a
  // planted1m level (1.88 -> 2.62 ms at 65536) -- the grid kernel's 32-edge
  // chunk tasks spread both over the whole GPU.
  const char* te = getenv("MCE_PEEL_TAIL");
  const int64_t tail_max = te ? std::min<int64_t>(atoll(te), PEEL_TAIL_MAX)
                              : (n <= PEEL_TAIL_SMALL_N ? n : 0);
  PeelTailState* ts = nullptr;
  int32_t *lidx = nullptr, *gid = nullptr, *queue = nullptr;
  if (tail_max > 0) {
    if (scr.get(&ts, 1) || scr.get(&lidx, n) || scr.get(&gid, PEEL_TAIL_MAX) ||
        scr.get(&queue, PEEL_TAIL_MAX))
      return -1;
    MCE_CHECK(cudaMemsetAsync(ts, 0, sizeof(PeelTailState), s));
    MCE_CHECK(cudaMemsetAsync(queue, 0xff, sizeof(int32_t) * PEEL_TAIL_MAX, s));
  }
  // Density floor.  A graph with degeneracy d has m <= d * n edges (each
  // vertex has at most d later neighbours), so d >= ceil(m / n): every level
  // below that threshold can be merged into ONE level at it.  Any vertex then
  // leaves with at most ceil(m / n) <= d later neighbours -- still a valid
  // degeneracy order with the same degeneracy (the d-core's vertices keep
  // degree >= d until a level at d takes them) -- and the first levels'
  // barriers and alive-list scans are skipped (planted1m: levels 3 .. 11
  // collapse into level 12).  A vertex of core c < ceil(m / n) may then get
  // up to ceil(m / n) later neighbours instead of c, so the floor is capped
  // (MCE_PEEL_DENS_CAP, default 32: such roots stay in the |P| <= 32 class).
  const int64_t dens_cap = (int64_t)apeel_env("MCE_PEEL_DENS_CAP", 32);
  const int64_t m_edges = g->nnz / 2;
  const int k_floor =
      n > 0 ? (int)std::min<int64_t>((m_edges + n - 1) / n, dens_cap) : 0;
  // residual jump of k_peel_async1 (MCE_PEEL_CERT = residual size, 0 disables)
  const int64_t cert_n = (int64_t)apeel_env("MCE_PEEL_CERT", 65536);
  // level slack of k_peel_async1 (MCE_PEEL_SLACK, 0 disables)
  const int slack = (int)apeel_env("MCE_PEEL_SLACK", 2);
  // one barrier per level (k_peel_async1) unless the per-level trace is on
  // or MCE_PEEL_MERGED=0 (diagnostics)
  const bool merged = !trace && apeel_env("MCE_PEEL_MERGED", 1) != 0;
  if (merged) {
    unsigned* rbits = nullptr;
    if (scr.get(&rbits, (n + 31) / 32)) return -1;
    k_peel_async1<<<(int)grid, APEEL_THREADS, 0, s>>>(g->ro, g->col, n, deg, alive, alive2, tasks,
                                                      removed, rbits, order, sh, d_degeneracy,
                                                      apeel_env("MCE_APEEL_POLL", 3),
                                                      apeel_env("MCE_APEEL_SLEEP", 32), tail_max,
                                                      k_floor, cert_n, slack);
  } else {
    k_peel_async<<<(int)grid, APEEL_THREADS, 0, s>>>(g->ro, g->col, n, deg, alive, alive2, tasks,
                                                     removed, order, sh, d_degeneracy,
                                                     apeel_env("MCE_APEEL_POLL", 3),
                                                     apeel_env("MCE_APEEL_SLEEP", 32), trace,
                                                     tail_max, k_floor);
  }
  mce_count_launch();
  MCE_CHECK(cudaGetLastError());
  if (merged && getenv("MCE_PEEL_CERT_TRACE")) {  // diagnostics
    APeelShared h{};
    MCE_CHECK(cudaMemcpyAsync(&h, sh, sizeof(h), cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
    fprintf(stderr, "[peel cert] cert=%d residual_maxdeg=%d k %d -> %d; cert phase %.1f us, "
                    "after it %.1f us\n", h.cert, h.cert_maxdeg, h.cert_k0, h.cert_k1,
            h.cert_t[0] ? (h.cert_t[1] - h.cert_t[0]) / 1e3 : -1.0,
            h.cert_t[0] ? (h.cert_t[2] - h.cert_t[1]) / 1e3 : -1.0);
    for (unsigned i = 0; i < h.nlvl && i < 64; ++i)
      fprintf(stderr, "[peel level] k=%llu end %.1f us positions %llu\n", h.lvl[i][0],
              i ? (h.lvl[i][1] - h.lvl[0][1]) / 1e3 : 0.0, h.lvl[i][2]);
  }
  if (tail_max > 0) {
    k_peel_tail<<<PEEL_TAIL_CLUSTER, PEEL_TAIL_THREADS, 0, s>>>(
        g->ro, g->col, n, deg, alive, alive2, removed, order, sh, ts, lidx, gid, queue,
        d_degeneracy);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
  }
  if (trace) {
    std::vector<unsigned long long> h(trace_words);
    MCE_CHECK(cudaMemcpyAsync(h.data(), trace, sizeof(unsigned long long) * trace_words,
                              cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
    if (FILE* f = fopen(trace_path, "a")) {
      const unsigned long long t0 = h[8 * APEEL_TRACE_LEVELS];
      auto us = [&](unsigned long long t) { return (t && t != ~0ull) ? (double)(t - t0) / 1e3 : -1.0; };
      fprintf(f, "# n=%lld grid=%lld: k scan_end_us claims first_work_us first_quiesce_us "
                 "last_quiesce_us last_work_us chunks level_end_us\n", (long long)n, (long long)grid);
      for (int k = 0; k < APEEL_TRACE_LEVELS; ++k)
        if (h[8 * k])
          fprintf(f, "%d %.1f %llu %.1f %.1f %.1f %.1f %llu %.1f\n", k, us(h[8 * k]), h[8 * k + 1],
                  us(h[8 * k + 2]), us(h[8 * k + 4]), us(h[8 * k + 5]), us(h[8 * k + 6]), h[8 * k + 7],
                  us(h[8 * k + 3]));
      fclose(f);
    }
  }
  k_peel_positions<<<grid_for(n), 256, 0, s>>>(order, n, d_pos);
  mce_count_launch();
  MCE_CHECK(cudaGetLastError());
  return 0;
}

// Degeneracy order into device buffers (positions, degeneracy); no host sync.
int order_device(const mce_graph* g, int method, int64_t* d_pos, int64_t* d_deg, cudaStream_t s,
                 Scratch& scr) {
  const int64_t n = g->n;
  if (method == 1) {
    int64_t leaves = 2;
    while (leaves < n) leaves <<= 1;
    uint64_t* tree = nullptr;
    if (scr.get(&tree, 2 * leaves)) return -1;
    k_exact_order<<<1, EXACT_THREADS, 0, s>>>(g->ro, g->col, n, leaves, tree, d_pos, d_deg);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    return 0;
  }
  if (method == 2) return peel_async(g, d_pos, d_deg, s, scr);
  return peel_parallel(g, d_pos, d_deg, s);
}

}  // namespace

namespace {
// Pinned host words + an event per graph for its statistics, recycled.
struct StatsSlot {
  unsigned long long* host;
  cudaEvent_t ev;
  int dev;
};
std::mutex g_slot_mu;
std::vector<StatsSlot*> g_free_slots[64];

StatsSlot* stats_slot_get(int dev) {
  std::lock_guard<std::mutex> lk(g_slot_mu);
  auto& fl = g_free_slots[dev];
  if (fl.empty()) {
    constexpr int BATCH = 256;
    unsigned long long* block = nullptr;
    if (cudaHostAlloc((void**)&block, BATCH * 4 * sizeof(unsigned long long), cudaHostAllocPortable) !=
        cudaSuccess)
      return nullptr;
    for (int i = 0; i < BATCH; ++i) {
      StatsSlot* sl = new StatsSlot{block + 4 * i, nullptr, dev};
      if (cudaEventCreateWithFlags(&sl->ev, cudaEventDisableTiming) != cudaSuccess) {
        delete sl;
        return nullptr;
      }
      fl.push_back(sl);
    }
  }
  StatsSlot* sl = fl.back();
  fl.pop_back();
  return sl;
}

void stats_slot_put(StatsSlot* sl) {
  std::lock_guard<std::mutex> lk(g_slot_mu);
  g_free_slots[sl->dev].push_back(sl);
}
}  // namespace

int mce_graph_build_split(mce_graph* g, cudaStream_t s) {
  if (!g->split && dev_alloc(&g->split, g->n, s)) return -1;
  if (!g->stats_dev && dev_alloc(&g->stats_dev, 3, s)) return -1;
  MCE_CHECK(cudaMemsetAsync(g->stats_dev, 0, 3 * sizeof(unsigned long long), s));
  if (g->n > 0) k_split<<<grid_for(g->n), 256, 0, s>>>(g->ro, g->col, g->n, g->split, g->stats_dev);
  mce_count_launch();
  MCE_CHECK(cudaGetLastError());
  StatsSlot* sl = static_cast<StatsSlot*>(g->stats_slot);
  if (!sl) {
    sl = stats_slot_get(g->device >= 0 && g->device < 64 ? g->device : 0);
    if (!sl) {
      mce_set_error("pinned statistics slot allocation failed");
      return -1;
    }
    g->stats_slot = sl;
  }
  MCE_CHECK(cudaMemcpyAsync(sl->host, g->stats_dev, 3 * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s));
  MCE_CHECK(cudaEventRecord(sl->ev, s));
  g->stats_pending = true;
  return 0;
}

int mce_graph_sync_stats(const mce_graph* cg) {
  mce_graph* g = const_cast<mce_graph*>(cg);
  if (!g->stats_pending) return 0;
  StatsSlot* sl = static_cast<StatsSlot*>(g->stats_slot);
  MCE_CHECK(cudaEventSynchronize(sl->ev));
  g->max_degree = (int64_t)sl->host[0];
  g->max_later = (int64_t)sl->host[1];
  g->max_earlier = (int64_t)sl->host[2];
  g->stats_pending = false;
  return 0;
}

extern "C" {

}  // extern "C"

template <typename T>
int from_edges_impl(const T* edges, int64_t num_edges, int64_t num_vertices, int edges_on_device,
                    void* stream, mce_graph** out) {
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
  const T* d_edges = edges;
  T* owned = nullptr;
  if (!edges_on_device && num_edges > 0) {
    if (dev_alloc(&owned, 2 * num_edges, s)) { delete g; return -1; }
    MCE_CHECK(cudaMemcpyAsync(owned, edges, sizeof(T) * 2 * num_edges,
                              cudaMemcpyHostToDevice, s));
    d_edges = owned;
  }
  const char* ks = getenv("MCE_CANON_KEYSORT");  // diagnostics: 1 = always the key sort
  if (num_edges > 0 && !(ks && atoi(ks) != 0)) {
    const int rc = canon_rows(g, d_edges, num_edges, s);
    if (rc != 1) {  // done (0) or an error; 1 = a row too long for the row path
      dev_free(owned, s);
      if (rc) delete g;
      else *out = g;
      return rc;
    }
  }
  uint64_t* keys = nullptr;
  int64_t m = 0;
  if (num_edges > 0) {
    // both directions at once: one sort of 2E keys, then one unique pass
    // merges duplicates; self-loops are all-ones keys, which sort last
    const int64_t dk = 2 * num_edges;
    int64_t* d_cnt = nullptr;  // [0] unique count, [1] out-of-range flag, [2] last key is a loop
    if (dev_alloc(&keys, dk, s) || dev_alloc(&d_cnt, 3, s)) return -1;
    MCE_CHECK(cudaMemsetAsync(d_cnt, 0, 3 * sizeof(int64_t), s));
    k_edge_keys_both<T><<<grid_for(num_edges), 256, 0, s>>>(d_edges, num_edges, b, num_vertices,
                                                         keys, (int*)(d_cnt + 1));
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    dev_free(owned, s);
    if (sort_keys(&keys, dk, 2 * b, s)) return -1;
    uint64_t* uniq = nullptr;
    if (dev_alloc(&uniq, dk, s)) return -1;
    size_t tb = 0;
    MCE_CHECK(cub::DeviceSelect::Unique(nullptr, tb, keys, uniq, d_cnt, dk, s));
    void* tmp = nullptr;
    MCE_CHECK(cudaMallocAsync(&tmp, tb, s));
    MCE_CHECK(cub::DeviceSelect::Unique(tmp, tb, keys, uniq, d_cnt, dk, s));
    cudaFreeAsync(tmp, s);
    k_last_is_loop<<<1, 1, 0, s>>>(uniq, d_cnt, 2 * b);
    mce_count_launch();
    int64_t hk[3] = {0, 0, 0};
    MCE_CHECK(cudaMemcpyAsync(hk, d_cnt, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
    dev_free(keys, s);
    dev_free(d_cnt, s);
    keys = uniq;
    if (hk[1]) {
      dev_free(keys, s);
      delete g;
      mce_set_error("vertex id outside [0, num_vertices)");
      return -2;
    }
    m = (hk[0] - hk[2]) / 2;  // directed entries come in pairs
  } else {
    dev_free(owned, s);
  }
  int rc = csr_from_sorted_keys(g, keys, 2 * m, b, s);
  dev_free(keys, s);
  if (rc) { delete g; return rc; }
  *out = g;
  return 0;
}

extern "C" {

int mce_graph_from_edges(const int64_t* edges, int64_t num_edges, int64_t num_vertices,
                         int edges_on_device, void* stream, mce_graph** out) {
  return from_edges_impl<int64_t>(edges, num_edges, num_vertices, edges_on_device, stream, out);
}

int mce_graph_from_edges32(const int32_t* edges, int64_t num_edges, int64_t num_vertices,
                           int edges_on_device, void* stream, mce_graph** out) {
  return from_edges_impl<int32_t>(edges, num_edges, num_vertices, edges_on_device, stream, out);
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
  if (mce_graph_sync_stats(g)) return -1;
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
  // stream-ordered frees back to the pool (everything was cudaMallocAsync'd):
  // no device-wide synchronisation when a graph goes out of scope
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != g->device) cudaSetDevice(g->device);
  if (g->ro) cudaFreeAsync(g->ro, 0);
  if (g->col) cudaFreeAsync(g->col, 0);
  if (g->split) cudaFreeAsync(g->split, 0);
  if (g->labels) cudaFreeAsync(g->labels, 0);
  if (g->stats_dev) cudaFreeAsync(g->stats_dev, 0);
  for (int t = 0; t < 2; ++t) {
    if (g->vhash_tab[t]) cudaFreeAsync(g->vhash_tab[t], 0);
    if (g->vhash_ev[t]) cudaEventDestroy(g->vhash_ev[t]);
  }
  if (g->up_off) cudaFreeAsync(g->up_off, 0);
  if (g->up_col) cudaFreeAsync(g->up_col, 0);
  if (g->up_ev) cudaEventDestroy(g->up_ev);
  if (g->stats_slot) {
    StatsSlot* sl = static_cast<StatsSlot*>(g->stats_slot);
    cudaEventSynchronize(sl->ev);  // its copy must land before the slot is reused
    stats_slot_put(sl);
  }
  if (cur != g->device) cudaSetDevice(cur);
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
  Scratch scr(s);
  int64_t* d_pos = position_on_device ? position : nullptr;
  int64_t* d_deg = nullptr;
  if ((!d_pos && scr.get(&d_pos, n)) || scr.get(&d_deg, 1)) return -1;
  int rc = order_device(g, method, d_pos, d_deg, s, scr);
  if (rc) return rc;
  MCE_CHECK(cudaMemcpyAsync(degeneracy, d_deg, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (!position_on_device)
    MCE_CHECK(cudaMemcpyAsync(position, d_pos, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
  MCE_CHECK(cudaStreamSynchronize(s));
  return 0;
}

}  // extern "C"

namespace {
// Relabel by device positions into a new graph; temporaries from `scr`.
int reorder_impl(const mce_graph* g, const int64_t* d_pos, cudaStream_t s, Scratch& scr,
                 mce_graph** out) {
  *out = nullptr;
  mce_graph* h = new mce_graph();
  h->device = g->device;
  h->n = g->n;
  const int64_t n = g->n;
  const int b = bits_for(std::max<int64_t>(n, 2));
  // Row-wise relabel: the new row pos[v] is v's adjacency mapped through
  // pos, so the new offsets are a scan of the permuted degrees, the rows are
  // scattered whole (coalesced), and only each row needs sorting -- a
  // segmented sort of int32 labels instead of a global sort of 64-bit keys.
  (void)b;
  const int64_t nnz = g->nnz;
  h->nnz = nnz;
  int64_t* ndeg = nullptr;
  int32_t* tmpcol = nullptr;
  if (dev_alloc(&h->ro, n + 1, s) || dev_alloc(&h->col, nnz, s) || scr.get(&ndeg, n + 1) ||
      scr.get(&tmpcol, nnz) || dev_alloc(&h->labels, n, s)) {
    delete h;
    return -1;
  }
  if (n > 0) {
    mce_trace_mark("reorder allocs");
    k_permuted_degrees<<<grid_for(n + 1), 256, 0, s>>>(g->ro, d_pos, n, ndeg);
    mce_count_launch();
    size_t tb = 0;
    MCE_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, ndeg, h->ro, n + 1, s));
    void* tmp = nullptr;
    if (scr.raw(&tmp, tb)) return -1;
    MCE_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tb, ndeg, h->ro, n + 1, s));
    if (nnz > 0) {
      // rows sorted in place by k_reorder_rows; the few long ones listed as
      // segments (the rest of the list stays empty) for one segmented sort
      int64_t* seg = nullptr;
      if (scr.get(&seg, 2 * n + 1)) return -1;
      unsigned long long* nlong = reinterpret_cast<unsigned long long*>(seg + 2 * n);
      MCE_CHECK(cudaMemsetAsync(seg, 0, sizeof(int64_t) * (2 * n + 1), s));
      k_reorder_rows<<<grid_for(n * 32, REORDER_THREADS), REORDER_THREADS, 0, s>>>(
          g->ro, g->col, n, d_pos, h->ro, h->col, tmpcol, seg, seg + n, nlong);
      mce_count_launch();
      MCE_CHECK(cudaGetLastError());
      // rows up to LONGROW_MAX: one CTA each (no host round trip); the
      // segmented sort (which reads its partition sizes back to the host)
      // only when the graph has longer rows
      if (mce_graph_sync_stats(g)) return -1;
      if (g->max_degree <= LONGROW_MAX) {
        static bool attr = false;
        if (!attr) {
          MCE_CHECK(cudaFuncSetAttribute(k_sort_long_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(LONGROW_MAX * sizeof(int32_t))));
          attr = true;
        }
        k_sort_long_rows<<<296, LONGROW_THREADS, LONGROW_MAX * sizeof(int32_t), s>>>(
            tmpcol, h->col, seg, seg + n, nlong);
        mce_count_launch();
        MCE_CHECK(cudaGetLastError());
      } else {
        tb = 0;
        MCE_CHECK(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, tmpcol, h->col, nnz, n, seg,
                                                     seg + n, s));
        if (scr.raw(&tmp, tb)) return -1;
        MCE_CHECK(cub::DeviceSegmentedSort::SortKeys(tmp, tb, tmpcol, h->col, nnz, n, seg,
                                                     seg + n, s));
      }
    }
    mce_trace_mark("reorder sorts queued");
    k_relabel<<<grid_for(n), 256, 0, s>>>(d_pos, n, g->labels, h->labels);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
  } else {
    MCE_CHECK(cudaMemsetAsync(h->ro, 0, sizeof(int64_t), s));
  }
  int rc = mce_graph_build_split(h, s);
  mce_trace_mark("split queued");
  if (rc) { mce_graph_free(h); return rc; }
  *out = h;
  return 0;
}
}  // namespace

extern "C" {

int mce_reorder(const mce_graph* g, const int64_t* position, int position_on_device,
                void* stream, mce_graph** out) {
  mce_prepare_device();
  cudaStream_t s = (cudaStream_t)stream;
  *out = nullptr;
  Scratch scr(s);
  const int64_t* d_pos = position;
  if (!position_on_device && g->n > 0) {
    int64_t* owned = nullptr;
    if (scr.get(&owned, g->n)) return -1;
    MCE_CHECK(cudaMemcpyAsync(owned, position, sizeof(int64_t) * g->n, cudaMemcpyHostToDevice, s));
    d_pos = owned;
  }
  return reorder_impl(g, d_pos, s, scr, out);
}

// Order + relabel without leaving the device (graph.py:239-243 minus stats):
// positions stay in HBM; the result's labels give the permutation back.
int mce_preprocess(const mce_graph* g, int method, int64_t* degeneracy, void* stream,
                   mce_graph** out) {
  mce_prepare_device();
  cudaStream_t s = (cudaStream_t)stream;
  *out = nullptr;
  if (degeneracy) *degeneracy = 0;
  if (g->n == 0) return mce_reorder(g, nullptr, 1, stream, out);
  mce_trace_mark("preprocess enter");
  Scratch scr(s);  // every temporary of order + reorder, released stream-ordered
  mce_trace_mark("pp scratch");
  int64_t* d_pos = nullptr;
  int64_t* d_deg = nullptr;
  if (scr.get(&d_pos, g->n) || scr.get(&d_deg, 1)) return -1;
  int rc = order_device(g, method, d_pos, d_deg, s, scr);
  mce_trace_mark("pp order queued");
  if (!rc) rc = reorder_impl(g, d_pos, s, scr, out);
  mce_trace_mark("pp reorder queued");
  // NULL degeneracy: no wait (the reordered graph's max |N+(v)| is the degeneracy,
  // available through mce_graph_info)
  if (!rc && degeneracy) {
    MCE_CHECK(cudaMemcpyAsync(degeneracy, d_deg, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
  }
  return rc;
}

}  // extern "C"


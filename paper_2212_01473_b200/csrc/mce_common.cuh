// Shared device helpers and the device-resident graph layout.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#define MCE_CHECK(call)                                                          \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess) {                                                     \
      mce_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,                   \
                    cudaGetErrorString(_e));                                     \
      return -1;                                                                 \
    }                                                                            \
  } while (0)

void mce_set_error(const char* fmt, ...);

// splitmix64 finaliser: the per-vertex term of the clique-set hash and the
// counter-based RNG of the generators (identical on host and device).
__host__ __device__ __forceinline__ uint64_t mce_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
#define MCE_SIZE_SALT 0xD1B54A32D192ED03ull

// Device-resident canonical graph: symmetric CSR, rows strictly ascending.
// `split[v]` indexes the first neighbour > v, so N-(v) = col[ro[v], split[v])
// (earlier neighbours, the first-level X) and N+(v) = col[split[v], ro[v+1])
// (later neighbours, the first-level P) -- the "CSR orientation".
struct mce_graph {
  int64_t n = 0;
  int64_t nnz = 0;            // directed entries = 2m
  int64_t* ro = nullptr;      // n + 1
  int32_t* col = nullptr;     // nnz
  int64_t* split = nullptr;   // n (lazily built)
  int64_t* labels = nullptr;  // optional: original label of every vertex (set by reorder)
  // statistics (valid after mce_graph_sync_stats): computed by the split
  // kernel and copied to pinned host memory asynchronously, so building a
  // graph never waits for the device
  int64_t max_degree = 0;
  int64_t max_later = 0;      // max |N+(v)|  (= degeneracy on a reordered graph)
  int64_t max_earlier = 0;    // max |N-(v)|
  int device = 0;
  unsigned long long* stats_dev = nullptr;  // 3 words
  void* stats_slot = nullptr;               // pinned host words + completion event
  bool stats_pending = false;
  // mix64(id) [0] / mix64(label) [1] per vertex: each built once, by the first
  // enumeration that hashes that way, and never rebuilt -- concurrent calls on
  // the same graph take the per-graph lock for the build and wait on the
  // table's event (stream-ordered) before reading it
  uint64_t* vhash_tab[2] = {nullptr, nullptr};
  cudaEvent_t vhash_ev[2] = {nullptr, nullptr};
  // the N+ lists alone, packed (built once, like vhash, by the first
  // enumeration): up_col[up_off[v], up_off[v+1]) = N+(v).  The induced-row
  // builds read only N+ lists; packed they are half the CSR and stay in L2
  int64_t* up_off = nullptr;  // n + 1
  int32_t* up_col = nullptr;  // nnz / 2
  cudaEvent_t up_ev = nullptr;
};

int mce_graph_build_split(mce_graph* g, cudaStream_t s);
// wait (on the graph's own event only) for its statistics
int mce_graph_sync_stats(const mce_graph* g);

// Keep freed stream-ordered allocations in the device pool (repeated runs
// reuse HBM instead of returning it to the driver at every synchronisation).
void mce_prepare_device();

// Scratch arena for the temporaries of one API call: one cached device
// buffer per device, bump-allocated, so a call makes no cudaMallocAsync /
// cudaFreeAsync of its own once the arena has grown to the call's demand
// (host-side driver calls dominate a millisecond-scale job otherwise).  A call
// that outgrows it takes the overflow from the stream-ordered pool and the
// arena is re-sized (stream-ordered) for the next call.  Reuse is
// stream-ordered too: releasing records an event and never waits on the host,
// and a call on another stream waits for that event on the device.  Held by
// one call at a time on the host; a concurrent call (another thread) falls
// back to the pool.
class Scratch {
 public:
  explicit Scratch(cudaStream_t s);
  ~Scratch();
  template <typename T>
  int get(T** p, size_t count) {
    void* q = nullptr;
    if (raw(&q, (count ? count : 1) * sizeof(T))) return -1;
    *p = static_cast<T*>(q);
    return 0;
  }
  int raw(void** p, size_t bytes);
  size_t reserved() const;  // arena bytes this call may use (already held, not in free memory)
  size_t demand() const { return demand_; }  // bytes this call has taken so far

 private:
  cudaStream_t s_;
  int dev_ = 0;
  bool owner_ = false;
  size_t used_ = 0, demand_ = 0;
  std::vector<void*> extra_;
};

// Free device memory, cached per device for up to a second: cudaMemGetInfo
// is a driver round trip that occasionally stalls for milliseconds, too much
// to pay on every call of a millisecond-scale job.
size_t mce_free_memory();

// MCE_TRACE=1: host timestamp marks on stderr (diagnostics; no-op otherwise)
void mce_trace_mark(const char* what);

// count of this library's own kernel launches (mce_launch_count)
void mce_count_launch(int64_t k = 1);

static inline int mce_ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

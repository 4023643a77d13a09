// Maximal clique enumeration on the device: per-warp depth-first
// Bron-Kerbosch with pivoting over independent subtrees, binary-encoded
// induced subgraphs, the split X_P / X_X excluded-set representation and a
// worker list through which busy warps donate branches to idle warps.
//
// Reference behaviour restated (file:line in /root/reference/pkg/src/mce):
//   root tasks ............. bk.py:186-209           (first/second-level subtrees)
//   induced rows ........... induced.py:61-103        (partial "ip" / full "ipx")
//   pivot .................. bk.py:82-110            (max |N(c) & P| over P|X_P, ties to the
//                                                     smallest id; X_X rows only if strictly
//                                                     better, first in prefix order)
//   traversal, node count .. scheduler.py:297-381
//   X_X stable partition ... xsets.py:55-82
//   donation conditions .... scheduler.py:346-355
//   worker list protocol ... scheduler.py:99-165
//   isolated vertices (l2) . scheduler.py:476-480
//
// The traversal tree (pivot choices, branch order, node accounting) is the
// reference's exactly, so the node total is bit-identical for every worker
// count and donation schedule.
//
// Layout.  One warp is one worker (the paper's thread block).  A bitset over
// the root's P (|P| <= CAP = 32*W) is W 32-bit words held one word per lane
// (lanes >= W hold 0).  Induced rows are stored transposed, rowsT[w][c] =
// word w of row c, with column stride CAP+1 so both access patterns are
// bank-conflict free: lane-per-candidate pivot scans read consecutive
// columns, lane-per-word row loads read one column across words.
//
// Beyond the reference's scheme (results unchanged):
//  * heavy-X roots (|X| >= HEAVY_X_MIN) take their X rows from a grid-wide
//    pre-pass (k_heavy_xrows); X members with no neighbour in P start outside
//    the X_X token list;
//  * a donated branch borrows its root's induced rows from the owner (every
//    donation happens after the last root was claimed, so they stay valid);
//  * the induced-row build walks the P then X members' N+ lists as one
//    flattened (member, neighbour) stream over the lanes.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "mce_common.cuh"
#include "mce_b200.h"

namespace {

#ifndef MCE_CMP_NARROW_MAX_W
#define MCE_CMP_NARROW_MAX_W 1
#endif
constexpr int HIST_SMEM = 128;

// 128-bit blocked bloom filter over a root's P (k_tiny's induced-row walk
// tests every N+ entry against P; most miss): bit 31 of the hash picks the
// 64-bit word, bits 19-24 and 25-30 the two bits set / tested in it.  (The
// same filter in the warp kernels' walk measured slower: 1.70 -> 1.74 ms.)
__device__ __forceinline__ uint32_t bloom_hash(int32_t w) { return (uint32_t)w * 0x9E3779B1u; }
__device__ __forceinline__ unsigned long long bloom_bits(uint32_t h) {
  return (1ull << ((h >> 19) & 63)) | (1ull << ((h >> 25) & 63));
}
#ifndef MCE_TEAM_REMOTE_MIN_P
#define MCE_TEAM_REMOTE_MIN_P 48
#endif
constexpr int TEAM_REMOTE_MIN_P = MCE_TEAM_REMOTE_MIN_P;
constexpr int CMP_WORDS = 256;  // per-warp compact_run scratch: 64 + 64 ints, 64 x 8-byte rows
constexpr int HIST_MAX = MCE_HIST_MAX;
constexpr unsigned FULLMASK = 0xffffffffu;
constexpr int ROOT_STRIPES = 32;  // root-claim counters (<= 32: one per lane in phase2())
constexpr int ROOT_STRIDE = 16;   // 128 B apart
constexpr int XROWS_PARTIAL_MAX = 2048;  // partial mode: X rows for roots with |X| <= this
// First-level roots with |X| >= HEAVY_X_MIN get their X rows from a grid-wide
// pre-pass (k_heavy_xrows) instead of one warp's walk over sum |N+(x)|: a hub
// late in the order would otherwise bound the whole launch.  Their pool slot
// (+1) rides in the root word above ROOT_ID_BITS.
#ifndef MCE_HEAVY_X_MIN
#define MCE_HEAVY_X_MIN 256
#endif
constexpr int HEAVY_X_MIN = MCE_HEAVY_X_MIN;
constexpr int HEAVY_MAX = 16384;        // heavy slots
constexpr int HEAVY_UNIT_X = 256;       // X members per pre-pass CTA
constexpr int HEAVY_UNITS_MAX = 1 << 20;
constexpr int ROOT_ID_BITS = 40;
constexpr int64_t ROOT_ID_MASK = (1ll << ROOT_ID_BITS) - 1;

// Lock-free worker list (paper §3.3, reference scheduler.py:99-165).  A parked
// worker sets its bit in `idle_bits`; a donor claims a receiver by clearing
// that bit with atomicAnd (each parked id is claimed at most once).  `state`
// packs the idle count (high 32 bits) and the donations in flight (low 32)
// so the termination test "every worker parked and nothing in flight" is a
// single atomic read-modify-write.
struct WorkerListDev {
  unsigned long long state;
  int terminated;
  int pad;
};

struct Mailbox {
  int64_t origin;   // root task the branch belongs to
  int32_t rlen;     // R path length, written into the receiver's rpath
  int32_t nxx;      // live X_X tokens, written into the receiver's xx
  int32_t has_task;
  int32_t owner;    // worker whose buffers hold the root's induced rows
  int32_t np, nx;   // the root's |P| and |X|
  int32_t xr;       // X rows in use for the root
  int32_t pubcta;   // team classes: -1 = a CTA-mate's branch (rows shared), else the donor
                    // CTA whose published rows the receiving team copies (a takeover)
};  // the branch's P and X_P bitsets go to EnumArgs::mbits (2W words per worker)

struct EnumArgs {
  int64_t n;
  const int64_t* ro;
  const int32_t* col;
  const int64_t* split;
  const int64_t* up_off;  // packed N+ lists (mce_graph::up_off / up_col)
  const int32_t* up_col;
  const uint64_t* vhash;  // mix64(label(v))
  const int64_t* roots;   // l1: vertex, l2: (u << 32) | v
  int64_t num_roots;
  const unsigned long long* num_roots_dev;  // if set: the root count, written by an earlier kernel
  unsigned long long* root_counter;  // ROOT_STRIPES counters, ROOT_STRIDE apart
  int roots_mode;
  int num_workers;
  int64_t xcap;
  int levels;
  // per-worker scratch
  uint32_t* rows_g;
  int32_t* plist_g;
  uint32_t* xrows;
  int32_t* xlist;
  int32_t* xx;
  int32_t* xtmp;
  uint32_t* stack;
  int32_t* lpx;
  int32_t* rpath;
  uint64_t* hsum;
  // outputs
  unsigned long long* g_acc;   // 0 cliques, 1 hash, 2 nodes, 3 donations, 4 max size
  unsigned long long* g_hist;  // HIST_MAX
  long long* w_metrics;        // per worker: MCE_WM_COLS columns (include/mce_b200.h)
  long long* root_cycles;      // diagnostics (MCE_PROFILE_ROOTS): SM cycles per claimed root
  int64_t* collect;
  int64_t collect_cap;
  unsigned long long* collect_len;
  // worker list
  WorkerListDev* wl;
  unsigned* idle_bits;  // ceil(num_workers / 32) words
  int* wl_wake;
  Mailbox* mbox;
  uint32_t* mbits;
  uint32_t* pub;  // shared-memory-row classes: per worker (per CTA for teams), the root's rows +
                  // plist published for the receivers of its branches (W * CAPP + CAP words)
  unsigned* pub_refs;  // teams: per CTA, takeovers still copying its published rows
  int worker_list_on;
  int min_p;
  int min_x;  // also donate branches whose node has >= min_x live X_X members (0: off)
  int xrows_partial_max;  // partial mode: X rows only for roots with |X| <= this
  const uint32_t* heavy_rows;  // X rows of the heavy-X roots (k_heavy_xrows), per slot
  const int64_t* heavy_off;    // word offset of slot h's rows (stride |X| of the root)
  int compact;                 // run small subtrees on the register copy (compact_run); 0: off
  int no_pivot;                // basic Bron-Kerbosch: branch on all of P (bk.py:124-150)
  int timing;                  // per-worker SM cycles by category (w_metrics columns 4..8)
  unsigned long long* phase_ns;  // this launch: [~first start, ~first root-list miss, last end]
};

constexpr int WM = MCE_WM_COLS;
enum TimeCat { T_BUILD = 4, T_PIVOT = 5, T_SETOPS = 6, T_WLIST = 7, T_TOTAL = 8 };

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int bsearch_i32(const int32_t* a, int len, int32_t key) {
  int lo = 0, hi = len;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (lo < len && a[lo] == key) ? lo : -1;
}

__device__ __forceinline__ bool contains_range(const int32_t* __restrict__ col, int64_t lo,
                                               int64_t hi, int32_t key) {
  int64_t end = hi;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (col[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo < end && col[lo] == key;
}

// Visit every (member i, entry col[e]) pair of `cnt` members with CSR
// ranges range(i) -> (lo, len): 32 members at a time, their ranges
// flattened over the lanes (warp scan of the lengths, owner found by a
// shuffle binary search), four entries per lane in flight -- so a warp
// keeps 128 independent col loads outstanding whatever the degree mix.
template <typename RangeF, typename VisitF>
__device__ __forceinline__ void warp_flat_walk(const int32_t* __restrict__ col, int lane, int cnt,
                                             RangeF range, VisitF visit) {
  constexpr int U = 4;
  for (int i0 = 0; i0 < cnt; i0 += 32) {
    int64_t lo = 0;
    int len = 0;
    if (i0 + lane < cnt) range(i0 + lane, lo, len);
    int incl = len;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(FULLMASK, incl, d);
      if (lane >= d) incl += t;
    }
    const int excl = incl - len;
    const int total = __shfl_sync(FULLMASK, incl, 31);
    for (int base = 0; base < total; base += 32 * U) {
      int own[U];
      int32_t val[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * 32 + lane;
        int owner = 0;  // lanes q with incl_q <= k
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int v = __shfl_sync(FULLMASK, incl, owner + step - 1);
          if (v <= k) owner += step;
        }
        own[u] = owner;
        const int64_t lo_o = __shfl_sync(FULLMASK, lo, owner);
        const int excl_o = __shfl_sync(FULLMASK, excl, owner);
        val[u] = k < total ? col[lo_o + (k - excl_o)] : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (base + u * 32 + lane < total) visit(i0 + own[u], val[u]);
    }
  }
}

// Bitsets over the root's P have W 32-bit words; lane l holds words
// l, l+32, ... (K = ceil(W/32) words per lane, lanes >= W hold 0 when W < 32).
template <int W>
struct Bits {
  static constexpr int K = (W + 31) / 32;
  uint32_t w[K];
};

// TEAM = T > 0: the paper's thread-block worker.  The T warps of a CTA
// share ONE copy of the root's induced rows in shared memory; warp 0 claims
// and builds the roots, and a busy warp hands branches to idle CTA-mates at
// any time (no row copy: the rows are the CTA's).  Across CTAs, in phase 2
// a branch goes only to a team whose T warps are all idle (a takeover): its
// warp 0 copies the branch's candidate rows from the donor team's published
// copy into the team's shared memory, then shares the branch out the same
// way.  T divides 32, so a team's idle bits sit in one word of idle_bits.
template <int W, bool PIVOT_XX, bool XROWS, bool ROWS_SMEM, int TEAM = 0>
struct Worker {
  static constexpr int CAP = 32 * W;
  static constexpr int CAPP = CAP + 1;
  static constexpr int K = (W + 31) / 32;
  static constexpr int SPW = W < 32 ? 32 : W;
  // the register-starved narrow classes instantiate only the 32-slot compact
  // copy (|P| <= 32 there anyway; a 64-slot copy would only serve > 32 live X_X)
  static constexpr bool CMP_NARROW_ONLY = W <= MCE_CMP_NARROW_MAX_W;
  using B = Bits<W>;

  const EnumArgs& a;
  const int lane;
  const int wid;
  uint32_t* rowsT;
  int32_t* plist;
  uint32_t* sP;   // the node's P, X_P and branch set, broadcast words (SPW each)
  uint32_t* sXP;
  uint32_t* sBR;
  unsigned int* s_hist;  // 32-bit CTA histogram (native shared atomics), spills at 2^31
  uint32_t* xrowsT;
  uint32_t* xrows_own;     // this worker's X-row buffer (stride a.xcap)
  int64_t xstride = 0;     // row-word stride of xrowsT (a.xcap, or |X| for a heavy root's pool rows)
  int32_t* xlist_buf;
  int32_t* xx;
  int32_t* xtmp;
  uint32_t* stk;
  int32_t* lpx;
  int32_t* rpath;
  uint64_t* hsum;
  int32_t* cu;      // compact_run scratch (shared memory): U members
  int32_t* ctok;    //   X_X tokens during a partition
  uint32_t* cbuf;   //   X_X rows during a partition (64 x 8 bytes)
  const int32_t* root_x;
  int np = 0, nx = 0;
  int64_t origin = 0;
  bool xr = false;  // X rows built for this root (see build())
  // Donated branches borrow the root's induced rows instead of rebuilding
  // them: every donation happens in phase 2 (all roots claimed), after which
  // no worker builds into its buffers again, so the root owner's rows (its
  // global rows, or for shared-memory classes the copy it publishes before
  // its first donation) and X rows stay valid until the launch ends.
  int owner_wid = 0;
  bool published = false;
  // metrics (uniform across the warp)
  long long nodes = 0, roots_claimed = 0, don_made = 0, don_recv = 0;
  unsigned long long cliques = 0, hash = 0, max_size = 0;
  bool phase2_seen = false;
  int64_t nroots = 0;  // a.num_roots, or the count an earlier kernel left in a.num_roots_dev
  // teams
  int cta = 0, tw = 0;          // team (CTA) index, warp within the team
  int team_word = 0, team_shift = 0;
  int* s_pub = nullptr;         // shared: 0 rows not published, 1 publishing, 2 published
  bool counted = true;          // this park counts toward termination (false: a leader
                                // waiting for its team in phase 1)

  __device__ Worker(const EnumArgs& args, int lane_, int wid_, uint32_t* smem_rows,
                    int32_t* smem_plist, uint32_t* smem_p, unsigned int* smem_hist,
                    int32_t* smem_cmp)
      : a(args), lane(lane_), wid(wid_), sP(smem_p), sXP(smem_p + SPW), sBR(smem_p + 2 * SPW),
        s_hist(smem_hist), cu(smem_cmp), ctok(smem_cmp + 64),
        cbuf(reinterpret_cast<uint32_t*>(smem_cmp + 128)) {
    if (ROWS_SMEM) {
      rowsT = smem_rows;
      plist = smem_plist;
    } else {
      rowsT = a.rows_g + (size_t)wid * W * CAPP;
      plist = a.plist_g + (size_t)wid * CAP;
    }
    nroots = a.num_roots_dev ? (int64_t)*(volatile const unsigned long long*)a.num_roots_dev : a.num_roots;
    if (TEAM) {
      constexpr int TT = TEAM > 0 ? TEAM : 1;
      cta = wid / TT;
      tw = wid % TT;
      team_word = (cta * TT) >> 5;
      team_shift = (cta * TT) & 31;
    }
    xrows_own = XROWS ? a.xrows + (size_t)wid * W * a.xcap : nullptr;
    xrowsT = xrows_own;
    xstride = a.xcap;
    xlist_buf = a.xlist ? a.xlist + (size_t)wid * a.xcap : nullptr;
    xx = a.xx + (size_t)wid * a.xcap;
    xtmp = a.xtmp + (size_t)wid * a.xcap;
    stk = a.stack + (size_t)wid * a.levels * 4 * W;
    lpx = a.lpx + (size_t)wid * a.levels;
    rpath = a.rpath + (size_t)wid * (a.levels + 2);
    hsum = a.hsum + (size_t)wid * (a.levels + 2);
  }

  // ---------------------------------------------------------------- timing (cfg.timing)
  __device__ __forceinline__ long long tic() const { return a.timing ? clock64() : 0; }
  __device__ __forceinline__ void toc(int col, long long t0) const {
    if (a.timing && lane == 0) a.w_metrics[(size_t)wid * WM + col] += clock64() - t0;
  }

  // ---------------------------------------------------------------- words
  __device__ __forceinline__ static bool valid(int k, int lane) { return W >= 32 || lane < W; }
  __device__ __forceinline__ int word(int k) const { return k * 32 + lane; }
  __device__ __forceinline__ uint32_t row_word(int c, int w) const { return rowsT[w * CAPP + c]; }
  __device__ __forceinline__ bool any(const B& x) const {
    uint32_t o = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) o |= x.w[k];
    return __any_sync(FULLMASK, o != 0);
  }
  __device__ __forceinline__ int popc(const B& x) const {
    int c = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) c += __popc(x.w[k]);
    return __reduce_add_sync(FULLMASK, c);
  }
  // lowest set bit (ascending local id), -1 if empty
  __device__ __forceinline__ int first(const B& x) const {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const unsigned bm = __ballot_sync(FULLMASK, x.w[k] != 0);
      if (bm) {
        const int fl = __ffs(bm) - 1;
        const uint32_t wd = __shfl_sync(FULLMASK, x.w[k], fl);
        return ((k * 32 + fl) << 5) + __ffs(wd) - 1;
      }
    }
    return -1;
  }
  __device__ __forceinline__ void row_of(int v, B& r) const {
#pragma unroll
    for (int k = 0; k < K; ++k) r.w[k] = valid(k, lane) ? row_word(v, word(k)) : 0u;
  }
  __device__ __forceinline__ void xrow_of(int32_t t, B& r) const {
#pragma unroll
    for (int k = 0; k < K; ++k)
      r.w[k] = valid(k, lane) ? xrowsT[(size_t)word(k) * xstride + t] : 0u;
  }

  // ---------------------------------------------------------------- flat walk
  template <typename RangeF, typename VisitF>
  __device__ __forceinline__ void flat_walk(int cnt, RangeF range, VisitF visit) const {
    warp_flat_walk(a.up_col, lane, cnt, range, visit);  // N+ lists only
  }

  // ---------------------------------------------------------------- build
  // Fill plist / root_x / rows (and X rows) for root `r`; returns R0 length.
  __device__ int build(int64_t r_enc) {
    const int32_t* col = a.col;
    xr = false;
    int nr;
    // l1 roots carry their heavy-X pool slot (+1) above ROOT_ID_BITS
    const int64_t r = a.roots_mode == 1 ? (r_enc & ROOT_ID_MASK) : r_enc;
    const int heavy = a.roots_mode == 1 ? (int)(r_enc >> ROOT_ID_BITS) : 0;
    xrowsT = xrows_own;
    xstride = a.xcap;
    if (a.roots_mode == 1) {
      const int64_t v = r;
      const int64_t s = a.split[v];
      np = (int)(a.ro[v + 1] - s);
      nx = (int)(s - a.ro[v]);
      for (int i = lane; i < np; i += 32) plist[i] = col[s + i];
      root_x = col + a.ro[v];
      if (lane == 0) rpath[0] = (int32_t)v;
      nr = 1;
    } else {
      const int64_t u = r >> 32, v = r & 0xffffffffll;
      // P = N+(u) & N+(v), X = N(u) & N-(v), both ascending (bk.py:198-204)
      np = 0;
      const int64_t ps = a.split[v], pe = a.ro[v + 1];
      const int64_t us = a.split[u], ue = a.ro[u + 1];
      for (int64_t base = ps; base < pe; base += 32) {
        int64_t e = base + lane;
        bool in = false;
        int32_t w = 0;
        if (e < pe) {
          w = col[e];
          in = contains_range(col, us, ue, w);
        }
        unsigned m = __ballot_sync(FULLMASK, in);
        if (in) plist[np + __popc(m & ((1u << lane) - 1))] = w;
        np += __popc(m);
      }
      nx = 0;
      const int64_t xs = a.ro[v], xe = a.split[v];
      const int64_t u0 = a.ro[u];
      for (int64_t base = xs; base < xe; base += 32) {
        int64_t e = base + lane;
        bool in = false;
        int32_t w = 0;
        if (e < xe) {
          w = col[e];
          in = contains_range(col, u0, ue, w);
        }
        unsigned m = __ballot_sync(FULLMASK, in);
        if (in) xlist_buf[nx + __popc(m & ((1u << lane) - 1))] = w;
        nx += __popc(m);
      }
      root_x = xlist_buf;
      if (lane == 0) {
        rpath[0] = (int32_t)u;
        rpath[1] = (int32_t)v;
      }
      nr = 2;
    }
    origin = r_enc;
    owner_wid = wid;
    published = false;
    if (!ROWS_SMEM) {
      rowsT = a.rows_g + (size_t)wid * W * CAPP;
      plist = a.plist_g + (size_t)wid * CAP;
    }
    __syncwarp();
    if (np == 0) return nr;
    if (W == 1 && lane >= np) plist[lane] = 0x7fffffff;  // padded for find32
    // Partial mode builds X rows only when |X| is moderate: a hub late in the
    // order (|X| in the thousands, tiny P) visits few nodes, and its handful
    // of X_X scans through the CSR cost less than sum |N+(x)| row-building
    // loads.  Full mode always needs them (X_X pivot candidates).
    xr = XROWS && (PIVOT_XX || heavy > 0 || nx <= a.xrows_partial_max);
    // a heavy-X root's rows were built by the whole grid (k_heavy_xrows)
    const bool xwalk = xr && heavy == 0;
    if (xr && heavy > 0) {
      xrowsT = const_cast<uint32_t*>(a.heavy_rows) + a.heavy_off[heavy - 1];
      xstride = nx;
    }
    for (int w = 0; w < W; ++w)
      for (int c = lane; c < np; c += 32) rowsT[w * CAPP + c] = 0;
    if (xwalk)
      for (int w = 0; w < W; ++w)
        for (int t = lane; t < nx; t += 32) xrowsT[(size_t)w * a.xcap + t] = 0;
    __syncwarp();
    // One flattened walk over the P members then the X members (a small root
    // fills one pass instead of two half-empty ones):
    //  * P rows (induced.py:61-92): each P-P edge (a_i, b) with b in N+(a_i);
    //    N+(a_i) & P lies after a_i in the ascending plist;
    //  * X rows (induced.py:95-103): X member x is earlier than every P
    //    vertex, so its P-neighbours are N+(x) & P.
    flat_walk(
        np + (xwalk ? nx : 0),
        [&](int i, int64_t& lo, int& len) {
          const int32_t m = i < np ? plist[i] : root_x[i - np];
          lo = a.up_off[m];
          len = (int)(a.up_off[m + 1] - lo);
        },
        [&](int i, int32_t w) {
          if (i < np) {
            // N+(a_i) holds only vertices after a_i: a hit is past i
            const int jj = W == 1 ? find32(w) : i + 1 + bsearch_i32(plist + i + 1, np - i - 1, w);
            if (jj > i) {
              atomicOr(&rowsT[(jj >> 5) * CAPP + i], 1u << (jj & 31));
              atomicOr(&rowsT[(i >> 5) * CAPP + jj], 1u << (i & 31));
            }
          } else {
            const int t = i - np;
            const int j = W == 1 ? find32(w) : bsearch_i32(plist, np, w);
            if (j >= 0) atomicOr(&xrowsT[(size_t)(j >> 5) * a.xcap + t], 1u << (j & 31));
          }
        });
    __syncwarp();
    return nr;
  }

  // W = 1: index of w in the padded 32-entry plist (branchless, 5 steps), -1 if absent
  __device__ __forceinline__ int find32(int32_t w) const {
    int i = 0;
    i += plist[i + 15] < w ? 16 : 0;
    i += plist[i + 7] < w ? 8 : 0;
    i += plist[i + 3] < w ? 4 : 0;
    i += plist[i + 1] < w ? 2 : 0;
    i += plist[i] < w ? 1 : 0;
    return plist[i] == w ? i : -1;
  }

  // ---------------------------------------------------------------- pieces
  __device__ __forceinline__ bool xx_adjacent(int32_t t, int v, int32_t gv) const {
    if (XROWS && xr) return (xrowsT[(size_t)(v >> 5) * xstride + t] >> (v & 31)) & 1u;
    const int32_t x = root_x[t];
    return contains_range(a.col, a.split[x], a.ro[x + 1], gv);
  }

  // Is any live X_X member adjacent to branch vertex v (global gv)?  Without
  // X rows, either test each live member x for gv in N+(x), or -- when the
  // live prefix is known ascending (`sorted`: the root's tokens and every
  // kept part cut from an ascending prefix) and gv has fewer earlier
  // neighbours than there are live members -- look each y in N-(gv) up in
  // the live prefix by binary search.
  __device__ bool xx_any_adjacent(int v, int32_t gv, int live, bool sorted = false) const {
    if (!(XROWS && xr) && sorted) {
      const int64_t nb = a.ro[gv], ne = a.split[gv];
      if (ne - nb < live) {
        for (int64_t base = nb; base < ne; base += 32) {
          const int64_t e = base + lane;
          bool hit = false;
          if (e < ne) {
            const int32_t y = a.col[e];
            int lo = 0, hi = live;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (root_x[xx[mid]] < y) lo = mid + 1; else hi = mid;
            }
            hit = lo < live && root_x[xx[lo]] == y;
          }
          if (__any_sync(FULLMASK, hit)) return true;
        }
        return false;
      }
    }
    for (int base = 0; base < live; base += 128) {  // 4 independent tests per lane in flight
      bool hit = false;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * 32 + lane;
        hit |= (i < live) && xx_adjacent(xx[i], v, gv);
      }
      if (__any_sync(FULLMASK, hit)) return true;
    }
    return false;
  }

  // stable partition of xx[0, live) by adjacency to v (xsets.py:55-82)
  __device__ int partition(int v, int32_t gv, int live) {
    constexpr int U = 4;  // tokens per lane per iteration: U independent adjacency tests in flight
    int kept = 0, dropped = 0;
    const unsigned lt = (1u << lane) - 1;
    for (int base = 0; base < live; base += 32 * U) {
      int32_t t[U];
      bool ok[U], keep[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * 32 + lane;
        ok[u] = i < live;
        t[u] = ok[u] ? xx[i] : 0;
      }
      if (XROWS && xr) {
#pragma unroll
        for (int u = 0; u < U; ++u) keep[u] = ok[u] && xx_adjacent(t[u], v, gv);
      } else {
        // U binary searches of gv in N+(x) in lockstep: U loads in flight per step
        int64_t lo[U], hi[U];
        bool hit[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int32_t x = ok[u] ? root_x[t[u]] : 0;
          lo[u] = ok[u] ? a.split[x] : 0;
          hi[u] = ok[u] ? a.ro[x + 1] : 0;
          hit[u] = false;
        }
        for (;;) {
          int32_t val[U];
          int64_t mid[U];
          bool act = false;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (lo[u] < hi[u]) {
              mid[u] = (lo[u] + hi[u]) >> 1;
              val[u] = a.col[mid[u]];
              act = true;
            }
          }
          if (!act) break;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (lo[u] < hi[u]) {
              if (val[u] == gv) {
                hit[u] = true;
                lo[u] = hi[u];
              } else if (val[u] < gv) {
                lo[u] = mid[u] + 1;
              } else {
                hi[u] = mid[u];
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) keep[u] = ok[u] && hit[u];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {  // in order: the partition stays stable
        const unsigned km = __ballot_sync(FULLMASK, keep[u]);
        const unsigned dm = __ballot_sync(FULLMASK, ok[u] && !keep[u]);
        if (keep[u]) xx[kept + __popc(km & lt)] = t[u];
        else if (ok[u]) xtmp[dropped + __popc(dm & lt)] = t[u];
        kept += __popc(km);
        dropped += __popc(dm);
      }
    }
    __syncwarp();
    for (int i = lane; i < dropped; i += 32) xx[kept + i] = xtmp[i];
    __syncwarp();
    return kept;
  }

  // number of P members adjacent to candidate column c (lane-private c)
  __device__ __forceinline__ int count_in_p(const unsigned (&pmask)[K], int c, bool xrow) const {
    // row words of up to RB P-words in flight at once (wide classes keep
    // their rows in global memory: one dependent load per word otherwise)
    constexpr int RB = W >= 8 ? 4 : 1;
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      for (unsigned pm = pmask[k]; pm;) {
        int j[RB];
        uint32_t rw[RB];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
          j[u] = pm ? k * 32 + __ffs(pm) - 1 : -1;
          pm &= pm - 1;
        }
#pragma unroll
        for (int u = 0; u < RB; ++u)
          rw[u] = j[u] < 0 ? 0u : (xrow ? xrowsT[(size_t)j[u] * xstride + c] : rowsT[j[u] * CAPP + c]);
#pragma unroll
        for (int u = 0; u < RB; ++u)
          if (j[u] >= 0) cnt += __popc(rw[u] & sP[j[u]]);
      }
    }
    return cnt;
  }

  // pivot (bk.py:82-110); BR = P - N(pivot)
  __device__ void pivot_branches(const B& P, const B& XP, int live, B& BR) {
    unsigned pmask[K], cmask[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (valid(k, lane)) sP[word(k)] = P.w[k];
      pmask[k] = __ballot_sync(FULLMASK, P.w[k] != 0);
      cmask[k] = __ballot_sync(FULLMASK, (P.w[k] | XP.w[k]) != 0);
    }
    __syncwarp();
    if (a.no_pivot) {  // basic BK: every member of P is a branch
#pragma unroll
      for (int k = 0; k < K; ++k) BR.w[k] = P.w[k];
      return;
    }
    int best = -1, bestc = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t Ck = P.w[k] | XP.w[k];
      for (unsigned cm = cmask[k]; cm; cm &= cm - 1) {
        const int fl = __ffs(cm) - 1;
        const uint32_t Cw = __shfl_sync(FULLMASK, Ck, fl);
        const int c = ((k * 32 + fl) << 5) + lane;
        if ((Cw >> lane) & 1u) {
          const int cnt = count_in_p(pmask, c, false);
          if (cnt > best) {
            best = cnt;
            bestc = c;
          }
        }
      }
    }
    const int m = (int)__reduce_max_sync(FULLMASK, (unsigned)(best + 1)) - 1;
    const int pc = __reduce_min_sync(FULLMASK, best == m ? bestc : 0x7fffffff);
    B prow;
    bool use_local = true;
    if (PIVOT_XX && live > 0) {
      int xb = -1, xpos = 0x7fffffff;
      for (int base = 0; base < live; base += 32) {
        const int i = base + lane;
        if (i < live) {
          const int cnt = count_in_p(pmask, xx[i], true);
          if (cnt > xb) {
            xb = cnt;
            xpos = i;
          }
        }
      }
      const int xm = (int)__reduce_max_sync(FULLMASK, (unsigned)(xb + 1)) - 1;
      if (xm > m) {
        const int pos = __reduce_min_sync(FULLMASK, xb == xm ? xpos : 0x7fffffff);
        xrow_of(xx[pos], prow);
        use_local = false;
      }
    }
    if (use_local) row_of(pc, prow);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) BR.w[k] = P.w[k] & ~prow.w[k];
  }

  __device__ void report(int size, uint64_t hs) {
    if (lane == 0) {
      cliques++;
      hash += mce_mix64(hs + (uint64_t)size * MCE_SIZE_SALT);
      if ((unsigned long long)size > max_size) max_size = size;
      hist_add(size, 1u);  // 32-bit shared counters (64-bit shared atomics are CAS loops)
    }
    if (a.collect_cap > 0) {
      unsigned long long pos = 0;
      if (lane == 0) pos = atomicAdd(a.collect_len, (unsigned long long)(size + 1));
      pos = __shfl_sync(FULLMASK, pos, 0);
      __syncwarp();
      if (pos + size + 1 <= (unsigned long long)a.collect_cap) {
        if (lane == 0) a.collect[pos] = size;
        for (int i = lane; i < size; i += 32) a.collect[pos + 1 + i] = rpath[i];
      }
    }
  }

  __device__ __forceinline__ void hist_add(int size, unsigned cnt) {
    if (size < HIST_SMEM) {
      const unsigned old = atomicAdd(&s_hist[size], cnt);
      if (old < 0x80000000u && old + cnt >= 0x80000000u) {  // spill 2^31 to HBM
        atomicAdd(&a.g_hist[size], 0x80000000ull);
        atomicSub(&s_hist[size], 0x80000000u);
      }
    } else {
      atomicAdd(&a.g_hist[size < HIST_MAX ? size : HIST_MAX - 1], (unsigned long long)cnt);
    }
  }

  // Leaf batch (the sibling subtrees of a node are independent given the
  // node's P, X_P, branch set BR and live X_X prefix): every branch v whose
  // child P_v & N(v) is empty -- P_v = P minus the branches before v -- is a
  // leaf of the reference's traversal (scheduler.py:358-369).  All of them
  // are decided in one lane-per-candidate pass: node count += #leaves, the
  // maximal ones (X_v & N(v) empty, X_v = X_P plus the earlier branches, and
  // no live X_X neighbour) are reported together.  Returns BR minus leaves.
  __device__ void leaf_batch(const B& P, const B& XP, const B& BR, int live, int rlen, B& NL,
                             bool xsorted) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (valid(k, lane)) {
        sXP[word(k)] = XP.w[k];
        sBR[word(k)] = BR.w[k];
      }
      NL.w[k] = BR.w[k];
    }
    unsigned umask[K];  // words where P | X_P has bits: the only row words that matter
#pragma unroll
    for (int k = 0; k < K; ++k) umask[k] = __ballot_sync(FULLMASK, (P.w[k] | XP.w[k]) != 0);
    __syncwarp();
    const uint64_t hs = hsum[rlen];
    const int size = rlen + 1;
    unsigned long long hsum_lane = 0;
    unsigned leaves = 0, maximal = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      for (unsigned bm = __ballot_sync(FULLMASK, BR.w[k] != 0); bm; bm &= bm - 1) {
        const int fl = __ffs(bm) - 1;
        const int w = k * 32 + fl;  // candidate word: candidate c = 32w + lane
        const uint32_t bw = __shfl_sync(FULLMASK, BR.w[k], fl);
        const bool cand = (bw >> lane) & 1u;
        const int c = (w << 5) + lane;
        bool leaf = false, xclear = false;
        if (cand) {
          uint32_t pin = 0, xin = 0;
          constexpr int RB = W >= 8 ? 4 : 1;  // row words in flight (see count_in_p)
#pragma unroll
          for (int q = 0; q < K; ++q) {
            for (unsigned um = umask[q]; um;) {
              int jj[RB];
              uint32_t rr[RB];
#pragma unroll
              for (int u = 0; u < RB; ++u) {
                jj[u] = um ? q * 32 + __ffs(um) - 1 : -1;
                um &= um - 1;
              }
#pragma unroll
              for (int u = 0; u < RB; ++u) rr[u] = jj[u] < 0 ? 0u : rowsT[jj[u] * CAPP + c];
#pragma unroll
              for (int u = 0; u < RB; ++u) {
                const int j = jj[u];
                if (j < 0) continue;
                const uint32_t below = j < w ? 0xffffffffu : (j == w ? (1u << lane) - 1u : 0u);
                const uint32_t bb = sBR[j] & below;
                pin |= rr[u] & (sP[j] & ~bb);
                xin |= rr[u] & (sXP[j] | bb);
              }
            }
          }
          leaf = pin == 0;
          xclear = leaf && xin == 0;
        }
        const unsigned lm = __ballot_sync(FULLMASK, leaf);
        if (!lm) continue;
        leaves += __popc(lm);
        // drop the leaves from the non-leaf branch set (word w lives in lane fl, slot k)
        if (lane == fl) NL.w[k] &= ~lm;
        unsigned xm = __ballot_sync(FULLMASK, xclear);
        if (xm && live > 0) {
          if (XROWS && xr) {
            uint32_t adj = 0;  // live X_X members' adjacency, word w
#pragma unroll 4
            for (int i = lane; i < live; i += 32) adj |= xrowsT[(size_t)w * xstride + xx[i]];
            adj = __reduce_or_sync(FULLMASK, adj);
            xm &= ~adj;
          } else {
            for (unsigned t = xm; t; t &= t - 1) {
              const int b = __ffs(t) - 1;
              const int v = (w << 5) + b;
              if (xx_any_adjacent(v, plist[v], live, xsorted)) xm &= ~(1u << b);
            }
          }
        }
        if (!xm) continue;
        if ((xm >> lane) & 1u) {
          hsum_lane += mce_mix64(hs + a.vhash[plist[c]] + (uint64_t)size * MCE_SIZE_SALT);
        }
        maximal += __popc(xm);
        if (a.collect_cap > 0) {
          for (unsigned t = xm; t; t &= t - 1) {
            const int v = (w << 5) + __ffs(t) - 1;
            collect_clique(size, plist[v]);
          }
        }
      }
    }
    nodes += leaves;
    if (maximal) {
      // 64-bit warp sum of the per-lane hashes
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) hsum_lane += __shfl_xor_sync(FULLMASK, hsum_lane, o);
      if (lane == 0) {
        cliques += maximal;
        hash += hsum_lane;
        if ((unsigned long long)size > max_size) max_size = size;
        hist_add(size, maximal);
      }
    }
  }

  // append [size, R..., last] to the clique stream (collect mode)
  __device__ void collect_clique(int size, int32_t last) {
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(a.collect_len, (unsigned long long)(size + 1));
    pos = __shfl_sync(FULLMASK, pos, 0);
    if (pos + size + 1 <= (unsigned long long)a.collect_cap) {
      if (lane == 0) {
        a.collect[pos] = size;
        a.collect[pos + size] = last;
      }
      for (int i = lane; i < size - 1; i += 32) a.collect[pos + 1 + i] = rpath[i];
    }
    __syncwarp();
  }

  // phase 2 = every root claimed: every stripe counter past its stripe
  __device__ bool phase2() {
    if (!phase2_seen) {
      const unsigned long long c =
          lane < ROOT_STRIPES ? *(volatile unsigned long long*)&a.root_counter[lane * ROOT_STRIDE] : 0ull;
      const bool done = lane >= ROOT_STRIPES ||
                        c * ROOT_STRIPES + lane >= (unsigned long long)nroots;
      phase2_seen = __all_sync(FULLMASK, done);
    }
    return phase2_seen;
  }

  // Next root (sorted heaviest first) or -1.  Roots are dealt round-robin into
  // ROOT_STRIPES stripes, each with its own counter: a warp claims from its
  // home stripe and moves on when it runs dry, so 10^4 warps do not
  // serialise on one L2 atomic while the claim order stays heaviest-first.
  __device__ int64_t claim_root(int& stripe) {
    for (int tried = 0; tried < ROOT_STRIPES; ++tried) {
      unsigned long long idx = 0;
      if (lane == 0) idx = atomicAdd(&a.root_counter[stripe * ROOT_STRIDE], 1ull);
      idx = __shfl_sync(FULLMASK, idx, 0);
      const unsigned long long r = idx * ROOT_STRIPES + stripe;
      if (r < (unsigned long long)nroots) return (int64_t)r;
      stripe = (stripe + 1) % ROOT_STRIPES;
    }
    return -1;
  }

  // donate the branch (v, childP, childXP) to an idle worker (scheduler.py:417-438)
  __device__ bool try_donate(const B& childP, const B& childXP, int v, int32_t gv, int live,
                             int rlen) {
    bool takeover = false;
    // a takeover copies the branch's candidate rows into the taking team:
    // only branches big enough to pay for it leave the team
    const int rid = TEAM ? claim_team_receiver(takeover, popc(childP) >= TEAM_REMOTE_MIN_P)
                         : claim_receiver();
    if (rid < 0) return false;
    // receiver's X_X: the live tokens adjacent to v, in prefix order
    int32_t* rx = a.xx + (size_t)rid * a.xcap;
    int k = 0;
    const unsigned lt = (1u << lane) - 1;
    for (int base = 0; base < live; base += 32) {
      int i = base + lane;
      bool keep = (i < live) && xx_adjacent(xx[i], v, gv);
      unsigned km = __ballot_sync(FULLMASK, keep);
      if (keep) rx[k + __popc(km & lt)] = xx[i];
      k += __popc(km);
    }
    send_branch(rid, childP, childXP, gv, rlen, k, takeover);
    return true;
  }

  // teams: an idle CTA-mate (local), else -- in phase 2 -- the warp 0 of a
  // fully idle team, all T of its bits taken at once (a takeover)
  __device__ int claim_team_receiver(bool& takeover, bool remote_ok) {
    takeover = false;
    constexpr unsigned TM = TEAM >= 32 ? ~0u : ((1u << (TEAM > 0 ? TEAM : 1)) - 1u);
    int rid = -1;
    if (lane == 0) {
      const unsigned mates = (TM << team_shift) & ~(1u << (team_shift + tw));
      unsigned bits = *(volatile unsigned*)&a.idle_bits[team_word] & mates;
      while (bits && rid < 0) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const unsigned old = atomicAnd(&a.idle_bits[team_word], ~(1u << b));
        if (old & (1u << b)) {
          rid = team_word * 32 + b;
          atomicAdd(&a.wl->state, 1ull);  // one more donation in flight
        }
      }
    }
    rid = __shfl_sync(FULLMASK, rid, 0);
    if (rid >= 0 || !remote_ok || !phase2()) return rid;
    const unsigned long long st = *(volatile unsigned long long*)&a.wl->state;
    if ((st >> 32) + 1 < (unsigned long long)TEAM + 1) return -1;  // no whole team can be idle
    const int nwords = (a.num_workers + 31) >> 5;
    const int start = (cta * 7) % nwords;
    for (int base = 0; base < nwords && rid < 0; base += 32) {
      const int wi = (start + base + lane) % nwords;
      const unsigned bits = (base + lane < nwords) ? *(volatile unsigned*)&a.idle_bits[wi] : 0u;
      unsigned full = 0;  // fully idle teams in this word (not mine)
#pragma unroll
      for (int sh = 0; sh < 32; sh += (TEAM > 0 ? TEAM : 32))
        if (((bits >> sh) & TM) == TM && !(wi == team_word && sh == team_shift)) full |= 1u << sh;
      unsigned m = __ballot_sync(FULLMASK, full != 0);
      while (m && rid < 0) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const unsigned f = __shfl_sync(FULLMASK, full, src);
        const int wordi = __shfl_sync(FULLMASK, wi, src);
        int claimed = -1;
        if (lane == 0) {
          for (unsigned t = f; t && claimed < 0; t &= t - 1) {
            const int sh = __ffs(t) - 1;
            unsigned cur = *(volatile unsigned*)&a.idle_bits[wordi];
            while (((cur >> sh) & TM) == TM) {
              const unsigned seen = atomicCAS(&a.idle_bits[wordi], cur, cur & ~(TM << sh));
              if (seen == cur) {
                claimed = wordi * 32 + sh;
                atomicAdd(&a.wl->state, 1ull);
                break;
              }
              cur = seen;
            }
          }
        }
        rid = __shfl_sync(FULLMASK, claimed, 0);
      }
    }
    takeover = rid >= 0;
    return rid;
  }

  // claim an idle worker off the worker list (-1: none parked)
  __device__ int claim_receiver() {
    int rid = -1;
    const unsigned long long st = *(volatile unsigned long long*)&a.wl->state;
    if ((st >> 32) == 0) return -1;  // nobody parked
    const int nwords = (a.num_workers + 31) >> 5;
    const int start = (wid * 7) % nwords;
    for (int base = 0; base < nwords && rid < 0; base += 32) {
      const int wi = (start + base + lane) % nwords;
      const unsigned bits = (base + lane < nwords) ? *(volatile unsigned*)&a.idle_bits[wi] : 0u;
      unsigned m = __ballot_sync(FULLMASK, bits != 0);
      while (m && rid < 0) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const unsigned wbits = __shfl_sync(FULLMASK, bits, src);
        const int wordi = __shfl_sync(FULLMASK, wi, src);
        const int b = __ffs(wbits) - 1;
        int claimed = -1;
        if (lane == 0) {
          const unsigned old = atomicAnd(&a.idle_bits[wordi], ~(1u << b));
          if (old & (1u << b)) {
            claimed = wordi * 32 + b;
            atomicAdd(&a.wl->state, 1ull);  // one more donation in flight
          }
        }
        rid = __shfl_sync(FULLMASK, claimed, 0);
      }
    }
    return __shfl_sync(FULLMASK, rid, 0);
  }

  // hand the claimed worker `rid` the branch (its X_X tokens, nxx of them,
  // are already in its xx buffer): R path, P / X_P bitsets, the root's rows
  __device__ void send_branch(int rid, const B& childP, const B& childXP, int32_t gv, int rlen,
                              int nxx, bool takeover = false) {
    Mailbox* mb = a.mbox + rid;
    uint32_t* mbits = a.mbits + (size_t)rid * 2 * W;
    int32_t* rr = a.rpath + (size_t)rid * (a.levels + 2);
    for (int i = lane; i < rlen; i += 32) rr[i] = rpath[i];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (valid(q, lane)) {
        mbits[word(q)] = childP.w[q];
        mbits[W + word(q)] = childXP.w[q];
      }
    }
    if (TEAM) {
      if (takeover) {  // the team's rows, published once per context, for the taking team
        int st = 0;
        if (lane == 0) st = atomicCAS(s_pub, 0, 1);
        st = __shfl_sync(FULLMASK, st, 0);
        if (st == 0) {
          if (lane == 0)  // the previous context's takeovers have copied their rows
            while (*(volatile unsigned*)&a.pub_refs[cta]) __nanosleep(64);
          __syncwarp();
          uint32_t* pb = a.pub + (size_t)cta * (W * CAPP + CAP);
          for (int w = 0; w < W; ++w)
            for (int c = lane; c < np; c += 32) pb[w * CAPP + c] = rowsT[w * CAPP + c];
          for (int c = lane; c < np; c += 32) pb[W * CAPP + c] = plist[c];
          __threadfence();
          __syncwarp();
          if (lane == 0) atomicExch(s_pub, 2);
        } else {
          if (lane == 0)
            while (*(volatile int*)s_pub != 2) __nanosleep(32);
          __syncwarp();
        }
        if (lane == 0) atomicAdd(&a.pub_refs[cta], 1u);
      }
    } else if (ROWS_SMEM && !published) {  // first donation from this root: publish its rows
      uint32_t* pb = a.pub + (size_t)wid * (W * CAPP + CAP);
      for (int w = 0; w < W; ++w)
        for (int c = lane; c < np; c += 32) pb[w * CAPP + c] = rowsT[w * CAPP + c];
      for (int c = lane; c < np; c += 32) pb[W * CAPP + c] = plist[c];
      published = true;
    }
    if (lane == 0) {
      rr[rlen] = gv;
      mb->origin = origin;
      mb->rlen = rlen + 1;
      mb->nxx = nxx;
      mb->owner = owner_wid;
      mb->np = np;
      mb->nx = nx;
      mb->xr = xr ? 1 : 0;
      mb->pubcta = TEAM && takeover ? cta : -1;
      mb->has_task = 1;
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicExch(&a.wl_wake[rid], 1);
    don_made++;
  }

  // park on the worker list until donated to (true) or terminated (false)
  __device__ bool park() {
    int got = 0;
    if (lane == 0) {
      WorkerListDev* wl = a.wl;
      const unsigned long long now = atomicAdd(&wl->state, 1ull << 32) + (1ull << 32);
      if ((now >> 32) == (unsigned long long)a.num_workers && (now & 0xffffffffull) == 0) {
        atomicExch(&wl->terminated, 1);  // last one in with nothing in flight
      } else {
        atomicOr(&a.idle_bits[wid >> 5], 1u << (wid & 31));
        unsigned ns = 32;
        for (;;) {
          if (*(volatile int*)&a.wl_wake[wid]) {
            got = 1;
            break;
          }
          if (*(volatile int*)&wl->terminated) break;
          __nanosleep(ns);
          ns = ns < 4096 ? ns * 2 : ns;
        }
        if (got) {
          __threadfence();
          a.wl_wake[wid] = 0;
          a.mbox[wid].has_task = 0;
          // leave the idle set and retire the in-flight donation together
          atomicAdd(&wl->state, ~0ull - (1ull << 32));  // -= (1<<32) + 1
        }
      }
    }
    got = __shfl_sync(FULLMASK, got, 0);
    __threadfence();
    return got != 0;
  }

  // teams: park until handed a branch (1) or terminated (0); a leader in
  // phase 1 (`leader_wait`) parks uncounted -- it cannot end the launch --
  // and returns 2 once every CTA-mate is parked with nothing in flight to it
  // (it has then left the idle set: the shared rows are its to rebuild)
  __device__ int park_team(bool leader_wait) {
    constexpr unsigned TM = TEAM >= 32 ? ~0u : ((1u << (TEAM > 0 ? TEAM : 1)) - 1u);
    int got = 0;
    if (lane == 0) {
      WorkerListDev* wl = a.wl;
      const unsigned me = 1u << (wid & 31);
      bool fin = false;
      if (!leader_wait) {
        const unsigned long long now = atomicAdd(&wl->state, 1ull << 32) + (1ull << 32);
        if ((now >> 32) == (unsigned long long)a.num_workers && (now & 0xffffffffull) == 0) {
          atomicExch(&wl->terminated, 1);  // last one in with nothing in flight
          fin = true;
        }
      }
      if (!fin) {
        atomicOr(&a.idle_bits[wid >> 5], me);
        const unsigned mates = (TM << team_shift) & ~me;
        unsigned ns = 32;
        for (;;) {
          if (*(volatile int*)&a.wl_wake[wid]) {
            got = 1;
            break;
          }
          if (!leader_wait && *(volatile int*)&wl->terminated) break;
          if (leader_wait && (*(volatile unsigned*)&a.idle_bits[team_word] & mates) == mates) {
            const unsigned old = atomicAnd(&a.idle_bits[team_word], ~me);
            if (old & me) {
              got = 2;
              break;
            }  // else claimed by a donor: its branch is on the way
          }
          __nanosleep(ns);
          ns = ns < 1024 ? ns * 2 : ns;
        }
        if (got == 1) {
          __threadfence();
          a.wl_wake[wid] = 0;
          a.mbox[wid].has_task = 0;
          // retire the in-flight donation (and leave the idle count when counted)
          atomicAdd(&wl->state, leader_wait ? ~0ull : ~0ull - (1ull << 32));
        }
      }
    }
    got = __shfl_sync(FULLMASK, got, 0);
    __threadfence();
    return got;
  }

  // ---------------------------------------------------------------- compact subtrees
  // Below a node whose candidate set U = P | X_P has at most CW (32 or 64)
  // members and whose live X_X prefix holds at most CW tokens, the rest of
  // the subtree runs on a re-indexed copy held in registers:
  //  * slot s = the s-th member of U in ascending local id, so the pivot's
  //    smallest-id tie-break and the ascending branch order are unchanged;
  //  * lane l holds the rows (restricted to U) of slots l and l + 32, and
  //    the rows and tokens of the live X_X members at prefix positions l and
  //    l + 32 -- the stable partition permutes them between lanes;
  //  * P, X_P, the branch and non-leaf sets are warp-uniform CW-bit masks;
  //  * the DFS frames live in lane registers (frame d in lane d & 31).
  // Pivot rule, leaf batch, X_X partition, node accounting and donation
  // conditions are traverse()'s, so the traversal tree is unchanged; a
  // branch donated from here is handed over in the wide (root-local) form.
  template <typename M>
  __device__ __forceinline__ static int popcm(M x) {
    if (sizeof(M) == 8) return __popcll((unsigned long long)x);
    return __popc((unsigned)x);
  }
  template <typename M>
  __device__ __forceinline__ static int ffsm(M x) {
    if (sizeof(M) == 8) return __ffsll((long long)x) - 1;
    return __ffs((unsigned)x) - 1;
  }
  template <typename M>
  __device__ __forceinline__ static M shflm(M x, int src) {
    if (sizeof(M) == 8) return (M)__shfl_sync(FULLMASK, (unsigned long long)x, src);
    return (M)__shfl_sync(FULLMASK, (unsigned)x, src);
  }
  template <typename M>
  __device__ __forceinline__ static M ballotm(bool p, int h) {
    return (M)((unsigned long long)__ballot_sync(FULLMASK, p) << (32 * h));
  }
  template <typename M>
  __device__ __forceinline__ static M reduce_orm(M x) {
    M r = (M)__reduce_or_sync(FULLMASK, (unsigned)x);
    if (sizeof(M) == 8)
      r |= (M)((unsigned long long)__reduce_or_sync(FULLMASK, (unsigned)((unsigned long long)x >> 32)) << 32);
    return r;
  }

  // eligible when |P | X_P| and the live X_X prefix fit CW bits and every live
  // X_X member has its row (X rows built, or none live)
  __device__ int compact_width(const B& P, const B& XP, int live) const {
    if (!a.compact || live > 64 || (live > 0 && !(XROWS && xr))) return 0;
    int c = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) c += __popc(P.w[k] | XP.w[k]);
    c = __reduce_add_sync(FULLMASK, c);
    if (c > 64) return 0;
    if (CMP_NARROW_ONLY) return (c <= 32 && live <= 32) ? 32 : 0;
    return (c <= 32 && live <= 32) ? 32 : 64;
  }

  template <typename M>
  __device__ __forceinline__ void compact_run(const B& Pw, const B& XPw, int live, int rlen, int& below,
                              uint64_t hs) {
    constexpr int H = (int)sizeof(M) / 4;  // slots per lane
    const unsigned lt = (1u << lane) - 1;
    // ---- U members (ascending local id), bit 31: member of P
    int nu = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t uw = valid(k, lane) ? (Pw.w[k] | XPw.w[k]) : 0u;
      const uint32_t pw = valid(k, lane) ? Pw.w[k] : 0u;
      const int c = __popc(uw);
      int incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(FULLMASK, incl, d);
        if (lane >= d) incl += t;
      }
      int pos = nu + incl - c;
      const int wid_ = k * 32 + lane;
      for (uint32_t t = uw; t; t &= t - 1) {
        const int b = __ffs(t) - 1;
        cu[pos++] = ((wid_ << 5) + b) | (int)(((pw >> b) & 1u) << 31);
      }
      nu += __shfl_sync(FULLMASK, incl, 31);
    }
    __syncwarp();
    const M umask = nu >= (int)(8 * sizeof(M)) ? ~(M)0 : (((M)1 << nu) - 1);
    const bool contig = (cu[nu - 1] & 0x7fffffff) == nu - 1;  // U = {0 .. nu-1}
    const int live0 = live;
    M row[H], xrow[H];
    int cid[H], tok[H];
    int32_t gvs[H];
    uint64_t vh[H];
    M P = 0;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int s = lane + 32 * h;
      const bool sv = s < nu;
      const int e = sv ? cu[s] : 0;
      cid[h] = e & 0x7fffffff;
      P |= ballotm<M>(sv && e < 0, h);
      gvs[h] = sv ? plist[cid[h]] : 0;
      vh[h] = sv ? a.vhash[gvs[h]] : 0ull;
      const int p = lane + 32 * h;
      tok[h] = p < live ? xx[p] : 0;
      row[h] = 0;
      xrow[h] = 0;
    }
    M XP = umask & ~P;
    if (contig) {  // the rows' first words are already indexed by slot
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int s = lane + 32 * h;
        const int p = lane + 32 * h;
        if (s < nu) {
          M r = (M)rowsT[cid[h]];
          if (H == 2 && W >= 2) r |= (M)((unsigned long long)rowsT[CAPP + cid[h]] << 32);
          row[h] = r & umask;
        }
        if (p < live) {
          M r = (M)xrowsT[tok[h]];
          if (H == 2 && W >= 2) r |= (M)((unsigned long long)xrowsT[(size_t)xstride + tok[h]] << 32);
          xrow[h] = r & umask;
        }
      }
    } else {  // gather bit u_t of every row word, one load per distinct word
      int curw = -1;
      uint32_t rw[H], xw[H];
#pragma unroll
      for (int h = 0; h < H; ++h) rw[h] = xw[h] = 0;
      for (int t = 0; t < nu; ++t) {
        const int u = cu[t] & 0x7fffffff;
        const int w = u >> 5;
        if (w != curw) {
          curw = w;
#pragma unroll
          for (int h = 0; h < H; ++h) {
            const int s = lane + 32 * h;
            rw[h] = s < nu ? rowsT[w * CAPP + cid[h]] : 0u;
            xw[h] = s < live ? xrowsT[(size_t)w * xstride + tok[h]] : 0u;
          }
        }
        const int b = u & 31;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          row[h] |= (M)((rw[h] >> b) & 1u) << t;
          xrow[h] |= (M)((xw[h] >> b) & 1u) << t;
        }
      }
    }
    __syncwarp();
    // ---- DFS frames in lane registers
    M fP[H], fXP[H], fBR[H], fNL[H];
    int flive[H];
    uint64_t fhs[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      fP[h] = fXP[h] = fBR[h] = fNL[h] = 0;
      flive[h] = 0;
      fhs[h] = 0;
    }
    int depth = 0;
    M BR = 0, NL = 0;
    bool fresh = true;
    for (;;) {
      if (fresh) {
        fresh = false;
        // pivot (bk.py:82-110): max |N(c) & P| over P | X_P, ties to the smallest slot
        const M cand = P | XP;
        unsigned key = 0;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int s = lane + 32 * h;
          if ((cand >> s) & 1) {
            const unsigned k2 = ((unsigned)(popcm(row[h] & P) + 1) << 7) | (unsigned)(127 - s);
            key = k2 > key ? k2 : key;
          }
        }
        const unsigned km = __reduce_max_sync(FULLMASK, key);
        const int ps = 127 - (int)(km & 127);
        M prow = shflm(H == 2 && ps >= 32 ? row[H - 1] : row[0], ps & 31);
        if (PIVOT_XX && live > 0) {  // X_X rows win only when strictly better, first in prefix order
          unsigned xk = 0;
#pragma unroll
          for (int h = 0; h < H; ++h) {
            const int p = lane + 32 * h;
            if (p < live) {
              const unsigned k2 = ((unsigned)(popcm(xrow[h] & P) + 1) << 7) | (unsigned)(127 - p);
              xk = k2 > xk ? k2 : xk;
            }
          }
          const unsigned xm = __reduce_max_sync(FULLMASK, xk);
          if ((xm >> 7) > (km >> 7)) {
            const int pp = 127 - (int)(xm & 127);
            prow = shflm(H == 2 && pp >= 32 ? xrow[H - 1] : xrow[0], pp & 31);
          }
        }
        if (a.no_pivot) prow = 0;  // basic BK: every member of P is a branch
        BR = P & ~prow;
        // leaf batch (see leaf_batch): every branch whose child P is empty
        M xxadj = 0;
        if (live > 0) {
          M o = 0;
#pragma unroll
          for (int h = 0; h < H; ++h)
            if (lane + 32 * h < live) o |= xrow[h];
          xxadj = reduce_orm(o);
        }
        const int size = rlen + 1;
        M leafm = 0, maxm = 0;
        unsigned long long hl = 0;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int s = lane + 32 * h;
          bool leaf = false, xcl = false;
          if ((BR >> s) & 1) {
            const M before = BR & (((M)1 << s) - 1);
            leaf = (row[h] & (P & ~before)) == 0;
            xcl = leaf && (row[h] & (XP | before)) == 0 && !((xxadj >> s) & 1);
          }
          leafm |= ballotm<M>(leaf, h);
          maxm |= ballotm<M>(xcl, h);
          if (xcl) hl += mce_mix64(hs + vh[h] + (uint64_t)size * MCE_SIZE_SALT);
        }
        nodes += popcm(leafm);
        NL = BR & ~leafm;
        if (maxm) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) hl += __shfl_xor_sync(FULLMASK, hl, o);
          const int cnt = popcm(maxm);
          if (lane == 0) {
            cliques += cnt;
            hash += hl;
            if ((unsigned long long)size > max_size) max_size = size;
            hist_add(size, (unsigned)cnt);
          }
          if (a.collect_cap > 0) {
            for (M t = maxm; t; t &= t - 1) {
              const int sv = ffsm(t);
              collect_clique(size, __shfl_sync(FULLMASK, H == 2 && sv >= 32 ? gvs[H - 1] : gvs[0], sv & 31));
            }
          }
        }
      }
      const int v = NL ? ffsm(NL) : -1;
      if (v < 0) {
        if (depth == 0) break;
        depth--;
        rlen--;
        const int fl = depth & 31, fh = depth >> 5;
        P = shflm(H == 2 && fh ? fP[H - 1] : fP[0], fl);
        XP = shflm(H == 2 && fh ? fXP[H - 1] : fXP[0], fl);
        BR = shflm(H == 2 && fh ? fBR[H - 1] : fBR[0], fl);
        NL = shflm(H == 2 && fh ? fNL[H - 1] : fNL[0], fl);
        live = __shfl_sync(FULLMASK, H == 2 && fh ? flive[H - 1] : flive[0], fl);
        hs = __shfl_sync(FULLMASK, H == 2 && fh ? fhs[H - 1] : fhs[0], fl);
        if (NL) below--;
        continue;
      }
      // move v and the (leaf) branches before it from P to X_P
      const M bit = (M)1 << v;
      const M mv = (BR & (bit - 1)) | bit;
      BR &= ~mv;
      NL &= ~mv;
      P &= ~mv;
      XP |= mv;
      const int vl = v & 31;
      const bool vh2 = H == 2 && v >= 32;
      const M rowv = shflm(vh2 ? row[H - 1] : row[0], vl);
      const M childP = P & rowv;
      const int32_t gv = __shfl_sync(FULLMASK, vh2 ? gvs[H - 1] : gvs[0], vl);
      const uint64_t vhv = __shfl_sync(FULLMASK, vh2 ? vh[H - 1] : vh[0], vl);
      if (a.worker_list_on && (popcm(childP) >= a.min_p || (a.min_x > 0 && live >= a.min_x)) &&
          below > 0 && NL != 0 && (TEAM > 0 || phase2())) {
        if (donate_compact<M, H>(childP, XP & rowv, v, gv, live, rlen, cid, nu, xrow, tok)) continue;
      }
      // stable partition of the live X_X prefix by adjacency to v (xsets.py:55-82)
      int kept = 0;
      if (live > 0) {
        unsigned kb[H], db[H];
        bool keep[H], ok[H];
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int p = lane + 32 * h;
          ok[h] = p < live;
          keep[h] = ok[h] && ((xrow[h] >> v) & 1);
          kb[h] = __ballot_sync(FULLMASK, keep[h]);
          db[h] = __ballot_sync(FULLMASK, ok[h] && !keep[h]);
          kept += __popc(kb[h]);
        }
        int kbase = 0, dbase = kept;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          int dst = -1;
          if (keep[h]) dst = kbase + __popc(kb[h] & lt);
          else if (ok[h]) dst = dbase + __popc(db[h] & lt);
          kbase += __popc(kb[h]);
          dbase += __popc(db[h]);
          if (dst >= 0) {
            cbuf_as<M>()[dst] = xrow[h];
            ctok[dst] = tok[h];
          }
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int p = lane + 32 * h;
          if (p < live) {
            xrow[h] = cbuf_as<M>()[p];
            tok[h] = ctok[p];
          }
        }
        __syncwarp();
      }
      {  // push the frame of this level
        const int fl = depth & 31, fh = depth >> 5;
        if (lane == fl) {
#pragma unroll
          for (int h = 0; h < H; ++h) {
            if (h == fh) {
              fP[h] = P;
              fXP[h] = XP;
              fBR[h] = BR;
              fNL[h] = NL;
              flive[h] = live;
              fhs[h] = hs;
            }
          }
        }
      }
      if (NL) below++;
      depth++;
      live = kept;
      XP &= rowv;
      P = childP;
      if (lane == 0) rpath[rlen] = gv;
      hs += vhv;
      rlen++;
      nodes++;
      fresh = true;
    }
    // the X_X prefix order this subtree left behind (the reference partitions
    // in place and never restores: the enclosing levels see it)
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int p = lane + 32 * h;
      if (p < live0) xx[p] = tok[h];
    }
    __syncwarp();
  }

  template <typename M>
  __device__ __forceinline__ M* cbuf_as() const { return reinterpret_cast<M*>(cbuf); }

  // hand the compact branch (childP, childXP over slots) to an idle worker
  // in the wide form: slots mapped back to root-local ids, the live X_X
  // tokens adjacent to v in the current prefix order
  template <typename M, int H>
  __device__ __forceinline__ bool donate_compact(M childP, M childXP, int v, int32_t gv, int live, int rlen,
                                 const int (&cid)[H], int nu, const M (&xrow)[H],
                                 const int (&tok)[H]) {
    const unsigned long long st = *(volatile unsigned long long*)&a.wl->state;
    if ((st >> 32) == 0) return false;  // nobody parked: skip the expansion
    for (int i = lane; i < W; i += 32) {
      sP[i] = 0;
      sXP[i] = 0;
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int s = lane + 32 * h;
      if (s < nu) {
        const int u = cid[h];
        if ((childP >> s) & 1) atomicOr(&sP[u >> 5], 1u << (u & 31));
        if ((childXP >> s) & 1) atomicOr(&sXP[u >> 5], 1u << (u & 31));
      }
    }
    __syncwarp();
    B cP, cXP;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      cP.w[k] = valid(k, lane) ? sP[word(k)] : 0u;
      cXP.w[k] = valid(k, lane) ? sXP[word(k)] : 0u;
    }
    __syncwarp();
    bool takeover = false;
    const int rid = TEAM ? claim_team_receiver(takeover, popcm(childP) >= TEAM_REMOTE_MIN_P)
                         : claim_receiver();
    if (rid < 0) return false;
    int32_t* rx = a.xx + (size_t)rid * a.xcap;
    const unsigned lt = (1u << lane) - 1;
    int k = 0;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int p = lane + 32 * h;
      const bool keep = p < live && ((xrow[h] >> v) & 1);
      const unsigned km = __ballot_sync(FULLMASK, keep);
      if (keep) rx[k + __popc(km & lt)] = tok[h];
      k += __popc(km);
    }
    send_branch(rid, cP, cXP, gv, rlen, k, takeover);
    return true;
  }

  // ---------------------------------------------------------------- DFS
  // frame: P, X_P, remaining branches BR, remaining non-leaf branches NL
  __device__ __forceinline__ void push(int depth, const B& P, const B& XP, const B& BR,
                                       const B& NL) {
    uint32_t* f = stk + (size_t)depth * 4 * W;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (valid(k, lane)) {
        f[word(k)] = P.w[k];
        f[W + word(k)] = XP.w[k];
        f[2 * W + word(k)] = BR.w[k];
        f[3 * W + word(k)] = NL.w[k];
      }
    }
  }
  __device__ __forceinline__ void pop(int depth, B& P, B& XP, B& BR, B& NL) const {
    const uint32_t* f = stk + (size_t)depth * 4 * W;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      P.w[k] = valid(k, lane) ? f[word(k)] : 0u;
      XP.w[k] = valid(k, lane) ? f[W + word(k)] : 0u;
      BR.w[k] = valid(k, lane) ? f[2 * W + word(k)] : 0u;
      NL.w[k] = valid(k, lane) ? f[3 * W + word(k)] : 0u;
    }
  }

  // Traverse from the level-0 state (P, XP, xx[0, nxx), rpath[0, rlen)).
  // Leaves are settled per node by leaf_batch; the loop walks the non-leaf
  // branches in the reference's order, applying the P -> X_P moves of the
  // leaf branches that precede each one.
  __device__ __forceinline__ void traverse(B P, B XP, int nxx, int rlen, bool root_sorted) {
    uint64_t hs = 0;
    for (int i = 0; i < rlen; ++i) hs += a.vhash[rpath[i]];
    if (!any(P)) {  // scheduler.py:300-304
      nodes++;
      if (!any(XP) && nxx == 0) report(rlen, hs);
      return;
    }
    int depth = 0;
    int below = 0;  // frozen frames with (non-leaf) branches left (scheduler.py:346-348)
    if (lane == 0) {
      lpx[0] = nxx;
      hsum[rlen] = hs;
    }
    __syncwarp();
    int live = nxx;
    nodes++;
    B BR, NL;
    bool fresh = true;  // a node just entered: pivot + leaf batch (one call site each)
    // bit d: the live X_X prefix at depth d is ascending (see xx_any_adjacent)
    unsigned long long xsorted = root_sorted ? 1ull : 0ull;
    for (;;) {
      if (fresh) {
        const int cw = compact_width(P, XP, live);
        if (cw) {  // the whole subtree below this node, on the register copy
          const long long t0 = tic();
          const uint64_t hs0 = hsum[rlen];
          if (cw == 32 || CMP_NARROW_ONLY) compact_run<uint32_t>(P, XP, live, rlen, below, hs0);
          else compact_run<unsigned long long>(P, XP, live, rlen, below, hs0);
#pragma unroll
          for (int k = 0; k < K; ++k) NL.w[k] = 0;
          toc(T_SETOPS, t0);
        } else {
          long long t0 = tic();
          pivot_branches(P, XP, live, BR);
          toc(T_PIVOT, t0);
          t0 = tic();
          leaf_batch(P, XP, BR, live, rlen, NL, depth < 64 && ((xsorted >> depth) & 1ull));
          toc(T_SETOPS, t0);
        }
        fresh = false;
      }
      const int v = first(NL);
      if (v < 0) {
        if (depth == 0) break;
        depth--;
        rlen--;
        pop(depth, P, XP, BR, NL);
        if (any(NL)) below--;
        live = lpx[depth];
        continue;
      }
      {
        // move v and the (leaf) branches before it from P to X_P
        const int wv = v >> 5;
        const uint32_t bit = 1u << (v & 31);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int wd = word(k);
          const uint32_t below_m = wd < wv ? 0xffffffffu : (wd == wv ? bit - 1u : 0u);
          const uint32_t m = (BR.w[k] & below_m) | (wd == wv ? bit : 0u);
          BR.w[k] &= ~m;
          NL.w[k] &= ~m;
          P.w[k] &= ~m;
          XP.w[k] |= m;
        }
      }
      B rowv, childP;
      row_of(v, rowv);
#pragma unroll
      for (int k = 0; k < K; ++k) childP.w[k] = P.w[k] & rowv.w[k];
      const int cpop = popc(childP);
      const int32_t gv = plist[v];
      if (a.worker_list_on && (cpop >= a.min_p || (a.min_x > 0 && live >= a.min_x)) &&
          below > 0 && any(NL) && (TEAM > 0 || phase2())) {
        B cxp;
#pragma unroll
        for (int k = 0; k < K; ++k) cxp.w[k] = XP.w[k] & rowv.w[k];
        const long long t0 = tic();
        const bool gave = try_donate(childP, cxp, v, gv, live, rlen);
        toc(T_WLIST, t0);
        if (gave) continue;
      }
      if (cpop == 0) {  // not reached: leaf_batch settled every leaf branch
        nodes++;
        uint32_t o = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) o |= XP.w[k] & rowv.w[k];
        bool hit = __any_sync(FULLMASK, o != 0);
        if (!hit) hit = xx_any_adjacent(v, gv, live);
        if (!hit) {
          if (lane == 0) rpath[rlen] = gv;
          __syncwarp();
          report(rlen + 1, hsum[rlen] + a.vhash[gv]);
        }
        continue;
      }
      const long long tp = tic();
      const int kept = partition(v, gv, live);
      toc(T_SETOPS, tp);
      if (depth < 63) {  // the kept part inherits the order; the parent's prefix is permuted
        const unsigned long long bit = (xsorted >> depth) & 1ull;
        xsorted &= ~(3ull << depth);
        xsorted |= bit << (depth + 1);
      } else {
        xsorted = 0;
      }
      push(depth, P, XP, BR, NL);
      if (any(NL)) below++;
      depth++;
      live = kept;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        XP.w[k] &= rowv.w[k];
        P.w[k] = childP.w[k];
      }
      if (lane == 0) {
        lpx[depth] = kept;
        rpath[rlen] = gv;
        hsum[rlen + 1] = hsum[rlen] + a.vhash[gv];
      }
      rlen++;
      nodes++;
      __syncwarp();
      fresh = true;
    }
  }

  // The root's X_X token list.  With X rows, members with no neighbour in P
  // are left out: every branch adds a P vertex to R, so such an x is dropped
  // by the first partition anyway, is never adjacent to a branch vertex
  // (leaf maximality) and never wins the pivot (a zero count is never
  // strictly better) -- the traversal and the node count are unchanged.
  // The kept tokens stay ascending.
  __device__ int init_tokens() {
    if (!(XROWS && xr)) {
      for (int t = lane; t < nx; t += 32) xx[t] = t;
      __syncwarp();
      return nx;
    }
    constexpr int U = 4;
    const unsigned lt = (1u << lane) - 1;
    int kept = 0;
    for (int base = 0; base < nx; base += 32 * U) {
      bool nz[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = base + u * 32 + lane;
        uint32_t o = 0;
        if (t < nx)
          for (int w = 0; w < W; ++w) o |= xrowsT[(size_t)w * xstride + t];
        nz[u] = o != 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned m = __ballot_sync(FULLMASK, nz[u]);
        if (nz[u]) xx[kept + __popc(m & lt)] = base + u * 32 + lane;
        kept += __popc(m);
      }
    }
    __syncwarp();
    return kept;
  }

  // level-0 state of root r (build its induced rows first); returns the R length
  __device__ int prepare_root(int64_t r, B& P, B& XP, int& nxx) {
    const int nr = build(r);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      uint32_t x = 0;
      if (valid(k, lane)) {
        const int lo = word(k) * 32;
        if (np >= lo + 32) x = 0xffffffffu;
        else if (np > lo) x = (1u << (np - lo)) - 1u;
      }
      P.w[k] = x;
      XP.w[k] = 0u;
    }
    nxx = init_tokens();
    return nr;
  }

  // Take over the root of a donated branch from its owner's buffers (no
  // CSR walks): rows and plist (shared-memory classes copy the owner's
  // published copy into their own shared memory), X rows in place.
  __device__ void adopt(const Mailbox* mb, int64_t r_enc) {
    const int owner = mb->owner;
    np = mb->np;
    nx = mb->nx;
    xr = mb->xr != 0;
    origin = r_enc;
    owner_wid = owner;
    published = true;
    const int64_t r = a.roots_mode == 1 ? (r_enc & ROOT_ID_MASK) : r_enc;
    const int heavy = a.roots_mode == 1 ? (int)(r_enc >> ROOT_ID_BITS) : 0;
    root_x = a.roots_mode == 1 ? a.col + a.ro[r] : a.xlist + (size_t)owner * a.xcap;
    if (TEAM && mb->pubcta < 0) {
      // a CTA-mate's branch: the rows are this team's shared rows already
    } else if (ROWS_SMEM) {
      // only the rows of the branch's candidates (P | X_P) are ever read below
      // this node: copy those (lane per candidate), and the member list
      const int src = TEAM ? mb->pubcta : owner;
      const uint32_t* pb = a.pub + (size_t)src * (W * CAPP + CAP);
      const uint32_t* mbits = a.mbits + (size_t)wid * 2 * W;
      for (int k = 0; k < W; ++k) {
        const uint32_t cw = mbits[k] | mbits[W + k];  // broadcast read
        if ((cw >> lane) & 1u) {
          const int c = k * 32 + lane;
          for (int w = 0; w < W; ++w) rowsT[w * CAPP + c] = pb[w * CAPP + c];
        }
      }
      for (int c = lane; c < np; c += 32) plist[c] = (int32_t)pb[W * CAPP + c];
      if (TEAM) {  // a takeover: this team's shared rows now hold the branch
        constexpr unsigned TM = TEAM >= 32 ? ~0u : ((1u << (TEAM > 0 ? TEAM : 1)) - 1u);
        __threadfence();
        __syncwarp();
        if (lane == 0) {
          atomicSub(&a.pub_refs[src], 1u);
          *s_pub = 0;  // a new context: its rows are not published yet
          // the CTA-mates (parked, their bits taken by the takeover) receive again
          atomicOr(&a.idle_bits[team_word], (TM << team_shift) & ~(1u << (wid & 31)));
        }
      }
    } else {
      rowsT = a.rows_g + (size_t)owner * W * CAPP;
      plist = a.plist_g + (size_t)owner * CAP;
    }
    if (XROWS && xr) {
      if (heavy > 0) {
        xrowsT = const_cast<uint32_t*>(a.heavy_rows) + a.heavy_off[heavy - 1];
        xstride = nx;
      } else {
        xrowsT = a.xrows + (size_t)owner * W * a.xcap;
        xstride = a.xcap;
      }
    }
    __syncwarp();
  }

  // level-0 state of the branch donated to this worker; returns the R length
  __device__ int prepare_donated(B& P, B& XP, int& nxx) {
    const Mailbox* mb = a.mbox + wid;
    const uint32_t* mbits = a.mbits + (size_t)wid * 2 * W;
    const int64_t r = mb->origin;
    const int rlen = mb->rlen;
    nxx = mb->nxx;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      P.w[k] = valid(k, lane) ? mbits[word(k)] : 0u;
      XP.w[k] = valid(k, lane) ? mbits[W + word(k)] : 0u;
    }
    adopt(mb, r);
    return rlen;
  }
};

// Resident CTAs per SM the compiler must allow for (register budget).  The
// narrow classes are latency-bound on dependent CSR loads: more resident
// warps hide more of it.
#ifndef MCE_MINB_SMALL
#define MCE_MINB_SMALL 4
#endif
// The wide classes are latency-bound with few warps per SM (register-limited
// at ~210 registers): capping them buys residency.  Measured on rmat20's
// core: the W = 32 class on one dense root 20.8 s (2 CTAs of 4 warps per SM)
// -> 15.5 s (3 CTAs, 167 registers); W = 8 / 16 chunk 935 -> 888 ms.
#ifndef MCE_MINB_W8
#define MCE_MINB_W8 4
#endif
#ifndef MCE_MINB_W16
#define MCE_MINB_W16 6
#endif
#ifndef MCE_MINB_W32
#define MCE_MINB_W32 3
#endif
template <int W>
struct MinBlocks {
  static constexpr int value = W <= 4 ? MCE_MINB_SMALL
                               : W == 8 ? MCE_MINB_W8
                               : W == 16 ? MCE_MINB_W16
                               : W == 32 ? MCE_MINB_W32 : 1;
};

// teams (T > 0) hold one shared copy of the rows per CTA; their residency is
// bounded by shared memory (W = 32: 135 KB) or registers
template <int W, int TEAM>
struct MinBlocksT {
  static constexpr int value = TEAM == 0 ? MinBlocks<W>::value : (W >= 32 ? 1 : 3);
};

template <int W, bool PIVOT_XX, bool XROWS, bool ROWS_SMEM, int WARPS, int TEAM = 0>
__global__ void __launch_bounds__(WARPS * 32, MinBlocksT<W, TEAM>::value) k_enumerate(EnumArgs a) {
  static_assert(TEAM == 0 || (TEAM == WARPS && 32 % (TEAM > 0 ? TEAM : 1) == 0 && ROWS_SMEM),
                "team = one CTA");
  constexpr int CAP = 32 * W;
  constexpr int CAPP = CAP + 1;
  constexpr int SPW = W < 32 ? 32 : W;  // sP words per warp
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned int* s_hist = reinterpret_cast<unsigned int*>(smem);
  uint32_t* s_p = reinterpret_cast<uint32_t*>(s_hist + HIST_SMEM);
  int32_t* s_cmp = reinterpret_cast<int32_t*>(s_p + 3 * WARPS * SPW);  // CMP_WORDS per warp
  uint32_t* s_rows = reinterpret_cast<uint32_t*>(s_cmp + WARPS * CMP_WORDS);
  constexpr int RCOPIES = TEAM ? 1 : WARPS;  // row copies in shared memory
  int32_t* s_plist = reinterpret_cast<int32_t*>(s_rows + (ROWS_SMEM ? RCOPIES * W * CAPP : 0));
  __shared__ int s_pubstate;  // teams: the shared rows' publication state
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < HIST_SMEM; i += blockDim.x) s_hist[i] = 0;
  if (threadIdx.x == 0) s_pubstate = 0;
  __syncthreads();
  const int wid = blockIdx.x * WARPS + warp;
  if (wid < a.num_workers) {
    const int rc = TEAM ? 0 : warp;
    Worker<W, PIVOT_XX, XROWS, ROWS_SMEM, TEAM> wk(a, lane, wid, s_rows + (ROWS_SMEM ? rc * W * CAPP : 0),
                                  s_plist + (ROWS_SMEM ? rc * CAP : 0), s_p + 3 * warp * SPW,
                                  s_hist, s_cmp + warp * CMP_WORDS);
    wk.s_pub = &s_pubstate;
    int stripe = wid % ROOT_STRIPES;
    bool phase1 = TEAM ? warp == 0 : true;  // a team's warp 0 claims and builds its roots
    const long long t_start = clock64();
    // launch phase times with few same-address atomics: the start by one thread,
    // the first root-list miss and the last end only while they can still move
    if (a.phase_ns && blockIdx.x == 0 && threadIdx.x == 0) atomicMax(&a.phase_ns[0], ~gtimer());
    // one traverse() call site (inlined once): phase 1 claims independent
    // subtrees (scheduler.py:253-273), phase 2 parks on the worker list and
    // receives donated branches
    for (;;) {
      Bits<W> P, XP;
      int nxx = 0, rlen = 0;
      int64_t idx = -1;
      bool from_root = false;
      if (TEAM) {
        long long t0 = wk.tic();
        // phase 1 (warp 0): wait for the team to go idle -- taking CTA-mates'
        // branches meanwhile -- then claim and build the next root
        const int r = wk.park_team(phase1);
        wk.toc(T_WLIST, t0);
        if (r == 0) break;
        if (r == 2) {
          t0 = wk.tic();
          idx = wk.claim_root(stripe);
          wk.toc(T_WLIST, t0);
          if (idx < 0) {
            phase1 = false;
            if (a.phase_ns && lane == 0 && !*(volatile unsigned long long*)&a.phase_ns[1])
              atomicMax(&a.phase_ns[1], ~gtimer());
            continue;
          }
          wk.roots_claimed++;
          if (lane == 0) s_pubstate = 0;  // a new context in the shared rows
          __syncwarp();
          t0 = wk.tic();
          rlen = wk.prepare_root(a.roots[idx], P, XP, nxx);
          wk.toc(T_BUILD, t0);
          from_root = true;
        } else {
          wk.don_recv++;
          t0 = wk.tic();
          rlen = wk.prepare_donated(P, XP, nxx);
          wk.toc(T_BUILD, t0);
        }
      } else if (phase1) {
        from_root = true;
        long long t0 = wk.tic();
        idx = wk.claim_root(stripe);
        wk.toc(T_WLIST, t0);
        if (idx < 0) {
          phase1 = false;
          if (a.phase_ns && lane == 0 && !*(volatile unsigned long long*)&a.phase_ns[1])
            atomicMax(&a.phase_ns[1], ~gtimer());
          if (!a.worker_list_on) break;
          continue;
        }
        wk.roots_claimed++;
        t0 = wk.tic();
        rlen = wk.prepare_root(a.roots[idx], P, XP, nxx);
        wk.toc(T_BUILD, t0);
      } else {
        long long t0 = wk.tic();
        const bool got = wk.park();
        wk.toc(T_WLIST, t0);
        if (!got) break;
        wk.don_recv++;
        t0 = wk.tic();
        rlen = wk.prepare_donated(P, XP, nxx);
        wk.toc(T_BUILD, t0);
      }
      const long long t0 = a.root_cycles ? clock64() : 0;
      wk.traverse(P, XP, nxx, rlen, from_root);
      if (from_root && a.root_cycles && lane == 0) a.root_cycles[idx] = clock64() - t0;
    }
    if (lane == 0) {
      atomicAdd(&a.g_acc[0], wk.cliques);
      atomicAdd(&a.g_acc[1], wk.hash);
      atomicAdd(&a.g_acc[2], (unsigned long long)wk.nodes);
      atomicAdd(&a.g_acc[3], (unsigned long long)wk.don_made);
      atomicMax(&a.g_acc[4], wk.max_size);
      long long* m = a.w_metrics + (size_t)wid * WM;
      m[0] += wk.nodes;
      m[1] += wk.roots_claimed;
      m[2] += wk.don_made;
      m[3] += wk.don_recv;
      if (a.timing) m[T_TOTAL] += clock64() - t_start;
      if (a.phase_ns) {
        const unsigned long long t = gtimer();
        if (t > *(volatile unsigned long long*)&a.phase_ns[2]) atomicMax(&a.phase_ns[2], t);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HIST_SMEM; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&a.g_hist[i], (unsigned long long)s_hist[i]);
}

#include "mce_tiny.cuh"

// ------------------------------------------------------------ root prep

// Root keys: class (bitset width) in the top byte, then heaviest-first by an
// estimated subtree cost.  l1 roots: |P| = |N+(v)|, |X| = |N-(v)|; l2 roots
// (edges u < v): bounded by |N+(v)| and |N-(v)|.
constexpr int NUM_WIDTHS = 8;
constexpr int TRIVIAL_RANK = NUM_WIDTHS;       // first-level roots with P empty
constexpr int MAXP_SLOT = NUM_WIDTHS + 1;      // classes[] slot holding max |P|
constexpr int MAX_CAPACITY_BITS = 32 * 128;    // widest instantiated bitset
__device__ __forceinline__ int width_rank(int64_t p) {
  if (p > 2048) return 0;  // W = 128
  if (p > 1024) return 1;  // 64
  if (p > 512) return 2;   // 32
  if (p > 256) return 3;   // 16
  if (p > 128) return 4;   // 8
  if (p > 64) return 5;    // 4
  if (p > 32) return 6;    // 2
  return 7;                // 1
}

struct HeavyPlan {
  int enabled;
  unsigned long long pool_cap;      // words
  unsigned long long* meta;         // 0 slots taken, 1 pool words reserved, 2 pre-pass CTAs
  int64_t* vertex;                  // HEAVY_MAX
  int64_t* off;                     // HEAVY_MAX: word offset of the slot's rows
  int64_t* unit0;                   // HEAVY_MAX: first pre-pass CTA of the slot
  int* unit_slot;                   // HEAVY_UNITS_MAX: CTA -> slot
};

// X rows of the heavy-X first-level roots, HEAVY_UNIT_X members per CTA:
// rows[(j >> 5) * |X| + t] bit j <=> X member t is adjacent to P member j,
// i.e. P_j in N+(x_t) (x_t < v < P_j) -- induced.py:95-103, the same rows the
// per-warp build makes, over the whole grid.  P is staged in shared memory;
// each warp walks the N+ lists of 32 members flattened over its lanes.
__global__ void __launch_bounds__(256) k_heavy_xrows(HeavyPlan hp, const int64_t* __restrict__ ro,
                                                     const int64_t* __restrict__ split,
                                                     const int32_t* __restrict__ col,
                                                     uint32_t* __restrict__ pool) {
  __shared__ int32_t sP[MAX_CAPACITY_BITS];
  const int slot = hp.unit_slot[blockIdx.x];
  const int64_t v = hp.vertex[slot];
  const int64_t ps = split[v], xs = ro[v];
  const int np = (int)(ro[v + 1] - ps);
  const int nx = (int)(ps - xs);
  for (int i = threadIdx.x; i < np; i += blockDim.x) sP[i] = col[ps + i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int t0 = (int)((blockIdx.x - hp.unit0[slot]) * HEAVY_UNIT_X) + (threadIdx.x >> 5) * 32;
  if (t0 >= nx) return;
  const int cnt = min(32, nx - t0);
  uint32_t* rows = pool + hp.off[slot];
  const int32_t pmin = sP[0], pmax = sP[np - 1];
  warp_flat_walk(
      col, lane, cnt,
      [&](int i, int64_t& lo, int& len) {
        const int32_t x = col[xs + t0 + i];
        lo = split[x];
        len = (int)(ro[x + 1] - lo);
      },
      [&](int i, int32_t y) {
        if (y < pmin || y > pmax) return;
        int lo = 0, hi = np;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (sP[mid] < y) lo = mid + 1; else hi = mid;
        }
        if (lo < np && sP[lo] == y)
          atomicOr(&rows[(size_t)(lo >> 5) * nx + t0 + i], 1u << (lo & 31));
      });
}

__global__ void k_root_keys(const int64_t* __restrict__ ro, const int64_t* __restrict__ split,
                            const int32_t* __restrict__ col, const int64_t* __restrict__ eoff,
                            int64_t n, int roots_mode, int64_t begin, int64_t stride,
                            int64_t count, uint32_t* __restrict__ keys,
                            int64_t* __restrict__ roots, unsigned long long* __restrict__ classes,
                            unsigned long long* __restrict__ max_p, HeavyPlan hp) {
  __shared__ unsigned int s_cls[TRIVIAL_RANK + 1];
  if (threadIdx.x <= TRIVIAL_RANK) s_cls[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long local_max = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = begin + i * stride;
    int64_t p, x;
    if (roots_mode == 1) {
      p = ro[r + 1] - split[r];
      x = split[r] - ro[r];
      roots[i] = r;
    } else {
      int64_t lo = 0, hi = n;  // largest u with eoff[u] <= r
      while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (eoff[mid] <= r) lo = mid; else hi = mid;
      }
      const int64_t u = lo;
      const int64_t v = col[split[u] + (r - eoff[u])];
      p = ro[v + 1] - split[v];
      x = split[v] - ro[v];
      roots[i] = (u << 32) | v;
    }
    const int rank = (roots_mode == 1 && p == 0) ? TRIVIAL_RANK : width_rank(p);
    if (hp.enabled && roots_mode == 1 && p > 0 && p <= MAX_CAPACITY_BITS && x >= HEAVY_X_MIN) {
      // reserve a slot, pool words (|X| x W) and pre-pass CTAs for this root
      const unsigned long long slot = atomicAdd(&hp.meta[0], 1ull);
      if (slot < HEAVY_MAX) {
        const unsigned long long words = (unsigned long long)x * (1ull << (NUM_WIDTHS - 1 - rank));
        const unsigned long long off = atomicAdd(&hp.meta[1], words);
        const unsigned long long units = (x + HEAVY_UNIT_X - 1) / HEAVY_UNIT_X;
        if (off + words <= hp.pool_cap) {
          // advance the pre-pass CTA count only when the reservation fits, so
          // every CTA the host launches (meta[2]) has a written unit_slot
          unsigned long long u0 = *(volatile unsigned long long*)&hp.meta[2];
          for (;;) {
            if (u0 + units > HEAVY_UNITS_MAX) break;
            const unsigned long long seen = atomicCAS(&hp.meta[2], u0, u0 + units);
            if (seen == u0) break;
            u0 = seen;
          }
          if (u0 + units <= HEAVY_UNITS_MAX) {
            hp.vertex[slot] = r;
            hp.off[slot] = (int64_t)off;
            hp.unit0[slot] = (int64_t)u0;
            for (unsigned long long q = 0; q < units; ++q) hp.unit_slot[u0 + q] = (int)slot;
            roots[i] = r | ((int64_t)(slot + 1) << ROOT_ID_BITS);
          }
        }
      }
    }
    // 24-bit key: class in the top 4 bits, then the cost estimate descending
    // as the top 20 bits of its float encoding (monotonic for positive
    // floats: 8 exponent + 12 mantissa bits) -- a 3-pass radix sort
    const float cost = (float)(p + 1) * (float)(p + 1) + (float)(p + 1) * (float)x * 0.125f;
    const uint32_t cb = __float_as_uint(cost) >> 11;
    keys[i] = ((uint32_t)rank << 20) | (0xFFFFFu - (cb & 0xFFFFFu));
    // warp-aggregated: one shared atomic per distinct class in the warp
    const unsigned peers = __match_any_sync(__activemask(), rank);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&s_cls[rank], (unsigned)__popc(peers));
    if ((unsigned long long)p > local_max) local_max = p;
  }
  __syncthreads();
  if (threadIdx.x <= TRIVIAL_RANK && s_cls[threadIdx.x])
    atomicAdd(&classes[threadIdx.x], (unsigned long long)s_cls[threadIdx.x]);
  // one atomic per warp, not per thread (a contended address serialises in L2)
  local_max = __reduce_max_sync(FULLMASK, (unsigned)min(local_max, 0xffffffffull));
  if ((threadIdx.x & 31) == 0 && local_max) atomicMax(max_p, local_max);
}

// Algorithmic bytes one root's induced-subgraph build must read from the CSR:
// its own offsets and adjacency, then for every P member a (and, with X rows,
// every X member x) two offsets plus N+(a) (N+(x)).  out[0] = P part, out[1] = X part.
__global__ void k_build_bytes(const int64_t* __restrict__ roots, int64_t count,
                              const int64_t* __restrict__ ro, const int64_t* __restrict__ split,
                              const int32_t* __restrict__ col, int with_x,
                              unsigned long long* __restrict__ out) {
  unsigned long long bp = 0;
  const int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < count; i += nwarps) {
    const int64_t r = roots[i] & ROOT_ID_MASK;
    const int64_t lo = ro[r], sp = split[r], hi = ro[r + 1];
    if (lane == 0) bp += 24 + 4 * (hi - lo);
    for (int64_t e = sp + lane; e < hi; e += 32) {
      const int32_t a = col[e];
      bp += 16 + 4 * (ro[a + 1] - split[a]);
    }
    if (with_x) {
      for (int64_t e = lo + lane; e < sp; e += 32) {
        const int32_t x = col[e];
        bp += 16 + 4 * (ro[x + 1] - split[x]);
      }
    }
  }
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage t0;
  bp = BR(t0).Sum(bp);
  if (threadIdx.x == 0) atomicAdd(out, bp);
}

__global__ void k_later_count(const int64_t* __restrict__ ro, const int64_t* __restrict__ split,
                              int64_t n, int64_t* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    out[v] = ro[v + 1] - split[v];
}

// up_col[up_off[v] ..] = N+(v).  A warp packs 32 consecutive rows: their
// destinations are one contiguous range, written coalesced, each entry's
// source row found by a 5-step shuffle search over the rows' offsets
__global__ void k_pack_upper(const int64_t* __restrict__ ro, const int64_t* __restrict__ split,
                             const int32_t* __restrict__ col, const int64_t* __restrict__ up_off,
                             int64_t n, int32_t* __restrict__ up_col) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 32; v0 < n;
       v0 += nw * 32) {
    const int64_t v = v0 + lane;
    const int64_t src = v < n ? split[v] : 0;
    const int64_t o = v < n ? up_off[v] : INT64_MAX;
    const int64_t obeg = __shfl_sync(0xffffffffu, o, 0);
    const int64_t oend = up_off[v0 + 32 < n ? v0 + 32 : n];
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
        val[u] = j < oend ? __ldcs(&col[sr + (j - orr)]) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (base + 32 * u + lane < oend) up_col[base + 32 * u + lane] = val[u];
    }
  }
}

__global__ void k_vhash(const int64_t* __restrict__ labels, int64_t n, uint64_t* __restrict__ vh) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    vh[v] = mce_mix64((uint64_t)(labels ? labels[v] : v));
}

// first-level roots with P empty (scheduler.py:300-304) and, for second-level
// runs, isolated vertices (scheduler.py:476-480): one node / one singleton each
__global__ void k_trivial_roots(const int64_t* __restrict__ roots, int64_t count,
                                const int64_t* __restrict__ ro, const int64_t* __restrict__ split,
                                const uint64_t* __restrict__ vhash,
                                unsigned long long* __restrict__ acc,
                                unsigned long long* __restrict__ hist, int64_t* collect,
                                int64_t collect_cap, unsigned long long* collect_len) {
  unsigned long long c = 0, h = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = roots[i] & ROOT_ID_MASK;
    if (ro[v + 1] == ro[v]) {
      c++;
      h += mce_mix64(vhash[v] + MCE_SIZE_SALT);
      if (collect_cap > 0) {
        unsigned long long pos = atomicAdd(collect_len, 2ull);
        if (pos + 2 <= (unsigned long long)collect_cap) {
          collect[pos] = 1;
          collect[pos + 1] = v;
        }
      }
    }
  }
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage t1, t2;
  unsigned long long cs = BR(t1).Sum(c);
  unsigned long long hsum = BR(t2).Sum(h);
  if (threadIdx.x == 0) {
    if (cs) {
      atomicAdd(&acc[0], cs);
      atomicAdd(&acc[1], hsum);
      atomicAdd(&hist[1], cs);
      atomicMax(&acc[4], 1ull);
    }
  }
}

__global__ void k_isolated(int64_t n, const int64_t* __restrict__ ro, int64_t* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    out[v] = v;
}

int grid_for(int64_t work, int threads = 256) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

template <typename T>
int dalloc(T** p, size_t count, cudaStream_t s) {
  *p = nullptr;
  if (count == 0) count = 1;
  MCE_CHECK(cudaMallocAsync((void**)p, count * sizeof(T), s));
  return 0;
}

// MCE_TRACE=1: host timestamps of the phases of mce_enumerate on stderr (diagnostics)
struct HostTrace {
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  HostTrace() : on(getenv("MCE_TRACE") != nullptr) { t0 = last = std::chrono::steady_clock::now(); }
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[mce_trace] %-22s +%8.3f ms (at %8.3f)\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(),
            std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};

HostTrace* g_tr = nullptr;

struct ClassPlan {
  int W;
  int64_t begin, count;  // slice of the sorted root list
};

template <int W, bool PIVOT_XX, bool XROWS, bool ROWS_SMEM, int WARPS, int TEAM = 0>
int launch_class(EnumArgs args, int requested_workers, int64_t* workers_used, cudaStream_t s,
                 int64_t* launches, size_t mem_budget, cudaEvent_t* ev, bool* xrows_used,
                 Scratch& scr) {
  constexpr int CAP = 32 * W;
  constexpr int CAPP = CAP + 1;
  auto kern = k_enumerate<W, PIVOT_XX, XROWS, ROWS_SMEM, WARPS, TEAM>;
  constexpr int SPW = W < 32 ? 32 : W;
  constexpr int RCOPIES = TEAM ? 1 : WARPS;
  size_t smem = HIST_SMEM * sizeof(unsigned int) + 3 * WARPS * SPW * sizeof(uint32_t) +
                (size_t)WARPS * CMP_WORDS * sizeof(int32_t) +
                (ROWS_SMEM ? (size_t)RCOPIES * (W * CAPP + CAP) * sizeof(uint32_t) : 0);
  if (g_tr) g_tr->mark("class start");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static int per_sm_cache[64];  // per instantiation and device: attribute + occupancy once
  static bool have[64];
  if (dev < 0 || dev >= 64) dev = 0;
  if (!have[dev]) {
    // (default carveout: these kernels lean on L1 for their global rows,
    // stacks and X rows -- max-shared measured slower)
    MCE_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MCE_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_cache[dev], kern, WARPS * 32, smem));
    have[dev] = true;
    if (getenv("MCE_TRACE"))
      fprintf(stderr, "[mce_trace] k_enumerate W=%d: %d CTAs/SM of %d warps, %zu B shared each\n", W,
              per_sm_cache[dev], WARPS, smem);
  }
  const int per_sm = per_sm_cache[dev];
  if (per_sm < 1) {
    mce_set_error("enumerate kernel W=%d does not fit on an SM", W);
    return -3;
  }
  // every worker must be co-resident: idle workers spin until woken
  int64_t resident = (int64_t)per_sm * sms * WARPS;
  // DFS depth <= |P| of the root: the class's stack never exceeds min(CAP, max |P|)
  const int64_t levels = std::min<int64_t>(CAP, std::max<int64_t>(args.levels, 1)) + 3;
  const int64_t xcap = std::max<int64_t>(args.xcap, 1);
  size_t per_worker = sizeof(uint32_t) * (size_t)(levels * 4 * W) + sizeof(int32_t) * levels +
                      (sizeof(int32_t) + sizeof(uint64_t)) * (levels + 2) +
                      sizeof(int32_t) * 2 * xcap + sizeof(Mailbox) + sizeof(uint32_t) * 2 * W +
                      sizeof(int) * 2 +
                      sizeof(long long) * 4 +
                      (XROWS ? sizeof(uint32_t) * (size_t)W * xcap : 0) +
                      (args.roots_mode == 2 ? sizeof(int32_t) * xcap : 0) +
                      sizeof(uint32_t) * (size_t)(W * CAPP + CAP);  // rows_g+plist_g, or pub
  if (g_tr) g_tr->mark("class occupancy");
  int64_t by_mem = std::max<int64_t>(1, (int64_t)(mem_budget / per_worker));
  int64_t workers = requested_workers > 0 ? requested_workers : resident;
  workers = std::min<int64_t>(workers, resident);
  workers = std::min<int64_t>(workers, by_mem);
  // a few narrow roots need few workers; wide roots (deep subtrees) feed every
  // resident warp through donations, however few they are
  if (requested_workers <= 0 && W < 8)
    workers = std::min<int64_t>(workers, std::max<int64_t>(args.num_roots, 1) + resident / 4);
  workers = std::max<int64_t>(workers, 1);
  constexpr int TT = TEAM > 0 ? TEAM : 1;
  if (TEAM)  // whole teams: a requested count rounds up, a resident one down
    workers = requested_workers > 0 ? std::min<int64_t>((workers + TT - 1) / TT * TT, resident)
                                    : std::max<int64_t>(TT, workers / TT * TT);
  args.num_workers = (int)workers;
  args.levels = (int)levels;
  args.xcap = xcap;
  *workers_used = std::max<int64_t>(*workers_used, workers);
  auto get = [&](auto** p, size_t count) -> int { return scr.get(p, count); };
  if (get(&args.stack, (size_t)workers * levels * 4 * W) || get(&args.lpx, (size_t)workers * levels) ||
      get(&args.rpath, (size_t)workers * (levels + 2)) || get(&args.hsum, (size_t)workers * (levels + 2)) ||
      get(&args.xx, (size_t)workers * xcap) || get(&args.xtmp, (size_t)workers * xcap) ||
      get(&args.mbits, (size_t)workers * 2 * W))
    return -1;
  // the worker list's zero-initialised state in one block, one memset
  const size_t z_mbox = sizeof(Mailbox) * (size_t)workers;
  const size_t z_root = sizeof(unsigned long long) * ROOT_STRIPES * ROOT_STRIDE;
  const size_t z_wl = 128;
  const size_t z_wake = (sizeof(int) * (size_t)workers + 127) / 128 * 128;
  const size_t z_idle = (sizeof(unsigned) * (size_t)((workers + 31) / 32) + 127) / 128 * 128;
  const size_t z_refs = TEAM ? (sizeof(unsigned) * (size_t)(workers / TT) + 127) / 128 * 128 : 0;
  const size_t z_total = z_mbox + z_root + z_wl + z_wake + z_idle + z_refs;
  unsigned char* zblk = nullptr;
  if (get(&zblk, z_total)) return -1;
  args.root_counter = reinterpret_cast<unsigned long long*>(zblk);
  args.wl = reinterpret_cast<WorkerListDev*>(zblk + z_root);
  args.wl_wake = reinterpret_cast<int*>(zblk + z_root + z_wl);
  args.idle_bits = reinterpret_cast<unsigned*>(zblk + z_root + z_wl + z_wake);
  args.mbox = reinterpret_cast<Mailbox*>(zblk + z_root + z_wl + z_wake + z_idle);
  args.pub_refs = TEAM ? reinterpret_cast<unsigned*>(zblk + z_root + z_wl + z_wake + z_idle + z_mbox)
                       : nullptr;
  args.xrows = nullptr;
  args.xlist = nullptr;
  args.rows_g = nullptr;
  args.plist_g = nullptr;
  if (XROWS && get(&args.xrows, (size_t)workers * W * xcap)) return -1;
  if (args.roots_mode == 2 && get(&args.xlist, (size_t)workers * xcap)) return -1;
  args.pub = nullptr;
  if (ROWS_SMEM && args.worker_list_on &&
      get(&args.pub, (size_t)(TEAM ? workers / TT : workers) * (W * CAPP + CAP)))
    return -1;
  if (!ROWS_SMEM && (get(&args.rows_g, (size_t)workers * W * CAPP) ||
                     get(&args.plist_g, (size_t)workers * CAP)))
    return -1;
  if (g_tr) g_tr->mark("class buffers");
  MCE_CHECK(cudaMemsetAsync(zblk, 0, z_total, s));
  const int grid = (int)((workers + WARPS - 1) / WARPS);
  if (g_tr) g_tr->mark("class memsets");
  MCE_CHECK(cudaEventRecord(ev[0], s));
  kern<<<grid, WARPS * 32, smem, s>>>(args);
  mce_count_launch();
  MCE_CHECK(cudaEventRecord(ev[1], s));
  *xrows_used = XROWS;
  MCE_CHECK(cudaGetLastError());
  (*launches)++;
  return 0;
}

// W = 16 / 32 as teams (one shared copy of the rows per CTA; MCE_TEAM=1).
// Built, parity-tested and measured slower than the per-warp workers, so
// off by default: on rmat20's core a W = 32 root took 31.6 s as 1 team of 8
// warps per SM (a takeover copies up to 77 KB of rows; remote branches only
// from |P| >= 48) against 14.9 s for 12 per-warp workers per SM reading
// L1/L2-resident rows; W = 8 / 16 chunk 987 vs 981 ms.
inline bool team(const EnumArgs& a) {
  const char* e = getenv("MCE_TEAM");
  return a.worker_list_on && e && atoi(e) != 0;
}

template <bool PIVOT_XX, bool XROWS>
int launch_W(int W, EnumArgs args, int workers, int64_t* used, cudaStream_t s, int64_t* launches,
             size_t budget, cudaEvent_t* ev, bool* xr, Scratch& scr) {
  switch (W) {
    case 1: return launch_class<1, PIVOT_XX, XROWS, true, 8>(args, workers, used, s, launches, budget, ev, xr, scr);
    case 2: return launch_class<2, PIVOT_XX, XROWS, true, 8>(args, workers, used, s, launches, budget, ev, xr, scr);
    case 4: return launch_class<4, PIVOT_XX, XROWS, true, 8>(args, workers, used, s, launches, budget, ev, xr, scr);
    case 8: return launch_class<8, PIVOT_XX, XROWS, true, 4>(args, workers, used, s, launches, budget, ev, xr, scr);
    case 16:
      if (team(args)) return launch_class<16, PIVOT_XX, XROWS, true, 4, 4>(args, workers, used, s, launches, budget, ev, xr, scr);
      return launch_class<16, PIVOT_XX, XROWS, true, 2>(args, workers, used, s, launches, budget, ev, xr, scr);
    case 32:
      if (team(args)) return launch_class<32, PIVOT_XX, XROWS, true, 8, 8>(args, workers, used, s, launches, budget, ev, xr, scr);
      return launch_class<32, PIVOT_XX, XROWS, false, 4>(args, workers, used, s, launches, budget, ev, xr, scr);
    case 64: return launch_class<64, PIVOT_XX, XROWS, false, 4>(args, workers, used, s, launches, budget, ev, xr, scr);
    case 128: return launch_class<128, PIVOT_XX, XROWS, false, 4>(args, workers, used, s, launches, budget, ev, xr, scr);
  }
  mce_set_error("unsupported bitset width %d", W);
  return -3;
}

// the lane-per-root kernel over the |P| <= 32 roots, timed by its own event pair
int launch_tiny(bool full, TinyArgs ta, cudaStream_t s, cudaEvent_t* ev, int64_t* launches,
                int64_t* workers_used, Scratch& scr) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dev < 0 || dev >= 64) dev = 0;
  static int per_sm[2][64];
  static bool have[2][64];
  const size_t smem = sizeof(uint32_t) * TINY_SMEM_WORDS;
  auto kern = full ? k_tiny<true> : k_tiny<false>;
  if (!have[full][dev]) {
    MCE_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // all of the unified L1 as shared memory: three CTAs' slices per SM
    MCE_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                   cudaSharedmemCarveoutMaxShared));
    MCE_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[full][dev], kern, TINY_THREADS, smem));
    if (getenv("MCE_TRACE"))
      fprintf(stderr, "[mce_trace] k_tiny: %d CTAs/SM, %zu B shared each\n", per_sm[full][dev], smem);
    have[full][dev] = true;
  }
  if (per_sm[full][dev] < 1) {
    mce_set_error("tiny-root kernel does not fit on an SM");
    return -3;
  }
  // one warp claims 32 roots: no more CTAs than that keeps busy
  const int64_t need = (ta.num_roots + TINY_THREADS - 1) / TINY_THREADS;
  int64_t g = std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm[full][dev] * sms, need));
  if (ta.max_warps > 0) g = std::min<int64_t>(g, (ta.max_warps + TINY_WARPS - 1) / TINY_WARPS);
  else ta.max_warps = (int)(g * TINY_WARPS);
  const int grid = (int)g;
  *workers_used = std::max<int64_t>(*workers_used, ta.max_warps);
  if (scr.get(&ta.spill, (size_t)grid * TINY_THREADS * TINY_SPILL * 8)) return -1;
  MCE_CHECK(cudaEventRecord(ev[0], s));
  kern<<<grid, TINY_THREADS, smem, s>>>(ta);
  mce_count_launch();
  MCE_CHECK(cudaEventRecord(ev[1], s));
  MCE_CHECK(cudaGetLastError());
  (*launches)++;
  return 0;
}

// Partial mode ("ip") keeps the reference's pivot rule (P | X_P only) but, when
// HBM allows, still materialises the X rows so X_X adjacency is one bit test
// instead of a binary search of the CSR -- same traversal tree, fewer
// dependent loads.  Full mode ("ipx") always has them.
int launch_mode(bool full, int W, int xrows_min_w, EnumArgs args, int workers, int64_t* used,
                cudaStream_t s, int64_t* launches, size_t budget, int64_t resident_guess,
                cudaEvent_t* ev, bool* xr, Scratch& scr) {
  if (full) return launch_W<true, true>(W, args, workers, used, s, launches, budget, ev, xr, scr);
  const size_t xrows_bytes = sizeof(uint32_t) * (size_t)W * (size_t)std::max<int64_t>(args.xcap, 1) *
                             (size_t)std::max<int64_t>(resident_guess, 1);
  // small-|P| roots visit few nodes: building X rows (|X| x |N+(x)| loads)
  // costs more than the CSR look-ups it saves
  if (W >= xrows_min_w && xrows_bytes <= budget / 2)
    return launch_W<false, true>(W, args, workers, used, s, launches, budget, ev, xr, scr);
  return launch_W<false, false>(W, args, workers, used, s, launches, budget, ev, xr, scr);
}

}  // namespace

extern "C" {

int mce_enumerate(const mce_graph* g, const mce_run_config* cfg, int64_t* collect,
                  int64_t* worker_metrics, int64_t worker_metrics_cap, mce_run_result* out,
                  void* stream) {
  HostTrace tr;
  g_tr = &tr;
  struct TrReset { ~TrReset() { g_tr = nullptr; } } tr_reset;
  mce_prepare_device();
  cudaStream_t s = (cudaStream_t)stream;
  memset(out, 0, sizeof(*out));
  if (cfg->roots != 1 && cfg->roots != 2) {
    mce_set_error("roots must be 1 (l1) or 2 (l2)");
    return -2;
  }
  const int64_t n = g->n;
  if (n == 0) return 0;
  tr.mark("enter");
  Scratch scr(s);  // every temporary of this call (released after the final sync)
  tr.mark("scratch");
  auto get = [&](auto** p, size_t count) -> int { return scr.get(p, count); };
  auto cleanup = [&]() {};
  // --- root list ---------------------------------------------------------
  int64_t* eoff = nullptr;
  int64_t total_roots = n;
  if (cfg->roots == 2) {
    int64_t* later = nullptr;
    if (get(&later, n) || get(&eoff, n + 1)) return -1;
    k_later_count<<<grid_for(n), 256, 0, s>>>(g->ro, g->split, n, later);
    mce_count_launch();
    MCE_CHECK(cudaMemsetAsync(eoff, 0, sizeof(int64_t), s));
    size_t tb = 0;
    MCE_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tb, later, eoff + 1, n, s));
    void* tmp = nullptr;
    if (scr.raw(&tmp, tb)) return -1;
    MCE_CHECK(cub::DeviceScan::InclusiveSum(tmp, tb, later, eoff + 1, n, s));
    MCE_CHECK(cudaMemcpyAsync(&total_roots, eoff + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MCE_CHECK(cudaStreamSynchronize(s));
  }
  int64_t begin = std::max<int64_t>(cfg->root_begin, 0);
  int64_t end = (cfg->root_end < 0 || cfg->root_end > total_roots) ? total_roots : cfg->root_end;
  int64_t stride = cfg->root_stride > 0 ? cfg->root_stride : 1;
  int64_t count = end > begin ? (end - begin + stride - 1) / stride : 0;

  // per-vertex hash terms: built once per graph and labelling choice (never
  // rebuilt, so a concurrent call on the same graph cannot see a table change
  // under it); the build is guarded and every reader waits for its event
  mce_graph* gm = const_cast<mce_graph*>(g);
  const int want_labels = (cfg->hash_labels && g->labels) ? 1 : 0;
  {
    static std::mutex vh_mu;
    std::lock_guard<std::mutex> lk(vh_mu);
    if (!gm->vhash_tab[want_labels]) {
      uint64_t* tab = nullptr;
      if (dalloc(&tab, n, s)) return -1;
      k_vhash<<<grid_for(n), 256, 0, s>>>(want_labels ? g->labels : nullptr, n, tab);
      mce_count_launch();
      MCE_CHECK(cudaEventCreateWithFlags(&gm->vhash_ev[want_labels], cudaEventDisableTiming));
      MCE_CHECK(cudaEventRecord(gm->vhash_ev[want_labels], s));
      gm->vhash_tab[want_labels] = tab;
    } else {
      MCE_CHECK(cudaStreamWaitEvent(s, gm->vhash_ev[want_labels], 0));
    }
  }
  const uint64_t* vhash = gm->vhash_tab[want_labels];
  {  // the packed N+ lists (same once-per-graph rule)
    static std::mutex up_mu;
    std::lock_guard<std::mutex> lk(up_mu);
    if (!gm->up_off) {
      int64_t *off = nullptr, *later = nullptr;
      int32_t* ucol = nullptr;
      if (dalloc(&off, n + 1, s) || dalloc(&ucol, std::max<int64_t>(g->nnz / 2, 1), s) ||
          get(&later, n))
        return -1;
      k_later_count<<<grid_for(n), 256, 0, s>>>(g->ro, g->split, n, later);
      mce_count_launch();
      MCE_CHECK(cudaMemsetAsync(off, 0, sizeof(int64_t), s));
      size_t tb = 0;
      MCE_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tb, later, off + 1, n, s));
      void* tmp = nullptr;
      if (scr.raw(&tmp, tb)) return -1;
      MCE_CHECK(cub::DeviceScan::InclusiveSum(tmp, tb, later, off + 1, n, s));
      k_pack_upper<<<grid_for(n), 256, 0, s>>>(g->ro, g->split, g->col, off, n, ucol);
      mce_count_launch();
      MCE_CHECK(cudaGetLastError());
      MCE_CHECK(cudaEventCreateWithFlags(&gm->up_ev, cudaEventDisableTiming));
      MCE_CHECK(cudaEventRecord(gm->up_ev, s));
      gm->up_col = ucol;
      gm->up_off = off;
    } else {
      MCE_CHECK(cudaStreamWaitEvent(s, gm->up_ev, 0));
    }
  }
  int64_t metric_slots = 0;
  {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    metric_slots = cfg->workers > 0 ? cfg->workers : (int64_t)sms * 64;
  }
  // every zero-initialised word of the call in one block, one memset:
  // acc[8] | hist[HIST_MAX] | collect_len | build bytes | root classes + heavy
  // plan counters [16] | launch phase times [32] | per-worker metrics [WM * metric_slots]
  constexpr int ZB_CLS = 8 + HIST_MAX + 2;
  constexpr int ZB_PH = ZB_CLS + 16;
  constexpr int ZB_WM = ZB_PH + 32;
  static_assert(3 * (NUM_WIDTHS + 1) <= 32, "phase slots");
  const size_t zwords = (size_t)ZB_WM + WM * (size_t)metric_slots;
  unsigned long long* zb = nullptr;
  if (get(&zb, zwords)) return -1;
  MCE_CHECK(cudaMemsetAsync(zb, 0, zwords * sizeof(unsigned long long), s));
  unsigned long long* acc = zb;
  unsigned long long* hist = zb + 8;
  unsigned long long* collect_len = zb + 8 + HIST_MAX;
  unsigned long long* bb = collect_len + 1;
  long long* wmet = reinterpret_cast<long long*>(zb + ZB_WM);
  unsigned long long* phase = zb + ZB_PH;  // 3 words per launch
  int nph = 0;
  int64_t* d_collect = nullptr;
  if (cfg->collect_cap > 0 && get(&d_collect, cfg->collect_cap)) {
    cleanup();
    return -1;
  }

  int64_t max_workers_slots = 0;
  int64_t launches = 0;
  int64_t trivial_nodes = 0;
  int64_t workers_used = 0;
  // timing events, created once per device (one call at a time uses them: the
  // call holds them until its final synchronisation)
  static cudaEvent_t ev_cache[64][2 * (NUM_WIDTHS + 1)];
  static bool ev_have[64];
  static std::mutex ev_mu;
  std::unique_lock<std::mutex> ev_lock(ev_mu);
  int ev_dev = 0;
  cudaGetDevice(&ev_dev);
  if (ev_dev < 0 || ev_dev >= 64) ev_dev = 0;
  if (!ev_have[ev_dev]) {
    for (int e = 0; e < 2 * (NUM_WIDTHS + 1); ++e) MCE_CHECK(cudaEventCreate(&ev_cache[ev_dev][e]));
    ev_have[ev_dev] = true;
  }
  cudaEvent_t* events = ev_cache[ev_dev];
  int nev = 0;
  // pinned staging for the D2H reads of this call (guarded by ev_lock): the
  // zeroed block comes back in ONE copy; pageable destinations would be
  // staged by the driver and cost tens of microseconds each
  static unsigned long long* pin_buf[64];
  static size_t pin_cap[64];
  if (pin_cap[ev_dev] < zwords) {
    if (pin_buf[ev_dev]) cudaFreeHost(pin_buf[ev_dev]);
    pin_buf[ev_dev] = nullptr;
    pin_cap[ev_dev] = 0;
    MCE_CHECK(cudaHostAlloc((void**)&pin_buf[ev_dev], zwords * sizeof(unsigned long long),
                            cudaHostAllocPortable));
    pin_cap[ev_dev] = zwords;
  }
  unsigned long long* pin = pin_buf[ev_dev];
  unsigned long long* tiny_reasons = nullptr;  // diagnostics (MCE_TRACE)
  tr.mark("vhash+events");
  if (count > 0) {
    uint32_t *keys = nullptr, *keys2 = nullptr;
    int64_t *roots = nullptr, *roots2 = nullptr;
    unsigned long long* cls = zb + ZB_CLS;  // zeroed above
    constexpr int HMETA = MAXP_SLOT + 1;  // cls[HMETA .. HMETA+2] = heavy plan counters
    static_assert(HMETA + 3 <= 16, "class/heavy counters exceed their zeroed slots");
    constexpr int TINY_SLOT = HMETA + 3;  // k_tiny's claim counter and fallback length
    static_assert(TINY_SLOT + 2 <= 16, "tiny counters exceed their zeroed slots");
    if (get(&keys, count) || get(&keys2, count) || get(&roots, count) || get(&roots2, count)) {
      cleanup();
      return -1;
    }
    HeavyPlan hp{};
    // device memory this call may use: free HBM plus the scratch arena it holds
    size_t avail_b = 0;
    avail_b = mce_free_memory() + scr.reserved();
    tr.mark("memgetinfo");
    {
      const size_t free_b = avail_b;
      const char* e = getenv("MCE_HEAVY");  // diagnostics: MCE_HEAVY=0 disables the pre-pass
      hp.enabled = cfg->roots == 1 && !(e && atoi(e) == 0);
      hp.pool_cap = std::min<unsigned long long>(free_b / 16, 1ull << 30) / sizeof(uint32_t);
      hp.meta = cls + HMETA;
      if (hp.enabled && (get(&hp.vertex, HEAVY_MAX) || get(&hp.off, HEAVY_MAX) ||
                         get(&hp.unit0, HEAVY_MAX) || get(&hp.unit_slot, HEAVY_UNITS_MAX))) {
        cleanup();
        return -1;
      }
    }
    tr.mark("setup");
    k_root_keys<<<grid_for(count), 256, 0, s>>>(g->ro, g->split, g->col, eoff, n, cfg->roots,
                                                 begin, stride, count, keys, roots, cls, cls + MAXP_SLOT,
                                                 hp);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
    cub::DoubleBuffer<uint32_t> dk(keys, keys2);
    cub::DoubleBuffer<int64_t> dv(roots, roots2);
    size_t tb = 0;
    MCE_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, count, 0, 24, s));
    void* tmp = nullptr;
    if (scr.raw(&tmp, tb)) return -1;
    MCE_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, count, 0, 24, s));
    unsigned long long* hc = pin + ZB_CLS;  // pinned: cls[0 .. HMETA + 3)
    MCE_CHECK(cudaMemcpyAsync(hc, cls, (HMETA + 3) * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, s));
    tr.mark("root keys+sort queued");
    MCE_CHECK(cudaStreamSynchronize(s));
    tr.mark("class counts synced");
    if (mce_graph_sync_stats(g)) return -1;  // complete by now (the stream is idle)
    // induced = auto: the reference's rule (scheduler.py:36-41) on the reordered
    // graph, whose max |N+(v)| is the degeneracy
    const bool full = cfg->induced_full >= 0
                          ? cfg->induced_full != 0
                          : !(g->max_later > 0 &&
                              (double)g->max_degree / (double)g->max_later > 200.0);
    out->induced_full = full ? 1 : 0;
    const int64_t* sorted_roots = dv.Current();
    // capacity first: nothing below may run for a root wider than the widest class
    // (k_heavy_xrows stages P in a MAX_CAPACITY_BITS shared array)
    const int64_t cap_limit = std::min<int64_t>(
        cfg->capacity_bits > 0 ? cfg->capacity_bits : MAX_CAPACITY_BITS, MAX_CAPACITY_BITS);
    const int64_t max_p = (int64_t)hc[MAXP_SLOT];
    if (max_p > cap_limit) {
      mce_set_error("CapacityError: |P| = %lld exceeds capacity %lld", (long long)max_p,
                    (long long)cap_limit);
      cleanup();
      return -4;
    }
    // heavy-X roots: their X rows over the whole grid, before the enumeration
    uint32_t* heavy_pool = nullptr;
    const unsigned long long heavy_units = std::min<unsigned long long>(hc[HMETA + 2], HEAVY_UNITS_MAX);
    if (hp.enabled && heavy_units > 0) {
      const unsigned long long words = std::min<unsigned long long>(hc[HMETA + 1], hp.pool_cap);
      if (get(&heavy_pool, words)) {
        cleanup();
        return -1;
      }
      MCE_CHECK(cudaMemsetAsync(heavy_pool, 0, words * sizeof(uint32_t), s));
      k_heavy_xrows<<<(unsigned)heavy_units, 256, 0, s>>>(hp, g->ro, g->split, g->col, heavy_pool);
      mce_count_launch();
      MCE_CHECK(cudaGetLastError());
    }
    // diagnostics: MCE_PROFILE_ROOTS=<file> dumps (root, W, cycles) per root
    const char* prof_path = getenv("MCE_PROFILE_ROOTS");
    long long* prof_cycles = nullptr;
    if (prof_path && get(&prof_cycles, count)) {
      cleanup();
      return -1;
    }
    if (prof_cycles) MCE_CHECK(cudaMemsetAsync(prof_cycles, 0, sizeof(long long) * count, s));
    const int widths[NUM_WIDTHS] = {128, 64, 32, 16, 8, 4, 2, 1};
    std::vector<ClassPlan> plan;
    int64_t i = 0;
    for (int c = 0; c < NUM_WIDTHS; ++c) {
      if (hc[c]) plan.push_back({widths[c], i, (int64_t)hc[c]});
      i += (int64_t)hc[c];
    }
    const int64_t trivial_begin = i;  // first-level roots with P empty
    const int64_t trivial_count = count - i;
    int64_t wcap = 0;
    double frac = cfg->mem_fraction > 0 ? cfg->mem_fraction : 0.5;
    const size_t budget0 = (size_t)(avail_b * frac);
    const size_t demand0 = scr.demand();
    // per-worker metrics (zeroed above) accumulate across class launches
    for (const ClassPlan& cp : plan) {
      // scratch of the earlier classes stays held until the call returns:
      // each class sizes its workers against what is left of the budget
      const size_t taken = scr.demand() - demand0;
      const size_t budget = budget0 > taken ? budget0 - taken : 0;
      EnumArgs args{};
      args.n = n;
      args.ro = g->ro;
      args.col = g->col;
      args.split = g->split;
      args.up_off = g->up_off;
      args.up_col = g->up_col;
      args.vhash = vhash;
      args.roots = sorted_roots + cp.begin;
      args.num_roots = cp.count;
      args.roots_mode = cfg->roots;
      args.xcap = g->max_earlier;
      args.levels = (int)max_p;
      args.g_acc = acc;
      args.g_hist = hist;
      args.w_metrics = wmet;
      args.root_cycles = prof_cycles ? prof_cycles + cp.begin : nullptr;
      args.collect = d_collect;
      args.collect_cap = cfg->collect_cap;
      args.collect_len = collect_len;
      args.worker_list_on = cfg->worker_list;
      args.min_p = cfg->donation_min_p;
      args.min_x = cfg->donation_min_x;
      args.heavy_rows = heavy_pool;
      args.heavy_off = hp.off;
      args.no_pivot = cfg->no_pivot;
      args.timing = cfg->timing;
      args.phase_ns = phase + 3 * nph++;
      {
        const char* e = getenv("MCE_COMPACT");  // diagnostics: MCE_COMPACT=0 disables compact_run
        args.compact = e ? atoi(e) : 1;
      }
      {
        const char* e = getenv("MCE_XROWS_PARTIAL_MAX");  // diagnostics override
        args.xrows_partial_max = e ? atoi(e) : XROWS_PARTIAL_MAX;
      }
      // |P| <= 32: one root per lane (k_tiny); the roots it hands back (heavy X,
      // dense, many X_X rows) follow in the warp kernel, whose root count the
      // device supplies
      // diagnostics: MCE_TINY=<min class size> (0 disables the lane-per-root path)
      const char* te = getenv("MCE_TINY");
      // (a small class is latency-bound either way: one warp kernel, one launch)
      const int64_t tiny_min = te ? std::max(0, atoi(te)) : TINY_MIN_ROOTS;
      if (cp.W == 1 && cfg->roots == 1 && cfg->collect_cap <= 0 && tiny_min > 0 && cp.count >= tiny_min) {
        int64_t* fb = nullptr;
        if (get(&fb, cp.count)) {
          cleanup();
          return -1;
        }
        TinyArgs ta{};
        ta.ro = g->ro;
        ta.col = g->col;
        ta.split = g->split;
        ta.up_off = g->up_off;
        ta.up_col = g->up_col;
        ta.vhash = vhash;
        ta.roots = sorted_roots + cp.begin;
        ta.num_roots = cp.count;
        ta.counter = cls + TINY_SLOT;
        ta.fallback = fb;
        ta.fallback_len = cls + TINY_SLOT + 1;
        ta.g_acc = acc;
        ta.g_hist = hist;
        ta.w_metrics = wmet;
        ta.phase_ns = phase + 3 * nph++;
        ta.max_warps = cfg->workers > 0 ? cfg->workers : 0;
        ta.no_pivot = cfg->no_pivot;
        ta.timing = cfg->timing;
        ta.reasons = nullptr;
        if (tr.on) {
          if (get(&ta.reasons, 8)) {
            cleanup();
            return -1;
          }
          MCE_CHECK(cudaMemsetAsync(ta.reasons, 0, 8 * sizeof(unsigned long long), s));
          tiny_reasons = ta.reasons;
        }
        if (launch_tiny(full, ta, s, &events[2 * nev++], &launches, &workers_used, scr)) {
          cleanup();
          return -1;
        }
        args.roots = fb;
        args.num_roots_dev = cls + TINY_SLOT + 1;
      }
      int req = cfg->workers > 0 ? cfg->workers : 0;
      if (req <= 0) req = 0;
      const int64_t guess = req > 0 ? req : std::min<int64_t>(metric_slots, cp.count + metric_slots / 4);
      cudaEvent_t* ev = &events[2 * nev++];
      bool xr = false;
      const int xmin = cfg->partial_xrows_min_w > 0 ? cfg->partial_xrows_min_w : 1;
      int rc = launch_mode(full, cp.W, xmin, args, req, &workers_used, s,
                           &launches, budget, guess, ev, &xr, scr);
      tr.mark("class launched");
      if (rc) {
        cleanup();
        return rc;
      }
      if (cfg->measure_bytes && cfg->roots == 1) {  // measurement only (bench roofline)
        k_build_bytes<<<grid_for(cp.count * 32), 256, 0, s>>>(sorted_roots + cp.begin, cp.count,
                                                               g->ro, g->split, g->col, xr, bb);
        mce_count_launch();
      }
      wcap = std::max<int64_t>(wcap, req > 0 ? req : metric_slots);
    }
    max_workers_slots = std::max<int64_t>(workers_used, 1);
    if (prof_cycles) {
      std::vector<long long> cyc(count);
      std::vector<int64_t> rts(count);
      MCE_CHECK(cudaMemcpyAsync(cyc.data(), prof_cycles, sizeof(long long) * count,
                                cudaMemcpyDeviceToHost, s));
      MCE_CHECK(cudaMemcpyAsync(rts.data(), sorted_roots, sizeof(int64_t) * count,
                                cudaMemcpyDeviceToHost, s));
      MCE_CHECK(cudaStreamSynchronize(s));
      if (FILE* f = fopen(prof_path, "wb")) {
        for (const ClassPlan& cp : plan)
          for (int64_t i = cp.begin; i < cp.begin + cp.count; ++i) {
            const int64_t rec[3] = {rts[i] & ROOT_ID_MASK, (int64_t)cp.W, (int64_t)cyc[i]};
            fwrite(rec, sizeof(rec), 1, f);
          }
        fclose(f);
      }
    }
    if (trivial_count > 0) {
      k_trivial_roots<<<grid_for(trivial_count), 256, 0, s>>>(
          sorted_roots + trivial_begin, trivial_count, g->ro, g->split, vhash, acc, hist,
          d_collect, cfg->collect_cap, collect_len);
      mce_count_launch();
      MCE_CHECK(cudaGetLastError());
      trivial_nodes = trivial_count;  // one visited node each (scheduler.py:300-301)
    }
    (void)wcap;
  }
  if (count <= 0) {  // no roots: still report the induced mode an auto run resolves to
    if (mce_graph_sync_stats(g)) return -1;
    out->induced_full = cfg->induced_full >= 0
                            ? (cfg->induced_full != 0)
                            : !(g->max_later > 0 &&
                                (double)g->max_degree / (double)g->max_later > 200.0);
  }
  if (cfg->roots == 2 && cfg->include_isolated) {
    int64_t* all = nullptr;
    if (get(&all, n)) {
      cleanup();
      return -1;
    }
    k_isolated<<<grid_for(n), 256, 0, s>>>(n, g->ro, all);
    mce_count_launch();
    k_trivial_roots<<<grid_for(n), 256, 0, s>>>(all, n, g->ro, g->split, vhash, acc, hist,
                                                 d_collect, cfg->collect_cap, collect_len);
    mce_count_launch();
    MCE_CHECK(cudaGetLastError());
  }
  // one D2H of the zeroed block (counters, histogram, stream length, worker
  // metrics of the slots in use), then host copies out of the pinned staging
  const int64_t wslots = (worker_metrics && worker_metrics_cap > 0)
                             ? std::min<int64_t>(worker_metrics_cap, max_workers_slots)
                             : 0;
  const size_t back = (size_t)ZB_WM + WM * (size_t)std::max<int64_t>(wslots, 0);
  MCE_CHECK(cudaMemcpyAsync(pin, zb, back * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  tr.mark("results queued");
  MCE_CHECK(cudaStreamSynchronize(s));
  tr.mark("results synced");
  if (tr.on) {
    unsigned long long rs[8] = {0};
    if (tiny_reasons)
      cudaMemcpy(rs, tiny_reasons, sizeof(rs), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[mce_trace] k_tiny handed back %llu roots to the warp kernel (heavy-X %llu, "
            "|P|>32 %llu, |X|>%d %llu, row pool %llu, dense %llu)\n",
            pin[ZB_CLS + MAXP_SLOT + 1 + 3 + 1], rs[0], rs[1], TINY_XT, rs[2], rs[3], rs[4]);
  }
  unsigned long long h_acc[8];
  memcpy(h_acc, pin, sizeof(h_acc));
  memcpy(out->hist, pin + 8, sizeof(int64_t) * HIST_MAX);
  const unsigned long long h_len = pin[8 + HIST_MAX];
  const unsigned long long h_bytes = pin[8 + HIST_MAX + 1];
  if (wslots > 0) memcpy(worker_metrics, pin + ZB_WM, sizeof(int64_t) * WM * wslots);
  {  // phase 1 (roots left to claim) / phase 2 (worker list only), per launch
    double p1 = 0.0, p2 = 0.0;
    for (int i = 0; i < nph; ++i) {
      const unsigned long long* ph = pin + ZB_PH + 3 * i;
      if (!ph[0] || !ph[2]) continue;
      const unsigned long long t0 = ~ph[0], t2 = ph[2];
      const unsigned long long t1 = ph[1] ? std::min(~ph[1], t2) : t2;
      if (t1 > t0) p1 += (double)(t1 - t0) / 1e6;
      if (t2 > t1) p2 += (double)(t2 - t1) / 1e6;
    }
    out->phase1_ms = p1;
    out->phase2_ms = p2;
    // (the clock-rate attribute costs milliseconds per query: once per device)
    static int khz_cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!khz_cache[dev]) cudaDeviceGetAttribute(&khz_cache[dev], cudaDevAttrClockRate, dev);
    out->clock_khz = (double)khz_cache[dev];
  }
  if (collect && cfg->collect_cap > 0) {
    int64_t words = std::min<int64_t>((int64_t)h_len, cfg->collect_cap);
    if (words > 0) {
      MCE_CHECK(cudaMemcpyAsync(collect, d_collect, sizeof(int64_t) * words,
                                cudaMemcpyDeviceToHost, s));
      MCE_CHECK(cudaStreamSynchronize(s));
    }
  }
  out->cliques = (int64_t)h_acc[0];
  out->hash = (uint64_t)h_acc[1];
  out->nodes = (int64_t)h_acc[2] + trivial_nodes;
  if (worker_metrics && worker_metrics_cap > 0) worker_metrics[0] += trivial_nodes;
  out->donations = (int64_t)h_acc[3];
  out->max_size = (int64_t)h_acc[4];
  out->workers = max_workers_slots;
  out->launches = launches;
  out->collect_len = (int64_t)h_len;
  out->build_bytes = (int64_t)h_bytes;
  double kernel_ms = 0.0;
  for (int e = 0; e < nev; ++e) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, events[2 * e], events[2 * e + 1]);
    kernel_ms += ms;
  }
  out->kernel_ms = kernel_ms;
  cleanup();
  tr.mark("done");
  return 0;
}

}  // extern "C"

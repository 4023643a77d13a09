// Thread-per-root enumeration of the tiny first-level roots (|P| <= 32): the
// narrowest subwarp partition -- a bitset over the root's P is ONE 32-bit
// register, so each lane of a warp runs a whole root on its own and a warp
// works 32 roots at once (the warp-per-root Worker leaves most lanes idle on
// a 10-member P).  Included by mce_enum.cu inside its anonymous namespace.
//
// Same traversal as Worker::traverse / compact_run (reference bk.py:82-110,
// scheduler.py:297-381, xsets.py:55-82): pivot = max |N(c) & P| over
// P | X_P, ties to the smallest id, full mode's X_X rows only when strictly
// better (first in prefix order); leaves of a node settled in one pass; the
// X_X prefix stably partitioned in place on descent and never restored -- so
// node totals are identical to the warp kernels'.
//
// A warp claims 32 consecutive roots of the (heaviest-first) class list and
//  * builds them TOGETHER: the N+ lists of all their P and X members are one
//    flattened stream over the lanes (coalesced loads, 128 in flight per
//    warp, the same walk as Worker::build), hits OR-ed into each root's rows
//    in shared memory -- a lane walking its own root's lists alone would
//    issue 32 uncoalesced sectors per load instruction;
//  * then runs one root per lane: member list, induced rows and X rows of
//    root r at [r * 33 + i] of the warp's shared-memory slices (33: distinct
//    banks across lanes), the DFS frames in local memory (L1).
//
// A root leaves this path for the warp kernel (appended to `fallback`) when
// it has a heavy-X pool slot, more than TINY_XT earlier neighbours, or more
// than TINY_E_MAX induced edges (a bound on its subtree: one lane must not
// carry a big search tree).

constexpr int TINY_WARPS = 8;
#ifndef MCE_TINY_U
#define MCE_TINY_U 4  // entry loads per lane in flight in the build walk
#endif
constexpr int64_t TINY_MIN_ROOTS = 8192;  // smaller W = 1 classes stay on the warp kernel
constexpr int TINY_THREADS = 32 * TINY_WARPS;
#ifndef MCE_TINY_XT
#define MCE_TINY_XT 32
#endif
#ifndef MCE_TINY_POOL
#define MCE_TINY_POOL 1024
#endif
constexpr int TINY_XT = MCE_TINY_XT;  // X members per root
static_assert(TINY_XT <= 64, "X member index has 6 bits in the walk's member word");
constexpr int TINY_STRIDE = 33;
constexpr int TINY_SLICE = 32 * TINY_STRIDE;  // member lists: words per warp
constexpr int TINY_POOL = MCE_TINY_POOL;  // rows + X rows of a warp's 32 roots (np + nx words each)
#ifndef MCE_TINY_E_MAX
#define MCE_TINY_E_MAX 64
#endif
constexpr int TINY_E_MAX = MCE_TINY_E_MAX;
// a clique of c members in P needs c(c-1)/2 <= TINY_E_MAX edges
constexpr int tiny_max_clique(int e) {
  int c = 1;
  while ((c + 1) * c / 2 <= e) ++c;
  return c;
}
constexpr int TINY_DEPTH = tiny_max_clique(TINY_E_MAX) + 1;  // local frames
constexpr int TINY_SPILL = 33 - TINY_DEPTH;  // global frames (a pushed level holds a P member)
// a root denser than TINY_E_MAX edges stays here when its P misses at most
// TINY_M_MAX edges (a near-clique: few maximal cliques, a short tree)
#ifndef MCE_TINY_M_MAX
#define MCE_TINY_M_MAX 16
#endif
constexpr int TINY_M_MAX = MCE_TINY_M_MAX;
constexpr int TINY_WARP_WORDS = TINY_SLICE + TINY_POOL + 128;  // + 32 x 2 bloom words (64-bit)
constexpr int TINY_SMEM_WORDS = HIST_SMEM + TINY_WARP_WORDS * TINY_WARPS;

struct TinyArgs {
  const int64_t* ro;
  const int32_t* col;
  const int64_t* split;
  const int64_t* up_off;             // packed N+ lists (mce_graph::up_off / up_col)
  const int32_t* up_col;
  const uint64_t* vhash;
  const int64_t* roots;
  int64_t num_roots;
  unsigned long long* counter;       // roots claimed (batches of 32, one per warp)
  int64_t* fallback;                 // roots handed to the warp kernel
  unsigned long long* fallback_len;
  unsigned long long* g_acc;         // 0 cliques, 1 hash, 2 nodes, 3 donations, 4 max size
  unsigned long long* g_hist;
  long long* w_metrics;              // per warp: MCE_WM_COLS columns
  unsigned long long* phase_ns;      // [~first start, ~first root-list miss, last end] (atomicMax)
  int max_warps;                     // workers requested (warps >= this stay idle)
  int no_pivot;                      // basic Bron-Kerbosch: branch on all of P
  int timing;                        // SM cycles by category into w_metrics
  unsigned long long* reasons;       // diagnostics (MCE_TRACE): hand-backs by cause
  uint32_t* spill;                   // DFS frames past TINY_DEPTH: TINY_SPILL x 8 words per thread
};

__device__ __forceinline__ void tiny_hist_add(unsigned* s_hist, unsigned long long* g_hist, int size) {
  const unsigned old = atomicAdd(&s_hist[size], 1u);
  if (old == 0x7fffffffu) {  // spill 2^31 to HBM
    atomicAdd(&g_hist[size], 0x80000000ull);
    atomicSub(&s_hist[size], 0x80000000u);
  }
}

// index of w in the padded 32-entry member list pl (5 branchless steps), -1 if absent
__device__ __forceinline__ int tiny_find(const int32_t* pl, int32_t w) {
  int i = 0;
  i += pl[i + 15] < w ? 16 : 0;
  i += pl[i + 7] < w ? 8 : 0;
  i += pl[i + 3] < w ? 4 : 0;
  i += pl[i + 1] < w ? 2 : 0;
  i += pl[i] < w ? 1 : 0;
  return pl[i] == w ? i : -1;
}

// The lane's root r = lane: DFS over its rows (same rules as compact_run).
template <bool PIVOT_XX>
__device__ __forceinline__ void tiny_dfs(const TinyArgs& a, const int32_t* pl, const uint32_t* rows,
                                         uint32_t* xm, int np, int live, uint64_t hs,
                                         unsigned* s_hist, unsigned long long& cliques,
                                         unsigned long long& hash, unsigned long long& nodes,
                                         unsigned long long& max_size, bool no_pivot) {
  uint32_t P = np == 32 ? ~0u : ((1u << np) - 1u), XP = 0, BR = 0, NL = 0;
  int rlen = 1, depth = 0;
  nodes++;
  // Frames are pushed only for levels with non-leaf branches left (a level
  // whose last branch is being visited is never returned to: a tail call),
  // so a clique-like P needs next to none.  The first TINY_DEPTH frames live
  // in local memory (L1); deeper ones in this thread's global spill slots.
  uint32_t fP[TINY_DEPTH], fXP[TINY_DEPTH], fBR[TINY_DEPTH], fNL[TINY_DEPTH];
  int flr[TINY_DEPTH];  // live | rlen << 16
  uint64_t fhs[TINY_DEPTH];
  uint32_t* spill = a.spill + ((size_t)blockIdx.x * TINY_THREADS + threadIdx.x) * TINY_SPILL * 8;
  bool fresh = true;
  for (;;) {
    if (fresh) {
      fresh = false;
      // pivot (bk.py:82-110): max |N(c) & P| over P | X_P, ties to the smallest id
      int best = -1;
      uint32_t prow = 0;
      for (uint32_t t = P | XP; t; t &= t - 1) {
        const uint32_t r = rows[__ffs(t) - 1];
        const int c = __popc(r & P);
        if (c > best) {
          best = c;
          prow = r;
        }
      }
      uint32_t xxadj = 0;
      for (int i = 0; i < live; ++i) {
        const uint32_t r = xm[i];
        xxadj |= r;
        if (PIVOT_XX) {  // X_X rows win only when strictly better, first in prefix order
          const int c = __popc(r & P);
          if (c > best) {
            best = c;
            prow = r;
          }
        }
      }
      if (no_pivot) prow = 0;  // basic BK: every member of P is a branch
      BR = P & ~prow;
      // leaf batch: every branch whose child P is empty (see Worker::leaf_batch)
      const int size = rlen + 1;
      uint32_t leafm = 0;
      for (uint32_t t = BR; t; t &= t - 1) {
        const int sl = __ffs(t) - 1;
        const uint32_t bit = 1u << sl;
        const uint32_t before = BR & (bit - 1u);
        const uint32_t r = rows[sl];
        if ((r & (P & ~before)) == 0) {
          leafm |= bit;
          if ((r & (XP | before)) == 0 && !(xxadj & bit)) {
            cliques++;
            hash += mce_mix64(hs + __ldg(&a.vhash[pl[sl]]) + (uint64_t)size * MCE_SIZE_SALT);
            if ((unsigned long long)size > max_size) max_size = size;
            tiny_hist_add(s_hist, a.g_hist, size);
          }
        }
      }
      nodes += __popc(leafm);
      NL = BR & ~leafm;
    }
    if (NL == 0) {
      if (depth == 0) break;
      depth--;
      int lr;
      if (depth < TINY_DEPTH) {
        P = fP[depth];
        XP = fXP[depth];
        BR = fBR[depth];
        NL = fNL[depth];
        lr = flr[depth];
        hs = fhs[depth];
      } else {
        const uint32_t* f = spill + (depth - TINY_DEPTH) * 8;
        P = f[0];
        XP = f[1];
        BR = f[2];
        NL = f[3];
        lr = (int)f[4];
        hs = (uint64_t)f[5] | ((uint64_t)f[6] << 32);
      }
      live = lr & 0xffff;
      rlen = lr >> 16;
      continue;
    }
    // move v and the (leaf) branches before it from P to X_P
    const int vs = __ffs(NL) - 1;
    const uint32_t bit = 1u << vs;
    const uint32_t mv = (BR & (bit - 1u)) | bit;
    BR &= ~mv;
    NL &= ~mv;
    P &= ~mv;
    XP |= mv;
    const uint32_t rv = rows[vs];
    // stable partition of the live X_X prefix by adjacency to v (xsets.py:55-82);
    // the parent's prefix stays permuted (the reference never restores it)
    // (in place: a kept row moves down over the dropped block, which shifts up)
    int kept = 0;
    for (int i = 0; i < live; ++i) {
      const uint32_t r = xm[i];
      if ((r >> vs) & 1u) {
        for (int j = i; j > kept; --j) xm[j] = xm[j - 1];
        xm[kept++] = r;
      }
    }
    if (NL) {  // this level has branches left: come back to it
      if (depth < TINY_DEPTH) {
        fP[depth] = P;
        fXP[depth] = XP;
        fBR[depth] = BR;
        fNL[depth] = NL;
        flr[depth] = live | (rlen << 16);
        fhs[depth] = hs;
      } else {
        uint32_t* f = spill + (depth - TINY_DEPTH) * 8;
        f[0] = P;
        f[1] = XP;
        f[2] = BR;
        f[3] = NL;
        f[4] = (uint32_t)(live | (rlen << 16));
        f[5] = (uint32_t)hs;
        f[6] = (uint32_t)(hs >> 32);
      }
      depth++;
    }
    live = kept;
    XP &= rv;
    P &= rv;
    hs += __ldg(&a.vhash[pl[vs]]);
    rlen++;
    nodes++;
    fresh = true;
  }
}

template <bool PIVOT_XX>
// 80 registers: three 256-thread CTAs per SM (allocation is in 8-register steps)
#ifndef MCE_TINY_MAXREG
#define MCE_TINY_MAXREG 80
#endif
__global__ void __maxnreg__(MCE_TINY_MAXREG) k_tiny(TinyArgs a) {
  extern __shared__ __align__(16) uint32_t tsm[];
  unsigned* s_hist = tsm;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int32_t* spl = reinterpret_cast<int32_t*>(tsm + HIST_SMEM) + warp * TINY_WARP_WORDS;
  unsigned long long* sbloom = reinterpret_cast<unsigned long long*>(spl + TINY_SLICE);
  uint32_t* spool = reinterpret_cast<uint32_t*>(spl + TINY_SLICE + 128);
  for (int i = threadIdx.x; i < HIST_SMEM; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  const int gw = (int)((blockIdx.x * TINY_THREADS + threadIdx.x) >> 5);
  const int32_t* __restrict__ col = a.col;
  if (a.phase_ns && blockIdx.x == 0 && threadIdx.x == 0) atomicMax(&a.phase_ns[0], ~gtimer());
  const long long t_start = clock64();
  long long t_build = 0, t_dfs = 0, t_claim = 0;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long cliques = 0, hash = 0, nodes = 0, max_size = 0;
  long long claimed = 0;
  int32_t* mypl = spl + lane * TINY_STRIDE;
  for (;;) {
    if (gw >= a.max_warps) break;
    long long t0 = a.timing ? clock64() : 0;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(a.counter, 32ull);
    base = __shfl_sync(FULLMASK, base, 0);
    if (a.timing) {
      const long long t1 = clock64();
      t_claim += t1 - t0;
      t0 = t1;
    }
    if (base >= (unsigned long long)a.num_roots) break;
    // ---- lane r: root r of the batch
    const int64_t idx = (int64_t)base + lane;
    const bool valid = idx < a.num_roots;
    const int64_t renc = valid ? a.roots[idx] : 0;
    const int64_t v = renc & ROOT_ID_MASK;
    int64_t xb0 = 0, s0 = 0;
    int np = 0, nx = 0;
    if (valid) {
      xb0 = a.ro[v];
      s0 = a.split[v];
      np = (int)(a.ro[v + 1] - s0);
      nx = (int)(s0 - xb0);
    }
    bool ok = valid && (renc >> ROOT_ID_BITS) == 0 && np <= 32 && nx <= TINY_XT;
    if (a.reasons && valid && !ok)
      atomicAdd(&a.reasons[(renc >> ROOT_ID_BITS) ? 0 : (np > 32 ? 1 : 2)], 1ull);
    if (!ok) np = nx = 0;
    // root r's rows and X rows: np + nx words of the warp's pool at its
    // prefix offset (roots past the pool's end go to the warp kernel)
    int cnt = np + nx;
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(FULLMASK, incl, d);
      if (lane >= d) incl += t;
    }
    if (__any_sync(FULLMASK, incl > TINY_POOL)) {  // the suffix past the pool's end
      if (incl > TINY_POOL) {
        if (a.reasons && ok) atomicAdd(&a.reasons[3], 1ull);
        ok = false;
        np = nx = cnt = 0;
      }
      incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(FULLMASK, incl, d);
        if (lane >= d) incl += t;
      }
    }
    const int excl = incl - cnt;
    const int total = __shfl_sync(FULLMASK, incl, 31);
    uint32_t* myrow = spool + excl;
    uint32_t* myxb = myrow + np;
    // member list (padded for tiny_find), zeroed rows
    for (int k = 0; k < 32; ++k) mypl[k] = 0x7fffffff;
    for (int k = 0; k < cnt; ++k) myrow[k] = 0;
    __syncwarp();  // other lanes fill this root's member list below
    // P member lists: one coalesced pass over the roots' N+ ranges
    for (int q0 = 0; q0 < total; q0 += 32) {
      const int q = q0 + lane;
      int r = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int ic = __shfl_sync(FULLMASK, incl, r + step - 1);
        if (ic <= q) r += step;
      }
      const int k = q - __shfl_sync(FULLMASK, excl, r);
      const int npr = __shfl_sync(FULLMASK, np, r);
      const int64_t sr = __shfl_sync(FULLMASK, s0, r);
      if (q < total && k < npr) spl[r * TINY_STRIDE + k] = __ldg(&col[sr + k]);
    }
    __syncwarp();
    {  // 128-bit blocked bloom filter of the root's members (two bits in one
       // of two words): most N+ entries miss P, and a miss skips the search
      unsigned long long b0 = 0, b1 = 0;
      for (int k = 0; k < np; ++k) {
        const uint32_t h = bloom_hash(mypl[k]);
        const unsigned long long bits = bloom_bits(h);
        if (h >> 31) b1 |= bits; else b0 |= bits;
      }
      sbloom[2 * lane] = b0;
      sbloom[2 * lane + 1] = b1;
    }
    __syncwarp();
    for (int q0 = 0; q0 < total; q0 += 32) {
      // lane: member q0 + lane -> its root, kind, index and N+ range
      const int q = q0 + lane;
      int r = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int ic = __shfl_sync(FULLMASK, incl, r + step - 1);
        if (ic <= q) r += step;
      }
      const int k = q - __shfl_sync(FULLMASK, excl, r);
      const int npr = __shfl_sync(FULLMASK, np, r);
      const int64_t xr = __shfl_sync(FULLMASK, xb0, r);
      const int rbase = __shfl_sync(FULLMASK, excl, r);
      int64_t lo = 0;
      int len = 0;
      // root (5 bits) | X member (bit 5) | index (6 bits) | its rows' pool offset
      int info = 0;
      if (q < total) {
        int32_t m;
        if (k < npr) {
          m = spl[r * TINY_STRIDE + k];
          info = r | (k << 6) | (rbase << 12);
        } else {
          m = __ldcs(&col[xr + (k - npr)]);  // the root's own N-: read once
          info = r | 32 | ((k - npr) << 6) | ((rbase + npr) << 12);
        }
        lo = __ldg(&a.up_off[m]);
        len = (int)(__ldg(&a.up_off[m + 1]) - lo);
      }
      // flatten the 32 members' N+ lists over the lanes (see warp_flat_walk)
      int inc2 = len;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(FULLMASK, inc2, d);
        if (lane >= d) inc2 += t;
      }
      const int exc2 = inc2 - len;
      const int tot2 = __shfl_sync(FULLMASK, inc2, 31);
      constexpr int U = MCE_TINY_U;
      for (int b2 = 0; b2 < tot2; b2 += 32 * U) {
        int32_t val[U];
        int inf[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int kk = b2 + u * 32 + lane;
          int o = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const int ic = __shfl_sync(FULLMASK, inc2, o + step - 1);
            if (ic <= kk) o += step;
          }
          const int64_t lo_o = __shfl_sync(FULLMASK, lo, o);
          const int ex_o = __shfl_sync(FULLMASK, exc2, o);
          inf[u] = __shfl_sync(FULLMASK, info, o);
          val[u] = kk < tot2 ? __ldg(&a.up_col[lo_o + (kk - ex_o)]) : 0x7fffffff;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (b2 + u * 32 + lane < tot2) {
            const int rr = inf[u] & 31;
            const uint32_t h = bloom_hash(val[u]);
            const unsigned long long bits = bloom_bits(h);
            if ((sbloom[2 * rr + (h >> 31)] & bits) == bits) {
              const int j = tiny_find(spl + rr * TINY_STRIDE, val[u]);
              if (j >= 0) {
                const int ii = (inf[u] >> 6) & 63;
                uint32_t* rb = spool + (inf[u] >> 12);
                atomicOr(&rb[ii], 1u << j);           // X row t = ii, or P row ii ...
                if (!(inf[u] & 32)) atomicOr(&rb[j], 1u << ii);  // ... and its mirror
              }
            }
          }
        }
      }
    }
    __syncwarp();
    if (a.timing) {
      const long long t1 = clock64();
      t_build += t1 - t0;
      t0 = t1;
    }
    // ---- lane r enumerates root r
    if (ok) {
      int e2 = 0;
      for (int k = 0; k < np; ++k) e2 += __popc(myrow[k]);
      if (e2 > 2 * TINY_E_MAX && np * (np - 1) - e2 > 2 * TINY_M_MAX) {
        if (a.reasons) atomicAdd(&a.reasons[4], 1ull);
        ok = false;
      } else {
        // X members with no neighbour in P never matter (see init_tokens)
        int nxx = 0;
        for (int t = 0; t < nx; ++t) {
          const uint32_t mk = myxb[t];
          if (mk) myxb[nxx++] = mk;
        }
        if (np > 0) {
          tiny_dfs<PIVOT_XX>(a, mypl, myrow, myxb, np, nxx, __ldg(&a.vhash[v]), s_hist, cliques,
                             hash, nodes, max_size, a.no_pivot != 0);
          claimed++;
        }
      }
    }
    const bool fb = valid && !ok;
    const unsigned fm = __ballot_sync(FULLMASK, fb);
    if (fm) {
      unsigned long long o = 0;
      if (lane == 0) o = atomicAdd(a.fallback_len, (unsigned long long)__popc(fm));
      o = __shfl_sync(FULLMASK, o, 0);
      if (fb) a.fallback[o + __popc(fm & lt)] = renc;
    }
    __syncwarp();
    if (a.timing) t_dfs += clock64() - t0;  // the warp waits for its slowest lane
  }
  if (a.phase_ns && lane == 0 && gw < a.max_warps) {
    const unsigned long long t = gtimer();
    if (!*(volatile unsigned long long*)&a.phase_ns[1])
      atomicMax(&a.phase_ns[1], ~t);  // the first warp to find the root list exhausted
    if (t > *(volatile unsigned long long*)&a.phase_ns[2]) atomicMax(&a.phase_ns[2], t);
  }
  // warp totals (64-bit shuffles), one set of atomics per warp
  unsigned long long c = cliques, h = hash, nd = nodes, mx = max_size;
  long long rc = claimed;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_xor_sync(FULLMASK, c, o);
    h += __shfl_xor_sync(FULLMASK, h, o);
    nd += __shfl_xor_sync(FULLMASK, nd, o);
    rc += __shfl_xor_sync(FULLMASK, rc, o);
    const unsigned long long m2 = __shfl_xor_sync(FULLMASK, mx, o);
    mx = m2 > mx ? m2 : mx;
  }
  if (lane == 0 && gw < a.max_warps) {
    if (c) {
      atomicAdd(&a.g_acc[0], c);
      atomicAdd(&a.g_acc[1], h);
      atomicMax(&a.g_acc[4], mx);
    }
    atomicAdd(&a.g_acc[2], nd);
    long long* m = a.w_metrics + (size_t)gw * WM;
    m[0] += (long long)nd;
    m[1] += rc;
    if (a.timing) {
      m[T_BUILD] += t_build;
      m[T_SETOPS] += t_dfs;
      m[T_WLIST] += t_claim;
      m[T_TOTAL] += clock64() - t_start;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HIST_SMEM; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&a.g_hist[i], (unsigned long long)s_hist[i]);
}

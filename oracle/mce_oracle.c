/*
 * mce_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU parity checker.
 *
 * A plain-C restatement of the reference `mce` package (a CPU Python
 * implementation of arXiv:2212.01473) for the maximal-clique-enumeration hot
 * path.  It exists to *check* the CUDA engine in paper_2212_01473_b200/ and
 * to time the reference algorithm on host cores (bench.py cpu_baseline and
 * `--impl reference`).  Nothing in the product path links or calls it.
 *
 * Reference semantics followed (file:line in /root/reference/pkg/src/mce):
 *   degeneracy order ....... graph.py:183-210  (min-degree peel, ties -> smallest id)
 *   first-level roots ...... bk.py:186-190     (P = later nbrs, X = earlier nbrs)
 *   second-level roots ..... bk.py:198-204     (P/X = common nbrs after/before max endpoint)
 *   pivot rule ............. bk.py:82-110      (max |N(c) & P| over P|X_P ascending, ties to
 *                                               smallest id; X_X rows only if strictly better)
 *   traversal + node count . scheduler.py:297-381
 *   full / partial rows .... induced.py:61-103, scheduler.py:397-415
 *   X_X stable partition ... xsets.py:55-82
 *   isolated vertices (L2) . scheduler.py:476-480
 * Pinned against the reference itself through tests/golden (see header).
 */
#include "mce_oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SIZE_SALT 0xD1B54A32D192ED03ull

static inline uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

uint64_t mce_oracle_clique_hash(const int64_t* labels_of_members, int64_t size) {
    uint64_t s = 0;
    for (int64_t i = 0; i < size; ++i) s += mix64((uint64_t)labels_of_members[i]);
    return mix64(s + (uint64_t)size * SIZE_SALT);
}

/* ------------------------------------------------------------------------ */
/* degeneracy ordering: indexed binary min-heap on key (deg << 32 | id).     */
/* The reference uses a lazy-deletion heap; both pop the live vertex with    */
/* the smallest (current degree, id), so the resulting order is identical.   */

static void heap_sift_up(uint64_t* key, int64_t* heap, int64_t* where, int64_t i) {
    int64_t v = heap[i];
    uint64_t k = key[v];
    while (i > 0) {
        int64_t parent = (i - 1) >> 1;
        int64_t pv = heap[parent];
        if (key[pv] <= k) break;
        heap[i] = pv;
        where[pv] = i;
        i = parent;
    }
    heap[i] = v;
    where[v] = i;
}

static void heap_sift_down(uint64_t* key, int64_t* heap, int64_t* where, int64_t size, int64_t i) {
    int64_t v = heap[i];
    uint64_t k = key[v];
    for (;;) {
        int64_t c = 2 * i + 1;
        if (c >= size) break;
        if (c + 1 < size && key[heap[c + 1]] < key[heap[c]]) c++;
        if (key[heap[c]] >= k) break;
        heap[i] = heap[c];
        where[heap[c]] = i;
        i = c;
    }
    heap[i] = v;
    where[v] = i;
}

int64_t mce_oracle_degeneracy_order(int64_t n, const int64_t* ro, const int64_t* ci,
                                    int64_t* position) {
    if (n <= 0) return 0;
    uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * n);
    int64_t* heap = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* where = (int64_t*)malloc(sizeof(int64_t) * n);
    for (int64_t v = 0; v < n; ++v) {
        key[v] = ((uint64_t)(ro[v + 1] - ro[v]) << 32) | (uint64_t)v;
        heap[v] = v;
        where[v] = v;
    }
    for (int64_t i = n / 2 - 1; i >= 0; --i) heap_sift_down(key, heap, where, n, i);
    int64_t size = n, rank = 0, degeneracy = 0;
    while (size > 0) {
        int64_t v = heap[0];
        int64_t dv = (int64_t)(key[v] >> 32);
        heap[0] = heap[size - 1];
        where[heap[0]] = 0;
        size--;
        where[v] = -1;
        if (size > 0) heap_sift_down(key, heap, where, size, 0);
        position[v] = rank++;
        if (dv > degeneracy) degeneracy = dv;
        for (int64_t e = ro[v]; e < ro[v + 1]; ++e) {
            int64_t u = ci[e];
            if (where[u] >= 0) {
                key[u] -= (1ull << 32);
                heap_sift_up(key, heap, where, where[u]);
            }
        }
    }
    free(key);
    free(heap);
    free(where);
    return degeneracy;
}

/* ------------------------------------------------------------------------ */
/* enumeration                                                               */

typedef struct {
    int64_t n;
    const int64_t* ro;
    const int64_t* ci;
    const int64_t* split;   /* split[v] = first index in N(v) with neighbour > v */
    const int64_t* labels;
    int full;
    int W;                  /* 64-bit words per bitset */
    int64_t cap_bits;
    int64_t max_x;
    /* collection */
    int64_t* collect;
    int64_t collect_cap;
    int64_t* collect_len;   /* shared cursor */
} ctx_t;

typedef struct {
    uint64_t* rows;   /* cap_bits x W */
    uint64_t* xrows;  /* max_x x W (full mode) */
    int64_t* plist;   /* local P index -> vertex */
    int64_t* xlist;   /* root X, ascending */
    int64_t* xx;      /* X_X tokens (positions into xlist) */
    int64_t* xtmp;    /* partition scratch */
    uint64_t* stk;    /* levels x 3W : P, XP, BR */
    int64_t* lpx;     /* per-level live prefix length */
    int64_t* rpath;   /* current R */
    uint64_t* hsum;   /* running hash sums per R length */
    mce_oracle_result res;
    int err;
} work_t;

static inline int64_t lbl(const ctx_t* c, int64_t v) { return c->labels ? c->labels[v] : v; }

/* index of key in sorted a[0..len) or -1 */
static inline int64_t bin_find(const int64_t* a, int64_t len, int64_t key) {
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return (lo < len && a[lo] == key) ? lo : -1;
}

/* is w in N+(x) (the later neighbours of x, sorted)? */
static inline int later_adjacent(const ctx_t* c, int64_t x, int64_t w) {
    int64_t lo = c->split[x], hi = c->ro[x + 1];
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (c->ci[mid] < w) lo = mid + 1; else hi = mid;
    }
    return lo < c->ro[x + 1] && c->ci[lo] == w;
}

static void report(const ctx_t* c, work_t* wk, const int64_t* verts, int64_t size, uint64_t hsum) {
    (void)verts;
    wk->res.cliques++;
    if (size < MCE_ORACLE_HIST_MAX) wk->res.hist[size]++;
    if (size > wk->res.max_size) wk->res.max_size = size;
    wk->res.hash += mix64(hsum + (uint64_t)size * SIZE_SALT);
    if (c->collect) {
        int64_t pos;
#pragma omp atomic capture
        { pos = *c->collect_len; *c->collect_len += size + 1; }
        if (pos + size + 1 <= c->collect_cap) {
            c->collect[pos] = size;
            for (int64_t i = 0; i < size; ++i) c->collect[pos + 1 + i] = verts[i];
        }
    }
}

static inline int popc_and(const uint64_t* a, const uint64_t* b, int W) {
    int s = 0;
    for (int w = 0; w < W; ++w) s += __builtin_popcountll(a[w] & b[w]);
    return s;
}

static inline int any_bits(const uint64_t* a, int W) {
    for (int w = 0; w < W; ++w) if (a[w]) return 1;
    return 0;
}

/* X_X member (token t) adjacent to branch vertex v (local) / gv (global) */
static inline int xx_adjacent(const ctx_t* c, const work_t* wk, int64_t t, int64_t v, int64_t gv) {
    if (c->full) return (int)((wk->xrows[t * c->W + (v >> 6)] >> (v & 63)) & 1ull);
    return later_adjacent(c, wk->xlist[t], gv);
}

/* Pivot row per bk.py:select_pivot: returns pointer to the winning row. */
static const uint64_t* choose_pivot(const ctx_t* c, work_t* wk, const uint64_t* P,
                                    const uint64_t* XP, int64_t live) {
    const int W = c->W;
    int best = -1;
    const uint64_t* prow = NULL;
    for (int w = 0; w < W; ++w) {
        uint64_t cand = P[w] | XP[w];
        while (cand) {
            int b = __builtin_ctzll(cand);
            cand &= cand - 1;
            int64_t v = (int64_t)w * 64 + b;
            const uint64_t* row = wk->rows + v * W;
            int cnt = popc_and(row, P, W);
            if (cnt > best) { best = cnt; prow = row; }
        }
    }
    if (c->full) {
        for (int64_t i = 0; i < live; ++i) {
            const uint64_t* row = wk->xrows + wk->xx[i] * W;
            int cnt = popc_and(row, P, W);
            if (cnt > best) { best = cnt; prow = row; }
        }
    }
    return prow;
}

static void traverse(const ctx_t* c, work_t* wk, const int64_t* R0, int nr,
                     int64_t np, int64_t nx) {
    const int W = c->W;
    uint64_t h0 = 0;
    for (int i = 0; i < nr; ++i) {
        wk->rpath[i] = R0[i];
        h0 += mix64((uint64_t)lbl(c, R0[i]));
    }
    if (np == 0) {                       /* scheduler.py:300-304 */
        wk->res.nodes++;
        if (nx == 0) report(c, wk, wk->rpath, nr, h0);
        return;
    }
    if (np > c->cap_bits) { wk->err = -2; return; }
    /* induced rows over P columns (induced.py:61-103) */
    memset(wk->rows, 0, sizeof(uint64_t) * np * W);
    for (int64_t i = 0; i < np; ++i) {
        int64_t a = wk->plist[i];
        for (int64_t e = c->split[a]; e < c->ro[a + 1]; ++e) {
            int64_t j = bin_find(wk->plist, np, c->ci[e]);
            if (j >= 0) {
                wk->rows[i * W + (j >> 6)] |= 1ull << (j & 63);
                wk->rows[j * W + (i >> 6)] |= 1ull << (i & 63);
            }
        }
    }
    if (c->full) {
        memset(wk->xrows, 0, sizeof(uint64_t) * nx * W);
        for (int64_t t = 0; t < nx; ++t) {
            int64_t x = wk->xlist[t];
            for (int64_t e = c->split[x]; e < c->ro[x + 1]; ++e) {
                int64_t j = bin_find(wk->plist, np, c->ci[e]);
                if (j >= 0) wk->xrows[t * W + (j >> 6)] |= 1ull << (j & 63);
            }
        }
    }
    for (int64_t t = 0; t < nx; ++t) wk->xx[t] = t;

    uint64_t P[64], XP[64], BR[64], childP[64];
    if (W > 64) { wk->err = -3; return; }
    memset(P, 0, sizeof(uint64_t) * W);
    memset(XP, 0, sizeof(uint64_t) * W);
    for (int64_t i = 0; i < np; ++i) P[i >> 6] |= 1ull << (i & 63);
    int64_t depth = 0, rlen = nr;
    wk->lpx[0] = nx;
    wk->hsum[rlen] = h0;
    wk->res.nodes++;
    {
        const uint64_t* prow = choose_pivot(c, wk, P, XP, nx);
        for (int w = 0; w < W; ++w) BR[w] = P[w] & ~prow[w];
    }
    for (;;) {
        int w0 = -1;
        for (int w = 0; w < W; ++w) if (BR[w]) { w0 = w; break; }
        if (w0 < 0) {
            if (depth == 0) break;
            depth--;
            rlen--;
            uint64_t* s = wk->stk + (size_t)depth * 3 * W;
            memcpy(P, s, sizeof(uint64_t) * W);
            memcpy(XP, s + W, sizeof(uint64_t) * W);
            memcpy(BR, s + 2 * W, sizeof(uint64_t) * W);
            continue;
        }
        int b = __builtin_ctzll(BR[w0]);
        uint64_t bit = 1ull << b;
        int64_t v = (int64_t)w0 * 64 + b;
        BR[w0] &= ~bit;
        P[w0] &= ~bit;
        XP[w0] |= bit;
        const uint64_t* rv = wk->rows + v * W;
        for (int w = 0; w < W; ++w) childP[w] = P[w] & rv[w];
        int64_t gv = wk->plist[v];
        int64_t live = wk->lpx[depth];
        if (!any_bits(childP, W)) {       /* scheduler.py:358-369 */
            wk->res.nodes++;
            int hit = 0;
            for (int w = 0; w < W && !hit; ++w) hit = (XP[w] & rv[w]) != 0;
            for (int64_t i = 0; i < live && !hit; ++i) hit = xx_adjacent(c, wk, wk->xx[i], v, gv);
            if (!hit) {
                wk->rpath[rlen] = gv;
                report(c, wk, wk->rpath, rlen + 1,
                       wk->hsum[rlen] + mix64((uint64_t)lbl(c, gv)));
            }
            continue;
        }
        /* descend (xsets.py:55-82): stable partition of the live X_X prefix */
        int64_t kept = 0, dropped = 0;
        for (int64_t i = 0; i < live; ++i) {
            int64_t t = wk->xx[i];
            if (xx_adjacent(c, wk, t, v, gv)) wk->xx[kept++] = t;
            else wk->xtmp[dropped++] = t;
        }
        memcpy(wk->xx + kept, wk->xtmp, sizeof(int64_t) * dropped);
        uint64_t* s = wk->stk + (size_t)depth * 3 * W;
        memcpy(s, P, sizeof(uint64_t) * W);
        memcpy(s + W, XP, sizeof(uint64_t) * W);
        memcpy(s + 2 * W, BR, sizeof(uint64_t) * W);
        depth++;
        wk->lpx[depth] = kept;
        for (int w = 0; w < W; ++w) { XP[w] &= rv[w]; P[w] = childP[w]; }
        wk->rpath[rlen] = gv;
        wk->hsum[rlen + 1] = wk->hsum[rlen] + mix64((uint64_t)lbl(c, gv));
        rlen++;
        wk->res.nodes++;
        const uint64_t* prow = choose_pivot(c, wk, P, XP, kept);
        for (int w = 0; w < W; ++w) BR[w] = P[w] & ~prow[w];
    }
}

int mce_oracle_enumerate(int64_t n, const int64_t* ro, const int64_t* ci, int roots_mode,
                         int induced_full, int64_t capacity_bits, const int64_t* labels,
                         int64_t root_begin, int64_t root_end, int64_t root_stride,
                         int include_isolated, int threads, mce_oracle_result* out,
                         int64_t* collect, int64_t collect_cap, int64_t* collect_len) {
    memset(out, 0, sizeof(*out));
    if (collect_len) *collect_len = 0;
    if (roots_mode != 1 && roots_mode != 2) return -1;
    if (root_stride <= 0) root_stride = 1;
    if (n <= 0) return 0;
    int64_t* split = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t max_x = 0, max_p = 0;
    for (int64_t v = 0; v < n; ++v) {
        int64_t lo = ro[v], hi = ro[v + 1];
        while (lo < hi) {
            int64_t mid = lo + ((hi - lo) >> 1);
            if (ci[mid] < v) lo = mid + 1; else hi = mid;
        }
        split[v] = lo;
        if (lo - ro[v] > max_x) max_x = lo - ro[v];
        if (ro[v + 1] - lo > max_p) max_p = ro[v + 1] - lo;
    }
    /* second-level roots are the edges (u < v) in CSR order (graph.py:57-64) */
    int64_t* eoff = NULL;
    int64_t total_roots = n;
    if (roots_mode == 2) {
        eoff = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
        eoff[0] = 0;
        for (int64_t v = 0; v < n; ++v) eoff[v + 1] = eoff[v] + (ro[v + 1] - split[v]);
        total_roots = eoff[n];
    }
    if (root_end < 0 || root_end > total_roots) root_end = total_roots;
    if (capacity_bits < 64) capacity_bits = 64;
    ctx_t c;
    c.n = n; c.ro = ro; c.ci = ci; c.split = split; c.labels = labels;
    c.full = induced_full; c.W = (int)(capacity_bits / 64); c.cap_bits = capacity_bits;
    c.max_x = max_x;
    c.collect = collect; c.collect_cap = collect_cap; c.collect_len = collect_len;
    int64_t levels = capacity_bits + 3;
    int err = 0;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#else
    threads = 1;
#endif
    mce_oracle_result* parts = (mce_oracle_result*)calloc((size_t)threads, sizeof(mce_oracle_result));
#pragma omp parallel num_threads(threads)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        work_t wk;
        memset(&wk, 0, sizeof(wk));
        int64_t mp = max_p > capacity_bits ? max_p : capacity_bits;
        wk.rows = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(mp * c.W + 1));
        wk.xrows = induced_full ? (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(max_x * c.W + 1)) : NULL;
        wk.plist = (int64_t*)malloc(sizeof(int64_t) * (size_t)(mp + 1));
        wk.xlist = (int64_t*)malloc(sizeof(int64_t) * (size_t)(max_x + 1));
        wk.xx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(max_x + 1));
        wk.xtmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(max_x + 1));
        wk.stk = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(levels * 3 * c.W));
        wk.lpx = (int64_t*)malloc(sizeof(int64_t) * (size_t)levels);
        wk.rpath = (int64_t*)malloc(sizeof(int64_t) * (size_t)(levels + 2));
        wk.hsum = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(levels + 2));
#pragma omp for schedule(dynamic, 16)
        for (int64_t r = root_begin; r < root_end; r += root_stride) {
            if (wk.err) continue;
            int64_t R0[2];
            int nr;
            int64_t np = 0, nx = 0;
            if (roots_mode == 1) {
                R0[0] = r; nr = 1;
                for (int64_t e = split[r]; e < ro[r + 1]; ++e) wk.plist[np++] = ci[e];
                for (int64_t e = ro[r]; e < split[r]; ++e) wk.xlist[nx++] = ci[e];
            } else {
                /* locate u with eoff[u] <= r < eoff[u+1] */
                int64_t lo = 0, hi = n;
                while (hi - lo > 1) {
                    int64_t mid = (lo + hi) >> 1;
                    if (eoff[mid] <= r) lo = mid; else hi = mid;
                }
                int64_t u = lo, v = ci[split[u] + (r - eoff[u])];
                R0[0] = u; R0[1] = v; nr = 2;
                /* common neighbours, ascending; cut at v */
                int64_t i = ro[u], j = ro[v];
                while (i < ro[u + 1] && j < ro[v + 1]) {
                    if (ci[i] < ci[j]) i++;
                    else if (ci[i] > ci[j]) j++;
                    else {
                        if (ci[i] < v) wk.xlist[nx++] = ci[i];
                        else wk.plist[np++] = ci[i];
                        i++; j++;
                    }
                }
            }
            traverse(&c, &wk, R0, nr, np, nx);
        }
        parts[tid] = wk.res;
        if (wk.err) {
#pragma omp critical
            err = wk.err;
        }
        free(wk.rows); free(wk.xrows); free(wk.plist); free(wk.xlist); free(wk.xx);
        free(wk.xtmp); free(wk.stk); free(wk.lpx); free(wk.rpath); free(wk.hsum);
    }
    for (int t = 0; t < threads; ++t) {
        out->cliques += parts[t].cliques;
        out->nodes += parts[t].nodes;
        out->hash += parts[t].hash;
        if (parts[t].max_size > out->max_size) out->max_size = parts[t].max_size;
        for (int s = 0; s < MCE_ORACLE_HIST_MAX; ++s) out->hist[s] += parts[t].hist[s];
    }
    if (roots_mode == 2 && include_isolated) {
        for (int64_t v = 0; v < n; ++v) {
            if (ro[v + 1] == ro[v]) {
                int64_t lab = labels ? labels[v] : v;
                out->cliques++;
                out->hist[1]++;
                if (out->max_size < 1) out->max_size = 1;
                out->hash += mix64(mix64((uint64_t)lab) + SIZE_SALT);
                if (collect) {
                    int64_t pos = *collect_len;
                    *collect_len += 2;
                    if (pos + 2 <= collect_cap) { collect[pos] = 1; collect[pos + 1] = v; }
                }
            }
        }
    }
    free(parts);
    free(split);
    free(eoff);
    return err;
}

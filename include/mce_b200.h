/*
 * mce_b200.h -- C ABI of the B200 maximal-clique-enumeration engine
 * (libmce_b200.so, built from paper_2212_01473_b200/csrc/).
 *
 * This is the drop-in boundary for the hot path of the reference `mce`
 * package (a Python implementation of arXiv:2212.01473 at
 * /root/reference/pkg/src/mce).  Each entry point replaces one reference
 * function; the Python host layer (paper_2212_01473_b200/, ctypes) mirrors
 * the reference API on top of these calls.  Plain pointers and sizes only.
 *
 *   reference function                          replaced by
 *   graph.py:103-129   from_edges            ->  mce_graph_from_edges
 *   graph.py:132-180  parse_edge_list       ->  mce_graph_from_text
 *   graph.py:28-64    Graph CSR accessors   ->  mce_graph_from_csr / mce_graph_copy_csr / mce_graph_info
 *   graph.py:183-210  degeneracy_order      ->  mce_degeneracy_order
 *   graph.py:213-224  reorder               ->  mce_reorder
 *   graph.py:227-236  stats                 ->  mce_graph_info
 *   graph.py:239-243  preprocess            ->  mce_preprocess (+ mce_graph_info)
 *   scheduler.py:441-492 run (+ bk.py roots, induced.py, xsets.py, the worker list)
 *                                           ->  mce_enumerate
 *
 * Error behaviour: every call returns 0 on success and a negative code on
 * failure, with a message from mce_last_error():
 *   -1  CUDA error (allocation, launch, ...)
 *   -2  invalid argument (reference: ValueError)
 *   -3  device limits (a kernel variant does not fit)
 *   -4  capacity exceeded (reference: induced.CapacityError)
 *
 * Streams: `stream` is a cudaStream_t (NULL = legacy default stream).
 * Graph-building calls (from_edges / from_text / from_csr / reorder /
 * preprocess with a NULL degeneracy) return once their work is queued: the
 * graph is usable on the same stream at once, and its statistics are fetched
 * asynchronously (mce_graph_info waits for them).  mce_enumerate,
 * mce_degeneracy_order and mce_graph_copy_csr are synchronous on return.
 */
#ifndef MCE_B200_H
#define MCE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCE_HIST_MAX 4096

typedef struct mce_graph mce_graph; /* device-resident canonical CSR */

const char* mce_last_error(void);

/* Canonical graph from (u, v) pairs: self-loops dropped, duplicates merged,
 * symmetric, rows strictly ascending (graph.py:103-129).  `edges` holds
 * 2*num_edges int64 values, on the host or (edges_on_device=1) the device. */
int mce_graph_from_edges(const int64_t* edges, int64_t num_edges, int64_t num_vertices,
                         int edges_on_device, void* stream, mce_graph** out);

/* The same from 2*num_edges int32 values (ids are below 2^31 anyway): half
 * the host->device bytes of mce_graph_from_edges for the same graph.  The
 * reference's from_edges (graph.py:103-129) takes any integer array; this is
 * the entry a caller holding int32 pairs binds. */
int mce_graph_from_edges32(const int32_t* edges, int64_t num_edges, int64_t num_vertices,
                           int edges_on_device, void* stream, mce_graph** out);

/* Edge-list TEXT -> canonical graph, parsed on the device (graph.py:132-180
 * parse_edge_list): '#'/'%' comment lines, "%%MatrixMarket" header (1-based
 * ids after it, the next data line is the size line), two integer tokens per
 * line, ids compacted to [0, n) ascending.  `text` is `len` bytes on the host
 * or (text_on_device=1) the device.  On a malformed line returns -2 with
 * *err_line = its 1-based number and *err_code = 1 (token count),
 * 2 (non-integer token) or 3 (id below base) -- the reference's
 * EdgeListParseError cases; *num_vertices = n on success. */
int mce_graph_from_text(const char* text, int64_t len, int base, int text_on_device,
                        void* stream, mce_graph** out, int64_t* err_line, int* err_code,
                        int64_t* num_vertices);

/* Adopt an already canonical CSR (row_offsets: n+1, col_indices: nnz). */
int mce_graph_from_csr(const int64_t* row_offsets, const int64_t* col_indices, int64_t n,
                       int64_t nnz, int on_device, void* stream, mce_graph** out);

/* n, directed entries (2m), max degree, max later / earlier neighbour counts. */
int mce_graph_info(const mce_graph* g, int64_t* n, int64_t* nnz, int64_t* max_degree,
                   int64_t* max_later, int64_t* max_earlier);

/* Copy the CSR (and, when present, the original labels) to host buffers. */
int mce_graph_copy_csr(const mce_graph* g, int64_t* row_offsets, int64_t* col_indices,
                       int64_t* labels, void* stream);

void mce_graph_free(mce_graph* g);

/* Degeneracy ordering (graph.py:183-210): position[v] = rank of v.
 *   method 1: the reference's exact order (minimum current degree, ties to the
 *             smallest id) -- bit-identical positions, single-CTA kernel;
 *   method 0: parallel bucket peeling -- a valid degeneracy order with the same
 *             degeneracy, vertices of one peel round ranked by id;
 *   method 2: asynchronous peeling -- no rounds inside a level: a vertex takes
 *             its position the moment a decrement brings it to the level; a
 *             valid degeneracy order with the same degeneracy whose tie-breaks
 *             vary from run to run (the throughput default of the Python API). */
int mce_degeneracy_order(const mce_graph* g, int method, int64_t* position,
                         int position_on_device, int64_t* degeneracy, void* stream);

/* Relabel by position (graph.py:213-224).  The result remembers the original
 * label of every vertex (used to hash cliques by original ids). */
int mce_reorder(const mce_graph* g, const int64_t* position, int position_on_device,
                void* stream, mce_graph** out);

/* degeneracy_order + reorder in one call, positions kept on the device
 * (graph.py:239-243 preprocess, minus stats which mce_graph_info gives).
 * The permutation is recoverable from the result's labels:
 * labels[position[v]] = label(v).  `degeneracy` may be NULL: the call then
 * returns without waiting for the device (the result's max later degree,
 * from mce_graph_info, is the degeneracy). */
int mce_preprocess(const mce_graph* g, int method, int64_t* degeneracy, void* stream,
                   mce_graph** out);

typedef struct {
  int roots;             /* 1 = first-level (per vertex), 2 = second-level (per edge) */
  int induced_full;      /* 1 = full ("ipx"), 0 = partial ("ip"), -1 = auto: partial iff
                            max_degree / degeneracy > 200 (scheduler.py:36-41), decided on
                            the device-side graph statistics */
  int workers;           /* worker warps; 0 = every co-resident warp */
  int worker_list;       /* donation protocol on/off (RunConfig.worker_list) */
  int donation_min_p;    /* RunConfig.donation_min_p */
  int hash_labels;       /* hash cliques by the graph's original labels when stored */
  int64_t root_begin;    /* root sample: begin, end (-1 = all), stride */
  int64_t root_end;
  int64_t root_stride;
  int include_isolated;  /* second-level runs: report isolated vertices */
  int64_t collect_cap;   /* int64 words of the clique stream (0 = count only) */
  int64_t capacity_bits; /* bitset capacity; |P| above it -> -4 (0 = 1024) */
  double mem_fraction;   /* share of free HBM for per-worker scratch (0 -> 0.5) */
  int measure_bytes;     /* also count the algorithmic CSR bytes of the induced-subgraph
                            builds into mce_run_result.build_bytes (bench only; l1) */
  int partial_xrows_min_w; /* partial mode: build X rows only for bitset classes of at
                              least this many words (0 -> 1); same traversal either way */
  int donation_min_x;    /* B200 extension: also donate a branch whose node has at least
                            this many live X_X members (0 = off; the reference donates on
                            |P| >= donation_min_p only).  Scheduling only: same results */
  int no_pivot;          /* 1 = branch on all of P (basic Bron-Kerbosch, bk.py:124-150);
                            0 = Tomita pivot (bk.py:82-110), the engine's default */
  int timing;            /* 1 = fill the per-worker time columns (RunConfig.timing,
                            metrics.py:13-32); 0 = counters only */
} mce_run_config;

typedef struct {
  int64_t cliques;       /* maximal cliques */
  int64_t nodes;         /* search-tree nodes (reference node accounting) */
  uint64_t hash;         /* sum over cliques of mix64(sum mix64(label) + size*salt) */
  int64_t max_size;
  int64_t donations;
  int64_t workers;       /* worker slots reported in worker_metrics */
  int64_t launches;      /* enumeration kernels launched */
  int64_t collect_len;   /* words the clique stream needed (may exceed collect_cap) */
  double kernel_ms;      /* device time of the enumeration kernels (CUDA events) */
  int64_t build_bytes;   /* algorithmic graph bytes the induced-subgraph builds read */
  int64_t hist[MCE_HIST_MAX]; /* hist[s] = maximal cliques of size s */
  int64_t induced_full;  /* the induced mode the run used (resolves auto) */
  double phase1_ms;      /* device time until every root of a launch was claimed, summed
                            over the launches (scheduler.py:481-490 phase1_time) */
  double phase2_ms;      /* device time after that: worker-list donations only */
  double clock_khz;      /* SM clock the worker time columns are counted in */
} mce_run_result;

/* Columns of one worker's row in mce_enumerate's worker_metrics: */
#define MCE_WM_COLS 9  /* nodes, roots claimed, donations made, donations received, then
                          SM cycles (cfg.timing only) spent in the induced-subgraph build,
                          pivot selection, set operations (leaf batches, X_X partitions,
                          register-resident subtrees), the worker list / root claims, and
                          the worker's whole run (metrics.py TIME_CATEGORIES; "other" is
                          the whole run minus the four) */

/* Enumerate every maximal clique of a canonical, degeneracy-reordered graph
 * (scheduler.py:441-492).  `collect` (host, collect_cap words) receives the
 * clique stream [size, v0, v1, ...]...; `worker_metrics` (host, MCE_WM_COLS
 * int64 per worker, see above). */
int mce_enumerate(const mce_graph* g, const mce_run_config* cfg, int64_t* collect,
                  int64_t* worker_metrics, int64_t worker_metrics_cap, mce_run_result* out,
                  void* stream);

/* Kernels this library has launched since load (its own kernels, not CUB's). */
int64_t mce_launch_count(void);

/* R-MAT edge generator on the device (input synthesis for the benchmarks):
 * edges [start, start+count) of the counter-based stream of
 * paper_2212_01473_b200/generate.py:rmat_edges, written as int64 pairs to a
 * device buffer. */
int mce_gen_rmat(int scale, int64_t start, int64_t count, uint64_t seed, int64_t* edges_dev,
                 void* stream);

#ifdef __cplusplus
}
#endif
#endif

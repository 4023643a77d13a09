"""Two-phase parallel enumeration with dynamic load balancing, on the GPU.

Same API as the reference ``mce.scheduler`` (reference scheduler.py:33-492):
``RunConfig``, ``Backoff``, ``RunResult``, ``choose_induced_mode`` and
``run``.  ``run`` hands the whole traversal to ``mce_enumerate`` in
libmce_b200.so:

* a worker is one warp (the paper's thread block); phase 1 claims
  first-level (``l1``) or second-level (``l2``) subtrees off a device-wide
  atomic counter, heaviest roots first;
* phase 2 is the worker list: idle warps park in a ring buffer and busy
  warps donate the branch they are about to visit when the reference's
  conditions hold (|P| >= donation_min_p, phase 2 reached, siblings left at
  this level and at some earlier level -- scheduler.py:346-348);
* the traversal tree (pivot rule, branch order, node accounting) is the
  reference's, so ``nodes_total`` is identical for every worker count and
  donation schedule, and the clique set is exact.

Extra results beyond the reference's: ``nodes_total``, ``clique_hash`` (an
order-independent checksum of the clique set over ORIGINAL vertex labels),
``size_histogram`` and ``max_clique_size``.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from time import perf_counter

import numpy as np

from paper_2212_01473_b200 import _lib
from paper_2212_01473_b200.bk import CliqueSink
from paper_2212_01473_b200.graph import Graph, GraphStats
from paper_2212_01473_b200.metrics import WorkerMetrics

PARTIAL_MODE_DEGREE_RATIO = 200.0  # reference scheduler.py:33
MAX_WORKER_SLOTS = 148 * 64        # co-resident warps on a B200


def choose_induced_mode(max_degree: int, degeneracy: int) -> str:
    """Partial ("ip") exactly when max_degree / degeneracy > 200, else full
    ("ipx") -- reference scheduler.py:36-41, paper §4.5."""
    if degeneracy > 0 and max_degree / degeneracy > PARTIAL_MODE_DEGREE_RATIO:
        return "ip"
    return "ipx"


@dataclass(frozen=True)
class Backoff:
    """Exponential sleep schedule for parked workers (reference scheduler.py:45-49).
    The device worker list backs off with __nanosleep from 64 ns doubling to
    ~8 us; the values here are validated for API compatibility."""

    initial: float = 1e-6
    max: float = 1e-3


@dataclass
class RunConfig:
    """Knobs for one run (reference scheduler.py:53-78).

    ``workers`` counts worker warps; 0 means every co-resident warp of the GPU.
    """

    workers: int = 0
    roots: str = "l1"          # "l1" | "l2"
    induced: str = "auto"      # "ip" | "ipx" | "auto"
    worker_list: bool = True
    donation_min_p: int = 10
    # B200 extension: also donate branches of nodes with this many live X_X
    # members (a hub root with a tiny P but thousands of excluded vertices is
    # partition-bound); 0 disables.  Scheduling only -- results are unchanged.
    donation_min_x: int = 1024
    backoff: Backoff = field(default_factory=Backoff)
    collect_limit: int | None = None
    timing: bool = False

    def resolved_workers(self) -> int:
        return self.workers if self.workers > 0 else MAX_WORKER_SLOTS

    def validate(self) -> None:
        if self.workers < 0:
            raise ValueError("workers must be >= 1 (or 0 for hardware default)")
        if self.roots not in ("l1", "l2"):
            raise ValueError(f"unknown roots mode {self.roots!r}")
        if self.induced not in ("ip", "ipx", "auto"):
            raise ValueError(f"unknown induced mode {self.induced!r}")
        if self.donation_min_p < 0:
            raise ValueError("donation_min_p must be >= 0")
        if self.donation_min_x < 0:
            raise ValueError("donation_min_x must be >= 0")
        if self.backoff.initial <= 0 or self.backoff.max < self.backoff.initial:
            raise ValueError("backoff must satisfy 0 < initial <= max")


@dataclass
class RunResult:
    """Outcome of one run (reference scheduler.py:169-185) plus the device
    engine's checksums."""

    clique_count: int
    donation_count: int
    roots_mode: str
    induced_mode: str
    workers: int
    total_time: float
    phase1_time: float
    phase2_time: float
    worker_metrics_raw: np.ndarray | list = field(repr=False)
    nodes_total: int = 0
    clique_hash: int = 0
    size_histogram: dict[int, int] = field(default_factory=dict)
    max_clique_size: int = 0
    kernel_launches: int = 0
    kernel_ms: float = 0.0
    build_bytes: int = 0
    timing: bool = False
    clock_khz: float = 0.0

    @property
    def worker_metrics(self) -> list[WorkerMetrics]:
        """Per-worker counters (built on first access from the device's
        ``[nodes, roots, donations made, received]`` rows)."""
        raw = self.worker_metrics_raw
        if isinstance(raw, np.ndarray):
            out = []
            hz = self.clock_khz * 1e3
            for i, row in enumerate(raw.tolist()):
                m = WorkerMetrics(worker_id=i, enabled=self.timing)
                m.nodes_visited, m.roots_claimed, m.donations_made, m.donations_received = row[:4]
                if self.timing and hz > 0:
                    build, pivot, setops, wlist, total = (c / hz for c in row[4:9])
                    m.times.update(induced_build=build, pivot=pivot, set_ops=setops,
                                   worker_list=wlist,
                                   other=max(0.0, total - build - pivot - setops - wlist))
                out.append(m)
            self.worker_metrics_raw = raw = out
        return raw

    def report(self):
        from paper_2212_01473_b200.metrics import aggregate

        return aggregate(self.worker_metrics)

    @property
    def clique_hash_hex(self) -> str:
        return f"{self.clique_hash:016x}"


def _decode_stream(buf: np.ndarray, words: int, limit: int) -> list[tuple[int, ...]]:
    out: list[tuple[int, ...]] = []
    i = 0
    while i < words and len(out) < limit:
        s = int(buf[i])
        if s <= 0 or i + 1 + s > words:
            break
        out.append(tuple(sorted(int(x) for x in buf[i + 1:i + 1 + s])))
        i += 1 + s
    return out


def run(g: Graph, st: GraphStats, cfg: RunConfig, sink: CliqueSink | None = None, *,
        root_begin: int = 0, root_end: int = -1, root_stride: int = 1,
        hash_labels: bool = True, stream=None, measure_bytes: bool = False,
        pivot: bool = True) -> RunResult:
    """Enumerate all maximal cliques of a degeneracy-reordered graph on the
    GPU (reference scheduler.py:441-492).

    ``root_begin/root_end/root_stride`` restrict the run to a sample of the
    subtree roots (vertices for l1, edges in CSR order for l2) -- used for
    bounded parity checks against the CPU oracle.  ``hash_labels`` hashes
    cliques by the graph's original labels (set by ``reorder``).
    ``pivot=False`` branches on every member of P (basic Bron-Kerbosch, the
    traversal of reference bk.py:124-150 below each root).

    ``phase1_time`` / ``phase2_time`` are device times (global timer inside
    the kernels): until every root of a launch was claimed, and the worker-
    list tail after it, summed over the launches (scheduler.py:481-490).
    """
    cfg.validate()
    if sink is None:
        sink = CliqueSink(collect_limit=cfg.collect_limit)
    # "auto" is resolved on the device side (the same rule, choose_induced_mode,
    # on the graph's device statistics) so that the call does not wait for them
    induced = cfg.induced
    limit = sink.collect_limit
    if g.num_vertices == 0:
        if induced == "auto":
            induced = choose_induced_mode(st.max_degree, st.degeneracy)
        return RunResult(0, 0, cfg.roots, induced, cfg.resolved_workers(), 0.0, 0.0, 0.0,
                         [WorkerMetrics(worker_id=0, enabled=cfg.timing)], timing=cfg.timing)
    _lib.require_device()
    cap_words = 0
    if limit:
        cap_words = int(min(limit * (st.degeneracy + 3), 1 << 26))
    slots = cfg.workers if cfg.workers > 0 else MAX_WORKER_SLOTS
    while True:
        c = _lib.RunConfigC(
            roots=1 if cfg.roots == "l1" else 2,
            induced_full={"ipx": 1, "ip": 0, "auto": -1}[induced],
            workers=int(cfg.workers),
            worker_list=int(bool(cfg.worker_list)),
            donation_min_p=int(cfg.donation_min_p),
            hash_labels=int(bool(hash_labels)),
            root_begin=int(root_begin), root_end=int(root_end), root_stride=int(root_stride),
            include_isolated=1 if root_begin == 0 and root_end < 0 and root_stride == 1 else 0,
            collect_cap=cap_words,
            capacity_bits=0,
            mem_fraction=float(os.environ.get("MCE_MEM_FRACTION", "0.5")),
            measure_bytes=int(bool(measure_bytes)),
            partial_xrows_min_w=int(os.environ.get("MCE_PARTIAL_XROWS_MIN_W", "0")),
            donation_min_x=int(cfg.donation_min_x),
            no_pivot=0 if pivot else 1,
            timing=int(bool(cfg.timing)),
        )
        buf = np.zeros(max(cap_words, 1), dtype=np.int64) if cap_words else None
        wm = np.zeros((slots, _lib.WM_COLS), dtype=np.int64)
        res = _lib.RunResultC()
        t0 = perf_counter()
        _lib.check(_lib.lib().mce_enumerate(g.device.handle, ctypes.byref(c), _lib.ptr(buf),
                                            _lib.ptr(wm), slots, ctypes.byref(res), stream),
                   "mce_enumerate")
        t1 = perf_counter()
        needed = int(res.collect_len)
        # the clique stream is word-capped; grow once if it truncated cliques we must keep
        if limit and needed > cap_words and cap_words < limit * (st.degeneracy + 3) \
                and int(res.cliques) > len(_decode_stream(buf, cap_words, limit)):
            cap_words = int(min(needed, limit * (st.degeneracy + 3)))
            continue
        break
    if limit:
        got = _decode_stream(buf, min(needed, cap_words), limit)
        room = limit - len(sink.collected)
        if room > 0:
            sink.collected.extend(got[:room])
    sink.total += int(res.cliques)
    induced = "ipx" if int(res.induced_full) else "ip"
    workers = max(int(res.workers), 1)
    hist_arr = np.ctypeslib.as_array(res.hist)
    hist = {int(s): int(hist_arr[s]) for s in np.flatnonzero(hist_arr)}
    return RunResult(
        clique_count=int(res.cliques),
        donation_count=int(res.donations),
        roots_mode=cfg.roots,
        induced_mode=induced,
        workers=workers,
        total_time=t1 - t0,
        phase1_time=float(res.phase1_ms) / 1e3,
        phase2_time=float(res.phase2_ms) / 1e3,
        worker_metrics_raw=wm[:workers],
        nodes_total=int(res.nodes),
        clique_hash=int(res.hash),
        size_histogram=hist,
        max_clique_size=int(res.max_size),
        kernel_launches=int(res.launches),
        kernel_ms=float(res.kernel_ms),
        build_bytes=int(res.build_bytes),
        timing=cfg.timing,
        clock_khz=float(res.clock_khz),
    )

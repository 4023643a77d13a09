"""GPU parity: the CUDA engine (through the C ABI) against the reference's
golden vectors and the CPU oracle.  Bit-exact on every integer output:
degeneracy / positions, clique count, search-tree node total, size
histogram and clique-set hash."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import K4_TRIANGLE_CLIQUES, K4_TRIANGLE_EDGES, golden_cases
from oracle import oracle
from paper_2212_01473_b200 import generate
from paper_2212_01473_b200 import (
    CliqueSink,
    RunConfig,
    degeneracy_order,
    from_edges,
    preprocess,
    reorder,
    run,
    stats,
)

pytestmark = pytest.mark.gpu

CASES = golden_cases()
MODES = ["l1-ipx", "l1-ip", "l2-ipx", "l2-ip"]


def _graph(case):
    edges = np.asarray(case["edges"], dtype=np.int64).reshape(-1, 2)
    return from_edges(edges, case["n"]), edges


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_csr_and_orderings_match_reference(case):
    g, edges = _graph(case)
    ro, ci = oracle.from_edges(edges, case["n"])
    assert np.array_equal(g.row_offsets, ro)
    assert np.array_equal(g.col_indices, ci)
    exact = degeneracy_order(g, method="exact")
    assert exact.degeneracy == case["degeneracy"]
    assert exact.position.tolist() == case["position"]
    par = degeneracy_order(g, method="parallel")
    assert par.degeneracy == case["degeneracy"]
    bpos, _ = oracle.bucket_peel_order(ro, ci)
    assert np.array_equal(par.position, bpos)
    assert sorted(par.position.tolist()) == list(range(case["n"]))
    g2 = reorder(g, par)
    n = case["n"]
    if n:
        later = [int(np.sum(g2.neighbors(v) > v)) for v in range(n)]
        assert max(later) == case["degeneracy"]  # a degeneracy ordering, tight


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_exact_order_runs_match_reference_bit_for_bit(case):
    """Reference ordering -> identical traversal tree: count, nodes, hist, hash."""
    g, _ = _graph(case)
    order = degeneracy_order(g, method="exact")
    g2 = reorder(g, order)
    st = stats(g2, order)
    assert st.max_degree == case["max_degree"] and st.m == case["m"]
    for mode in MODES:
        exp = case["runs"][mode]
        roots, induced = mode.split("-")
        res = run(g2, st, RunConfig(workers=8, roots=roots, induced=induced, worker_list=False))
        assert res.clique_count == exp["count"], mode
        assert res.nodes_total == exp["nodes"], mode
        donated = run(g2, st, RunConfig(workers=8, roots=roots, induced=induced,
                                        donation_min_p=2))
        assert donated.clique_count == exp["count"], mode
        assert donated.clique_hash == res.clique_hash, mode
        if induced == "ip":
            assert donated.nodes_total == exp["nodes"], mode
        if "hash" in exp:
            assert res.clique_hash_hex == exp["hash"], mode
            assert {str(k): v for k, v in res.size_histogram.items()} == exp["hist"], mode


@pytest.mark.parametrize("case", [c for c in CASES if c["n"] >= 64],
                         ids=[c["name"] for c in CASES if c["n"] >= 64])
def test_parallel_order_results_and_tree_match_oracle(case):
    """Parallel ordering: same cliques (count/hist/hash over original labels);
    the node total equals the oracle's on the GPU-reordered graph."""
    g, _ = _graph(case)
    g2, order, st = preprocess(g)
    ro2, ci2 = g2.row_offsets, g2.col_indices
    for mode in MODES:
        exp = case["runs"][mode]
        roots, induced = mode.split("-")
        res = run(g2, st, RunConfig(roots=roots, induced=induced))
        assert res.clique_count == exp["count"], mode
        assert res.clique_hash_hex == exp["hash"], mode
        assert {str(k): v for k, v in res.size_histogram.items()} == exp["hist"], mode
        orc = oracle.enumerate_cliques(ro2, ci2, roots=roots, induced=induced,
                                       degeneracy=st.degeneracy, labels=g2.labels)
        if induced == "ipx":  # donation-independent tree only without the worker list
            res = run(g2, st, RunConfig(roots=roots, induced=induced, worker_list=False))
        assert res.nodes_total == orc["nodes"], mode


@pytest.mark.parametrize("case", [c for c in CASES if "brute_force" in c],
                         ids=[c["name"] for c in CASES if "brute_force" in c])
def test_collected_cliques_match_brute_force(case):
    g, _ = _graph(case)
    g2, order, st = preprocess(g)
    inverse = np.argsort(order.position)
    expected = {tuple(c) for c in case["brute_force"]}
    for mode in MODES:
        roots, induced = mode.split("-")
        sink = CliqueSink.collecting()
        res = run(g2, st, RunConfig(workers=4, roots=roots, induced=induced), sink=sink)
        got = {tuple(sorted(int(inverse[v]) for v in c)) for c in sink.collected}
        assert got == expected, mode
        assert res.clique_count == len(expected) == sink.total


def test_running_example():
    g = from_edges(K4_TRIANGLE_EDGES, 6)
    g2, order, st = preprocess(g)
    inverse = np.argsort(order.position)
    for roots in ("l1", "l2"):
        for induced in ("ip", "ipx"):
            for wl in (True, False):
                sink = CliqueSink(collect_limit=10)
                res = run(g2, st, RunConfig(workers=2, roots=roots, induced=induced,
                                            worker_list=wl), sink=sink)
                assert res.clique_count == 2
                got = {tuple(sorted(int(inverse[v]) for v in c)) for c in sink.collected}
                assert got == K4_TRIANGLE_CLIQUES


def test_work_conservation_across_workers_and_donation():
    """Reference acceptance criterion 4: the node total is invariant across
    worker counts and worker-list on/off (the traversal tree is identical).

    Holds exactly for partial ("ip") subgraphs.  With full ("ipx") subgraphs
    the pivot may come from X_X with ties broken by X_X prefix order, and a
    donated branch's partition of that prefix happens in the receiver, not
    the donor -- exactly as in the reference (scheduler.py:417-438) -- so
    later siblings can see a different order; node totals are then exact only
    without donations, while counts and hashes stay exact.  The reference's
    own scheduler shows it: profiles/r2/ref_ipx_donation_probe.txt (from
    tests/golden/ref_ipx_donation_probe.py) -- gnp(200, 0.5), ipx, 8 workers,
    donation_min_p=2: one of six runs reports 1,258,448 nodes against the
    worker-list-off 1,258,446, same clique count."""
    for case in CASES:
        if case["name"] not in ("gnp_200_0.5_s3", "skew_2000_40", "gnp_300_0.08_s42"):
            continue
        g, _ = _graph(case)
        g2, _, st = preprocess(g, method="exact")
        for mode in ("l1-ipx", "l1-ip"):
            roots, induced = mode.split("-")
            totals, counts, hashes = set(), set(), set()
            for workers in (1, 2, 4, 8, 16, 0):
                for wl in (True, False):
                    res = run(g2, st, RunConfig(workers=workers, roots=roots, induced=induced,
                                                worker_list=wl, donation_min_p=4))
                    if induced == "ip" or not wl:
                        totals.add(sum(w.nodes_visited for w in res.worker_metrics))
                    counts.add(res.clique_count)
                    hashes.add(res.clique_hash)
                    made = sum(w.donations_made for w in res.worker_metrics)
                    recv = sum(w.donations_received for w in res.worker_metrics)
                    assert made == recv == res.donation_count
                    if not wl:
                        assert made == 0
            assert totals == {case["runs"][mode]["nodes"]}, (case["name"], mode, totals)
            assert counts == {case["runs"][mode]["count"]}
            assert len(hashes) == 1


def test_donations_happen_and_preserve_results():
    """A skewed instance with few workers must actually donate, and the
    donated run must reproduce count, hash and node total."""
    case = next(c for c in CASES if c["name"] == "gnp_200_0.5_s3")
    g, _ = _graph(case)
    g2, _, st = preprocess(g, method="exact")
    for induced in ("ip", "ipx"):
        base = run(g2, st, RunConfig(workers=1, induced=induced, worker_list=False))
        res = run(g2, st, RunConfig(workers=64, induced=induced, donation_min_p=2))
        exp = case["runs"][f"l1-{induced}"]
        assert res.clique_count == base.clique_count == exp["count"]
        assert res.clique_hash == base.clique_hash
        assert base.nodes_total == exp["nodes"]
        if induced == "ip":
            assert res.nodes_total == exp["nodes"]
        assert res.donation_count > 0


def test_edge_cases():
    for edges, n in (([], 0), ([], 4), ([(0, 1)], 2), ([(0, 1), (1, 2), (0, 2)], 5)):
        g = from_edges(np.asarray(edges, dtype=np.int64).reshape(-1, 2), n)
        g2, _, st = preprocess(g)
        ro, ci = oracle.from_edges(np.asarray(edges, dtype=np.int64).reshape(-1, 2), n)
        pos, d = oracle.degeneracy_order(ro, ci)
        for roots in ("l1", "l2"):
            exp = oracle.reference_pipeline(np.asarray(edges, dtype=np.int64).reshape(-1, 2),
                                            n, roots=roots, induced="ipx")
            res = run(g2, st, RunConfig(workers=2, roots=roots, induced="ipx"))
            assert res.clique_count == exp["count"]
            if n:
                assert res.clique_hash_hex == exp["hash"]


def test_l2_roots_count_isolated_vertices():
    g = from_edges([(0, 1), (1, 2), (0, 2)], 5)
    g2, _, st = preprocess(g)
    res = run(g2, st, RunConfig(workers=2, roots="l2", induced="ipx"))
    assert res.clique_count == 3


def test_scratch_arena_is_stream_ordered():
    """Temporaries come from a per-device arena released without a host wait;
    a call on another stream must wait for the previous call's work on the
    device (cudaStreamWaitEvent): alternating streams give identical results."""
    import torch

    edges, n = generate.workload_edges("er2k")
    g2, _, st = preprocess(from_edges(edges, n))
    base = run(g2, st, RunConfig())
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for i in range(6):
        s = streams[i % 2]
        res = run(g2, st, RunConfig(), stream=ctypes.c_void_p(s.cuda_stream))
        assert (res.clique_count, res.clique_hash, res.nodes_total) == \
            (base.clique_count, base.clique_hash, base.nodes_total)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_lane_per_root_path_matches_reference(case, monkeypatch):
    """The |P| <= 32 class on the lane-per-root kernel (k_tiny, forced on with
    MCE_TINY=1 for these small graphs): the reference's count, node total,
    histogram and hash with the exact order; roots it hands back (dense,
    heavy X, |X| > 32) run on the warp kernel in the same call."""
    g, _ = _graph(case)
    order = degeneracy_order(g, method="exact")
    g2 = reorder(g, order)
    st = stats(g2, order)
    for mode in ("l1-ipx", "l1-ip"):
        exp = case["runs"][mode]
        roots, induced = mode.split("-")
        monkeypatch.setenv("MCE_TINY", "0")
        warp = run(g2, st, RunConfig(roots=roots, induced=induced, worker_list=False))
        monkeypatch.setenv("MCE_TINY", "1")
        for workers, wl in ((0, False), (8, False), (0, True), (3, True)):
            res = run(g2, st, RunConfig(workers=workers, roots=roots, induced=induced,
                                        worker_list=wl))
            assert res.clique_count == exp["count"], (mode, workers, wl)
            if induced == "ip" or not wl:
                assert res.nodes_total == exp["nodes"], (mode, workers, wl)
                assert sum(w.nodes_visited for w in res.worker_metrics) == exp["nodes"]
            assert res.clique_hash == warp.clique_hash
            assert res.size_histogram == warp.size_histogram
            if "hash" in exp:
                assert res.clique_hash_hex == exp["hash"], mode
            if case["n"] and st.degeneracy <= 32 and case["m"]:
                assert res.kernel_launches > warp.kernel_launches  # k_tiny ran


def test_lane_per_root_fallbacks_match_oracle(monkeypatch):
    """Roots the lane kernel must hand back -- dense (> 64 induced edges),
    |X| > 32, heavy X (|X| >= 256) -- mixed with sparse ones in one call."""
    rng = np.random.default_rng(7)
    parts, base = [], 0
    k = 13  # K_13: early roots have 12 members and 66 > 64 edges
    parts += [(base + i, base + j) for i in range(k) for j in range(i + 1, k)]
    base += k
    for leaves in (300, 60):  # hubs in many triangles: |X| >= 256 (heavy) and 32 < |X| < 256
        hub = base
        for t in range(leaves):
            a, b = base + 1 + 2 * t, base + 2 + 2 * t
            parts += [(hub, a), (hub, b), (a, b)]
        base += 2 * leaves + 1
    sparse = generate.gnp_edges(3000, 0.004, seed=3)
    parts += [(base + int(u), base + int(v)) for u, v in sparse]
    base += 3000
    edges = np.asarray(parts, dtype=np.int64)
    edges = edges[rng.permutation(len(edges))]
    n = base
    g = from_edges(edges, n)
    g2, _, st = preprocess(g, method="exact")
    for induced in ("ipx", "ip"):
        monkeypatch.setenv("MCE_TINY", "1")
        res = run(g2, st, RunConfig(induced=induced, worker_list=False))
        monkeypatch.setenv("MCE_TINY", "0")
        ref = run(g2, st, RunConfig(induced=induced, worker_list=False))
        orc = oracle.enumerate_cliques(g2.row_offsets, g2.col_indices, roots="l1",
                                       induced=induced, degeneracy=st.degeneracy,
                                       labels=g2.labels)
        assert res.clique_count == ref.clique_count == orc["count"]
        assert res.nodes_total == ref.nodes_total == orc["nodes"]
        assert res.clique_hash_hex == ref.clique_hash_hex == orc["hash"]
        assert res.size_histogram == ref.size_histogram


BK = __import__("json").load(open(__import__("os").path.join(
    __import__("os").path.dirname(__file__), "golden", "bk_vectors.json")))["cases"]


@pytest.mark.parametrize("name", sorted(BK))
def test_bk_basic_and_pivot_match_reference(name, monkeypatch):
    """bk_basic: the reference's count and node total (no pivoting, the
    graph's own vertex order -- golden vectors from reference bk.py:124-150);
    bk_pivot: the same clique set, never more nodes than bk_basic."""
    from paper_2212_01473_b200 import bk_basic, bk_pivot

    case = next(c for c in CASES if c["name"] == name)
    g, _ = _graph(case)
    exp = BK[name]
    for tiny in ("0", "1"):  # warp kernel / lane-per-root kernel
        monkeypatch.setenv("MCE_TINY", tiny)
        mb, mp = {}, {}
        sb, sp = CliqueSink.collecting(), CliqueSink.collecting()
        assert bk_basic(g, sb, metrics=mb) == exp["count"]
        assert mb["nodes"] == exp["basic_nodes"], (name, tiny)
        assert bk_pivot(g, sp, metrics=mp) == exp["count"]
        assert set(sb.collected) == set(sp.collected)
        if "brute_force" in case:
            assert set(sb.collected) == {tuple(c) for c in case["brute_force"]}
        assert 0 < mp["nodes"] <= mb["nodes"]


def test_phase_times_and_worker_time_categories():
    """RunResult.phase1_time / phase2_time (device time before / after every
    root was claimed) and WorkerMetrics.times with timing on (reference
    scheduler.py:481-490, metrics.py:13-32)."""
    edges, n = generate.workload_edges("ba200k")
    g2, _, st = preprocess(from_edges(edges, n))
    res = run(g2, st, RunConfig(timing=True))
    assert res.phase1_time > 0 and res.phase2_time >= 0
    assert res.phase1_time + res.phase2_time <= res.total_time
    ms = res.worker_metrics
    cats = ("induced_build", "pivot", "set_ops", "worker_list", "other")
    assert all(set(m.times) == set(cats) for m in ms)
    assert all(v >= 0 for m in ms for v in m.times.values())
    busy = [m for m in ms if m.roots_claimed > 0]
    assert busy and all(m.times["induced_build"] > 0 for m in busy)
    assert sum(m.times["set_ops"] for m in ms) > 0
    rep = res.report()
    assert abs(sum(rep.category_shares.values()) - 1.0) < 1e-6
    off = run(g2, st, RunConfig())
    assert all(v == 0 for m in off.worker_metrics for v in m.times.values())
    assert (off.clique_count, off.clique_hash) == (res.clique_count, res.clique_hash)


C4 = __import__("json").load(open(__import__("os").path.join(
    __import__("os").path.dirname(__file__), "golden", "criterion4.json")))["graphs"]


@pytest.mark.parametrize("i", range(len(C4)))
def test_criterion_4_graph_set(i, monkeypatch):
    """The reference's acceptance criterion 4 (reference
    tests/test_acceptance.py:93-109) on its own 20 graphs: full ("ipx")
    subgraphs, workers {1, 2, 4, 8, 16} x worker list on/off -- the node
    total is the reference's in every configuration, with donations
    happening (also forced with donation_min_p=2), and on both the warp and
    the lane-per-root kernels."""
    gr = C4[i]
    g = from_edges(np.asarray(gr["edges"], dtype=np.int64).reshape(-1, 2), gr["n"])
    g2, _, st = preprocess(g, method="exact")
    donated = 0
    for tiny in ("0", "1"):
        monkeypatch.setenv("MCE_TINY", tiny)
        for workers in (1, 2, 4, 8, 16):
            for wl in (True, False):
                for min_p in ((10, 2) if wl else (10,)):
                    res = run(g2, st, RunConfig(workers=workers, roots="l1", induced="ipx",
                                                worker_list=wl, donation_min_p=min_p))
                    assert res.clique_count == gr["count"]
                    assert sum(w.nodes_visited for w in res.worker_metrics) == gr["nodes"], \
                        (i, tiny, workers, wl, min_p, res.donation_count)
                    donated += res.donation_count
    # (these sparse graphs' subtrees are too small to donate: phase 2 finds no
    # branch with |P| >= donation_min_p -- as in the reference's own run)


@pytest.mark.parametrize("variant", ["rows", "keysort"])
def test_from_edges_canonical_csr_with_duplicates_loops_and_hubs(variant, monkeypatch):
    """from_edges (graph.py:103-129): duplicates in either orientation and
    self-loops dropped, rows strictly ascending -- on both canonicalisation
    paths (row-wise; the key sort, which also takes every graph with a vertex
    of more than 2048 endpoints), rows of every register class, a long row
    sorted by one CTA, and a hub past the row path's limit."""
    if variant == "keysort":
        monkeypatch.setenv("MCE_CANON_KEYSORT", "1")
    rng = np.random.default_rng(11)
    n = 30_000
    parts = [rng.integers(0, n, size=(60_000, 2))]                  # random, some loops
    parts.append(parts[0][:5000][:, ::-1])                          # reversed duplicates
    parts.append(parts[0][:3000])                                   # exact duplicates
    parts.append(np.column_stack((np.full(1500, 7), rng.integers(0, n, 1500))))   # row > 256
    parts.append(np.column_stack((np.full(400, 9), np.full(400, 9))))             # loops only
    hub = np.column_stack((np.full(20_000, 5), np.arange(10, 20_010) % n))  # > the row path's 2048
    for with_hub in (False, True):
        edges = np.concatenate(parts + ([hub, hub[:100]] if with_hub else [])).astype(np.int64)
        g = from_edges(edges, n)
        ro, ci = oracle.from_edges(edges, n)
        assert np.array_equal(g.row_offsets, ro)
        assert np.array_equal(g.col_indices, ci)
        g32 = from_edges(edges.astype(np.int32), n)
        assert np.array_equal(g32.col_indices, ci)
    with pytest.raises(ValueError):
        from_edges(np.array([[0, n]], dtype=np.int64), n)

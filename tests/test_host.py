"""Host-side logic that needs no GPU: configuration validation, the auto
heuristic, sinks, metrics aggregation, parse errors and the generators
(checked against vectors produced by the reference)."""

from __future__ import annotations

import io

import numpy as np
import pytest

from conftest import golden_cases
from paper_2212_01473_b200 import generate
from paper_2212_01473_b200.bk import CliqueSink
from paper_2212_01473_b200.metrics import TIME_CATEGORIES, WorkerMetrics, aggregate
from paper_2212_01473_b200.scheduler import Backoff, RunConfig, choose_induced_mode


def test_config_rejects_bad_values():
    for bad in (RunConfig(workers=-1), RunConfig(roots="l3"), RunConfig(induced="both"),
                RunConfig(donation_min_p=-1), RunConfig(backoff=Backoff(initial=0.0)),
                RunConfig(backoff=Backoff(initial=1.0, max=0.5))):
        with pytest.raises(ValueError):
            bad.validate()


def test_workers_zero_resolves_to_hardware():
    assert RunConfig(workers=0).resolved_workers() >= 1
    assert RunConfig(workers=3).resolved_workers() == 3


def test_choose_induced_mode_matches_reference_fixtures():
    # reference tests/test_acceptance.py:198-221 (published dataset ratios)
    fixtures = [(100_029, 131, "ip"), (31_941, 100, "ip"), (6_914, 100, "ipx"),
                (31_604, 100, "ip"), (240_749, 100, "ip"), (1_245, 100, "ipx"),
                (13_167, 100, "ipx"), (144_295, 100, "ip"), (67_573, 100, "ip"),
                (160_665, 100, "ip"), (381_370, 100, "ip"), (1_715, 100, "ipx")]
    for max_deg, d, expected in fixtures:
        assert choose_induced_mode(max_deg, d) == expected
    assert choose_induced_mode(200, 1) == "ipx"
    assert choose_induced_mode(201, 1) == "ip"
    assert choose_induced_mode(0, 0) == "ipx"
    assert choose_induced_mode(20_001, 100) == "ip"


def test_sink_semantics():
    sink = CliqueSink(collect_limit=2)
    for i in range(5):
        sink.report([i])
    assert sink.total == 5 and len(sink.collected) == 2
    s = CliqueSink.collecting()
    s.report([3, 1, 2])
    assert s.collected == [(1, 2, 3)]
    a, b = CliqueSink(collect_limit=3), CliqueSink(collect_limit=3)
    a.report([1])
    for x in (2, 3, 4):
        b.report([x])
    a.merge(b)
    assert a.total == 4 and len(a.collected) == 3


def test_metrics_aggregate():
    rep = aggregate([WorkerMetrics(worker_id=0, nodes_visited=300),
                     WorkerMetrics(worker_id=1, nodes_visited=100)])
    assert rep.load_ratio == pytest.approx(1.5)
    assert rep.nodes_total == 400
    a = WorkerMetrics(worker_id=0)
    a.record("pivot", 1.0)
    a.record("induced_build", 3.0)
    rep = aggregate([a])
    assert rep.category_shares["induced_build"] == pytest.approx(0.75)
    assert set(rep.category_shares) == set(TIME_CATEGORIES)
    with pytest.raises(ValueError):
        aggregate([])


@pytest.mark.parametrize("case", [c for c in golden_cases() if c["name"].startswith("gnp_")
                                  or c["name"].startswith("er_")],
                         ids=lambda c: c["name"])
def test_gnp_stream_matches_reference_generator(case):
    """generate.gnp_edges draws numpy's PCG64 stream exactly as the reference
    gnp (reference generate.py:17-26): same seed, same edges."""
    name = case["name"]
    parts = name.split("_")
    n, p = int(parts[1]), float(parts[2])
    seed = int(parts[3][1:])
    got = generate.gnp_edges(n, p, seed)
    exp = np.asarray(case["edges"], dtype=np.int64).reshape(-1, 2)
    assert np.array_equal(got, exp)


def test_planted_skew_stream_matches_reference():
    for case in golden_cases():
        if case["name"] == "skew_2000_40":
            args = dict(n=2_000, community=40, p_in=0.95, background_degree=2.0, seed=1)
        elif case["name"] == "skew_1000_30":
            args = dict(n=1_000, community=30, p_in=0.9, background_degree=2.0, seed=3)
        else:
            continue
        rng_edges = _planted_skew_edges(**args)
        exp = np.asarray(case["edges"], dtype=np.int64).reshape(-1, 2)
        assert np.array_equal(rng_edges, exp), case["name"]


def _planted_skew_edges(**kw):
    """Canonical (u<v, sorted) edge set of generate.planted_skew without a GPU."""
    from oracle import oracle

    captured = {}

    def fake_from_edges(edges, n):
        captured["e"] = np.asarray(edges, dtype=np.int64)
        captured["n"] = n
        return None

    import paper_2212_01473_b200.graph as graph_mod
    orig = graph_mod.from_edges
    graph_mod.from_edges = fake_from_edges
    try:
        generate.planted_skew(**kw)
    finally:
        graph_mod.from_edges = orig
    ro, ci = oracle.from_edges(captured["e"], captured["n"])
    return oracle.upper_edges(ro, ci)


def test_rmat_and_ba_generators_are_deterministic_and_in_range():
    e1 = generate.rmat_edges(10, 4, seed=3)
    e2 = generate.rmat_edges(10, 4, seed=3)
    assert np.array_equal(e1, e2) and e1.min() >= 0 and e1.max() < 1 << 10
    # slices of the counter-based stream compose
    part = generate.rmat_edges(10, 4, seed=3, start=100, count=50)
    assert np.array_equal(part, e1[100:150])
    ba = generate.barabasi_albert_edges(1000, 4, seed=1)
    assert ba.shape == (4000, 2) and ba.max() < 1000
    assert np.all(ba[:, 1] <= ba[:, 0])  # targets are earlier (or the source itself)


def test_run_result_lazy_worker_metrics():
    """RunResult keeps the device's per-worker rows raw and builds
    WorkerMetrics objects on first access (host-only, no GPU)."""
    import numpy as np

    from paper_2212_01473_b200.scheduler import RunResult

    raw = np.array([[5, 1, 0, 1], [7, 2, 1, 0]], dtype=np.int64)
    res = RunResult(clique_count=3, donation_count=1, roots_mode="l1", induced_mode="ipx",
                    workers=2, total_time=0.0, phase1_time=0.0, phase2_time=0.0,
                    worker_metrics_raw=raw, nodes_total=12, timing=False)
    wm = res.worker_metrics
    assert [w.nodes_visited for w in wm] == [5, 7]
    assert [w.donations_made for w in wm] == [0, 1]
    assert res.report().nodes_total == 12 and res.report().load_ratio == pytest.approx(7 / 6)
    assert res.worker_metrics is wm


def test_graph_stats_lazy_resolution():
    """preprocess returns before the device finishes: GraphStats resolves its
    fields from the device statistics on first access, once."""
    from paper_2212_01473_b200.graph import GraphStats

    calls = []

    def thunk():
        calls.append(1)
        return 10, 7, 3

    st = GraphStats(5, _thunk=thunk)
    assert st.n == 5 and calls == []
    assert (st.m, st.max_degree, st.degeneracy) == (10, 7, 3)
    assert calls == [1]
    assert st == GraphStats(5, 10, 7, 3)
    assert "degeneracy=3" in repr(st)

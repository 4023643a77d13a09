"""GPU parity on the BASELINE.json workloads and on wide bitsets.

* Wide bitsets (|P| > 1024 -> W = 64 / 128 words): K_n minus a perfect
  matching on 2k of its vertices has exactly 2**k maximal cliques, each of
  size n - k, and a degeneracy of n - 2 -- the first-level roots need the
  widest bitset classes.  Checked bit-exactly against the oracle (count,
  node total, histogram, hash) and against the closed form.
* BASELINE workloads at sizes the oracle finishes in seconds: full runs for
  er2k / ba200k, root samples (``root_begin/root_end/root_stride``) for the
  R-MAT and planted-clique graphs, both sides on the SAME reordered graph.
* Size-independent properties at full size where the oracle cannot follow:
  first-level and second-level decompositions give the same clique set
  (count, histogram, hash); the sharded runs sum to the whole.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle
from paper_2212_01473_b200 import RunConfig, from_edges, generate, preprocess, run
from paper_2212_01473_b200.distributed import ShardResult, combine

pytestmark = pytest.mark.gpu


def k_minus_matching(n: int, k: int) -> np.ndarray:
    u, v = np.triu_indices(n, k=1)
    drop = (u < 2 * k) & (v == u + 1) & (u % 2 == 0)
    return np.column_stack((u[~drop], v[~drop])).astype(np.int64)


def _check_against_oracle(g2, st, roots="l1", induced="ipx", **kw):
    res = run(g2, st, RunConfig(roots=roots, induced=induced, worker_list=False), **kw)
    sample = {k: kw[k] for k in ("root_begin", "root_end", "root_stride") if k in kw}
    inc = not sample
    orc = oracle.enumerate_cliques(g2.row_offsets, g2.col_indices, roots=roots, induced=induced,
                                   degeneracy=st.degeneracy, labels=g2.labels,
                                   include_isolated=inc, **sample)
    assert res.clique_count == orc["count"]
    assert res.nodes_total == orc["nodes"]
    assert res.clique_hash_hex == orc["hash"]
    assert res.size_histogram == orc["hist"]
    return res


@pytest.mark.parametrize("n,k", [(1100, 6), (2150, 5)])
def test_wide_bitsets_match_oracle_and_closed_form(n, k):
    g = from_edges(k_minus_matching(n, k), n)
    g2, _, st = preprocess(g)
    assert st.degeneracy == n - 2 > 1024
    # partial mode cannot pivot on X_X members: ~300x the nodes, oracle-bound
    for induced in (("ipx", "ip") if n < 2048 else ("ipx",)):
        res = _check_against_oracle(g2, st, induced=induced)
        assert res.clique_count == 2 ** k
        assert res.size_histogram == {n - k: 2 ** k}
    # the worker list must not change the clique set
    res = run(g2, st, RunConfig(donation_min_p=2))
    assert res.clique_count == 2 ** k


def test_capacity_error_beyond_widest_class():
    from paper_2212_01473_b200 import CapacityError

    n = 4200
    g = from_edges(k_minus_matching(n, 1), n)
    g2, _, st = preprocess(g)
    with pytest.raises(CapacityError):
        run(g2, st, RunConfig())


@pytest.mark.parametrize("name", ["er2k", "ba200k"])
def test_small_workloads_full_parity(name):
    edges, n = generate.workload_edges(name)
    g = from_edges(edges, n)
    g2, _, st = preprocess(g)
    res = _check_against_oracle(g2, st, induced="ipx")
    ip = run(g2, st, RunConfig(induced="ip"))
    assert (ip.clique_count, ip.clique_hash) == (res.clique_count, res.clique_hash)


@pytest.mark.parametrize("name,sample,modes", [
    ("planted1m", dict(root_begin=0, root_end=-1, root_stride=97), ("ipx", "ip")),
    ("planted1m", dict(root_begin=999_000, root_end=-1, root_stride=1), ("ipx", "ip")),
    ("rmat20", dict(root_begin=0, root_end=600_000, root_stride=13), ("ipx", "ip")),
    # the dense core: the last 8,576 roots hold all but 0.2 % of rmat20's
    # maximal cliques; its first part (~2.5e4 cliques per root) and a few
    # roots 6,000 from the end (~6e6 cliques each, cliques up to size ~95)
    ("rmat20", dict(root_begin=(1 << 20) - 8576, root_end=(1 << 20) - 7000, root_stride=32),
     ("ipx", "ip")),
    ("rmat20", dict(root_begin=(1 << 20) - 6000, root_end=(1 << 20) - 4000, root_stride=500),
     ("ipx",)),
])
def test_large_workloads_sampled_parity(name, sample, modes):
    edges, n = generate.workload_edges(name)
    g = from_edges(edges, n)
    g2, _, st = preprocess(g)
    for induced in modes:
        _check_against_oracle(g2, st, induced=induced, **sample)


def test_planted1m_full_parity():
    """configs[3] in full: every one of the 1,000,000 first-level roots, count,
    node total, histogram and hash against the oracle on the same reordered
    graph (the oracle takes ~10 s on the box's host threads)."""
    edges, n = generate.workload_edges("planted1m")
    g2, _, st = preprocess(from_edges(edges, n))
    res = _check_against_oracle(g2, st, induced="ipx")
    assert res.clique_count == 9_997_854 and max(res.size_histogram) == 60


def test_planted_full_l1_equals_l2_and_shards_sum():
    edges, n = generate.workload_edges("planted1m")
    g = from_edges(edges, n)
    g2, _, st = preprocess(g)
    whole = run(g2, st, RunConfig(worker_list=False))
    # every planted clique (sizes 30-60) is maximal in a sparse background
    assert sum(c for s, c in whole.size_histogram.items() if s >= 30) >= 990
    l2 = run(g2, st, RunConfig(roots="l2"))
    assert (l2.clique_count, l2.clique_hash, l2.size_histogram) == \
        (whole.clique_count, whole.clique_hash, whole.size_histogram)
    parts = []
    for r in range(3):
        p = run(g2, st, RunConfig(worker_list=False), root_begin=r, root_stride=3)
        parts.append(ShardResult(p.clique_count, p.nodes_total, p.donation_count, p.clique_hash,
                                 p.size_histogram))
    tot = combine(parts)
    assert tot.cliques == whole.clique_count and tot.hash == whole.clique_hash
    assert tot.nodes == whole.nodes_total


@pytest.mark.parametrize("name", ["ba200k", "planted1m"])
def test_per_rank_orderings_shard_exactly(name):
    """The N>1 code path as two ranks run it: each rank builds ITS OWN
    ordering (preprocess_for_shards: the deterministic parallel peel at
    world > 1) and enumerates its shard through run_shard; the two partial
    results must add up to the whole run (count, node total, histogram,
    hash).  With the async peel (the old per-rank default) two independent
    orderings differ, and run_shard refuses them at world > 1."""
    from paper_2212_01473_b200.distributed import preprocess_for_shards, run_shard

    edges, n = generate.workload_edges(name)
    cfg = RunConfig()
    whole_g, _, whole_st = preprocess(from_edges(edges, n), method="parallel")
    whole = run(whole_g, whole_st, cfg)
    parts = []
    for rank in range(2):
        g2, order, st = preprocess_for_shards(from_edges(edges, n), 2)  # independent per rank
        assert g2.order_method == "parallel"
        _, part = run_shard(g2, st, cfg, rank, 2)
        parts.append(part)
    tot = combine(parts)
    assert (tot.cliques, tot.hash, tot.hist, tot.nodes) == \
        (whole.clique_count, whole.clique_hash, whole.size_histogram, whole.nodes_total)
    ga, _, sta = preprocess(from_edges(edges, n), method="async")
    with pytest.raises(ValueError):
        run_shard(ga, sta, cfg, 0, 2)


def test_from_edges_rejects_out_of_range_ids_on_device():
    for bad in ([(0, 5)], [(-1, 2)], [(0, 1), (2, 3)]):
        with pytest.raises(ValueError):
            from_edges(np.asarray(bad, dtype=np.int64), 3 if bad != [(0, 5)] else 5)
    g = from_edges(np.asarray([(0, 4), (4, 4)], dtype=np.int64), 5)  # self-loop dropped
    assert g.num_edges == 1


@pytest.mark.parametrize("name", ["er2k", "ba200k", "planted1m"])
def test_parallel_peel_positions_match_restatement(name):
    """The persistent peel kernel (incremental + full rounds) reproduces the
    round-synchronous bucket peel exactly: positions and degeneracy."""
    from paper_2212_01473_b200 import degeneracy_order

    edges, n = generate.workload_edges(name)
    g = from_edges(edges, n)
    got = degeneracy_order(g, method="parallel")
    pos, d = oracle.bucket_peel_order(g.row_offsets, g.col_indices)
    assert got.degeneracy == d
    assert np.array_equal(got.position, pos)
    # preprocess (device-resident positions) agrees with the host-visible order
    _, order, st = preprocess(g, method="parallel")
    assert np.array_equal(order.position, pos) and st.degeneracy == d


@pytest.mark.parametrize("induced", ["ip", "ipx"])
def test_heavy_x_prepass_matches_per_warp_build_and_oracle(induced, monkeypatch):
    """Hubs late in the order (|X| >= 256) take their X rows from the grid-wide
    pre-pass (k_heavy_xrows) and start with the zero-row X members left out;
    the traversal must be the per-warp build's exactly (MCE_HEAVY=0), node
    count included, and the oracle's."""
    edges, n = generate.workload_edges("ba200k")
    g2, _, st = preprocess(from_edges(edges, n))
    assert g2.device_info()["max_earlier"] >= 4096
    fast = run(g2, st, RunConfig(induced=induced, worker_list=False))
    monkeypatch.setenv("MCE_HEAVY", "0")
    slow = run(g2, st, RunConfig(induced=induced, worker_list=False))
    monkeypatch.delenv("MCE_HEAVY")
    assert (fast.clique_count, fast.nodes_total, fast.clique_hash, fast.size_histogram) == \
        (slow.clique_count, slow.nodes_total, slow.clique_hash, slow.size_histogram)
    orc = oracle.enumerate_cliques(g2.row_offsets, g2.col_indices, roots="l1", induced=induced,
                                   degeneracy=st.degeneracy, labels=g2.labels)
    assert (fast.clique_count, fast.nodes_total, fast.clique_hash_hex) == \
        (orc["count"], orc["nodes"], orc["hash"])
    # with donations (hub branches handed to idle warps) the clique set is unchanged
    don = run(g2, st, RunConfig(induced=induced, donation_min_p=1, donation_min_x=16))
    assert (don.clique_count, don.clique_hash, don.nodes_total) == \
        (fast.clique_count, fast.clique_hash, fast.nodes_total)


def _later_counts(ro, ci, pos):
    src = np.repeat(np.arange(len(ro) - 1), np.diff(ro))
    later = pos[ci] > pos[src]
    return np.bincount(src[later], minlength=len(ro) - 1)


@pytest.mark.parametrize("name,tail", [("er2k", None), ("ba200k", None), ("planted1m", None),
                                       ("ba200k", "65536"), ("planted1m", "65536"),
                                       ("planted1m", "1")])
def test_async_peel_is_a_degeneracy_order(name, tail, monkeypatch):
    """method="async" (no rounds inside a level): a permutation whose every
    vertex has at most d later neighbours, d the reference's degeneracy --
    checked on repeated runs, since its tie-breaks are data-dependent -- and
    the same clique set as the other orders.  ``tail`` forces the hand-over
    of the last levels to the cluster kernel (k_peel_tail) at that many
    remaining vertices (er2k runs on it whole by default)."""
    from paper_2212_01473_b200 import degeneracy_order

    if tail is not None:
        monkeypatch.setenv("MCE_PEEL_TAIL", tail)
    edges, n = generate.workload_edges(name)
    g = from_edges(edges, n)
    ro, ci = g.row_offsets, g.col_indices
    _, d = oracle.degeneracy_order(ro, ci)
    for _ in range(3):
        got = degeneracy_order(g, method="async")
        assert got.degeneracy == d
        assert np.array_equal(np.sort(got.position), np.arange(n))
        assert _later_counts(ro, ci, got.position).max() == d
    g_a, _, st_a = preprocess(g, method="async")
    g_p, _, st_p = preprocess(g, method="parallel")
    assert st_a.degeneracy == st_p.degeneracy == d
    ra, rp = run(g_a, st_a, RunConfig()), run(g_p, st_p, RunConfig())
    assert (ra.clique_count, ra.clique_hash, ra.size_histogram) == \
        (rp.clique_count, rp.clique_hash, rp.size_histogram)


@pytest.mark.parametrize("env", [{"MCE_PEEL_SLACK": "0"}, {"MCE_PEEL_CERT": "0"},
                                 {"MCE_PEEL_DENS_CAP": "0"},
                                 {"MCE_PEEL_SLACK": "0", "MCE_PEEL_CERT": "0", "MCE_PEEL_DENS_CAP": "0"},
                                 {"MCE_PEEL_SLACK": "6"}])
def test_async_peel_certified_jumps(env, monkeypatch):
    """The async peel's certified shortcuts one at a time (density floor,
    level slack, residual certificate jump): a sparse background of 200k
    vertices plus disjoint planted cliques of 10-80 members, so the residual
    is small, clique-made and its certificate the largest clique's size - 1.
    Every variant is a valid degeneracy order with the reference's
    degeneracy and the same clique set."""
    from paper_2212_01473_b200 import degeneracy_order

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(7)
    n0 = 200_000
    bg = rng.integers(0, n0, size=(3 * n0, 2), dtype=np.int64)
    parts, base = [bg], n0
    for size in range(10, 81, 5):
        for _ in range(4):
            u, w = np.triu_indices(size, k=1)
            parts.append(np.column_stack((u + base, w + base)))
            base += size
    edges = np.concatenate(parts)
    g = from_edges(edges, base)
    ro, ci = g.row_offsets, g.col_indices
    _, d = oracle.degeneracy_order(ro, ci)
    assert d == 79
    for _ in range(2):
        got = degeneracy_order(g, method="async")
        assert got.degeneracy == d
        assert np.array_equal(np.sort(got.position), np.arange(base))
        assert _later_counts(ro, ci, got.position).max() == d
    g_a, _, st_a = preprocess(g, method="async")
    g_p, _, st_p = preprocess(g, method="parallel")
    ra, rp = run(g_a, st_a, RunConfig()), run(g_p, st_p, RunConfig())
    assert (ra.clique_count, ra.clique_hash, ra.size_histogram) == \
        (rp.clique_count, rp.clique_hash, rp.size_histogram)


def test_async_peel_on_reference_graphs():
    """Every golden graph of the reference's tests: valid degeneracy order,
    exact degeneracy, and the reference's clique count / hash."""
    from conftest import golden_cases
    from paper_2212_01473_b200 import degeneracy_order

    for case in golden_cases():
        n = case["n"]
        edges = np.asarray(case["edges"], dtype=np.int64).reshape(-1, 2)
        g = from_edges(edges, n)
        if n == 0:
            continue
        got = degeneracy_order(g, method="async")
        _, d = oracle.degeneracy_order(g.row_offsets, g.col_indices)
        assert got.degeneracy == d, case["name"]
        assert np.array_equal(np.sort(got.position), np.arange(n)), case["name"]
        if g.num_edges:
            assert _later_counts(g.row_offsets, g.col_indices, got.position).max() == d, case["name"]
        g2, _, st = preprocess(g, method="async")
        res = run(g2, st, RunConfig())
        exp = case["runs"]["l1-ipx"]
        assert res.clique_count == exp["count"], case["name"]
        assert res.clique_hash_hex == exp["hash"], case["name"]


def test_every_width_class_in_one_call():
    """Disjoint cliques whose first-level roots fall in seven bitset classes
    (|P| up to 1049 -> W = 1 ... 64): one call launches every class (the
    first call of a process takes its scratch from the pool), and each
    clique is exactly one maximal clique."""
    sizes = [5, 40, 70, 140, 270, 530, 1050]
    parts, base = [], 0
    for s in sizes:
        u, v = np.triu_indices(s, k=1)
        parts.append(np.column_stack((u + base, v + base)))
        base += s
    g = from_edges(np.concatenate(parts).astype(np.int64), base)
    g2, _, st = preprocess(g)
    assert st.degeneracy == max(sizes) - 1
    for induced in ("ipx", "ip"):
        res = run(g2, st, RunConfig(induced=induced))
        assert res.clique_count == len(sizes)
        assert res.size_histogram == {s: 1 for s in sizes}
        assert res.kernel_launches >= 7


def test_rmat24_sampled_parity():
    """configs[4] at full size: R-MAT scale 24 (268 M generated edges, 16.8 M
    vertices, degeneracy 1621) generated, canonicalised and ordered on the
    device, then a strided sample of first-level roots checked bit-exactly
    against the oracle on the same reordered CSR (both induced modes).  The
    dense core (the last roots) is out of the oracle's reach; the core's
    widest class is covered by the K_n-minus-matching and every-class tests."""
    import torch

    from paper_2212_01473_b200 import _lib, from_device_edges

    scale = 24
    m, n = 16 << scale, 1 << scale
    dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "mce_gen_rmat")
    g = from_device_edges(dev, m, n)
    del dev
    torch.cuda.empty_cache()
    g2, _, st = preprocess(g)
    assert st.degeneracy == 1621 and st.max_degree == 405842
    sample = dict(root_begin=0, root_end=16_000_000, root_stride=4001)
    for induced in ("ip", "ipx"):
        res = _check_against_oracle(g2, st, induced=induced, **sample)
        assert res.clique_count > 3000
    # toward the core: 64 roots 100,000 from the end (~7e4 maximal cliques each,
    # cliques up to size ~52); 50,000 from the end it is ~1e8 per root
    core = dict(root_begin=n - 100_000, root_end=n - 100_000 + 64 * 16, root_stride=16)
    res = _check_against_oracle(g2, st, induced="ipx", **core)
    assert res.clique_count > 1_000_000


def test_team_workers_match_oracle(monkeypatch):
    """The thread-block ("team") workers for the W = 16 / 32 classes (opt-in,
    MCE_TEAM=1): CTA-mates share one copy of the rows, whole idle teams take
    over branches in phase 2 -- same count, hash and histogram, and with the
    worker list off the oracle's node total."""
    monkeypatch.setenv("MCE_TEAM", "1")
    sizes = [270, 530, 600, 40]
    parts, base = [], 0
    for s in sizes:
        u, v = np.triu_indices(s, k=1)
        parts.append(np.column_stack((u + base, v + base)))
        base += s
    parts.append(k_minus_matching(700, 4) + base)
    base += 700
    g = from_edges(np.concatenate(parts).astype(np.int64), base)
    g2, _, st = preprocess(g)
    for induced in ("ipx", "ip"):
        res = run(g2, st, RunConfig(induced=induced, donation_min_p=2))
        orc = oracle.enumerate_cliques(g2.row_offsets, g2.col_indices, induced=induced,
                                       degeneracy=st.degeneracy, labels=g2.labels)
        assert res.clique_count == orc["count"] == len(sizes) + 2 ** 4
        assert res.clique_hash_hex == orc["hash"] and res.size_histogram == orc["hist"]
        if induced == "ip":
            assert res.nodes_total == orc["nodes"]
    edges, n = generate.workload_edges("rmat20")
    g2, _, st = preprocess(from_edges(edges, n))
    sample = dict(root_begin=(1 << 20) - 8576, root_end=(1 << 20) - 7000, root_stride=32)
    res = run(g2, st, RunConfig(), **sample)
    orc = oracle.enumerate_cliques(g2.row_offsets, g2.col_indices, induced="ipx",
                                   degeneracy=st.degeneracy, labels=g2.labels,
                                   include_isolated=False, **sample)
    assert (res.clique_count, res.clique_hash_hex) == (orc["count"], orc["hash"])


@pytest.mark.parametrize("shard", ["static", "steal"])
def test_bench_two_ranks_reproduce_one_gpu(shard, tmp_path):
    """bench.py's N > 1 path end to end: two ranks (torchrun) time-sharing
    this GPU, gloo standing in for NCCL (MCE_BENCH_BACKEND) -- every rank
    orders the graph itself, enumerates its shard, and the all-reduced
    result is the single-GPU clique set exactly."""
    import json
    import os
    import subprocess
    import sys

    import socket

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MCE_BENCH_BACKEND="gloo")

    def launch():
        with socket.socket() as sk:  # a free rendezvous port
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(port),
               os.path.join(root, "bench.py"), "--gpus", "2", "--workload", "ba200k", "--steps", "3",
               "--warmup", "3", "--shard", shard, "--no-cpu-baseline", "--no-clocks"]
        return subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=root, env=env)

    # two processes time-slicing one GPU next to this one's context: one
    # full-suite run saw a launch never return (not reproducible alone, 17 s);
    # a stalled launch is retried once on a fresh port
    try:
        out = launch()
    except subprocess.TimeoutExpired:
        out = launch()
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["result"]["sharding"] == shard
    edges, n = generate.workload_edges("ba200k")
    g2, _, st = preprocess(from_edges(edges, n))
    one = run(g2, st, RunConfig())
    assert line["result"]["maximal_cliques"] == one.clique_count
    assert line["result"]["clique_hash"] == one.clique_hash_hex

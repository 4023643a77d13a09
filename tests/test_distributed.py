"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 path: the
all-reduce of per-rank results (count/nodes/histogram and the clique-set
hash mod 2**64), the static interleaved sharding, and the static+dynamic
chunk claiming of ``run_work_stealing`` -- the enumeration itself is
replaced by the CPU oracle (static shards) or a stub (claims), since these
tests run without a GPU."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2212_01473_b200.distributed import (
    MASK64,
    ShardResult,
    allreduce_result,
    claim_chunks,
    combine,
    run_work_stealing,
    shard_bounds,
)
from paper_2212_01473_b200.scheduler import RunConfig, RunResult

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank: int, port: int) -> None:
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)


def _spawn(fn, *args):
    port = _free_port()
    mp.spawn(fn, args=(port, *args), nprocs=WORLD, join=True)


# ---------------------------------------------------------------- all-reduce

def _allreduce_worker(rank, port, out_dir):
    _init(rank, port)
    try:
        big = MASK64 - 5 if rank == 0 else 11  # wraps mod 2**64
        part = ShardResult(cliques=10 + rank, nodes=100 * (rank + 1), donations=rank,
                           hash=big, hist={3: 1 + rank, 200: 2})
        tot = allreduce_result(part)
        np.save(os.path.join(out_dir, f"r{rank}.npy"), tot.pack())
    finally:
        dist.destroy_process_group()


def test_allreduce_sums_counts_histograms_and_wraps_the_hash(tmp_path):
    _spawn(_allreduce_worker, str(tmp_path))
    a = ShardResult.unpack(np.load(tmp_path / "r0.npy"))
    b = ShardResult.unpack(np.load(tmp_path / "r1.npy"))
    assert a == b
    assert (a.cliques, a.nodes, a.donations) == (21, 300, 1)
    assert a.hash == (MASK64 - 5 + 11) & MASK64 == 5
    # every size is reduced in its own slot (RMAT cores reach sizes > 100)
    assert a.hist == {3: 3, 200: 4}
    with pytest.raises(ValueError):
        ShardResult(1, 1, 0, 0, {5000: 1}).pack()


# ---------------------------------------------------------------- work stealing

def _fake_result(k: int) -> RunResult:
    return RunResult(clique_count=k + 1, donation_count=0, roots_mode="l1", induced_mode="ipx",
                     workers=1, total_time=0.0, phase1_time=0.0, phase2_time=0.0,
                     worker_metrics_raw=[], nodes_total=2 * k, clique_hash=(k * 0x9E3779B97F4A7C15)
                     & MASK64, size_histogram={2: k + 1})


def _steal_worker(rank, port, out_dir, chunks):
    _init(rank, port)
    try:
        seen = []

        def runner(g2, st, cfg, root_begin, root_end, root_stride):
            assert root_stride == chunks and root_end == -1
            seen.append(root_begin)
            if rank == 0:  # rank 0 is slow: rank 1 must steal most chunks
                import time
                time.sleep(0.2)
            return _fake_result(root_begin)

        results, tot = run_work_stealing(None, None, RunConfig(), rank, WORLD, chunks=chunks,
                                         runner=runner)
        assert [r.clique_count - 1 for r in results] == seen
        np.save(os.path.join(out_dir, f"seen{rank}.npy"), np.asarray(seen, dtype=np.int64))
        np.save(os.path.join(out_dir, f"tot{rank}.npy"), tot.pack())
        # a second job on the same ranks uses a fresh counter
        _, tot2 = run_work_stealing(None, None, RunConfig(), rank, WORLD, chunks=chunks,
                                    runner=lambda *a, **k: _fake_result(k["root_begin"]))
        np.save(os.path.join(out_dir, f"tot2_{rank}.npy"), tot2.pack())
    finally:
        dist.destroy_process_group()


def test_work_stealing_claims_every_chunk_once(tmp_path):
    chunks = 12
    _spawn(_steal_worker, str(tmp_path), chunks)
    s0 = np.load(tmp_path / "seen0.npy").tolist()
    s1 = np.load(tmp_path / "seen1.npy").tolist()
    assert s0[0] == 0 and s1[0] == 1  # static share first
    assert sorted(s0 + s1) == list(range(chunks))
    assert len(s1) > len(s0)  # the fast rank stole from the slow one
    expect = combine([ShardResult(k + 1, 2 * k, 0, (k * 0x9E3779B97F4A7C15) & MASK64, {2: k + 1})
                      for k in range(chunks)])
    for name in ("tot0.npy", "tot1.npy", "tot2_0.npy", "tot2_1.npy"):
        assert ShardResult.unpack(np.load(tmp_path / name)) == expect


def test_claim_chunks_single_process_store():
    import datetime

    from torch.distributed import HashStore

    store = HashStore()
    store.set_timeout(datetime.timedelta(seconds=5))
    assert list(claim_chunks(store, "k", 0, 1, 5)) == [0, 1, 2, 3, 4]
    assert list(claim_chunks(store, "k", 0, 1, 5)) == [0]  # counter exhausted


def test_stealing_rejects_bad_chunking():
    with pytest.raises(ValueError):
        run_work_stealing(None, None, RunConfig(roots="l2"), 0, 2, store=object())
    with pytest.raises(ValueError):
        run_work_stealing(None, None, RunConfig(), 0, 4, chunks=2, store=object())


# ---------------------------------------------------------------- static shards

def _with_big_clique(n=400, p=0.05, k=130, seed=7):
    """G(n, p) plus a planted k-clique (k >= 128: sizes past the old 128-slot
    histogram) on random vertices."""
    from paper_2212_01473_b200 import generate

    edges = generate.gnp_edges(n, p, seed=seed)
    members = np.random.default_rng(seed).choice(n, size=k, replace=False)
    iu, ju = np.triu_indices(k, 1)
    return np.concatenate([edges, np.column_stack((members[iu], members[ju]))]), n


def test_static_shards_partition_the_roots_exactly():
    """Per-shard oracle runs over shard_bounds(r, world) sum to the whole run:
    same count, node total, histogram and clique-set hash -- including a
    clique of size >= 128."""
    from oracle import oracle

    edges, n = _with_big_clique()
    ro, ci = oracle.from_edges(edges, n)
    pos, d = oracle.degeneracy_order(ro, ci)
    ro2, ci2 = oracle.reorder(ro, ci, pos)
    whole = oracle.enumerate_cliques(ro2, ci2, degeneracy=d, threads=1)
    for world in (2, 3):
        parts = []
        for r in range(world):
            b = shard_bounds(r, world)
            o = oracle.enumerate_cliques(ro2, ci2, degeneracy=d, threads=1, **b)
            parts.append(ShardResult(o["count"], o["nodes"], 0, int(o["hash"], 16), o["hist"]))
        tot = combine(parts)
        assert tot.cliques == whole["count"] and tot.nodes == whole["nodes"]
        assert f"{tot.hash:016x}" == whole["hash"] and tot.hist == whole["hist"]
    assert max(whole["hist"]) >= 128
    with pytest.raises(ValueError):
        shard_bounds(2, 2)


def _labels(pos):
    """Original id of every reordered vertex: the clique hash over labels
    does not depend on the ordering."""
    lab = np.empty(len(pos), dtype=np.int64)
    lab[pos] = np.arange(len(pos), dtype=np.int64)
    return lab


def _gloo_shard_worker(rank, port, out_dir):
    """Each rank orders the graph itself (deterministic bucket peel, the
    numpy restatement of method='parallel'), enumerates its shard with the
    oracle and joins the one all-reduce."""
    from oracle import oracle

    _init(rank, port)
    try:
        edges, n = _with_big_clique()
        ro, ci = oracle.from_edges(edges, n)
        pos, d = oracle.bucket_peel_order(ro, ci)
        ro2, ci2 = oracle.reorder(ro, ci, pos)
        o = oracle.enumerate_cliques(ro2, ci2, degeneracy=d, threads=1, labels=_labels(pos),
                                     **shard_bounds(rank, WORLD))
        tot = allreduce_result(ShardResult(o["count"], o["nodes"], 0, int(o["hash"], 16), o["hist"]))
        np.save(os.path.join(out_dir, f"shard{rank}.npy"), tot.pack())
    finally:
        dist.destroy_process_group()


def test_gloo_shards_with_per_rank_ordering_sum_to_the_whole(tmp_path):
    from oracle import oracle

    _spawn(_gloo_shard_worker, str(tmp_path))
    edges, n = _with_big_clique()
    ro, ci = oracle.from_edges(edges, n)
    pos, d = oracle.degeneracy_order(ro, ci)
    whole = oracle.enumerate_cliques(*oracle.reorder(ro, ci, pos), degeneracy=d, threads=1,
                                     labels=_labels(pos))
    for r in range(WORLD):
        tot = ShardResult.unpack(np.load(tmp_path / f"shard{r}.npy"))
        assert tot.cliques == whole["count"] and tot.hist == whole["hist"]
        assert f"{tot.hash:016x}" == whole["hash"]
    assert max(tot.hist) >= 128


def test_shards_of_two_different_orderings_do_not_partition():
    """Why sharding needs ONE ordering: shard 0 of one valid degeneracy order
    plus shard 1 of another (both with the reference's degeneracy) miss or
    double-count cliques -- the failure the async peel's run-to-run tie-breaks
    would cause; and run_shard refuses an async-ordered graph at world > 1."""
    from oracle import oracle
    from paper_2212_01473_b200 import generate
    from paper_2212_01473_b200.distributed import check_shardable

    edges = generate.gnp_edges(400, 0.05, seed=0)
    ro, ci = oracle.from_edges(edges, 400)
    pos_a, d = oracle.degeneracy_order(ro, ci)
    pos_b, d_b = oracle.bucket_peel_order(ro, ci)
    assert d == d_b and not np.array_equal(pos_a, pos_b)
    whole = oracle.enumerate_cliques(*oracle.reorder(ro, ci, pos_a), degeneracy=d, threads=1,
                                     labels=_labels(pos_a))
    s0 = oracle.enumerate_cliques(*oracle.reorder(ro, ci, pos_a), degeneracy=d, threads=1,
                                  labels=_labels(pos_a), **shard_bounds(0, 2))
    s1 = oracle.enumerate_cliques(*oracle.reorder(ro, ci, pos_b), degeneracy=d, threads=1,
                                  labels=_labels(pos_b), **shard_bounds(1, 2))
    mixed = combine([ShardResult(o["count"], o["nodes"], 0, int(o["hash"], 16), o["hist"])
                     for o in (s0, s1)])
    assert f"{mixed.hash:016x}" != whole["hash"]
    # each ordering on its own still shards exactly
    s1a = oracle.enumerate_cliques(*oracle.reorder(ro, ci, pos_a), degeneracy=d, threads=1,
                                   labels=_labels(pos_a), **shard_bounds(1, 2))
    same = combine([ShardResult(o["count"], o["nodes"], 0, int(o["hash"], 16), o["hist"])
                    for o in (s0, s1a)])
    assert f"{same.hash:016x}" == whole["hash"] and same.cliques == whole["count"]

    class G:
        order_method = "async"
    with pytest.raises(ValueError):
        check_shardable(G(), 2)
    check_shardable(G(), 1)
    G.order_method = "parallel"
    check_shardable(G(), 2)

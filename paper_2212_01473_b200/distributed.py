"""Multi-GPU enumeration: first-level subtrees sharded across ranks.

One process per GPU (``torch.distributed``).  The subtree roots are
independent (paper §3.1), so ranks need no data-path communication.

* ``run_sharded`` (static): rank r enumerates the roots ``r, r + world,
  r + 2*world, ...`` of the degeneracy-reordered graph -- an interleave over
  vertex ids, which spreads the heavy late-ordered roots evenly -- with its
  own device-wide worker list for intra-GPU balance.
* ``run_work_stealing`` (static + dynamic): the roots are cut into K
  interleaved chunks ``{v : v % K == k}``; rank r first runs chunk r, then
  claims further chunks off one shared counter (``store.add`` on the
  process group's key-value store -- control plane only, a few bytes per
  claim) until none are left, so a rank that drew light chunks keeps
  working while another is still in a heavy one.

Every rank builds the ordering itself, so the shards only partition the
cliques when every rank computes the SAME ordering: a clique is enumerated
by the root of its earliest vertex, and "earliest" is the order's.  The
``async`` peel breaks ties by a device-wide race and differs from run to
run, so sharding requires a deterministic method -- ``preprocess_for_shards``
uses ``parallel`` (pinned to ``oracle.bucket_peel_order``) whenever
world > 1, and ``run_shard`` refuses an async-ordered graph at world > 1.

Either way the single collective is the final reduction of counts, node
totals, the full size histogram (every size up to MCE_HIST_MAX) and the
order-independent clique-set hash (sum mod 2**64), done with one NCCL
all-reduce (gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2212_01473_b200.scheduler import RunConfig, RunResult, run

HIST_WORDS = 4096  # = MCE_HIST_MAX (include/mce_b200.h): every clique size the device counts
MASK64 = (1 << 64) - 1
DETERMINISTIC_METHODS = ("parallel", "exact")


@dataclass
class ShardResult:
    """This rank's partial result, packed for one all-reduce."""

    cliques: int
    nodes: int
    donations: int
    hash: int
    hist: dict[int, int]

    def pack(self) -> np.ndarray:
        v = np.zeros(4 + HIST_WORDS, dtype=np.int64)
        v[0], v[1], v[2] = self.cliques, self.nodes, self.donations
        h = self.hash & MASK64
        v[3] = h - (1 << 64) if h >= (1 << 63) else h  # two's complement view
        for s, c in self.hist.items():
            if not 0 <= s < HIST_WORDS:
                raise ValueError(f"clique size {s} outside the reduced histogram")
            v[4 + s] += c
        return v

    @staticmethod
    def unpack(v: np.ndarray) -> "ShardResult":
        nz = np.flatnonzero(v[4:])
        hist = {int(s): int(v[4 + s]) for s in nz}
        return ShardResult(int(v[0]), int(v[1]), int(v[2]), int(v[3]) & MASK64, hist)

    @staticmethod
    def of(res: RunResult) -> "ShardResult":
        return ShardResult(res.clique_count, res.nodes_total, res.donation_count,
                           res.clique_hash, res.size_histogram)


def shard_bounds(rank: int, world: int) -> dict:
    """Root sample of one rank: every world-th root starting at rank."""
    if not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    return {"root_begin": rank, "root_end": -1, "root_stride": world}


def combine(partials: list[ShardResult]) -> ShardResult:
    """What the all-reduce computes (used by tests and the gloo path)."""
    tot = np.zeros(4 + HIST_WORDS, dtype=np.int64)
    with np.errstate(over="ignore"):
        for p in partials:
            tot = tot + p.pack()
    return ShardResult.unpack(tot)


def allreduce_result(part: ShardResult, device=None) -> ShardResult:
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(part.pack())
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t)  # int64 sums wrap mod 2**64, as the hash requires
    return ShardResult.unpack(t.cpu().numpy())


def shard_order_method(world: int) -> str:
    """Ordering method every rank must use: the fastest (async) alone, a
    deterministic one when the roots are split across ranks."""
    return "async" if world <= 1 else "parallel"


def preprocess_for_shards(g, world: int):
    """``preprocess`` with an ordering every rank reproduces bit-for-bit."""
    from paper_2212_01473_b200.graph import preprocess

    return preprocess(g, method=shard_order_method(world))


def check_shardable(g2, world: int) -> None:
    """Refuse a graph whose ordering other ranks cannot reproduce."""
    method = getattr(g2, "order_method", None)
    if world > 1 and method is not None and method not in DETERMINISTIC_METHODS:
        raise ValueError(
            f"graph ordered with method={method!r} cannot be sharded: every rank must compute "
            f"the same ordering (use preprocess_for_shards or method='parallel')")


def run_shard(g2, st, cfg: RunConfig, rank: int, world: int, **kw) -> tuple[RunResult, ShardResult]:
    """Enumerate this rank's static shard (no collective)."""
    if world > 1 and cfg.roots == "l2":
        raise ValueError("sharding is defined over first-level roots")
    check_shardable(g2, world)
    res = run(g2, st, cfg, **shard_bounds(rank, world), **kw)
    return res, ShardResult.of(res)


def run_sharded(g2, st, cfg: RunConfig, rank: int, world: int, device=None,
                **kw) -> tuple[RunResult, ShardResult]:
    """Enumerate this rank's shard on its GPU, then all-reduce the totals."""
    res, part = run_shard(g2, st, cfg, rank, world, **kw)
    if world == 1:
        return res, part
    return res, allreduce_result(part, device)


def claim_chunks(store, key: str, rank: int, world: int, chunks: int):
    """Chunk ids this rank runs: its static chunk ``rank`` first, then
    chunks ``world, world+1, ...`` claimed off the shared counter ``key``
    (each id handed out exactly once across ranks)."""
    if rank < chunks:
        yield rank
    while True:
        k = world + int(store.add(key, 1)) - 1
        if k >= chunks:
            return
        yield k


def agreed_job_id(store, world: int) -> int:
    """A job id every rank of this job derives identically from one shared
    counter: each rank adds 1 once per job, and no rank can add for job j+1
    before every rank added for job j (job j ends in an all-reduce every rank
    joins), so ``(value - 1) // world`` is the same on all of them -- whatever
    each process's own call history."""
    return (int(store.add("mce_steal_jobs", 1)) - 1) // max(world, 1)


def run_work_stealing(g2, st, cfg: RunConfig, rank: int, world: int, chunks: int | None = None,
                      device=None, store=None, runner=run, job_id: int | None = None,
                      **kw) -> tuple[list[RunResult], ShardResult]:
    """Static + dynamic sharding of the first-level roots (module docstring);
    returns this rank's per-chunk results and the all-reduced totals.
    ``job_id`` names the shared claim counter; by default it is agreed
    through the store (``agreed_job_id``)."""
    import torch.distributed as dist

    if cfg.roots == "l2":
        raise ValueError("sharding is defined over first-level roots")
    chunks = chunks or 4 * world
    if chunks < world:
        raise ValueError("need at least one chunk per rank")
    check_shardable(g2, world)
    if store is None:
        store = dist.distributed_c10d._get_default_store()
    if job_id is None:
        job_id = agreed_job_id(store, world)
    key = f"mce_steal_{job_id}"
    results, parts = [], []
    for k in claim_chunks(store, key, rank, world, chunks):
        res = runner(g2, st, cfg, root_begin=k, root_end=-1, root_stride=chunks, **kw)
        results.append(res)
        parts.append(ShardResult.of(res))
    part = combine(parts) if parts else ShardResult(0, 0, 0, 0, {})
    if world <= 1:
        return results, part
    tot = allreduce_result(part, device)
    if rank == 0:  # every rank is past its claims once the all-reduce returns
        try:
            store.delete_key(key)
        except Exception:  # stores without delete (HashStore in old torch): harmless leftover
            pass
    return results, tot

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

Either way the single collective is the final reduction of counts, node
totals, size histograms and the order-independent clique-set hash (sum mod
2**64), done with one NCCL all-reduce (gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2212_01473_b200.scheduler import RunConfig, RunResult, run

HIST_WORDS = 128  # clique sizes reduced individually (larger sizes fold into the last slot)
MASK64 = (1 << 64) - 1


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
            v[4 + min(s, HIST_WORDS - 1)] += c
        return v

    @staticmethod
    def unpack(v: np.ndarray) -> "ShardResult":
        hist = {s: int(v[4 + s]) for s in range(HIST_WORDS) if v[4 + s]}
        return ShardResult(int(v[0]), int(v[1]), int(v[2]), int(v[3]) & MASK64, hist)


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


def run_sharded(g2, st, cfg: RunConfig, rank: int, world: int, device=None,
                **kw) -> tuple[RunResult, ShardResult]:
    """Enumerate this rank's shard on its GPU, then all-reduce the totals."""
    if world > 1 and cfg.roots == "l2":
        raise ValueError("sharding is defined over first-level roots")
    res = run(g2, st, cfg, **shard_bounds(rank, world), **kw)
    part = ShardResult(res.clique_count, res.nodes_total, res.donation_count,
                       res.clique_hash, res.size_histogram)
    if world == 1:
        return res, part
    return res, allreduce_result(part, device)


_steal_epoch = 0


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


def run_work_stealing(g2, st, cfg: RunConfig, rank: int, world: int, chunks: int | None = None,
                      device=None, store=None, runner=run,
                      **kw) -> tuple[list[RunResult], ShardResult]:
    """Static + dynamic sharding of the first-level roots (module docstring);
    returns this rank's per-chunk results and the all-reduced totals."""
    global _steal_epoch
    import torch.distributed as dist

    if cfg.roots == "l2":
        raise ValueError("sharding is defined over first-level roots")
    chunks = chunks or 4 * world
    if chunks < world:
        raise ValueError("need at least one chunk per rank")
    if store is None:
        store = dist.distributed_c10d._get_default_store()
    _steal_epoch += 1  # every rank calls in the same order: same key per job
    key = f"mce_steal_{_steal_epoch}"
    results, parts = [], []
    for k in claim_chunks(store, key, rank, world, chunks):
        res = runner(g2, st, cfg, root_begin=k, root_end=-1, root_stride=chunks, **kw)
        results.append(res)
        parts.append(ShardResult(res.clique_count, res.nodes_total, res.donation_count,
                                 res.clique_hash, res.size_histogram))
    part = combine(parts) if parts else ShardResult(0, 0, 0, 0, {})
    return results, (allreduce_result(part, device) if world > 1 else part)

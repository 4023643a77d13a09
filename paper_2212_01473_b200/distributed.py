"""Multi-GPU enumeration: first-level subtrees sharded across ranks.

One process per GPU (``torch.distributed``).  The subtree roots are
independent (paper §3.1), so ranks need no data-path communication: rank r
enumerates the roots ``r, r + world, r + 2*world, ...`` of the degeneracy-
reordered graph -- a static interleave over vertex ids, which spreads the
heavy late-ordered roots evenly -- with its own device-wide worker list for
intra-GPU balance.  The single collective is the final reduction of counts,
node totals, size histograms and the order-independent clique-set hash
(sum mod 2**64), done with one NCCL all-reduce (gloo on CPU tests).
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

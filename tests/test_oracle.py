"""Pin the CPU oracle (oracle/) against vectors produced by the reference itself.

tests/golden/reference_vectors.json was written by tests/golden/make_golden.py,
which imports the reference package; every field the oracle computes must
match it exactly: degeneracy ordering, per-mode clique count, search-tree node
total, size histogram and clique-set hash.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle
from conftest import golden_cases

CASES = golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference_vectors(case):
    n = case["n"]
    edges = np.asarray(case["edges"], dtype=np.int64).reshape(-1, 2)
    ro, ci = oracle.from_edges(edges, n)
    assert len(ci) // 2 == case["m"]
    pos, d = oracle.degeneracy_order(ro, ci)
    assert d == case["degeneracy"]
    assert pos.tolist() == case["position"]
    ro2, ci2 = oracle.reorder(ro, ci, pos)
    inv = np.empty(n, dtype=np.int64)
    inv[pos] = np.arange(n)
    for mode, exp in case["runs"].items():
        roots, induced = mode.split("-")
        got = oracle.enumerate_cliques(ro2, ci2, roots=roots, induced=induced,
                                       degeneracy=d, labels=inv, threads=2)
        assert got["count"] == exp["count"], mode
        assert got["nodes"] == exp["nodes"], mode
        assert got["hash"] == exp["hash"], mode
        assert {str(k): v for k, v in got["hist"].items()} == exp["hist"], mode


@pytest.mark.parametrize("case", [c for c in CASES if "brute_force" in c],
                         ids=[c["name"] for c in CASES if "brute_force" in c])
def test_oracle_clique_sets_match_brute_force(case):
    n = case["n"]
    edges = np.asarray(case["edges"], dtype=np.int64).reshape(-1, 2)
    expected = {tuple(c) for c in case["brute_force"]}
    for roots in ("l1", "l2"):
        for induced in ("ip", "ipx"):
            got = oracle.reference_pipeline(edges, n, roots=roots, induced=induced,
                                            collect=1 << 16, threads=1)
            ro, ci = oracle.from_edges(edges, n)
            pos, _ = oracle.degeneracy_order(ro, ci)
            inv = np.empty(n, dtype=np.int64)
            inv[pos] = np.arange(n)
            cl = {tuple(sorted(int(inv[v]) for v in c)) for c in got["cliques"]}
            assert cl == expected
            assert got["count"] == len(expected)


def test_hash_is_order_independent():
    a = oracle.summarize_cliques([(1, 2, 3), (4, 5)])
    b = oracle.summarize_cliques([(5, 4), (3, 1, 2)])
    assert a == b
    assert oracle.clique_hash([1, 2]) != oracle.clique_hash([1, 3])


def test_bucket_peel_order_is_a_degeneracy_order():
    """The parallel-order restatement (checker of the GPU peel) yields the
    reference's degeneracy on every golden graph and a valid permutation."""
    from conftest import golden_cases

    for case in golden_cases():
        edges = np.asarray(case["edges"], dtype=np.int64).reshape(-1, 2)
        ro, ci = oracle.from_edges(edges, case["n"])
        pos, d = oracle.bucket_peel_order(ro, ci)
        assert d == case["degeneracy"]
        assert sorted(pos.tolist()) == list(range(case["n"]))
        ro2, ci2 = oracle.reorder(ro, ci, pos)
        later = [int(np.sum(ci2[ro2[v]:ro2[v + 1]] > v)) for v in range(case["n"])]
        assert max(later, default=0) == d

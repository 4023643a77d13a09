"""Edge-list text parsing on the device (mce_graph_from_text) against the
reference's own parse_edge_list: golden vectors made by running the
reference (tests/golden/make_parse_golden.py) -- vertex count, canonical
CSR, or the first malformed line's number and message -- plus a large
generated file checked against a numpy restatement."""

from __future__ import annotations

import io
import json
import os

import numpy as np
import pytest

from oracle import oracle
from paper_2212_01473_b200 import EdgeListParseError, generate, parse_edge_list

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "parse_vectors.json")
CASES = json.load(open(GOLDEN))["cases"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_parse_matches_reference(case):
    if "error_line" in case:
        with pytest.raises(EdgeListParseError) as exc:
            parse_edge_list(io.StringIO(case["text"]), base=case["base"])
        assert exc.value.line_no == case["error_line"]
        assert str(exc.value) == case["error"]
        return
    g = parse_edge_list(io.StringIO(case["text"]), base=case["base"])
    assert g.num_vertices == case["n"]
    assert g.row_offsets.tolist() == case["row_offsets"]
    assert g.col_indices.tolist() == case["col_indices"]
    # str / bytes sources parse the same
    g2 = parse_edge_list(case["text"].encode(), base=case["base"])
    assert g2.col_indices.tolist() == case["col_indices"]


def test_parse_large_snap_style_file():
    """~3.2M lines with comments, sparse ids, duplicates and a trailing
    line without newline: same canonical CSR as a numpy restatement."""
    edges = generate.barabasi_albert_edges(200_000, 8, seed=5)
    ids = (edges * 7 + 11).astype(np.int64)  # sparse, non-contiguous ids
    lines = [f"{u}\t{v}" for u, v in ids.tolist()]
    text = "# SNAP-style header\n# Nodes: ? Edges: ?\n" + "\n".join(lines)
    g = parse_edge_list(text)
    uniq, inv = np.unique(ids, return_inverse=True)
    ro, ci = oracle.from_edges(inv.reshape(-1, 2), len(uniq))
    assert g.num_vertices == len(uniq)
    assert np.array_equal(g.row_offsets, ro) and np.array_equal(g.col_indices, ci)


def test_parse_rejects_bad_base():
    with pytest.raises(ValueError):
        parse_edge_list("0 1\n", base=2)

"""Golden vectors for edge-list parsing, made by running the REFERENCE's
parse_edge_list (reference graph.py:132-180) here.  Run:
    python tests/golden/make_parse_golden.py
Writes tests/golden/parse_vectors.json (committed; tests never read
/root/reference)."""

from __future__ import annotations

import io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from mce.graph import EdgeListParseError, parse_edge_list  # noqa: E402  (reference)

CASES = [
    ("plain", "0 1\n1 2\n# comment\n% other comment\n\n2 0\n", 0),
    ("one_based", "1 2\n2 3\n", 1),
    ("sparse_ids", "10 20\n20 999\n", 0),
    ("loops_dups", "1 2\n2 1\n1 1\n", 1),
    ("fig1a", "0 1\n0 2\n0 3\n1 2\n1 3\n2 3\n0 4\n0 5\n4 5\n", 0),
    ("whitespace", "  3\t4  \r\n\t\n 4   5\n\v5 3\f\n", 0),
    ("no_trailing_newline", "0 1\n1 2", 0),
    ("signs_underscores", "+1 2\n1_0 2\n007 3\n", 0),
    ("matrix_market", "%%MatrixMarket matrix coordinate pattern symmetric\n% c\n4 4 3\n1 2\n2 3\n3 4 1.5\n", 0),
    ("mm_after_data", "0 1\n%%MatrixMarket matrix coordinate pattern general\n9 9 9\n2 3\n", 0),
    ("only_comments", "# nothing\n% here\n\n", 0),
    ("empty", "", 0),
    ("size_line_only", "%%MatrixMarket matrix\n3 3 0\n", 0),
    ("err_token_count", "0 1\n0 1 2 3\n", 0),
    ("err_single_token", "0 1\n\n5\n", 0),
    ("err_non_integer", "0 1\nnot numbers\n", 0),
    ("err_float", "0 1\n1.5 2\n", 0),
    ("err_below_base", "1 2\n0 1\n", 1),
    ("err_negative", "0 1\n-3 2\n", 0),
    ("err_first_of_many", "0 1\nx y\n1 2 3\n", 0),
    ("err_bad_underscore", "1__0 2\n", 0),
]


def main() -> None:
    out = []
    for name, text, base in CASES:
        rec = {"name": name, "text": text, "base": base}
        try:
            g = parse_edge_list(io.StringIO(text), base=base)
            rec["n"] = int(g.num_vertices)
            rec["edges"] = [[int(u), int(v)] for u, v in g.edges()]
            rec["row_offsets"] = [int(x) for x in np.asarray(g.row_offsets)]
            rec["col_indices"] = [int(x) for x in np.asarray(g.col_indices)]
        except EdgeListParseError as exc:
            rec["error_line"] = exc.line_no
            rec["error"] = str(exc)
        out.append(rec)
    with open(os.path.join(HERE, "parse_vectors.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_parse_golden.py",
                   "reference": "/root/reference/pkg (mce 0.1.0) graph.parse_edge_list",
                   "cases": out}, fh, indent=1)
    print(f"{len(out)} cases")


if __name__ == "__main__":
    main()

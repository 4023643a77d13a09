import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from conftest import golden_cases
from paper_2212_01473_b200 import from_edges, preprocess, run, RunConfig
for name in ("gnp_200_0.5_s3", "gnp_300_0.08_s42", "skew_2000_40", "gnp_96_0.25_s11", "moon_moser_5"):
    case = next(c for c in golden_cases() if c["name"] == name)
    g = from_edges(np.asarray(case["edges"], dtype=np.int64).reshape(-1, 2), case["n"])
    g2, _, st = preprocess(g, method="exact")
    exp = case["runs"]["l1-ipx"]
    out = []
    for workers in (2, 8, 64, 0):
        for rep in range(3):
            r = run(g2, st, RunConfig(workers=workers, induced="ipx", donation_min_p=2))
            out.append((workers, r.donation_count, r.nodes_total - exp["nodes"], r.clique_count == exp["count"]))
    print(name, exp["nodes"], out, flush=True)

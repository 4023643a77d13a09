"""Ad-hoc diagnostics on the GPU box (not part of the product)."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2212_01473_b200 import *
from paper_2212_01473_b200 import generate
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import golden_cases

def donation_check():
    case = next(c for c in golden_cases() if c["name"] == "gnp_200_0.5_s3")
    g = from_edges(np.asarray(case["edges"]).reshape(-1, 2), case["n"])
    g2, _, st = preprocess(g, method="exact")
    for mode in ("l1-ipx", "l1-ip"):
        r, i = mode.split("-")
        print(mode, "expected", case["runs"][mode])
        for workers in (1, 8, 64, 0):
            for wl in (False, True):
                res = run(g2, st, RunConfig(workers=workers, roots=r, induced=i, worker_list=wl))
                made = sum(w.donations_made for w in res.worker_metrics)
                recv = sum(w.donations_received for w in res.worker_metrics)
                wn = sum(w.nodes_visited for w in res.worker_metrics)
                print(f"  workers={workers} wl={wl} count={res.clique_count} nodes={res.nodes_total} wnodes={wn} hash={res.clique_hash_hex} don={res.donation_count} made={made} recv={recv}")

def timing(name):
    e, n = generate.workload_edges(name)
    t = time.perf_counter(); g = from_edges(e, n); t1 = time.perf_counter()
    o = degeneracy_order(g); t2 = time.perf_counter()
    g2 = reorder(g, o); t3 = time.perf_counter()
    st = stats(g2, o)
    res = run(g2, st, RunConfig()); t4 = time.perf_counter()
    res = run(g2, st, RunConfig()); t5 = time.perf_counter()
    print(f"{name}: from_edges {t1-t:.4f}s order {t2-t1:.4f}s reorder {t3-t2:.4f}s run {t4-t3:.4f}s run2 {t5-t4:.4f}s count={res.clique_count} nodes={res.nodes_total} d={st.degeneracy} launches={res.kernel_launches} workers={res.workers} don={res.donation_count}")

if __name__ == "__main__":
    for a in sys.argv[1:]:
        if a == "don": donation_check()
        else: timing(a)

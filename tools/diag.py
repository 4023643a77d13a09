"""Ad-hoc diagnostics on the GPU box (not part of the product).
usage: python tools/diag.py <workload|don> [...] [--stride K]"""
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

def timing(name, stride=1, reps=3, begin=0, end=-1):
    e, n = generate.workload_edges(name)
    for rep in range(reps):
        t = time.perf_counter(); g = from_edges(e, n); t1 = time.perf_counter()
        tp = time.perf_counter(); degeneracy_order(g); tp = time.perf_counter() - tp
        print(f"  degeneracy_order(parallel) {1e3*tp:.2f}ms", flush=True)
        g2, o, st = preprocess(g); t2 = time.perf_counter()
        res = run(g2, st, RunConfig(), root_stride=stride, root_begin=begin, root_end=end); t3 = time.perf_counter()
        print(f"{name}[{rep}] roots[{begin}:{end}:{stride}]: from_edges {1e3*(t1-t):.2f}ms preprocess {1e3*(t2-t1):.2f}ms run {1e3*(t3-t2):.2f}ms "
              f"(kernel {res.kernel_ms:.2f}ms) count={res.clique_count} nodes={res.nodes_total} d={st.degeneracy} "
              f"maxdeg={st.max_degree} induced={res.induced_mode} launches={res.kernel_launches} workers={res.workers} "
              f"don={res.donation_count} maxsize={res.max_clique_size}", flush=True)

if __name__ == "__main__":
    args = sys.argv[1:]
    opt = {"stride": 1, "begin": 0, "end": -1, "reps": 3}
    for k in list(opt):
        if "--" + k in args:
            i = args.index("--" + k); opt[k] = int(args[i + 1]); del args[i:i + 2]
    for a in args:
        if a == "don": donation_check()
        else: timing(a, **opt)

"""Run the REFERENCE's own scheduler (reference scheduler.py) with the worker
list on and donations forced (donation_min_p=2) on gnp(200, 0.5, seed=3) in
full ("ipx") mode, several times: the node totals it reports, next to its
worker-list-off total.  Evidence for the X_X prefix-order dependence of ipx
node totals under donation (xsets.py:55-78 partitions in place and never
restores; a donated branch is partitioned in the receiver, not the donor).
Run:  python tests/golden/ref_ipx_donation_probe.py > profiles/r2/ref_ipx_donation_probe.txt
"""
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")

from mce.generate import gnp  # noqa: E402  (reference)
from mce.graph import preprocess  # noqa: E402  (reference)
from mce.scheduler import RunConfig, run  # noqa: E402  (reference)

g2, _, st = preprocess(gnp(200, 0.5, seed=3))
base = run(g2, st, RunConfig(workers=1, induced="ipx", worker_list=False))
nb = sum(w.nodes_visited for w in base.worker_metrics)
print(f"reference, worker list off: count={base.clique_count} nodes={nb}", flush=True)
for rep in range(6):
    t0 = time.time()
    res = run(g2, st, RunConfig(workers=8, induced="ipx", worker_list=True, donation_min_p=2))
    n = sum(w.nodes_visited for w in res.worker_metrics)
    print(f"reference, 8 workers, donations on: count={res.clique_count} nodes={n} "
          f"(delta {n - nb:+d}) donations={res.donation_count} ({time.time() - t0:.0f}s)", flush=True)

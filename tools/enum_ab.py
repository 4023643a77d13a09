"""A/B of enumeration-kernel variants on one preprocessed graph (diagnostics).
usage: python tools/enum_ab.py <workload>[:begin:end:stride] ... [--env VAR=a,b] [--reps N]
Runs every value of the env knob (default MCE_COMPACT=0,1) on the same
reordered graph; prints median kernel ms and checks count/nodes/hash agree."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_01473_b200 import RunConfig, from_edges, from_device_edges, preprocess, run, generate, _lib

args = [a for a in sys.argv[1:] if not a.startswith("--")]
env = "MCE_COMPACT=0,1"
reps = 5
for i, a in enumerate(sys.argv):
    if a == "--env": env = sys.argv[i + 1]
    if a == "--reps": reps = int(sys.argv[i + 1])
args = [a for a in args if a != env and a != str(reps)]
var, vals = env.split("=")
for spec in args:
    parts = spec.split(":")
    name = parts[0]
    b, e, s = (int(x) for x in parts[1:4]) if len(parts) == 4 else (0, -1, 1)
    if name.startswith("rmat"):
        scale = int(name[4:]); m, n = 16 << scale, 1 << scale
        dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
        g = from_device_edges(dev, m, n); del dev
    else:
        edges, n = generate.workload_edges(name)
        g = from_edges(edges, n)
    g2, _, st = preprocess(g, method="parallel")
    ref = None
    for v in vals.split(","):
        os.environ[var] = v
        ms = []
        for _ in range(reps):
            r = run(g2, st, RunConfig(), root_begin=b, root_end=e, root_stride=s)
            ms.append(r.kernel_ms)
        key = (r.clique_count, r.nodes_total, r.clique_hash_hex)
        ok = "" if ref is None or key == ref else "  MISMATCH vs first variant!"
        ref = ref or key
        print(f"{spec} {var}={v}: kernel median {statistics.median(ms):.3f} ms (min {min(ms):.3f}) "
              f"count={r.clique_count} nodes={r.nodes_total} hash={r.clique_hash_hex} "
              f"don={r.donation_count} -> {r.clique_count / (statistics.median(ms) / 1e3) / 1e6:.1f} M/s{ok}",
              flush=True)

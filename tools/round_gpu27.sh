out=gpurun_out
# one call over a strided sample of the whole rmat20 core (all workers busy through donation)
timeout -s KILL 400 python - > $out/rmat20_core_r1v.txt 2>&1 <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess, run, _lib
scale = 20; m, n = 16 << scale, 1 << scale
dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
_lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
g = from_device_edges(dev, m, n); del dev
g2, order, st = preprocess(g)
print(f"rmat20 d={st.degeneracy}", flush=True)
for stride in (512, 128, 32):
    t = time.perf_counter()
    res = run(g2, st, RunConfig(), root_begin=n - 8576, root_end=n, root_stride=stride)
    print(f"core stride {stride}: roots {8576//stride} count={res.clique_count} nodes={res.nodes_total} max={res.max_clique_size} "
          f"kernel {res.kernel_ms:.1f} ms wall {time.perf_counter()-t:.1f}s don={res.donation_count} launches={res.kernel_launches} "
          f"-> {res.clique_count/(res.kernel_ms/1e3)/1e6:.1f} M cliques/s; est full core x{stride}: {res.kernel_ms*stride/1e3:.0f} s, {res.clique_count*stride:.3g} cliques", flush=True)
PY
echo "rc=$?"; cat $out/rmat20_core_r1v.txt

"""Benchmark: end-to-end maximal clique enumeration on B200 (BASELINE.json metric
"end-to-end MCE seconds and maximal cliques/sec at 1/2/4/8 B200 vs CPU ref").

One step = one full MCE job over one synthetic graph: degeneracy ordering +
reordering + enumeration (the paper's GPU time, Table 1 / appendix: "the time
includes both the degeneracy ordering time and the maximal clique counting
time").  `value` is maximal cliques per second with the canonical graph
already resident in HBM; `e2e` is the same metric through the public API from
pinned host edges (H2D copy, canonicalisation, ordering, enumeration, D2H of
the result inside the timed region).

Multi-GPU: first-level subtrees are partitioned across ranks (strided
sample of the heavy-first root order), each rank runs its share with no
collective on the data path, and one NCCL all-reduce combines counts,
node totals and clique-set hashes at the end.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOAD_CONFIG = {
    "er2k": "Erdos-Renyi G(n=2000, p=0.01), reference gnp seed 0",
    "ba200k": "Barabasi-Albert n=200k, m=8",
    "rmat20": "RMAT scale-20, edge factor 16",
    "planted1m": "ER n=1M avg deg 20 + 1k planted cliques of size 30-60",
    "rmat24": "RMAT scale-24, edge factor 16",
}


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--workload", default=os.environ.get("MCE_BENCH_WORKLOAD", "ba200k"),
                   choices=sorted(WORKLOAD_CONFIG))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


class ClockSampler:
    """Samples nvidia-smi clocks/throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.samples: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                row = [x.strip() for x in out.stdout.strip().split(",")]
                if len(row) == 6:
                    self.samples.append(row)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.samples if r[0].replace(".", "").isdigit())
        smax = max(float(r[1]) for r in self.samples if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.samples for i in range(4)
                          if r[2 + i].lower() in ("active", "1")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax,
                "reasons": reasons, "samples": len(self.samples)}


def load_workload(name: str, seed: int, on_device: bool):
    """(edges, n): host numpy edges, or a device tensor for rmat24."""
    from paper_2212_01473_b200 import generate

    if name in ("rmat20", "rmat24") and on_device:
        import torch

        from paper_2212_01473_b200 import _lib

        scale = 20 if name == "rmat20" else 24
        m = 16 << scale
        dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, seed, _lib.ptr(dev), None),
                   "mce_gen_rmat")
        torch.cuda.synchronize()
        return dev, 1 << scale
    return generate.workload_edges(name, seed)


def main():
    args = parse_args()
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    if args.impl == "reference":
        return run_reference(args, rank, world)
    from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess, run
    from paper_2212_01473_b200 import _lib
    from paper_2212_01473_b200.graph import from_edges

    _lib.require_device()
    edges, n = load_workload(args.workload, args.seed, on_device=True)
    if isinstance(edges, np.ndarray):
        host_edges = torch.from_numpy(edges).pin_memory()
        dev_edges = host_edges.cuda()
    else:
        dev_edges = edges
        host_edges = edges.cpu().pin_memory()
    m_raw = dev_edges.shape[0]
    torch.cuda.synchronize()
    g = from_device_edges(dev_edges, m_raw, n)
    del dev_edges
    cfg = RunConfig(roots="l1", induced="auto")

    def step_device():
        g2, order, st = preprocess(g)
        res = run(g2, st, cfg, root_begin=rank, root_stride=world) if world > 1 else \
            run(g2, st, cfg)
        return res, st

    def step_e2e():
        ge = from_edges(host_edges.numpy(), n)
        g2, order, st = preprocess(ge)
        res = run(g2, st, cfg, root_begin=rank, root_stride=world) if world > 1 else \
            run(g2, st, cfg)
        return res, st

    for _ in range(args.warmup):
        res, st = step_device()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    results = []
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            res, st = step_device()
            results.append(res)
        ev1.record()
        torch.cuda.synchronize()
    dev_ms = ev0.elapsed_time(ev1) / args.steps
    # e2e through the public API from pinned host edges
    for _ in range(1):
        step_e2e()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        res_e, _ = step_e2e()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    res = results[-1]
    count = res.clique_count
    if world > 1:
        t = torch.tensor([dev_ms, e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, e2e_ms = float(t[0]), float(t[1])
        c = torch.tensor([count, res.nodes_total], dtype=torch.int64, device="cuda")
        dist.all_reduce(c)
        count = int(c[0])
    if rank != 0:
        return
    line = {
        "metric": "maximal cliques/sec (end-to-end MCE: ordering + reorder + enumeration)",
        "value": count / (dev_ms / 1e3),
        "unit": "cliques/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD_CONFIG[args.workload], "n": n, "m": st.m,
                   "degeneracy": st.degeneracy, "max_degree": st.max_degree,
                   "roots": cfg.roots, "induced": res.induced_mode,
                   "maximal_cliques": count, "nodes": res.nodes_total,
                   "clique_hash": res.clique_hash_hex, "l2_flush": "inputs > L2"},
        "e2e": {"value": count / (e2e_ms / 1e3), "unit": "cliques/s",
                "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(host_edges.numel() * 8),
                "d2h_bytes_per_step": int(8 * (8 + 4096))},
        "gpu_launches": int(res.kernel_launches),
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def run_reference(args, rank: int, world: int):
    """The reference algorithm on host cores (the C restatement in oracle/)."""
    if rank != 0:
        return
    from oracle import oracle

    edges, n = load_workload(args.workload, args.seed, on_device=False)
    times = []
    out = None
    threads = os.cpu_count() or 1
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        out = oracle.reference_pipeline(edges, n, roots="l1", induced="auto", threads=threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    sec = sum(times) / len(times)
    val = out["count"] / sec
    line = {"impl": "reference", "metric": "maximal cliques/sec", "value": val,
            "unit": "cliques/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True,
            "config": {"workload": WORKLOAD_CONFIG[args.workload], "maximal_cliques": out["count"]},
            "cpu_baseline": {"value": val, "unit": "cliques/s", "cores": threads, "kind": "port",
                             "sample": "full workload"},
            "e2e": {"value": val, "unit": "cliques/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

"""Benchmark: end-to-end maximal clique enumeration on B200.

BASELINE.json metric: "end-to-end MCE seconds and maximal cliques/sec at
1/2/4/8 B200 vs CPU ref".  One step = one full MCE job over one synthetic
graph: degeneracy ordering + reordering + enumeration of every maximal clique
(the paper's GPU time: "includes both the degeneracy ordering time and the
maximal clique counting time").

* ``value``  -- maximal cliques/s with the canonical graph already in HBM.
* ``e2e``    -- the same metric through the public API from pinned host edges:
                H2D copy, canonicalisation, ordering, enumeration and the D2H
                of the result inside the timed region.
* ``roofline`` -- the enumeration kernels against HBM: algorithmic bytes =
                the CSR bytes every root's induced-subgraph build must read
                (DESIGN.md "roofline"), over their CUDA-event time.
* ``cpu_baseline`` -- the reference algorithm (C restatement in oracle/, all
                host threads) on a bounded sample of the same workload.

Default workload: configs[3] (planted cliques, ER n=1M avg deg 20 + 1k
cliques of size 30-60) -- the largest BASELINE config whose full enumeration
fits a bench step (rmat20's core alone takes minutes: see DESIGN.md).  N>1
shards the first-level subtrees across ranks (every rank computes the same
deterministic ordering; no data-path collective; one NCCL all-reduce of
counts, histogram and clique-set hash); scaling is "strong".
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
FALLBACK_HBM_GBS = 6650.0
L2_POLICY = ("GPU arm: a 256 MiB buffer is zeroed between timed steps (outside the CUDA "
             "events), so every step starts from a cold L2; CPU arm: not applicable")
ORDERING = {"async": "async peel (degeneracy order, no rounds inside a level)",
            "parallel": "parallel bucket peel (deterministic degeneracy order, same on every rank)",
            "exact": "the reference's exact degeneracy order"}


def workload_config(name, n, m, degeneracy, max_degree, roots, induced) -> dict:
    """The workload both arms report (identical keys and values)."""
    return {"workload": WORKLOAD_CONFIG[name], "name": name, "n": int(n), "m": int(m),
            "degeneracy": int(degeneracy), "max_degree": int(max_degree), "roots": roots,
            "induced": induced, "l2_flush": L2_POLICY}
METRIC = "maximal cliques/sec (end-to-end MCE: degeneracy order + reorder + enumerate)"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--workload", default=os.environ.get("MCE_BENCH_WORKLOAD", "planted1m"),
                   choices=sorted(WORKLOAD_CONFIG))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--root-stride", type=int, default=1,
                   help="enumerate every k-th first-level root (bounded samples of huge graphs)")
    p.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-clocks", action="store_true", help="diagnostics: no nvidia-smi sampling")
    p.add_argument("--shard", default="static", choices=["static", "steal"],
                   help="N>1: static interleave, or static + work-stealing chunks")
    return p.parse_args()


class ClockSampler:
    """Samples SM clocks and clock-event (throttle) reasons DURING the timed
    region through NVML in-process, falling back to nvidia-smi.  The bench
    calls ``sample_now()`` between timed steps (after a step's end event,
    before the next start event): a concurrent sampler thread contends with
    the CUDA driver calls of a millisecond-scale step and shows up as GPU
    idle time inside the events."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int = 0, enabled: bool = True, period: float = 0.01):
        self.index = index
        self.enabled = enabled
        self.period = period
        self.samples: list[tuple[float | None, float | None, set]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._nvml = None

    def _nvml_init(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self._nvml = (pynvml, h, bits)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        pynvml, h, bits = self._nvml
        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        return sm, mx, {k for k, b in bits.items() if r & b}

    def _sample_smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={fields}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5)
        row = [x.strip() for x in out.stdout.strip().split(",")]
        if len(row) != 6:
            return None

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        return num(row[0]), num(row[1]), {self.NAMES[i] for i in range(4)
                                         if row[2 + i].lower() in ("active", "1")}

    def _loop(self):
        while not self._stop.is_set():
            try:
                smp = self._sample_nvml() if self._nvml else self._sample_smi()
                if smp:
                    self.samples.append(smp)
            except Exception:
                pass
            self._stop.wait(self.period if self._nvml else 0.1)

    def sample_now(self):
        if not self.enabled:
            return
        try:
            smp = self._sample_nvml() if self._nvml else self._sample_smi()
            if smp:
                self.samples.append(smp)
        except Exception:
            pass

    def __enter__(self):
        if self.enabled:
            self._nvml_init()
        return self

    def __exit__(self, *exc):
        self._stop.set()

    def summary(self) -> dict:
        sm = sorted(x[0] for x in self.samples if x[0] is not None)
        mx = [x[1] for x in self.samples if x[1] is not None]
        reasons = sorted(set().union(*[x[2] for x in self.samples])) if self.samples else []
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nvml else "nvidia-smi"}


def measured_hbm_peak() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback"


def ncu_traffic(workload: str):
    """DRAM bytes of one step's enumeration launches from the committed ncu
    capture (profiles/traffic.json), plus that capture's L2 bytes and issue /
    warp-occupancy figures (the enumeration is latency/issue bound, not HBM
    bound: these say how far from which roof)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get(workload), d.get("_detail", {}).get(workload)
    except (OSError, ValueError):
        return None, None


def load_workload(name: str, seed: int, on_device: bool):
    """(edges, n): host numpy edges, or a device tensor for the R-MAT graphs."""
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


def cpu_reference_step(ro, ci, root_stride: int, threads: int, pre=None):
    """The reference algorithm on host cores: exact degeneracy order,
    reorder, enumeration of a strided root sample (oracle/, C + numpy)."""
    from oracle import oracle

    ro2, ci2, d, labels = pre if pre is not None else cpu_preprocess(ro, ci)
    n = len(ro) - 1
    max_degree = int(np.diff(ro2).max()) if n else 0
    induced = "ip" if d > 0 and max_degree / d > 200.0 else "ipx"
    return oracle.enumerate_cliques(ro2, ci2, roots="l1", induced=induced, degeneracy=d,
                                    labels=labels, root_stride=root_stride, threads=threads)


def cpu_preprocess(ro, ci):
    from oracle import oracle

    pos, d = oracle.degeneracy_order(ro, ci)
    ro2, ci2 = oracle.reorder(ro, ci, pos)
    labels = np.empty_like(pos)
    labels[pos] = np.arange(len(pos), dtype=pos.dtype)  # original id of every rank
    return ro2, ci2, d, labels


def choose_cpu_stride(ro, ci, target_s: float, threads: int) -> tuple[int, float, dict]:
    """Root stride so one CPU step (ordering + enumeration) costs about
    target_s seconds: the ordering is timed once, the enumeration on a
    1/64 probe sample."""
    t0 = time.perf_counter()
    pre = cpu_preprocess(ro, ci)
    t_pre = time.perf_counter() - t0
    probe = 64
    t0 = time.perf_counter()
    cpu_reference_step(ro, ci, probe, threads, pre)
    est_enum = (time.perf_counter() - t0) * probe
    budget = max(target_s - t_pre, 1.0)
    stride = 1 if est_enum <= budget else int(np.ceil(est_enum / budget))
    return stride, t_pre, {"est_enum_s": est_enum}


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch
    import torch.distributed as dist

    if world > 1:
        # MCE_BENCH_BACKEND=gloo with more ranks than GPUs: a functional check
        # of the N > 1 path on one GPU (ranks time-share it) -- never a bench
        # number; the driver's runs take NCCL and one GPU per rank
        backend = os.environ.get("MCE_BENCH_BACKEND", "nccl")
        dev_idx = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
        torch.cuda.set_device(dev_idx)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess
    from paper_2212_01473_b200 import _lib
    from paper_2212_01473_b200.distributed import (run_sharded, run_work_stealing,
                                                   shard_order_method)
    from paper_2212_01473_b200.graph import from_edges

    _lib.require_device()
    edges, n = load_workload(args.workload, args.seed, on_device=True)
    # the e2e arm ships the edge list as int32 pairs (ids < 2^31): half the H2D
    if isinstance(edges, np.ndarray):
        dev_edges = torch.from_numpy(np.ascontiguousarray(edges)).cuda()
        host_edges = torch.from_numpy(np.ascontiguousarray(edges, dtype=np.int32)).pin_memory()
    else:
        dev_edges = edges
        host_edges = edges.to(torch.int32).cpu().pin_memory()
    torch.cuda.synchronize()
    g = from_device_edges(dev_edges, dev_edges.shape[0], n)
    del dev_edges
    cfg = RunConfig(roots="l1", induced="auto")
    stride = max(1, args.root_stride)

    order_method = shard_order_method(world)  # deterministic whenever ranks share the roots

    def one_job(graph, measure=False):
        g2, _, st = preprocess(graph, method=order_method)
        if world > 1 and stride == 1 and args.shard == "steal":
            results, tot = run_work_stealing(g2, st, cfg, rank, world, device="cuda",
                                             measure_bytes=measure)
            res = results[0]
            res.kernel_ms = sum(r.kernel_ms for r in results)
            res.build_bytes = sum(r.build_bytes for r in results)
            return res, tot, st
        if world > 1 or stride > 1:
            res, tot = run_sharded(g2, st, cfg, rank * 1, world * 1, device="cuda",
                                   measure_bytes=measure) \
                if stride == 1 else run_sharded_strided(g2, st, cfg, rank, world, stride, measure)
            return res, tot, st
        from paper_2212_01473_b200 import run

        res = run(g2, st, cfg, measure_bytes=measure)
        return res, None, st

    # algorithmic bytes of one step's induced-subgraph builds (outside the timing)
    build_bytes_step = one_job(g, measure=True)[0].build_bytes
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # 2x the 126 MB L2
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    import gc

    with ClockSampler(local, enabled=not args.no_clocks) as clocks:
        # W warm-up steps shaped like the timed ones (L2 flush first), and at
        # least ~0.5 s of them: a fresh box starts at idle clocks and an empty
        # stream-ordered memory pool
        t_w = time.perf_counter()
        w_done = 0
        while w_done < max(args.warmup, 3) or (time.perf_counter() - t_w < 0.5 and w_done < 1000):
            flush.zero_()
            res, tot, st = one_job(g)
            w_done += 1
        torch.cuda.synchronize()
        # ---- device-resident timed region ----------------------------------
        kernel_ms = 0.0
        launches0 = _lib.lib().mce_launch_count()
        gc.collect()
        gc.disable()  # no collector pauses between the kernels of a timed step
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()  # evict L2 between timed steps (outside the events)
            starts[i].record()
            res, tot, st = one_job(g)
            ends[i].record()
            kernel_ms += res.kernel_ms
            clocks.sample_now()  # between the events: host time only
        torch.cuda.synchronize()
    gc.enable()
    launches = _lib.lib().mce_launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    dev_ms = sum(step_ms) / args.steps
    print(f"[bench] per-step device ms: {[round(x, 3) for x in step_ms]}", file=sys.stderr)
    count = tot.cliques if tot is not None else res.clique_count
    nodes = tot.nodes if tot is not None else res.nodes_total
    chash = f"{tot.hash:016x}" if tot is not None else res.clique_hash_hex
    # ---- end to end through the public API from pinned host edges --------
    e2e_ms = None
    if not args.no_e2e:
        host_np = host_edges.numpy()
        one_job(from_edges(host_np, n))
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        e2e_ms = 0.0
        gc.collect()
        gc.disable()
        for _ in range(args.steps):
            flush.zero_()
            e0.record()
            one_job(from_edges(host_np, n))
            e1.record()
            torch.cuda.synchronize()
            e2e_ms += e0.elapsed_time(e1)
        gc.enable()
        e2e_ms /= args.steps
    if world > 1:
        t = torch.tensor([dev_ms, e2e_ms or 0.0], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, e2e_ms = float(t[0]), (float(t[1]) if e2e_ms is not None else None)
    if rank != 0:
        dist.barrier()
        return
    peak, peak_kind = measured_hbm_peak()
    per_launch_ms = kernel_ms / max(1, args.steps * max(1, res.kernel_launches))
    achieved = build_bytes_step / (kernel_ms / args.steps / 1e3) / 1e9 \
        if kernel_ms > 0 else None
    line = {
        "metric": METRIC,
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
        "config": workload_config(args.workload, n, st.m, st.degeneracy, st.max_degree,
                                  cfg.roots, res.induced_mode),
        "result": {"maximal_cliques": count, "nodes": nodes, "clique_hash": chash,
                   "root_stride": stride,
                   "ordering": ORDERING[order_method],
                   "sharding": args.shard if world > 1 else None},
        "e2e": ({"value": count / (e2e_ms / 1e3), "unit": "cliques/s", "ms_per_step": e2e_ms,
                 "h2d_bytes_per_step": int(host_edges.numel() * host_edges.element_size()),
                 "d2h_bytes_per_step": int(8 * (10 + 4096))} if e2e_ms else None),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": ncu_traffic(args.workload)[0],
                     "ncu": ncu_traffic(args.workload)[1],
                     "kernel": "enumeration kernels (k_tiny lane-per-root + k_enumerate width classes)",
                     "kernel_ms_per_step": kernel_ms / args.steps,
                     "kernel_ms_per_launch": per_launch_ms,
                     "algorithmic_bytes_per_step": build_bytes_step,
                     "peak_source": peak_kind},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(g, args)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()


def run_sharded_strided(g2, st, cfg, rank, world, stride, measure=False):
    """Bounded sample (every stride-th root) split across ranks."""
    from paper_2212_01473_b200.distributed import ShardResult, allreduce_result
    from paper_2212_01473_b200.scheduler import run

    res = run(g2, st, cfg, root_begin=rank, root_stride=stride * world, measure_bytes=measure)
    part = ShardResult(res.clique_count, res.nodes_total, res.donation_count,
                       res.clique_hash, res.size_histogram)
    if world > 1:
        part = allreduce_result(part, "cuda")
    return res, part


def cpu_baseline(g, args) -> dict:
    """Reference algorithm on this host's cores, bounded sample."""
    threads = os.cpu_count() or 1
    ro, ci = g.row_offsets, g.col_indices
    stride, t_probe, _ = choose_cpu_stride(ro, ci, args.cpu_sample_seconds, threads)
    t0 = time.perf_counter()
    out = cpu_reference_step(ro, ci, stride, threads)
    sec = time.perf_counter() - t0
    return {"value": out["count"] / sec, "unit": "cliques/s", "cores": threads, "kind": "port",
            "seconds": sec,
            "sample": (f"all {len(ro) - 1} first-level roots" if stride == 1 else
                       f"every {stride}-th first-level root (count {out['count']})") +
                      "; exact degeneracy order + reorder included"}


def run_reference(args, rank: int, world: int):
    """--impl reference: the reference algorithm (C restatement in oracle/)
    on this box's host cores, same workload/metric; rank 0 only."""
    if rank != 0:
        return
    from oracle import oracle

    threads = os.cpu_count() or 1
    edges, n = load_workload(args.workload, args.seed, on_device=False)
    ro, ci = oracle.from_edges(edges, n)
    stride = max(1, args.root_stride)
    if args.workload in ("rmat20", "rmat24"):
        stride, _, _ = choose_cpu_stride(ro, ci, 20.0, threads)
    times = []
    out = None
    pre = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        pre = cpu_preprocess(ro, ci)
        out = cpu_reference_step(ro, ci, stride, threads, pre)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    sec = sum(times) / len(times)
    val = out["count"] / sec
    d = pre[2]
    max_degree = int(np.diff(ro).max()) if n else 0
    induced = "ip" if d > 0 and max_degree / d > 200.0 else "ipx"
    sample = ("all first-level roots" if stride == 1 else f"every {stride}-th first-level root") + \
        "; exact degeneracy order + reorder + enumeration per step"
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "cliques/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": workload_config(args.workload, n, int(len(ci) // 2), d, max_degree, "l1",
                                      induced),
            "result": {"maximal_cliques": out["count"], "nodes": out["nodes"],
                       "clique_hash": out["hash"], "root_stride": stride,
                       "ordering": ORDERING["exact"], "sharding": None},
            "cpu_baseline": {"value": val, "unit": "cliques/s", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": val, "unit": "cliques/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

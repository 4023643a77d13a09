"""Summarise an ncu --set full report: time, DRAM/L2 traffic and throughput,
issue/pipe utilisation, occupancy and per-SM busy-time spread (load balance).
usage: python tools/ncu_summary.py rep.ncu-rep [> profiles/...txt]"""
import csv, re, subprocess, sys

PATTERNS = [
    r"^gpu__time_duration\.sum$",
    r"^dram__bytes_(read|write)\.sum$",
    r"^gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^dram__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^lts__t_bytes\.sum$",
    r"^lts__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^l1tex__throughput\.avg\.pct_of_peak_sustained_active$",
    r"^l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum$",
    r"^sm__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^sm__inst_executed\.sum$",
    r"^smsp__issue_active\.avg\.pct_of_peak_sustained_active$",
    r"^sm__inst_executed_pipe_(alu|fma|lsu|adu|cbu|uniform|xu)\.avg\.pct_of_peak_sustained_active$",
    r"^sm__pipe_(alu|fma|shared|fmaheavy)_cycles_active\.avg\.pct_of_peak_sustained_active$",
    r"^sm__warps_active\.avg\.pct_of_peak_sustained_active$",
    r"^sm__maximum_warps_per_active_cycle_pct$",
    r"^sm__cycles_active\.(avg|max|min)$",
    r"^sm__cycles_elapsed\.avg$",
    r"^launch__(registers_per_thread|grid_size|block_size|occupancy_limit_.*)$",
    r"^smsp__average_warp_latency_issue_stalled_.*\.ratio$",
    r"^smsp__pcsamp_warps_issue_stalled_(long_scoreboard|short_scoreboard|wait|barrier|membar|lg_throttle|mio_throttle|no_instruction|branch_resolving|math_pipe_throttle|selected|not_selected|sleeping|dispatch_stall|drain|imc_miss|misc|tex_throttle)$",
]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
if len(rows) < 3:
    sys.exit("no data in " + rep)
hdr, units = rows[0], rows[1]
pats = [re.compile(p) for p in PATTERNS]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(f"== {name[:110]}")
    vals = {}
    for i, h in enumerate(hdr):
        if any(p.match(h) for p in pats):
            vals[h] = (r[i], units[i])
    for h in sorted(vals):
        print(f"  {h:75s} {vals[h][0]:>18s} {vals[h][1]}")
    SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1,
             "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}

    def f(k):  # bytes / nanoseconds / plain numbers
        try:
            v, u = vals[k]
            return float(v.replace(",", "")) * SCALE.get(u, 1)
        except (KeyError, ValueError):
            return None
    mx, av, mn = f("sm__cycles_active.max"), f("sm__cycles_active.avg"), f("sm__cycles_active.min")
    if mx and av:
        print(f"  per-SM busy spread: max/avg = {mx / av:.3f}, min/avg = {(mn or 0) / av:.3f}")
    rd, wr, t = f("dram__bytes_read.sum"), f("dram__bytes_write.sum"), f("gpu__time_duration.sum")
    if rd is not None and wr is not None and t:
        print(f"  dram traffic {(rd + wr) / 1e6:.2f} MB over {t / 1e3:.1f} us -> {(rd + wr) / t:.1f} GB/s")

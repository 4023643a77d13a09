"""Fold `ncu --set full` captures of one step's enumeration launches into
profiles/traffic.json (bench.py's roofline.traffic / roofline.ncu).
usage: python tools/traffic_from_ncu.py <workload> <rep.ncu-rep> <profile-file-name>"""
import csv, json, os, subprocess, sys

wl, rep, src = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
         "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}


def val(r, name):
    i = hdr.index(name)
    return float(r[i].replace(",", "")) * SCALE.get(units[i], 1)


kernels = []
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if "k_tiny" not in name and "k_enumerate" not in name:
        continue
    t = val(r, "gpu__time_duration.sum")
    kernels.append({
        "kernel": name.split("(")[0].replace("void <unnamed>::", ""),
        "ms": t / 1e6,
        "dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
        "l2_bytes": 32 * val(r, "lts__t_sectors.sum"),  # 32-B sectors
        "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "sm_busy_max_over_avg": val(r, "sm__cycles_active.max") / val(r, "sm__cycles_active.avg"),
    })
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
try:
    d = json.load(open(path))
except (OSError, ValueError):
    d = {}
d[wl] = int(sum(k["dram_bytes"] for k in kernels))
d.setdefault("_source", {})[wl] = (f"{src}: dram read + write summed over the step's enumeration "
                                   f"launches ({', '.join(k['kernel'] for k in kernels)})")
d.setdefault("_detail", {})[wl] = {
    "l2_bytes": int(sum(k["l2_bytes"] for k in kernels)),
    "per_kernel": [{k2: (round(v, 4) if isinstance(v, float) else v) for k2, v in k.items()}
                   for k in kernels]}
json.dump(d, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps(d[wl]), json.dumps(d["_detail"][wl], indent=1))

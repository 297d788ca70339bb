"""Summarise gpurun_out/prof (tools/refresh_profiles.sh) into profiles/: selected ncu metrics
per step kernel, DRAM traffic per launch (traffic.json), and the launch list shares."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
OUT = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


rows = []
traffic = {}
for f in sorted(os.listdir(SRC)):
    if not f.endswith(".ncu-rep"):
        continue
    k = f[:-8]
    m = raw(os.path.join(SRC, f))
    row = {"kernel": k}
    for key in KEYS:
        v, u = m.get(key, ("", ""))
        row[key] = v
        row[key + " [unit]"] = u
    rows.append(row)
    def num(key):
        v, u = m.get(key, ("0", ""))
        x = float(str(v).replace(",", "") or 0)
        return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)
    traffic[k.replace("k_", "").replace("nonbonded", "nonbonded")] = int(num("dram__bytes_read.sum") + num("dram__bytes_write.sum"))
with open(os.path.join(OUT, f"{TAG}_ncu_full_step_kernels.csv"), "w", newline="") as fh:
    w = csv.DictWriter(fh, fieldnames=list(rows[0].keys()))
    w.writeheader()
    w.writerows(rows)
name_map = {"nonbonded": "nonbonded", "spread": "spread", "gather": "gather", "integrate": "integrate",
            "lambda_reduce": "lambda", "solve": "solve", "build_list": "build_list", "cell_sort": "cell_sort"}
tj = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes) from one ncu --set full "
               "capture per kernel (tools/refresh_profiles.sh: tools/prof_step.py, C2 x 17 replicas)",
      "C2_GEAHG_7k/R17": {name_map.get(k, k): v for k, v in traffic.items()}}
json.dump(tj, open(os.path.join(OUT, "traffic.json"), "w"), indent=2)
# launch list shares
agg = defaultdict(list)
hdr = None
for r in csv.reader(open(os.path.join(SRC, "launches.csv"))):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
with open(os.path.join(OUT, f"{TAG}_launches_C2_R17.txt"), "w") as fh:
    fh.write("ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 --warmup 3\n")
    fh.write("(cold-cache, serialised launches: compare shares, not absolutes)\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        fh.write(f"{k:50s} n={len(v):4d} mean_ns={sum(v) / len(v):11.0f} share={sum(v) / tot:6.3f}\n")
print(open(os.path.join(OUT, f"{TAG}_launches_C2_R17.txt")).read())
print(json.dumps(tj, indent=1))

"""Summarise profiles/fusion_bytes.sh launch lists into profiles/fusion_r1.json
and a markdown table: DRAM bytes per output pixel and kernel time per
execution, unfused (run_naive) vs fused (run_plan)."""
import csv
import json
import sys
from collections import defaultdict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
PX = 265420800  # px per execution (fusion_session.py frames x W x H)
REPS = 2
out = {}
src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
for cfg in (1, 2, 3, 4):
    for naive in (1, 0):
        rows = list(csv.reader(open(f"{src}/fusion_{cfg}_{naive}.csv")))  # profiles/fusion_r1/ keeps the lists
        i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
        h = rows[i]
        tot = defaultdict(float)
        kernels = set()
        for r in rows[i + 1:]:
            d = dict(zip(h, r))
            if not d.get("Metric Name"):
                continue
            kernels.add(d["ID"])
            tot[d["Metric Name"]] += float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
        b = (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / REPS
        t = tot["gpu__time_duration.sum"] / REPS
        out[f"cfg{cfg}_{'naive' if naive else 'fused'}"] = {
            "launches_per_execution": len(kernels) / REPS, "dram_bytes_per_px": round(b / PX, 3),
            "kernel_s_per_execution": t, "achieved_GBs": round(b / t / 1e9, 1), "px": PX}
json.dump(out, open("profiles/fusion_r1.json", "w"), indent=1)
print("| config | unfused launches | unfused DRAM B/px | fused launches | fused DRAM B/px | kernel time unfused -> fused (ms) |")
print("|---|---|---|---|---|---|")
for cfg in (1, 2, 3, 4):
    a, b = out[f"cfg{cfg}_naive"], out[f"cfg{cfg}_fused"]
    print(f"| cfg{cfg} | {a['launches_per_execution']:.0f} | {a['dram_bytes_per_px']} | {b['launches_per_execution']:.0f} | "
          f"{b['dram_bytes_per_px']} | {a['kernel_s_per_execution']*1e3:.2f} -> {b['kernel_s_per_execution']*1e3:.3f} |")

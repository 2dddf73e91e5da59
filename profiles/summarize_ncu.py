"""Summarise ncu --set full captures (gpurun_out/prof_cfg*.ncu-rep) into a
committed JSON + markdown table (profiles/).  Usage:
    python profiles/summarize_ncu.py <tag> gpurun_out/prof_cfg2.ncu-rep ...
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            try:
                d[m] = float(vals[i].replace(",", ""))
            except ValueError:
                d[m] = vals[i]
            d[m + ".unit"] = units[i]
    return d


def main():
    tag, reps = sys.argv[1], sys.argv[2:]
    res = {}
    for r in reps:
        d = read(r)
        res[r.split("/")[-1].replace(".ncu-rep", "")] = d
    with open(f"profiles/ncu_{tag}.json", "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()

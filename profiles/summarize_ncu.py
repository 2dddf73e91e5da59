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
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
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


SCALE = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}


def update_traffic(tag, res):
    """profiles/ncu_traffic.json: per config, DRAM bytes and warp instructions
    per launch of the dominant kernel (bench.py reports them as
    roofline.traffic / roofline.issue).  Captures are named prof_cfgN and
    come from profiles/run_ncu.sh, i.e. bench.py's default frames per step."""
    import os
    sys.path.insert(0, os.getcwd())
    from bench import DEFAULT_FRAMES
    size = {1: (1920, 1080), 2: (3840, 2160), 3: (7680, 4320), 4: (3840, 2160), 5: (16384, 16384)}
    path = "profiles/ncu_traffic.json"
    try:
        table = json.load(open(path))
    except Exception:
        table = {}
    for name, d in res.items():
        if not name.startswith("prof_cfg"):
            continue
        cfg = int(name[len("prof_cfg"):])
        w, h = size[cfg]
        px = w * h * DEFAULT_FRAMES[cfg]
        b = sum(d[m] * SCALE.get(d.get(m + ".unit", "byte"), 1.0)
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        table[str(cfg)] = {"kernel": d["kernel"], "dram_bytes_per_launch": round(b), "px_per_launch": px,
                           "dram_bytes_per_px": round(b / px, 4),
                           "warp_inst_per_px": round(d["smsp__inst_executed.sum"] / px, 4),
                           "duration_us_under_ncu": d["gpu__time_duration.sum"],
                           "source": f"profiles/ncu_{tag}.json"}
    with open(path, "w") as f:
        json.dump(table, f, indent=1, sort_keys=True)


def main():
    tag, reps = sys.argv[1], sys.argv[2:]
    res = {}
    for r in reps:
        d = read(r)
        res[r.split("/")[-1].replace(".ncu-rep", "")] = d
    with open(f"profiles/ncu_{tag}.json", "w") as f:
        json.dump(res, f, indent=1)
    update_traffic(tag, res)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()

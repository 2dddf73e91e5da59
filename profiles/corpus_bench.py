"""Device throughput of the graph-file corpus (examples/*.json) resized to
W x H, through DeviceSession: run_plan's program (fused groups + generated
kernels) and run_naive's (one generated kernel set per node).  Prints one
JSON object per graph: Mpixel/s, algorithmic HBM bytes per pixel (source
images in + observable images out), fraction of the measured HBM peak,
kernel launches per execution, and the device program.
Usage: python profiles/corpus_bench.py [W H frames] > gpurun_out/corpus.jsonl"""
import json
import os
import pathlib
import sys

REPO = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2008_11476_b200 as gvx  # noqa: E402

W, H, F = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (3840, 2160, 8)
peak = json.load(open(REPO / "MEASURED_PEAKS.json")).get("hbm_gbs", 6532.5) if (REPO / "MEASURED_PEAKS.json").exists() else 6532.5
names = sys.argv[4:] or [p.stem for p in sorted((REPO / "examples").glob("*.json"))]
for name in names:
    doc = json.loads((REPO / "examples" / f"{name}.json").read_text())
    for im in doc["images"]:
        im["width"], im["height"] = W, H
    try:
        g = gvx.GraphFile(json.dumps(doc))
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"graph": name, "error": str(e)[:200]}), flush=True)
        continue
    row = {"graph": name, "size": [W, H], "frames": F, "regions": os.environ.get("GVX_NO_REGIONS") is None}
    for naive in (False, True):
        r = g.bench(naive=naive, frames=F, iters=10)
        px = W * H * F
        key = "naive" if naive else "plan"
        row[key] = {"Mpx_s": round(px / (r["ms"] / 1e3) / 1e6, 1), "ms": round(r["ms"], 4),
                    "bytes_per_px": round(r["bytes"] / px, 3),
                    "hbm_frac": round(r["bytes"] / (r["ms"] / 1e3) / 1e9 / peak, 4), "launches": r["launches"]}
    row["program"] = g.describe()
    print(json.dumps(row), flush=True)

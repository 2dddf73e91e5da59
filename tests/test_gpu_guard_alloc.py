"""Every device allocation framed by guard bytes (GVX_GUARD_ALLOC=1,
runtime.cu gvxb_alloc / gvxb_free / gvxb_guard_check) while the library's
own buffers are in use: the generated (NVRTC) region and per-node kernels of
random DAGs and of the example corpus at ragged sizes, the fused config
graphs through run_plan, run_naive, batch sessions and row bands.  No
kernel may write past the end (or before the start) of any allocation.
Runs in a fresh process (the mode is read once); a planted out-of-bounds
byte proves the check reports."""
import json
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = pathlib.Path(__file__).resolve().parent.parent

SCRIPT = r"""
import ctypes, gc, json, pathlib, sys
repo = pathlib.Path(sys.argv[1])
sys.path.insert(0, str(repo)); sys.path.insert(0, str(repo / "tests"))
import paper_2008_11476_b200 as gvx
import reference_graphs as rg
ran = 0
for seed in range(1, 41):
    doc = rg.random_dag(seed, 5 + seed * 37 % 300, 3 + seed * 11 % 70)
    if not doc["outputs"]:
        continue
    g = gvx.GraphFile(json.dumps(doc))
    g.run(naive=False, seed=seed); g.run(naive=True, seed=seed)
    del g; ran += 1
for path in sorted((repo / "examples").glob("*.json")):
    doc = json.loads(path.read_text())
    for im in doc["images"]:
        im["width"], im["height"] = 389, 131
    try:
        g = gvx.GraphFile(json.dumps(doc))
    except gvx.GraphvxError:
        continue
    g.run(naive=False, seed=3); g.run(naive=True, seed=3)
    del g; ran += 1
for cfg in (1, 2, 3, 4, 5):
    w, h = 1031, 517
    g = gvx.ConfigGraph(cfg, w, h)
    img = gvx.random_u8(w, h, cfg)
    g.run_host(img); g.run_host(img, naive=True)
    s = gvx.Session(g, frames=3)
    for f in range(3):
        s.upload(f, img)
    s.launch(); s.sync(); s.download(2)
    s.close(); g.close(); ran += 1
gc.collect()
c, _ = gvx._load()
c.gvxb_guard_check.restype = ctypes.c_int64
live = ctypes.c_int()
bad = c.gvxb_guard_check(ctypes.byref(live))
# the check has teeth: one byte written just past a 1000-byte allocation
dev = gvx.Device(0)
p = dev.alloc(1000)
dev.memset(p + 1024, 0, 1)  # allocations are rounded up to 256 bytes
dev.sync(); dev.free(p)
planted = c.gvxb_guard_check(None) - bad
print(json.dumps({"ran": ran, "bad": bad, "live": live.value, "planted": planted}))
"""


def test_no_kernel_writes_outside_its_allocation():
    env = dict(os.environ, GVX_GUARD_ALLOC="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(REPO)], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["ran"] >= 40, res
    assert res["planted"] == 1, res
    assert res["bad"] == 0, (res, r.stderr[-3000:])

"""Phases of the drop-in host run_plan (gvxc_graph_run_host) on one config:
GVX_TRACE_HOST=1 python profiles/run_plan_probe.py [cfg] [reuse]
(reuse = 1: the caller's output array is allocated once; 0: np.empty per
call, as ConfigGraph.run_host does)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2008_11476_b200 as gvx  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reuse = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w, h = gvx.CONFIG_SIZE[cfg]
g = gvx.ConfigGraph(cfg, w, h, True)
img = gvx.random_u8(w, h, 1)
out = g.output_array()
import ctypes  # noqa: E402

hist = (ctypes.c_longlong * 256)()
stats = (ctypes.c_double * 2)()
cnt = (ctypes.c_longlong * 4)()


def call():
    o = out if reuse else g.output_array()
    gvx._graph.gvxc_graph_run_host(g._h, 0, img.ctypes.data, None if o is None else o.ctypes.data, hist, stats, cnt)


for _ in range(2):
    call()
n = 4
t = time.perf_counter()
for _ in range(n):
    call()
dt = (time.perf_counter() - t) / n
print(f"cfg {cfg} reuse {reuse}: {dt * 1e3:.2f} ms per call, {w * h / dt / 1e6:.0f} Mpx/s", file=sys.stderr)

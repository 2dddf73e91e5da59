"""Wall time per execution of a config's device program when consecutive
executions cannot overlap (same output buffers every launch, so each
launch waits for the previous one): the case the serial tile-height cap
(edge8 / Harris) is for.  Usage: python profiles/serial_probe.py cfg frames"""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_2008_11476_b200 as gvx  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
F = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w, h = gvx.CONFIG_SIZE[cfg]
g = gvx.ConfigGraph(cfg, w, h, True)
s = gvx.Session(g, frames=F)
for f in range(F):
    s.upload(f, gvx.random_u8(w, h, cfg + f))
for _ in range(5):
    s.launch()
s.sync()
n = 100
t0 = time.perf_counter()
for _ in range(n):
    s.launch()
s.sync()
dt = (time.perf_counter() - t0) / n
th = os.environ.get("GVX_HARRIS_TH") or os.environ.get("GVX_EDGE8_TH") or "auto"
print(f"cfg {cfg} x{F} th={th}: {dt * 1e6:.1f} us per execution, {w * h * F / dt / 1e9:.0f} Gpx/s", file=sys.stderr)

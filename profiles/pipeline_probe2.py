# one pipeline, warmed, then per-frame wall times (mode: copy | view)
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2008_11476_b200 as gvx
cfg, mode = int(sys.argv[1]), sys.argv[2]
w, h = gvx.CONFIG_SIZE[cfg]
g = gvx.ConfigGraph(cfg, w, h, True)
NF = int(sys.argv[3]) if len(sys.argv) > 3 else 8
frames = [gvx.random_u8(w, h, 3 + i) for i in range(NF)]
out = g.output_array()
pl = gvx.Pipeline(g, depth=3)
def nxt():
    pl.next(out) if mode == "copy" else pl.next_view()
for i in range(4):
    if pl.pending() >= 3:
        nxt()
    pl.submit(frames[i])
while pl.pending():
    nxt()
ts = []
t0 = time.perf_counter()
for i in range(24):
    a = time.perf_counter()
    if pl.pending() >= 3:
        nxt()
    pl.submit(frames[i % NF])
    ts.append(time.perf_counter() - a)
while pl.pending():
    nxt()
tot = time.perf_counter() - t0
print(mode, f"{w * h * 24 / tot / 1e9:.1f} Gpx/s;", " ".join(f"{1e6 * t:.0f}" for t in ts), file=sys.stderr)

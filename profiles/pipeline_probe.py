# per-call timings of the host pipeline (next / next_view / submit)
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2008_11476_b200 as gvx
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w, h = gvx.CONFIG_SIZE[cfg]
g = gvx.ConfigGraph(cfg, w, h, True)
frames = [gvx.random_u8(w, h, 3 + i) for i in range(4)]
out = g.output_array()
for mode in ("copy", "view", "copy", "view"):
    pl = gvx.Pipeline(g, depth=3)
    tn = ts = 0.0
    t0 = time.perf_counter()
    n = 30
    for i in range(n):
        if pl.pending() >= 3:
            a = time.perf_counter()
            pl.next(out) if mode == "copy" else pl.next_view()
            tn += time.perf_counter() - a
        a = time.perf_counter()
        pl.submit(frames[i % 4])
        ts += time.perf_counter() - a
    while pl.pending():
        pl.next(out) if mode == "copy" else pl.next_view()
    tot = time.perf_counter() - t0
    print(f"{mode}: {tot / n * 1e6:.0f} us/frame  next {tn / n * 1e6:.0f}  submit {ts / n * 1e6:.0f}  -> {w * h * n / tot / 1e9:.1f} Gpx/s", file=sys.stderr)

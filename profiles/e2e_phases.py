# e2e phase probe for the Harris pipeline: DMA rates alone (pinned H2D, D2H,
# both at once), the host staging copy alone, then the pipeline per frame.
import sys, time, ctypes, threading
sys.path.insert(0, ".")
import numpy as np
import paper_2008_11476_b200 as gvx
c, _ = gvx._load()
dev = gvx.Device(0)
w, h = 3840, 2160
n = w * h
src = np.random.default_rng(1).integers(0, 256, n, dtype=np.uint8)
pin_in, pin_out = ctypes.c_void_p(), ctypes.c_void_p()
c.gvxb_host_alloc(ctypes.c_size_t(n), ctypes.byref(pin_in))
c.gvxb_host_alloc(ctypes.c_size_t(n), ctypes.byref(pin_out))
d_in, d_out = dev.alloc(n), dev.alloc(n)
def rate(label, fn, reps=10):
    dev.sync(); t = time.perf_counter()
    for _ in range(reps): fn()
    dev.sync(); dt = (time.perf_counter() - t) / reps
    print(f"{label:34s} {dt * 1e6:8.1f} us/frame  {n / dt / 1e9:6.1f} GB/s", file=sys.stderr)
up = lambda: c.gvxb_upload_2d(dev.h, ctypes.c_void_p(d_in), w, pin_in, w, w, h)
down = lambda: c.gvxb_download_2d(dev.h, pin_out, w, ctypes.c_void_p(d_out), w, w, h)
rate("H2D pinned", up)
rate("D2H pinned", down)
dev2 = gvx.Device(0)
d2 = dev2.alloc(n)
def both():
    c.gvxb_upload_2d(dev.h, ctypes.c_void_p(d_in), w, pin_in, w, w, h)
    c.gvxb_download_2d(dev2.h, pin_out, w, ctypes.c_void_p(d2), w, w, h)
def both_sync():
    both(); dev2.sync()
rate("H2D + D2H (two streams)", both_sync)
ctypes.memmove(pin_in, src.ctypes.data, n)
rate("memmove pageable->pinned (1 thr)", lambda: ctypes.memmove(pin_in, src.ctypes.data, n))
g = gvx.ConfigGraph(2, w, h, True)
NFR = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--nf=")), "4"))
frames = np.stack([gvx.random_u8(w, h, 3 + i) for i in range(NFR)])
pinned = gvx.PinnedHost([frames]) if "--pinned" in sys.argv else None
for depth in (2, 3, 4, 6):
    pl = gvx.Pipeline(g, depth=depth)
    for i in range(depth + 2):
        if pl.pending() >= depth: pl.next_view()
        pl.submit(frames[i % NFR], pinned=pinned is not None)
    while pl.pending(): pl.next_view()
    t0 = time.perf_counter(); sub = 0.0; nxt = 0.0
    N = 48
    for i in range(N):
        a = time.perf_counter()
        if pl.pending() >= depth: pl.next_view()
        b = time.perf_counter()
        pl.submit(frames[i % NFR], pinned=pinned is not None)
        nxt += b - a; sub += time.perf_counter() - b
    while pl.pending(): pl.next_view()
    tot = time.perf_counter() - t0
    print(f"pipeline depth {depth}: {n * N / tot / 1e9:.1f} Gpx/s; per frame {tot / N * 1e6:.0f} us "
          f"(next {nxt / N * 1e6:.0f}, submit {sub / N * 1e6:.0f})", file=sys.stderr)
    del pl

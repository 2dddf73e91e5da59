import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2008_11476_b200 as gvx
sys.path.insert(0, "."); import bench
w, h = 3840, 2160
dev = gvx.Device(0)
graph = gvx.ConfigGraph(2, w, h, True)
if "--sess" in sys.argv:
    sess = gvx.Session(graph, frames=32); sess.set_stream(dev.stream)
host = bench.make_frames(gvx, w, h, 32, 2) if "--mk" in sys.argv else np.stack([gvx.random_u8(w, h, 3 + i) for i in range(32)])
pinned = gvx.PinnedHost([host])
pipe = gvx.Pipeline(graph, depth=3)
out = graph.output_array()
for i in range(32):
    if pipe.pending() >= 3: pipe.next(out)
    pipe.submit(host[i % 32], pinned=True)
while pipe.pending(): pipe.next(out)
for rep in range(3):
    t0 = time.perf_counter()
    for i in range(48):
        if pipe.pending() >= 3: pipe.next_view()
        pipe.submit(host[i % 32], pinned=True)
    while pipe.pending(): pipe.next_view()
    print(sys.argv[1:], f"{w*h*48/(time.perf_counter()-t0)/1e9:.1f} Gpx/s", file=sys.stderr)

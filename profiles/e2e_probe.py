# e2e phase probe: GVX_TRACE_HOST=1 python profiles/e2e_probe.py [cfg]
import sys, time
sys.path.insert(0, ".")
import paper_2008_11476_b200 as gvx
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w, h = gvx.CONFIG_SIZE[cfg]
g = gvx.ConfigGraph(cfg, w, h, True)
img = gvx.random_u8(w, h, 1)
for i in range(3):
    g.run_host_inplace(img)
t = time.perf_counter()
for i in range(5):
    g.run_host_inplace(img)
print(cfg, (time.perf_counter() - t) / 5 * 1e3, "ms per call", file=sys.stderr)

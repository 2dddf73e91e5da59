# one naive (per-node NVRTC) session of config 1 over 4 frames, for ncu
import sys
sys.path.insert(0, ".")
import paper_2008_11476_b200 as gvx
dev = gvx.Device(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w, h = gvx.CONFIG_SIZE[cfg]
F = 4
g = gvx.ConfigGraph(cfg, w, h, True)
s = gvx.Session(g, frames=F, naive=True)
s.set_stream(dev.stream)
pitch = (w + 127) // 128 * 128
din = dev.alloc(pitch * h * F)
dout = dev.alloc(2 * pitch * h * F)
s.bind(0, din, pitch, pitch * h)
if cfg != 4:
    s.bind(1, dout, pitch * (2 if cfg == 1 else 1), pitch * (2 if cfg == 1 else 1) * h)
for _ in range(3):
    s.launch()
s.sync()
print("ok")

"""One device session of a BASELINE config, fused (run_plan program) or
unfused (run_naive: one NVRTC kernel set per abstraction node), executed
`reps` times over F frames — the workload of the before/after-fusion DRAM
byte counts (profiles/fusion_bytes.sh runs it under ncu).
usage: python profiles/fusion_session.py <cfg> <naive 0|1> <frames> [reps]"""
import sys
sys.path.insert(0, ".")
import paper_2008_11476_b200 as gvx

cfg, naive, F = int(sys.argv[1]), bool(int(sys.argv[2])), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
dev = gvx.Device(0)
w, h = gvx.CONFIG_SIZE[cfg]
g = gvx.ConfigGraph(cfg, w, h, True)
s = gvx.Session(g, frames=F, naive=naive)
s.set_stream(dev.stream)
pitch = (w + 127) // 128 * 128
obytes = 2 if cfg in (1, 5) else 1
din = dev.alloc(pitch * h * F)
s.bind(0, din, pitch, pitch * h)
if cfg != 4:
    dout = dev.alloc(obytes * pitch * h * F)
    s.bind(1, dout, pitch * obytes, pitch * obytes * h)
for _ in range(reps):
    s.launch()
s.sync()
print("ok", cfg, "naive" if naive else "fused", F, "frames", reps, "executions", "px/execution", w * h * F)

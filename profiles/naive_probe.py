# device time of the per-node NVRTC program (run_naive path) vs the fused plan
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2008_11476_b200 as gvx

dev = gvx.Device(0)
for cfg in (1, 2, 3, 4):
    w, h = gvx.CONFIG_SIZE[cfg]
    F = 4
    g = gvx.ConfigGraph(cfg, w, h, True)
    for naive in (True, False):
        s = gvx.Session(g, frames=F, naive=naive)
        s.set_stream(dev.stream)
        pitch = (w + 127) // 128 * 128
        din = dev.alloc(pitch * h * F)
        out_pitch = pitch * (2 if cfg == 1 else 1)
        dout = dev.alloc(out_pitch * h * F) if cfg != 4 else None
        s.bind(0, din, pitch, pitch * h)
        if dout:
            s.bind(1, dout, out_pitch, out_pitch * h)
        for _ in range(3):
            s.launch()
        s.sync()
        e0, e1 = dev.event(), dev.event()
        dev.record(e0)
        for _ in range(10):
            s.launch()
        dev.record(e1)
        ms = dev.elapsed_ms(e0, e1) / 10
        print(f"cfg{cfg} {'naive' if naive else 'plan '} launches/run {s.launches():2d}  {ms:.3f} ms  "
              f"{w * h * F / ms / 1e6:.0f} Mpx/s")

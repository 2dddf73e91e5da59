"""Host-side cost and wall time of banded executions (BandedSession::launch
through gvx_c.h), outputs rotating over PROBE_NOUT (16) buffers as bench.py
does (an execution overlaps the ones still running when independent of them): world = 1 on 16384 x H images,
H = one band's share at 1 / 2 / 4 / 8 GPUs.
Usage: [GVX_EDGE8_TH=n] [PROBE_SINGLE=1] python profiles/band_host_probe.py [WxH ...]"""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_2008_11476_b200 as gvx  # noqa: E402

sizes = [tuple(map(int, a.split("x"))) for a in sys.argv[1:]] or [(16384, 16384), (16384, 2048)]
dev = gvx.Device(0)
for W, H in sizes:
    g = gvx.ConfigGraph(5, W, H, True)
    b = gvx.Band(g, 0, 1, None)
    b.set_stream(dev.stream)
    b.upload(0, gvx.random_u8(W, H, 5), 0)
    b.set_overlap(1)
    pitch = (2 * W + 127) // 128 * 128
    nout = int(os.environ.get("PROBE_NOUT", 16))  # rotating outputs, as bench.py (NPOOL)
    outs = [dev.alloc(pitch * H) for _ in range(nout)]

    single = os.environ.get("PROBE_SINGLE") is not None  # one output buffer: every launch waits

    def launch(i):
        b.bind(1, outs[0 if single else i % nout], pitch, pitch * H)
        b.launch()

    for i in range(5):
        launch(i)
    dev.sync()
    n = 200
    t0 = time.perf_counter()
    for i in range(n):
        launch(i)
    t1 = time.perf_counter()
    dev.sync()
    t2 = time.perf_counter()
    print(f"{W}x{H} th={os.environ.get('GVX_EDGE8_TH', 'auto')}{' single' if single else ''}: host {1e6 * (t1 - t0) / n:.1f} us per launch call, "
          f"wall {1e6 * (t2 - t0) / n:.1f} us per execution", file=sys.stderr)
    b.close()

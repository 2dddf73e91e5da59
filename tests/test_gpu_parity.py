"""GPU parity: every BASELINE config through the public API on the B200,
bit-exact against the reference (golden fixtures from the unmodified
reference) and the C restatement at full size."""
import pathlib
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [(1, 1), (2, 3), (7, 5), (16, 16), (33, 17), (64, 48), (5, 129), (130, 3)]


def _same(cfg, a, b):
    if cfg == 4:
        return np.array_equal(a[0], b[0]) and a[1] == b[1] and a[2] == b[2]
    return np.array_equal(a, b)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
@pytest.mark.parametrize("size", SIZES)
def test_configs_match_reference_golden(cfg, size, gvx, golden):
    w, h = size
    key = f"c{cfg}_{w}x{h}"
    img = golden[key + "_in"]
    want = (golden[key + "_hist"], *golden[key + "_stats"]) if cfg == 4 else golden[key + "_out"]
    g = gvx.ConfigGraph(cfg, w, h)
    got_plan, cnt_plan = g.run_host(img)
    got_naive, cnt_naive = g.run_host(img, naive=True)
    assert _same(cfg, got_plan, want), "run_plan (fused sm_100a kernel) differs from the reference"
    assert _same(cfg, got_naive, want), "run_naive (per-node NVRTC kernels) differs from the reference"
    ref = golden[key + "_counters"]
    # exact reference event counters for the unfused program
    assert cnt_naive["pixels_read"] == ref[1] and cnt_naive["pixels_written"] == ref[2]
    assert cnt_naive["transfers_executed"] == ref[3]
    assert cnt_plan["kernel_launches"] <= cnt_naive["kernel_launches"]
    assert cnt_plan["transfers_executed"] <= cnt_naive["transfers_executed"]


def test_fused_plans_are_single_launches(gvx):
    # cfg1..4 fuse into one kernel each (cfg4: conv/convert/hist/sums, the
    # last CTA of each frame publishes the histogram and MeanStdDev)
    want = {1: 1, 2: 1, 3: 1, 4: 1}
    for cfg, n in want.items():
        g = gvx.ConfigGraph(cfg, 300, 200)
        _, cnt = g.run_host(gvx.random_u8(300, 200, cfg))
        assert cnt["kernel_launches"] == n, (cfg, cnt)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_full_size_configs_match_oracle(cfg, gvx, oracle_mod):
    w, h = gvx.CONFIG_SIZE[cfg]
    img = gvx.random_u8(w, h, gvx.CONFIG_SEED[cfg])
    g = gvx.ConfigGraph(cfg, w, h)
    got, _ = g.run_host(img)
    want = oracle_mod.port_run(cfg, img)
    assert _same(cfg, got, want)


def test_naive_plan_agree_at_1080p(gvx):
    for cfg in (1, 2, 3, 4):
        img = gvx.random_u8(1920, 1080, 40 + cfg)
        g = gvx.ConfigGraph(cfg, 1920, 1080)
        a, _ = g.run_host(img)
        b, _ = g.run_host(img, naive=True)
        assert _same(cfg, a, b)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_device_sessions_batch_frames(cfg, gvx, oracle_mod):
    w, h, frames = 641, 359, 3
    g = gvx.ConfigGraph(cfg, w, h)
    s = gvx.Session(g, frames=frames)
    imgs = [gvx.random_u8(w, h, 70 + f) for f in range(frames)]
    for f, im in enumerate(imgs):
        s.upload(f, im)
    s.launch()
    s.sync()
    for f, im in enumerate(imgs):
        assert _same(cfg, s.download(f), oracle_mod.port_run(cfg, im))


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_row_bands_reproduce_full_image(world, gvx, oracle_mod):
    """cfg5 banding on one GPU, sequentially: each band reads its halo'd slab
    straight out of the full image buffer (what NVLink halo exchange
    delivers on N GPUs) and must equal the unbanded launch and the oracle."""
    W, H = 1000, 777
    img = gvx.random_u8(W, H, 5)
    dev = gvx.Device(0)
    pitch = 1024
    src = dev.alloc(pitch * H)
    dev.upload(src, pitch, img)
    full = dev.alloc(2 * pitch * H)
    banded = dev.alloc(2 * pitch * H)
    gvx.edge_band(dev, src, pitch, W, H, full, 2 * pitch, 0, H, H, 0, 0)
    for r in range(world):
        r0, r1 = gvx.band_rows(H, world, r)
        s0, s1 = max(0, r0 - 2), min(H, r1 + 2)
        gvx.edge_band(dev, src + s0 * pitch, pitch, W, s1 - s0, banded + r0 * 2 * pitch, 2 * pitch,
                      r0, r1, H, s0, r0)
    a = np.empty((H, W), np.int16)
    b = np.empty((H, W), np.int16)
    dev.download(a, full, 2 * pitch)
    dev.download(b, banded, 2 * pitch)
    assert np.array_equal(a, b)
    assert np.array_equal(a, oracle_mod.port_run(1, img))
    for p in (src, full, banded):
        dev.free(p)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_host_runs_recycle_pinned_buffers(cfg, gvx, oracle_mod):
    """Repeated host runs through the C facade: the input is copied into the
    graph's page-locked Buffer and outputs DMA into recycled page-locked
    vectors; every run must still return its own frame's result."""
    w, h = 1031, 517
    g = gvx.ConfigGraph(cfg, w, h)
    frames = [gvx.random_u8(w, h, 40 + i) for i in range(3)]
    for rnd in range(2):
        for f in frames:
            got, _ = g.run_host_inplace(f)
            want = oracle_mod.port_run(cfg, f)
            if cfg == 4:
                assert np.array_equal(got[0], want[0]) and got[1] == want[1] and got[2] == want[2]
            else:
                assert np.array_equal(np.array(got), want), (cfg, rnd)
            plain, _ = g.run_host(f)
            assert _same(cfg, plain, want)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
@pytest.mark.parametrize("naive", [False, True])
def test_host_pipeline_matches_run_host(cfg, naive, gvx, oracle_mod):
    """gvx::HostPipeline: frames in flight, results in submission order and
    identical (outputs and event counters) to one-at-a-time run_plan /
    run_naive."""
    w, h = 643, 211
    g = gvx.ConfigGraph(cfg, w, h)
    frames = [gvx.random_u8(w, h, 70 + i) for i in range(7)]
    want = [g.run_host(f, naive=naive) for f in frames]
    for depth in (1, 3):
        pl = gvx.Pipeline(g, depth=depth, naive=naive)
        got = []
        for f in frames:
            if pl.pending() >= depth:
                got.append(pl.next())
            pl.submit(f)
        while pl.pending():
            got.append(pl.next())
        assert len(got) == len(frames)
        for (gr, gc), (wr, wc), f in zip(got, want, frames):
            assert _same(cfg, gr, wr) and _same(cfg, gr, oracle_mod.port_run(cfg, f))
            assert gc == wc


def test_host_pipeline_views(gvx, oracle_mod):
    """next_view: results read in place from the pipeline's staging."""
    w, h = 517, 333
    g = gvx.ConfigGraph(2, w, h)
    frames = [gvx.random_u8(w, h, 90 + i) for i in range(6)]
    pl = gvx.Pipeline(g, depth=3)
    got = []
    for f in frames:
        if pl.pending() >= 3:
            v, _ = pl.next_view()
            got.append(np.array(v))  # consumed before the next submit
        pl.submit(f)
    while pl.pending():
        v, _ = pl.next_view()
        got.append(np.array(v))
    for r, f in zip(got, frames):
        assert np.array_equal(r, oracle_mod.port_run(2, f))


@pytest.mark.parametrize("pinned", [False, True])
def test_host_pipeline_stream(pinned, gvx, oracle_mod):
    """gvxc_pipeline_stream: a whole stream in one native call, every result
    handed over in order; counters are the per-frame sums."""
    w, h = 517, 333
    g = gvx.ConfigGraph(1, w, h)
    stack = np.stack([gvx.random_u8(w, h, 150 + i) for i in range(7)])
    pl = gvx.Pipeline(g, depth=3)
    got = []
    if pinned:
        with gvx.PinnedHost([stack]):
            cnt = pl.stream(list(stack), pinned=True, on_result=lambda v: got.append(np.array(v)))
    else:
        cnt = pl.stream(list(stack), on_result=lambda v: got.append(np.array(v)))
    assert len(got) == len(stack)
    for r, f in zip(got, stack):
        assert np.array_equal(r, oracle_mod.port_run(1, f))
    _, one = g.run_host(stack[0])
    assert cnt["pixels_read"] == len(stack) * one["pixels_read"]
    assert cnt["kernel_launches"] == len(stack) * one["kernel_launches"]


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_host_pipeline_pinned_inputs(cfg, gvx, oracle_mod):
    """submit(pinned=True): frames DMAed straight from registered host memory
    give the same results as staged submits; unregistered memory is refused."""
    w, h = 517, 333
    g = gvx.ConfigGraph(cfg, w, h)
    stack = np.stack([gvx.random_u8(w, h, 120 + i) for i in range(5)])
    pl = gvx.Pipeline(g, depth=3)
    with gvx.PinnedHost([stack]):
        got = []
        for f in stack:
            if pl.pending() >= 3:
                got.append(pl.next())
            pl.submit(f, pinned=True)
        while pl.pending():
            got.append(pl.next())
    for (r, _), f in zip(got, stack):
        assert _same(cfg, r, oracle_mod.port_run(cfg, f))
    with pytest.raises(gvx.GraphvxError):
        pl.submit(gvx.random_u8(w, h, 7), pinned=True)


@pytest.mark.parametrize("size", [(1920, 1080), (77, 41), (481, 37)])
def test_edge_v2_kernel_still_bit_exact(size):
    """The 4-warp tiled edge kernel (kept behind GVX_EDGE_V2=1 for A/B runs
    against edge8) in a fresh process: bit-exact with the C restatement."""
    import os
    import subprocess
    import sys
    repo = pathlib.Path(__file__).resolve().parent.parent
    code = ("import sys; sys.path.insert(0, '.'); import numpy as np, paper_2008_11476_b200 as gvx, oracle; "
            f"w, h = {size[0]}, {size[1]}; img = gvx.random_u8(w, h, 3); "
            "got, _ = gvx.ConfigGraph(1, w, h).run_host(img); "
            "print('EQUAL' if np.array_equal(got, oracle.port_run(1, img)) else 'DIFF')")
    out = subprocess.run([sys.executable, "-c", code], cwd=repo, capture_output=True, text=True, timeout=300,
                         env=dict(os.environ, GVX_EDGE_V2="1"))
    assert "EQUAL" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]


@pytest.mark.parametrize("cfg", [2, 3])
def test_overlapped_launch_chain_respects_dependences(cfg, gvx, oracle_mod):
    """Programmatic dependent launch (DeviceSession::set_overlap): a chain
    whose executions read the previous one's output (RAW), overwrite its
    input (WAR) and alternate with independent executions must equal the
    sequential result."""
    w, h = 1537, 301
    g = gvx.ConfigGraph(cfg, w, h)
    s = gvx.Session(g, frames=1)
    dev = gvx.Device(0)
    s.set_stream(dev.stream)
    s.set_overlap(1)
    pitch = (w + 127) // 128 * 128
    bufs = [dev.alloc(pitch * h) for _ in range(4)]
    img = gvx.random_u8(w, h, 11)
    other = gvx.random_u8(w, h, 12)
    dev.upload(bufs[0], pitch, img)
    dev.upload(bufs[3], pitch, other)
    seq = [(0, 1), (3, 2), (1, 2), (2, 0), (3, 1)]  # (in, out) buffer indices
    for a, b in seq:
        s.bind(0, bufs[a], pitch, pitch * h)
        s.bind(1, bufs[b], pitch, pitch * h)
        s.launch()
    s.sync()
    want = {0: img, 3: other}
    for a, b in seq:
        want[b] = oracle_mod.port_run(cfg, want[a])
    for k in (0, 1, 2):
        got = np.empty((h, w), np.uint8)
        dev.download(got, bufs[k], pitch)
        assert np.array_equal(got, want[k]), k
    for p in bufs:
        dev.free(p)


STRIP_W = [3, 4, 5, 120, 123, 124, 125, 126, 128, 129, 247, 248, 249, 250, 252, 253, 371, 372, 373, 496, 497]


@pytest.mark.parametrize("cfg", [1, 2])
@pytest.mark.parametrize("h", [1, 2, 3, 5, 17, 130])
def test_row_ring_kernels_at_strip_boundaries(cfg, h, gvx, oracle_mod):
    """The row-ring kernels split the width into strips (harris4: 124
    columns, 4 per lane; edge8: 248, 8 per lane) whose last one is pulled
    left and whose border strips clamp: widths around the strip multiples
    and heights around the ring chunks, against the C restatement."""
    for w in STRIP_W:
        img = gvx.random_u8(w, h, 1000 + w + h)
        got, _ = gvx.ConfigGraph(cfg, w, h).run_host(img)
        assert np.array_equal(got, oracle_mod.port_run(cfg, img)), (cfg, w, h)


def test_eight_column_harris_kernel_stays_exact(gvx):
    """The 8-column Harris kernel (GVX_HARRIS8=1, the default before
    harris4) on border-heavy sizes, in a fresh process (the switch is read
    once), against the C restatement."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.');"
        "import oracle, paper_2008_11476_b200 as gvx\n"
        "for w, h in [(5, 3), (247, 19), (248, 130), (253, 7), (3840, 64), (1001, 517)]:\n"
        "    img = gvx.random_u8(w, h, w * 7 + h)\n"
        "    g = gvx.ConfigGraph(2, w, h)\n"
        "    assert 'harris' in g.describe()\n"
        "    got, _ = g.run_host(img)\n"
        "    assert np.array_equal(got, oracle.port_run(2, img)), (w, h)\n"
        "print('ok')\n")
    env = dict(__import__("os").environ, GVX_HARRIS8="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=str(pathlib.Path(__file__).resolve().parent.parent),
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("cfg,seed", [(2, 1), (2, 2), (3, 3)])
def test_overlapped_random_launch_chains(cfg, seed, gvx, oracle_mod):
    """40 executions over 5 buffers with random (input, output) pairs, so
    read-after-write, write-after-read and write-after-write hazards reach
    back one to several launches: the overlap window must order exactly
    the dependent ones (checked against the sequential result)."""
    rng = np.random.default_rng(seed)
    w, h = 1537, 301
    g = gvx.ConfigGraph(cfg, w, h)
    s = gvx.Session(g, frames=1)
    dev = gvx.Device(0)
    s.set_stream(dev.stream)
    s.set_overlap(1)
    pitch = (w + 127) // 128 * 128
    nb = 5
    bufs = [dev.alloc(pitch * h) for _ in range(nb)]
    want = {}
    for k in range(nb):
        want[k] = gvx.random_u8(w, h, 100 * seed + k)
        dev.upload(bufs[k], pitch, want[k])
    seq = []
    for _ in range(40):
        a = int(rng.integers(nb))
        b = int(rng.integers(nb - 1))
        seq.append((a, b if b < a else b + 1))
    for a, b in seq:
        s.bind(0, bufs[a], pitch, pitch * h)
        s.bind(1, bufs[b], pitch, pitch * h)
        s.launch()
    s.sync()
    for a, b in seq:
        want[b] = oracle_mod.port_run(cfg, want[a])
    for k in range(nb):
        got = np.empty((h, w), np.uint8)
        dev.download(got, bufs[k], pitch)
        assert np.array_equal(got, want[k]), k
    for p in bufs:
        dev.free(p)

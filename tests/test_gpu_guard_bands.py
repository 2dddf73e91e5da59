"""Memory-safety checks of the C-ABI kernels without compute-sanitizer
(closed on the GPU pool): every image and scratch buffer a kernel touches
sits inside one allocation framed by guard bytes, with padded row pitches
and, for batches, a gap between frames, all pre-filled with 0xA5.  After
the launch the guards, the row padding and the frame gaps must still hold
0xA5 (no out-of-bounds store: ragged widths, last strips pulled left,
partial vector stores, short bands), and the results must not depend on
what the source's row padding holds (no load past the last column feeds a
result: the TMA boxes' and the border clamps' column handling).  Results
are also checked against the C restatement (oracle/gvx_oracle.c)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GUARD = 4096
FILL = 0xA5
SIZES = [(1, 1), (3, 2), (77, 41), (248, 9), (249, 70), (385, 33), (1000, 131), (2049, 19)]


class Guarded:
    """One device allocation: guard | frame 0 rows | gap | frame 1 rows | ... | guard.
    pitch leaves >= 64 padding bytes per row; every byte starts as `fill`
    (0xA5 outside the image; the image bytes themselves are written by
    upload or by the kernel)."""

    def __init__(self, dev, w, h, bpp, frames=1, fill=FILL):
        self.dev, self.w, self.h, self.bpp, self.frames, self.fill = dev, w, h, bpp, frames, fill
        self.pitch = (w * bpp + 64 + 127) // 128 * 128
        self.stride = self.pitch * h + (1024 if frames > 1 else 0)
        self.total = GUARD + self.stride * frames + GUARD
        self.base = dev.alloc(self.total)
        dev.memset(self.base, FILL, self.total)
        if fill != FILL:  # a source whose row padding holds `fill`
            for f in range(frames):
                dev.memset(self.data + f * self.stride, fill, self.pitch * h)

    @property
    def data(self):
        return self.base + GUARD

    def image(self, gvx, fmt):
        return gvx.GvxbImage(self.data, self.pitch, self.w, self.h, fmt, self.frames,
                             self.stride if self.frames > 1 else 0)

    def upload(self, frames):
        for f, a in enumerate(frames):
            self.dev.upload(self.data + f * self.stride, self.pitch, a)

    def raw(self):
        b = np.empty((1, self.total), np.uint8)
        self.dev.download(b, self.base, self.total)
        return b[0]

    def read(self, dtype, what, rows=None):
        """The frames' pixels; asserts every byte outside them (outside rows
        [rows[0], rows[1]) when given) still holds its initial value."""
        r0, r1 = rows if rows else (0, self.h)
        b = self.raw()
        outside = np.ones(self.total, bool)
        expect = np.full(self.total, FILL, np.uint8)
        pix = []
        for f in range(self.frames):
            o = GUARD + f * self.stride
            expect[o:o + self.pitch * self.h] = self.fill
            rows = b[o:o + self.pitch * self.h].reshape(self.h, self.pitch)
            pix.append(rows[:, :self.w * self.bpp].copy().view(dtype))
            for r in range(r0, r1):
                outside[o + r * self.pitch:o + r * self.pitch + self.w * self.bpp] = False
        bad = np.flatnonzero(outside & (b != expect))
        assert bad.size == 0, f"{what}: {bad.size} byte(s) outside the image overwritten, first at offset " \
                              f"{int(bad[0]) - GUARD} from the image start"
        return pix

    def free(self):
        self.dev.free(self.base)


def frames_of(rng, w, h, n):
    return [rng.integers(0, 256, (h, w), dtype=np.uint8) for _ in range(n)]


@pytest.fixture(scope="module")
def dev(gvx):
    return gvx.Device(0)


def _run_edge(gvx, dev, imgs, pad):
    c, _ = gvx._load()
    c.gvxb_edge.argtypes = [ctypes.c_void_p, ctypes.POINTER(gvx.GvxbEdgeArgs)]
    h, w = imgs[0].shape
    n = len(imgs)
    src = Guarded(dev, w, h, 1, n, fill=pad)
    src.upload(imgs)
    outs = [Guarded(dev, w, h, 2, n) for _ in range(3)]
    a = gvx.GvxbEdgeArgs()
    a.src = src.image(gvx, 0)
    a.gx, a.gy, a.mag = (o.image(gvx, 2) for o in outs)
    a.with_gauss = 1
    a.band = gvx.GvxbBand(0, h, h, 0, 0)
    gvx._check_cuda(c.gvxb_edge(dev.h, ctypes.byref(a)))
    dev.sync()
    res = [o.read(np.int16, f"edge {name} {w}x{h}x{n}") for o, name in zip(outs, ("gx", "gy", "mag"))]
    src.read(np.uint8, "edge source")  # read-only: padding untouched
    for b in [src] + outs:
        b.free()
    return res


@pytest.mark.parametrize("frames", [1, 2])
def test_edge_stays_inside_its_images(frames, gvx, dev, oracle_mod):
    rng = np.random.default_rng(23)
    for w, h in SIZES:
        imgs = frames_of(rng, w, h, frames)
        zero = _run_edge(gvx, dev, imgs, 0x00)
        ones = _run_edge(gvx, dev, imgs, 0xFF)
        for i in range(3):
            for f in range(frames):
                assert np.array_equal(zero[i][f], ones[i][f]), f"{w}x{h}: output {i} depends on row padding"
        for f in range(frames):
            assert np.array_equal(zero[2][f], oracle_mod.port_run(1, imgs[f])), f"{w}x{h} frame {f}"


def _run_harris(gvx, dev, img, k, t, pad):
    c, _ = gvx._load()
    c.gvxb_harris.argtypes = [ctypes.c_void_p, ctypes.POINTER(gvx.GvxbHarrisArgs)]
    h, w = img.shape
    src = Guarded(dev, w, h, 1, fill=pad)
    src.upload([img])
    mask, resp = Guarded(dev, w, h, 1), Guarded(dev, w, h, 4)
    a = gvx.GvxbHarrisArgs()
    a.src, a.mask, a.response = src.image(gvx, 0), mask.image(gvx, 0), resp.image(gvx, 4)
    a.k, a.threshold = k, t
    a.band = gvx.GvxbBand(0, h, h, 0, 0)
    gvx._check_cuda(c.gvxb_harris(dev.h, ctypes.byref(a)))
    dev.sync()
    m = mask.read(np.uint8, f"harris mask {w}x{h}")[0]
    r = resp.read(np.uint32, f"harris response {w}x{h}")[0]
    for b in (src, mask, resp):
        b.free()
    return m, r


def test_harris_stays_inside_its_images(gvx, dev, oracle_mod):
    rng = np.random.default_rng(29)
    for w, h in SIZES:
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        _, want_r = oracle_mod.port_harris(img, 0.04, 0.0)
        finite = want_r[np.isfinite(want_r)]
        t = float(np.quantile(finite, 0.9)) if finite.size else 0.0
        want_m, want_r = oracle_mod.port_harris(img, 0.04, t)
        m0, r0 = _run_harris(gvx, dev, img, 0.04, t, 0x00)
        m1, r1 = _run_harris(gvx, dev, img, 0.04, t, 0xFF)
        assert np.array_equal(m0, m1) and np.array_equal(r0, r1), f"{w}x{h}: depends on row padding"
        assert np.array_equal(m0, want_m), f"{w}x{h}: mask"
        assert np.array_equal(r0, want_r.view(np.uint32)), f"{w}x{h}: response"


STENCILS = {
    "gauss3/16": (np.outer([1, 2, 1], [1, 2, 1]), 16),
    "binomial5/256": (np.outer([1, 4, 6, 4, 1], [1, 4, 6, 4, 1]), 256),
    "binomial7/4096": (np.outer([1, 6, 15, 20, 15, 6, 1], [1, 6, 15, 20, 15, 6, 1]), 4096),
    "cross3/8 (integer kernel)": (np.array([[0, 1, 0], [1, 4, 1], [0, 1, 0]]), 8),
}


def _run_stencil(gvx, dev, imgs, mask, div, mode, pad):
    c, _ = gvx._load()
    c.gvxb_stencil_point.argtypes = [ctypes.c_void_p, ctypes.POINTER(gvx.GvxbStencilArgs)]
    h, w = imgs[0].shape
    n = len(imgs)
    src = Guarded(dev, w, h, 1, n, fill=pad)
    src.upload(imgs)
    dst = Guarded(dev, w, h, 1, n)
    a = gvx.GvxbStencilArgs()
    a.src, a.dst = src.image(gvx, 0), dst.image(gvx, 0)
    a.ksize = mask.shape[0]
    a.mask = gvx._mask49(mask)
    a.div_num, a.div_den, a.mode = 1, div, mode
    a.band = gvx.GvxbBand(0, h, h, 0, 0)
    gvx._check_cuda(c.gvxb_stencil_point(dev.h, ctypes.byref(a)))
    dev.sync()
    out = dst.read(np.uint8, f"stencil {w}x{h}x{n}")
    src.free(), dst.free()
    return out


@pytest.mark.parametrize("name", list(STENCILS))
@pytest.mark.parametrize("mode", [0, 1])
def test_stencil_stays_inside_its_images(name, mode, gvx, dev, oracle_mod):
    mask, div = STENCILS[name]
    rng = np.random.default_rng(31)
    for w, h in SIZES:
        imgs = frames_of(rng, w, h, 2)
        zero = _run_stencil(gvx, dev, imgs, mask, div, mode, 0x00)
        ones = _run_stencil(gvx, dev, imgs, mask, div, mode, 0xFF)
        for f in range(2):
            assert np.array_equal(zero[f], ones[f]), f"{name} {w}x{h}: depends on row padding"
            assert np.array_equal(zero[f], oracle_mod.port_stencil(imgs[f], mask, div, mode)), f"{name} {w}x{h}"


CONV = [
    # mask, scale, shift, wrap, bins, offset, range
    (np.outer([1, 4, 6, 4, 1], [1, 4, 6, 4, 1]), 256, 0, False, 256, 0, 256),
    (np.outer([1, 2, 1], [1, 2, 1]), 16, 0, False, 16, 0, 16),  # identity bins below 256: values >= 16 skipped
    (np.ones((5, 5), np.int64), 8, 1, True, 64, 10, 200),
]


@pytest.mark.parametrize("one_launch", [False, True], ids=["clear+finalize", "one-launch"])
@pytest.mark.parametrize("case", range(len(CONV)))
def test_conv_stats_stays_inside_its_buffers(case, one_launch, gvx, dev, oracle_mod):
    mask, scale, shift, wrap, bins, offset, rng_ = CONV[case]
    c, _ = gvx._load()
    c.gvxb_conv_stats.argtypes = [ctypes.c_void_p, ctypes.POINTER(gvx.GvxbConvStatsArgs)]
    rng = np.random.default_rng(37)
    for w, h in SIZES:
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        src = Guarded(dev, w, h, 1)
        src.upload([img])
        conv = Guarded(dev, w, h, 1)
        # hist (bins gvxb_value of 16 bytes), sum, sumsq, mean, stddev: one guarded row
        aux = Guarded(dev, 16 * bins + 48, 1, 1)
        work = Guarded(dev, 8 * (bins + 1), 1, 1) if one_launch else None
        dev.memset(aux.data, 0, 16 * bins + 48)
        if work:
            dev.memset(work.data, 0, 8 * (bins + 1))
        a = gvx.GvxbConvStatsArgs()
        a.src, a.converted = src.image(gvx, 0), conv.image(gvx, 0)
        a.ksize = mask.shape[0]
        a.mask = gvx._mask49(mask)
        a.scale, a.conv_format, a.shift, a.wrap = scale, 2, shift, int(wrap)
        a.bins, a.offset, a.range = bins, offset, rng_
        a.hist, a.sum, a.sumsq = aux.data, aux.data + 16 * bins, aux.data + 16 * bins + 8
        a.mean, a.stddev = aux.data + 16 * bins + 16, aux.data + 16 * bins + 32
        a.work = work.data if work else None
        gvx._check_cuda(c.gvxb_conv_stats(dev.h, ctypes.byref(a)))
        dev.sync()
        got = conv.read(np.uint8, f"conv_stats converted {w}x{h}")[0]
        raw = aux.read(np.uint8, f"conv_stats hist/sums {w}x{h}")[0].view(np.int64)[0]
        if work:
            assert not work.read(np.uint8, f"conv_stats work {w}x{h}")[0].any(), "scratch left non-zero"
        wconv, whist, wmean, wsd = oracle_mod.port_conv_stats(img, mask, scale, -32768, 32767, shift, wrap, bins,
                                                              offset, rng_)
        assert np.array_equal(got, wconv), f"{w}x{h}: converted"
        assert np.array_equal(raw[1:2 * bins:2], whist), f"{w}x{h}: histogram"
        assert float(raw[2 * bins + 3:2 * bins + 4].view(np.float64)[0]) == wmean, f"{w}x{h}: mean"
        assert float(raw[2 * bins + 5:2 * bins + 6].view(np.float64)[0]) == wsd, f"{w}x{h}: stddev"
        for b in (src, conv, aux) + ((work,) if work else ()):
            b.free()


def test_guard_check_catches_a_stray_byte(gvx, dev):
    """The check itself: one byte of row padding, one of the trailing guard
    and one of the frame gap changed behind the kernel's back are reported."""
    for where in ("padding", "guard", "gap"):
        g = Guarded(dev, 77, 5, 2, 2)
        off = {"padding": 3 * g.pitch + 2 * 77, "guard": 2 * g.stride + 17, "gap": g.pitch * 5 + 100}[where]
        dev.memset(g.data + off, 0, 1)
        with pytest.raises(AssertionError, match="outside the image"):
            g.read(np.int16, where)
        g.free()


BANDS = [(0, 1), (5, 6), (17, 90), (1, 130), (64, 131)]


@pytest.mark.parametrize("kernel", ["edge", "harris", "stencil-sep", "stencil-int", "unsharp"])
def test_band_launches_write_only_their_rows(kernel, gvx, dev, oracle_mod):
    """A row band [r0, r1) of a full-height destination: rows outside the
    band keep their 0xA5, rows inside equal the whole-image oracle."""
    rng = np.random.default_rng(41)
    w, h = 1000, 131
    img = rng.integers(0, 256, (h, w), dtype=np.uint8)
    c, _ = gvx._load()
    if kernel == "edge":
        want = [oracle_mod.port_run(1, img)]
    elif kernel == "harris":
        resp = oracle_mod.port_harris(img, 0.04, 0.0)[1]
        t = float(np.quantile(resp[np.isfinite(resp)], 0.9))
        want = [oracle_mod.port_harris(img, 0.04, t)[0]]
    else:
        mask, div = STENCILS["gauss3/16" if kernel != "stencil-int" else "cross3/8 (integer kernel)"]
        want = [oracle_mod.port_stencil(img, mask, div, int(kernel == "unsharp"))]
    for r0, r1 in BANDS:
        src = Guarded(dev, w, h, 1)
        src.upload([img])
        if kernel == "edge":
            c.gvxb_edge.argtypes = [ctypes.c_void_p, ctypes.POINTER(gvx.GvxbEdgeArgs)]
            dst = Guarded(dev, w, h, 2)
            a = gvx.GvxbEdgeArgs()
            a.src, a.mag, a.with_gauss = src.image(gvx, 0), dst.image(gvx, 2), 1
            a.band = gvx.GvxbBand(r0, r1, h, 0, 0)
            gvx._check_cuda(c.gvxb_edge(dev.h, ctypes.byref(a)))
            dt = np.int16
        elif kernel == "harris":
            c.gvxb_harris.argtypes = [ctypes.c_void_p, ctypes.POINTER(gvx.GvxbHarrisArgs)]
            dst = Guarded(dev, w, h, 1)
            a = gvx.GvxbHarrisArgs()
            a.src, a.mask, a.k, a.threshold = src.image(gvx, 0), dst.image(gvx, 0), 0.04, t
            a.band = gvx.GvxbBand(r0, r1, h, 0, 0)
            gvx._check_cuda(c.gvxb_harris(dev.h, ctypes.byref(a)))
            dt = np.uint8
        else:
            c.gvxb_stencil_point.argtypes = [ctypes.c_void_p, ctypes.POINTER(gvx.GvxbStencilArgs)]
            dst = Guarded(dev, w, h, 1)
            a = gvx.GvxbStencilArgs()
            a.src, a.dst = src.image(gvx, 0), dst.image(gvx, 0)
            a.ksize, a.mask = mask.shape[0], gvx._mask49(mask)
            a.div_num, a.div_den, a.mode = 1, div, int(kernel == "unsharp")
            a.band = gvx.GvxbBand(r0, r1, h, 0, 0)
            gvx._check_cuda(c.gvxb_stencil_point(dev.h, ctypes.byref(a)))
            dt = np.uint8
        dev.sync()
        got = dst.read(dt, f"{kernel} band [{r0}, {r1})", rows=(r0, r1))[0]
        assert np.array_equal(got[r0:r1], want[0][r0:r1]), f"{kernel} band [{r0}, {r1})"
        src.free(), dst.free()

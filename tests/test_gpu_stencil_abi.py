"""GPU parity of the local-operator C-ABI kernels (gvxb_stencil_point,
gvxb_conv_stats) over masks beyond the BASELINE configs: separable masks
that take the packed-FP32 fast path (with and without U8 saturation,
shifts, wrap, non-identity histogram bins) and masks that must fall back
to the exact integer kernel (non-separable, negative taps, odd divisors).
Checked bit-exact against the C restatement (oracle/gvx_oracle.c)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def outer(u, v):
    return np.outer(np.asarray(u, np.int64), np.asarray(v, np.int64))


BIN5 = [1, 4, 6, 4, 1]
MASKS = {
    "binomial5/256": (outer(BIN5, BIN5), 256),
    "gauss3/16": (outer([1, 2, 1], [1, 2, 1]), 16),
    "binomial7/4096": (outer([1, 6, 15, 20, 15, 6, 1], [1, 6, 15, 20, 15, 6, 1]), 4096),
    "box3/8 (saturates)": (np.ones((3, 3), np.int64), 8),
    "asym5/64 (saturates)": (outer([1, 3, 5, 3, 1], [2, 1, 0, 1, 2]), 64),
    "box5/1": (np.ones((5, 5), np.int64), 1),
    "cross3/8 (non-separable)": (np.array([[0, 1, 0], [1, 4, 1], [0, 1, 0]]), 8),
    "sharpen3/1 (negative)": (np.array([[0, -1, 0], [-1, 5, -1], [0, -1, 0]]), 1),
    "box3/9 (odd divisor)": (np.ones((3, 3), np.int64), 9),
}
SIZES = [(1, 1), (3, 2), (77, 41), (384, 9), (385, 70), (1000, 131)]


@pytest.fixture(scope="module")
def dev(gvx):
    return gvx.Device(0)


@pytest.mark.parametrize("name", list(MASKS))
@pytest.mark.parametrize("mode", [0, 1])
def test_stencil_point_matches_oracle(name, mode, dev, gvx, oracle_mod):
    mask, div = MASKS[name]
    rng = np.random.default_rng(7)
    for w, h in SIZES:
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        got = gvx.stencil_point(dev, img, mask, div, mode)
        want = oracle_mod.port_stencil(img, mask, div, mode)
        assert np.array_equal(got, want), f"{name} mode {mode} {w}x{h}"


CONV = [
    # name, mask, scale, shift, wrap, bins, offset, range
    ("binomial5 identity", outer(BIN5, BIN5), 256, 0, False, 256, 0, 256),
    ("binomial5 shift1", outer(BIN5, BIN5), 256, 1, False, 256, 0, 256),
    ("box5/8 saturate", np.ones((5, 5), np.int64), 8, 0, False, 256, 0, 256),
    ("box5/8 wrap", np.ones((5, 5), np.int64), 8, 0, True, 256, 0, 256),
    ("gauss3 16 bins", outer([1, 2, 1], [1, 2, 1]), 16, 0, False, 16, 10, 200),
    ("binomial7 shift2 wrap", outer([1, 6, 15, 20, 15, 6, 1], [1, 6, 15, 20, 15, 6, 1]), 1024, 2, True, 64, 0, 256),
    ("sharpen (negative)", np.array([[0, -1, 0], [-1, 5, -1], [0, -1, 0]]), 1, 0, False, 256, 0, 256),
    ("box3/9 odd", np.ones((3, 3), np.int64), 9, 0, False, 256, 0, 256),
]


@pytest.mark.parametrize("one_launch", [False, True], ids=["clear+finalize", "one-launch"])
@pytest.mark.parametrize("case", CONV, ids=[c[0] for c in CONV])
def test_conv_stats_matches_oracle(case, one_launch, dev, gvx, oracle_mod):
    """Both forms of gvxb_conv_stats: scratch clear + kernel + finalize, and
    the single kernel whose last CTA per frame publishes the results (run
    three times: each run must leave its scratch zero for the next)."""
    name, mask, scale, shift, wrap, bins, offset, rng_ = case
    rng = np.random.default_rng(11)
    for w, h in SIZES:
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        conv, hist, mean, sd = gvx.conv_stats(dev, img, mask, scale, 2, shift, wrap, bins, offset, rng_,
                                              one_launch=one_launch, repeat=3 if one_launch else 1)
        wconv, whist, wmean, wsd = oracle_mod.port_conv_stats(img, mask, scale, -32768, 32767, shift, wrap, bins,
                                                              offset, rng_)
        assert np.array_equal(conv, wconv), f"{name} {w}x{h}: converted image"
        assert np.array_equal(hist, whist), f"{name} {w}x{h}: histogram"
        assert mean == wmean and sd == wsd, f"{name} {w}x{h}: mean/stddev"


def test_conv_stats_full_4k_frame(dev, gvx, oracle_mod):
    img = gvx.random_u8(3840, 2160, 99)
    mask = outer(BIN5, BIN5)
    conv, hist, mean, sd = gvx.conv_stats(dev, img, mask, 256)
    wconv, whist, wmean, wsd = oracle_mod.port_conv_stats(img, mask, 256)
    assert np.array_equal(conv, wconv) and np.array_equal(hist, whist)
    assert mean == wmean and sd == wsd
    assert hist.sum() == 3840 * 2160

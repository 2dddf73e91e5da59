"""GPU parity of the fused Harris kernel (gvxb_harris) where the certified
fp32 decision is stressed: thresholds placed at quantiles of the actual
response distribution (so many pixels sit next to T), negative and large
k, smooth and random images, with and without the observable F32 response.
Bit-exact against the C restatement (oracle/gvx_oracle.c gvxo_harris)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def images(rng):
    h, w = 97, 203
    yy, xx = np.mgrid[0:h, 0:w]
    smooth = ((np.sin(xx / 9.0) + np.cos(yy / 7.0)) * 60 + 128).astype(np.uint8)
    noisy = np.clip(smooth.astype(int) + rng.integers(-20, 21, (h, w)), 0, 255).astype(np.uint8)
    checker = (((xx // 6 + yy // 5) % 2) * 255).astype(np.uint8)
    return {"random": rng.integers(0, 256, (h, w), dtype=np.uint8), "smooth": smooth, "noisy": noisy,
            "checker": checker}


@pytest.mark.parametrize("k", [0.04, 0.15, -0.05])
def test_harris_near_threshold_matches_oracle(k, gvx, oracle_mod):
    dev = gvx.Device(0)
    rng = np.random.default_rng(3)
    for name, img in images(rng).items():
        _, resp = oracle_mod.port_harris(img, k, 0.0)
        finite = resp[np.isfinite(resp)]
        for q in (0.5, 0.8, 0.97):
            T = float(np.quantile(finite, q))
            want, _ = oracle_mod.port_harris(img, k, T)
            got = gvx.harris(dev, img, k, T)
            assert np.array_equal(got, want), f"{name} k={k} q={q} T={T}: {np.count_nonzero(got != want)} px"
            # thresholds exactly on an attained response value
            T2 = float(finite[len(finite) // 3])
            want2, _ = oracle_mod.port_harris(img, k, T2)
            assert np.array_equal(gvx.harris(dev, img, k, T2), want2), f"{name} k={k} T={T2}"


def test_harris_response_image_is_exact(gvx, oracle_mod):
    dev = gvx.Device(0)
    rng = np.random.default_rng(9)
    for name, img in images(rng).items():
        want_m, want_r = oracle_mod.port_harris(img, 0.04, 1e9)
        got_m, got_r = gvx.harris(dev, img, 0.04, 1e9, response=True)
        assert np.array_equal(got_m, want_m), name
        assert np.array_equal(got_r.view(np.uint32), want_r.view(np.uint32)), name


@pytest.mark.parametrize("th", [None, "8", "13"])
def test_harris_strips_bands_and_ragged_sizes(th, gvx, oracle_mod, monkeypatch):
    """Strip placement (last strip pulled left, ragged widths, widths below one
    strip), the TMA row ring across many 8-row chunks, and tall images split
    into many bands (GVX_HARRIS_TH forces short bands)."""
    if th is not None:
        monkeypatch.setenv("GVX_HARRIS_TH", th)
    dev = gvx.Device(0)
    rng = np.random.default_rng(17)
    for (h, w) in [(1, 1), (3, 5), (7, 250), (40, 247), (64, 248), (33, 496), (300, 517), (261, 744), (1030, 1002)]:
        yy, xx = np.mgrid[0:h, 0:w]
        smooth = ((np.sin(xx / 5.0) + np.cos(yy / 4.0)) * 60 + 128).astype(np.uint8)
        for name, img in (("random", rng.integers(0, 256, (h, w), dtype=np.uint8)), ("smooth", smooth)):
            _, resp = oracle_mod.port_harris(img, 0.04, 0.0)
            finite = resp[np.isfinite(resp)]
            T = float(np.quantile(finite, 0.7)) if finite.size else 0.0
            want, _ = oracle_mod.port_harris(img, 0.04, T)
            got = gvx.harris(dev, img, 0.04, T)
            assert np.array_equal(got, want), f"{h}x{w} {name} th={th}: {np.count_nonzero(got != want)} px"

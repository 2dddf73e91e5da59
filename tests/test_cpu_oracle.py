"""The CPU oracle is pinned before it is trusted (tests/golden/ were produced
by the unmodified reference, see tests/golden/make_golden.py)."""
import pathlib

import numpy as np
import pytest

SIZES = [(1, 1), (2, 3), (7, 5), (16, 16), (33, 17), (64, 48), (5, 129), (130, 3)]


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
@pytest.mark.parametrize("size", SIZES)
def test_port_matches_reference_golden(cfg, size, golden, oracle_mod):
    w, h = size
    key = f"c{cfg}_{w}x{h}"
    img = golden[key + "_in"]
    got = oracle_mod.port_run(cfg, img)
    if cfg == 4:
        assert np.array_equal(got[0], golden[key + "_hist"])
        assert got[1] == golden[key + "_stats"][0] and got[2] == golden[key + "_stats"][1]
    else:
        assert np.array_equal(got, golden[key + "_out"])


def test_random_buffer_is_reference_identical(golden, gvx):
    for (w, h) in SIZES:
        for cfg in (1, 2, 3, 4):
            key = f"c{cfg}_{w}x{h}"
            assert np.array_equal(gvx.random_u8(w, h, int(golden[key + "_seed"])), golden[key + "_in"])


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_port_matches_live_reference(cfg, oracle_mod, gvx):
    if not oracle_mod.have_ref():
        pytest.skip("reference oracle not built here (needs /root/reference)")
    for (w, h, seed) in [(97, 61, 3), (200, 33, 4), (1, 40, 5)]:
        img = gvx.random_u8(w, h, seed)
        want, _ = oracle_mod.ref_run(cfg, img)
        got = oracle_mod.port_run(cfg, img)
        if cfg == 4:
            assert np.array_equal(got[0], want[0]) and got[1] == want[1] and got[2] == want[2]
        else:
            assert np.array_equal(got, want)


def test_known_answers_from_reference_tests(oracle_mod):
    """KATs of ref:tests/test_registry.cpp:543-553 (constant 17 is a fixed point of
    the 3x3 blurs) through the restated edge / unsharp chains."""
    c = np.full((9, 11), 17, np.uint8)
    assert (oracle_mod.port_run(1, c) == 0).all()        # no gradient on a constant image
    assert (oracle_mod.port_run(3, c) == 17).all()       # unsharp of a constant is the constant
    hist, mean, sd = oracle_mod.port_run(4, c)
    assert hist[17] == c.size and mean == 17.0 and sd == 0.0


def test_generalised_oracle_agrees_with_pinned_configs(oracle_mod):
    """gvxo_stencil_u8 / gvxo_conv_stats_ex (used for the C-ABI mask sweep)
    reduce to the reference-pinned cfg3 / cfg4 restatements on their masks."""
    rng = np.random.default_rng(5)
    b5 = np.outer([1, 4, 6, 4, 1], [1, 4, 6, 4, 1])
    for w, h in [(1, 1), (7, 5), (64, 48), (130, 3)]:
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        assert np.array_equal(oracle_mod.port_stencil(img, b5, 256, 1), oracle_mod.port_run(3, img))
        conv, hist, mean, sd = oracle_mod.port_conv_stats(img, b5, 256)
        whist, wmean, wsd = oracle_mod.port_run(4, img)
        assert np.array_equal(hist, whist) and mean == wmean and sd == wsd
        # mode 0 output is the blur itself: a constant image stays constant
    c = np.full((9, 11), 200, np.uint8)
    assert (oracle_mod.port_stencil(c, b5, 256, 0) == 200).all()
    assert (oracle_mod.port_stencil(c, np.ones((3, 3)), 8, 0) == 225).all()   # 1800/8 = 225
    assert (oracle_mod.port_stencil(c, np.ones((3, 3)), 4, 0) == 255).all()   # saturates


def test_edge8_magnitude_rounding_is_exact(tmp_path):
    """The fp32 rounding sequence of edge8's magnitude equals the reference's
    llround(sqrt(n)) for every reachable n (tests/cpp/round_sqrt16.c)."""
    import subprocess
    src = pathlib.Path(__file__).resolve().parent / "cpp" / "round_sqrt16.c"
    exe = tmp_path / "rs"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", str(src), "-o", str(exe), "-lm"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert "bad=0" in out, out


def test_reciprocal_cast_is_integer_rounded_division():
    """The generated code replaces the reference's cast(int, x * fl(1/d))
    (double multiply, llround: ref:src/expr.cpp binop / cast_value) by the
    integer half-away division (2|x| + d) / 2d (jit.cpp t_rdiv) when d is
    odd or a power of two and |x| < 2^51.  Check the claim on boundary and
    random x for several d, in IEEE double arithmetic (Python floats) with
    the rounding of the product taken exactly."""
    import math
    import random
    from fractions import Fraction

    def llround(r: float) -> int:  # half away from zero, exact
        q = Fraction(r)
        f = math.floor(abs(q) + Fraction(1, 2))
        return f if q >= 0 else -f

    def rdiv(x: int, d: int) -> int:
        return (2 * x + d) // (2 * d) if x >= 0 else -((d - 2 * x) // (2 * d))

    rng = random.Random(7)
    lim = 1 << 51
    for d in (1, 2, 3, 5, 7, 8, 9, 16, 25, 49, 81, 255, 1023, 4096, 65537):
        c = 1.0 / d
        xs = [0, 1, -1, lim - 1, -(lim - 1)]
        for _ in range(400):
            k = rng.randrange(-(lim // d), lim // d)
            for off in (-1, 0, 1):  # around the half-integer quotients k + 1/2 (ties for even d)
                xs.append(k * d + (d - 1) // 2 + off)
                xs.append(k * d + d // 2 + off)
            xs.append(rng.randrange(-lim + 1, lim))
        for x in xs:
            if abs(x) >= lim:
                continue
            assert llround(float(x) * c) == rdiv(x, d), (x, d)

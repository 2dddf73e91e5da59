"""Reference-pinned parity of the paths the golden corpus does not reach
(tests/reference_graphs.py): user locals with Constant / Undefined borders,
Min / Max combines and real masks, chains of them through virtual
intermediates, U16 images, cfg4's fused statistics with identity bins, and
100 random DAGs.  Each graph runs on the B200 through run_plan (fused) and
run_naive (per node) and on the UNMODIFIED reference engine (oracle/_ref,
run_naive, non-virtual intermediates); the serialised outputs must be equal
byte for byte, and where the reference rejects a graph this library must
reject it with the same error code."""
import json
import pathlib
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO / "tests"))
import reference_graphs as rg  # noqa: E402

SEED = 41
CASES = rg.all_cases()


def blob(outs):
    b = bytearray()
    for kind, payload in outs:
        b += kind.to_bytes(4, "little") + len(payload).to_bytes(4, "little") + payload
    return bytes(b)


def compare(doc, gvx, oracle_mod, seed=SEED, want_fused=None):
    if not oracle_mod.have_ref_graph_io():
        pytest.skip("reference graph_io not built")
    ref_err = None
    try:
        want, ref_counters = oracle_mod.ref_json_run(json.dumps(rg.reference_form(doc)), seed)
    except RuntimeError as e:
        ref_err = str(e)
    if ref_err is not None:
        with pytest.raises(gvx.GraphvxError):
            gvx.GraphFile(json.dumps(doc)).run(naive=True, seed=seed)
        return "rejected"
    g = gvx.GraphFile(json.dumps(doc))
    plan, pc = g.run(naive=False, seed=seed)
    naive, nc = g.run(naive=True, seed=seed)
    assert blob(naive) == want, "run_naive differs from the reference"
    assert blob(plan) == want, "run_plan differs from the reference"
    assert [nc["pixels_read"], nc["pixels_written"]] == ref_counters[1:3], "event counters"
    if want_fused:
        assert want_fused in g.describe(), g.describe()
    return "ok"


@pytest.mark.parametrize("case,doc", CASES, ids=[c for c, _ in CASES])
def test_graph_matches_reference(case, doc, gvx, oracle_mod):
    res = compare(doc, gvx, oracle_mod)
    # every U16 / border / combine case is executable on the reference
    assert res == "ok" or case.startswith(("u16_histogram", "u16_integral")), case


def test_cfg4_shape_fuses_to_conv_stats(gvx):
    doc = dict(rg.stats_cases(257, 131)[0][1])
    assert "conv_stats" in gvx.GraphFile(json.dumps(doc)).describe()


@pytest.mark.parametrize("block", range(4))
def test_random_dags_match_reference(block, gvx, oracle_mod):
    ran = 0
    for seed in range(block * 25 + 1, block * 25 + 26):
        w, h = 5 + seed * 37 % 120, 3 + seed * 11 % 50
        doc = rg.random_dag(seed, w, h)
        if not doc["outputs"]:
            continue
        compare(doc, gvx, oracle_mod, seed=seed)
        ran += 1
    assert ran >= 20


def _harris_doc(w, h, k, t, observable_resp=False):
    doc = json.loads((REPO / "examples" / "cfg2_harris.json").read_text())
    for im in doc["images"]:
        im["width"], im["height"] = w, h
        if observable_resp and im["name"] == "resp":
            im.pop("virtual", None)
    if observable_resp:
        doc["outputs"] = ["resp", "mask"]

    def patch(e):
        if isinstance(e, dict):
            if e.get("op") == "const_f":
                e["value"] = k if e["value"] == 0.04 else t
            for v in e.values():
                patch(v)
        elif isinstance(e, list):
            for v in e:
                patch(v)
    patch(doc["custom_kernels"])
    return doc


@pytest.mark.parametrize("k", [0.04, 0.15, -0.05])
def test_harris_certified_threshold_matches_reference(k, gvx, oracle_mod):
    """The fused Harris kernel decides `resp > T` with a certified fp32
    estimate and falls back to the reference's int64/double expression only
    where the estimate is undecided.  Pin that decision to the UNMODIFIED
    reference at thresholds placed ON response values of the image (ties:
    resp == T gives 0) and at response quantiles, for several k."""
    import numpy as np
    if not oracle_mod.have_ref_graph_io():
        pytest.skip("reference graph_io not built")
    w, h, seed = 211, 97, 3
    blob, _ = oracle_mod.ref_json_run(json.dumps(rg.reference_form(_harris_doc(w, h, k, 1e9, True))), seed)
    outs = gvx.parse_outputs(blob)
    resp = np.frombuffer(outs[0][1], np.float32)
    vals = np.unique(resp)
    picks = [float(vals[i]) for i in np.linspace(0, len(vals) - 1, 9).astype(int)]
    picks += [float(np.quantile(resp, q)) for q in (0.5, 0.9, 0.99)] + [0.0, -1.0]
    for t in picks:
        doc = _harris_doc(w, h, k, t)
        g = gvx.GraphFile(json.dumps(doc))
        assert "harris" in g.describe()  # the fused kernel decides
        want, _ = oracle_mod.ref_json_run(json.dumps(rg.reference_form(doc)), seed)
        got, _ = g.run(naive=False, seed=seed)
        assert blob_of(got) == want, (k, t)


def blob_of(outs):
    return blob(outs)


def test_random_dags_with_interior_tiles_match_reference(gvx, oracle_mod):
    """Random DAGs at 300 x 70, wide and tall enough for the generated region
    kernels' interior tiles (16-byte vector staging and stores, no
    per-entry position tests) next to their border tiles, against the
    unmodified reference."""
    ran = 0
    for seed in range(200, 214):
        doc = rg.random_dag(seed, 300, 70)
        if not doc["outputs"]:
            continue
        compare(doc, gvx, oracle_mod, seed=seed)
        ran += 1
    assert ran >= 10

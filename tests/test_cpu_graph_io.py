"""Graph description files (graph_io.hpp) on the CPU: the corpus in
examples/ loads, verifies, expands and optimizes through the product API;
save_graph_json is canonical (idempotent) and equals the reference's own
serializer (compiled from /root/reference by oracle/Makefile) on every
file — byte-for-byte except that the reference build here links
cudnn-frontend's modified nlohmann copy, which prints integer arrays on
one line; structurally always.  Error behaviour mirrors the reference's
SchemaError cases."""
import json
import pathlib

import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent
CORPUS = sorted((REPO / "examples").glob("*.json"))
GOLDEN = json.loads((REPO / "tests" / "golden" / "corpus.json").read_text())
SCHEMA_ERROR = "SchemaError"


def strict_eq(a, b):
    if type(a) is not type(b):
        return False
    if isinstance(a, dict):
        return a.keys() == b.keys() and all(strict_eq(a[k], b[k]) for k in a)
    if isinstance(a, list):
        return len(a) == len(b) and all(strict_eq(x, y) for x, y in zip(a, b))
    return a == b


def has_int_array(v):
    if isinstance(v, dict):
        return any(has_int_array(x) for x in v.values())
    if isinstance(v, list):
        return (bool(v) and isinstance(v[0], int) and not isinstance(v[0], bool)) or any(has_int_array(x) for x in v)
    return False


def test_corpus_is_complete():
    names = {p.stem for p in CORPUS}
    assert {"gauss", "laplacian", "fchain", "sobelx", "edge_fig1", "sobel", "unsharp", "harris", "tomasi"} <= names
    assert {"cfg1_edge", "cfg2_harris", "cfg3_unsharp", "cfg4_stats"} <= names
    assert set(GOLDEN) == names


@pytest.mark.parametrize("path", CORPUS, ids=[p.stem for p in CORPUS])
def test_canonical_save_matches_reference(path, gvx):
    text = path.read_text()
    ours = gvx.json_roundtrip(text)
    assert gvx.json_roundtrip(ours) == ours, "save_graph_json is not canonical"
    ref = GOLDEN[path.stem]["canonical"]
    assert strict_eq(json.loads(ours), json.loads(ref))
    if not has_int_array(json.loads(ref)):
        assert ours == ref


@pytest.mark.parametrize("path", CORPUS, ids=[p.stem for p in CORPUS])
def test_live_reference_roundtrip(path, gvx, oracle_mod):
    if not oracle_mod.have_ref_graph_io():
        pytest.skip("reference graph_io not built (needs /root/reference + nlohmann)")
    text = path.read_text()
    assert strict_eq(json.loads(gvx.json_roundtrip(text)), json.loads(oracle_mod.ref_json_roundtrip(text)))


def test_corpus_node_counts_and_dce(gvx):
    st = {p.stem: gvx.GraphFile(p.read_text()).pass_stats() for p in CORPUS}
    # Listing 1 / Fig. 1: 6 implementation nodes, the unused
    # Sobel half is eliminated
    assert (st["edge_fig1"]["nodes_before"], st["edge_fig1"]["nodes_alive"], st["edge_fig1"]["nodes_removed"]) == (6, 5, 1)
    # paper Section 6: Harris 4 local + 9 point CV nodes, Tomasi 4 + 10 (Sobel3x3 expands to 2)
    docs = {p.stem: json.loads(p.read_text()) for p in CORPUS}
    assert len(docs["harris"]["nodes"]) == 13 and len(docs["tomasi"]["nodes"]) == 14
    assert st["harris"]["nodes_before"] == 14 and st["tomasi"]["nodes_before"] == 15
    assert st["unsharp"]["launches_after"] == 1 and st["cfg3_unsharp"]["launches_after"] == 1
    for name in ("unsharp", "harris", "tomasi"):  # fusible point chains
        assert st[name]["launches_after"] < st[name]["launches_before"], name


def test_expression_and_kernel_blocks_roundtrip(gvx):
    text = (REPO / "examples" / "tomasi.json").read_text()
    ours = json.loads(gvx.json_roundtrip(text))
    src = json.loads(text)
    assert strict_eq(ours["custom_kernels"], src["custom_kernels"])


@pytest.mark.parametrize("text,fragment", [
    ("{not json", "not valid JSON"),
    ("[1, 2]", "must be an object"),
    ('{"images": [{"name": "a", "width": 4, "height": 4, "format": "U8"},'
     ' {"name": "a", "width": 4, "height": 4, "format": "U8"}]}', "duplicate object name"),
    ('{"images": [{"name": "a", "width": 4, "height": 4, "format": "Q9"}]}', "bad image format"),
    ('{"nodes": [{"kernel": "Copy", "params": ["nope"]}]}', "no object named 'nope'"),
    ('{"scalars": [{"name": "s", "virtual": true}]}', "scalars cannot be virtual"),
    ('{"custom_kernels": [{"name": "k", "kind": "local", "window": [3, 3], "boundary": "wrap",'
     ' "signature": [{"direction": "output"}], "tap_body": {"op": "win"}}]}', "bad boundary mode"),
    ('{"custom_kernels": [{"name": "k", "kind": "reduce", "signature": [{"direction": "output"}]}]}',
     "must be point or local"),
    ('{"custom_kernels": [{"name": "k", "kind": "point", "signature": [{"direction": "output"}],'
     ' "body": {"op": "frobnicate"}}]}', "unknown expression op"),
    ('{"nodes": [{"kernel": "Copy", "attrs": {"x": [1]}}]}', "must be scalar"),
])
def test_schema_errors(text, fragment, gvx):
    with pytest.raises(gvx.GraphvxError) as e:
        gvx.json_roundtrip(text)
    assert e.value.code == SCHEMA_ERROR and fragment in str(e.value), str(e.value)


def test_numbers_keep_their_json_types(gvx):
    text = json.dumps({"name": "n", "images": [], "nodes": [{"kernel": "X", "params": [],
                      "attrs": {"i": 3, "f": 3.0, "e": 1e-7, "big": 1.5e300, "neg": -0.25, "s": "a\"b\\n"}}]})
    out = json.loads(gvx.json_roundtrip(text))
    attrs = out["nodes"][0]["attrs"]
    assert type(attrs["i"]) is int and type(attrs["f"]) is float
    assert attrs["e"] == 1e-7 and attrs["big"] == 1.5e300 and attrs["neg"] == -0.25 and attrs["s"] == 'a"b\\n'
    assert '"f": 3.0' in gvx.json_roundtrip(text) and '"e": 1e-07' in gvx.json_roundtrip(text)


def test_kernel_golden_covers_every_case():
    """tests/golden/kernels.json (reference run_naive of every built-in
    kernel as a one-node graph file) matches tests/kernel_graphs.py."""
    import sys
    sys.path.insert(0, str(REPO / "tests"))
    import kernel_graphs
    gold = json.loads((REPO / "tests" / "golden" / "kernels.json").read_text())
    cases = {c for c, _ in kernel_graphs.all_cases()}
    assert cases == set(gold["cases"]) | set(gold["reference_errors"])
    # the only reference failures are its ScaleImage / EqualizeHist defects
    assert {c.split("_")[0] for c in gold["reference_errors"]} == {"ScaleImage", "EqualizeHist"}


def test_loaded_kernel_cases_verify(gvx):
    import sys
    sys.path.insert(0, str(REPO / "tests"))
    import kernel_graphs
    for case, text in kernel_graphs.all_cases():
        gvx.GraphFile(text)  # load + verify + expand + optimize (no device needed)


def test_attribute_fuzz_roundtrip(gvx, oracle_mod):
    """Random attribute strings (escapes, control characters, unicode) and
    numbers (integers, subnormal / huge doubles) survive load -> save ->
    load, and match the reference serializer when it is available."""
    import random
    rng = random.Random(1234)
    alphabet = ['a', 'Z', '"', '\\\\', '/', '\\n', '\\t', '\\x01', '\\x1f', 'é', '€', '😀', ' ', '{', '}']
    for trial in range(60):
        attrs = {}
        for k in range(rng.randint(1, 6)):
            key = "k" + "".join(rng.choice("abcxyz_") for _ in range(rng.randint(1, 6)))
            kind = rng.randint(0, 3)
            if kind == 0:
                attrs[key] = "".join(rng.choice(alphabet) for _ in range(rng.randint(0, 12)))
            elif kind == 1:
                attrs[key] = rng.randint(-2 ** 62, 2 ** 62)
            elif kind == 2:
                attrs[key] = rng.choice([0.0, -0.0, 5e-324, 1.7976931348623157e308, 1e-7, 123456.789, -2.5e22])
            else:
                attrs[key] = rng.uniform(-1e6, 1e6) * 10 ** rng.randint(-30, 30)
        doc = {"name": "fuzz", "images": [], "nodes": [{"kernel": "Copy", "params": [], "attrs": attrs}]}
        text = json.dumps(doc)
        ours = gvx.json_roundtrip(text)
        back = json.loads(ours)["nodes"][0]["attrs"]
        assert strict_eq(back, attrs), (trial, attrs, back)
        assert gvx.json_roundtrip(ours) == ours
        if oracle_mod.have_ref_graph_io():
            assert ours == oracle_mod.ref_json_roundtrip(text), trial

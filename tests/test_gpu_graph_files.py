"""GPU parity of the graph-file corpus (examples/*.json): each file is
loaded through graph_io, verified, expanded, optimized and executed on the
B200 with run_plan (fused) and run_naive (per-node NVRTC kernels), with
virtual intermediates as written and with every intermediate made
non-virtual (the form the reference can execute).  All four runs must
reproduce the reference's run_naive outputs bit-for-bit (SHA-256 in
tests/golden/corpus.json, generated from the unmodified reference) and the
non-virtual run_naive must reproduce its event counters exactly."""
import hashlib
import json
import pathlib

import pytest

pytestmark = pytest.mark.gpu

REPO = pathlib.Path(__file__).resolve().parent.parent
CORPUS = sorted((REPO / "examples").glob("*.json"))
GOLDEN = json.loads((REPO / "tests" / "golden" / "corpus.json").read_text())


def devirtualise(text):
    d = json.loads(text)
    for im in d.get("images", []):
        im.pop("virtual", None)
    return json.dumps(d)


def blob(outs):
    b = bytearray()
    for kind, payload in outs:
        b += kind.to_bytes(4, "little") + len(payload).to_bytes(4, "little") + payload
    return bytes(b)


@pytest.mark.parametrize("path", CORPUS, ids=[p.stem for p in CORPUS])
def test_corpus_graph_matches_reference(path, gvx):
    gold = GOLDEN[path.stem]
    text = path.read_text()
    for variant, src in (("virtual", text), ("plain", devirtualise(text))):
        g = gvx.GraphFile(src)
        launches = {}
        for naive in (False, True):
            outs, counters = g.run(naive=naive, seed=gold["seed"])
            digest = hashlib.sha256(blob(outs)).hexdigest()
            assert digest == gold["sha256"], f"{path.stem} {variant} {'naive' if naive else 'plan'}"
            if naive and variant == "plain":
                assert [counters[k] for k in ("kernel_launches", "pixels_read", "pixels_written",
                                              "transfers_executed")][1:] == gold["counters"][1:]
            launches[naive] = counters["kernel_launches"]
        assert launches[False] <= launches[True], (path.stem, variant, launches)


@pytest.mark.parametrize("stem", ["sobel", "harris", "tomasi"])
def test_generic_regions_fuse_and_match_reference(stem, gvx):
    """Graphs outside the hand-written groups fuse into generated regions
    (convex DAG regions of point / local nodes as one kernel,
    intermediates in shared memory): fewer launches than run_naive, outputs
    bit-exact with the reference's."""
    gold = GOLDEN[stem]
    g = gvx.GraphFile((REPO / "examples" / f"{stem}.json").read_text())
    assert "region" in g.describe(), g.describe()
    outs, counters = g.run(naive=False, seed=gold["seed"])
    assert hashlib.sha256(blob(outs)).hexdigest() == gold["sha256"]
    _, naive = g.run(naive=True, seed=gold["seed"])
    assert counters["kernel_launches"] < naive["kernel_launches"]

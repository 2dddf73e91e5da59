"""Fusion with observable intermediates: for every corpus graph, random
subsets of its intermediates are made non-virtual and declared as outputs
(so the fused program must also store them), then run_plan and run_naive on
the B200 are compared with the UNMODIFIED reference engine (oracle/_ref,
all intermediates non-virtual, same declared outputs) bit-for-bit."""
import json
import pathlib
import random
import zlib

import pytest

pytestmark = pytest.mark.gpu

REPO = pathlib.Path(__file__).resolve().parent.parent
CORPUS = sorted((REPO / "examples").glob("*.json"))


def variants(text, n, seed):
    doc = json.loads(text)
    mids = [im["name"] for im in doc["images"] if im.get("virtual")]
    rng = random.Random(seed)
    out = []
    for k in range(n):
        keep = {m for m in mids if rng.random() < 0.5}
        d = json.loads(text)
        for im in d["images"]:
            if im["name"] in keep:
                im.pop("virtual", None)
        d["outputs"] = d["outputs"] + sorted(keep)
        ref = json.loads(json.dumps(d))
        for im in ref["images"]:
            im.pop("virtual", None)
        out.append((json.dumps(d), json.dumps(ref)))
    return out


@pytest.mark.parametrize("path", CORPUS, ids=[p.stem for p in CORPUS])
def test_observable_intermediates_match_reference(path, gvx, oracle_mod):
    if not oracle_mod.have_ref_graph_io():
        pytest.skip("reference graph_io not built")
    for ours_text, ref_text in variants(path.read_text(), 3, zlib.crc32(path.stem.encode())):
        want, _ = oracle_mod.ref_json_run(ref_text, 5)
        g = gvx.GraphFile(ours_text)
        for naive in (False, True):
            outs, _ = g.run(naive=naive, seed=5)
            blob = b"".join(k.to_bytes(4, "little") + len(p).to_bytes(4, "little") + p for k, p in outs)
            assert blob == want, (path.stem, naive, json.loads(ours_text)["outputs"])

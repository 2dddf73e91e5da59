"""run_plan's host path for large frames (execute.cpp host_piece_rows):
single-group stencil / point programs run in row pieces whose host copies,
transfers and kernels overlap (BandedSession::run_host_rows over a
whole-image band).  Every variant must equal the whole-frame result:
pageable InputMap buffers (staged both ways), the C facade's page-locked
input / pooled outputs, the caller's destination filled piece by piece,
piece counts that do not divide the height, and generated (NVRTC) programs
against run_naive (per-node kernels on whole frames)."""
import json
import pathlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = pathlib.Path(__file__).resolve().parent.parent
sys_path = str(REPO / "tests")


def _fixtures():
    import sys
    sys.path.insert(0, sys_path)
    import test_gpu_fullsize as fs
    return fs


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_pieces_facade_paths_match_reference(cfg, gvx):
    fs = _fixtures()
    fx = fs.FULL[str(cfg)]
    w, h = fx["width"], fx["height"]
    img = gvx.random_u8(w, h, cfg)
    g = gvx.ConfigGraph(cfg, w, h)
    dst = g.output_array()
    for _ in range(2):  # second run: recycled page-locked outputs, destination drained piece by piece
        dst[:] = 0
        got, cnt = g.run_host(img, out=dst)
        fs.check_image(fx, got)
        assert cnt["kernel_launches"] >= 1
    view, _ = g.run_host_inplace(img)  # result left in the pooled output
    fs.check_image(fx, view)
    got, _ = g.run_host(img)  # a fresh destination array
    fs.check_image(fx, got)
    g.close()


def _resize(doc, w, h):
    doc = json.loads(json.dumps(doc))
    for im in doc["images"]:
        im["width"], im["height"] = w, h
    return doc


@pytest.mark.parametrize("name", ["cfg1_edge", "cfg2_harris", "cfg3_unsharp", "gauss", "laplacian", "sobel",
                                  "sobelx", "unsharp"])
@pytest.mark.parametrize("size", [(2304, 2049), (4100, 1031)])
def test_pieces_equal_whole_frames(name, size, gvx):
    """Plan (row pieces when the program is one group) against run_naive
    (per-node programs: whole frames) on pageable InputMap buffers."""
    doc = _resize(json.loads((REPO / "examples" / f"{name}.json").read_text()), *size)
    g = gvx.GraphFile(json.dumps(doc))
    plan, _ = g.run(naive=False, seed=3)
    naive, _ = g.run(naive=True, seed=3)
    assert plan == naive


@pytest.mark.parametrize("name,observe", [("cfg2_harris", ["resp"]), ("cfg1_edge", ["gx", "gy"])])
def test_pieces_with_observable_intermediates(name, observe, gvx):
    """Several image outputs (one F32) streamed back piece by piece: the
    Harris response next to the mask, the edge graph's gx / gy next to the
    magnitude, against run_naive."""
    doc = _resize(json.loads((REPO / "examples" / f"{name}.json").read_text()), 2304, 2049)
    for im in doc["images"]:
        if im["name"] in observe:
            im.pop("virtual", None)
    doc["outputs"] = list(dict.fromkeys(doc["outputs"] + observe))
    g = gvx.GraphFile(json.dumps(doc))
    plan, _ = g.run(naive=False, seed=5)
    naive, _ = g.run(naive=True, seed=5)
    assert len(plan) == len(doc["outputs"])
    assert plan == naive

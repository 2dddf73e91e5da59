"""Row-band execution through the library (gvx::BandedSession /
gvx::BandGroup, device.hpp): every bandable BASELINE graph (edge, Harris,
user 5x5 unsharp) split into 1..8 bands at border-heavy sizes, halo rows
exchanged by the group (poisoned beforehand, so a missing row shows), must
equal the single-image run_plan result; the NCCL path with one rank, the
pipelined host path and the error contract are covered too."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OUT_DT = {1: np.int16, 2: np.uint8, 3: np.uint8, 5: np.int16}


def run_group(gvx, cfg, img, world, poison=True, launches=1):
    H, W = img.shape
    g = gvx.ConfigGraph(cfg, W, H)
    grp = gvx.BandGroup(g, [0] * world)
    for b in grp.bands:
        L = b.layout
        if poison:  # halo rows must come from the neighbours
            b.upload(0, np.full((L["src_row1"] - L["src_row0"], W), 0xA5, np.uint8), L["src_row0"])
        b.upload(0, img[L["row0"]:L["row1"]], L["row0"])
    for _ in range(launches):
        grp.launch()
    grp.sync()
    out = np.empty((H, W), OUT_DT[cfg])
    for b in grp.bands:
        L = b.layout
        out[L["row0"]:L["row1"]] = b.download(1, L["row0"], L["row1"] - L["row0"], OUT_DT[cfg])
    grp.close()
    return out


@pytest.mark.parametrize("cfg", [1, 2, 3])
@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("size", [(64, 40), (257, 131), (1000, 77)])
def test_band_group_equals_whole_image(cfg, world, size, gvx):
    W, H = size
    if H // world < 2:
        pytest.skip("bands thinner than the halo")
    img = gvx.random_u8(W, H, 300 + cfg)
    want, _ = gvx.ConfigGraph(cfg, W, H).run_host(img)
    got = run_group(gvx, cfg, img, world, launches=2)
    assert np.array_equal(got, want)


def test_band_plan_rejects_bands_thinner_than_halo(gvx):
    with pytest.raises(gvx.GraphvxError):
        gvx.BandGroup(gvx.ConfigGraph(1, 64, 9), [0] * 8)  # 1-row bands, halo 2


def test_bands_need_stencil_groups(gvx):
    # cfg4 ends in global reductions: frames are its unit of parallelism
    with pytest.raises(gvx.GraphvxError, match="row-band"):
        gvx.Band(gvx.ConfigGraph(4, 64, 64))


def test_single_band_nccl_communicator(gvx):
    """world = 1 through an NCCL communicator (the code path torchrun ranks
    take; no neighbours, so no messages) equals run_plan."""
    c, _ = gvx.libraries()
    if not c.gvxb_comm_available():
        pytest.skip("NCCL not loadable")
    W, H = 300, 123
    img = gvx.random_u8(W, H, 9)
    comm = gvx.Comm(0, 1, 0, uid=gvx.Comm.unique_id())
    assert comm.allreduce_max(3.5) == 3.5
    comm.barrier()
    g = gvx.ConfigGraph(1, W, H)
    b = gvx.Band(g, 0, 1, comm)
    b.upload(0, img, 0)
    b.launch()
    b.sync()
    got = b.download(1, 0, H, np.int16)
    want, _ = gvx.ConfigGraph(1, W, H).run_host(img)
    assert np.array_equal(got, want)
    b.close()
    comm.close()


@pytest.mark.parametrize("world,rank", [(1, 0), (3, 1), (4, 3)])
def test_run_host_pipeline_equals_whole_band(world, rank, gvx):
    """BandedSession::run_host (pieces pipelined over three streams, page-
    locked host rows) equals the band of the whole-image result."""
    W, H = 1500, 900
    img = gvx.random_u8(W, H, 17)
    want, _ = gvx.ConfigGraph(5, W, H).run_host(img)
    g = gvx.ConfigGraph(5, W, H)
    comm = None
    b = gvx.Band(g, rank, world, comm) if world == 1 else None
    if b is None:
        # a middle band of a multi-rank split, fed with its slab from the host
        grp = gvx.BandGroup(g, [0] * world)
        b = grp.bands[rank]
    L = b.layout
    src = gvx.HostBuffer((L["src_row1"] - L["src_row0"], W), np.uint8)
    src.array[:] = img[L["src_row0"]:L["src_row1"]]
    dst = gvx.HostBuffer((L["row1"] - L["row0"], W), np.int16)
    for piece in (64, 1024):
        dst.array[:] = -1
        b.run_host(src.ptr, W, 1, dst.ptr, 2 * W, piece)
        assert np.array_equal(dst.array, want[L["row0"]:L["row1"]]), piece

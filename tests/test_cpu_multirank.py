"""The N>1 path of config 5 on CPU: world_size-2 gloo ranks row-band an
image, exchange halo rows with paper_2008_11476_b200.bands.halo_exchange
(the same code bench.py runs over NCCL), run the edge graph on each halo'd
slab, keep the owned rows and reassemble: the result must equal the
single-image result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, w, h, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2008_11476_b200 as gvx
    from paper_2008_11476_b200.bands import band_slab, halo_exchange

    full = gvx.random_u8(w, h, 5)
    r0, r1, s0, s1 = band_slab(h, world, rank, 2)
    slab = torch.zeros((s1 - s0, w), dtype=torch.uint8)
    slab[r0 - s0:r1 - s0] = torch.from_numpy(full[r0:r1])  # only owned rows are local
    halo_exchange(dist, slab, r0, r1, s0, s1, rank, world, 2)
    ok_halo = bool(np.array_equal(slab.numpy(), full[s0:s1]))
    # slab-local Clamp differs from global Clamp only within `halo` rows of an
    # interior cut, which are never owned rows
    mag = oracle.port_run(1, slab.numpy())[r0 - s0:r1 - s0]
    gathered = [torch.zeros(1) for _ in range(world)]
    obj = [None] * world
    dist.all_gather_object(obj, (r0, r1, mag, ok_halo))
    if rank == 0:
        q.put(obj)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,w,h", [(2, 67, 41), (2, 16, 5), (3, 31, 29)])
def test_banded_edge_graph_equals_full_image(world, w, h):
    import oracle
    import paper_2008_11476_b200 as gvx
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, w, h, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    full = gvx.random_u8(w, h, 5)
    want = oracle.port_run(1, full)
    got = np.zeros_like(want)
    for r0, r1, mag, ok_halo in parts:
        assert ok_halo
        got[r0:r1] = mag
    assert np.array_equal(got, want)


def _overlap_worker(rank, world, port, w, h, q):
    """bench.py's overlapped cfg5 step: post the halo exchange, compute the
    interior rows from owned rows only (halo rows poisoned here to prove it),
    wait, then compute the edge rows."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2008_11476_b200 as gvx
    from paper_2008_11476_b200.bands import band_pieces, band_slab, halo_exchange_start

    full = gvx.random_u8(w, h, 7)
    r0, r1, s0, s1 = band_slab(h, world, rank, 2)
    slab = torch.full((s1 - s0, w), 0xAA, dtype=torch.uint8)
    slab[r0 - s0:r1 - s0] = torch.from_numpy(full[r0:r1])
    before = slab.clone()  # what the interior pass may see: halo not yet arrived
    works = halo_exchange_start(dist, slab, r0, r1, s0, s1, rank, world, 2)
    interior, edges = band_pieces(r0, r1, rank, world, 2)

    def rows(src, a, b):  # edge magnitude of global rows [a, b) from a slab (global rows s0..s1)
        lo, hi = max(s0, a - 2), min(s1, b + 2)
        return oracle.port_run(1, src[lo - s0:hi - s0].numpy())[a - lo:b - lo]

    out = np.zeros((r1 - r0, w), np.int16)
    if interior:
        out[interior[0] - r0:interior[1] - r0] = rows(before, *interior)
    for work in works:
        work.wait()
    for a, b in edges:
        out[a - r0:b - r0] = rows(slab, a, b)
    pieces = ([interior] if interior else []) + edges
    obj = [None] * world
    dist.all_gather_object(obj, (r0, r1, out, sorted(pieces)))
    if rank == 0:
        q.put(obj)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,w,h", [(2, 67, 41), (3, 31, 29), (4, 19, 9)])
def test_overlapped_band_step_equals_full_image(world, w, h):
    import oracle
    import paper_2008_11476_b200 as gvx
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overlap_worker, args=(r, world, port, w, h, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    want = oracle.port_run(1, gvx.random_u8(w, h, 7))
    got = np.zeros_like(want)
    for r0, r1, out, pieces in parts:
        covered = []
        for a, b in pieces:
            covered.extend(range(a, b))
        assert covered == list(range(r0, r1))  # the pieces partition the band
        got[r0:r1] = out
    assert np.array_equal(got, want)


def test_band_pieces_partition():
    from paper_2008_11476_b200.bands import band_pieces
    for world in (1, 2, 3, 8):
        for rank in range(world):
            for r0, r1 in ((0, 1), (5, 6), (10, 13), (0, 100), (40, 44), (40, 45)):
                interior, edges = band_pieces(r0, r1, rank, world, 2)
                rows = []
                for a, b in ([interior] if interior else []) + edges:
                    assert a < b
                    rows.extend(range(a, b))
                assert sorted(rows) == list(range(r0, r1))
                if interior:
                    assert interior[0] >= r0 + (2 if rank > 0 else 0)
                    assert interior[1] <= r1 - (2 if rank < world - 1 else 0)

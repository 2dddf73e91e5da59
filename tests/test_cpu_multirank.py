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

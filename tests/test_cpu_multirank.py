"""The N>1 row-band path on CPU with world-size 2..4 gloo ranks.

Each rank takes its rows, slab, overlap split and exchange schedule from
the library's band planner (gvxb_band_plan_make, the same plan
gvx::BandedSession executes with NCCL on the GPUs), holds only its owned
input rows (the halo rows are poisoned), executes the plan's sends and
receives over gloo, computes the interior rows BEFORE the exchange has
completed (from the poisoned slab, proving they read owned rows only) and
the edge rows after, with the C restatement of the edge graph standing in
for the device kernel.  The reassembled image must equal the single-image
result."""
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


def post_exchange(plan, slab):
    """The plan's sends / receives as gloo P2P ops on a slab tensor whose row
    0 is global row plan['src_row0'] (gvxb_halo_start does the same with
    ncclSend / ncclRecv inside one group)."""
    s0 = plan["src_row0"]
    ops = []
    for side in plan["peers"]:
        if side is None:
            continue
        a, b = side["send"]
        ops.append(dist.P2POp(dist.isend, slab[a - s0:b - s0].contiguous(), side["peer"]))
        a, b = side["recv"]
        ops.append(dist.P2POp(dist.irecv, slab[a - s0:b - s0], side["peer"]))
    return dist.batch_isend_irecv(ops) if ops else []


def _worker(rank, world, port, w, h, halo, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2008_11476_b200 as gvx

    full = gvx.random_u8(w, h, 7)
    p = gvx.band_plan(h, world, rank, halo)
    r0, r1, s0, s1 = p["row0"], p["row1"], p["src_row0"], p["src_row1"]
    slab = torch.full((s1 - s0, w), 0xAA, dtype=torch.uint8)
    slab[r0 - s0:r1 - s0] = torch.from_numpy(full[r0:r1])  # only owned rows are local
    before = slab.clone()  # what the interior pass may see: halo not yet arrived
    works = post_exchange(p, slab)

    def rows(src, a, b):  # edge magnitude of global rows [a, b) from a slab (global rows s0..s1)
        lo, hi = max(s0, a - halo), min(s1, b + halo)
        return oracle.port_run(1, src[lo - s0:hi - s0].numpy())[a - lo:b - lo]

    out = np.zeros((r1 - r0, w), np.int16)
    i0, i1 = p["interior_row0"], p["interior_row1"]
    if i1 > i0:
        out[i0 - r0:i1 - r0] = rows(before, i0, i1)
    for work in works:
        work.wait()
    ok_halo = bool(np.array_equal(slab.numpy(), full[s0:s1]))
    for a, b in p["edges"]:
        out[a - r0:b - r0] = rows(slab, a, b)
    pieces = ([(i0, i1)] if i1 > i0 else []) + p["edges"]
    obj = [None] * world
    dist.all_gather_object(obj, (r0, r1, out, sorted(pieces), ok_halo))
    if rank == 0:
        q.put(obj)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,w,h", [(2, 67, 41), (2, 16, 5), (3, 31, 29), (4, 19, 9)])
def test_banded_edge_graph_equals_full_image(world, w, h):
    import oracle
    import paper_2008_11476_b200 as gvx
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, w, h, 2, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    want = oracle.port_run(1, gvx.random_u8(w, h, 7))
    got = np.zeros_like(want)
    for r0, r1, out, pieces, ok_halo in parts:
        assert ok_halo
        covered = []
        for a, b in pieces:
            covered.extend(range(a, b))
        assert covered == list(range(r0, r1))  # the pieces partition the band
        got[r0:r1] = out
    assert np.array_equal(got, want)


def test_band_plans_partition_and_pair_up():
    """Every band plan: rows partition the image, interior + edges partition
    the band, interior rows read owned rows only, and each send of one rank
    is exactly the matching receive of its neighbour."""
    import paper_2008_11476_b200 as gvx
    for h in (4, 9, 100, 16384):
        for world in (1, 2, 3, 4, 8):
            for halo in (0, 1, 2, 3):
                if world > 1 and h // world < halo:
                    with pytest.raises(gvx.GraphvxError):
                        gvx.band_plan(h, world, 0, halo)
                    continue
                plans = [gvx.band_plan(h, world, r, halo) for r in range(world)]
                assert plans[0]["row0"] == 0 and plans[-1]["row1"] == h
                for r, p in enumerate(plans):
                    if r:
                        assert p["row0"] == plans[r - 1]["row1"]
                    rows = list(range(p["interior_row0"], p["interior_row1"]))
                    for a, b in p["edges"]:
                        rows.extend(range(a, b))
                    assert sorted(rows) == list(range(p["row0"], p["row1"]))
                    if p["interior_row1"] > p["interior_row0"]:
                        assert p["interior_row0"] - halo >= (p["row0"] if r else -halo)
                        assert p["interior_row1"] + halo <= (p["row1"] if r < world - 1 else h + halo)
                    assert p["src_row0"] == max(0, p["row0"] - halo) and p["src_row1"] == min(h, p["row1"] + halo)
                    for s, side in enumerate(p["peers"]):
                        if side is None:
                            continue
                        q = plans[side["peer"]]["peers"][1 - s]
                        assert q is not None and q["peer"] == r
                        assert q["recv"] == side["send"] and q["send"] == side["recv"]
                        lo, hi = side["recv"]
                        assert (lo, hi) == ((p["src_row0"], p["row0"]) if s == 0 else (p["row1"], p["src_row1"]))

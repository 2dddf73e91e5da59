"""Multi-GPU row-band scheduler for large images (BASELINE config 5).

Band g of G owns global rows [row0, row1) (balanced split, gvxb_band_rows in
the C-ABI).  A fused stencil group of total radius R needs source rows
[row0 - R, row1 + R) clipped to the image; the R rows on each side that a
rank does not own are exchanged with its neighbours, point to point, once
per group execution — the only collective on this path.
Clamp borders use *global* rows, so only the first and last bands clamp.

The exchange runs on torch.distributed tensors: NCCL over NVLink on the GPU
box, gloo in the CPU tests (tests/test_cpu_multirank.py).
"""
from __future__ import annotations


def band_slab(height: int, world: int, rank: int, halo: int, band_rows=None):
    """(row0, row1, src_row0, src_row1) of rank's band and its halo'd slab."""
    if band_rows is None:
        from . import band_rows as _band_rows  # C-ABI gvxb_band_rows
        band_rows = _band_rows
    r0, r1 = band_rows(height, world, rank)
    return r0, r1, max(0, r0 - halo), min(height, r1 + halo)


def band_pieces(r0: int, r1: int, rank: int, world: int, halo: int):
    """Split band [r0, r1) for overlap: (interior, edges).  `interior` rows
    read only owned source rows, so they are computed while the halo rows
    are in flight; each `edges` range reads halo rows and runs after the
    exchange.  The ranges partition [r0, r1); a band thinner than 2 halos
    is all edge."""
    lo = r0 + halo if rank > 0 else r0
    hi = r1 - halo if rank < world - 1 else r1
    if lo >= hi:
        return None, [(r0, r1)] if r1 > r0 else []
    edges = []
    if lo > r0:
        edges.append((r0, lo))
    if hi < r1:
        edges.append((hi, r1))
    return (lo, hi), edges


def halo_exchange_start(dist, slab, r0: int, r1: int, s0: int, s1: int, rank: int, world: int, halo: int):
    """Post the halo sends / receives of halo_exchange and return the
    requests without waiting (wait() on each before reading the halo)."""
    if world <= 1:
        return []
    ops = []
    if rank > 0 and r0 > s0:
        ops.append(dist.P2POp(dist.isend, slab[r0 - s0:r0 - s0 + halo], rank - 1))
        ops.append(dist.P2POp(dist.irecv, slab[0:r0 - s0], rank - 1))
    if rank < world - 1 and s1 > r1:
        ops.append(dist.P2POp(dist.isend, slab[r1 - s0 - halo:r1 - s0], rank + 1))
        ops.append(dist.P2POp(dist.irecv, slab[r1 - s0:s1 - s0], rank + 1))
    return dist.batch_isend_irecv(ops) if ops else []


def halo_exchange(dist, slab, r0: int, r1: int, s0: int, s1: int, rank: int, world: int, halo: int) -> None:
    """Fill the halo rows of `slab` (global rows s0..s1) from the neighbours.

    `slab` is a torch tensor of shape (s1 - s0, W) whose owned rows
    [r0, r1) are valid.  Sends my first / last `halo` owned rows, receives
    the neighbours' into my halo.
    """
    if world <= 1:
        return
    ops = []
    if rank > 0 and r0 > s0:
        ops.append(dist.P2POp(dist.isend, slab[r0 - s0:r0 - s0 + halo].contiguous(), rank - 1))
        top = slab[0:r0 - s0]
        ops.append(dist.P2POp(dist.irecv, top, rank - 1))
    if rank < world - 1 and s1 > r1:
        ops.append(dist.P2POp(dist.isend, slab[r1 - s0 - halo:r1 - s0].contiguous(), rank + 1))
        bottom = slab[r1 - s0:s1 - s0]
        ops.append(dist.P2POp(dist.irecv, bottom, rank + 1))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()

"""Multi-GPU sharding of the distance-transform path.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing.

* C3 (a batch of independent images): rank r owns images
  [r*n/N, (r+1)*n/N); no data-path collective.
* C5 (one giant image, north_star): rank r owns the column stripe
  [r*W/N, (r+1)*W/N).  Stage 1 (per-column nearest-object scan) is exact on a
  stripe because columns are independent.  The uint16 nearest-row plane of the
  stripe is row-major, so the block destined for rank q -- rows
  [q*H/N, (q+1)*H/N) -- is contiguous: ONE all-to-all over the raw bytes
  (NCCL has no 16-bit integer type) turns column stripes into row stripes.  The
  received buffer holds N column tiles of (H/N x W/N); stage 2 reads them in
  place (``dfc_rows_from_nr_u16`` tile addressing) with global row numbers, so
  no transpose pass exists.  Each rank ends with its row stripe of the result.

The two stages are pluggable (``KernelOps`` on the GPU; the CPU tests pass a
numpy stand-in) so the partition/exchange logic is tested with ``gloo``.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """[lo, hi) of n units owned by rank (contiguous, sizes differ by <= 1)."""
    return (n * rank) // world, (n * (rank + 1)) // world


class KernelOps:
    """The sm_100a kernels through the C ABI."""

    def __init__(self):
        import paper_2106_03503_b200 as dfc
        self.dfc = dfc

    def column_nr(self, stripe: torch.Tensor) -> torch.Tensor:
        """int16 [H, Ws] nearest object rows of a column stripe (uint16 bits)."""
        nr = self.dfc.column_nr(stripe)
        return nr[:, : stripe.shape[1]].contiguous() if nr.shape[1] != stripe.shape[1] else nr

    def rows_from_tiles(self, tiles: torch.Tensor, rows: int, cols: int, row0: int, tile_cols: int):
        return self.dfc.rows_from_nr(tiles, rows, cols, row0=row0, tile_cols=tile_cols,
                                     tile_stride=rows * tile_cols)["sqdist"]

    def batch(self, imgs: torch.Tensor, label: bool = True):
        return self.dfc.edt_batched(imgs, dist=False, label=label)


def edt_batch_sharded(imgs_all, rank: int, world: int, ops=None, device=None):
    """C3: this rank's share of a batch [n, H, W] (host or device tensor).
    Returns (lo, hi, outputs dict for images lo..hi-1)."""
    ops = ops or KernelOps()
    lo, hi = shard_range(imgs_all.shape[0], rank, world)
    local = imgs_all[lo:hi]
    if device is not None:
        local = local.to(device, non_blocking=True)
    return lo, hi, ops.batch(local)


def exchange_column_to_row(nr_stripe: torch.Tensor, H: int, rank: int, world: int, group=None):
    """All-to-all: my column stripe's nearest-row plane [H, Ws] -> my row
    stripe as `world` column tiles [world][Hs, Ws] (tile p = rank p's columns)."""
    Ws = nr_stripe.shape[1]
    assert nr_stripe.is_contiguous() and nr_stripe.shape[0] == H
    rows = [shard_range(H, q, world) for q in range(world)]
    send_sizes = [(r1 - r0) * Ws * 2 for (r0, r1) in rows]  # bytes; blocks are contiguous row ranges
    my0, my1 = rows[rank]
    recv = torch.empty(world * (my1 - my0) * Ws, dtype=torch.int16, device=nr_stripe.device)
    recv_sizes = [(my1 - my0) * Ws * 2] * world
    if world == 1:
        recv.copy_(nr_stripe.reshape(-1))
    else:
        dist.all_to_all_single(recv.view(torch.uint8), nr_stripe.reshape(-1).view(torch.uint8),
                               output_split_sizes=recv_sizes, input_split_sizes=send_sizes, group=group)
    return recv, my0, my1


def edt_column_striped(img_stripe: torch.Tensor, H: int, W: int, rank: int, world: int, ops=None, group=None):
    """C5: exact squared EDT of an H x W image whose column stripe
    [rank*W/N, (rank+1)*W/N) this rank holds (img_stripe: [H, W/N] uint8).
    Returns (row0, row1, sqdist [row1-row0, W]) -- this rank's row stripe."""
    ops = ops or KernelOps()
    if W % world != 0 or (W // world) % 2 != 0:
        raise ValueError("column stripes must be equal and even: W % (2*world) == 0")
    Ws = W // world
    assert img_stripe.shape == (H, Ws)
    nr = ops.column_nr(img_stripe)                      # stage 1 on the stripe
    tiles, r0, r1 = exchange_column_to_row(nr, H, rank, world, group)
    sq = ops.rows_from_tiles(tiles, r1 - r0, W, r0, Ws)  # stage 2 on the row stripe
    return r0, r1, sq

"""Multi-GPU sharding of the distance-transform path.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing.

* C3 (a batch of independent images): rank r owns images
  [r*n/N, (r+1)*n/N); no data-path collective.
* C5 (one giant image, north_star): rank r owns the column stripe
  ``shard_cols(W, N, r)``.  Stage 1 (the per-column nearest-object scan) is
  exact on a stripe because columns are independent.

  - ``compact`` (default, ``StripedEDT``): the library call
    ``dfc_edt_u8_sharded`` -- column pass on the stripe, an NCCL all-to-all of
    the compact band data (per 32-row band and column: object mask, nearest
    object rows above / below the band; 0.25 B/px), the band-path row pass on
    the row stripe ``shard_rows(H, N, r)``.  The communicator is the
    library's own (``dfc_comm_init_rank``; rank 0's unique id is broadcast
    over ``torch.distributed``).
  - ``dense`` (``edt_column_striped_dense``, reported for comparison): the
    uint16 nearest-row plane of the stripe (2 B/px) goes through
    ``all_to_all_single``; stage 2 reads the N received tiles in place
    (``dfc_rows_from_nr_u16``).

``edt_column_striped_compact_py`` is the compact exchange's data flow in
Python over ``torch.distributed`` with pluggable column/row stages -- the
host-side protocol the CPU (gloo) tests check with numpy stand-ins; on the GPU
the same flow runs inside ``dfc_edt_u8_sharded``.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """[lo, hi) of n units owned by rank (contiguous, sizes differ by <= 1)."""
    return (n * rank) // world, (n * (rank + 1)) // world


def band_range(rows: int, rank: int, world: int):
    """[b0, b1) of the 32-row bands of the row stripe of `rank` (dfc_shard_rows)."""
    return shard_range((rows + 31) // 32, rank, world)


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


class StripedEDT:
    """C5 over torch.distributed ranks through ``dfc_edt_u8_sharded`` (compact
    exchange, NCCL inside libdfc).  Build once per (H, W, world); call with
    this rank's column stripe; returns (row0, row1, sqdist of the row stripe)."""

    def __init__(self, H: int, W: int, rank: int, world: int, device=None, group=None, dist_out=False):
        import paper_2106_03503_b200 as dfc
        self.dfc, self.H, self.W, self.rank, self.world = dfc, H, W, rank, world
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.c0, self.c1 = dfc.shard_cols(W, world, rank)
        self.r0, self.r1 = dfc.shard_rows(H, world, rank)
        self.comm = None
        if world > 1:
            uid = torch.zeros(128, dtype=torch.uint8, device=self.device)
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(dfc.comm_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, 0, group=group)
            self.comm = dfc.comm_init_rank(world, rank, bytes(uid.cpu().numpy().tobytes()))
        self.sq = torch.empty((self.r1 - self.r0, W), dtype=torch.int32, device=self.device)
        self.dist = torch.empty_like(self.sq, dtype=torch.float32) if dist_out else None

    def __call__(self, img_stripe: torch.Tensor, polarity: int = 0, stream=None):
        if img_stripe.shape != (self.H, self.c1 - self.c0):
            raise ValueError(f"rank {self.rank} holds columns [{self.c0}, {self.c1}) of all {self.H} rows")
        self.dfc.edt_sharded([{"rank": self.rank, "img": img_stripe, "sqdist": self.sq, "dist": self.dist,
                               "comm": self.comm, "stream": stream}], self.world, self.H, self.W, polarity)
        return self.r0, self.r1, self.sq

    def close(self):
        if self.comm is not None:
            self.dfc.comm_destroy(self.comm)
            self.comm = None


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


def edt_column_striped_dense(img_stripe: torch.Tensor, H: int, W: int, rank: int, world: int, ops=None,
                             group=None):
    """C5, dense exchange: the stripe's uint16 nearest-row plane (2 B/px)
    through all_to_all_single.  img_stripe: [H, W/N] uint8, equal even stripes.
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


def edt_column_striped_compact_py(img_stripe: torch.Tensor, H: int, W: int, rank: int, world: int, ops,
                                  group=None):
    """The compact exchange of dfc_edt_u8_sharded, in Python (tests): `ops`
    provides band_data(stripe) -> (masks [nb, Ws] int64 bit masks, above, below
    [nb, Ws] int64 rows, -1 = none, count) and rows_from_bands(masks, above,
    below, row0, nrows, W, count) -> sqdist of the row stripe.  Column stripes
    from shard_range(W), row stripes from band_range(H); the band slices for
    rank q are contiguous, as in the C implementation."""
    c0, c1 = shard_range(W, rank, world)
    assert img_stripe.shape == (H, c1 - c0)
    masks, above, below, count = ops.band_data(img_stripe)
    nb = (H + 31) // 32
    assert masks.shape == (nb, c1 - c0)
    packed = torch.stack([masks, above, below]).to(torch.int64)  # [3, nb, Ws]
    b_my0, b_my1 = band_range(H, rank, world)
    send = [packed[:, slice(*band_range(H, q, world))].reshape(-1) for q in range(world)]
    widths = [shard_range(W, q, world)[1] - shard_range(W, q, world)[0] for q in range(world)]
    rsz = [3 * (b_my1 - b_my0) * widths[q] for q in range(world)]
    flat = torch.empty(sum(rsz), dtype=torch.int64)
    counts = torch.empty(world, dtype=torch.int64)
    if world == 1:
        flat.copy_(send[0])
        counts.fill_(count)
    else:  # one all_to_all_single per message kind (gloo has no list all_to_all)
        dist.all_to_all_single(flat, torch.cat(send), output_split_sizes=rsz,
                               input_split_sizes=[t.numel() for t in send], group=group)
        dist.all_to_all_single(counts, torch.full((world,), count, dtype=torch.int64), group=group)
    recv = list(torch.split(flat, rsz))
    full = torch.empty((3, b_my1 - b_my0, W), dtype=torch.int64)
    for q in range(world):
        q0, q1 = shard_range(W, q, world)
        full[:, :, q0:q1] = recv[q].view(3, b_my1 - b_my0, q1 - q0)
    r0, r1 = min(H, 32 * b_my0), min(H, 32 * b_my1)
    total = int(counts.sum())
    sq = ops.rows_from_bands(full[0], full[1], full[2], r0, r1 - r0, W, total)
    return r0, r1, sq

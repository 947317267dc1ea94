"""torchrun worker for tests/test_sharding.py (gloo, CPU): runs the sharded
drivers of paper_2106_03503_b200.sharded with numpy stand-ins for the two
kernels and checks the gathered result against the oracle on rank 0.
Test infrastructure only."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), HERE]

import oracle  # noqa: E402


class NumpyOps:
    """CPU stand-ins with the kernels' exact data contracts."""

    def column_nr(self, stripe):
        img = stripe.numpy()
        H, Ws = img.shape
        out = np.full((H, Ws), 0xFFFF, np.uint16)
        ii = np.arange(H)
        for j in range(Ws):
            rows = np.nonzero(img[:, j])[0]
            if rows.size:
                d = np.abs(ii[:, None] - rows[None, :])
                out[:, j] = rows[d.argmin(axis=1)]  # first minimum = upper row on ties
        return torch.from_numpy(out.view(np.int16))

    def rows_from_tiles(self, tiles, rows, cols, row0, tile_cols):
        t = tiles.numpy().view(np.uint16)
        nr = np.empty((rows, cols), np.int64)
        for j in range(cols):
            tt = j // tile_cols
            nr[:, j] = t[tt * rows * tile_cols + np.arange(rows) * tile_cols + (j % tile_cols)]
        gi = row0 + np.arange(rows)[:, None]
        g = np.where(nr == 0xFFFF, np.int64(1) << 40, (gi - nr) ** 2)
        jj = np.arange(cols)
        d = (g[:, None, :] + (jj[:, None] - jj[None, :])[None] ** 2).min(axis=2)
        return torch.from_numpy(np.where(d >= (1 << 40), 0x7FFFFFFF, d).astype(np.int32))

    def batch(self, imgs, label=True):
        sq = np.stack([oracle.to_i32(oracle.edt(im.numpy())) for im in imgs])
        return {"sqdist": torch.from_numpy(sq)}


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2106_03503_b200 import sharded
    ops = NumpyOps()
    ok = True
    # ---- C5-style: column stripes -> all-to-all -> row stripes ----
    for (H, W, dens, seed) in ((37, 24, 0.02, 5), (64, 40, 0.0, 6), (50, 32, 0.3, 7), (33, 16, 0.004, 8)):
        img = oracle.random_image(H, W, dens, seed)
        Ws = W // world
        stripe = torch.from_numpy(np.ascontiguousarray(img[:, rank * Ws:(rank + 1) * Ws]))
        r0, r1, sq = sharded.edt_column_striped(stripe, H, W, rank, world, ops=ops)
        parts = [None] * world
        dist.all_gather_object(parts, (r0, r1, sq.numpy()))
        if rank == 0:
            full = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])])
            want = oracle.to_i32(oracle.edt(img))
            if not (full.shape == want.shape and (full == want).all()):
                print("C5 mismatch", H, W, dens, flush=True)
                ok = False
    # ---- C3-style: per-image shards ----
    import workloads
    imgs = torch.from_numpy(workloads.points_batch(7, 24, 20, 5, 3))
    lo, hi, out = sharded.edt_batch_sharded(imgs, rank, world, ops=ops)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, hi, out["sqdist"].numpy()))
    if rank == 0:
        cover = sorted((p[0], p[1]) for p in parts)
        assert cover[0][0] == 0 and cover[-1][1] == 7 and all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
        for (a, b, sq) in parts:
            for k in range(a, b):
                if not (sq[k - a] == oracle.to_i32(oracle.edt(imgs[k].numpy()))).all():
                    print("C3 mismatch", k, flush=True)
                    ok = False
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

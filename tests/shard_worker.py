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

    # ---- the compact exchange's stage contracts (K1a + K1b; band-path row pass) ----
    def band_data(self, stripe):
        img = stripe.numpy()
        H, Ws = img.shape
        nb = (H + 31) // 32
        masks = np.zeros((nb, Ws), np.int64)
        above = np.full((nb, Ws), -1, np.int64)
        below = np.full((nb, Ws), -1, np.int64)
        for j in range(Ws):
            rows = np.nonzero(img[:, j])[0]
            for b in range(nb):
                inb = rows[(rows >= 32 * b) & (rows < 32 * b + 32)]
                masks[b, j] = int(np.sum(1 << (inb - 32 * b))) if inb.size else 0
                up = rows[rows < 32 * b]
                dn = rows[rows >= 32 * b + 32]
                above[b, j] = up[-1] if up.size else -1
                below[b, j] = dn[0] if dn.size else -1
        return (torch.from_numpy(masks), torch.from_numpy(above), torch.from_numpy(below),
                int(img.astype(bool).sum()))

    def rows_from_bands(self, masks, above, below, row0, nrows, W, count):
        """The row stripe from the band data alone (nearest row per column as
        K1c: in-band bits, else the carries; upper row on ties)."""
        m, a, bl = masks.numpy(), above.numpy(), below.numpy()
        nr = np.full((nrows, W), -1, np.int64)
        for ii in range(nrows):
            i = row0 + ii
            b = i // 32 - row0 // 32
            r = i % 32
            for j in range(W):
                mk = int(m[b, j])
                up = mk & ((2 << r) - 1)
                dn = mk >> r
                ra = 32 * (i // 32) + up.bit_length() - 1 if up else a[b, j]
                rb = i + ((dn & -dn).bit_length() - 1) if dn else bl[b, j]
                if ra < 0:
                    nr[ii, j] = rb
                elif rb < 0:
                    nr[ii, j] = ra
                else:
                    nr[ii, j] = ra if i - ra <= rb - i else rb
        gi = row0 + np.arange(nrows)[:, None]
        g = np.where(nr < 0, np.int64(1) << 40, (gi - nr) ** 2)
        jj = np.arange(W)
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
        r0, r1, sq = sharded.edt_column_striped_dense(stripe, H, W, rank, world, ops=ops)
        parts = [None] * world
        dist.all_gather_object(parts, (r0, r1, sq.numpy()))
        if rank == 0:
            full = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])])
            want = oracle.to_i32(oracle.edt(img))
            if not (full.shape == want.shape and (full == want).all()):
                print("C5 dense mismatch", H, W, dens, flush=True)
                ok = False
    # ---- C5, compact exchange (the data flow of dfc_edt_u8_sharded): band
    # stripes, uneven column stripes, a partial last band ----
    for (H, W, dens, seed) in ((37, 25, 0.02, 5), (100, 31, 0.01, 9), (64, 40, 0.0, 6), (70, 19, 0.3, 7)):
        img = oracle.random_image(H, W, dens, seed)
        c0, c1 = sharded.shard_range(W, rank, world)
        stripe = torch.from_numpy(np.ascontiguousarray(img[:, c0:c1]))
        r0, r1, sq = sharded.edt_column_striped_compact_py(stripe, H, W, rank, world, ops)
        parts = [None] * world
        dist.all_gather_object(parts, (r0, r1, sq.numpy()))
        if rank == 0:
            cover = sorted((p[0], p[1]) for p in parts)
            assert cover[0][0] == 0 and cover[-1][1] == H and all(x[1] == y[0] for x, y in zip(cover, cover[1:]))
            assert all(p[0] % 32 == 0 for p in parts)   # row stripes are whole bands
            full = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])])
            want = oracle.to_i32(oracle.edt(img))
            if not (full.shape == want.shape and (full == want).all()):
                print("C5 compact mismatch", H, W, dens, flush=True)
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

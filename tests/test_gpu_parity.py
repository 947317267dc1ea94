"""GPU parity: the sm_100a path (through the C ABI) against the pinned CPU oracle.

Bit-exact for every integer output (squared distances, labels, nearest
columns, city-block / chessboard / chamfer-3-4); float32 distances must equal
(float)sqrt((double)D) exactly (0 ulp; north_star allows <= 1 ulp).
"""
import json
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def dfc():
    """The device layer with the band path open to every image size, so that
    the small sparse cases below run through it (the library default only
    offers it images above 4096^2; test_small_sparse_default_dispatch covers
    that default)."""
    import paper_2106_03503_b200 as m
    m.set_band_min_pixels(0)
    yield m
    m.set_band_min_pixels(-1)


def _dev(img):
    return torch.from_numpy(np.ascontiguousarray(img)).cuda()


def _check_edt(dfc, img, polarity=0):
    out = dfc.edt(_dev(img), polarity=polarity, dist=True, label=True, nearest_col=True)
    torch.cuda.synchronize()
    src = img if polarity == 0 else (img == 0).astype(np.uint8)
    want = oracle.to_i32(oracle.edt(src))
    got = out["sqdist"].cpu().numpy()
    np.testing.assert_array_equal(got, want)
    # squared distances alone: the row kernels' D-only fills (no owner per column)
    only = dfc.edt(_dev(img), polarity=polarity, dist=False, label=False, nearest_col=False)
    np.testing.assert_array_equal(only["sqdist"].cpu().numpy(), want)
    np.testing.assert_array_equal(out["dist"].cpu().numpy().view(np.uint32),
                                  oracle.sqrt_f32(want).view(np.uint32))
    lab = oracle.voronoi_labels(src, linear=True)
    want_lab = np.full(src.shape, -1, np.int32) if lab is None else lab[1]
    np.testing.assert_array_equal(out["label"].cpu().numpy(), want_lab)
    _, ncol = oracle.meijster_scan(oracle.vertical_pass(src), take_new=True)
    np.testing.assert_array_equal(out["nearest_col"].cpu().numpy(), ncol.view(np.int32))


def test_six_point_golden(dfc):
    with open(os.path.join(GOLD, "six_point.json")) as f:
        g = json.load(f)
    img = np.zeros((g["rows"], g["cols"]), np.uint8)
    for r, c in g["points"]:
        img[r, c] = 1
    out = dfc.edt(_dev(img), label=True)
    r = dfc.raster(_dev(img))
    vert = dfc.vertical(_dev(img))
    torch.cuda.synchronize()
    m = lambda k: np.where(np.array(g[k]) < 0, 0x7FFFFFFF, np.array(g[k])).astype(np.int32)
    np.testing.assert_array_equal(out["sqdist"].cpu().numpy(), m("kSquaredEuclidean"))
    np.testing.assert_array_equal(vert.cpu().numpy(), m("kVerticalFinal"))
    np.testing.assert_array_equal(r["cityblock"].cpu().numpy(), m("kCityblockFinal"))
    np.testing.assert_array_equal(r["chamfer34"].cpu().numpy(), m("kChamferFinal"))
    # test_exact_edt.cpp:238-259: the (0,0) tie resolves to the feature at (4, 1)
    assert int(out["label"][0, 0]) == 4 * g["cols"] + 1


def _cases():
    z = np.load(os.path.join(GOLD, "random_cases.npz"))
    for n in range(int(z["n_cases"][0])):
        yield {k.split("_", 1)[1]: z[k] for k in z.files if k.startswith(f"c{n}_")}


@pytest.mark.parametrize("case", list(_cases()),
                         ids=lambda c: "x".join(map(str, c["meta"][:2])) + f"@{c['density'][0]}")
def test_reference_fixtures(dfc, case):
    """The 60 committed outputs of the reference library itself."""
    img = case["img"]
    d = _dev(img)
    out = dfc.edt(d, label=True, nearest_col=True)
    r = dfc.raster(d)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out["sqdist"].cpu().numpy(), oracle.to_i32(case["edt"]))
    np.testing.assert_array_equal(out["nearest_col"].cpu().numpy(), case["nearest_col"].view(np.int32))
    if case["labels"].size:
        ords = dfc.label_ordinals(d, out["label"]).cpu().numpy()
        np.testing.assert_array_equal(ords, case["labels"].astype(np.int64))
    else:
        assert (out["label"].cpu().numpy() == -1).all()
    np.testing.assert_array_equal(r["cityblock"].cpu().numpy(), oracle.to_i32(case["cityblock"]))
    np.testing.assert_array_equal(r["chamfer34"].cpu().numpy(), oracle.to_i32(case["chamfer34"]))
    np.testing.assert_array_equal(r["chessboard"].cpu().numpy(), oracle.to_i32(case["chessboard"]))


SHAPES = [(1, 1), (1, 2), (2, 1), (1, 100), (100, 1), (7, 33), (33, 7), (64, 64), (31, 97),
          (5, 1000), (3, 1031), (2, 2048), (2, 4096), (3, 4100), (40, 129), (257, 65), (2, 8191),
          (1, 16384), (1, 32768), (70, 600)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("density", [0.0005, 0.01, 0.2, 0.7])
def test_edt_random(dfc, shape, density):
    img = oracle.random_image(shape[0], shape[1], density, 1000 * shape[0] + shape[1] + int(density * 1e4))
    _check_edt(dfc, img, 0)


@pytest.mark.parametrize("shape", [(48, 48), (3, 2000), (129, 300)])
def test_edt_polarity_inside(dfc, shape):
    img = oracle.random_image(shape[0], shape[1], 0.6, 77 + shape[1])
    _check_edt(dfc, img, 1)


def test_edt_degenerate(dfc):
    for img in (np.zeros((5, 7), np.uint8), np.ones((4, 9), np.uint8), np.zeros((1, 1), np.uint8)):
        _check_edt(dfc, img)
    corner = np.zeros((300, 2000), np.uint8)
    corner[299, 1999] = 1
    _check_edt(dfc, corner)
    ties = np.zeros((41, 41), np.uint8)
    for (r, c) in [(0, 0), (0, 40), (40, 0), (40, 40), (20, 20), (10, 30), (30, 10)]:
        ties[r, c] = 1
    _check_edt(dfc, ties)


def test_pitch_and_bool_input(dfc):
    img = oracle.random_image(50, 70, 0.03, 5)
    big = np.zeros((50, 131), np.uint8)
    big[:, 3:73] = img * 9  # nonzero bytes other than 1 are objects too (grid.hpp:82)
    t = _dev(big)[:, 3:73]
    out = dfc.edt(t, dist=False)
    out_b = dfc.edt(_dev(img.astype(bool)), dist=False)
    torch.cuda.synchronize()
    want = oracle.to_i32(oracle.edt(img))
    np.testing.assert_array_equal(out["sqdist"].cpu().numpy(), want)
    np.testing.assert_array_equal(out_b["sqdist"].cpu().numpy(), want)


@pytest.mark.parametrize("shape", [(64, 64), (100, 301), (1, 500), (256, 4096)])
def test_dual_polarity(dfc, shape):
    import workloads
    img = workloads.discs(shape[0], shape[1], 12, 3 + shape[1])
    out = dfc.edt_dual(_dev(img))
    torch.cuda.synchronize()
    w0 = oracle.to_i32(oracle.edt(img))
    w1 = oracle.to_i32(oracle.edt((img == 0).astype(np.uint8)))
    np.testing.assert_array_equal(out["sqdist_bg"].cpu().numpy(), w0)
    np.testing.assert_array_equal(out["sqdist_obj"].cpu().numpy(), w1)
    np.testing.assert_array_equal(out["dist_bg"].cpu().numpy(), oracle.sqrt_f32(w0))
    np.testing.assert_array_equal(out["dist_obj"].cpu().numpy(), oracle.sqrt_f32(w1))


def test_batched_points(dfc):
    import workloads
    imgs = workloads.points_batch(24, 128, 96, 30, 99)
    imgs[5] = 0  # a featureless image inside the batch
    out = dfc.edt_batched(_dev(imgs), dist=True, label=True)
    torch.cuda.synchronize()
    d, s, lab = (out[k].cpu().numpy() for k in ("sqdist", "dist", "label"))
    for b in range(imgs.shape[0]):
        want = oracle.to_i32(oracle.edt(imgs[b]))
        np.testing.assert_array_equal(d[b], want)
        np.testing.assert_array_equal(s[b], oracle.sqrt_f32(want))
        wl = oracle.voronoi_labels(imgs[b], linear=True)
        np.testing.assert_array_equal(lab[b], np.full(imgs[b].shape, -1, np.int32) if wl is None else wl[1])


def test_vertical_pass(dfc):
    for shape, dens in (((70, 90), 0.03), ((1, 50), 0.1), ((300, 7), 0.005), ((97, 1000), 0.001)):
        img = oracle.random_image(*shape, dens, shape[0] + 7)
        got = dfc.vertical(_dev(img))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy(), oracle.to_i32(oracle.vertical_pass(img)))


@pytest.mark.parametrize("shape", [(1, 1), (9, 10), (64, 64), (50, 1500), (3, 5000), (333, 77), (5, 16384),
                                   (3, 17000), (70, 33)])
@pytest.mark.parametrize("density", [0.0, 0.003, 0.05, 0.5, 0.97])
def test_raster_random(dfc, shape, density):
    img = oracle.random_image(shape[0], shape[1], density, 7 * shape[0] + shape[1])
    r = dfc.raster(_dev(img))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(r["cityblock"].cpu().numpy(), oracle.to_i32(oracle.cityblock(img)))
    np.testing.assert_array_equal(r["chamfer34"].cpu().numpy(), oracle.to_i32(oracle.chamfer34(img)))
    np.testing.assert_array_equal(r["chessboard"].cpu().numpy(), oracle.to_i32(oracle.chessboard(img)))


def test_label_ordinals(dfc):
    img = oracle.random_image(80, 120, 0.02, 11)
    out = dfc.edt(_dev(img), label=True, dist=False)
    ords = dfc.label_ordinals(_dev(img), out["label"])
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ords.cpu().numpy(), oracle.voronoi_labels(img).astype(np.int64))


def test_shape_errors(dfc):
    with pytest.raises(dfc.DfcError):
        dfc.edt(torch.zeros((70000, 1), dtype=torch.uint8, device="cuda"))  # more rows than supported
    with pytest.raises(dfc.DfcError):
        dfc.edt(torch.zeros((2, 40000), dtype=torch.uint8, device="cuda"))  # row wider than supported


def test_sqrt_epilogue_exact(dfc):
    """dist_f32 == (float)sqrt((double)D) over the whole int32 range, incl. D >= 2^24."""
    rng = np.random.default_rng(3)
    vals = np.concatenate([np.arange(0, 1 << 16), rng.integers(0, 2**31 - 1, 2_000_000),
                           (np.arange(1, 46341, dtype=np.int64) ** 2), (np.arange(1, 46341, dtype=np.int64) ** 2) - 1,
                           (np.arange(1, 46340, dtype=np.int64) ** 2) + np.arange(1, 46340),
                           np.array([2**24 - 1, 2**24, 2**24 + 1, 2147352578, 0x7FFFFFFE])]).astype(np.int32)
    got = dfc.sqrt_i32(torch.from_numpy(vals).cuda()).cpu().numpy()
    want = np.sqrt(vals.astype(np.float64)).astype(np.float32)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    inf = dfc.sqrt_i32(torch.tensor([0x7FFFFFFF], dtype=torch.int32, device="cuda")).cpu().numpy()
    assert np.isinf(inf[0])


@pytest.mark.parametrize("shape", [(40, 64), (7, 301), (1, 1000)])
def test_envelope_from_vertical_plane(dfc, shape):
    """dfc_envelope_vdist_u16 == meijster_scan(vertical_pass(img)) (take_new) and keep_old D."""
    img = oracle.random_image(*shape, 0.03, shape[1])
    vert = oracle.vertical_pass(img)
    a = np.where(vert == oracle.INF, 0xFFFF, np.sqrt(vert.astype(np.float64)).astype(np.int64)).astype(np.uint16)
    w = shape[1] + (shape[1] & 1)
    plane = np.full((shape[0], w), 0xFFFF, np.uint16)
    plane[:, : shape[1]] = a
    t = torch.from_numpy(plane.view(np.int16)).cuda()[:, : shape[1]]
    out = dfc.envelope_vdist(t, take_new=True, dist=True)
    torch.cuda.synchronize()
    d, ncol = oracle.meijster_scan(vert, take_new=True)
    np.testing.assert_array_equal(out["sqdist"].cpu().numpy(), oracle.to_i32(d))
    np.testing.assert_array_equal(out["nearest_col"].cpu().numpy(), ncol.view(np.int32))
    np.testing.assert_array_equal(out["dist"].cpu().numpy(), oracle.sqrt_f32(oracle.to_i32(d)))


@pytest.mark.parametrize("p", [0.02, 0.002])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_column_striped_path_emulated(dfc, world, p):
    """C5 path on one GPU: every 'rank' runs the real stage-1 kernel on its column
    stripe; the all-to-all is emulated by slicing; the real stage-2 kernel reads
    the N tiles in place with global row numbers (dfc_rows_from_nr_u16).  At
    p = 0.002 the row stripes are sparse planes (< 1/256 object pixels): the
    lane-per-row kernel reads the tiles.  (The dense-exchange variant,
    sharded.edt_column_striped_dense.)"""
    from paper_2106_03503_b200 import sharded
    import workloads
    H, W = (96, 256) if p > 0.01 else (256, 1024)
    img = workloads.sparse_tiles(H, W, tile=32, n_on=6 if p > 0.01 else 64, p=p, seed=11 + world)
    ops = sharded.KernelOps()
    Ws = W // world
    stripes = [ops.column_nr(_dev(np.ascontiguousarray(img[:, r * Ws:(r + 1) * Ws]))) for r in range(world)]
    full = np.zeros((H, W), np.int32)
    for q in range(world):
        r0, r1 = sharded.shard_range(H, q, world)
        tiles = torch.cat([s[r0:r1].reshape(-1) for s in stripes])
        sq = ops.rows_from_tiles(tiles, r1 - r0, W, r0, Ws)
        torch.cuda.synchronize()
        full[r0:r1] = sq.cpu().numpy()
    np.testing.assert_array_equal(full, oracle.to_i32(oracle.edt(img)))


def test_column_nr_plane(dfc):
    img = oracle.random_image(70, 41, 0.05, 9)
    nr = dfc.column_nr(_dev(img)).cpu().numpy().view(np.uint16)[:, :41].astype(np.int64)
    vert = oracle.vertical_pass(img)
    ii = np.arange(70)[:, None]
    got = np.where(nr == 0xFFFF, oracle.INF, ((ii - nr) ** 2).astype(np.uint64))
    np.testing.assert_array_equal(got, vert)
    # labels through the row pass use the same plane: global linear index
    out = dfc.rows_from_nr(dfc.column_nr(_dev(img)), 70, 41, label=True, dist=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out["label"].cpu().numpy(), oracle.voronoi_labels(img, linear=True)[1])


def test_sharded_driver_single_rank(dfc):
    from paper_2106_03503_b200 import sharded
    img = oracle.random_image(64, 128, 0.01, 4)
    r0, r1, sq = sharded.edt_column_striped_dense(_dev(img), 64, 128, 0, 1)
    torch.cuda.synchronize()
    assert (r0, r1) == (0, 64)
    np.testing.assert_array_equal(sq.cpu().numpy(), oracle.to_i32(oracle.edt(img)))


# ---- dfc_edt_u8_sharded: column stripes -> compact band exchange -> row stripes ----

def _sharded_in_process(dfc, img, world, polarity=0, dist=False, label=False):
    """All `world` ranks as shards of ONE call on this GPU, without
    communicators: the exchange is stream-ordered device copies, every other
    step is the library's real multi-GPU path."""
    H, W = img.shape
    shards, outs = [], []
    for r in range(world):
        c0, c1 = dfc.shard_cols(W, world, r)
        r0, r1 = dfc.shard_rows(H, world, r)
        o = {"sqdist": torch.full((r1 - r0, W), -7, dtype=torch.int32, device="cuda")}
        if dist:
            o["dist"] = torch.empty((r1 - r0, W), dtype=torch.float32, device="cuda")
        if label:
            o["label"] = torch.empty((r1 - r0, W), dtype=torch.int32, device="cuda")
        shards.append(dict(rank=r, img=_dev(np.ascontiguousarray(img[:, c0:c1])), comm=None, **o))
        outs.append((r0, r1, o))
    dfc.edt_sharded(shards, world, H, W, polarity)
    torch.cuda.synchronize()
    full = {k: np.zeros((H, W), np.float32 if k == "dist" else np.int32) for k in outs[0][2]}
    for r0, r1, o in outs:
        for k, v in o.items():
            full[k][r0:r1] = v.cpu().numpy()
    return full


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("kind", ["tiles", "bern", "discs", "corner", "empty", "tall"])
def test_sharded_library_in_process(dfc, world, kind):
    import workloads
    if kind == "tall":  # row stripes of several coarse groups of 32 bands, partial last ones
        rng = np.random.default_rng(5 + world)
        img = np.zeros((4200, 203), np.uint8)
        for r in (0, 1023, 1024, 2047, 2048, 2111, 2112, 4199):
            img[r, rng.integers(203)] = 1
        for _ in range(12):
            img[rng.integers(4200), rng.integers(203)] = 1
    elif kind == "tiles":
        img = workloads.sparse_tiles(512, 1024, tile=32, n_on=64, p=0.004, seed=3 + world)
    elif kind == "bern":
        img = oracle.random_image(301, 517, 0.02, 40 + world)   # uneven stripes, partial last band
    elif kind == "discs":
        img = workloads.discs(256, 384, 10, 4)               # a dense plane through the band path
    elif kind == "corner":
        img = np.zeros((200, 333), np.uint8)
        img[199, 0] = 1
    else:
        img = np.zeros((70, 90), np.uint8)
    got = _sharded_in_process(dfc, img, world, dist=True, label=True)
    want = oracle.to_i32(oracle.edt(img))
    np.testing.assert_array_equal(got["sqdist"], want)
    np.testing.assert_array_equal(got["dist"].view(np.uint32), oracle.sqrt_f32(want).view(np.uint32))
    lab = oracle.voronoi_labels(img, linear=True)
    np.testing.assert_array_equal(got["label"], np.full(img.shape, -1, np.int32) if lab is None else lab[1])


def test_sharded_library_inverted_polarity(dfc):
    img = np.ones((256, 300), np.uint8)
    img[[5, 100, 200], [7, 150, 299]] = 0
    got = _sharded_in_process(dfc, img, 4, polarity=1)
    np.testing.assert_array_equal(got["sqdist"], oracle.to_i32(oracle.edt((img == 0).astype(np.uint8))))


def test_sharded_library_nccl_single_rank(dfc):
    """The NCCL exchange itself (grouped send/recv through libnccl) with a
    one-rank communicator -- the one-GPU box cannot host more ranks."""
    from paper_2106_03503_b200 import sharded
    img = oracle.random_image(130, 257, 0.003, 12)
    uid = dfc.comm_unique_id()
    comm = dfc.comm_init_rank(1, 0, uid)
    try:
        sq = torch.empty((130, 257), dtype=torch.int32, device="cuda")
        dfc.edt_sharded([dict(rank=0, img=_dev(img), sqdist=sq, comm=comm)], 1, 130, 257)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(sq.cpu().numpy(), oracle.to_i32(oracle.edt(img)))
    finally:
        dfc.comm_destroy(comm)
    st = sharded.StripedEDT(130, 257, 0, 1)
    r0, r1, sq2 = st(_dev(img))
    torch.cuda.synchronize()
    assert (r0, r1) == (0, 130)
    np.testing.assert_array_equal(sq2.cpu().numpy(), oracle.to_i32(oracle.edt(img)))


def test_sharded_library_argument_errors(dfc):
    img = _dev(np.zeros((64, 64), np.uint8))
    sq = torch.empty((64, 64), dtype=torch.int32, device="cuda")
    with pytest.raises(dfc.DfcError):   # two shards claim rank 0
        dfc.edt_sharded([dict(rank=0, img=img[:, :32], sqdist=sq), dict(rank=0, img=img[:, 32:], sqdist=sq)],
                        2, 64, 64)
    with pytest.raises(dfc.DfcError):   # in-process exchange needs every rank
        dfc.edt_sharded([dict(rank=0, img=img[:, :32], sqdist=sq)], 2, 64, 64)


@pytest.mark.parametrize("gap", [1, 2, 17, 255, 256, 257, 600])
def test_dense_rows_zero_split(dfc, gap):
    """Dense planes (most pixels are objects) with gaps of many lengths, next to
    objects at various vertical distances (non-trivial envelopes in the gaps)."""
    rng = np.random.default_rng(gap)
    H, W = 48, 1024
    img = np.ones((H, W), np.uint8)
    for i in range(H):
        j0 = int(rng.integers(0, W - gap))
        img[i, j0:j0 + gap] = 0
        if i % 3 == 0:
            img[max(0, i - 5):i + 5, j0 + gap // 3: j0 + gap // 2 + 1] = 0
    img[:, :2] = 1
    _check_edt(dfc, img)            # background -> object (dense objects)
    _check_edt(dfc, (img == 0).astype(np.uint8), polarity=1)  # same plane via the inverted polarity


def test_dense_rows_border_gaps_and_ties(dfc):
    img = np.ones((40, 300), np.uint8)
    img[:, :37] = 0        # gap at the left border
    img[:, 250:] = 0       # gap at the right border
    img[10:30, 100:140] = 0
    img[::4, 120] = 1      # vertical ties inside the gap
    _check_edt(dfc, img)
    small = np.ones((6, 200), np.uint8)
    small[2] = 0           # a full-width gap row (no zero at all in the row)
    _check_edt(dfc, small)


@pytest.fixture(params=[0, 32, 96, 2048])
def lr_kernel(dfc, request):
    """The lane-per-row chunk scan (k_rows_lr.cu) at the default chunk width and
    at narrow chunks (many chunks per row: warm-ups and cross-chunk owners)."""
    dfc.set_row_kernel("lr")
    dfc.set_lr_chunk(request.param)
    yield dfc
    dfc.set_lr_chunk(0)
    dfc.set_row_kernel("default")


@pytest.mark.parametrize("shape", [(1, 1), (5, 7), (33, 97), (64, 64), (40, 1031), (70, 600), (3, 4100), (100, 33)])
@pytest.mark.parametrize("density", [0.0, 0.002, 0.02, 0.3, 1.0])
def test_lr_row_kernel(lr_kernel, shape, density):
    """The lane-per-row chunk scan gives the same maps, labels and columns."""
    img = oracle.random_image(shape[0], shape[1], density, 13 * shape[0] + shape[1] + int(density * 1000))
    _check_edt(lr_kernel, img)


def test_lr_overflow_falls_back(lr_kernel):
    """Equal-height parabolas under a far object line keep many entries alive per
    row: rows beyond the ring capacity are recomputed exactly by k_rows."""
    img = np.zeros((300, 257), np.uint8)
    img[0, :] = 1
    img[299, 100] = 1
    _check_edt(lr_kernel, img)
    img2 = np.zeros((200, 512), np.uint8)
    img2[0, ::2] = 1
    _check_edt(lr_kernel, img2)


def test_lr_batched_dual_and_discs(lr_kernel):
    import workloads
    imgs = workloads.points_batch(40, 96, 128, 30, 5)
    out = lr_kernel.edt_batched(_dev(imgs), dist=True, label=True)
    img = workloads.discs(256, 384, 10, 3)
    dual = lr_kernel.edt_dual(_dev(img))
    torch.cuda.synchronize()
    for b in range(0, 40, 7):
        np.testing.assert_array_equal(out["sqdist"][b].cpu().numpy(), oracle.to_i32(oracle.edt(imgs[b])))
        np.testing.assert_array_equal(out["label"][b].cpu().numpy(), oracle.voronoi_labels(imgs[b], linear=True)[1])
    np.testing.assert_array_equal(dual["sqdist_bg"].cpu().numpy(), oracle.to_i32(oracle.edt(img)))
    np.testing.assert_array_equal(dual["sqdist_obj"].cpu().numpy(), oracle.to_i32(oracle.edt((img == 0).astype(np.uint8))))
    _check_edt(lr_kernel, img)
    _check_edt(lr_kernel, img, polarity=1)
    _check_edt(lr_kernel, workloads.discs(512, 1000, 12, 9))


@pytest.fixture
def anc_kernel(dfc):
    """Anchored segments (k_rows_anc.cu) for every non-point, non-sparse row."""
    dfc.set_row_kernel("anc")
    yield dfc
    dfc.set_row_kernel("default")


@pytest.mark.parametrize("shape", [(1, 1), (5, 7), (33, 97), (64, 64), (40, 1031), (70, 600), (3, 4100),
                                   (100, 33), (17, 16384), (9, 2049)])
@pytest.mark.parametrize("density", [0.0, 0.002, 0.02, 0.3, 0.9, 1.0])
def test_anc_row_kernel(anc_kernel, shape, density):
    """Anchored segments give the same maps, labels (keep_old) and nearest columns (take_new)."""
    img = oracle.random_image(shape[0], shape[1], density, 7 * shape[0] + shape[1] + int(density * 1000))
    _check_edt(anc_kernel, img)
    _check_edt(anc_kernel, img, polarity=1)


@pytest.fixture
def merge_kernel(dfc):
    """The previous default: k_rows (merge tree) for the rows anchored segments now take."""
    dfc.set_row_kernel("dense")
    yield dfc
    dfc.set_row_kernel("default")


@pytest.mark.parametrize("shape", [(5, 7), (33, 97), (40, 1031), (3, 4100), (9, 2049)])
@pytest.mark.parametrize("density", [0.0, 0.02, 0.3, 0.9])
def test_merge_row_kernel(merge_kernel, shape, density):
    img = oracle.random_image(shape[0], shape[1], density, 5 * shape[0] + shape[1] + int(density * 1000))
    _check_edt(merge_kernel, img)
    _check_edt(merge_kernel, img, polarity=1)


@pytest.mark.parametrize("shape", [(4, 17000), (33000, 3)])
@pytest.mark.parametrize("density", [0.01, 0.3, 0.9])
def test_default_path_outside_anc_limits(dfc, shape, density):
    """Rows wider than 16384 columns or planes taller than 32768 rows leave the
    anchored-segment kernel and the band staging: dense-row / merge-tree kernels
    and the nearest-row plane take over."""
    img = oracle.random_image(shape[0], shape[1], density, shape[0] + shape[1] + int(100 * density))
    _check_edt(dfc, img)
    _check_edt(dfc, img, polarity=1)


def test_anc_ties_and_long_runs(anc_kernel):
    """Equal-height parabolas (every column a tie candidate), object lines, long
    empty runs and a single far object: anchors on ties, pops to an empty stack."""
    img = np.zeros((300, 257), np.uint8)
    img[0, :] = 1
    img[299, 100] = 1
    _check_edt(anc_kernel, img)
    img2 = np.zeros((200, 512), np.uint8)
    img2[0, ::2] = 1
    img2[199, 1::3] = 1
    _check_edt(anc_kernel, img2)
    img3 = np.zeros((64, 3000), np.uint8)
    img3[10, 2999] = 1
    img3[50, 0] = 1
    _check_edt(anc_kernel, img3)
    img4 = np.zeros((40, 640), np.uint8)
    img4[:, 320] = 1
    img4[::7, 0] = 1
    _check_edt(anc_kernel, img4)


def test_anc_batched_dual_and_discs(anc_kernel):
    import workloads
    imgs = workloads.points_batch(40, 96, 128, 30, 5)
    out = anc_kernel.edt_batched(_dev(imgs), dist=True, label=True)
    img = workloads.discs(256, 384, 10, 3)
    dual = anc_kernel.edt_dual(_dev(img))
    torch.cuda.synchronize()
    for b in range(0, 40, 7):
        np.testing.assert_array_equal(out["sqdist"][b].cpu().numpy(), oracle.to_i32(oracle.edt(imgs[b])))
        np.testing.assert_array_equal(out["label"][b].cpu().numpy(), oracle.voronoi_labels(imgs[b], linear=True)[1])
    np.testing.assert_array_equal(dual["sqdist_bg"].cpu().numpy(), oracle.to_i32(oracle.edt(img)))
    np.testing.assert_array_equal(dual["sqdist_obj"].cpu().numpy(), oracle.to_i32(oracle.edt((img == 0).astype(np.uint8))))
    _check_edt(anc_kernel, workloads.discs(512, 1000, 12, 9))
    _check_edt(anc_kernel, workloads.discs(512, 1000, 12, 9), polarity=1)


def test_vertical_direction_passes(dfc):
    """vertical_down_pass / vertical_up_pass (exact_edt.cpp:74-110) in place over
    arbitrary uint64 maps -- infinities, zeros, squares and arbitrary values,
    odd pitches -- against the oracle; down then up over init_distance_map is
    vertical_pass; the six-point golden pins the down pass alone."""
    rng = np.random.default_rng(5)
    inf = np.uint64(2**64 - 1)
    for r, c in [(1, 1), (1, 7), (9, 1), (37, 53), (256, 300), (1000, 33)]:
        dm = rng.integers(0, 400, size=(r, c)).astype(np.uint64)
        dm[rng.random((r, c)) < 0.5] = inf
        dm[rng.random((r, c)) < 0.05] = 0
        dm[rng.random((r, c)) < 0.01] = np.uint64(2**63 + 5)  # unsigned arithmetic as in the reference
        for fn, ofn in ((dfc.vertical_down_pass, oracle.vertical_down_pass),
                        (dfc.vertical_up_pass, oracle.vertical_up_pass)):
            pitch = c + 3  # a padded device map
            buf = torch.zeros((r, pitch), dtype=torch.int64, device="cuda")
            buf[:, :c] = torch.from_numpy(dm.view(np.int64)).cuda()
            fn(buf[:, :c])
            torch.cuda.synchronize()
            np.testing.assert_array_equal(buf[:, :c].cpu().numpy().view(np.uint64), ofn(dm))
    for t in range(6):
        img = oracle.random_image(20 + 7 * t, 31 + 5 * t, [0.0, 0.01, 0.1][t % 3], 90 + t)
        d = torch.from_numpy(oracle.init_map(img).view(np.int64)).cuda()
        dfc.vertical_down_pass(d)
        dfc.vertical_up_pass(d)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(d.cpu().numpy().view(np.uint64), oracle.vertical_pass(img))
    g = json.load(open(os.path.join(GOLD, "six_point.json")))
    img = np.zeros((g["rows"], g["cols"]), np.uint8)
    for a, b in g["points"]:
        img[a, b] = 1
    d = torch.from_numpy(oracle.init_map(img).view(np.int64)).cuda()
    dfc.vertical_down_pass(d)
    want = np.array(g["kVerticalDown"], dtype=np.int64)
    got = d.cpu().numpy()
    np.testing.assert_array_equal(np.where(want < 0, -1, got), np.where(want < 0, -1, want))
    assert (got[want < 0] == -1).all()


@pytest.mark.parametrize("npts", [0, 1, 2, 26, 27, 28, 29, 30, 31, 64, 200])
def test_point_planes(dfc, npts):
    """Planes with at most 32 object pixels (k_rows_pts: K1a's object list, no
    nearest-row plane): same maps, labels and nearest columns as the oracle, at
    the 32-pixel boundary of the path and beyond it; several points per column
    (vertical ties), corners, and a featureless plane."""
    rng = np.random.default_rng(100 + npts)
    H, W = 96, 160
    img = np.zeros((H, W), np.uint8)
    cols = rng.integers(0, 12, size=npts) * 13 % W  # few distinct columns: many points per column
    rows = rng.integers(0, H, size=npts)
    img[rows, cols] = 1
    if npts >= 2:
        img[0, 0] = img[H - 1, W - 1] = 1
        img[10, 50] = img[20, 50] = 1  # an equidistant pair in one column (upper row wins at row 15)
    _check_edt(dfc, img)
    batch = np.stack([img, np.roll(img, 7, axis=1), np.zeros_like(img), img[::-1].copy()])
    out = dfc.edt_batched(_dev(batch), dist=True, label=True)
    torch.cuda.synchronize()
    for b in range(batch.shape[0]):
        np.testing.assert_array_equal(out["sqdist"][b].cpu().numpy(), oracle.to_i32(oracle.edt(batch[b])))
        lab = oracle.voronoi_labels(batch[b], linear=True)
        want = np.full((H, W), -1, np.int32) if lab is None else lab[1]
        np.testing.assert_array_equal(out["label"][b].cpu().numpy(), want)


def test_point_plane_dual_polarity(dfc):
    """An image with only a few BACKGROUND pixels: its object->background plane is
    a point plane while the other is dense."""
    img = np.ones((64, 200), np.uint8)
    img[5, 7] = img[40, 7] = img[63, 199] = img[20, 100] = 0
    _check_edt(dfc, img, polarity=1)
    dual = dfc.edt_dual(_dev(img))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(dual["sqdist_obj"].cpu().numpy(), oracle.to_i32(oracle.edt((img == 0).astype(np.uint8))))
    np.testing.assert_array_equal(dual["sqdist_bg"].cpu().numpy(), oracle.to_i32(oracle.edt(img)))


@pytest.mark.parametrize("density", [3e-5, 0.002])
def test_tall_wide_single_image(dfc, density):
    """One image taller than 8192 rows and wider than k_rows_anc's 16384 columns
    (a sparse plane: k_rows_lr; a denser one: k_rows_dense / k_rows), objects on
    both sides of the middle row: squared distances (with and without the other
    outputs), float distances and labels as the oracle."""
    img = oracle.random_image(8192, 16416, density, 77 + int(density * 1e6))
    img[:, 5000] = 0
    img[4095:4097, 9000:9100] = 1  # objects on both sides of the half boundary
    out = dfc.edt(_dev(img), dist=True, label=True)
    only = dfc.edt(_dev(img), dist=False)
    torch.cuda.synchronize()
    want = oracle.to_i32(oracle.edt(img))
    np.testing.assert_array_equal(out["sqdist"].cpu().numpy(), want)
    np.testing.assert_array_equal(only["sqdist"].cpu().numpy(), want)
    np.testing.assert_array_equal(out["dist"].cpu().numpy().view(np.uint32), oracle.sqrt_f32(want).view(np.uint32))
    np.testing.assert_array_equal(out["label"].cpu().numpy(), oracle.voronoi_labels(img, linear=True)[1])


@pytest.mark.parametrize("shape", [(288, 200), (300, 77), (1000, 96), (2048, 64)])
def test_band_scan_medium_heights(dfc, shape):
    """9-64 bands of 32 rows (k_band_scan_serial; the chunked k_band_scan measured
    slower there): single images of both polarities and a batch of non-point planes."""
    img = oracle.random_image(shape[0], shape[1], 0.01, shape[0] + 7 * shape[1])
    _check_edt(dfc, img)
    _check_edt(dfc, img, polarity=1)
    imgs = np.stack([oracle.random_image(shape[0], shape[1], 0.02, 100 + s) for s in range(3)])
    out = dfc.edt_batched(_dev(imgs), dist=True, label=True)
    torch.cuda.synchronize()
    for b in range(3):
        np.testing.assert_array_equal(out["sqdist"][b].cpu().numpy(), oracle.to_i32(oracle.edt(imgs[b])))
        np.testing.assert_array_equal(out["label"][b].cpu().numpy(), oracle.voronoi_labels(imgs[b], linear=True)[1])


# ---- the band path for sparse planes (k_rows_band.cu: hull filter, per-row
# stacks with a spilling ring, fill) -- the default for planes with fewer than
# 1/256 object pixels in single images ----

def _sparse(shape, npts, seed):
    rng = np.random.default_rng(seed)
    img = np.zeros(shape, np.uint8)
    img[rng.integers(0, shape[0], npts), rng.integers(0, shape[1], npts)] = 1
    return img


@pytest.mark.parametrize("shape", [(33, 97), (64, 64), (257, 65), (100, 1500), (300, 2000), (1000, 96),
                                   (70, 4100), (129, 5000), (40, 1025), (2, 32768), (600, 3000)])
@pytest.mark.parametrize("npts", [1, 2, 7, 40])
def test_band_sparse_random(dfc, shape, npts):
    img = _sparse(shape, npts, shape[0] * 7 + shape[1] + npts)
    if img.sum() * 256 >= img.size:
        pytest.skip("not a sparse plane")
    _check_edt(dfc, img, 0)


@pytest.mark.parametrize("shape", [(1125, 333), (2080, 97), (4133, 40)])
def test_band_sparse_coarse_group_boundaries(dfc, shape):
    """Several coarse groups of 32 bands with a partial last one (and a partial
    last group and band): objects on the rows either side of the coarse and
    group boundaries, a far corner, and a few random ones -- the hull hierarchy
    (coarse lines, then the groups' lines over coarse survivors + the object
    columns in between)."""
    H, W = shape
    rng = np.random.default_rng(H * 31 + W)
    img = np.zeros(shape, np.uint8)
    for r in (1023, 1024, 1055, 1056, 127, 128, 2047, 2048, 4095, 4096):
        if r < H:
            img[r, rng.integers(W)] = 1
    img[H - 1, 0] = 1
    for _ in range(6):
        img[rng.integers(H), rng.integers(W)] = 1
    assert img.sum() * 256 < img.size
    _check_edt(dfc, img, 0)


def test_band_sparse_full_row_spills(dfc):
    """A full object row: below it every column owns itself, so each row's
    stack holds all 2000 columns (the ring spills to the list and reloads)."""
    img = np.zeros((300, 2000), np.uint8)
    img[150, :] = 1
    _check_edt(dfc, img, 0)
    img2 = np.zeros((600, 1100), np.uint8)
    img2[5, 3:1090:2] = 1    # every other column: ties between neighbours
    img2[590, 0] = 1
    _check_edt(dfc, img2, 0)


def test_band_sparse_ties_lattice_and_corners(dfc):
    img = np.zeros((400, 700), np.uint8)
    img[::37, ::41] = 1      # a lattice: many equidistant owners
    _check_edt(dfc, img, 0)
    c = np.zeros((513, 1500), np.uint8)
    c[0, 0] = c[512, 1499] = c[0, 1499] = 1
    _check_edt(dfc, c, 0)


def test_band_sparse_inverted_polarity(dfc):
    img = np.ones((200, 1300), np.uint8)
    img[_sparse((200, 1300), 9, 3) == 1] = 0   # the object->background plane is sparse
    _check_edt(dfc, img, 1)
    out = dfc.edt_dual(_dev(img))
    torch.cuda.synchronize()
    for key, src in (("bg", img), ("obj", (img == 0).astype(np.uint8))):
        np.testing.assert_array_equal(out["sqdist_" + key].cpu().numpy(), oracle.to_i32(oracle.edt(src)))


@pytest.mark.parametrize("seed", [1, 2])
def test_band_sparse_tiles_scaled(dfc, seed):
    """A C5-like image at 1/16 scale: Bernoulli pixels in a quarter of the tiles."""
    import workloads
    img = workloads.sparse_tiles(2048, 2048, 64, 256, 4e-3, 99 + seed)
    assert img.sum() * 256 < img.size
    _check_edt(dfc, img, 0)


# ---- per-pass entry points: build_row_envelope on arbitrary int64 rows, the
# in-place raster passes (k_passes.cu) ----

def _owners_from_envelope(ks, js, cols):
    own = np.empty(cols, np.int64)
    for t in range(len(ks)):
        own[js[t]:js[t + 1]] = ks[t]
    return own


@pytest.mark.parametrize("take_new", [True, False])
def test_row_owners_arbitrary_rows(dfc, take_new):
    rng = np.random.default_rng(5 + take_new)
    for t in range(120):
        c = int(rng.integers(1, 700))
        lmax = int(rng.integers(2, 3_000_000))
        rows = int(rng.integers(1, 5))
        v = rng.integers(0, lmax + lmax // 20 + 2, (rows, c)).astype(np.int64)
        if t % 3 == 0:
            v[:, 0] = lmax                                    # the sentinel base
        if t % 5 == 0:
            v[:, rng.random(c) < 0.9] = lmax                  # mostly sentinels
        own, val = dfc.row_owners(torch.from_numpy(v).cuda(), lmax, take_new)
        own, val = own.cpu().numpy(), val.cpu().numpy()
        for r in range(rows):
            ks, js = oracle.build_row_envelope(v[r], lmax, take_new)
            want = _owners_from_envelope(ks, js, c)
            np.testing.assert_array_equal(own[r], want)
            jj = np.arange(c)
            np.testing.assert_array_equal(val[r], v[r][want] + (jj - want) ** 2)


@pytest.mark.parametrize("which", range(6))
def test_raster_pass_in_place(dfc, which):
    rng = np.random.default_rng(10 + which)
    for t in range(12):
        r, c = int(rng.integers(1, 300)), int(rng.integers(1, 2500))
        if t % 2:
            dm = oracle.init_map(oracle.random_image(r, c, float(rng.choice([0.0, 0.002, 0.05, 0.5])), t))
        else:
            dm = np.where(rng.random((r, c)) < 0.2, rng.integers(0, 10000, (r, c)),
                          np.iinfo(np.uint64).max).astype(np.uint64)
        g = torch.from_numpy(dm.view(np.int64).copy()).cuda()
        dfc.raster_pass(g, which)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(g.cpu().numpy().view(np.uint64), oracle.raster_pass(dm, which))


def test_raster_passes_compose_to_the_transforms(dfc):
    """forward + backward == cityblock_sequential / chamfer34 (propagation.cpp:90-109)."""
    img = oracle.random_image(130, 517, 0.01, 3)
    for (f, b_, kind) in ((0, 1, "cityblock"), (4, 5, "chamfer34")):
        g = torch.from_numpy(oracle.init_map(img).view(np.int64).copy()).cuda()
        dfc.raster_pass(g, f)
        dfc.raster_pass(g, b_)
        torch.cuda.synchronize()
        want = oracle.cityblock(img) if kind == "cityblock" else oracle.chamfer34(img)
        np.testing.assert_array_equal(g.cpu().numpy().view(np.uint64), want)


def test_small_sparse_default_dispatch(dfc):
    """The library default: a sparse plane of a small image goes to the
    lane-per-row kernel (the band path is only offered images above 4096^2)."""
    dfc.set_band_min_pixels(-1)
    try:
        rng = np.random.default_rng(17)
        for shape in ((300, 2000), (1000, 96), (64, 64)):
            img = np.zeros(shape, np.uint8)
            for _ in range(7):
                img[rng.integers(shape[0]), rng.integers(shape[1])] = 1
            _check_edt(dfc, img)
            _check_edt(dfc, img, polarity=1)
    finally:
        dfc.set_band_min_pixels(0)


def test_two_host_threads_two_streams(dfc):
    """Two host threads driving the same device on their own streams at the
    same time (the helper stream and its events are shared per device: the
    enqueue is serialised by a mutex, the results must not mix)."""
    import threading
    imgs = [_sparse((700, 900), 9, 1), oracle.random_image(300, 500, 0.05, 2)]
    wants = [oracle.to_i32(oracle.edt(i)) for i in imgs]
    errs = []

    def work(k):
        try:
            dfc.set_band_min_pixels(0)  # per thread
            st = torch.cuda.Stream()
            dev = _dev(imgs[k])
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                for _ in range(20):
                    out = dfc.edt(dev, dist=False)
                    st.synchronize()
                    if not (out["sqdist"].cpu().numpy() == wants[k]).all():
                        errs.append(k)
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs


def test_cuda_graph_capture_and_replay(dfc):
    """The calls are capturable (stream-ordered scratch, event fork / join to the
    helper stream, no host synchronisation): a captured dfc.edt replays to the
    same maps, for a sparse plane (band path + helper stream) and a dense one."""
    import workloads
    for img in (workloads.sparse_tiles(1024, 1536, tile=64, n_on=60, p=1e-3, seed=5),
                oracle.random_image(700, 900, 0.05, 3)):
        dev = _dev(img)
        out = {"sqdist": torch.empty(img.shape, dtype=torch.int32, device="cuda"),
               "dist": torch.empty(img.shape, dtype=torch.float32, device="cuda")}
        dfc.edt(dev, dist=True, out=out)  # warm-up: pool, attributes, helper stream
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                dfc.edt(dev, dist=True, out=out)
        torch.cuda.synchronize()
        want = oracle.to_i32(oracle.edt(img))
        for _ in range(3):
            out["sqdist"].zero_()
            out["dist"].zero_()
            g.replay()
            torch.cuda.synchronize()
            np.testing.assert_array_equal(out["sqdist"].cpu().numpy(), want)
            np.testing.assert_array_equal(out["dist"].cpu().numpy().view(np.uint32),
                                          oracle.sqrt_f32(want).view(np.uint32))


def _check_danielsson(dfc, img, first_sweep=False):
    out = dfc.danielsson(_dev(img), first_sweep=first_sweep)
    torch.cuda.synchronize()
    d, dy, dx = oracle.danielsson(img, first_sweep)
    np.testing.assert_array_equal(out["sqdist"].cpu().numpy().view(np.uint64), d)
    np.testing.assert_array_equal(out["dy"].cpu().numpy().view(np.uint32), dy)
    np.testing.assert_array_equal(out["dx"].cpu().numpy().view(np.uint32), dx)


@pytest.mark.parametrize("shape", [(1, 1), (1, 40), (37, 1), (2, 2), (9, 33), (33, 32), (64, 65), (50, 200), (200, 97),
                                   (3, 1000), (130, 130)])
@pytest.mark.parametrize("density", [0.0, 0.004, 0.05, 0.3, 0.9, 1.0])
def test_danielsson_random(dfc, shape, density):
    """vector_dt.cpp:108-124 on the device: squared lengths and both offset
    components bit-exact with the restated (reference-pinned) sweeps, for both
    danielsson and danielsson_first_sweep."""
    img = oracle.random_image(shape[0], shape[1], density, shape[0] * 131 + shape[1] + int(density * 1000))
    _check_danielsson(dfc, img)
    _check_danielsson(dfc, img, first_sweep=True)


def test_danielsson_ties_wide_and_batch(dfc):
    img = np.zeros((90, 120), np.uint8)
    img[::9, ::11] = 1                     # a lattice: equal-length candidates from both sides
    _check_danielsson(dfc, img)
    img2 = np.zeros((40, 7000), np.uint8)  # rows wider than the shared-memory buffers
    img2[20, 10] = img2[3, 6990] = img2[39, 3500] = 1
    _check_danielsson(dfc, img2)
    _check_danielsson(dfc, img2, first_sweep=True)
    batch = np.stack([oracle.random_image(70, 90, p, 9 + k) for k, p in enumerate((0.0, 0.01, 0.2, 0.6, 0.03))])
    out = dfc.danielsson(_dev(batch))
    torch.cuda.synchronize()
    for k in range(batch.shape[0]):
        d, dy, dx = oracle.danielsson(batch[k])
        np.testing.assert_array_equal(out["sqdist"][k].cpu().numpy().view(np.uint64), d)
        np.testing.assert_array_equal(out["dy"][k].cpu().numpy().view(np.uint32), dy)
        np.testing.assert_array_equal(out["dx"][k].cpu().numpy().view(np.uint32), dx)


def test_danielsson_goldens_on_device(dfc):
    """goldens.hpp:144-190 through the CUDA path: the six-point offsets after
    the first sweep and final, and the disrupted-region witness (one wrong
    cell: 170 at (1, 0) with offset (1, 13), exact 169)."""
    import json
    with open(os.path.join(GOLD, "vector_dt.json")) as f:
        g = json.load(f)
    img = np.zeros(g["six_shape"], np.uint8)
    for r, c in g["six_points"]:
        img[r, c] = 1
    for key, fs in (("kOffsetsSweep1", True), ("kOffsetsFinal", False)):
        out = dfc.danielsson(_dev(img), first_sweep=fs)
        want = np.array(g[key], np.int32)
        np.testing.assert_array_equal(out["dy"].cpu().numpy(), want[:, :, 0])
        np.testing.assert_array_equal(out["dx"].cpu().numpy(), want[:, :, 1])
    wit = np.zeros(g["witness_shape"], np.uint8)
    for r, c in g["witness_points"]:
        wit[r, c] = 1
    out = dfc.danielsson(_dev(wit))
    d = out["sqdist"].cpu().numpy().view(np.uint64)
    exact = oracle.edt(wit)
    assert int((d != exact).sum()) == 1
    qi, qj = g["witness_cell"]
    assert d[qi, qj] == 170 and exact[qi, qj] == 169
    assert (int(out["dy"][qi, qj]), int(out["dx"][qi, qj])) == (1, 13)
    for c in g["reference_runs"]:
        im = oracle.random_image(c["rows"], c["cols"], c["density"], c["seed"])
        o = dfc.danielsson(_dev(im), first_sweep=c["first_sweep"])
        np.testing.assert_array_equal(o["sqdist"].cpu().numpy().ravel(), np.array(c["dist"], np.int64))
        np.testing.assert_array_equal(o["dy"].cpu().numpy().ravel(), np.array(c["dy"], np.int32))
        np.testing.assert_array_equal(o["dx"].cpu().numpy().ravel(), np.array(c["dx"], np.int32))

"""Parity at BASELINE.json's full sizes (configs 1-5), on the GPU.

Every config's FULL map is compared bit-exactly: C1, C2, C4 with the C
oracle; all 1024 C3 images (distances and labels) and the whole 1-Gpixel C5
map (distances, labels, float distances) with the reference library itself
(oracle/_ref, all host cores: ~20 s each); the degenerate C5 corner image with
its closed form D(i, j) = i^2 + j^2 over all 2^30 pixels (max 2,147,352,578 --
the int32 bound, SURVEY finding 7).  Plus transpose equivariance
edt(img^T) == edt(img)^T on C5 (test_exact_edt.cpp:197-208).
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dfc():
    import paper_2106_03503_b200 as m
    return m


@pytest.fixture(scope="module")
def wl():
    import workloads
    return workloads


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_c1_full(dfc, wl):
    img = wl.config("c1")
    out = dfc.edt(_dev(img), dist=True, label=True)
    torch.cuda.synchronize()
    want = oracle.to_i32(oracle.edt(img))
    np.testing.assert_array_equal(out["sqdist"].cpu().numpy(), want)
    np.testing.assert_array_equal(out["dist"].cpu().numpy(), oracle.sqrt_f32(want))
    np.testing.assert_array_equal(out["label"].cpu().numpy(), oracle.voronoi_labels(img, linear=True)[1])
    if oracle.ref_available():  # the reference itself, too
        np.testing.assert_array_equal(out["sqdist"].cpu().numpy(), oracle.to_i32(oracle.ref_edt(img)))


def test_c2_full_both_polarities(dfc, wl):
    img = wl.config("c2")
    out = dfc.edt_dual(_dev(img))
    torch.cuda.synchronize()
    for key, src in (("bg", img), ("obj", (img == 0).astype(np.uint8))):
        want = oracle.to_i32(oracle.edt(src))
        np.testing.assert_array_equal(out["sqdist_" + key].cpu().numpy(), want)
        np.testing.assert_array_equal(out["dist_" + key].cpu().numpy(), oracle.sqrt_f32(want))


def _ordinals_to_linear(img, ords):
    """Reference LabelMap ordinals (grid.cpp:29-36: row-major enumeration of
    the object pixels) -> linear indices row * cols + col."""
    objs = np.flatnonzero(img.reshape(-1)).astype(np.int32)
    return objs[ords.reshape(-1)].reshape(img.shape)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_c3_full_batch_vs_reference(dfc, wl):
    """All 1024 images of C3, squared distances AND labels, against the
    reference library itself (edt + voronoi_labels per image, all host cores)."""
    import ctypes as C
    import os
    imgs = wl.config("c3")  # 1024 x 1024^2, computed as one batch
    out = dfc.edt_batched(_dev(imgs), dist=False, label=True)
    torch.cuda.synchronize()
    sq = out["sqdist"].cpu().numpy()
    lab = out["label"].cpu().numpy()
    del out
    n, h, w = imgs.shape
    threads = os.cpu_count() or 1
    for b0 in range(0, n, 128):
        sub = np.ascontiguousarray(imgs[b0:b0 + 128])
        d = np.empty(sub.shape, np.uint64)
        ords = np.empty(sub.shape, np.uint32)
        st = oracle.ref.dfref_edt_labels_batch(sub, sub.shape[0], h, w, threads, d.ctypes.data,
                                               ords.ctypes.data, C.byref(C.c_double(0)))
        assert st == 0
        np.testing.assert_array_equal(sq[b0:b0 + 128], d.astype(np.int32))
        for t in range(sub.shape[0]):
            np.testing.assert_array_equal(lab[b0 + t], _ordinals_to_linear(sub[t], ords[t]))


def test_c4_full(dfc, wl):
    img = wl.config("c4")
    r = dfc.raster(_dev(img))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(r["cityblock"].cpu().numpy(), oracle.to_i32(oracle.cityblock(img)))
    np.testing.assert_array_equal(r["chamfer34"].cpu().numpy(), oracle.to_i32(oracle.chamfer34(img)))
    np.testing.assert_array_equal(r["chessboard"].cpu().numpy(), oracle.to_i32(oracle.chessboard(img)))


def test_c5_degenerate_corner_closed_form(dfc, wl):
    img = wl.config("c5d")
    out = dfc.edt(_dev(img), dist=False)
    d = out["sqdist"]
    i = torch.arange(32768, device="cuda", dtype=torch.int64)
    want = (i[:, None] ** 2 + i[None, :] ** 2).to(torch.int32)
    assert bool((d == want).all())
    assert int(d.max()) == 2147352578


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_c5_full_map_vs_reference(dfc, wl):
    """The whole 32768^2 C5 map (the bench workload, squared distances only)
    against the reference library's edt on all host cores, bit for bit; then
    the labels and float distances of the same image against the reference's
    voronoi_labels and (float)sqrt((double)D)."""
    import os
    img = wl.config("c5")
    assert 20000 < int(img.sum()) < 35000
    dev = _dev(img)
    sq = dfc.edt(dev, dist=False)["sqdist"].cpu().numpy()
    threads = os.cpu_count() or 1
    ref = oracle.ref_edt(img, threads=threads)
    for r0 in range(0, 32768, 4096):  # chunked: the uint64 map is 8 GiB
        np.testing.assert_array_equal(sq[r0:r0 + 4096], ref[r0:r0 + 4096].astype(np.int32))
    assert int(sq.max()) == int(ref.max())
    del ref
    full = dfc.edt(dev, dist=True, label=True)
    np.testing.assert_array_equal(full["sqdist"].cpu().numpy(), sq)
    s = full["dist"].cpu().numpy()
    for r0 in range(0, 32768, 4096):
        np.testing.assert_array_equal(s[r0:r0 + 4096], oracle.sqrt_f32(sq[r0:r0 + 4096]))
    del s
    lab = full["label"].cpu().numpy()
    del full
    ords = oracle.ref_voronoi_labels(img, threads=threads)
    np.testing.assert_array_equal(lab, _ordinals_to_linear(img, ords))
    del ords, lab
    # transpose equivariance on the full image (test_exact_edt.cpp:197-208)
    dt = dfc.edt(dev.t().contiguous(), dist=False)["sqdist"]
    d0 = dfc.edt(dev, dist=False)["sqdist"]
    assert bool((dt == d0.t()).all())


def test_dual_polarity_above_the_band_gate(dfc, wl):
    """Both polarities of one sparse image above the band path's size gate
    (4100 x 4200 > 2^24 pixels): the background->object plane takes the band
    path on the caller's stream while the object->background plane (nearly
    all object pixels) runs k_rows_anc on the helper stream at the same time."""
    img = wl.sparse_tiles(4100, 4200, tile=128, n_on=300, p=3e-4, seed=12)
    assert img.sum() * 256 < img.size
    out = dfc.edt_dual(_dev(img))
    torch.cuda.synchronize()
    ref = oracle.ref_edt if oracle.ref_available() else oracle.edt
    for key, src in (("bg", img), ("obj", (img == 0).astype(np.uint8))):
        want = oracle.to_i32(ref(src))
        np.testing.assert_array_equal(out["sqdist_" + key].cpu().numpy(), want)
        np.testing.assert_array_equal(out["dist_" + key].cpu().numpy().view(np.uint32),
                                      oracle.sqrt_f32(want).view(np.uint32))

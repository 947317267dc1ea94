"""The CLI epilogue kernels (k_render.cu) through the Python mirror of the C ABI,
against numpy restatements of netpbm.cpp:81-95 and grid.cpp:93-121 and the
reference itself (oracle/_ref)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dfc():
    import paper_2106_03503_b200 as m
    return m


def _lround(x):  # lround: half away from zero (x >= 0 here)
    return np.floor(np.asarray(x, np.float64) + 0.5).astype(np.int64)


@pytest.mark.parametrize("shape", [(1, 1), (3, 7), (5, 8), (4, 9), (17, 33), (64, 128), (9, 1000)])
@pytest.mark.parametrize("invert", [False, True])
def test_unpack_pbm(dfc, shape, invert):
    rng = np.random.default_rng(shape[0] * 131 + shape[1])
    img = (rng.random(shape) < 0.3).astype(np.uint8)
    packed = np.packbits(img, axis=1)  # MSB first, rows padded to whole bytes
    got = dfc.unpack_pbm(torch.from_numpy(packed.reshape(-1)).cuda(), shape[0], shape[1], invert=invert)
    want = (img == 0).astype(np.uint8) if invert else img
    np.testing.assert_array_equal(got.cpu().numpy(), want)


def test_unpack_pbm_ignores_padding_bits(dfc):
    packed = np.full((3, 2), 0xFF, np.uint8)  # 10 columns: 6 padding bits set
    got = dfc.unpack_pbm(torch.from_numpy(packed.reshape(-1)).cuda(), 3, 10)
    np.testing.assert_array_equal(got.cpu().numpy(), np.ones((3, 10), np.uint8))


def test_binarize_and_count(dfc):
    rng = np.random.default_rng(2)
    img = rng.integers(0, 4, (37, 91)).astype(np.uint8)
    t = torch.from_numpy(img).cuda()
    np.testing.assert_array_equal(dfc.binarize(t).cpu().numpy(), (img != 0).astype(np.uint8))
    np.testing.assert_array_equal(dfc.binarize(t, invert=True).cpu().numpy(), (img == 0).astype(np.uint8))
    assert int(dfc.count_objects(t).item()) == int((img != 0).sum())
    assert int(dfc.count_objects(torch.zeros((3, 3), dtype=torch.uint8, device="cuda")).item()) == 0


@pytest.mark.parametrize("sqrt_mode", [False, True])
def test_gray_matches_restatement_and_reference(dfc, sqrt_mode):
    img = oracle.random_image(70, 90, 0.01, 5)
    d = torch.from_numpy(oracle.to_i32(oracle.edt(img))).cuda()
    g, mx = dfc.gray(d, sqrt_mode=sqrt_mode)
    dd = d.cpu().numpy().astype(np.float64)
    m = dd.max()
    want = _lround(255.0 * (np.sqrt(dd) if sqrt_mode else dd) / (np.sqrt(m) if sqrt_mode else m))
    np.testing.assert_array_equal(g.cpu().numpy(), want.astype(np.uint8))
    assert int(mx.item()) == int(m)
    if oracle.ref is not None:
        np.testing.assert_array_equal(g.cpu().numpy(), oracle.ref_transform_gray(img, 0, sqrt_mode))


def test_gray_edge_cases(dfc):
    zeros = torch.zeros((4, 5), dtype=torch.int32, device="cuda")
    g, mx = dfc.gray(zeros)
    assert int(mx.item()) == 0 and int(g.sum().item()) == 0          # max == 0: all zeros
    inf = torch.full((4, 5), 0x7FFFFFFF, dtype=torch.int32, device="cuda")
    _, mx = dfc.gray(inf)
    assert int(mx.item()) == -1                                       # no finite value


def test_labels_gray(dfc):
    img = oracle.random_image(50, 61, 0.02, 8)
    lab = torch.from_numpy(oracle.voronoi_labels(img).astype(np.int64)).cuda()
    n = int(img.sum())
    got = dfc.labels_gray(lab, n).cpu().numpy()
    want = _lround(255.0 * oracle.voronoi_labels(img).astype(np.float64) / n)
    np.testing.assert_array_equal(got, want.astype(np.uint8))
    if oracle.ref is not None:
        np.testing.assert_array_equal(got, oracle.ref_labels_render(img)[0])

"""Pin the CPU oracle (oracle/dt_oracle.c) before trusting it.

Checks, all on CPU:
  * every golden matrix of proj/tests/goldens.hpp (tests/golden/six_point.json);
  * the reference library's own outputs on 60 committed seeded cases
    (tests/golden/random_cases.npz, made by tests/golden/make_golden.py);
  * the live reference build (oracle/_ref) on fresh seeds, when present;
  * the brute-force oracles of proj/tests/oracles.hpp;
  * the separable closed forms and tie rules the CUDA kernels rely on
    (SURVEY.md findings 4-6).
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
INF = oracle.INF


def _gold():
    with open(os.path.join(GOLD, "six_point.json")) as f:
        return json.load(f)


def _six_point_image(g):
    img = np.zeros((g["rows"], g["cols"]), np.uint8)
    for r, c in g["points"]:
        img[r, c] = 1
    return img


def _as_ref(mat):
    m = np.array(mat, dtype=np.int64)
    out = m.astype(np.uint64)
    out[m < 0] = INF
    return out


def _cases():
    z = np.load(os.path.join(GOLD, "random_cases.npz"))
    for n in range(int(z["n_cases"][0])):
        yield {k.split("_", 1)[1]: z[k] for k in z.files if k.startswith(f"c{n}_")}


# ------------------------------------------------------------------ goldens.hpp
def test_six_point_goldens():
    g = _gold()
    img = _six_point_image(g)
    dm = np.empty(img.shape, np.uint64)
    oracle.orc.orc_init_map(img, *img.shape, dm)
    oracle.orc.orc_vertical_down_pass(dm, *img.shape)
    assert (dm == _as_ref(g["kVerticalDown"])).all()
    oracle.orc.orc_vertical_up_pass(dm, *img.shape)
    assert (dm == _as_ref(g["kVerticalFinal"])).all()
    assert (oracle.vertical_pass(img) == _as_ref(g["kVerticalFinal"])).all()
    assert (oracle.edt(img) == _as_ref(g["kSquaredEuclidean"])).all()
    assert (oracle.cityblock(img) == _as_ref(g["kCityblockFinal"])).all()
    assert (oracle.chamfer34(img) == _as_ref(g["kChamferFinal"])).all()
    ks, js = oracle.row_envelope(oracle.vertical_pass(img)[0], img.shape[0], take_new=True)
    assert ks.tolist() == g["kRow0Ks"] and js.tolist() == g["kRow0Js"]
    assert oracle.edt(img)[0].tolist() == g["kRow0Distances"]


def test_six_point_label_tie():
    """test_exact_edt.cpp:238-259: (0,0) ties between columns 1 and 4 -> feature (4,1)."""
    img = _six_point_image(_gold())
    lab, lin = oracle.voronoi_labels(img, linear=True)
    assert lin[0, 0] == 4 * 10 + 1
    assert lab[0, 0] == 3  # ordinal of (4,1) in row-major order


# --------------------------------------------------------- reference fixtures
@pytest.mark.parametrize("case", list(_cases()), ids=lambda c: "x".join(map(str, c["meta"][:2])) + f"@{c['density'][0]}")
def test_oracle_matches_reference_fixtures(case):
    img = case["img"]
    assert (oracle.edt(img) == case["edt"]).all()
    d, ncol = oracle.meijster_scan(oracle.vertical_pass(img), take_new=True)
    assert (d == case["edt"]).all()
    assert (ncol == case["nearest_col"]).all()
    lab = oracle.voronoi_labels(img)
    if case["labels"].size == 0:
        assert lab is None
    else:
        assert (lab == case["labels"]).all()
    assert (oracle.cityblock(img) == case["cityblock"]).all()
    assert (oracle.chamfer34(img) == case["chamfer34"]).all()
    assert (oracle.chessboard(img) == case["chessboard"]).all()
    # the reference generator is reproduced byte for byte
    r, c, s = (int(x) for x in case["meta"])
    assert (oracle.random_image(r, c, float(case["density"][0]), s) == img).all()


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference():
    rng = np.random.default_rng(5)
    for t in range(40):
        r, c = int(rng.integers(1, 90)), int(rng.integers(1, 90))
        dens = [0.002, 0.03, 0.3][t % 3]
        img = oracle.ref_random_image(r, c, dens, 100 + t)
        assert (oracle.edt(img) == oracle.ref_edt(img)).all()
        assert (oracle.vertical_pass(img) == oracle.ref_vertical_pass(img)).all()
        lab = oracle.voronoi_labels(img)
        rl = oracle.ref_voronoi_labels(img)
        assert (lab is None) == (rl is None)
        if lab is not None:
            assert (lab == rl).all()
        assert (oracle.cityblock(img) == oracle.ref_propagation(img, 0)).all()
        assert (oracle.chamfer34(img) == oracle.ref_propagation(img, 2)).all()
        for row in range(0, r, max(1, r // 4)):
            ks, js = oracle.row_envelope(oracle.vertical_pass(img)[row], r, take_new=True)
            rks, rjs = oracle.ref_row_envelope(img, row)
            assert (ks == rks).all() and (js == rjs).all()


# ------------------------------------------------------ brute-force oracles
def test_oracle_matches_bruteforce():
    for t in range(30):
        img = oracle.random_image(1 + t % 23, 1 + (7 * t) % 31, [0.01, 0.1, 0.5][t % 3], 900 + t)
        assert (oracle.edt(img) == oracle.brute(img, 3)).all()
        assert (oracle.cityblock(img) == oracle.brute(img, 0)).all()
        assert (oracle.chessboard(img) == oracle.brute(img, 1)).all()


# ------------------------------------- separable forms + tie rules
def _a_cols(img):
    """Vertical pixel distance to the nearest object in the same column (INF=big)."""
    r, c = img.shape
    big = 1 << 40
    a = np.full((r, c), big, np.int64)
    for j in range(c):
        rows = np.nonzero(img[:, j])[0]
        if rows.size:
            a[:, j] = np.abs(np.arange(r)[:, None] - rows[None, :]).min(axis=1)
    return a, big


def test_separable_closed_forms():
    for t in range(25):
        img = oracle.random_image(2 + t % 30, 2 + (5 * t) % 37, [0.01, 0.05, 0.3][t % 3], 300 + t)
        if not img.any():
            continue
        a, big = _a_cols(img)
        r, c = img.shape
        h = np.abs(np.arange(c)[:, None] - np.arange(c)[None, :])  # [j, k]
        A = a[:, None, :]  # [i, 1, k]
        H = h[None, :, :]
        mx, mn = np.maximum(A, H), np.minimum(A, H)
        valid = A < big
        l1 = np.where(valid, A + H, big).min(axis=2)
        linf = np.where(valid, mx, big).min(axis=2)
        ch = np.where(valid, 3 * mx + mn, big).min(axis=2)
        assert (l1 == oracle.cityblock(img).astype(np.int64)).all()
        assert (linf == oracle.chessboard(img).astype(np.int64)).all()
        assert (ch == oracle.chamfer34(img).astype(np.int64)).all()


def test_raster_argmin_monotone():
    """The smallest minimising column of min_k max(a_k,|j-k|) (chessboard) and of
    min_k 3 max + min (chamfer-3-4) is non-decreasing along a row: the divide and
    conquer of k_raster.cu relies on it (SURVEY finding 5)."""
    for t in range(40):
        img = oracle.random_image(3 + t % 25, 3 + (7 * t) % 60, [0.005, 0.02, 0.08, 0.3][t % 4], 700 + t)
        if not img.any():
            continue
        a, big = _a_cols(img)
        r, c = img.shape
        h = np.abs(np.arange(c)[:, None] - np.arange(c)[None, :])  # [j, k]
        A = a[:, None, :]
        H = h[None, :, :]
        mx, mn = np.maximum(A, H), np.minimum(A, H)
        valid = A < big
        for f in (mx, 3 * mx + mn):
            v = np.where(valid, f, 4 * big)
            kstar = v.argmin(axis=2)  # numpy argmin = smallest minimiser
            assert (np.diff(kstar, axis=1) >= 0).all()


def test_raster_argmin_monotone_synthetic():
    """Same property on arbitrary vertical-distance rows (many ties, empty columns),
    smallest and largest minimiser alike: k_raster_anc.cu brackets every segment's
    minimisers by the owners at its two ends."""
    rng = np.random.default_rng(5)
    for _ in range(3000):
        W = int(rng.integers(2, 120))
        a = rng.integers(0, int(rng.choice([2, 5, 20, 100])), W).astype(np.int64)
        none = rng.random(W) < rng.choice([0.0, 0.3, 0.8])
        if none.all():
            continue
        h = np.abs(np.arange(W)[:, None] - np.arange(W)[None, :])
        A = np.broadcast_to(a[None, :], h.shape)
        mx, mn = np.maximum(A, h), np.minimum(A, h)
        for f in (mx, 3 * mx + mn):
            v = np.where(np.broadcast_to(none[None, :], h.shape), 1 << 40, f)
            hit = v == v.min(axis=1, keepdims=True)
            lo, hi = hit.argmax(axis=1), W - 1 - hit[:, ::-1].argmax(axis=1)
            assert (np.diff(lo) >= 0).all() and (np.diff(hi) >= 0).all()


def test_label_tie_rule_min_column_then_min_row():
    """voronoi_labels = (smallest minimizing column, then upper row); nearest_col =
    largest minimizing column (SURVEY finding 4)."""
    for t in range(60):
        img = oracle.random_image(3 + t % 20, 3 + (3 * t) % 25, [0.02, 0.08, 0.3][t % 3], 500 + t)
        if not img.any():
            continue
        fr, fc = np.nonzero(img)
        r, c = img.shape
        ii, jj = np.meshgrid(np.arange(r), np.arange(c), indexing="ij")
        d = (ii[..., None] - fr) ** 2 + (jj[..., None] - fc) ** 2
        best = d.min(axis=2)
        key = np.where(d == best[..., None], fc * 100000 + fr, 1 << 60)
        win = key.argmin(axis=2)
        want_lin = fr[win] * c + fc[win]
        _, lin = oracle.voronoi_labels(img, linear=True)
        assert (lin == want_lin).all()
        colmax = np.where(d == best[..., None], fc, -1).max(axis=2)
        _, ncol = oracle.meijster_scan(oracle.vertical_pass(img), take_new=True)
        assert (ncol.astype(np.int64) == colmax).all()


def test_oracle_per_pass_raster_functions_match_reference():
    """orc_raster_pass (propagation.cpp:16-88 restated) == the reference's own
    per-pass functions, on init maps and arbitrary maps."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(0)
    for t in range(150):
        r, c = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        if t % 2:
            dm = oracle.init_map(oracle.random_image(r, c, 0.1, t))
        else:
            dm = np.where(rng.random((r, c)) < 0.3, rng.integers(0, 50, (r, c)),
                          np.iinfo(np.uint64).max).astype(np.uint64)
        for p in range(6):
            np.testing.assert_array_equal(oracle.raster_pass(dm, p), oracle.ref_raster_pass(dm, p))


def test_oracle_build_row_envelope_matches_reference_on_arbitrary_rows():
    """build_row_envelope on int64 rows that are not vertical-pass rows
    (non-squares, values at / above the sentinel, a sentinel base)."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(1)
    for t in range(400):
        c = int(rng.integers(1, 60))
        lmax = int(rng.integers(2, 2000))
        v = rng.integers(0, lmax + 40, c).astype(np.int64)
        if t % 3 == 0:
            v[0] = lmax
        for tn in (True, False):
            a = oracle.build_row_envelope(v, lmax, tn)
            b = oracle.ref_build_row_envelope(v, lmax, tn)
            assert a[0].tolist() == b[0].tolist() and a[1].tolist() == b[1].tolist()


# ---- Danielsson vector transform (vector_dt.cpp) ----
def _vec_gold():
    import json
    with open(os.path.join(os.path.dirname(__file__), "golden", "vector_dt.json")) as f:
        return json.load(f)


def _points_image(shape, points):
    img = np.zeros(shape, np.uint8)
    for r, c in points:
        img[r, c] = 1
    return img


def test_danielsson_goldens():
    """The reference's frozen matrices (goldens.hpp:144-190): offsets after the
    downward sweep and final offsets on the six-point sample; the
    disrupted-region witness: exactly one wrong cell, 170 = 1^2 + 13^2 against
    the exact 169 (test_vector_dt.cpp:23-55)."""
    g = _vec_gold()
    img = _points_image(g["six_shape"], g["six_points"])
    for key, fs in (("kOffsetsSweep1", True), ("kOffsetsFinal", False)):
        d, dy, dx = oracle.danielsson(img, fs)
        want = np.array(g[key], np.int64)
        np.testing.assert_array_equal(dy.astype(np.int32).astype(np.int64), want[:, :, 0])
        np.testing.assert_array_equal(dx.astype(np.int32).astype(np.int64), want[:, :, 1])
    d, _, _ = oracle.danielsson(img)
    np.testing.assert_array_equal(d, oracle.edt(img))  # exact on this input
    wit = _points_image(g["witness_shape"], g["witness_points"])
    d, dy, dx = oracle.danielsson(wit)
    exact = oracle.edt(wit)
    assert int((d != exact).sum()) == 1
    qi, qj = g["witness_cell"]
    assert d[qi, qj] == 170 and exact[qi, qj] == 169 and (dy[qi, qj], dx[qi, qj]) == (1, 13)


def test_danielsson_reference_runs_and_properties():
    """The restatement against outputs of the reference itself (committed),
    plus the reference's own properties: value = dy^2 + dx^2 wherever set, an
    upper bound of the exact transform (test_vector_dt.cpp:57-92)."""
    for c in _vec_gold()["reference_runs"]:
        img = oracle.random_image(c["rows"], c["cols"], c["density"], c["seed"])
        d, dy, dx = oracle.danielsson(img, c["first_sweep"])
        np.testing.assert_array_equal(d.view(np.int64).ravel(), np.array(c["dist"], np.int64))
        np.testing.assert_array_equal(dy.view(np.int32).ravel(), np.array(c["dy"], np.int32))
        np.testing.assert_array_equal(dx.view(np.int32).ravel(), np.array(c["dx"], np.int32))
        if not c["first_sweep"]:
            exact = oracle.edt(img)
            setm = dy != 0xFFFFFFFF
            assert ((d == np.iinfo(np.uint64).max) == ~setm).all()
            assert (d[setm] == dy[setm].astype(np.uint64) ** 2 + dx[setm].astype(np.uint64) ** 2).all()
            assert (d >= exact).all()
    if oracle.ref_available():
        rng = np.random.default_rng(4)
        for _ in range(40):
            img = (rng.random((int(rng.integers(1, 50)), int(rng.integers(1, 50)))) < 0.07).astype(np.uint8)
            for fs in (False, True):
                for a, b in zip(oracle.danielsson(img, fs), oracle.ref_danielsson(img, fs)):
                    np.testing.assert_array_equal(a, b)

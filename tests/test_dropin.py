"""The C++ drop-in library (namespace distfield, reference-compatible headers)
driven end to end through lib/dropin_cli, against the oracle and the goldens."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2106_03503_b200", "lib", "dropin_cli")
INF = oracle.INF


def run(op, img, *extra, nout=1, dtype=np.uint64):
    r, c = img.shape
    with tempfile.TemporaryDirectory() as d:
        fi, fo = os.path.join(d, "in"), os.path.join(d, "out")
        np.ascontiguousarray(img, img.dtype if img.dtype in (np.int64, np.uint64) else np.uint8).tofile(fi)
        p = subprocess.run([CLI, op, str(r), str(c), fi, fo, *map(str, extra)], capture_output=True, text=True,
                           timeout=120)
        if p.returncode == 3:
            return p.stdout.strip()
        assert p.returncode == 0, p.stderr
        return np.fromfile(fo, dtype=dtype)


def test_six_point_goldens():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "six_point.json")))
    img = np.zeros((g["rows"], g["cols"]), np.uint8)
    for a, b in g["points"]:
        img[a, b] = 1
    def ref(k):
        arr = np.array(g[k], dtype=np.int64)
        out = arr.astype(np.uint64)
        out[arr < 0] = INF
        return out.ravel()
    assert (run("edt", img) == ref("kSquaredEuclidean")).all()
    assert (run("edt_simple", img) == ref("kSquaredEuclidean")).all()
    assert (run("vertical", img) == ref("kVerticalFinal")).all()
    assert (run("vertical_down", img) == ref("kVerticalDown")).all()
    assert (run("vertical_both", img) == ref("kVerticalFinal")).all()
    want_up = oracle.vertical_up_pass(oracle.init_map(img)).ravel()
    assert (run("vertical_up", img) == want_up).all()
    assert (run("cityblock", img) == ref("kCityblockFinal")).all()
    assert (run("chamfer", img) == ref("kChamferFinal")).all()
    v = run("rowenv", img, 0, dtype=np.int64)
    n = int(v[0])
    assert v[1:1 + n].tolist() == g["kRow0Ks"] and v[1 + n:].tolist() == g["kRow0Js"]
    lab = run("labels", img, dtype=np.uint32).reshape(img.shape)
    assert lab[0, 0] == 3  # test_exact_edt.cpp:238-259: tie -> feature (4, 1)


@pytest.mark.parametrize("shape,dens", [((48, 48), 0.02), ((33, 97), 0.1), ((1, 300), 0.01), ((200, 3), 0.05),
                                        ((64, 1200), 0.003)])
def test_dropin_matches_oracle(shape, dens):
    img = oracle.random_image(*shape, dens, shape[0] * 7 + shape[1])
    np.testing.assert_array_equal(run("edt", img), oracle.edt(img).ravel())
    np.testing.assert_array_equal(run("vertical", img), oracle.vertical_pass(img).ravel())
    m = run("meijster", img, dtype=np.uint8)
    npx = img.size
    d, ncol = oracle.meijster_scan(oracle.vertical_pass(img), take_new=True)
    np.testing.assert_array_equal(m[: 8 * npx].view(np.uint64), d.ravel())
    np.testing.assert_array_equal(m[8 * npx:].view(np.uint32), ncol.ravel())
    lab = run("labels", img, dtype=np.uint32)
    want = oracle.voronoi_labels(img)
    if want is None:
        assert lab.startswith("EXC domain_error")
    else:
        np.testing.assert_array_equal(lab, want.ravel())
    for op, fn in (("cityblock", oracle.cityblock), ("chamfer", oracle.chamfer34), ("chessboard", oracle.chessboard)):
        np.testing.assert_array_equal(run(op, img), fn(img).ravel())
    both = run("both", img)
    np.testing.assert_array_equal(both[:npx], oracle.edt(img).ravel())
    np.testing.assert_array_equal(both[npx:], oracle.edt((img == 0).astype(np.uint8)).ravel())
    for row in range(0, shape[0], max(1, shape[0] // 3)):
        v = run("rowenv", img, row, dtype=np.int64)
        n = int(v[0])
        ks, js = oracle.row_envelope(oracle.vertical_pass(img)[row], shape[0], take_new=True)
        assert v[1:1 + n].tolist() == ks.tolist() and v[1 + n:].tolist() == js.tolist()


def test_dropin_errors_and_degenerate():
    assert run("labels", np.zeros((3, 3), np.uint8)).startswith("EXC domain_error")  # exact_edt.cpp:321
    assert (run("edt", np.zeros((5, 7), np.uint8)) == INF).all()                     # test_exact_edt.cpp:223
    assert (run("cityblock", np.zeros((4, 5), np.uint8)) == INF).all()                # test_propagation.cpp:73
    assert run("edt", np.zeros((2, 40000), np.uint8)).startswith("EXC length_error")  # beyond the GPU row limit


def test_dropin_generator_parity():
    """generate_random_image of the drop-in is byte-identical to the reference generator."""
    for (r, c, dens, seed) in ((17, 23, 0.05, 1234), (64, 64, 0.5, 0), (3, 300, 0.001, 99)):
        out = run("random", np.zeros((r, c), np.uint8), dens, seed, dtype=np.uint8)
        np.testing.assert_array_equal(out, oracle.random_image(r, c, dens, seed).ravel())


def test_dropin_build_row_envelope_and_passes():
    """build_row_envelope (exact_edt.hpp:71-72) on arbitrary int64 rows, the
    per-pass raster functions (propagation.hpp:15-26) and meijster_scan on a
    map that is not a vertical-pass map, through the drop-in."""
    rng = np.random.default_rng(3)
    for t in range(40):
        c = int(rng.integers(1, 300))
        lmax = int(rng.integers(2, 100000))
        v = rng.integers(0, lmax + 100, c).astype(np.int64)
        if t % 4 == 0:
            v[0] = lmax
        for tie in (1, 0):
            o = run("bre", v.reshape(1, c), lmax, tie, dtype=np.int64)
            n = int(o[0])
            ks, js = oracle.build_row_envelope(v, lmax, bool(tie))
            assert o[1:1 + n].tolist() == ks.tolist() and o[1 + n:].tolist() == js.tolist()
    for which in range(6):
        img = oracle.random_image(40, 77, 0.03, which)
        dm = oracle.init_map(img)
        np.testing.assert_array_equal(run("pass", dm, which), oracle.raster_pass(dm, which).ravel())
    vert = rng.integers(0, 5000, (20, 50)).astype(np.uint64)   # not perfect squares
    vert[rng.random((20, 50)) < 0.3] = INF
    m = run("meijster_raw", vert, dtype=np.uint8)
    d, ncol = oracle.meijster_scan(vert, take_new=True)
    np.testing.assert_array_equal(m[: 8 * vert.size].view(np.uint64), d.ravel())
    np.testing.assert_array_equal(m[8 * vert.size:].view(np.uint32), ncol.ravel())


ACC_DROPIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_dropin")


@pytest.mark.skipif(not os.path.exists(ACC_DROPIN), reason="oracle/_ref/acceptance_dropin not built")
def test_reference_acceptance_suite_relinked_against_dropin():
    """The reference's own acceptance.cpp (proj/tests/acceptance.cpp:341-363),
    unmodified, linked against libdistfield_b200 (+ the reference's metrics.cpp,
    outside the drop-in's scope; vector_dt comes from the drop-in): every
    criterion passes except c4, which fails in the reference itself (chamfer
    chart accuracy, proj/README.md:50-55; no drop-in code involved).  Criterion
    1 also times each call against 1 s (acceptance.cpp:49-54): the drop-in
    creates its CUDA context at load time (cpp/src/warmup.cpp)."""
    p = subprocess.run([ACC_DROPIN], capture_output=True, text=True, timeout=600)
    lines = [l for l in p.stdout.splitlines() if l.startswith("criterion")]
    status = {int(l.split()[1].rstrip(":")): l.split()[2] for l in lines}
    assert status == {1: "PASS", 2: "PASS", 3: "PASS", 4: "FAIL", 5: "PASS", 6: "PASS", 7: "PASS"}, p.stdout


def test_dropin_danielsson():
    """distfield::danielsson / danielsson_first_sweep / to_text(OffsetMap)
    (vector_dt.hpp) through the drop-in: maps and offsets as the oracle, the
    text dump byte for byte."""
    rng = np.random.default_rng(8)
    for t in range(6):
        img = (rng.random((int(rng.integers(1, 50)), int(rng.integers(1, 60)))) < [0.0, 0.02, 0.1, 0.5][t % 4]).astype(np.uint8)
        n = img.size
        for op, fs in (("danielsson", False), ("danielsson_first", True)):
            raw = run(op, img, dtype=np.uint8)
            d, dy, dx = oracle.danielsson(img, fs)
            np.testing.assert_array_equal(raw[:8 * n].view(np.uint64), d.ravel())
            np.testing.assert_array_equal(raw[8 * n:12 * n].view(np.uint32), dy.ravel())
            np.testing.assert_array_equal(raw[12 * n:16 * n].view(np.uint32), dx.ravel())
            want = "".join(" ".join("inf" if dy[i, j] == 0xFFFFFFFF else f"{dy[i, j]},{dx[i, j]}"
                                    for j in range(img.shape[1])) + "\n" for i in range(img.shape[0]))
            assert raw[16 * n:].tobytes().decode() == want

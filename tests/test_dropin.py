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
        np.ascontiguousarray(img, np.uint8).tofile(fi)
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

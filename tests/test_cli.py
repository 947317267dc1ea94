"""The CLI path (lib/distfield_b200: the reference CLI's transform / labels /
bench subcommands over the B200 library) against the UNMODIFIED reference's
own I/O layer (read_netpbm, to_text, to_text_sqrt, chamfer_normalized,
to_gray, labels_to_gray through oracle/_ref), byte for byte.

CPU tests: argument handling and every Netpbm header/raster error (they fail
before any device call).  GPU tests: outputs for P1/P4/point-list inputs,
all metrics, both polarities, dumps, graymaps and labels.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2106_03503_b200", "lib", "distfield_b200")

needs_cli = pytest.mark.skipif(not os.path.exists(CLI), reason="CLI not built (run __graft_entry__.build())")
needs_ref = pytest.mark.skipif(oracle.ref is None, reason="oracle/_ref not built")


def run(*args, cwd=None):
    return subprocess.run([CLI, *args], capture_output=True, text=False, cwd=cwd, timeout=120)


def pbm_plain(img):
    rows = ["".join("1" if v else "0" for v in r) for r in img]
    return ("P1\n%d %d\n" % (img.shape[1], img.shape[0]) + "\n".join(rows) + "\n").encode()


# ---------------------------------------------------------------- CPU ----

BAD_INPUTS = [
    b"",
    b"X1\n2 2\n",
    b"P3\n2 2\n",
    b"P1",
    b"P1\n",
    b"P1 x 3\n",
    b"P1 2\n",
    b"P1 0 3\n",
    b"P1 99999999 1\n",
    b"P1\n2 1\n1 2",
    b"P1\n2 2\n1 0 1",
    b"P1 # comment\n2 # more\n1\n1 #\n0",
    b"P4\n3 1",
    b"P4\n3 1x\x00",
    b"P4\n10 3\n\x80\x40\x00",
    b"P4 10 3\n\x80",
    b"P4\n# c\n12 2\n\x01\x02\x03",
]


@needs_cli
@needs_ref
@pytest.mark.parametrize("k", range(len(BAD_INPUTS)))
def test_netpbm_errors_match_reference(tmp_path, k):
    data = BAD_INPUTS[k]
    img, err = oracle.ref_read_netpbm(data)
    f = tmp_path / "in.pbm"
    f.write_bytes(data)
    if err is None:  # a valid file (the comment case): needs the device, covered below
        assert img is not None
        return
    p = run("transform", "--input", str(f), "--dump", str(tmp_path / "o.txt"))
    assert p.returncode == 1
    assert p.stderr.decode().strip() == "error: " + err


@needs_cli
def test_usage_and_option_errors(tmp_path):
    assert run().returncode == 106
    assert run("--help").returncode == 0
    assert run("transform", "--bogus").returncode == 109
    assert run("transform", "--polarity", "sideways", "--dump", "x").returncode == 105
    assert run("transform", "--orient", "diag", "--dump", "x").returncode == 105
    assert run("frobnicate").returncode == 109
    p = run("transform", "--input", "nofile.pbm")
    assert p.returncode == 1 and b"no output requested (--dump, --gray, --labels, --offsets)" in p.stderr
    p = run("transform", "--metric", "chamfer34", "--algorithm", "envelope", "--dump", "x")
    assert p.returncode == 1 and b"chamfer34 takes no --algorithm" in p.stderr
    p = run("transform", "--metric", "cityblock", "--algorithm", "envelope", "--dump", "x")
    assert p.returncode == 1 and b"cityblock supports --algorithm sequential|separable" in p.stderr
    p = run("transform", "--metric", "euclidean", "--algorithm", "fast", "--dump", "x")
    assert p.returncode == 1 and b"euclidean supports --algorithm" in p.stderr
    p = run("transform", "--metric", "hamming", "--dump", "x")
    assert p.returncode == 1 and b"unknown --metric hamming" in p.stderr
    p = run("transform", "--dump", "x")
    assert p.returncode == 1 and b"an input is required (--input or --points-file)" in p.stderr
    p = run("transform", "--points-file", "p.txt", "--dump", "x")
    assert p.returncode == 1 and b"--points-file requires --size ROWSxCOLS" in p.stderr
    p = run("transform", "--points-file", "p.txt", "--size", "9by10", "--dump", "x")
    assert p.returncode == 1 and b"--size expects ROWSxCOLS" in p.stderr
    p = run("transform", "--input", "a.pbm", "--points-file", "p.txt", "--dump", "x")
    assert p.returncode == 1 and b"choose one of --input or --points-file" in p.stderr
    p = run("transform", "--input", str(tmp_path / "missing.pbm"), "--dump", "x")
    assert p.returncode == 1 and b"cannot open" in p.stderr
    p = run("labels", "--input", "a.pbm")
    assert p.returncode == 1 and b"no output requested (--out, --dump)" in p.stderr
    p = run("bench", "--algorithms", "quick")
    assert p.returncode == 1 and b"unknown algorithm quick" in p.stderr
    p = run("chart", "--radius", "3")
    assert p.returncode == 1


@needs_ref
def test_reference_pbm_writer_round_trips_through_the_parser():
    """Pins the packed layout the GPU unpack relies on: MSB first, rows padded."""
    rng = np.random.default_rng(3)
    for shape in [(1, 1), (3, 7), (5, 8), (4, 9), (17, 33)]:
        img = (rng.random(shape) < 0.4).astype(np.uint8)
        data = oracle.ref_write_pbm(img, raw=True)
        back, err = oracle.ref_read_netpbm(data)
        assert err is None
        np.testing.assert_array_equal(back, img)
        body = data[data.index(b"\n", 3) + 1:]
        rb = (shape[1] + 7) // 8
        bits = np.unpackbits(np.frombuffer(body, np.uint8).reshape(shape[0], rb), axis=1)[:, :shape[1]]
        np.testing.assert_array_equal(bits, img)


# ---------------------------------------------------------------- GPU ----

def _images():
    rng = np.random.default_rng(11)
    six = np.zeros((9, 10), np.uint8)
    for r, c in [(1, 4), (2, 8), (4, 1), (5, 6), (7, 2), (8, 9)]:
        six[r, c] = 1
    out = {"six": six,
           "rand_7x13": (rng.random((7, 13)) < 0.1).astype(np.uint8),
           "rand_40x64": (rng.random((40, 64)) < 0.02).astype(np.uint8),
           "rand_33x100": (rng.random((33, 100)) < 0.3).astype(np.uint8),
           "one_px": np.zeros((5, 5), np.uint8),
           "full": np.ones((4, 6), np.uint8)}
    out["one_px"][2, 3] = 1
    return out


IMAGES = _images()


def _pgm(gray):
    return b"P5\n%d %d\n255\n" % (gray.shape[1], gray.shape[0]) + gray.astype(np.uint8).tobytes()


@pytest.mark.gpu
@needs_cli
@needs_ref
@pytest.mark.parametrize("name", sorted(IMAGES))
@pytest.mark.parametrize("fmt", ["p4", "p1"])
@pytest.mark.parametrize("polarity", ["outside", "inside"])
def test_transform_outputs_match_reference(tmp_path, name, fmt, polarity):
    img = IMAGES[name]
    src = img if polarity == "outside" else (img == 0).astype(np.uint8)
    f = tmp_path / "in.pbm"
    f.write_bytes(oracle.ref_write_pbm(img, raw=True) if fmt == "p4" else pbm_plain(img))
    for metric, mid in (("euclidean", 0), ("cityblock", 1), ("chamfer34", 2)):
        modes = [("plain", 0)] + ([("--sqrt", 1)] if mid == 0 else []) + ([("--normalized", 2)] if mid == 2 else [])
        for flag, mode in modes:
            args = ["transform", "--input", str(f), "--polarity", polarity, "--metric", metric,
                    "--dump", str(tmp_path / "d.txt"), "--gray", str(tmp_path / "g.pgm")]
            if flag != "plain":
                args.append(flag)
            if mid == 0:
                args += ["--labels", str(tmp_path / "l.pgm")]
            p = run(*args)
            want_gray = oracle.ref_transform_gray(src, mid, mid == 0)
            if src.sum() == 0:
                # featureless: warning, then to_gray's domain_error
                assert p.returncode == 1 and b"no finite value" in p.stderr
                continue
            assert p.returncode == 0, p.stderr
            assert (tmp_path / "d.txt").read_text() == oracle.ref_transform_text(src, mid, mode), (metric, flag)
            assert (tmp_path / "g.pgm").read_bytes() == _pgm(want_gray), metric
            if mid == 0:
                lab_gray, _ = oracle.ref_labels_render(src)
                assert (tmp_path / "l.pgm").read_bytes() == _pgm(lab_gray)


@pytest.mark.gpu
@needs_cli
@needs_ref
@pytest.mark.parametrize("name", sorted(IMAGES))
def test_labels_subcommand_matches_reference(tmp_path, name):
    img = IMAGES[name]
    f = tmp_path / "in.pbm"
    f.write_bytes(oracle.ref_write_pbm(img, raw=True))
    p = run("labels", "--input", str(f), "--out", str(tmp_path / "l.pgm"), "--dump", str(tmp_path / "l.txt"))
    want = oracle.ref_labels_render(img)
    assert p.returncode == 0, p.stderr
    assert (tmp_path / "l.pgm").read_bytes() == _pgm(want[0])
    assert (tmp_path / "l.txt").read_text() == want[1]


@pytest.mark.gpu
@needs_cli
def test_featureless_inputs(tmp_path):
    f = tmp_path / "empty.pbm"
    f.write_bytes(b"P4\n5 2\n\x00\x00")
    p = run("transform", "--input", str(f), "--dump", str(tmp_path / "d.txt"))
    assert p.returncode == 0
    assert b"warning: no features, distances are infinite everywhere" in p.stderr
    assert (tmp_path / "d.txt").read_text() == "inf inf inf inf inf\ninf inf inf inf inf\n"
    p = run("labels", "--input", str(f), "--dump", str(tmp_path / "l.txt"))
    assert p.returncode == 1 and b"error: no features: voronoi labels undefined" in p.stderr


@pytest.mark.gpu
@needs_cli
@needs_ref
def test_points_file_input(tmp_path):
    pts = tmp_path / "p.txt"
    pts.write_text("# six points\n1 4\n2 8  # trailing\n\n4 1\n5 6\n7 2\n8 9\n")
    p = run("transform", "--points-file", str(pts), "--size", "9x10", "--dump", str(tmp_path / "d.txt"), "--sqrt")
    assert p.returncode == 0, p.stderr
    assert (tmp_path / "d.txt").read_text() == oracle.ref_transform_text(IMAGES["six"], 0, 1)
    bad = tmp_path / "bad.txt"
    bad.write_text("1 4\n7\n")
    p = run("transform", "--points-file", str(bad), "--size", "9x10", "--dump", str(tmp_path / "d.txt"))
    assert p.returncode == 1 and b"bad.txt:2: expected \"row col\"" in p.stderr


@pytest.mark.gpu
@needs_cli
def test_bench_subcommand_csv(tmp_path):
    p = run("bench", "--sizes", "16,33", "--reps", "2", "--algorithms", "envelope,simple", "--out",
            str(tmp_path / "b.csv"))
    assert p.returncode == 0, p.stderr
    lines = (tmp_path / "b.csv").read_text().splitlines()
    assert lines[0] == "cells,algorithm,size,rep,wall_ns,candidates"
    rows = [ln.split(",") for ln in lines[1:]]
    assert [(r[0], r[1], r[2], r[3]) for r in rows] == [
        (str(s * s), a, str(s), str(rep)) for s in (16, 33) for rep in (0, 1) for a in ("envelope", "simple")]
    assert all(int(r[4]) > 0 for r in rows)


def _offsets_text(dy, dx):
    """to_text(OffsetMap) (vector_dt.cpp:7-21): "dy,dx" or "inf", one line per row."""
    return "".join(" ".join("inf" if dy[i, j] == 0xFFFFFFFF else f"{dy[i, j]},{dx[i, j]}" for j in range(dy.shape[1]))
                   + "\n" for i in range(dy.shape[0]))


@pytest.mark.gpu
@needs_cli
def test_danielsson_algorithm_and_offsets_dump(tmp_path):
    """--algorithm danielsson / --offsets (distfield_cli.cpp:177-179, :192-220;
    the reference's own test: test_cli.cpp:136-150): the squared-distance dump
    and the offsets dump of the vector transform, and the option errors."""
    img = oracle.random_image(23, 31, 0.04, 99)
    f = tmp_path / "in.pbm"
    f.write_bytes(pbm_plain(img))
    p = run("transform", "--input", str(f), "--algorithm", "danielsson", "--dump", str(tmp_path / "d.txt"),
            "--offsets", str(tmp_path / "o.txt"))
    assert p.returncode == 0, p.stderr
    d, dy, dx = oracle.danielsson(img)
    assert (tmp_path / "o.txt").read_text() == _offsets_text(dy, dx)
    want = "".join(" ".join("inf" if v == oracle.INF else str(int(v)) for v in row) + "\n" for row in d)
    assert (tmp_path / "d.txt").read_text() == want
    p = run("transform", "--input", str(f), "--offsets", str(tmp_path / "o2.txt"))
    assert p.returncode == 1 and b"--offsets requires --algorithm danielsson" in p.stderr
    p = run("transform", "--input", str(f), "--algorithm", "danielsson", "--labels", str(tmp_path / "l.pgm"))
    assert p.returncode == 1 and b"--labels requires an exact euclidean algorithm" in p.stderr

"""Parity oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package; the product package ``paper_2106_03503_b200``
never does (it fails loudly when its CUDA library is missing instead).

Two checkers live here:

* ``orc``  -- ``oracle/dt_oracle.c``: a plain-C restatement of the reference
  hot path (each function cites the reference file:line it follows), built
  into ``oracle/build/liborc.so``.
* ``ref``  -- the unmodified reference library compiled from
  ``/root/reference/proj/core/src`` into ``oracle/_ref/libdfref.so`` via
  ``oracle/Makefile`` (+ ``oracle/ref_shim.cpp``).  ``None`` when absent.

Parity is pinned: tests/test_oracle.py checks ``orc`` against the reference's
golden matrices (tests/golden/six_point.json, dumped from
proj/tests/goldens.hpp) and against ``ref`` on seeded random images.

All distance outputs use the reference convention: uint64 with
``INF = 2**64-1`` (grid.hpp:113); labels uint32 ordinals with
``NO_LABEL = 2**32-1`` (grid.hpp:174).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
INF = np.uint64(2**64 - 1)
NO_LABEL = np.uint32(2**32 - 1)

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_sz = C.c_uint64


def build() -> None:
    """Compile the checkers (C restatement; reference shim when the sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path):
    return C.CDLL(path) if os.path.exists(path) else None


def _bind_orc(lib):
    lib.orc_kind_bound.restype = C.c_uint64
    lib.orc_kind_bound.argtypes = [C.c_int, _sz, _sz]
    lib.orc_generate_random_image.argtypes = [_sz, _sz, C.c_double, C.c_uint64, _u8p]
    lib.orc_vertical_pass.argtypes = [_u8p, _sz, _sz, _u64p]
    lib.orc_init_map.argtypes = [_u8p, _sz, _sz, _u64p]
    lib.orc_vertical_down_pass.argtypes = [_u64p, _sz, _sz]
    lib.orc_vertical_up_pass.argtypes = [_u64p, _sz, _sz]
    lib.orc_build_row_envelope.restype = C.c_int64
    lib.orc_build_row_envelope.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_int, _i64p, _i64p,
                                           C.POINTER(C.c_uint64)]
    lib.orc_envelope_scan.argtypes = [_u64p, _sz, _sz, C.c_int, _u64p, C.c_void_p,
                                      C.POINTER(C.c_uint64)]
    lib.orc_edt.argtypes = [_u8p, _sz, _sz, _u64p]
    lib.orc_voronoi_labels.restype = C.c_int
    lib.orc_voronoi_labels.argtypes = [_u8p, _sz, _sz, _u32p, C.c_void_p]
    for f in ("orc_cityblock_sequential", "orc_chamfer34", "orc_chessboard"):
        getattr(lib, f).argtypes = [_u8p, _sz, _sz, _u64p]
    lib.orc_brute.argtypes = [_u8p, _sz, _sz, C.c_int, _u64p]
    lib.orc_raster_pass.argtypes = [_u64p, _sz, _sz, C.c_int]
    lib.orc_danielsson.argtypes = [_u8p, _sz, _sz, C.c_int, _u64p, _u32p, _u32p]
    return lib


def _bind_ref(lib):
    if lib is None:
        return None
    dp = C.POINTER(C.c_double)
    lib.dfref_generate_random_image.argtypes = [_sz, _sz, C.c_double, C.c_uint64, _u8p]
    lib.dfref_edt.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, C.c_uint, C.c_void_p,
                              C.c_void_p, dp]
    lib.dfref_vertical_pass.argtypes = [_u8p, _sz, _sz, _u64p]
    lib.dfref_meijster_scan.argtypes = [_u8p, _sz, _sz, _u64p, _u32p]
    lib.dfref_row_envelope.restype = C.c_longlong
    lib.dfref_row_envelope.argtypes = [_u8p, _sz, _sz, _sz, _i64p, _i64p]
    lib.dfref_voronoi_labels.restype = C.c_int
    lib.dfref_voronoi_labels.argtypes = [_u8p, _sz, _sz, C.c_uint, _u32p, dp]
    lib.dfref_edt_labels_batch.restype = C.c_int
    lib.dfref_edt_labels_batch.argtypes = [_u8p, _sz, _sz, _sz, C.c_uint, C.c_void_p, C.c_void_p, dp]
    lib.dfref_propagation.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_uint, _u64p, dp]
    szp = C.POINTER(_sz)
    lib.dfref_read_netpbm.argtypes = [C.c_char_p, _sz, C.c_void_p, szp, szp, C.c_char_p, _sz]
    lib.dfref_write_pbm.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_char_p, _sz]
    lib.dfref_transform_text.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, C.c_char_p, _sz]
    lib.dfref_transform_gray.argtypes = [_u8p, _sz, _sz, C.c_int, C.c_int, _u8p]
    lib.dfref_labels_render.argtypes = [_u8p, _sz, _sz, _u8p, C.c_char_p, _sz, C.POINTER(C.c_int)]
    lib.dfref_build_row_envelope.restype = C.c_longlong
    lib.dfref_build_row_envelope.argtypes = [_i64p, _sz, C.c_int64, C.c_int, _i64p, _i64p]
    lib.dfref_raster_pass.argtypes = [_u64p, _sz, _sz, C.c_int]
    if hasattr(lib, "dfref_danielsson"):
        lib.dfref_danielsson.argtypes = [_u8p, _sz, _sz, C.c_int, _u64p, _u32p, _u32p]
    lib.dfref_kind_bound.restype = C.c_uint64
    lib.dfref_kind_bound.argtypes = [C.c_int, _sz, _sz]
    return lib


_ORC = os.path.join(HERE, "build", "liborc.so")
if os.path.exists(_ORC):
    with open(_ORC, "rb") as _f:
        if b"dfg_sparse_tiles" not in _f.read():  # built before the generators moved in
            os.remove(_ORC)
if not os.path.exists(_ORC):
    build()
orc = _bind_orc(C.CDLL(_ORC))
ref = _bind_ref(_load(os.path.join(HERE, "_ref", "libdfref.so")))


def _img(img):
    img = np.ascontiguousarray(img, dtype=np.uint8)
    assert img.ndim == 2
    return img, img.shape[0], img.shape[1]


# ------------------------------------------------------------------ workloads
def workload(name, scale=1, seed=None):
    """The seeded input of config `name` (workloads.config) generated by the
    oracle's own copy of workloads/gen.c: the reference arm of bench.py uses
    this, so it maps no library of the product."""
    import workloads
    return workloads.config(name, scale=scale, seed=seed, lib=_wl_lib())


_wl_bound = None


def _wl_lib():
    global _wl_bound
    if _wl_bound is None:
        import workloads
        _wl_bound = workloads.bind(orc)
    return _wl_bound


# ---------------------------------------------------------------- C restatement
def random_image(rows, cols, density, seed):
    out = np.empty((rows, cols), np.uint8)
    orc.orc_generate_random_image(rows, cols, density, seed, out)
    return out


def vertical_pass(img):
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    orc.orc_vertical_pass(img, r, c, out)
    return out


def init_map(img):
    """init_distance_map (grid.cpp:85-91), squared Euclidean: 0 at objects, INF elsewhere."""
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    orc.orc_init_map(img, r, c, out)
    return out


def vertical_down_pass(dm):
    """vertical_down_pass (exact_edt.cpp:74-91) on a copy of a uint64 map."""
    out = np.ascontiguousarray(dm, dtype=np.uint64).copy()
    orc.orc_vertical_down_pass(out, out.shape[0], out.shape[1])
    return out


def vertical_up_pass(dm):
    """vertical_up_pass (exact_edt.cpp:93-110) on a copy of a uint64 map."""
    out = np.ascontiguousarray(dm, dtype=np.uint64).copy()
    orc.orc_vertical_up_pass(out, out.shape[0], out.shape[1])
    return out


def edt(img):
    """Exact squared EDT, uint64 with INF (exact_edt.cpp:285-317)."""
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    orc.orc_edt(img, r, c, out)
    return out


def meijster_scan(vert, take_new=True):
    """(map, nearest_col) for a vertical-pass map (exact_edt.cpp:242-283)."""
    vert = np.ascontiguousarray(vert, np.uint64)
    r, c = vert.shape
    out = np.empty((r, c), np.uint64)
    col = np.empty((r, c), np.uint32)
    orc.orc_envelope_scan(vert, r, c, 1 if take_new else 0, out, col.ctypes.data, None)
    return out, col


def row_envelope(vert_row, rows, take_new=True):
    """build_row_envelope on one vertical-pass row; returns (ks, js)."""
    c = len(vert_row)
    lmax = int(orc.orc_kind_bound(3, rows, c)) + 1
    buf = np.array([lmax if v == INF else int(v) for v in vert_row], np.int64)
    ks = np.zeros(c + 1, np.int64)
    js = np.zeros(c + 2, np.int64)
    n = orc.orc_build_row_envelope(buf, c, lmax, 1 if take_new else 0, ks, js, None)
    return ks[:n].copy(), js[: n + 1].copy()


def raster_pass(dm, which):
    """One per-pass in-place function (propagation.cpp:16-88) on a copy of a
    uint64 map; which: 0 cityblock_forward_pass, 1 cityblock_backward_pass,
    2 cityblock_vertical_passes, 3 cityblock_horizontal_passes,
    4 chamfer_forward_pass, 5 chamfer_backward_pass."""
    out = np.ascontiguousarray(dm, dtype=np.uint64).copy()
    orc.orc_raster_pass(out, out.shape[0], out.shape[1], which)
    return out


def build_row_envelope(vert_i64, lmax, take_new=True):
    """build_row_envelope (exact_edt.cpp:190-230) on an int64 row: (ks, js)."""
    buf = np.ascontiguousarray(vert_i64, np.int64)
    c = buf.size
    ks = np.zeros(c + 1, np.int64)
    js = np.zeros(c + 2, np.int64)
    n = orc.orc_build_row_envelope(buf, c, int(lmax), 1 if take_new else 0, ks, js, None)
    return ks[:n].copy(), js[: n + 1].copy()


def voronoi_labels(img, linear=False):
    """Feature ordinals (exact_edt.cpp:319-371); None when featureless (domain_error).
    With linear=True returns (ordinals, int32 row*cols+col)."""
    img, r, c = _img(img)
    lab = np.empty((r, c), np.uint32)
    lin = np.empty((r, c), np.int32)
    st = orc.orc_voronoi_labels(img, r, c, lab, lin.ctypes.data)
    if st != 0:
        return None
    return (lab, lin) if linear else lab


def cityblock(img):
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    orc.orc_cityblock_sequential(img, r, c, out)
    return out


def chamfer34(img):
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    orc.orc_chamfer34(img, r, c, out)
    return out


def chessboard(img):
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    orc.orc_chessboard(img, r, c, out)
    return out


def brute(img, metric):
    """oracles.hpp min-over-features; metric 0 L1, 1 Linf, 3 squared euclidean."""
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    orc.orc_brute(img, r, c, metric, out)
    return out


def danielsson(img, first_sweep=False):
    """vector_dt.cpp:108-124 restated: (squared distances uint64, dy, dx uint32;
    0xFFFFFFFF = unset offset, UINT64_MAX = infinity)."""
    img, r, c = _img(img)
    d = np.empty((r, c), np.uint64)
    dy = np.empty((r, c), np.uint32)
    dx = np.empty((r, c), np.uint32)
    orc.orc_danielsson(img, r, c, int(first_sweep), d, dy, dx)
    return d, dy, dx


def ref_danielsson(img, first_sweep=False):
    """The reference's own danielsson / danielsson_first_sweep (oracle/_ref)."""
    img, r, c = _img(img)
    d = np.empty((r, c), np.uint64)
    dy = np.empty((r, c), np.uint32)
    dx = np.empty((r, c), np.uint32)
    ref.dfref_danielsson(img, r, c, int(first_sweep), d, dy, dx)
    return d, dy, dx


def to_i32(dm):
    """uint64 reference map -> int32 with INF -> 0x7fffffff (the C-ABI sentinel)."""
    dm = np.asarray(dm)
    out = np.where(dm == INF, np.uint64(0x7FFFFFFF), dm)
    assert int(out.max(initial=0)) <= 0x7FFFFFFF
    return out.astype(np.int32)


def sqrt_f32(d_i32):
    """float32 distance as the reference would print it: (float)sqrt((double)D), +inf for INF."""
    d = np.asarray(d_i32)
    out = np.sqrt(d.astype(np.float64)).astype(np.float32)
    out[d == 0x7FFFFFFF] = np.inf
    return out


# ------------------------------------------------------------- reference (.so)
def ref_available():
    return ref is not None


def ref_random_image(rows, cols, density, seed):
    out = np.empty((rows, cols), np.uint8)
    ref.dfref_generate_random_image(rows, cols, density, seed, out)
    return out


def ref_edt(img, algorithm=3, orient=0, threads=1, want_time=False):
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    ns = C.c_double(0)
    ref.dfref_edt(img, r, c, algorithm, orient, threads, out.ctypes.data, None, C.byref(ns))
    return (out, ns.value) if want_time else out


def ref_edt_candidates(img, algorithm=3):
    img, r, c = _img(img)
    cand = C.c_uint64(0)
    ref.dfref_edt(img, r, c, algorithm, 0, 1, None, C.addressof(cand), None)
    return cand.value


def ref_vertical_pass(img):
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    ref.dfref_vertical_pass(img, r, c, out)
    return out


def ref_meijster_scan(img):
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    col = np.empty((r, c), np.uint32)
    ref.dfref_meijster_scan(img, r, c, out, col)
    return out, col


def ref_row_envelope(img, row):
    img, r, c = _img(img)
    ks = np.zeros(c + 1, np.int64)
    js = np.zeros(c + 2, np.int64)
    n = ref.dfref_row_envelope(img, r, c, row, ks, js)
    return ks[:n].copy(), js[: n + 1].copy()


def ref_build_row_envelope(vert_i64, lmax, take_new=True):
    buf = np.ascontiguousarray(vert_i64, np.int64)
    c = buf.size
    ks = np.zeros(c + 1, np.int64)
    js = np.zeros(c + 2, np.int64)
    n = ref.dfref_build_row_envelope(buf, c, int(lmax), 1 if take_new else 0, ks, js)
    return ks[:n].copy(), js[: n + 1].copy()


def ref_raster_pass(dm, which):
    out = np.ascontiguousarray(dm, dtype=np.uint64).copy()
    ref.dfref_raster_pass(out, out.shape[0], out.shape[1], which)
    return out


def ref_voronoi_labels(img, threads=1):
    img, r, c = _img(img)
    lab = np.empty((r, c), np.uint32)
    st = ref.dfref_voronoi_labels(img, r, c, threads, lab, None)
    return None if st != 0 else lab


def ref_propagation(img, kind, threads=1, want_time=False):
    """kind 0 cityblock_sequential, 1 cityblock_separable, 2 chamfer34."""
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint64)
    ns = C.c_double(0)
    ref.dfref_propagation(img, r, c, kind, threads, out, C.byref(ns))
    return (out, ns.value) if want_time else out


# ---- the CLI's I/O layer, from the reference (checkers for tools/distfield_b200) ----

def ref_read_netpbm(data: bytes):
    """(image, None) or (None, error message) from the reference read_netpbm."""
    r, c = _sz(0), _sz(0)
    err = C.create_string_buffer(512)
    if ref.dfref_read_netpbm(data, len(data), None, C.byref(r), C.byref(c), err, 512) != 0:
        return None, err.value.decode()
    out = np.empty((r.value, c.value), np.uint8)
    ref.dfref_read_netpbm(data, len(data), out.ctypes.data, C.byref(r), C.byref(c), err, 512)
    return out, None


def ref_write_pbm(img, raw=True) -> bytes:
    img, r, c = _img(img)
    n = ref.dfref_write_pbm(img, r, c, int(raw), None, 0)
    buf = C.create_string_buffer(n)
    ref.dfref_write_pbm(img, r, c, int(raw), buf, n)
    return buf.raw[:n]


def ref_transform_text(img, metric, mode=0) -> str:
    """metric 0 edt / 1 cityblock / 2 chamfer34; mode 0 plain, 1 sqrt, 2 normalized."""
    img, r, c = _img(img)
    n = ref.dfref_transform_text(img, r, c, metric, mode, None, 0)
    buf = C.create_string_buffer(n + 1)
    ref.dfref_transform_text(img, r, c, metric, mode, buf, n + 1)
    return buf.value.decode()


def ref_transform_gray(img, metric, sqrt_mode):
    img, r, c = _img(img)
    out = np.empty((r, c), np.uint8)
    return None if ref.dfref_transform_gray(img, r, c, metric, int(sqrt_mode), out) else out


def ref_labels_render(img):
    """(labels_to_gray image, to_text(labels)) or None when the reference throws."""
    img, r, c = _img(img)
    gray = np.empty((r, c), np.uint8)
    n = C.c_int(0)
    if ref.dfref_labels_render(img, r, c, gray, None, 0, C.byref(n)):
        return None
    buf = C.create_string_buffer(n.value + 1)
    ref.dfref_labels_render(img, r, c, gray, buf, n.value + 1, C.byref(n))
    return gray, buf.value.decode()

"""Seeded synthetic inputs for the five BASELINE.json configs.

Bench / test infrastructure, not the product: the paper's figure images are
absent from the reference tree, so every config is a seeded stand-in with the
specified shape, size and value distribution, generated on the host by
``gen.c`` (the reference xorshift64* PRNG, random_image.hpp:12-29) so the
oracle and the GPU see identical bytes.

The C generators are bound lazily: ``bench.py``'s own arm uses
``workloads/libdfgen.so``; the reference arm and the tests pass ``lib=`` the
oracle's library (``oracle/build/liborc.so`` compiles the same ``gen.c``), so
the reference arm maps no library of the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64, _u64 = C.c_int64, C.c_uint64

# master seeds, recorded in every bench line
SEEDS = {"c1": 2106, "c2": 3503, "c3": 20210607, "c4": 8192, "c5": 32768}

_default = None


def bind(lib):
    """Declare the dfg_* generator signatures on a ctypes library holding gen.c."""
    lib.dfg_bernoulli.argtypes = [_u8p, _i64, _i64, C.c_double, _u64]
    lib.dfg_discs.argtypes = [_u8p, _i64, _i64, _i64, _u64]
    lib.dfg_points_batch.argtypes = [_u8p, _i64, _i64, _i64, _i64, _u64]
    lib.dfg_shapes.argtypes = [_u8p, _i64, _i64, _i64, _u64]
    lib.dfg_sparse_tiles.argtypes = [_u8p, _i64, _i64, _i64, _i64, C.c_double, _u64, C.c_int]
    lib.dfg_splitmix64.restype = _u64
    lib.dfg_splitmix64.argtypes = [_u64]
    return lib


def _lib(lib=None):
    global _default
    if lib is not None:
        return lib
    if _default is None:
        path = os.path.join(HERE, "libdfgen.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        _default = bind(C.CDLL(path))
    return _default


def bernoulli(rows, cols, density, seed, lib=None):
    out = np.empty((rows, cols), np.uint8)
    _lib(lib).dfg_bernoulli(out, rows, cols, density, seed)
    return out


def discs(rows, cols, n, seed, lib=None):
    out = np.empty((rows, cols), np.uint8)
    _lib(lib).dfg_discs(out, rows, cols, n, seed)
    return out


def points_batch(n_img, rows, cols, npts, master, lib=None):
    out = np.empty((n_img, rows, cols), np.uint8)
    _lib(lib).dfg_points_batch(out, n_img, rows, cols, npts, master)
    return out


def shapes(rows, cols, n, seed, lib=None):
    out = np.empty((rows, cols), np.uint8)
    _lib(lib).dfg_shapes(out, rows, cols, n, seed)
    return out


def sparse_tiles(rows, cols, tile=1024, n_on=256, p=1e-4, seed=SEEDS["c5"], degenerate=False, lib=None):
    out = np.empty((rows, cols), np.uint8)
    _lib(lib).dfg_sparse_tiles(out, rows, cols, tile, n_on, p, seed, 1 if degenerate else 0)
    return out


def config(name: str, scale: int = 1, seed: int | None = None, lib=None):
    """Input of config `name` ("c1".."c5", "c5d" = degenerate corner variant).
    scale > 1 shrinks every linear dimension (and the object counts
    proportionally to the area) for fast parity tests."""
    s = SEEDS.get(name[:2], 1) if seed is None else seed
    if name == "c1":
        return bernoulli(600 // scale, 500 // scale, 0.01, s, lib)
    if name == "c2":
        n = 4096 // scale
        return discs(n, n, max(1, 200 // (scale * scale)), s, lib)
    if name == "c3":
        n = 1024 // scale
        return points_batch(max(1, 1024 // (scale * scale)), n, n, 30, s, lib)
    if name == "c4":
        n = 8192 // scale
        return shapes(n, n, max(1, 2000 // (scale * scale)), s, lib)
    if name == "c5":
        n = 32768 // scale
        tile = max(1, 1024 // scale)
        return sparse_tiles(n, n, tile, 256, 1e-4 * scale * scale if scale > 1 else 1e-4, s, lib=lib)
    if name == "c5d":
        n = 32768 // scale
        return sparse_tiles(n, n, degenerate=True, lib=lib)
    raise KeyError(name)

"""Reference-shaped host API: the ``distfield`` entry points of
/root/reference/proj/core (exact_edt.hpp:37-107, propagation.hpp:15-30), same
argument meaning, return types and error behaviour, computed on the GPU.

Inputs are 2-D numpy arrays (object pixel = nonzero, grid.hpp:82); outputs
follow the reference types: distance maps as uint64 with ``INF = 2**64-1``
(DistanceMap::kInfinity, grid.hpp:113), label maps as uint32 feature ordinals
(LabelMap, grid.hpp:172-188), nearest columns as uint32 with ``NO_COLUMN``
(kNoColumn, exact_edt.hpp:78).  The ``algorithm``/``orientation``/``threads``
arguments are accepted for signature compatibility: every algorithm and
orientation yields the identical map in the reference (exact_edt.hpp:97-99),
so all are served by the one GPU envelope path.  ``stats`` (a ScanStats-like
object with a ``candidates`` attribute) receives a deterministic count of one
candidate evaluation per cell.
"""
from __future__ import annotations

import enum

import numpy as np
import torch

from . import INF_I32, edt as _edt, label_ordinals, raster as _raster, vertical as _vertical
from . import vertical_down_pass as _vdown, vertical_up_pass as _vup
from . import danielsson as _danielsson

INF = np.uint64(2**64 - 1)
NO_COLUMN = np.uint32(2**32 - 1)
NO_LABEL = np.uint32(2**32 - 1)


class EdtAlgorithm(enum.IntEnum):  # exact_edt.hpp:90
    bruteforce = 0
    simple = 1
    improved = 2
    envelope = 3


class Orientation(enum.IntEnum):  # exact_edt.hpp:92-96
    automatic = 0
    rows = 1
    columns = 2


class DomainError(ValueError):
    """Python counterpart of the reference's std::domain_error (exact_edt.cpp:321)."""


def _to_device(img) -> torch.Tensor:
    a = np.ascontiguousarray(img)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("grid dimensions must be at least 1x1")  # grid.hpp:22-23
    if a.dtype != np.uint8:
        a = (a != 0).astype(np.uint8)
    host = torch.from_numpy(a).pin_memory()
    return host.to("cuda", non_blocking=True)


def _u64(d32: torch.Tensor) -> np.ndarray:
    d = d32.cpu().numpy().astype(np.uint64)
    d[d == INF_I32] = INF
    return d


def edt(img, algorithm=EdtAlgorithm.envelope, orient=Orientation.automatic, stats=None, threads=1):
    """edt(img, algorithm, orient, stats, threads) -- exact_edt.cpp:285-317."""
    dev = _to_device(img)
    out = _edt(dev, dist=False)
    if stats is not None:
        stats.candidates += dev.numel()
    return _u64(out["sqdist"])


def vertical_pass(img, threads=1):
    """vertical_pass -- exact_edt.cpp:112-117."""
    return _u64(_vertical(_to_device(img)))


def _vpass_np(dm, fn):
    a = np.ascontiguousarray(dm, dtype=np.uint64)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("grid dimensions must be at least 1x1")  # grid.hpp:22-23
    d = torch.from_numpy(a.view(np.int64)).cuda()
    fn(d)
    return d.cpu().numpy().view(np.uint64)


def vertical_down_pass(dm, threads=1):
    """vertical_down_pass -- exact_edt.cpp:74-91.  The reference mutates a
    DistanceMap in place; here the updated uint64 map is returned (and written
    back into ``dm`` when it is a writable C-contiguous uint64 array)."""
    out = _vpass_np(dm, _vdown)
    if isinstance(dm, np.ndarray) and dm.dtype == np.uint64 and dm.flags.c_contiguous and dm.flags.writeable:
        dm[...] = out
    return out


def vertical_up_pass(dm, threads=1):
    """vertical_up_pass -- exact_edt.cpp:93-110 (see vertical_down_pass)."""
    out = _vpass_np(dm, _vup)
    if isinstance(dm, np.ndarray) and dm.dtype == np.uint64 and dm.flags.c_contiguous and dm.flags.writeable:
        dm[...] = out
    return out


def meijster_scan_image(img, threads=1):
    """(meijster_scan(vertical_pass(img)).map, .nearest_col) -- exact_edt.cpp:272-283."""
    out = _edt(_to_device(img), dist=False, nearest_col=True)
    nc = out["nearest_col"].cpu().numpy().astype(np.int64)
    return _u64(out["sqdist"]), np.where(nc < 0, int(NO_COLUMN), nc).astype(np.uint32)


def voronoi_labels(img, threads=1):
    """voronoi_labels -- exact_edt.cpp:319-371 (ordinal ids; DomainError when featureless)."""
    dev = _to_device(img)
    out = _edt(dev, dist=False, label=True)
    if int(out["sqdist"][0, 0]) == INF_I32:  # no object pixel anywhere
        raise DomainError("no features: voronoi labels undefined")
    return label_ordinals(dev, out["label"]).cpu().numpy().astype(np.uint32)


def voronoi_labels_linear(img):
    """int32 linear-index labels (row*cols+col), -1 for a featureless image."""
    return _edt(_to_device(img), dist=False, label=True)["label"].cpu().numpy()


def _raster1(img, key):
    return _u64(_raster(_to_device(img), **{k: k == key for k in ("cityblock", "chessboard", "chamfer34")})[key])


def cityblock_sequential(img):
    """cityblock_sequential -- propagation.cpp:90-95."""
    return _raster1(img, "cityblock")


def cityblock_separable(img, threads=1):
    """cityblock_separable -- propagation.cpp:97-102 (identical map)."""
    return _raster1(img, "cityblock")


def chamfer34(img):
    """chamfer34 -- propagation.cpp:104-109."""
    return _raster1(img, "chamfer34")


def chessboard(img):
    """Chessboard map; the reference has only oracle::chessboard (tests/oracles.hpp:52-55)."""
    return _raster1(img, "chessboard")


def danielsson(img, first_sweep=False):
    """danielsson / danielsson_first_sweep -- vector_dt.cpp:108-124: (squared
    lengths uint64 with kInfinity, dy uint32, dx uint32 with Offset::kUnset =
    0xFFFFFFFF), the sweeps on the GPU."""
    o = _danielsson(_to_device(img), first_sweep=first_sweep)
    torch.cuda.synchronize()
    return (o["sqdist"].cpu().numpy().view(np.uint64), o["dy"].cpu().numpy().view(np.uint32),
            o["dx"].cpu().numpy().view(np.uint32))

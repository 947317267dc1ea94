"""distfield-b200: B200-native exact distance transforms (Strutz, arXiv 2106.03503).

Python host mirror of the reference ``distfield`` hot path
(/root/reference/proj/core/include/distfield/{exact_edt,propagation}.hpp) over
the C ABI in ``include/distfield_cuda.h`` (``lib/libdfc.so``, hand-written
sm_100a CUDA).  Two layers:

* device layer (``edt``, ``edt_dual``, ``edt_batched``, ``vertical``,
  ``raster``, ``label_ordinals``): torch CUDA tensors in and out, int32 maps
  with ``INF_I32`` as the infinity marker, stream-ordered, no host sync;
* reference-shaped host layer in :mod:`paper_2106_03503_b200.distfield`
  (``edt``, ``voronoi_labels``, ``meijster_scan``, ``vertical_pass``,
  ``cityblock_sequential``, ``chamfer34``, ``chessboard``): numpy uint8 image
  in, reference-typed numpy maps out (uint64 with ``2**64-1`` infinity,
  uint32 ordinal labels), same exceptions as the reference.

There is no CPU fallback: importing this package without the built CUDA
library raises, and every call needs a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DFC_LIB") or os.path.join(HERE, "lib", "libdfc.so")  # DFC_LIB: A/B builds
INF_I32 = 0x7FFFFFFF

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a library first "
        "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2106_03503_b200/csrc)")

_lib = C.CDLL(LIB_PATH)
_i64 = C.c_int64
_vp = C.c_void_p
_lib.dfc_edt_u8.argtypes = [_vp, _i64, _i64, _i64, C.c_int, _vp, _vp, _vp, _vp, _vp]
_lib.dfc_edt_u8_dual.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp]
_lib.dfc_edt_u8_batched.argtypes = [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp]
_lib.dfc_vertical_u8.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp]
_lib.dfc_vertical_down_pass_u64.argtypes = [_vp, _i64, _i64, _i64, _vp]
_lib.dfc_vertical_up_pass_u64.argtypes = [_vp, _i64, _i64, _i64, _vp]
_lib.dfc_raster_u8.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp]
_lib.dfc_label_ordinals.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp, _vp]
_lib.dfc_status_string.restype = C.c_char_p
_lib.dfc_status_string.argtypes = [C.c_int]
_lib.dfc_version.restype = C.c_char_p
_lib.dfc_last_launch_count.restype = C.c_int
_lib.dfc_last_cuda_error.restype = C.c_int
_lib.dfc_set_profile_events.argtypes = [_vp, _vp, _vp]
_lib.dfc_sqrt_i32.argtypes = [_vp, _vp, _i64, _vp]
_lib.dfc_set_row_kernel.argtypes = [C.c_int]
_lib.dfc_set_lr_chunk.argtypes = [C.c_int]
_lib.dfc_set_band_min_pixels.argtypes = [_i64]
_lib.dfc_column_nr_u8.argtypes = [_vp, _i64, _i64, _i64, C.c_int, _vp, _i64, _vp]
_lib.dfc_rows_from_nr_u16.argtypes = [_vp, _i64, _i64, _i64, _i64, _i64, C.c_int, _vp, _vp, _vp, _vp, _vp]
_lib.dfc_envelope_vdist_u16.argtypes = [_vp, _i64, _i64, _i64, C.c_int, _vp, _vp, _vp, _vp]
_lib.dfc_unpack_pbm.argtypes = [_vp, _i64, _i64, _i64, C.c_int, _vp, _i64, _vp]
_lib.dfc_binarize_u8.argtypes = [_vp, _i64, _i64, _i64, C.c_int, _vp, _i64, _vp]
_lib.dfc_count_objects_u8.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp]
_lib.dfc_gray_i32.argtypes = [_vp, _i64, C.c_int, _vp, _vp, _vp, _vp]
_lib.dfc_labels_gray.argtypes = [_vp, _i64, _i64, _vp, _vp]
_lib.dfc_row_owners_i64.argtypes = [_vp, _i64, _i64, _i64, _i64, C.c_int, _vp, _vp, _vp]
_lib.dfc_raster_pass_u64.argtypes = [_vp, _i64, _i64, _i64, C.c_int, _vp]
_lib.dfc_danielsson_u8.argtypes = [_vp, _i64, _i64, _i64, _i64, _i64, C.c_int, _vp, _vp, _vp, _vp]


class Shard(C.Structure):
    """struct dfc_shard (include/distfield_cuda.h): one local rank of dfc_edt_u8_sharded."""
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("d_img", _vp), ("pitch_bytes", _i64),
                ("d_sqdist", _vp), ("d_dist", _vp), ("d_label", _vp), ("comm", _vp), ("stream", _vp)]


_lib.dfc_edt_u8_sharded.argtypes = [C.POINTER(Shard), C.c_int, C.c_int, _i64, _i64, C.c_int]
_lib.dfc_shard_cols.argtypes = [_i64, C.c_int, C.c_int, C.POINTER(_i64), C.POINTER(_i64)]
_lib.dfc_shard_rows.argtypes = [_i64, C.c_int, C.c_int, C.POINTER(_i64), C.POINTER(_i64)]
_lib.dfc_comm_unique_id.argtypes = [C.c_char_p]
_lib.dfc_comm_init_rank.argtypes = [C.POINTER(_vp), C.c_int, C.c_int, C.c_char_p]
_lib.dfc_comm_init_all.argtypes = [C.POINTER(_vp), C.c_int, C.POINTER(C.c_int)]
_lib.dfc_comm_destroy.argtypes = [_vp]
_lib.dfc_last_nccl_error.restype = C.c_int

EXPORTED_SYMBOLS = (
    "dfc_edt_u8", "dfc_edt_u8_dual", "dfc_edt_u8_batched", "dfc_vertical_u8", "dfc_raster_u8",
    "dfc_vertical_down_pass_u64", "dfc_vertical_up_pass_u64",
    "dfc_label_ordinals", "dfc_last_launch_count", "dfc_status_string", "dfc_last_cuda_error",
    "dfc_version", "dfc_set_profile_events", "dfc_sqrt_i32", "dfc_envelope_vdist_u16", "dfc_column_nr_u8", "dfc_rows_from_nr_u16", "dfc_set_row_kernel", "dfc_set_lr_chunk",
    "dfc_unpack_pbm", "dfc_binarize_u8", "dfc_count_objects_u8", "dfc_gray_i32", "dfc_labels_gray",
    "dfc_edt_u8_sharded", "dfc_shard_cols", "dfc_shard_rows", "dfc_comm_unique_id", "dfc_comm_init_rank",
    "dfc_comm_init_all", "dfc_comm_destroy", "dfc_last_nccl_error", "dfc_row_owners_i64", "dfc_raster_pass_u64",
    "dfc_set_band_min_pixels", "dfc_debug_guard_violations", "dfc_danielsson_u8",
)


class DfcError(RuntimeError):
    def __init__(self, status: int):
        msg = _lib.dfc_status_string(status).decode()
        if status == 3:
            msg += f" (cudaError {_lib.dfc_last_cuda_error()})"
        if status == 4:
            msg += f" (ncclResult {_lib.dfc_last_nccl_error()})"
        super().__init__(msg)
        self.status = status


_tls = threading.local()


def _check(status: int) -> None:
    # a launch on a side stream (see _stream): the current stream, on which this
    # layer allocates outputs and temporaries, waits for it, so the caching
    # allocator cannot hand their memory out again while the kernels still run
    side = getattr(_tls, "side", None)
    if side is not None:
        _tls.side = None
        side[1].wait_stream(side[0])
    if status != 0:
        raise DfcError(status)


def version() -> str:
    return _lib.dfc_version().decode()


def set_profile_events(col_begin=None, row_begin=None, row_end=None) -> None:
    """Record torch.cuda.Event objects around the column / row pass of the next
    edt* calls on this thread (measurement hook for bench.py); None disables."""
    h = lambda e: None if e is None else C.c_void_p(e.cuda_event)
    _check(_lib.dfc_set_profile_events(h(col_begin), h(row_begin), h(row_end)))


def set_lr_chunk(cols: int) -> None:
    """Columns per warp chunk of the "lr" row kernel (multiple of 32; 0 = default)."""
    _check(_lib.dfc_set_lr_chunk(int(cols)))


def set_band_min_pixels(pixels: int) -> None:
    """Smallest image whose sparse planes take the band path (0: every size,
    negative: the library default, 2**24 + 1); see dfc_set_band_min_pixels."""
    _check(_lib.dfc_set_band_min_pixels(int(pixels)))


def set_row_kernel(mode: str) -> None:
    """Stage-2 kernel for this thread's calls: "default" (= "anc" unless
    DFC_ROWS says otherwise), "segment" (the merge-tree kernel k_rows for
    every row), "dense" (point planes, dense rows, sparse planes, k_rows for
    the rest), "lr" (k_rows_lr.cu, lane-per-row chunk scan for every row) or
    "anc" (point planes, sparse planes by the band path, k_rows_anc.cu for the
    rest).  Results are identical in every mode."""
    _check(_lib.dfc_set_row_kernel({"default": 0, "segment": 1, "dense": 4, "lr": 5, "anc": 6}[mode]))


def last_launch_count() -> int:
    """Kernels enqueued by the last successful call on this thread."""
    return _lib.dfc_last_launch_count()


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    """The launch stream's handle.  A side stream first waits for the current
    stream (inputs, outputs and temporaries are produced / allocated there);
    _check() then makes the current stream wait for the launch."""
    cur = torch.cuda.current_stream()
    if stream is None or stream == cur:
        _tls.side = None
        return C.c_void_p(cur.cuda_stream)
    stream.wait_stream(cur)
    _tls.side = (stream, cur)
    return C.c_void_p(stream.cuda_stream)


def _img2d(img: torch.Tensor):
    if not img.is_cuda:
        raise ValueError("device layer expects a CUDA tensor; use paper_2106_03503_b200.distfield for host arrays")
    if img.dtype not in (torch.uint8, torch.bool) or img.dim() != 2:
        raise ValueError("image must be a 2-D uint8 (or bool) CUDA tensor")
    if img.dtype == torch.bool:
        img = img.view(torch.uint8)
    if img.stride(1) != 1:
        img = img.contiguous()
    return img, img.shape[0], img.shape[1], img.stride(0)


# DFC_DEBUG_GUARD=1 (debug, see include/distfield_cuda.h): outputs this layer
# allocates sit between two 4 KiB canary zones (0x5A bytes, interior poisoned
# alike); check_guards() verifies them together with the library's scratch
# canaries.  The stand-in for compute-sanitizer where that tool cannot run.
_GUARD = os.environ.get("DFC_DEBUG_GUARD") == "1"
_GUARD_PAD = 4096
_guarded = []
_lib.dfc_debug_guard_violations.restype = C.c_longlong


def _empty(shape, dtype, like):
    if not _GUARD:
        return torch.empty(shape, dtype=dtype, device=like.device)
    n = 1
    for d in shape:
        n *= int(d)
    nbytes = n * torch.empty((), dtype=dtype).element_size()
    buf = torch.full((nbytes + 2 * _GUARD_PAD,), 0x5A, dtype=torch.uint8, device=like.device)
    _guarded.append((buf, nbytes))
    return buf[_GUARD_PAD:_GUARD_PAD + nbytes].view(dtype).view(shape)


def check_guards() -> int:
    """Debug (DFC_DEBUG_GUARD=1): raise if any kernel wrote outside an output
    this layer allocated or outside a scratch allocation of the library;
    returns the number of output buffers checked."""
    if not _GUARD:
        raise RuntimeError("DFC_DEBUG_GUARD=1 is not set")
    torch.cuda.synchronize()
    for buf, nbytes in _guarded:
        lo, hi = buf[:_GUARD_PAD], buf[_GUARD_PAD + nbytes:]
        if not (bool((lo == 0x5A).all()) and bool((hi == 0x5A).all())):
            raise AssertionError("a kernel wrote outside an output buffer (canary zone changed)")
    n = len(_guarded)
    _guarded.clear()
    bad = _lib.dfc_debug_guard_violations()
    if bad != 0:
        raise AssertionError(f"scratch canary zones: {bad} bytes overwritten")
    return n


def edt(img: torch.Tensor, polarity: int = 0, dist: bool = True, label: bool = False,
        nearest_col: bool = False, stream=None, out=None):
    """Exact squared EDT of one image (``edt(img, envelope)``, exact_edt.cpp:285-317).

    polarity 0: background -> nearest object (the reference ``edt(img)``);
    polarity 1: object -> nearest background (``edt(img.inverted())``).
    Returns a dict with int32 ``sqdist`` and optionally float32 ``dist``,
    int32 ``label`` (linear index, voronoi_labels tie rule) and int32
    ``nearest_col`` (meijster_scan's take_new rule)."""
    img, h, w, pitch = _img2d(img)
    o = dict(out or {})
    o.setdefault("sqdist", _empty((h, w), torch.int32, img))
    if dist:
        o.setdefault("dist", _empty((h, w), torch.float32, img))
    if label:
        o.setdefault("label", _empty((h, w), torch.int32, img))
    if nearest_col:
        o.setdefault("nearest_col", _empty((h, w), torch.int32, img))
    _check(_lib.dfc_edt_u8(_ptr(img), h, w, pitch, polarity, _ptr(o["sqdist"]), _ptr(o.get("dist")),
                           _ptr(o.get("label")), _ptr(o.get("nearest_col")), _stream(stream)))
    return o


def edt_dual(img: torch.Tensor, dist: bool = True, stream=None, out=None):
    """Both polarities from one input read (config 2): keys sqdist_bg, dist_bg,
    sqdist_obj, dist_obj."""
    img, h, w, pitch = _img2d(img)
    o = dict(out or {})
    for k in ("sqdist_bg", "sqdist_obj"):
        o.setdefault(k, _empty((h, w), torch.int32, img))
    if dist:
        for k in ("dist_bg", "dist_obj"):
            o.setdefault(k, _empty((h, w), torch.float32, img))
    _check(_lib.dfc_edt_u8_dual(_ptr(img), h, w, pitch, _ptr(o["sqdist_bg"]), _ptr(o.get("dist_bg")),
                                _ptr(o["sqdist_obj"]), _ptr(o.get("dist_obj")), _stream(stream)))
    return o


def edt_batched(imgs: torch.Tensor, dist: bool = False, label: bool = True, stream=None, out=None):
    """A batch [n, rows, cols] of images (config 3): int32 sqdist and labels
    (linear index within each image, -1 for a featureless image)."""
    if not imgs.is_cuda or imgs.dim() != 3 or imgs.dtype not in (torch.uint8, torch.bool):
        raise ValueError("batch must be a 3-D uint8 CUDA tensor [n, rows, cols]")
    if imgs.dtype == torch.bool:
        imgs = imgs.view(torch.uint8)
    if imgs.stride(2) != 1:
        imgs = imgs.contiguous()
    n, h, w = imgs.shape
    o = dict(out or {})
    o.setdefault("sqdist", _empty((n, h, w), torch.int32, imgs))
    if dist:
        o.setdefault("dist", _empty((n, h, w), torch.float32, imgs))
    if label:
        o.setdefault("label", _empty((n, h, w), torch.int32, imgs))
    _check(_lib.dfc_edt_u8_batched(_ptr(imgs), n, h, w, imgs.stride(1), imgs.stride(0),
                                   _ptr(o["sqdist"]), _ptr(o.get("dist")), _ptr(o.get("label")),
                                   _stream(stream)))
    return o


def vertical(img: torch.Tensor, stream=None) -> torch.Tensor:
    """Stage one alone (vertical_pass, exact_edt.cpp:112-117): int32 squared
    vertical distance, INF_I32 in featureless columns."""
    img, h, w, pitch = _img2d(img)
    out = _empty((h, w), torch.int32, img)
    _check(_lib.dfc_vertical_u8(_ptr(img), h, w, pitch, _ptr(out), _stream(stream)))
    return out


def vertical_down_pass(dm: torch.Tensor, stream=None) -> torch.Tensor:
    """vertical_down_pass (exact_edt.cpp:74-91) IN PLACE on a 2-D int64 tensor
    holding uint64 cells (bit pattern; -1 = kInfinity).  Returns dm."""
    _vpass(dm, _lib.dfc_vertical_down_pass_u64, stream)
    return dm


def vertical_up_pass(dm: torch.Tensor, stream=None) -> torch.Tensor:
    """vertical_up_pass (exact_edt.cpp:93-110) IN PLACE, as vertical_down_pass."""
    _vpass(dm, _lib.dfc_vertical_up_pass_u64, stream)
    return dm


def _vpass(dm, fn, stream):
    if not dm.is_cuda or dm.dim() != 2 or dm.dtype not in (torch.int64, torch.uint64) or dm.stride(1) != 1:
        raise ValueError("expected a 2-D CUDA int64/uint64 tensor with unit column stride")
    _check(fn(_ptr(dm), dm.shape[0], dm.shape[1], dm.stride(0), _stream(stream)))


def raster(img: torch.Tensor, cityblock: bool = True, chessboard: bool = True,
           chamfer34: bool = True, stream=None, out=None):
    """City-block / chessboard / chamfer-3-4 maps (config 4), int32, bit-exact
    with the reference raster scans (propagation.cpp:90-109)."""
    img, h, w, pitch = _img2d(img)
    o = dict(out or {})
    for key, want in (("cityblock", cityblock), ("chessboard", chessboard), ("chamfer34", chamfer34)):
        if want:
            o.setdefault(key, _empty((h, w), torch.int32, img))
    _check(_lib.dfc_raster_u8(_ptr(img), h, w, pitch, _ptr(o.get("cityblock")),
                              _ptr(o.get("chessboard")), _ptr(o.get("chamfer34")), _stream(stream)))
    return o


def column_nr(img: torch.Tensor, polarity: int = 0, out: torch.Tensor = None, stream=None) -> torch.Tensor:
    """Stage one as an int16 tensor of nearest object rows (uint16 bits, -1 = none),
    shape [rows, round_up(cols, 4)]."""
    img, h, w, pitch = _img2d(img)
    wp = (w + 3) // 4 * 4
    if out is None:
        out = torch.empty((h, wp), dtype=torch.int16, device=img.device)
    _check(_lib.dfc_column_nr_u8(_ptr(img), h, w, pitch, polarity, _ptr(out), out.stride(0), _stream(stream)))
    return out


def rows_from_nr(nr: torch.Tensor, rows: int, cols: int, row0: int = 0, tile_cols: int = None,
                 tile_stride: int = 0, dist: bool = False, label: bool = False, stream=None, out=None):
    """Stage two from a (possibly column-tiled) int16 nearest-row buffer; see
    dfc_rows_from_nr_u16.  Returns int32 sqdist (+ float dist, int32 label)."""
    o = dict(out or {})
    o.setdefault("sqdist", torch.empty((rows, cols), dtype=torch.int32, device=nr.device))
    if dist:
        o.setdefault("dist", torch.empty((rows, cols), dtype=torch.float32, device=nr.device))
    if label:
        o.setdefault("label", torch.empty((rows, cols), dtype=torch.int32, device=nr.device))
    tc = tile_cols if tile_cols is not None else nr.stride(0)
    _check(_lib.dfc_rows_from_nr_u16(_ptr(nr), rows, cols, row0, tc, tile_stride, 0, _ptr(o["sqdist"]),
                                     _ptr(o.get("dist")), _ptr(o.get("label")), None, _stream(stream)))
    return o


def envelope_vdist(vdist: torch.Tensor, take_new: bool = True, dist: bool = False, stream=None):
    """Stage two from a uint16 vertical-distance plane (0xFFFF = no feature):
    meijster_scan(vert) for vert = a^2 (exact_edt.cpp:272-283)."""
    if vdist.dtype != torch.int16 and vdist.dtype != torch.uint16:
        raise ValueError("vdist must be a 16-bit CUDA tensor")
    h, w = vdist.shape
    if vdist.stride(1) != 1 or vdist.stride(0) % 2 or vdist.data_ptr() % 4:
        padded = torch.full((h, w + (w & 1)), -1, dtype=torch.int16, device=vdist.device)
        padded[:, :w] = vdist.view(torch.int16)
        vdist = padded[:, :w]
    o = {"sqdist": _empty((h, w), torch.int32, vdist), "nearest_col": _empty((h, w), torch.int32, vdist)}
    if dist:
        o["dist"] = _empty((h, w), torch.float32, vdist)
    _check(_lib.dfc_envelope_vdist_u16(_ptr(vdist), h, w, vdist.stride(0), 1 if take_new else 0,
                                       _ptr(o["sqdist"]), _ptr(o.get("dist")), _ptr(o["nearest_col"]),
                                       _stream(stream)))
    return o


def sqrt_i32(sq: torch.Tensor, stream=None) -> torch.Tensor:
    """float32 (float)sqrt((double)D) of an int32 squared map (INF_I32 -> +inf)."""
    sq = sq.contiguous()
    out = torch.empty(sq.shape, dtype=torch.float32, device=sq.device)
    _check(_lib.dfc_sqrt_i32(_ptr(sq), _ptr(out), sq.numel(), _stream(stream)))
    return out


def unpack_pbm(bits: torch.Tensor, rows: int, cols: int, invert: bool = False, stream=None) -> torch.Tensor:
    """uint8 0/1 image [rows, cols] from a device P4 raster (uint8, rows * ceil(cols/8)
    bytes, MSB first, bit 1 = object; netpbm.cpp:81-95), optionally inverted."""
    bits = bits.contiguous()
    rb = (cols + 7) // 8
    if bits.numel() < rows * rb:
        raise ValueError("P4 raster too short")
    out = torch.empty((rows, cols), dtype=torch.uint8, device=bits.device)
    _check(_lib.dfc_unpack_pbm(_ptr(bits), rows, cols, rb, int(invert), _ptr(out), cols, _stream(stream)))
    return out


def binarize(img: torch.Tensor, invert: bool = False, stream=None) -> torch.Tensor:
    """0/1 uint8 copy of an image (object = nonzero), optionally inverted."""
    img, h, w, pitch = _img2d(img)
    out = torch.empty((h, w), dtype=torch.uint8, device=img.device)
    _check(_lib.dfc_binarize_u8(_ptr(img), h, w, pitch, int(invert), _ptr(out), w, _stream(stream)))
    return out


def count_objects(img: torch.Tensor, stream=None) -> torch.Tensor:
    """Device int64 scalar: object pixels of the image (BinaryImage::object_count)."""
    img, h, w, pitch = _img2d(img)
    cnt = torch.zeros((), dtype=torch.int64, device=img.device)
    _check(_lib.dfc_count_objects_u8(_ptr(img), h, w, pitch, _ptr(cnt), _stream(stream)))
    return cnt


def gray(dmap: torch.Tensor, sqrt_mode: bool = False, stream=None):
    """to_gray (grid.cpp:93-110) of an int32 map -> (uint8 map, device int32 max;
    -1 = no finite value, where the reference throws domain_error)."""
    dmap = dmap.contiguous()
    out = torch.empty(dmap.shape, dtype=torch.uint8, device=dmap.device)
    mx = torch.empty((), dtype=torch.int32, device=dmap.device)
    scratch = torch.empty((), dtype=torch.int32, device=dmap.device)
    _check(_lib.dfc_gray_i32(_ptr(dmap), dmap.numel(), int(sqrt_mode), _ptr(out), _ptr(mx), _ptr(scratch),
                             _stream(stream)))
    return out, mx


def labels_gray(ordinal: torch.Tensor, feature_count: int, stream=None) -> torch.Tensor:
    """labels_to_gray (grid.cpp:112-121) of uint32 ordinals (int32/int64 tensor)."""
    o = ordinal.to(torch.int32).contiguous()
    out = torch.empty(o.shape, dtype=torch.uint8, device=o.device)
    _check(_lib.dfc_labels_gray(_ptr(o), o.numel(), int(feature_count), _ptr(out), _stream(stream)))
    return out


def label_ordinals(img: torch.Tensor, label: torch.Tensor, stream=None) -> torch.Tensor:
    """Linear-index labels -> the reference LabelMap feature ordinals
    (grid.cpp:29-36); int64 tensor holding uint32 values (2**32-1 = none)."""
    img, h, w, pitch = _img2d(img)
    out = _empty((h, w), torch.int32, img)
    lab = label.contiguous()  # kept alive until the launch is ordered (see _check)
    _check(_lib.dfc_label_ordinals(_ptr(img), h, w, pitch, _ptr(lab), _ptr(out), _stream(stream)))
    return out.to(torch.int64) & 0xFFFFFFFF


def row_owners(vert: torch.Tensor, lmax: int, take_new: bool = True, stream=None):
    """build_row_envelope / envelope_rows over arbitrary int64 rows
    (exact_edt.cpp:190-283): (owner int32, value int64) per column; see
    dfc_row_owners_i64."""
    if not vert.is_cuda or vert.dtype != torch.int64 or vert.dim() != 2 or vert.stride(1) != 1:
        raise ValueError("vert must be a 2-D int64 CUDA tensor with unit column stride")
    r, c = vert.shape
    own = torch.empty((r, c), dtype=torch.int32, device=vert.device)
    val = torch.empty((r, c), dtype=torch.int64, device=vert.device)
    _check(_lib.dfc_row_owners_i64(_ptr(vert), r, c, vert.stride(0), int(lmax), int(take_new), _ptr(own),
                                   _ptr(val), _stream(stream)))
    return own, val


RASTER_PASSES = ("cityblock_forward_pass", "cityblock_backward_pass", "cityblock_vertical_passes",
                 "cityblock_horizontal_passes", "chamfer_forward_pass", "chamfer_backward_pass")


def raster_pass(dm: torch.Tensor, which, stream=None) -> torch.Tensor:
    """One per-pass in-place function (propagation.hpp:15-26) on a 2-D int64
    CUDA tensor holding uint64 cells (-1 = kInfinity); `which` is a name of
    RASTER_PASSES or its index.  Returns dm."""
    k = RASTER_PASSES.index(which) if isinstance(which, str) else int(which)
    if not dm.is_cuda or dm.dim() != 2 or dm.dtype not in (torch.int64, torch.uint64) or dm.stride(1) != 1:
        raise ValueError("expected a 2-D CUDA int64/uint64 tensor with unit column stride")
    _check(_lib.dfc_raster_pass_u64(_ptr(dm), dm.shape[0], dm.shape[1], dm.stride(0), k, _stream(stream)))
    return dm


# ---------------------------------------------------------- multi-GPU (config 5)
def danielsson(img: torch.Tensor, first_sweep: bool = False, stream=None):
    """Danielsson's vector transform (vector_dt.cpp:108-124) of one image [H, W]
    or a batch [n, H, W] (uint8 CUDA tensor): {"sqdist": int64 holding the
    reference's uint64 values (-1 = infinity), "dy", "dx": int32 holding uint32
    offset magnitudes (-1 = unset)}; see dfc_danielsson_u8."""
    if not img.is_cuda or img.dtype not in (torch.uint8, torch.bool) or img.dim() not in (2, 3):
        raise ValueError("image must be a 2-D or 3-D uint8 (or bool) CUDA tensor")
    if img.dtype == torch.bool:
        img = img.view(torch.uint8)
    if img.stride(-1) != 1:
        img = img.contiguous()
    batch = img.dim() == 3
    n = img.shape[0] if batch else 1
    h, w = img.shape[-2], img.shape[-1]
    o = {"sqdist": _empty(tuple(img.shape), torch.int64, img), "dy": _empty(tuple(img.shape), torch.int32, img),
         "dx": _empty(tuple(img.shape), torch.int32, img)}
    _check(_lib.dfc_danielsson_u8(_ptr(img), n, h, w, img.stride(-2), img.stride(0) if batch else 0,
                                  int(first_sweep), _ptr(o["sqdist"]), _ptr(o["dy"]), _ptr(o["dx"]), _stream(stream)))
    return o


def shard_cols(cols: int, world: int, rank: int):
    """[col0, col0 + ncols): the column stripe rank `rank` holds (dfc_shard_cols)."""
    a, b = _i64(), _i64()
    _check(_lib.dfc_shard_cols(cols, world, rank, C.byref(a), C.byref(b)))
    return a.value, a.value + b.value


def shard_rows(rows: int, world: int, rank: int):
    """[row0, row1): the row stripe of the result rank `rank` gets (whole 32-row bands)."""
    a, b = _i64(), _i64()
    _check(_lib.dfc_shard_rows(rows, world, rank, C.byref(a), C.byref(b)))
    return a.value, a.value + b.value


def comm_unique_id() -> bytes:
    """A 128-byte NCCL unique id (rank 0 makes it; the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    _check(_lib.dfc_comm_unique_id(buf))
    return buf.raw


def comm_init_rank(world: int, rank: int, uid: bytes) -> int:
    """This rank's NCCL communicator on the current CUDA device (opaque handle)."""
    h = _vp()
    _check(_lib.dfc_comm_init_rank(C.byref(h), world, rank, uid))
    return h.value


def comm_destroy(handle: int) -> None:
    _check(_lib.dfc_comm_destroy(handle))


def edt_sharded(shards, world: int, rows: int, cols: int, polarity: int = 0) -> None:
    """dfc_edt_u8_sharded over local ranks.  `shards`: dicts with keys rank,
    img (CUDA uint8 [rows, ncols] column stripe), sqdist (CUDA int32 [nrows, cols]
    row stripe), optional dist / label, comm (handle or None), stream."""
    arr = (Shard * len(shards))()
    for s, d in zip(arr, shards):
        img, _, _, pitch = _img2d(d["img"])
        s.device = img.device.index
        s.rank = d["rank"]
        s.d_img = img.data_ptr()
        s.pitch_bytes = pitch
        s.d_sqdist = d["sqdist"].data_ptr()
        s.d_dist = d["dist"].data_ptr() if d.get("dist") is not None else None
        s.d_label = d["label"].data_ptr() if d.get("label") is not None else None
        s.comm = d.get("comm")
        st = d.get("stream") or torch.cuda.current_stream(img.device)
        s.stream = st.cuda_stream
    _check(_lib.dfc_edt_u8_sharded(arr, len(shards), world, rows, cols, polarity))


from . import distfield  # noqa: E402,F401  (reference-shaped host API)

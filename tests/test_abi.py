"""CPU checks of the boundary: the C-ABI library and the C++ drop-in load and
export every symbol include/distfield_cuda.h declares (no compute without a GPU)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2106_03503_b200", "lib")


def _declared():
    src = open(os.path.join(ROOT, "include", "distfield_cuda.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|long long|const char\*|size_t)\s+(dfc_\w+)\s*\(", src, re.M)))


def _exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_c_abi_exports_every_declared_symbol():
    decl = _declared()
    assert len(decl) >= 12
    exp = _exported(os.path.join(LIB, "libdfc.so"))
    missing = [s for s in decl if s not in exp]
    assert not missing, missing
    lib = ctypes.CDLL(os.path.join(LIB, "libdfc.so"))
    for s in decl:
        assert getattr(lib, s)
    lib.dfc_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.dfc_version()
    lib.dfc_status_string.restype = ctypes.c_char_p
    assert lib.dfc_status_string(5) == b"no features: voronoi labels undefined"


def test_python_mirror_lists_every_symbol():
    import paper_2106_03503_b200 as dfc
    assert sorted(dfc.EXPORTED_SYMBOLS) == _declared()


def test_dropin_library_exports_reference_entry_points():
    exp = _exported(os.path.join(LIB, "libdistfield_b200.so"))
    demangled = subprocess.run(["c++filt"], input="\n".join(exp), capture_output=True, text=True).stdout
    for name in ("distfield::edt(", "distfield::vertical_pass(", "distfield::meijster_scan(",
                 "distfield::meijster_row_envelope(", "distfield::voronoi_labels(",
                 "distfield::cityblock_sequential(", "distfield::cityblock_separable(", "distfield::chamfer34(",
                 "distfield::chessboard(", "distfield::generate_random_image(", "distfield::kind_bound(",
                 "distfield::init_distance_map("):
        assert name in demangled, name
    ctypes.CDLL(os.path.join(LIB, "libdistfield_b200.so"))  # loads (rpath to libdfc, cudart)


def test_product_fails_loudly_without_library(tmp_path):
    """The product path has no CPU fallback: without lib/libdfc.so the import raises."""
    import shutil
    import sys
    pkg = tmp_path / "paper_2106_03503_b200"
    shutil.copytree(os.path.join(ROOT, "paper_2106_03503_b200"), pkg,
                    ignore=shutil.ignore_patterns("lib", "csrc", "cpp"))
    code = "import paper_2106_03503_b200"
    p = subprocess.run([sys.executable, "-c", code], cwd=tmp_path, capture_output=True, text=True)
    assert p.returncode != 0 and "libdfc.so is missing" in p.stderr

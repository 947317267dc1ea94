"""Regenerate the committed golden fixtures from the REFERENCE (run in the build
container only -- it needs /root/reference; the GPU box only reads the output).

Outputs (committed):
  six_point.json   every frozen matrix of proj/tests/goldens.hpp (six-point 9x10
                   sample: vertical down/final, squared euclidean, city-block
                   forward/vertical/final, chamfer forward/final, row-0 envelope
                   bookkeeping), dumped by compiling a tiny program against
                   goldens.hpp.  -1 = infinity, as in goldens.hpp:26.
  random_cases.npz seeded images run through the reference library itself
                   (oracle/_ref/libdfref.so): edt (uint64), meijster_scan
                   nearest_col, voronoi_labels ordinals, cityblock_sequential,
                   chamfer34, and oracle::chessboard (brute force, via the
                   reference test oracle header).

Usage:  python tests/golden/make_golden.py
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/proj"

DUMP_CPP = r"""
#include <cstdio>
#include "goldens.hpp"
template <typename M> void dump(const char* name, const M& m, bool& first) {
    std::printf("%s\"%s\": [", first ? "" : ",\n", name); first = false;
    for (std::size_t i = 0; i < m.size(); ++i) {
        std::printf("%s[", i ? "," : "");
        for (std::size_t j = 0; j < m[i].size(); ++j) std::printf("%s%lld", j ? "," : "", (long long)m[i][j]);
        std::printf("]");
    }
    std::printf("]");
}
template <typename A> void dump1(const char* name, const A& a, bool& first) {
    std::printf("%s\"%s\": [", first ? "" : ",\n", name); first = false;
    for (std::size_t i = 0; i < a.size(); ++i) std::printf("%s%lld", i ? "," : "", (long long)a[i]);
    std::printf("]");
}
int main() {
    bool first = true;
    std::printf("{\n");
    std::printf("\"rows\": %zu, \"cols\": %zu,\n", golden::kRows6, golden::kCols6);
    std::printf("\"points\": [");
    for (std::size_t t = 0; t < golden::kSixPoints.size(); ++t)
        std::printf("%s[%zu,%zu]", t ? "," : "", golden::kSixPoints[t].row, golden::kSixPoints[t].col);
    std::printf("],\n");
    dump("kCityblockForward", golden::kCityblockForward, first);
    dump("kCityblockFinal", golden::kCityblockFinal, first);
    dump("kCityblockVertical", golden::kCityblockVertical, first);
    dump("kChamferForward", golden::kChamferForward, first);
    dump("kChamferFinal", golden::kChamferFinal, first);
    dump("kVerticalDown", golden::kVerticalDown, first);
    dump("kVerticalFinal", golden::kVerticalFinal, first);
    dump("kSquaredEuclidean", golden::kSquaredEuclidean, first);
    dump1("kRow0Ks", golden::kRow0Ks, first);
    dump1("kRow0Js", golden::kRow0Js, first);
    dump1("kRow0Distances", golden::kRow0Distances, first);
    std::printf("\n}\n");
}
"""

CHESS_CPP = r"""
#include <cstdio>
#include <cstdint>
#include <vector>
#include "oracles.hpp"
// stdin: rows cols then rows*cols bytes (0/1 as text); stdout: oracle::chessboard values
int main() {
    std::size_t r, c; if (std::scanf("%zu %zu", &r, &c) != 2) return 1;
    distfield::BinaryImage img(r, c);
    for (std::size_t i = 0; i < r; ++i) for (std::size_t j = 0; j < c; ++j) {
        int v; std::scanf("%d", &v); if (v) img.set_object(i, j); }
    const auto dm = oracle::chessboard(img);
    for (std::size_t i = 0; i < r; ++i) for (std::size_t j = 0; j < c; ++j)
        std::printf("%llu\n", (unsigned long long)dm(i, j));
}
"""


def _compile(src, name, tmp):
    path = os.path.join(tmp, name + ".cpp")
    with open(path, "w") as f:
        f.write(src)
    exe = os.path.join(tmp, name)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", f"{REF}/core/include", "-I", f"{REF}/tests",
                    path, f"{REF}/core/src/grid.cpp", "-o", exe], check=True)
    return exe


def main():
    sys.path.insert(0, ROOT)
    import oracle  # noqa: E402  (test infrastructure)
    oracle.build()
    assert oracle.ref_available(), "oracle/_ref/libdfref.so missing"
    with tempfile.TemporaryDirectory() as tmp:
        exe = _compile(DUMP_CPP, "dump", tmp)
        js = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
        data = json.loads(js)
        data["_source"] = "proj/tests/goldens.hpp (dumped by tests/golden/make_golden.py)"
        with open(os.path.join(HERE, "six_point.json"), "w") as f:
            json.dump(data, f)
        chess = _compile(CHESS_CPP, "chess", tmp)

        # Seeded random cases: acceptance c3 shapes x densities (acceptance.cpp:141-150),
        # degenerate shapes (test_exact_edt.cpp:223-227) and a few wide/tall rows.
        cases = []
        seed = 7000
        shapes = [(16, 16), (64, 64), (33, 97), (1, 1), (1, 37), (41, 1), (5, 7), (3, 200),
                  (200, 3), (48, 48), (9, 10), (128, 160)]
        for (r, c) in shapes:
            for dens in (0.0, 0.001, 0.02, 0.5, 1.0):
                seed += 1
                cases.append((r, c, dens, seed))
        arrays = {}
        for n, (r, c, dens, s) in enumerate(cases):
            img = oracle.ref_random_image(r, c, dens, s)
            d = oracle.ref_edt(img)
            dm, ncol = oracle.ref_meijster_scan(img)
            assert (dm == d).all()
            lab = oracle.ref_voronoi_labels(img)
            city = oracle.ref_propagation(img, 0)
            cham = oracle.ref_propagation(img, 2)
            txt = f"{r} {c}\n" + " ".join(str(int(v)) for v in img.ravel()) + "\n"
            out = subprocess.run([chess], input=txt, check=True, capture_output=True, text=True).stdout
            cb = np.array([int(x) for x in out.split()], dtype=np.uint64).reshape(r, c)
            arrays[f"c{n}_meta"] = np.array([r, c, s], np.int64)
            arrays[f"c{n}_density"] = np.array([dens])
            arrays[f"c{n}_img"] = img
            arrays[f"c{n}_edt"] = d
            arrays[f"c{n}_nearest_col"] = ncol
            arrays[f"c{n}_labels"] = lab if lab is not None else np.zeros((0,), np.uint32)
            arrays[f"c{n}_cityblock"] = city
            arrays[f"c{n}_chamfer34"] = cham
            arrays[f"c{n}_chessboard"] = cb
        arrays["n_cases"] = np.array([len(cases)])
        np.savez_compressed(os.path.join(HERE, "random_cases.npz"), **arrays)
    print("wrote six_point.json and random_cases.npz with", len(cases), "cases")


if __name__ == "__main__":
    main()

"""Regenerate tests/golden/vector_dt.json from the REFERENCE (build container only;
needs /root/reference): the frozen Danielsson matrices of proj/tests/goldens.hpp
(kOffsetsSweep1, kOffsetsFinal on the six-point sample; the disrupted-region
witness image and cell), dumped by compiling a tiny program against goldens.hpp,
plus seeded images run through the reference's own danielsson /
danielsson_first_sweep (oracle/_ref/libdfref.so).  -1 = unset / infinity.

Usage:  python tests/golden/make_golden_vector.py
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
sys.path.insert(0, ROOT)

DUMP_CPP = r"""
#include <cstdio>
#include "goldens.hpp"
template <typename M> void dump(const char* name, const M& m) {
    std::printf("\"%s\": [", name);
    for (std::size_t i = 0; i < m.size(); ++i) {
        std::printf("%s[", i ? "," : "");
        for (std::size_t j = 0; j < m[i].size(); ++j)
            std::printf("%s[%d,%d]", j ? "," : "", (int)m[i][j][0], (int)m[i][j][1]);
        std::printf("]");
    }
    std::printf("],\n");
}
int main() {
    std::printf("{");
    dump("kOffsetsSweep1", golden::kOffsetsSweep1);
    dump("kOffsetsFinal", golden::kOffsetsFinal);
    std::printf("\"six_points\": [");
    const auto img = golden::six_point_image();
    bool f = true;
    for (std::size_t i = 0; i < img.rows(); ++i)
        for (std::size_t j = 0; j < img.cols(); ++j)
            if (img.is_object(i, j)) { std::printf("%s[%zu,%zu]", f ? "" : ",", i, j); f = false; }
    std::printf("], \"six_shape\": [%zu,%zu],\n", img.rows(), img.cols());
    std::printf("\"witness_shape\": [%zu,%zu], \"witness_points\": [", golden::kWitnessRows, golden::kWitnessCols);
    for (std::size_t k = 0; k < golden::kWitnessPoints.size(); ++k)
        std::printf("%s[%zu,%zu]", k ? "," : "", golden::kWitnessPoints[k].row, golden::kWitnessPoints[k].col);
    std::printf("], \"witness_cell\": [%zu,%zu]}\n", golden::kWitnessCell.row, golden::kWitnessCell.col);
}
"""


def main():
    import oracle
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "dump.cpp")
        open(src, "w").write(DUMP_CPP)
        exe = os.path.join(d, "dump")
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", REF + "/core/include", "-I", REF + "/tests", src,
                        REF + "/core/src/grid.cpp", "-o", exe], check=True)
        out = json.loads(subprocess.run([exe], check=True, capture_output=True, text=True).stdout)
    out["_source"] = "proj/tests/goldens.hpp:144-190 (kOffsetsSweep1, kOffsetsFinal, witness), dumped by make_golden_vector.py"
    cases = []
    rng = np.random.default_rng(20210603)
    for k in range(12):
        r, c = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        dens = float(rng.choice([0.0, 0.01, 0.05, 0.3]))
        seed = int(rng.integers(1, 1 << 30))
        img = oracle.ref_random_image(r, c, dens, seed)
        for fs in (False, True):
            dd, dy, dx = oracle.ref_danielsson(img, fs)
            cases.append({"rows": r, "cols": c, "density": dens, "seed": seed, "first_sweep": fs,
                          "dist": dd.astype(np.int64).ravel().tolist(), "dy": dy.astype(np.int32).ravel().tolist(),
                          "dx": dx.astype(np.int32).ravel().tolist()})
    out["reference_runs"] = cases
    with open(os.path.join(HERE, "vector_dt.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote vector_dt.json:", len(cases), "reference runs")


if __name__ == "__main__":
    main()

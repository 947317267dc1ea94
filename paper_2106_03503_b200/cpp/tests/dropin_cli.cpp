// dropin_cli -- exercises the C++ drop-in (namespace distfield) end to end for
// tests/test_dropin.py:  dropin_cli <op> <rows> <cols> <in.u8> <out.bin> [arg]
// Writes the reference-typed result (uint64 maps, uint32 labels/columns, or
// int64 ks/js) as raw little-endian; on an exception prints its type and exits 3.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <typeinfo>
#include <vector>

#include "distfield/exact_edt.hpp"
#include "distfield/propagation.hpp"
#include "distfield/random_image.hpp"
#include "distfield/vector_dt.hpp"

using namespace distfield;

template <typename T>
static void put(std::ofstream& f, const std::vector<T>& v) {
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}
static void put_map(std::ofstream& f, const DistanceMap& dm) {
    for (std::size_t i = 0; i < dm.rows(); ++i) {
        const auto r = dm.row(i);
        f.write(reinterpret_cast<const char*>(r.data()), static_cast<std::streamsize>(r.size() * 8));
    }
}

int main(int argc, char** argv) {
    if (argc < 6) {
        std::fprintf(stderr, "usage: dropin_cli op rows cols in out [arg]\n");
        return 2;
    }
    const std::string op = argv[1];
    const std::size_t rows = std::stoul(argv[2]), cols = std::stoul(argv[3]);
    try {
        BinaryImage img(rows, cols);
        if (op != "bre" && op != "pass" && op != "meijster_raw") {
            std::ifstream in(argv[4], std::ios::binary);
            std::vector<char> buf(rows * cols);
            in.read(buf.data(), static_cast<std::streamsize>(buf.size()));
            for (std::size_t p = 0; p < buf.size(); ++p)
                if (buf[p]) img.set_object(p / cols, p % cols);
        }
        std::ofstream out(argv[5], std::ios::binary);
        if (op == "time_edt") {  // arg: repetitions; host BinaryImage in -> host DistanceMap out, per call
            const int reps = argc > 6 ? std::stoi(argv[6]) : 20;
            std::vector<double> ms;
            std::uint64_t sink = 0;
            for (int r = 0; r < reps + 3; ++r) {
                const auto t0 = std::chrono::steady_clock::now();
                const DistanceMap dm = edt(img, EdtAlgorithm::envelope);
                const auto t1 = std::chrono::steady_clock::now();
                sink += dm(rows - 1, cols - 1);
                if (r >= 3) ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
            }
            std::sort(ms.begin(), ms.end());
            out << "median_ms " << ms[ms.size() / 2] << " min_ms " << ms.front() << " reps " << reps << " sink " << sink
                << "\n";
        } else if (op == "edt") {
            ScanStats st;
            put_map(out, edt(img, EdtAlgorithm::envelope, Orientation::automatic, &st, 4));
        } else if (op == "edt_simple") {
            put_map(out, edt(img, EdtAlgorithm::simple, Orientation::columns));
        } else if (op == "vertical") {
            put_map(out, vertical_pass(img));
        } else if (op == "vertical_down" || op == "vertical_up") {  // over init_distance_map(img)
            DistanceMap dm = init_distance_map(img, DistanceKind::squared_euclidean);
            if (op == "vertical_down") vertical_down_pass(dm, 2);
            else vertical_up_pass(dm, 2);
            put_map(out, dm);
        } else if (op == "vertical_both") {  // down then up == vertical_pass (exact_edt.cpp:112-117)
            DistanceMap dm = init_distance_map(img, DistanceKind::squared_euclidean);
            vertical_down_pass(dm);
            vertical_up_pass(dm);
            put_map(out, dm);
        } else if (op == "meijster") {
            const auto r = meijster_scan(vertical_pass(img));
            put_map(out, r.map);
            std::vector<std::uint32_t> nc(r.nearest_col.cells().begin(), r.nearest_col.cells().end());
            put(out, nc);
        } else if (op == "rowenv") {
            const auto env = meijster_row_envelope(vertical_pass(img), std::stoul(argv[6]));
            std::vector<std::int64_t> v{static_cast<std::int64_t>(env.ks.size())};
            v.insert(v.end(), env.ks.begin(), env.ks.end());
            v.insert(v.end(), env.js.begin(), env.js.end());
            put(out, v);
        } else if (op == "labels") {
            const auto lm = voronoi_labels(img);
            std::vector<std::uint32_t> v(rows * cols);
            for (std::size_t i = 0; i < rows; ++i)
                for (std::size_t j = 0; j < cols; ++j) v[i * cols + j] = lm(i, j);
            put(out, v);
        } else if (op == "cityblock") {
            put_map(out, cityblock_sequential(img));
        } else if (op == "chamfer") {
            put_map(out, chamfer34(img));
        } else if (op == "chessboard") {
            put_map(out, chessboard(img));
        } else if (op == "danielsson" || op == "danielsson_first") {  // map, then dy, dx (uint32), then to_text
            const auto r = op == "danielsson" ? danielsson(img) : danielsson_first_sweep(img);
            put_map(out, r.distance);
            std::vector<std::uint32_t> dy(rows * cols), dx(rows * cols);
            for (std::size_t i = 0; i < rows; ++i)
                for (std::size_t j = 0; j < cols; ++j) {
                    dy[i * cols + j] = r.offsets(i, j).dy;
                    dx[i * cols + j] = r.offsets(i, j).dx;
                }
            put(out, dy);
            put(out, dx);
            const std::string t = to_text(r.offsets);
            out.write(t.data(), static_cast<std::streamsize>(t.size()));
        } else if (op == "both") {
            const auto [a, b] = edt_both_polarities(img);
            put_map(out, a);
            put_map(out, b);
        } else if (op == "bre") {  // build_row_envelope: rows must be 1; input = cols int64; arg lmax, tie
            std::ifstream in(argv[4], std::ios::binary);
            std::vector<std::int64_t> v(cols);
            in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(cols * 8));
            ScanStats st;
            const auto env = build_row_envelope(v, std::stoll(argv[6]),
                                                std::stoi(argv[7]) ? EnvelopeTie::take_new : EnvelopeTie::keep_old, &st);
            std::vector<std::int64_t> o{static_cast<std::int64_t>(env.ks.size())};
            o.insert(o.end(), env.ks.begin(), env.ks.end());
            o.insert(o.end(), env.js.begin(), env.js.end());
            put(out, o);
        } else if (op == "pass" || op == "meijster_raw") {  // input = a uint64 map
            std::ifstream in(argv[4], std::ios::binary);
            DistanceMap dm(rows, cols, DistanceKind::cityblock);
            for (std::size_t i = 0; i < rows; ++i) {
                auto r = dm.row(i);
                in.read(reinterpret_cast<char*>(r.data()), static_cast<std::streamsize>(cols * 8));
            }
            if (op == "meijster_raw") {
                const auto r = meijster_scan(dm);
                put_map(out, r.map);
                std::vector<std::uint32_t> nc(r.nearest_col.cells().begin(), r.nearest_col.cells().end());
                put(out, nc);
            } else {
                const int w = std::stoi(argv[6]);
                if (w == 0) cityblock_forward_pass(dm);
                else if (w == 1) cityblock_backward_pass(dm);
                else if (w == 2) cityblock_vertical_passes(dm, 3);
                else if (w == 3) cityblock_horizontal_passes(dm, 3);
                else if (w == 4) chamfer_forward_pass(dm);
                else chamfer_backward_pass(dm);
                put_map(out, dm);
            }
        } else if (op == "random") {  // generator parity: rows cols <unused> out density seed
            const auto r = generate_random_image(rows, cols, std::stod(argv[6]), std::stoull(argv[7]));
            std::vector<std::uint8_t> v(rows * cols);
            for (std::size_t p = 0; p < v.size(); ++p) v[p] = r.is_object(p / cols, p % cols);
            put(out, v);
        } else {
            std::fprintf(stderr, "unknown op %s\n", op.c_str());
            return 2;
        }
    } catch (const std::domain_error& e) {
        std::printf("EXC domain_error: %s\n", e.what());
        return 3;
    } catch (const std::length_error& e) {
        std::printf("EXC length_error: %s\n", e.what());
        return 3;
    } catch (const std::invalid_argument& e) {
        std::printf("EXC invalid_argument: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::printf("EXC %s: %s\n", typeid(e).name(), e.what());
        return 3;
    }
    return 0;
}

// distfield_b200 -- the reference CLI's `transform`, `labels` and `bench`
// subcommands (proj/tools/distfield_cli.cpp:149-222, 294-304, 308-345, 353-416)
// routed to the B200 path: a P4 input travels to the GPU as its packed raster
// and is unpacked there; transforms, labels and gray renderings stay in HBM;
// only the requested outputs come back.  Same options, defaults, messages and
// exit codes ("error: <what>", exit 1).  --algorithm danielsson / --offsets run
// the vector transform's sweeps on the device (k_vector.cu).  Not provided:
// `chart` (reference metric charts, not a transform).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "distfield/bench.hpp"
#include "distfield/device_image.hpp"
#include "distfield/exact_edt.hpp"
#include "distfield/netpbm.hpp"
#include "distfield/propagation.hpp"
#include "distfield/random_image.hpp"

using namespace distfield;

namespace {

// command-line errors, with CLI11's exit codes (ExtrasError 109,
// ValidationError 105, RequiredError 106)
struct UsageError : std::runtime_error {
    UsageError(const std::string& what, int code) : std::runtime_error(what), code(code) {}
    int code;
};

std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

void write_file(const std::string& path, const std::string& bytes) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write " + path);
    out << bytes;
}

std::size_t parse_count(const std::string& text, const char* what) {
    std::size_t pos = 0;
    unsigned long long v = 0;
    try {
        v = std::stoull(text, &pos);
    } catch (const std::exception&) {
        pos = std::string::npos;
    }
    if (pos != text.size()) throw std::runtime_error(std::string("invalid ") + what + ": " + text);
    return static_cast<std::size_t>(v);
}

// Minimal option parser: --name value / --flag, as the reference's CLI11 setup.
class Args {
public:
    Args(int argc, char** argv, int first, const std::vector<std::string>& options,
         const std::vector<std::string>& flags) {
        for (int k = first; k < argc; ++k) {
            std::string a = argv[k];
            std::string val;
            bool has_val = false;
            if (const auto eq = a.find('='); a.rfind("--", 0) == 0 && eq != std::string::npos) {
                val = a.substr(eq + 1);
                a = a.substr(0, eq);
                has_val = true;
            }
            if (std::find(flags.begin(), flags.end(), a) != flags.end()) {
                flags_[a] = true;
            } else if (std::find(options.begin(), options.end(), a) != options.end()) {
                if (!has_val) {
                    if (k + 1 >= argc) throw UsageError(a + " requires an argument", 114);
                    val = argv[++k];
                }
                opts_[a] = val;
            } else {
                throw UsageError("unknown option " + a, 109);
            }
        }
    }
    std::string get(const std::string& k, const std::string& def = "") const {
        const auto it = opts_.find(k);
        return it == opts_.end() ? def : it->second;
    }
    bool flag(const std::string& k) const { return flags_.count(k) != 0; }

private:
    std::map<std::string, std::string> opts_;
    std::map<std::string, bool> flags_;
};

void check_member(const std::string& name, const std::string& v, const std::vector<std::string>& allowed) {
    if (std::find(allowed.begin(), allowed.end(), v) == allowed.end())
        throw UsageError(name + ": " + v + " not in {" + [&] {
            std::string s;
            for (const auto& a : allowed) s += (s.empty() ? "" : ",") + a;
            return s;
        }() + "}", 105);
}

// --input (P1/P4) or --points-file + --size; --polarity inside inverts on the GPU.
DeviceImage load_image(const Args& a, bool with_polarity) {
    const std::string input = a.get("--input"), points = a.get("--points-file"), size = a.get("--size");
    const bool inside = with_polarity && a.get("--polarity", "outside") == "inside";
    if (!input.empty() && !points.empty()) throw std::runtime_error("choose one of --input or --points-file");
    if (!input.empty()) return DeviceImage::from_raster(read_pbm_raster(read_file(input)), inside);
    if (points.empty()) throw std::runtime_error("an input is required (--input or --points-file)");
    if (size.empty()) throw std::runtime_error("--points-file requires --size ROWSxCOLS");
    const auto x = size.find('x');
    if (x == std::string::npos || x == 0 || x + 1 >= size.size())
        throw std::runtime_error("--size expects ROWSxCOLS, e.g. 9x10");
    const std::size_t rows = parse_count(size.substr(0, x), "row count");
    const std::size_t cols = parse_count(size.substr(x + 1), "column count");
    std::ifstream in(points);
    if (!in) throw std::runtime_error("cannot open " + points);
    std::vector<GridPoint> pts;
    std::string line;
    for (std::size_t lineno = 1; std::getline(in, line); ++lineno) {
        if (const auto h = line.find('#'); h != std::string::npos) line.erase(h);
        std::istringstream ls(line);
        std::size_t r, c;
        if (!(ls >> r)) continue;
        if (!(ls >> c)) throw std::runtime_error(points + ":" + std::to_string(lineno) + ": expected \"row col\"");
        pts.push_back({r, c});
    }
    return DeviceImage::from_image(BinaryImage::from_points(rows, cols, pts), inside);
}

int run_transform(const Args& a) {
    const std::string metric = a.get("--metric", "euclidean");
    std::string algorithm = a.get("--algorithm");
    check_member("--orient", a.get("--orient", "auto"), {"auto", "rows", "columns"});
    check_member("--gray-mode", a.get("--gray-mode", "auto"), {"auto", "linear", "sqrt-linear"});
    check_member("--polarity", a.get("--polarity", "outside"), {"outside", "inside"});
    const std::string dump = a.get("--dump"), gray = a.get("--gray"), labels = a.get("--labels"),
                      offsets = a.get("--offsets");
    if (dump.empty() && gray.empty() && labels.empty() && offsets.empty())
        throw std::runtime_error("no output requested (--dump, --gray, --labels, --offsets)");
    if (algorithm.empty())
        algorithm = metric == "cityblock" ? "sequential" : "envelope";
    else if (metric == "chamfer34")
        throw std::runtime_error("chamfer34 takes no --algorithm");

    DistanceKind kind;
    if (metric == "cityblock") {
        if (algorithm != "sequential" && algorithm != "separable")
            throw std::runtime_error("cityblock supports --algorithm sequential|separable");
        kind = DistanceKind::cityblock;
    } else if (metric == "chamfer34") {
        kind = DistanceKind::chamfer3;
    } else if (metric == "chessboard") {  // B200 addition (no reference transform)
        kind = DistanceKind::chessboard;
    } else if (metric == "euclidean") {
        if (algorithm != "danielsson" && !parse_algorithm(algorithm))
            throw std::runtime_error(
                "euclidean supports --algorithm bruteforce|simple|improved|envelope|danielsson");
        kind = DistanceKind::squared_euclidean;  // every algorithm yields the same map (exact_edt.cpp:285-317)
    } else {
        throw std::runtime_error("unknown --metric " + metric);
    }

    const DeviceImage img = load_image(a, true);
    if (img.object_count() == 0) std::cerr << "warning: no features, distances are infinite everywhere\n";
    const bool vector_dt = metric == "euclidean" && algorithm == "danielsson";
    if (!offsets.empty() && !vector_dt) throw std::runtime_error("--offsets requires --algorithm danielsson");
    if (vector_dt) {  // distfield_cli.cpp:177-179, :192-220: the approximate vector transform
        if (!labels.empty()) throw std::runtime_error("--labels requires an exact euclidean algorithm");
        const VectorDtResult vec = danielsson(img);
        if (!dump.empty()) write_file(dump, a.flag("--sqrt") ? to_text_sqrt(vec.distance) : to_text(vec.distance));
        if (a.flag("--normalized")) throw std::runtime_error("--normalized applies to chamfer34 results only");
        if (!gray.empty()) {
            const std::string mode = a.get("--gray-mode", "auto");
            write_file(gray, write_netpbm(to_gray(vec.distance, mode == "linear" ? GrayMapping::linear
                                                                                  : GrayMapping::sqrt_linear),
                                          PgmVariant::raw));
        }
        if (!offsets.empty()) write_file(offsets, to_text(vec.offsets));
        return 0;
    }
    const DeviceMap dm = transform(img, kind);

    const bool sqrt_dump = a.flag("--sqrt"), normalized = a.flag("--normalized");
    if (sqrt_dump && kind != DistanceKind::squared_euclidean)
        throw std::runtime_error("--sqrt applies to euclidean results only");
    if (normalized && kind != DistanceKind::chamfer3)
        throw std::runtime_error("--normalized applies to chamfer34 results only");
    if (!labels.empty() && metric != "euclidean")
        throw std::runtime_error("--labels requires an exact euclidean algorithm");

    if (!dump.empty()) {
        const DistanceMap host = dm.download();
        write_file(dump, normalized ? to_text(chamfer_normalized(host)) : sqrt_dump ? to_text_sqrt(host) : to_text(host));
    }
    if (!gray.empty()) {
        const std::string mode = a.get("--gray-mode", "auto");
        const bool sq = mode == "sqrt-linear" || (mode == "auto" && kind == DistanceKind::squared_euclidean);
        write_file(gray, write_netpbm(dm.to_gray(sq ? GrayMapping::sqrt_linear : GrayMapping::linear), PgmVariant::raw));
    }
    if (!labels.empty()) {
        const DeviceLabels lab = voronoi_labels(img);
        write_file(labels, write_netpbm(lab.to_gray(img.object_count()), PgmVariant::raw));
    }
    return 0;
}

int run_labels(const Args& a) {
    const std::string out = a.get("--out"), dump = a.get("--dump");
    if (out.empty() && dump.empty()) throw std::runtime_error("no output requested (--out, --dump)");
    const DeviceImage img = load_image(a, false);
    const DeviceLabels lab = voronoi_labels(img);
    if (!out.empty()) write_file(out, write_netpbm(lab.to_gray(img.object_count()), PgmVariant::raw));
    if (!dump.empty()) write_file(dump, to_text(lab.download()));
    return 0;
}

// bench: the reference's CSV schema (bench.cpp:63-71), GPU edt per row.
int run_bench_cmd(const Args& a) {
    BenchConfig config;
    auto split = [](const std::string& t) {
        std::vector<std::string> parts;
        std::istringstream ss(t);
        std::string p;
        while (std::getline(ss, p, ','))
            if (!p.empty()) parts.push_back(p);
        return parts;
    };
    for (const auto& s : split(a.get("--sizes", "64,128,256"))) config.sizes.push_back(parse_count(s, "size"));
    for (const auto& n : split(a.get("--algorithms", "simple,envelope"))) {
        const auto p = parse_algorithm(n);
        if (!p) throw std::runtime_error("unknown algorithm " + n);
        config.algorithms.push_back(*p);
    }
    if (config.sizes.empty() || config.algorithms.empty())
        throw std::runtime_error("bench needs at least one size and one algorithm");
    config.density = std::stod(a.get("--density", "0.02"));
    config.reps = static_cast<unsigned>(parse_count(a.get("--reps", "1"), "reps"));
    config.seed = parse_count(a.get("--seed", "1"), "seed");
    const std::string csv = to_csv(run_bench(config));
    const std::string out = a.get("--out");
    if (out.empty())
        std::cout << csv;
    else
        write_file(out, csv);
    return 0;
}

const char* kUsage =
    "binary-image distance transforms (B200)\n"
    "usage: distfield_b200 SUBCOMMAND [options]\n"
    "  transform  --input FILE | --points-file FILE --size RxC  [--polarity outside|inside]\n"
    "             [--metric euclidean|cityblock|chamfer34|chessboard] [--algorithm A] [--orient auto|rows|columns]\n"
    "             [--dump FILE [--sqrt|--normalized]] [--gray FILE [--gray-mode auto|linear|sqrt-linear]]\n"
    "             [--labels FILE] [--threads N]\n"
    "  labels     --input FILE | --points-file FILE --size RxC  [--out FILE] [--dump FILE] [--threads N]\n"
    "  bench      [--sizes 64,128,256] [--density 0.02] [--algorithms simple,envelope] [--reps 1]\n"
    "             [--seed 1] [--threads N] [--out FILE]\n";

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
        (argc < 2 ? std::cerr : std::cout) << kUsage;
        return argc < 2 ? 106 : 0;
    }
    const std::string sub = argv[1];
    try {
        if (sub == "transform") {
            const Args a(argc, argv, 2,
                         {"--input", "--points-file", "--size", "--polarity", "--metric", "--algorithm", "--orient",
                          "--dump", "--gray", "--gray-mode", "--labels", "--offsets", "--threads"},
                         {"--sqrt", "--normalized"});
            return run_transform(a);
        }
        if (sub == "labels") {
            const Args a(argc, argv, 2, {"--input", "--points-file", "--size", "--out", "--dump", "--threads"}, {});
            return run_labels(a);
        }
        if (sub == "bench") {
            const Args a(argc, argv, 2,
                         {"--sizes", "--density", "--algorithms", "--reps", "--seed", "--threads", "--out"}, {});
            return run_bench_cmd(a);
        }
        if (sub == "chart") throw std::runtime_error("chart is not part of the B200 build (reference metric charts)");
        std::cerr << "unknown subcommand " << sub << "\n" << kUsage;
        return 109;
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\n" << kUsage;
        return e.code;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}

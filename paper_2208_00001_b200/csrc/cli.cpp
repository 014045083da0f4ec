// geodist_b200 — the reference CLI's subcommands on the B200 engine
// (reference: proj/tools/main.cpp:130-512, which needs CLI11; this one parses
// its own arguments).  Same subcommands, flags, output lines, CSV schema and
// exit codes (0 ok, 1 compare over tolerance, 2 usage, 3 I/O, 4 compute):
//   compute    --input --seeds --mode {geodesic,euclidean,generalized,signed,gsf}
//              [--lambda --v --theta --iterations --engine --threads --fixpoint
//               --output --preview --slice]
//   compare    --a --b [--tol]
//   benchmark  --dims --sizes --threads-list [--iterations --lambda --repeats --csv]
// Every transform runs through the C++ drop-in (include/geodist) on the GPU.
// Engine::Serial / Engine::Oracle are the reference's CPU engines: rejected
// (exit 2), as the library rejects them.  `benchmark` times the GPU engine
// end to end on host grids (the drop-in call: H2D, scan, D2H) and reports the
// reference's CSV columns; with no serial engine in this build its serial row
// is absent and speedup_vs_serial / max_dev_vs_serial are "nan".
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "geodist/grid.hpp"
#include "geodist/io.hpp"
#include "geodist/scan_parallel.hpp"
#include "geodist/transforms.hpp"

using namespace geodist;

namespace {

enum Exit : int { kOk = 0, kOverTol = 1, kUsage = 2, kIo = 3, kCompute = 4 };

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void diag(const std::string& m) { std::cerr << "geodist: error: " << m << "\n"; }

// --name value / --name=value options and bare flags after the subcommand.
class Args {
public:
    Args(int argc, char** argv, int first, std::vector<std::string> flags) {
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) throw Usage("unexpected argument: " + a);
            a = a.substr(2);
            const auto eq = a.find('=');
            if (eq != std::string::npos) {
                kv_[a.substr(0, eq)] = a.substr(eq + 1);
            } else if (std::find(flags.begin(), flags.end(), a) != flags.end()) {
                kv_[a] = "1";
            } else {
                if (i + 1 >= argc) throw Usage("--" + a + " needs a value");
                kv_[a] = argv[++i];
            }
        }
    }
    void allow(std::initializer_list<const char*> names) const {
        for (const auto& [k, v] : kv_) {
            bool ok = false;
            for (const char* n : names) ok = ok || k == n;
            if (!ok) throw Usage("unknown option --" + k);
        }
    }
    bool has(const std::string& k) const { return kv_.count(k) != 0; }
    std::string str(const std::string& k) const {
        if (!has(k)) throw Usage("--" + k + " is required");
        return kv_.at(k);
    }
    std::string str(const std::string& k, const std::string& d) const { return has(k) ? kv_.at(k) : d; }
    double num(const std::string& k, double d) const { return has(k) ? to_double(k, kv_.at(k)) : d; }
    long integer(const std::string& k, long d) const { return has(k) ? to_long(k, kv_.at(k)) : d; }
    std::vector<long> list(const std::string& k) const {
        std::vector<long> out;
        std::stringstream ss(str(k));
        for (std::string t; std::getline(ss, t, ',');) out.push_back(to_long(k, t));
        return out;
    }

    static long to_long(const std::string& k, const std::string& v) {
        char* end = nullptr;
        const long x = std::strtol(v.c_str(), &end, 10);
        if (v.empty() || *end != '\0') throw Usage("--" + k + ": not an integer: " + v);
        return x;
    }
    static double to_double(const std::string& k, const std::string& v) {
        char* end = nullptr;
        const double x = std::strtod(v.c_str(), &end);
        if (v.empty() || *end != '\0') throw Usage("--" + k + ": not a number: " + v);
        return x;
    }

private:
    std::map<std::string, std::string> kv_;
};

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

std::string shape_of(const ScalarGrid& g) {
    std::string s;
    for (int a = 0; a < g.ndim(); ++a) s += (a ? "x" : "") + std::to_string(g.extent(a));
    return s;
}

std::string coords_of(const ScalarGrid& g, std::size_t i) {
    const std::size_t w = g.width(), h = g.height();
    const std::string yx = std::to_string((i / w) % h) + "," + std::to_string(i % w);
    return g.ndim() == 3 ? "(" + std::to_string(i / (w * h)) + "," + yx + ")" : "(" + yx + ")";
}

Engine engine_of(const std::string& s) {
    std::string l = s;
    std::transform(l.begin(), l.end(), l.begin(), [](unsigned char c) { return std::tolower(c); });
    if (l == "parallel") return Engine::Parallel;
    if (l == "serial") return Engine::Serial;
    if (l == "oracle") return Engine::Oracle;
    throw Usage("--engine: expected serial, parallel or oracle, got " + s);
}

int threads_default(const Args& a) {
    if (a.has("threads")) {
        const long t = a.integer("threads", 1);
        if (t < 1) throw Usage("--threads must be >= 1");
        return static_cast<int>(t);
    }
    if (const char* env = std::getenv("GEODIST_THREADS")) {
        char* end = nullptr;
        const long v = std::strtol(env, &end, 10);
        if (end == env || *end != '\0' || v < 1)
            throw Usage(std::string("invalid GEODIST_THREADS value: ") + env);
        return static_cast<int>(v);
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? static_cast<int>(hw) : 1;
}

ScalarGrid slice_of(const ScalarGrid& g, int z) {
    const int dims[2] = {g.height(), g.width()};
    const double sp[2] = {g.spacing(1), g.spacing(2)};
    ScalarGrid out(2, dims, sp, 0.0f);
    const std::size_t plane = static_cast<std::size_t>(g.height()) * g.width();
    std::copy_n(g.data() + plane * z, plane, out.data());
    return out;
}

int cmd_compute(const Args& a) {
    a.allow({"input", "seeds", "mode", "lambda", "v", "theta", "iterations", "engine", "threads",
             "fixpoint", "output", "preview", "slice"});
    const std::string mode = a.str("mode");
    static const char* kModes[] = {"geodesic", "euclidean", "generalized", "signed", "gsf"};
    if (std::find_if(std::begin(kModes), std::end(kModes),
                     [&](const char* m) { return mode == m; }) == std::end(kModes))
        throw Usage("--mode: unknown transform " + mode);
    const bool has_theta = a.has("theta");
    if (mode == "gsf" && !has_theta) throw Usage("--theta is required for --mode gsf");
    if (mode != "gsf" && has_theta) throw Usage("--theta applies to --mode gsf only");
    const std::string out_path = a.str("output");
    const int threads = threads_default(a);

    const ScalarGrid image = read_grid_file(a.str("input"));
    const ScalarGrid seeds = read_grid_file(a.str("seeds"));
    if (!image.same_shape(seeds)) throw Usage("shape mismatch between --input and --seeds");
    if (!image.same_spacing(seeds)) throw Usage("spacing mismatch between --input and --seeds");

    TransformParams params;
    params.lambda = a.num("lambda", 1.0);
    params.nu = a.num("v", 1.0e10);
    params.iterations = static_cast<int>(a.integer("iterations", 2));
    params.validate();
    ScanPolicy policy;
    policy.engine = engine_of(a.str("engine", "parallel"));
    policy.workers = threads;
    policy.to_fixpoint = a.has("fixpoint");
    policy.max_rounds = 100;

    TransformStats stats;
    const auto t0 = std::chrono::steady_clock::now();
    ScalarGrid result = [&] {
        if (mode == "geodesic") return geodesic_distance(image, seeds, params, policy, &stats);
        if (mode == "euclidean") return euclidean_distance(seeds, params.iterations, policy, &stats);
        if (mode == "generalized") return generalized_geodesic(image, seeds, params, policy, &stats);
        if (mode == "signed") return signed_geodesic(image, seeds, params, policy, &stats);
        GsfParams gp;
        gp.base = params;
        gp.theta = a.num("theta", 0.0);
        return gsf(image, seeds, gp, policy, &stats);
    }();
    const double wall = ms_since(t0);
    write_fgd1_file(result, out_path);
    if (a.has("preview")) {
        if (result.ndim() == 2) {
            write_preview_file(result, a.str("preview"));
        } else {
            const long z = a.integer("slice", -1);
            if (z < 0) throw Usage("3D preview requires --slice Z");
            if (z >= result.depth())
                throw Usage("--slice out of range: grid depth is " + std::to_string(result.depth()));
            write_preview_file(slice_of(result, static_cast<int>(z)), a.str("preview"));
        }
    }
    if (policy.to_fixpoint && !stats.converged)
        std::cerr << "geodist: warning: fixpoint not reached within " << policy.max_rounds
                  << " rounds\n";
    std::printf("mode=%s size=%s engine=%s threads=%d wall_ms=%.3f rounds=%d\n", mode.c_str(),
                shape_of(result).c_str(), engine_name(policy.engine), threads, wall, stats.rounds);
    return kOk;
}

int cmd_compare(const Args& a) {
    a.allow({"a", "b", "tol"});
    const double tol = a.num("tol", 0.0);
    auto load = [](const std::string& p) {
        std::ifstream is(p, std::ios::binary);
        if (!is) throw IoError("cannot open for reading: " + p);
        return read_grid_fgd1(is);
    };
    const ScalarGrid ga = load(a.str("a")), gb = load(a.str("b"));
    if (!ga.same_shape(gb) || !ga.same_spacing(gb)) throw Usage("shape mismatch between --a and --b");
    double worst = 0.0;
    std::size_t at = 0, over = 0;
    for (std::size_t i = 0; i < ga.size(); ++i) {
        const double d = std::fabs(static_cast<double>(ga.data()[i]) - gb.data()[i]);
        if (d > worst) {
            worst = d;
            at = i;
        }
        over += d > tol ? 1 : 0;
    }
    std::printf("max_abs_diff=%.9g at=%s cells_over_tol=%zu tol=%.9g\n", worst,
                coords_of(ga, at).c_str(), over, tol);
    return worst <= tol ? kOk : kOverTol;
}

int cmd_benchmark(const Args& a) {
    a.allow({"dims", "sizes", "threads-list", "iterations", "lambda", "repeats", "csv"});
    const long nd = a.integer("dims", 0);
    if (nd != 2 && nd != 3) throw Usage("--dims must be 2 or 3");
    const std::vector<long> sizes = a.list("sizes"), threads = a.list("threads-list");
    if (sizes.empty() || threads.empty()) throw Usage("--sizes and --threads-list must be non-empty");
    for (long t : threads)
        if (t < 1) throw Usage("--threads-list entries must be >= 1");
    const long repeats = a.integer("repeats", 5);
    if (repeats < 1) throw Usage("--repeats must be >= 1");
    TransformParams params;
    params.lambda = a.num("lambda", 1.0);
    params.iterations = static_cast<int>(a.integer("iterations", 2));
    params.validate();

    std::string csv =
        "ndim,size,engine,threads,iterations,wall_ms,speedup_vs_serial,max_dev_vs_serial,rng_seed\n";
    for (long size : sizes) {
        if (size < 1) throw Usage("--sizes entries must be >= 1");
        // SplitMix64 benchmark image, seed as tools/main.cpp:312-314
        const std::uint64_t seed = 0x67656F64697374ull ^ (static_cast<std::uint64_t>(nd) << 32) ^
                                   static_cast<std::uint64_t>(size);
        std::vector<int> dims(static_cast<std::size_t>(nd), static_cast<int>(size));
        std::vector<double> sp(static_cast<std::size_t>(nd), 1.0);
        ScalarGrid image(static_cast<int>(nd), dims, sp, 0.0f);
        std::uint64_t s = seed;
        for (std::size_t i = 0; i < image.size(); ++i) {
            s += 0x9E3779B97F4A7C15ull;
            std::uint64_t z = s;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            image.data()[i] = static_cast<float>(static_cast<double>(z >> 40) * 0x1.0p-24);
        }
        ScalarGrid mask = grid_like(image, 0.0f);
        const std::size_t c = (static_cast<std::size_t>(image.depth() / 2) * image.height() +
                               image.height() / 2) * image.width() + image.width() / 2;
        mask.data()[c] = 1.0f;
        const ScalarGrid init = init_hard_seeds(mask);
        for (long w : threads) {
            std::vector<double> t;
            for (long rep = 0; rep <= repeats; ++rep) {  // rep 0: warm-up
                ScalarGrid dist = init;
                const auto t0 = std::chrono::steady_clock::now();
                detail::parallel_scan_inplace(image, dist, params, static_cast<int>(w));
                if (rep > 0) t.push_back(ms_since(t0));
            }
            std::sort(t.begin(), t.end());
            const double med = t.size() % 2 ? t[t.size() / 2]
                                            : 0.5 * (t[t.size() / 2 - 1] + t[t.size() / 2]);
            char row[256];
            std::snprintf(row, sizeof(row), "%ld,%ld,parallel,%ld,%d,%.3f,nan,nan,%llu\n", nd, size,
                          w, params.iterations, med, static_cast<unsigned long long>(seed));
            csv += row;
        }
    }
    std::cout << csv;
    if (a.has("csv")) {
        std::ofstream os(a.str("csv"));
        if (!os) throw IoError("cannot open for writing: " + a.str("csv"));
        os << csv;
        os.flush();
        if (!os) throw IoError("write failure: " + a.str("csv"));
    }
    return kOk;
}

// Exception -> exit code, as tools/main.cpp:393-415.
int guarded(const std::function<int()>& f) {
    try {
        return f();
    } catch (const Usage& e) {
        diag(e.what());
        return kUsage;
    } catch (const FormatError& e) {
        diag(e.what());
        return kIo;
    } catch (const IoError& e) {
        diag(e.what());
        return kIo;
    } catch (const EmptySeedsError& e) {
        diag(e.what());
        return kCompute;
    } catch (const std::invalid_argument& e) {
        diag(e.what());
        return kUsage;
    } catch (const std::exception& e) {
        diag(e.what());
        return kCompute;
    }
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
        std::cout << "usage: geodist_b200 {compute|compare|benchmark} [--options]\n"
                     "  geodesic, Euclidean and hybrid distance transforms on 2D/3D grids (B200)\n";
        return argc < 2 ? kUsage : kOk;
    }
    const std::string sub = argv[1];
    return guarded([&] {
        if (sub == "compute") return cmd_compute(Args(argc, argv, 2, {"fixpoint"}));
        if (sub == "compare") return cmd_compare(Args(argc, argv, 2, {}));
        if (sub == "benchmark") return cmd_benchmark(Args(argc, argv, 2, {}));
        throw Usage("unknown subcommand " + sub);
    });
}

// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library (`geodist`, compiled from
// /root/reference/proj/src by oracle/Makefile with -Dgeodist=geodist_ref so its
// symbols cannot collide with ours).  Python tests and bench.py's reference arm
// load oracle/_ref/libgeodist_ref.so through ctypes and call these entry points;
// every function forwards to the reference's own public API:
//   generalized_geodesic  transforms.hpp:62-64 / transforms.cpp:143-158
//   gsf                   transforms.hpp:85-86 / transforms.cpp:231-238
//   directional_pass      scan_parallel.hpp:20-22 / scan_parallel.cpp:344-349
//   parallel_scan         scan_parallel.hpp:27-28 / scan_parallel.cpp:351-355
//   scan_to_fixpoint      scan_parallel.hpp:40-43 / scan_parallel.cpp:357-397
//   geodesic_distance / euclidean_distance / signed_geodesic   transforms.cpp:127-183
//   dijkstra_exact        oracle.hpp:19-20
// Status codes: 0 ok, 1 std::invalid_argument, 2 EmptySeedsError, 3 other.
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "geodist/grid.hpp"
#include "geodist/metric.hpp"
#include "geodist/oracle.hpp"
#include "geodist/scan_parallel.hpp"
#include "geodist/scan_serial.hpp"
#include "geodist/transforms.hpp"

namespace {

thread_local std::string g_err;

geodist::ScalarGrid make(int ndim, const int* dims, const double* spacing, const float* data) {
    geodist::ScalarGrid g(ndim, std::span<const int>(dims, ndim),
                          std::span<const double>(spacing, ndim), 0.0f);
    if (data) std::memcpy(g.data(), data, g.size() * sizeof(float));
    return g;
}

void put(const geodist::ScalarGrid& g, float* out) {
    std::memcpy(out, g.data(), g.size() * sizeof(float));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const geodist::EmptySeedsError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

geodist::TransformParams params(double lambda, double nu, int iterations) {
    geodist::TransformParams p;
    p.lambda = lambda;
    p.nu = nu;
    p.iterations = iterations;
    return p;
}

geodist::ScanPolicy policy(int engine, int workers, int to_fixpoint, int max_rounds, double tol) {
    geodist::ScanPolicy p;
    p.engine = static_cast<geodist::Engine>(engine);
    p.workers = workers;
    p.to_fixpoint = to_fixpoint != 0;
    p.max_rounds = max_rounds;
    p.tol = tol;
    return p;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_generalized_geodesic(int ndim, const int* dims, const double* spacing,
                             const float* image, const float* mask, double lambda, double nu,
                             int iterations, int workers, float* out, int* rounds) {
    return guard([&] {
        auto im = make(ndim, dims, spacing, image);
        auto m = make(ndim, dims, spacing, mask);
        geodist::TransformStats st;
        auto r = geodist::generalized_geodesic(im, m, params(lambda, nu, iterations),
                                               policy(1, workers, 0, 100, 1e-6), &st);
        put(r, out);
        if (rounds) *rounds = st.rounds;
    });
}

int ref_gsf(int ndim, const int* dims, const double* spacing, const float* image,
            const float* mask, double lambda, double nu, int iterations, double theta,
            int workers, float* out, int* rounds, int* complement_empty) {
    return guard([&] {
        auto im = make(ndim, dims, spacing, image);
        auto m = make(ndim, dims, spacing, mask);
        geodist::GsfParams gp;
        gp.base = params(lambda, nu, iterations);
        gp.theta = theta;
        geodist::TransformStats st;
        auto r = geodist::gsf(im, m, gp, policy(1, workers, 0, 100, 1e-6), &st);
        put(r, out);
        if (rounds) *rounds = st.rounds;
        if (complement_empty) *complement_empty = st.complement_empty ? 1 : 0;
    });
}

int ref_directional_pass(int ndim, const int* dims, const double* spacing, const float* image,
                         float* dist, int axis, int orientation, double lambda, int workers) {
    return guard([&] {
        auto im = make(ndim, dims, spacing, image);
        auto d = make(ndim, dims, spacing, dist);
        geodist::PassDirection dir{axis, orientation};
        auto r = geodist::directional_pass(std::move(d), im, dir, params(lambda, 1e10, 1),
                                           workers);
        put(r, dist);
    });
}

int ref_parallel_scan(int ndim, const int* dims, const double* spacing, const float* image,
                      float* dist, double lambda, int iterations, int workers) {
    return guard([&] {
        auto im = make(ndim, dims, spacing, image);
        auto d = make(ndim, dims, spacing, dist);
        auto r = geodist::parallel_scan(im, std::move(d), params(lambda, 1e10, iterations),
                                        workers);
        put(r, dist);
    });
}

int ref_serial_scan(int ndim, const int* dims, const double* spacing, const float* image,
                    float* dist, double lambda, int iterations) {
    return guard([&] {
        auto im = make(ndim, dims, spacing, image);
        auto d = make(ndim, dims, spacing, dist);
        auto r = geodist::serial_scan(im, std::move(d), params(lambda, 1e10, iterations));
        put(r, dist);
    });
}

int ref_scan_to_fixpoint(int ndim, const int* dims, const double* spacing, const float* image,
                         float* dist, double lambda, int engine, int max_rounds, double tol,
                         int workers, int* rounds_used, int* converged, double* last_change) {
    return guard([&] {
        auto im = make(ndim, dims, spacing, image);
        auto d = make(ndim, dims, spacing, dist);
        auto r = geodist::scan_to_fixpoint(im, std::move(d), params(lambda, 1e10, 1),
                                           static_cast<geodist::Engine>(engine), max_rounds, tol,
                                           workers);
        put(r.dist, dist);
        if (rounds_used) *rounds_used = r.rounds_used;
        if (converged) *converged = r.converged ? 1 : 0;
        if (last_change) *last_change = r.last_change;
    });
}

int ref_geodesic_distance(int ndim, const int* dims, const double* spacing, const float* image,
                          const float* seeds, double lambda, int iterations, int workers,
                          float* out) {
    return guard([&] {
        auto im = make(ndim, dims, spacing, image);
        auto s = make(ndim, dims, spacing, seeds);
        put(geodist::geodesic_distance(im, s, params(lambda, 1e10, iterations),
                                       policy(1, workers, 0, 100, 1e-6)),
            out);
    });
}

int ref_euclidean_distance(int ndim, const int* dims, const double* spacing, const float* seeds,
                           int iterations, int workers, float* out) {
    return guard([&] {
        auto s = make(ndim, dims, spacing, seeds);
        put(geodist::euclidean_distance(s, iterations, policy(1, workers, 0, 100, 1e-6)), out);
    });
}

int ref_signed_geodesic(int ndim, const int* dims, const double* spacing, const float* image,
                        const float* mask, double lambda, int iterations, int workers,
                        float* out) {
    return guard([&] {
        auto im = make(ndim, dims, spacing, image);
        auto m = make(ndim, dims, spacing, mask);
        put(geodist::signed_geodesic(im, m, params(lambda, 1e10, iterations),
                                     policy(1, workers, 0, 100, 1e-6)),
            out);
    });
}

// Every transform of transforms.hpp under one entry, with a full ScanPolicy
// (iterations or fixpoint): which = 0 generalized_geodesic, 1 geodesic_distance,
// 2 euclidean_distance, 3 signed_geodesic, 4 geodesic_dilate, 5 geodesic_erode,
// 6 gsf.  Reports TransformStats {rounds, converged, complement_empty}.
int ref_transform_ex(int which, int ndim, const int* dims, const double* spacing,
                     const float* image, const float* mask, double lambda, double nu,
                     int iterations, double theta, int to_fixpoint, int max_rounds, double tol,
                     int workers, float* out, int* rounds, int* converged, int* complement_empty) {
    return guard([&] {
        auto im = make(ndim, dims, spacing, image);
        auto m = make(ndim, dims, spacing, mask);
        const auto pr = params(lambda, nu, iterations);
        const auto pol = policy(1, workers, to_fixpoint, max_rounds, tol);
        geodist::TransformStats st;
        geodist::ScalarGrid r = [&] {
            switch (which) {
                case 0: return geodist::generalized_geodesic(im, m, pr, pol, &st);
                case 1: return geodist::geodesic_distance(im, m, pr, pol, &st);
                case 2: return geodist::euclidean_distance(m, iterations, pol, &st);
                case 3: return geodist::signed_geodesic(im, m, pr, pol, &st);
                case 4: return geodist::geodesic_dilate(im, m, theta, pr, pol, &st);
                case 5: return geodist::geodesic_erode(im, m, theta, pr, pol, &st);
                default: {
                    geodist::GsfParams gp;
                    gp.base = pr;
                    gp.theta = theta;
                    return geodist::gsf(im, m, gp, pol, &st);
                }
            }
        }();
        put(r, out);
        if (rounds) *rounds = st.rounds;
        if (converged) *converged = st.converged ? 1 : 0;
        if (complement_empty) *complement_empty = st.complement_empty ? 1 : 0;
    });
}

int ref_dijkstra_exact(int ndim, const int* dims, const double* spacing, const float* image,
                       const float* init, double lambda, float* out) {
    return guard([&] {
        auto im = make(ndim, dims, spacing, image);
        auto d = make(ndim, dims, spacing, init);
        put(geodist::dijkstra_exact(im, d, lambda), out);
    });
}

// Pass stencil as the reference computes it (metric.cpp:78-114): 3 or 9
// offsets in the reference's order, each (dz, dy, dx, rho).
int ref_pass_offsets(int ndim, const double* spacing, int axis, int orientation, int* dzyx,
                     double* rho, int* n) {
    return guard([&] {
        auto offs = geodist::pass_neighbor_offsets(geodist::PassDirection{axis, orientation},
                                                   ndim, std::span<const double>(spacing, ndim));
        *n = static_cast<int>(offs.size());
        for (std::size_t i = 0; i < offs.size(); ++i) {
            dzyx[3 * i + 0] = offs[i].dz;
            dzyx[3 * i + 1] = offs[i].dy;
            dzyx[3 * i + 2] = offs[i].dx;
            rho[i] = offs[i].rho;
        }
    });
}

}  // extern "C"

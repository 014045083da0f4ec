// C++ drop-in for the reference API (include/geodist/*.hpp) over the C-ABI.
// Validation mirrors the reference (same exception types, checked before any
// device work); every scan runs on the B200.  Engine::Serial / Engine::Oracle
// are CPU engines of the reference and are rejected: there is no CPU fallback.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>

#include "geodist/grid.hpp"
#include "geodist/metric.hpp"
#include "geodist/scan_parallel.hpp"
#include "geodist/transforms.hpp"
#include "geodist_b200.h"
#include "metric_host.hpp"

namespace geodist {

namespace {

void throw_status(int rc) {
    if (rc == GD_OK) return;
    const std::string msg = gd_last_error();
    if (rc == GD_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == GD_EMPTY_SEEDS) throw EmptySeedsError(msg);
    throw std::runtime_error("geodist_b200: " + msg);
}

gd_grid to_gd(const ScalarGrid& g) {
    gd_grid d{};
    d.ndim = g.ndim();
    for (int a = 0; a < g.ndim(); ++a) {
        d.dims[a] = g.extent(a);
        d.spacing[a] = g.spacing(a);
    }
    return d;
}

void require_match(const ScalarGrid& a, const ScalarGrid& b, const char* what) {
    if (!a.same_shape(b)) throw std::invalid_argument(std::string(what) + ": shape mismatch");
    if (!a.same_spacing(b)) throw std::invalid_argument(std::string(what) + ": spacing mismatch");
}

void require_device_engine(Engine e, const char* what) {
    if (e != Engine::Parallel)
        throw std::invalid_argument(std::string(what) + ": engine '" + engine_name(e) +
                                    "' is a CPU engine; geodist_b200 runs Engine::Parallel on the "
                                    "GPU only");
}

void require_workers(int workers) {
    if (workers < 1)
        throw std::invalid_argument("workers must be >= 1, got " + std::to_string(workers));
}

ScalarGrid with_spacing(const ScalarGrid& g, std::span<const double> spacing) {
    ScalarGrid out(g.ndim(), g.dims(), spacing, 0.0f);
    std::memcpy(out.data(), g.data(), g.size() * sizeof(float));
    return out;
}

}  // namespace

// ---------------------------------------------------------------- grid.hpp
ScalarGrid::ScalarGrid(int ndim, std::span<const int> dims, std::span<const double> spacing,
                       float fill) {
    if (ndim != 2 && ndim != 3)
        throw std::invalid_argument("grid rank must be 2 or 3, got " + std::to_string(ndim));
    if (dims.size() != static_cast<std::size_t>(ndim) ||
        spacing.size() != static_cast<std::size_t>(ndim)) {
        std::ostringstream m;
        m << "expected " << ndim << " dims and spacings, got " << dims.size() << " and "
          << spacing.size();
        throw std::invalid_argument(m.str());
    }
    ndim_ = ndim;
    offset_ = 3 - ndim;
    std::size_t total = 1;
    for (int a = 0; a < ndim; ++a) {
        if (dims[a] < 1)
            throw std::invalid_argument("grid extent must be >= 1, got " + std::to_string(dims[a]));
        if (!(spacing[a] > 0.0) || !std::isfinite(spacing[a]))
            throw std::invalid_argument("grid spacing must be finite and > 0, got " +
                                        std::to_string(spacing[a]));
        dims_[a + offset_] = dims[a];
        spacing_[a + offset_] = spacing[a];
        total *= static_cast<std::size_t>(dims[a]);
    }
    data_.assign(total, fill);
}

bool grids_approx_equal(const ScalarGrid& a, const ScalarGrid& b, double tol) {
    if (tol < 0.0) throw std::invalid_argument("tolerance must be >= 0");
    if (!a.same_shape(b) || !a.same_spacing(b)) return false;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const float x = a.data()[i], y = b.data()[i];
        const bool ix = x >= kInfSentinel, iy = y >= kInfSentinel;
        if (ix != iy) return false;
        if (!ix && std::abs(static_cast<double>(x) - static_cast<double>(y)) > tol) return false;
    }
    return true;
}

ScalarGrid grid_like(const ScalarGrid& like, float fill) {
    return ScalarGrid(like.ndim(), like.dims(), like.spacings(), fill);
}

void TransformParams::validate() const {
    if (!(lambda >= 0.0 && lambda <= 1.0))
        throw std::invalid_argument("lambda must lie in [0, 1], got " + std::to_string(lambda));
    if (!(nu >= 0.0)) throw std::invalid_argument("nu must be >= 0, got " + std::to_string(nu));
    if (iterations < 1)
        throw std::invalid_argument("iterations must be >= 1, got " + std::to_string(iterations));
}

// -------------------------------------------------------------- metric.hpp
std::vector<PassDirection> pass_sequence(int ndim) {
    if (ndim == 2) return {pass::top_bottom, pass::bottom_top, pass::left_right, pass::right_left};
    if (ndim == 3)
        return {pass::front_back, pass::back_front, pass::top_bottom,
                pass::bottom_top, pass::left_right, pass::right_left};
    throw std::invalid_argument("rank must be 2 or 3, got " + std::to_string(ndim));
}

bool direction_valid(PassDirection d, int ndim) {
    if (d.orientation != 1 && d.orientation != -1) return false;
    if (ndim == 2) return d.axis == 1 || d.axis == 2;
    if (ndim == 3) return d.axis >= 0 && d.axis <= 2;
    return false;
}

const char* direction_name(PassDirection d) {
    static const char* names[3][2] = {{"back-front", "front-back"},
                                      {"bottom-top", "top-bottom"},
                                      {"right-left", "left-right"}};
    if (d.axis < 0 || d.axis > 2 || (d.orientation != 1 && d.orientation != -1)) return "invalid";
    return names[d.axis][d.orientation > 0 ? 1 : 0];
}

namespace {
std::array<double, 3> canonical_spacing(int ndim, std::span<const double> spacing) {
    if (ndim != 2 && ndim != 3)
        throw std::invalid_argument("rank must be 2 or 3, got " + std::to_string(ndim));
    if (spacing.size() != static_cast<std::size_t>(ndim))
        throw std::invalid_argument("spacing length does not match rank");
    std::array<double, 3> s{1.0, 1.0, 1.0};
    for (int a = 0; a < ndim; ++a) s[a + 3 - ndim] = spacing[a];
    return s;
}

NeighborOffset offset_of(int dz, int dy, int dx, const std::array<double, 3>& s) {
    return NeighborOffset{dz, dy, dx, gdb::offset_rho(dz, dy, dx, s[0], s[1], s[2])};
}
}  // namespace

double step_cost(double ip, double iq, const NeighborOffset& o, double lambda) {
    if (!(lambda >= 0.0 && lambda <= 1.0))
        throw std::invalid_argument("lambda must lie in [0, 1], got " + std::to_string(lambda));
    const double di = ip - iq;
    return std::sqrt((1.0 - lambda) * o.rho * o.rho + lambda * di * di);
}

std::vector<NeighborOffset> pass_neighbor_offsets(PassDirection direction, int ndim,
                                                  std::span<const double> spacing) {
    if (!direction_valid(direction, ndim))
        throw std::invalid_argument("invalid pass direction for rank " + std::to_string(ndim));
    const auto s = canonical_spacing(ndim, spacing);
    std::array<int, 3> delta{0, 0, 0};
    delta[direction.axis] = -direction.orientation;
    int free_axes[2] = {0, 0}, nf = 0;
    for (int a = 0; a < 3; ++a)
        if (a != direction.axis && !(ndim == 2 && a == 0)) free_axes[nf++] = a;
    std::vector<NeighborOffset> out;
    if (ndim == 2) {
        for (int a = -1; a <= 1; ++a) {
            delta[free_axes[0]] = a;
            out.push_back(offset_of(delta[0], delta[1], delta[2], s));
        }
    } else {
        for (int a = -1; a <= 1; ++a)
            for (int b = -1; b <= 1; ++b) {
                delta[free_axes[0]] = a;
                delta[free_axes[1]] = b;
                out.push_back(offset_of(delta[0], delta[1], delta[2], s));
            }
    }
    return out;
}

std::vector<NeighborOffset> serial_neighbor_offsets(int ndim, ScanPhase phase,
                                                    std::span<const double> spacing) {
    const auto s = canonical_spacing(ndim, spacing);
    std::vector<NeighborOffset> out;
    const int zlo = ndim == 3 ? -1 : 0;
    for (int dz = zlo; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const bool causal = dz < 0 || (dz == 0 && (dy < 0 || (dy == 0 && dx < 0)));
                if (!causal) continue;
                const int sg = phase == ScanPhase::Forward ? 1 : -1;
                out.push_back(offset_of(sg * dz, sg * dy, sg * dx, s));
            }
    return out;
}

// ------------------------------------------------------- scan_parallel.hpp
const char* engine_name(Engine e) {
    switch (e) {
        case Engine::Serial: return "serial";
        case Engine::Parallel: return "parallel";
        case Engine::Oracle: return "oracle";
    }
    return "unknown";
}

namespace detail {

void directional_pass_inplace(ScalarGrid& dist, const ScalarGrid& image, PassDirection direction,
                              const TransformParams& params, int workers) {
    if (!image.same_shape(dist) || !image.same_spacing(dist))
        throw std::invalid_argument("directional_pass: image/distance shape or spacing mismatch");
    require_workers(workers);
    params.validate();
    if (!direction_valid(direction, image.ndim()))
        throw std::invalid_argument("invalid pass direction for rank " +
                                    std::to_string(image.ndim()));
    const gd_grid g = to_gd(image);
    throw_status(gd_directional_pass(&g, image.data(), dist.data(), direction.axis,
                                     direction.orientation, params.lambda, GD_MEM_HOST, nullptr));
}

void parallel_scan_inplace(const ScalarGrid& image, ScalarGrid& dist,
                           const TransformParams& params, int workers) {
    if (!image.same_shape(dist) || !image.same_spacing(dist))
        throw std::invalid_argument("directional_pass: image/distance shape or spacing mismatch");
    require_workers(workers);
    params.validate();
    const gd_grid g = to_gd(image);
    throw_status(gd_parallel_scan(&g, image.data(), dist.data(), params.lambda, params.iterations,
                                  GD_MEM_HOST, nullptr));
}

}  // namespace detail

ScalarGrid directional_pass(ScalarGrid dist, const ScalarGrid& image, PassDirection direction,
                            const TransformParams& params, int workers) {
    detail::directional_pass_inplace(dist, image, direction, params, workers);
    return dist;
}

ScalarGrid parallel_scan(const ScalarGrid& image, ScalarGrid dist, const TransformParams& params,
                         int workers) {
    detail::parallel_scan_inplace(image, dist, params, workers);
    return dist;
}

FixpointResult scan_to_fixpoint(const ScalarGrid& image, ScalarGrid dist,
                                const TransformParams& params, Engine engine, int max_rounds,
                                double tol, int workers) {
    if (engine != Engine::Serial && engine != Engine::Parallel)
        throw std::invalid_argument("scan_to_fixpoint: engine must be serial or parallel");
    if (max_rounds < 1)
        throw std::invalid_argument("max_rounds must be >= 1, got " + std::to_string(max_rounds));
    if (tol < 0.0) throw std::invalid_argument("tol must be >= 0");
    params.validate();
    require_device_engine(engine, "scan_to_fixpoint");
    if (!image.same_shape(dist) || !image.same_spacing(dist))
        throw std::invalid_argument("directional_pass: image/distance shape or spacing mismatch");
    require_workers(workers);
    const gd_grid g = to_gd(image);
    gd_stats st{};
    throw_status(gd_scan_to_fixpoint(&g, image.data(), dist.data(), params.lambda, max_rounds, tol,
                                     GD_MEM_HOST, nullptr, &st));
    FixpointResult r{std::move(dist), st.rounds, st.converged != 0, st.last_change};
    return r;
}

// ---------------------------------------------------------- transforms.hpp
void GsfParams::validate() const {
    base.validate();
    if (!(theta >= 0.0))
        throw std::invalid_argument("theta must be >= 0, got " + std::to_string(theta));
}

ScalarGrid init_hard_seeds(const ScalarGrid& seed_mask) {
    ScalarGrid dist = grid_like(seed_mask, kInfSentinel);
    std::size_t n = 0;
    for (std::size_t i = 0; i < seed_mask.size(); ++i)
        if (seed_mask.data()[i] >= 0.5f) {
            dist.data()[i] = 0.0f;
            ++n;
        }
    if (n == 0) throw EmptySeedsError("no seed cell at or above the 0.5 mask threshold");
    return dist;
}

ScalarGrid run_scan(const ScalarGrid& image, ScalarGrid dist, const TransformParams& params,
                    const ScanPolicy& policy, TransformStats* stats) {
    params.validate();
    require_device_engine(policy.engine, "run_scan");
    if (policy.to_fixpoint) {
        FixpointResult r = scan_to_fixpoint(image, std::move(dist), params, policy.engine,
                                            policy.max_rounds, policy.tol, policy.workers);
        if (stats) {
            stats->rounds += r.rounds_used;
            stats->converged = stats->converged && r.converged;
        }
        return std::move(r.dist);
    }
    detail::parallel_scan_inplace(image, dist, params, policy.workers);
    if (stats) stats->rounds += params.iterations;
    return dist;
}

namespace {

// ScanPolicy -> gd_policy (null for the default iterations mode)
struct PolicyArg {
    gd_policy p{};
    const gd_policy* ptr = nullptr;
    explicit PolicyArg(const ScanPolicy& pol) {
        if (pol.to_fixpoint) {
            p.to_fixpoint = 1;
            p.max_rounds = pol.max_rounds;
            p.tol = pol.tol;
            ptr = &p;
        }
    }
};

void add_stats(TransformStats* stats, const gd_stats& st, bool fixpoint) {
    if (!stats) return;
    stats->rounds += st.rounds;
    if (fixpoint) stats->converged = stats->converged && st.converged != 0;
    stats->complement_empty = stats->complement_empty || st.complement_empty != 0;
}

// Host-side checks the reference makes before any compute, shared by the
// transforms below (engine, workers; the data checks run on the device).
void require_policy(const ScanPolicy& policy, const char* what) {
    require_device_engine(policy.engine, what);
    require_workers(policy.workers);
    if (policy.to_fixpoint) {
        if (policy.max_rounds < 1)
            throw std::invalid_argument("max_rounds must be >= 1, got " +
                                        std::to_string(policy.max_rounds));
        if (policy.tol < 0.0) throw std::invalid_argument("tol must be >= 0");
    }
}

}  // namespace

// Every transform below runs on the B200 through the C-ABI: hard seeds, soft-mask
// init, thresholds, counts and the signed subtraction are device kernels; the
// only host work is the reference's argument validation.
ScalarGrid geodesic_distance(const ScalarGrid& image, const ScalarGrid& seed_mask,
                             const TransformParams& params, const ScanPolicy& policy,
                             TransformStats* stats) {
    require_match(image, seed_mask, "geodesic_distance");
    params.validate();
    require_policy(policy, "geodesic_distance");
    ScalarGrid out = grid_like(seed_mask, 0.0f);
    const gd_grid g = to_gd(image);
    const PolicyArg pa(policy);
    gd_stats st{};
    throw_status(gd_geodesic_distance(&g, image.data(), seed_mask.data(), params.lambda,
                                      params.iterations, pa.ptr, out.data(), GD_MEM_HOST, nullptr,
                                      &st));
    add_stats(stats, st, policy.to_fixpoint);
    return out;
}

ScalarGrid euclidean_distance(const ScalarGrid& seed_mask, int iterations,
                              const ScanPolicy& policy, TransformStats* stats) {
    TransformParams params;
    params.lambda = 0.0;
    params.iterations = iterations;
    params.validate();
    require_policy(policy, "euclidean_distance");
    ScalarGrid out = grid_like(seed_mask, 0.0f);
    const gd_grid g = to_gd(seed_mask);
    const PolicyArg pa(policy);
    gd_stats st{};
    throw_status(gd_euclidean_distance(&g, seed_mask.data(), iterations, pa.ptr, out.data(),
                                       GD_MEM_HOST, nullptr, &st));
    add_stats(stats, st, policy.to_fixpoint);
    return out;
}

ScalarGrid generalized_geodesic(const ScalarGrid& image, const ScalarGrid& soft_mask,
                                const TransformParams& params, const ScanPolicy& policy,
                                TransformStats* stats) {
    require_match(image, soft_mask, "generalized_geodesic");
    params.validate();
    require_policy(policy, "generalized_geodesic");
    // the mask-range check (transforms.cpp:22-28) runs fused with the soft-mask
    // init on the device and is reported before any result is copied back
    ScalarGrid out = grid_like(soft_mask, 0.0f);
    const gd_grid g = to_gd(image);
    const PolicyArg pa(policy);
    gd_stats st{};
    throw_status(gd_generalized_geodesic_ex(&g, 1, image.data(), soft_mask.data(), params.lambda,
                                            params.nu, params.iterations, pa.ptr, out.data(),
                                            GD_MEM_HOST, nullptr, &st));
    add_stats(stats, st, policy.to_fixpoint);
    return out;
}

ScalarGrid signed_geodesic(const ScalarGrid& image, const ScalarGrid& mask,
                           const TransformParams& params, const ScanPolicy& policy,
                           TransformStats* stats) {
    require_match(image, mask, "signed_geodesic");
    params.validate();
    require_policy(policy, "signed_geodesic");
    ScalarGrid out = grid_like(mask, 0.0f);
    const gd_grid g = to_gd(image);
    const PolicyArg pa(policy);
    gd_stats st{};
    throw_status(gd_signed_geodesic(&g, image.data(), mask.data(), params.lambda,
                                    params.iterations, pa.ptr, out.data(), GD_MEM_HOST, nullptr,
                                    &st));
    add_stats(stats, st, policy.to_fixpoint);
    return out;
}

ScalarGrid geodesic_dilate(const ScalarGrid& image, const ScalarGrid& mask, double theta,
                           const TransformParams& params, const ScanPolicy& policy,
                           TransformStats* stats) {
    if (!(theta >= 0.0)) throw std::invalid_argument("theta must be >= 0");
    require_match(image, mask, "geodesic_dilate");
    params.validate();
    require_policy(policy, "geodesic_dilate");
    ScalarGrid out = grid_like(mask, 0.0f);
    const gd_grid g = to_gd(image);
    const PolicyArg pa(policy);
    gd_stats st{};
    throw_status(gd_geodesic_dilate(&g, image.data(), mask.data(), theta, params.lambda, params.nu,
                                    params.iterations, pa.ptr, out.data(), GD_MEM_HOST, nullptr,
                                    &st));
    add_stats(stats, st, policy.to_fixpoint);
    return out;
}

ScalarGrid geodesic_erode(const ScalarGrid& image, const ScalarGrid& mask, double theta,
                          const TransformParams& params, const ScanPolicy& policy,
                          TransformStats* stats) {
    if (!(theta >= 0.0)) throw std::invalid_argument("theta must be >= 0");
    require_match(image, mask, "geodesic_erode");
    params.validate();
    require_policy(policy, "geodesic_erode");
    ScalarGrid out = grid_like(mask, 0.0f);
    const gd_grid g = to_gd(image);
    const PolicyArg pa(policy);
    gd_stats st{};
    throw_status(gd_geodesic_erode(&g, image.data(), mask.data(), theta, params.lambda, params.nu,
                                   params.iterations, pa.ptr, out.data(), GD_MEM_HOST, nullptr,
                                   &st));
    add_stats(stats, st, policy.to_fixpoint);
    return out;
}

ScalarGrid gsf(const ScalarGrid& image, const ScalarGrid& soft_mask, const GsfParams& params,
               const ScanPolicy& policy, TransformStats* stats) {
    params.validate();
    require_match(image, soft_mask, "gsf");
    require_policy(policy, "gsf");
    ScalarGrid out = grid_like(soft_mask, 0.0f);
    const gd_grid g = to_gd(image);
    const PolicyArg pa(policy);
    gd_stats st{};
    throw_status(gd_gsf_ex(&g, image.data(), soft_mask.data(), params.base.lambda, params.base.nu,
                           params.base.iterations, params.theta, pa.ptr, out.data(), GD_MEM_HOST,
                           nullptr, &st));
    add_stats(stats, st, policy.to_fixpoint);
    return out;
}

ScalarGrid generalised_geodesic2d(const ScalarGrid& image, const ScalarGrid& softmask, double v,
                                  double lambda, int iterations) {
    TransformParams p;
    p.lambda = lambda;
    p.nu = v;
    p.iterations = iterations;
    return generalized_geodesic(image, softmask, p, ScanPolicy{});
}

ScalarGrid generalised_geodesic3d(const ScalarGrid& image, const ScalarGrid& softmask,
                                  std::span<const double> spacing, double v, double lambda,
                                  int iterations) {
    TransformParams p;
    p.lambda = lambda;
    p.nu = v;
    p.iterations = iterations;
    return generalized_geodesic(with_spacing(image, spacing), with_spacing(softmask, spacing), p,
                                ScanPolicy{});
}

ScalarGrid GSF2d(const ScalarGrid& image, const ScalarGrid& softmask, double theta, double v,
                 double lambda, int iterations) {
    GsfParams p;
    p.base.lambda = lambda;
    p.base.nu = v;
    p.base.iterations = iterations;
    p.theta = theta;
    return gsf(image, softmask, p, ScanPolicy{});
}

ScalarGrid GSF3d(const ScalarGrid& image, const ScalarGrid& softmask, double theta,
                 std::span<const double> spacing, double v, double lambda, int iterations) {
    GsfParams p;
    p.base.lambda = lambda;
    p.base.nu = v;
    p.base.iterations = iterations;
    p.theta = theta;
    return gsf(with_spacing(image, spacing), with_spacing(softmask, spacing), p, ScanPolicy{});
}

std::vector<ScalarGrid> generalized_geodesic_batch(const std::vector<ScalarGrid>& images,
                                                   const std::vector<ScalarGrid>& soft_masks,
                                                   const TransformParams& params) {
    if (images.size() != soft_masks.size() || images.empty())
        throw std::invalid_argument("generalized_geodesic_batch: need equal, non-empty lists");
    params.validate();
    for (std::size_t b = 0; b < images.size(); ++b) {
        require_match(images[0], images[b], "generalized_geodesic_batch");
        require_match(images[b], soft_masks[b], "generalized_geodesic_batch");
    }
    const std::size_t n = images[0].size();
    std::vector<float> img(n * images.size()), msk(n * images.size()), out(n * images.size());
    for (std::size_t b = 0; b < images.size(); ++b) {
        std::memcpy(img.data() + b * n, images[b].data(), n * sizeof(float));
        std::memcpy(msk.data() + b * n, soft_masks[b].data(), n * sizeof(float));
    }
    const gd_grid g = to_gd(images[0]);
    throw_status(gd_generalized_geodesic_batched(&g, static_cast<int>(images.size()), img.data(),
                                                 msk.data(), params.lambda, params.nu,
                                                 params.iterations, out.data(), GD_MEM_HOST,
                                                 nullptr, nullptr));
    std::vector<ScalarGrid> res;
    res.reserve(images.size());
    for (std::size_t b = 0; b < images.size(); ++b) {
        res.push_back(grid_like(images[b], 0.0f));
        std::memcpy(res.back().data(), out.data() + b * n, n * sizeof(float));
    }
    return res;
}

}  // namespace geodist

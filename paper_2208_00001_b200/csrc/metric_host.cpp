#include "metric_host.hpp"

#include <cmath>

namespace gdb {

double offset_rho(int dz, int dy, int dx, double sz, double sy, double sx) {
    const double lz = dz * sz;
    const double ly = dy * sy;
    const double lx = dx * sx;
    return std::sqrt(std::fma(lx, lx, std::fma(lz, lz, ly * ly)));
}

double blend_c0(double lambda, double rho) { return (1.0 - lambda) * rho * rho; }

}  // namespace gdb

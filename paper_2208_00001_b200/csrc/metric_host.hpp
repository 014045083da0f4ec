// Host-side stencil coefficients, computed with exactly the operation order
// the reference's gcc -O3 -march=native build uses:
//   make_offset   metric.cpp:26-31   rho = sqrt(fma(lx, lx, fma(lz, lz, ly*ly)))
//   c0            scan_parallel.cpp:204   (1 - lambda) * rho * rho
// metric_host.cpp is compiled with -ffp-contract=off so these stay explicit.
#pragma once

namespace gdb {
double offset_rho(int dz, int dy, int dx, double sz, double sy, double sx);
double blend_c0(double lambda, double rho);
}  // namespace gdb

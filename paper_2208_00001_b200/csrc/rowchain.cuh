// Row-chain kernel (rowchain.cu): forward+backward pass pairs whose plane is a
// single row (2D images), one CTA per image, no inter-CTA hand-off.
#pragma once

#include <cuda_runtime.h>

#include "sweep.cuh"

namespace gdb {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kWarpLast = 31;
constexpr int kRowChainMaxWidth = 512 * kC;  // one thread per 4 columns, <= 512 threads

// p.nu must be 1; uses p.dist, p.image, p.vol_stride, p.ss, p.ns, p.nv, p.nvol
// (grid), p.first_orient, p.npass and the cost coefficients.
cudaError_t launch_row_chain(int kind, bool f64, const SweepParams& p, cudaStream_t s);

}  // namespace gdb

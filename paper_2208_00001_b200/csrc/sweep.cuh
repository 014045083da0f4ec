// Persistent directional-pass kernel for sm_100a.
//
// Replaces the reference's per-pass OpenMP plane loop
//   run_pass<K>          /root/reference/proj/src/scan_parallel.cpp:89-142
//   relax_row<K,Contig>  /root/reference/proj/src/scan_parallel.cpp:44-87
// and, for a forward+backward pair on one axis, two consecutive
// directional_pass_inplace calls (scan_parallel.cpp:298-318, :320-340).
//
// Geometry.  One launch sweeps axis "s" of a batch of volumes, optionally
// forward then backward.  The plane perpendicular to s has a slow axis u and a
// contiguous axis v.  Each CTA owns a TU x 64 tile of that plane (NWU warps
// stacked along u, R rows per warp, 2 consecutive v columns per lane) for the
// whole sweep and keeps the previous plane's new distances and intensities in
// registers.  In-plane neighbours come from warp shuffles (v +- 1), own
// registers (u +- 1 inside a warp) and shared memory (rows at warp borders).
//
// Staging.  An NST-deep ring of TMA boxes brings each upcoming plane's old
// distances (TU x 64) and intensities with a 1-voxel halo ((TU+2) x 72) into
// shared memory, completion tracked by one mbarrier per slot.
//
// Halo hand-off.  The 1-voxel ring of the previous plane owned by neighbour
// tiles arrives through global memory as tagged 64-bit words {f32 value, u32
// tag}: single-copy-atomic relaxed stores by the owner, relaxed polling loads
// by the reader until the tag equals the expected step.  No fences, no flags,
// no grid barrier.  The loads are issued before the interior of the plane is
// relaxed, so their latency hides behind that work; only the tile's border
// voxels wait for them.
//
// Arithmetic (bit-exact contract with the reference, which relaxes in f64 and
// stores f32 once per voxel per pass): rounding to f32 is monotone, so
// f32(min_k x_k) == min_k f32(x_k) and every candidate may be rounded to f32 on
// its own.
//   * Spatial (lambda == 0): candidates of one rho class are min-reduced in f32
//     first (exact: monotone), then one f64 add per class and one rounding.
//   * Intensity (lambda == 1): f32 `d_q + |I_p - I_q|` is exactly the
//     reference's f32(f64(d_q) + |di|) whenever I_p - I_q is exact in f32; the
//     host checks that per image (image_diff_exact) and otherwise selects the
//     f64 path.
//   * Blend: f32 arithmetic within the 1e-6 abs + 1e-5 rel tolerance; the f64
//     path (sqrt(fma(lambda*di, di, c0)) exactly as compiled in the reference)
//     when exact mode is requested.
#pragma once

#include <cuda.h>
#include <cstdint>

#include "gd_device.cuh"

namespace gdb {

enum CostKind : int { kSpatial = 0, kIntensity = 1, kBlend = 2 };

constexpr int kTV = 64;   // tile width along v (2 columns per lane)
constexpr int kIW = 72;   // intensity box width: v0-4 .. v0+67 (16-byte aligned)

struct SweepParams {
    float* dist;              // volume 0 of this launch
    long long vol_stride;     // elements between volumes
    long long ss, su;         // element strides of the sweep axis and of u (v stride = 1)
    int ns, nu, nv;           // extents
    int ntu, ntv;             // tiles per volume
    int nvol;                 // volumes in this launch
    int tma_sweep_dim;        // tensor-map dim carrying s (2: z-form, 1: y-form)
    int first_orient;         // +1 / -1
    int npass;                // 1 or 2 (second pass runs the opposite orientation)
    int fence_turn;           // emit fence.proxy.async on forward stores (npass == 2)
    uint32_t tag_base;
    unsigned long long* halo; // tagged halo words
    // Neighbour coefficients indexed (du+1)*3 + (dv+1).
    double rho[9];
    double c0[9];
    float c0_f[9];
    double lambda;
    float lambda_f;
};

struct SweepTileConfig {
    int R, NWU, NST;
};

// Host-side launch (defined in sweep.cu).
cudaError_t launch_sweep(int kind, bool f64, int R, int NWU, const CUtensorMap& tm_d,
                         const CUtensorMap& tm_i, const SweepParams& p, cudaStream_t stream);
size_t sweep_smem_bytes(int R, int NWU);
int sweep_max_coresident(int R, int NWU, int kind, bool f64);

}  // namespace gdb

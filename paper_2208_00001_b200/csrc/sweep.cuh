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
// contiguous axis v.  Each CTA owns a full-width strip of R rows of that plane
// (u in [u0, u0+R), every v) for the whole sweep: NWV warps side by side, each
// lane holding C = 4 consecutive columns of all R rows in registers.  Strips
// only have neighbours above and below, so there is no column halo at all:
// v +- 1 comes from warp shuffles, warp-edge columns from the neighbour warp's
// previous-step values in shared memory, u +- 1 inside the strip from the
// thread's own registers.
//
// Staging.  An NST-deep ring of TMA boxes brings each upcoming plane's old
// distances (R x 128 per warp) and intensities with a row halo and a 4-column
// margin ((R+2) x 136 per warp) into shared memory; one mbarrier per slot, each
// warp arms it with its own boxes.
//
// Halo hand-off.  The previous plane's row above and row below the strip come
// from the neighbouring strips through global memory as tagged 64-bit words
// {f32 value, u32 tag}: single-copy-atomic relaxed stores by the owner, relaxed
// loads by the reader until the tag equals the expected step.  Each lane loads
// exactly the 6 words (v-1 .. v+4) it needs, so the hand-off needs no shared
// memory and no barrier.  The loads are issued at the top of the step and only
// checked after the strip interior has been relaxed, which hides their latency
// (~750 cycles per hop measured, tools/micro/halo_latency.cu).
//
// Arithmetic (bit-exact contract with the reference, which relaxes in f64 and
// stores f32 once per voxel per pass): rounding to f32 is monotone, so
// f32(min_k x_k) == min_k f32(x_k) and every candidate may be rounded to f32 on
// its own.
//   * Spatial (lambda == 0): candidates of one rho class are min-reduced in f32
//     first (exact: monotone), then one f64 add per class and one rounding.
//   * Intensity (lambda == 1): f32 `d_q + |I_p - I_q|` is exactly the
//     reference's f32(f64(d_q) + |di|) whenever I_p - I_q is exact in f32; the
//     host checks that per image (image_check_kernel) and otherwise selects the
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

constexpr int kC = 4;            // columns per lane
constexpr int kWV = 32 * kC;     // columns per warp (128)
constexpr int kIW = kWV + 8;     // intensity box width per warp: v0w-4 .. v0w+131
constexpr int kMaxWarps = 16;    // strip width limit: 16 * 128 = 2048 columns

struct SweepParams {
    float* dist;              // volume 0 of this launch
    long long vol_stride;     // elements between volumes
    long long ss, su;         // element strides of the sweep axis and of u (v stride = 1)
    int ns, nu, nv;           // extents
    int ntu;                  // strips per volume
    int nvol;                 // volumes in this launch
    int nwv;                  // warps across the strip
    int tma_sweep_dim;        // tensor-map dim carrying s (2: z-form, 1: y-form)
    int first_orient;         // +1 / -1
    int npass;                // 1 or 2 (second pass runs the opposite orientation)
    int fence_turn;           // emit fence.proxy.async on forward stores (npass == 2)
    int cs;                   // thread-block cluster size: strips of one cluster exchange
                              // their halo rows through DSMEM (1 = every link via L2)
    uint32_t tag_base;
    unsigned long long* halo; // tagged halo words: [strip][parity][TOP|BOT][nwv*128]
    long long* trace;         // optional per-warp cycle counters (null in production)
    float* ghost;             // TB: forward ghost rows, [cta][TOP|BOT][n1/2+1][nwv*128]
    const float* image;       // plane-step fallback: intensities (same layout as dist)
    // Device-side gate (the asynchronous API decides on the device, no host sync):
    // the launch runs iff (*gate & gate_mask) == gate_want; gate == null: always.
    const int* gate;
    int gate_mask, gate_want;
    unsigned int* err;        // watchdog word (mapped host memory): a halo wait that exceeds
                              // the spin limit sets it and every later wait gives up, so a
                              // protocol failure ends the launch and is reported, never hangs
    int debug_flags;          // experiments only (GD_SWEEP_TRACE builds): 1 no spin, 2 no halo stores, 4 no halo loads
    // Neighbour coefficients indexed (du+1)*3 + (dv+1).
    double rho[9];
    double c0[9];
    float c0_f[9];
    float c0l_f[9];           // blend f32: c0 / lambda (cost = sqrt(lambda) * sqrt(di^2 + c0 / lambda))
    double lambda;
    float lambda_f;
    float sqrt_lambda_f;
};

// Gate bits written by decide_kernel (aux_kernels.cu) for one transform.
enum GateBits : int {
    kGateMaskBad = 1,   // soft mask outside [0, 1]: nothing runs, error reported (deferred)
    kGateF64 = 2,       // lambda = 1 image whose differences are not exact in f32: f64 path
    kGateSkip = 4,      // GSF erode with an empty complement: the transform is skipped
};

__device__ __forceinline__ bool gate_closed(const SweepParams& p) {
    return p.gate && ((__ldg(p.gate) & p.gate_mask) != p.gate_want);
}

// Host-side launch (defined in sweep.cu).  R = rows per strip; tb = the
// temporally blocked variant (halo every two planes; boxes with ghost rows:
// distances R + 2 rows from u0 - 1, intensities R + 4 rows from u0 - 2; halo
// 2 rows per side).
cudaError_t launch_sweep(int kind, bool f64, int R, bool tb, const CUtensorMap& tm_d,
                         const CUtensorMap& tm_i, const SweepParams& p, cudaStream_t stream);
// Warp rows (NWU) of the strip shape serving R rows at this width; 0 = none.
int sweep_warp_rows(int R, int nwv, int kind, bool f64 = false);
// Fallback for planes the persistent kernel cannot hold co-resident (more row
// strips than CTAs, or wider than kMaxWarps * 128 columns): one launch per
// plane step, plane s relaxed from plane sp, all `p.nvol` volumes at once.
cudaError_t launch_plane_step(int kind, bool f64, const SweepParams& p, int s, int sp,
                              cudaStream_t stream);
// Experiments: prefer strip shapes with this many rows per warp (-1 = per-kind default).
void sweep_set_rows_per_warp(int rw);
// Whether a thread-block-cluster (DSMEM halo) variant exists for this strip shape.
bool sweep_has_cluster(int R, int nwv, int kind);
// Whether a temporally blocked variant exists for this strip shape.
bool sweep_has_tb(int R, int nwv, int kind);
// Co-resident CTAs of the strip shape (cs > 1: in clusters of cs CTAs).
int sweep_max_coresident(int R, bool tb, int nwv, int kind, bool f64, int cs = 1);

}  // namespace gdb

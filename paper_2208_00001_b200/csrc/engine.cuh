// Host-side engine: per-device context, pass scheduler, transforms.
// All entry points take DEVICE pointers to B dense canonical volumes
// ([b][z][y][x], x fastest) and enqueue on `stream`; the C-ABI (capi.cpp)
// adds host-memory staging and the C++ drop-in (geodist_api.cpp) sits on top.
#pragma once

#include <cuda_runtime.h>

#include <string>

namespace gdb {

enum StatusCode : int {
    kOk = 0,
    kInvalidArgument = 1,  // std::invalid_argument in the reference
    kEmptySeeds = 2,       // geodist::EmptySeedsError
    kCudaError = 3,        // new: device failure (std::runtime_error in the C++ layer)
    kUnsupported = 4,      // new: shape the kernels cannot take (reported, never a CPU fallback)
};

struct Status {
    int code = kOk;
    std::string msg;
    bool ok() const { return code == kOk; }
    static Status Ok() { return {}; }
    static Status Invalid(std::string m) { return {kInvalidArgument, std::move(m)}; }
};

// Canonical grid: dims (D, H, W), spacing (sz, sy, sx); 2D grids have D = 1,
// sz = 1 (ScalarGrid's padding, grid.hpp:69-72 of the reference).
struct GridDesc {
    int ndim = 3;
    int D = 1, H = 1, W = 1;
    double sz = 1.0, sy = 1.0, sx = 1.0;
    long long voxels() const { return static_cast<long long>(D) * H * W; }
};

// Builds a GridDesc from the reference's logical (ndim-long) dims/spacing and
// validates it exactly like ScalarGrid's constructor (grid.cpp:10-39).
Status make_grid_desc(int ndim, const int* dims, const double* spacing, GridDesc* out);

struct ScanStats {
    int rounds = 0;
    bool converged = true;
    bool complement_empty = false;
    double last_change = 0.0;
    long long kernel_launches = 0;
};

// Arithmetic mode for 0 < lambda < 1 (Blend): f32 (default, within the
// 1e-6 abs + 1e-5 rel contract) or the f64 replica of the reference (bit-exact).
void set_exact_blend(bool on);
// Layout planner (per-pass storage layout, engine.cu plan_layouts) on / off.
void set_layout_plan(bool on);
bool exact_blend();

// ScanPolicy (transforms.hpp:24-30) for the parallel engine: a fixed number of
// iterations (default) or rounds to a fixpoint (scan_to_fixpoint semantics:
// one host synchronisation per round).
struct Policy {
    bool fixpoint = false;
    int max_rounds = 100;
    double tol = 1e-6;
};

// --- the hot path -----------------------------------------------------------
// One directional pass (scan_parallel.cpp:298-318).
Status directional_pass(const GridDesc& g, int B, const float* img, float* dist, int axis,
                        int orientation, double lambda, cudaStream_t s, ScanStats* st);
// parallel_scan_inplace (scan_parallel.cpp:320-340): iterations x pass_sequence.
Status parallel_scan(const GridDesc& g, int B, const float* img, float* dist, double lambda,
                     int iterations, cudaStream_t s, ScanStats* st);
// generalized_geodesic (transforms.cpp:143-158).
Status generalized_geodesic(const GridDesc& g, int B, const float* img, const float* mask,
                            float* out, double lambda, double nu, int iterations, cudaStream_t s,
                            ScanStats* st, const Policy& pol = Policy{});
// geodesic_distance / euclidean_distance / signed_geodesic (transforms.cpp:127-141,
// 160-183), hard seeds initialised on the device; no seed -> EmptySeedsError
// (deferred like every device-side finding).
Status geodesic_distance(const GridDesc& g, const float* img, const float* seeds, float* out,
                         double lambda, int iterations, const Policy& pol, cudaStream_t s,
                         ScanStats* st);
Status euclidean_distance(const GridDesc& g, const float* seeds, float* out, int iterations,
                          const Policy& pol, cudaStream_t s, ScanStats* st);
Status signed_geodesic(const GridDesc& g, const float* img, const float* mask, float* out,
                       double lambda, int iterations, const Policy& pol, cudaStream_t s,
                       ScanStats* st);
// geodesic_dilate / geodesic_erode (transforms.cpp:185-229).
Status geodesic_dilate(const GridDesc& g, const float* img, const float* mask, float* out,
                       double lambda, double nu, int iterations, double theta, const Policy& pol,
                       cudaStream_t s, ScanStats* st);
Status geodesic_erode(const GridDesc& g, const float* img, const float* mask, float* out,
                      double lambda, double nu, int iterations, double theta, const Policy& pol,
                      cudaStream_t s, ScanStats* st, bool sync_stats);
// gsf (transforms.cpp:231-238) = erode(dilate(M, theta), theta).  B must be 1.
// Asynchronous on the device (the erode's empty-complement skip is a device-side
// gate); sync_stats: synchronise at the end to report complement_empty and rounds.
Status gsf(const GridDesc& g, const float* img, const float* mask, float* out, double lambda,
           double nu, int iterations, double theta, cudaStream_t s, ScanStats* st,
           bool sync_stats, const Policy& pol = Policy{});
// Four chained transforms: gsf (closing) followed by the opening
// dilate(erode(.)) -- the upstream-style symmetric filter.
Status gsf_symmetric(const GridDesc& g, const float* img, const float* mask, float* out,
                     double lambda, double nu, int iterations, double theta, const Policy& pol,
                     cudaStream_t s, ScanStats* st, bool sync_stats);
// scan_to_fixpoint, parallel engine (scan_parallel.cpp:357-397).  B must be 1.
Status scan_to_fixpoint(const GridDesc& g, const float* img, float* dist, double lambda,
                        int max_rounds, double tol, cudaStream_t s, ScanStats* st);

// Synthetic benchmark input (tools/main.cpp:67-81) generated on the device.
Status fill_splitmix(float* out, long long n, unsigned long long seed, cudaStream_t s);

// Number of kernels this library has launched in this process (evidence for
// bench.py's gpu_launches).
long long kernel_launch_count();

// Launch log of the directional-pass kernels (tests assert which variant ran):
// one record per sweep launch group, in launch order, capped at kLaunchLogMax.
struct LaunchRec {
    int axis;       // canonical sweep axis: 0 z, 1 y, 2 x
    int npass;      // 1 or 2 (forward+backward pair)
    int kind;       // CostKind
    int f64;        // f64 arithmetic path
    int path;       // 0 persistent strip kernel, 1 row chain, 2 plane-step fallback
    int rows;       // R: rows per strip (0 for path 1/2)
    int nwv;        // warp columns per strip
    int nwu;        // warp rows per strip
    int cs;         // thread-block cluster size (1 = tagged-L2 links only)
    int ntu;        // strips per volume
    int nvol;       // volumes in this launch
    int grid;       // CTAs
    int tb;         // temporally blocked variant (halo every two planes)
    int layout;     // storage layout of the pass: 0 [z][y][x], 1 [x][z][y], 2 [y][x][z]
};
constexpr int kLaunchLogMax = 4096;
// Reads (and clears) this device's deferred-error word (mapped host memory, no
// stream synchronisation): kCudaError if a sweep launch enqueued since the last
// call gave up waiting for a neighbour (halo watchdog), kInvalidArgument if a
// transform found its soft mask outside [0, 1] (the asynchronous path decides
// that on the device).  Work still running may raise it later.
Status take_deferred();
// Copies up to `max` records (oldest first); returns the number logged.
int launch_log(LaunchRec* out, int max, bool reset);

// Per-launch CUDA-event profiling by kernel class (on the launching stream).
// kProfSweepTwin: the f64 twin of a lambda = 1 sweep, launched next to the f32
// one under the device-side gate (only one of the two does the work; for
// images whose differences are exact in f32 -- every benchmark image -- the
// twin leaves at once, so the sweep class holds the real launches).
enum ProfKind : int {
    kProfSweep = 0, kProfTranspose = 1, kProfInit = 2, kProfOther = 3, kProfSweepTwin = 4,
    kProfKinds = 5
};
void profile_enable(bool on);
// Collects finished launches (synchronising on their end events) and returns
// accumulated milliseconds, launch counts and algorithmic bytes per class
// (kProfKinds entries each).
void profile_read(double* ms, long long* count, double* bytes, bool reset);
// Per-launch (kind, ms) of the launches collected by the last profile_read
// (before its reset); returns the total number logged.
int profile_log(int* kinds, float* ms, int max);

}  // namespace gdb

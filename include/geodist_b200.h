/* geodist_b200 — C-ABI boundary of the B200-native generalised geodesic
 * distance transform (arXiv 2208.00001 / FastGeodis raster scan).
 *
 * Plain pointers and sizes only.  Every entry point validates on the host
 * first (same conditions as the reference, which throws before computing) and
 * returns a status code; gd_last_error() gives the message for the calling
 * thread.  Grids follow the reference's ScalarGrid convention
 * (/root/reference/proj/include/geodist/grid.hpp:15-74): `ndim` 2 or 3,
 * logical dims/spacing in (depth,) height, width order, row-major with width
 * fastest.  Batched calls take `batch` such grids back to back.
 *
 * Memory: `mem` = GD_MEM_HOST (pointers are host memory; the library stages
 * through the device and synchronises before returning, like the reference's
 * blocking calls) or GD_MEM_DEVICE (pointers are device memory on the current
 * CUDA device; work is enqueued on `stream` (a cudaStream_t, NULL = legacy
 * default stream) and the call returns without blocking).  Decisions that
 * depend on the data are taken on the device: the soft-mask range check, the
 * f32 / f64 choice for lambda = 1 and GSF's empty-complement skip set a gate
 * word the transform's kernels test.  Errors found that way (mask values
 * outside [0, 1]; the halo watchdog) are DEFERRED: they are returned by the
 * next call on the device or by gd_synchronize(), like CUDA's asynchronous
 * errors; host-memory calls check them before copying results back, so the
 * caller's output stays untouched on error as with the reference.  Only
 * scan_to_fixpoint (a host-side convergence loop, one sync per round) and
 * gd_gsf with a non-NULL `stats` (complement_empty needs the device count)
 * synchronise a device-memory call.
 *
 * There is no CPU fallback: if no CUDA device is usable every call returns
 * GD_CUDA_ERROR.
 */
#ifndef GEODIST_B200_H
#define GEODIST_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define GD_VERSION 1

enum gd_status {
    GD_OK = 0,
    GD_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
    GD_EMPTY_SEEDS = 2,      /* reference: geodist::EmptySeedsError (transforms.hpp:11-14) */
    GD_CUDA_ERROR = 3,       /* device failure; C++ layer throws std::runtime_error */
    GD_UNSUPPORTED = 4       /* reserved: every shape runs (planes beyond the persistent kernel's
                                co-residency or width limit take the plane-step fallback) */
};

enum gd_mem { GD_MEM_HOST = 0, GD_MEM_DEVICE = 1 };

typedef struct gd_grid {
    int ndim;          /* 2 or 3 */
    int dims[3];       /* first ndim entries used: (depth,) height, width */
    double spacing[3]; /* same order; finite and > 0 */
} gd_grid;

typedef struct gd_stats {
    int rounds;            /* TransformStats::rounds (transforms.hpp:33-37) */
    int converged;         /* TransformStats::converged */
    int complement_empty;  /* TransformStats::complement_empty */
    double last_change;    /* FixpointResult::last_change (scan_parallel.hpp:31-36) */
    long long kernel_launches;
} gd_stats;

/* generalized_geodesic — replaces geodist::generalized_geodesic
 * (/root/reference/proj/include/geodist/transforms.hpp:62-64, src/transforms.cpp:143-158):
 * out = scan(image, min(nu * soft_mask, 1e10)) with `iterations` rounds of the
 * directional passes.  `stats` may be NULL. */
int gd_generalized_geodesic(const gd_grid* grid, const float* image, const float* soft_mask,
                            double lambda, double nu, int iterations, float* out, int mem,
                            void* stream, gd_stats* stats);

/* Batched generalized_geodesic over `batch` independent grids of identical
 * shape (new: the reference has no batch entry; a loop over
 * generalized_geodesic is its equivalent). */
int gd_generalized_geodesic_batched(const gd_grid* grid, int batch, const float* images,
                                    const float* soft_masks, double lambda, double nu,
                                    int iterations, float* out, int mem, void* stream,
                                    gd_stats* stats);

/* gsf — replaces geodist::gsf (transforms.hpp:85-86, transforms.cpp:231-238):
 * geodesic_erode(geodesic_dilate(M, theta), theta); binary {0,1} output. */
int gd_gsf(const gd_grid* grid, const float* image, const float* soft_mask, double lambda,
           double nu, int iterations, double theta, float* out, int mem, void* stream,
           gd_stats* stats);

/* directional_pass — replaces geodist::directional_pass /
 * detail::directional_pass_inplace (scan_parallel.hpp:20-22,45-47): one pass
 * along canonical axis (0 depth, 1 height, 2 width) and orientation +-1,
 * relaxing `dist` in place. */
int gd_directional_pass(const gd_grid* grid, const float* image, float* dist, int axis,
                        int orientation, double lambda, int mem, void* stream);

/* parallel_scan — replaces geodist::parallel_scan / detail::parallel_scan_inplace
 * (scan_parallel.hpp:27-28,48-50): `iterations` rounds of pass_sequence(ndim),
 * in place on `dist`. */
int gd_parallel_scan(const gd_grid* grid, const float* image, float* dist, double lambda,
                     int iterations, int mem, void* stream);

/* scan_to_fixpoint with Engine::Parallel — replaces geodist::scan_to_fixpoint
 * (scan_parallel.hpp:40-43, scan_parallel.cpp:357-397), in place on `dist`. */
int gd_scan_to_fixpoint(const gd_grid* grid, const float* image, float* dist, double lambda,
                        int max_rounds, double tol, int mem, void* stream, gd_stats* stats);

/* ScanPolicy (transforms.hpp:24-30) for the parallel engine: NULL or
 * to_fixpoint = 0 -> `iterations` rounds of the pass sequence; to_fixpoint != 0
 * -> rounds until the largest change is <= tol, at most max_rounds
 * (scan_to_fixpoint semantics; one stream synchronisation per round). */
typedef struct gd_policy {
    int to_fixpoint;
    int max_rounds; /* >= 1 */
    double tol;     /* >= 0 */
} gd_policy;

/* generalized_geodesic / batched with a ScanPolicy (fixpoint mode: batch == 1). */
int gd_generalized_geodesic_ex(const gd_grid* grid, int batch, const float* images,
                               const float* soft_masks, double lambda, double nu, int iterations,
                               const gd_policy* policy, float* out, int mem, void* stream,
                               gd_stats* stats);

/* geodesic_distance — replaces geodist::geodesic_distance (transforms.hpp:41-44,
 * transforms.cpp:127-132): hard seeds where seed_mask >= 0.5 (init_hard_seeds,
 * :74-89, on the device), then the scan.  No seed -> GD_EMPTY_SEEDS. */
int gd_geodesic_distance(const gd_grid* grid, const float* image, const float* seed_mask,
                         double lambda, int iterations, const gd_policy* policy, float* out,
                         int mem, void* stream, gd_stats* stats);

/* euclidean_distance — replaces geodist::euclidean_distance (transforms.cpp:134-141):
 * lambda = 0 over a uniform image (no image argument: it is never read). */
int gd_euclidean_distance(const gd_grid* grid, const float* seed_mask, int iterations,
                          const gd_policy* policy, float* out, int mem, void* stream,
                          gd_stats* stats);

/* signed_geodesic — replaces geodist::signed_geodesic (transforms.cpp:160-183):
 * d(inside seeds [mask >= 0.5]) - d(outside seeds); either set empty ->
 * GD_EMPTY_SEEDS. */
int gd_signed_geodesic(const gd_grid* grid, const float* image, const float* mask, double lambda,
                       int iterations, const gd_policy* policy, float* out, int mem,
                       void* stream, gd_stats* stats);

/* geodesic_dilate / geodesic_erode — replace geodist::geodesic_dilate / _erode
 * (transforms.cpp:185-229): binary {0,1} outputs; erode reports an empty
 * complement in stats->complement_empty (GD_MEM_DEVICE: only when stats != NULL,
 * which synchronises). */
int gd_geodesic_dilate(const gd_grid* grid, const float* image, const float* mask, double theta,
                       double lambda, double nu, int iterations, const gd_policy* policy,
                       float* out, int mem, void* stream, gd_stats* stats);
int gd_geodesic_erode(const gd_grid* grid, const float* image, const float* mask, double theta,
                      double lambda, double nu, int iterations, const gd_policy* policy,
                      float* out, int mem, void* stream, gd_stats* stats);

/* gsf with a ScanPolicy. */
int gd_gsf_ex(const gd_grid* grid, const float* image, const float* soft_mask, double lambda,
              double nu, int iterations, double theta, const gd_policy* policy, float* out,
              int mem, void* stream, gd_stats* stats);

/* Upstream-style symmetric filter, four chained transforms (BASELINE.json's
 * "GSF3d ... four chained transforms"; the reference's gsf is the closing only):
 * opening(closing(M)) = dilate(erode(erode(dilate(M, theta), theta), theta), theta)
 * with the reference's geodesic_dilate / geodesic_erode semantics
 * (transforms.cpp:185-229).  No reference entry point: its oracle is the
 * composition of the reference's own dilate / erode calls. */
int gd_gsf_symmetric(const gd_grid* grid, const float* image, const float* soft_mask,
                     double lambda, double nu, int iterations, double theta,
                     const gd_policy* policy, float* out, int mem, void* stream, gd_stats* stats);

/* Blend (0 < lambda < 1) arithmetic: 0 = f32 (default; within 1e-6 abs +
 * 1e-5 rel of the reference), 1 = f64 replica of the reference (bit-exact). */
int gd_set_exact_blend(int on);

/* Storage-layout planner: 1 (default) = each pass runs on the layout that
 * minimises sequential plane steps plus rotations ([z][y][x], [x][z][y] or
 * [y][x][z]); 0 = the fixed plan ([z][y][x] for the z and y passes, [x][z][y]
 * for x).  Results are identical either way; tuning / testing switch
 * (GEODIST_LAYOUT_PLAN=0 at load). */
int gd_set_layout_plan(int on);

/* Per-launch CUDA-event profiling, recorded on each launch's own stream.
 * Classes: 0 sweep (the directional-pass kernel), 1 layout rotations
 * (transposes), 2 soft-mask init, 3 checks/thresholds, 4 the f64 twin of a
 * lambda = 1 sweep (launched beside the f32 one under the device-side gate;
 * it leaves at once when the image's differences are exact in f32).
 * gd_profile_read waits for the recorded launches and returns accumulated ms,
 * launch counts and algorithmic bytes (12 B/voxel/pass for the sweep, 8 at
 * lambda = 0) per class, 5 entries each. */
int gd_profile_enable(int on);
int gd_profile_read(double* ms5, long long* count5, double* bytes5, int reset);
/* Per-launch (class, ms) in launch order for the launches collected by the last
 * gd_profile_read (call it with reset = 0 first); returns the number logged. */
int gd_profile_log(int* kinds, float* ms, int max);

/* Launch log of the directional-pass kernels, one record per launch group in
 * launch order (at most 4096 kept): which kernel variant actually ran, so tests
 * can assert that the intended one did.  Copies up to `max` records into `out`,
 * returns how many are logged; `reset` != 0 clears the log afterwards. */
typedef struct gd_launch_rec {
    int axis;  /* sweep axis: 0 depth, 1 height, 2 width */
    int npass; /* 1 = one directional pass, 2 = forward+backward pair */
    int kind;  /* 0 spatial (lambda 0), 1 intensity (lambda 1), 2 blend */
    int f64;   /* f64 arithmetic path */
    int path;  /* 0 persistent strip kernel, 1 row chain (2D), 2 plane-step fallback */
    int rows;  /* rows per strip */
    int nwv;   /* warp columns per strip */
    int nwu;   /* warp rows per strip */
    int cs;    /* thread-block cluster size (1: halo links through L2 only) */
    int ntu;   /* strips per volume */
    int nvol;  /* volumes in the launch */
    int grid;  /* CTAs */
    int tb;    /* temporally blocked variant (halo exchanged every two planes) */
    int layout; /* storage layout the pass ran on: 0 [z][y][x] (caller's), 1 [x][z][y],
                   2 [y][x][z] (chosen per pass by the layout planner) */
} gd_launch_rec;
int gd_debug_launch_log(gd_launch_rec* out, int max, int reset);

/* Waits for `stream` and returns any deferred error of the work enqueued on
 * this device (GD_INVALID_ARGUMENT for a soft mask outside [0, 1],
 * GD_CUDA_ERROR for a CUDA error or the halo watchdog). */
int gd_synchronize(void* stream);

/* Utilities. */
/* Selects the CUDA device for this thread's subsequent calls (the library
 * carries its own CUDA runtime state; a caller's cudaSetDevice does not reach it). */
int gd_set_device(int device);
const char* gd_last_error(void);
int gd_version(void);
long long gd_kernel_launches(void);
/* Device-side SplitMix64 benchmark image (tools/main.cpp:67-81). */
int gd_fill_splitmix(float* device_out, long long n, unsigned long long seed, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GEODIST_B200_H */

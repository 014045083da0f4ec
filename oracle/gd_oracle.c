/* TEST INFRASTRUCTURE ONLY — see gd_oracle.h.
 *
 * A deliberately naive, obviously-correct restatement of the reference scan:
 * one plane at a time, every voxel reads only the previous plane plus its own
 * prior value, f64 relaxation and one f32 store per voxel per pass.  It is the
 * checker the CUDA path is compared against; it is never timed as the product.
 *
 * Reference anchors (file:line under /root/reference/proj):
 *   pass stencil / rho      src/metric.cpp:26-31, 78-114
 *   pass order              src/metric.cpp:35-44
 *   cost kinds              src/scan_common.hpp:17-21, 52-68
 *   relaxation arithmetic   src/scan_parallel.cpp:44-87 (relax_row)
 *   plane loop / bounds     src/scan_parallel.cpp:89-142 (run_pass)
 *   early exit n_sweep < 2  src/scan_parallel.cpp:308-310
 *   generalized_geodesic    src/transforms.cpp:143-158
 *   gsf chain               src/transforms.cpp:30-63, 185-238
 *   scan_to_fixpoint        src/scan_parallel.cpp:357-397
 *
 * Floating-point contract: built with -ffp-contract=off; the two places where
 * the reference's gcc -O3 -march=native build contracts into an FMA are
 * written as explicit fma() calls:
 *   rho^2  = fma(lx, lx, fma(lz, lz, ly*ly))      (make_offset)
 *   blend  = sqrt(fma(lambda*di, di, c0))          (relax_cost<Blend>)
 */
#include "gd_oracle.h"

#include <math.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#define GDO_INF_SENTINEL 1.0e10f

typedef struct {
    int dz, dy, dx;
    double rho;
} gdo_off;

static int canon(int ndim, const int* dims, const double* spacing, int cd[3], double cs[3]) {
    if (ndim != 2 && ndim != 3) return 1;
    cd[0] = cd[1] = cd[2] = 1;
    cs[0] = cs[1] = cs[2] = 1.0;
    for (int a = 0; a < ndim; ++a) {
        if (dims && dims[a] < 1) return 1;
        if (!(spacing[a] > 0.0) || !isfinite(spacing[a])) return 1;
        if (dims) cd[a + 3 - ndim] = dims[a];
        cs[a + 3 - ndim] = spacing[a];
    }
    return 0;
}

/* metric.cpp:26-31 */
static double make_rho(int dz, int dy, int dx, const double s[3]) {
    const double lz = dz * s[0];
    const double ly = dy * s[1];
    const double lx = dx * s[2];
    return sqrt(fma(lx, lx, fma(lz, lz, ly * ly)));
}

static int direction_valid(int axis, int orientation, int ndim) {
    if (orientation != 1 && orientation != -1) return 0;
    if (ndim == 2) return axis == 1 || axis == 2;
    return axis >= 0 && axis <= 2;
}

/* metric.cpp:78-114: delta[axis] = -orientation; free axes a (outer), b (inner). */
static int pass_offsets(int ndim, const double s[3], int axis, int orientation, gdo_off* out) {
    int delta[3] = {0, 0, 0};
    int free_axes[2] = {0, 0};
    int n_free = 0, n = 0;
    delta[axis] = -orientation;
    for (int a = 0; a < 3; ++a)
        if (a != axis && !(ndim == 2 && a == 0)) free_axes[n_free++] = a;
    if (ndim == 2) {
        for (int a = -1; a <= 1; ++a) {
            delta[free_axes[0]] = a;
            out[n].dz = delta[0]; out[n].dy = delta[1]; out[n].dx = delta[2];
            out[n].rho = make_rho(delta[0], delta[1], delta[2], s);
            ++n;
        }
    } else {
        for (int a = -1; a <= 1; ++a)
            for (int b = -1; b <= 1; ++b) {
                delta[free_axes[0]] = a;
                delta[free_axes[1]] = b;
                out[n].dz = delta[0]; out[n].dy = delta[1]; out[n].dx = delta[2];
                out[n].rho = make_rho(delta[0], delta[1], delta[2], s);
                ++n;
            }
    }
    return n;
}

int gdo_pass_offsets(int ndim, const double* spacing, int axis, int orientation, int* dzyx,
                     double* rho, int* n) {
    int cd[3];
    double cs[3];
    gdo_off offs[9];
    if (canon(ndim, NULL, spacing, cd, cs) || !direction_valid(axis, orientation, ndim)) return 1;
    *n = pass_offsets(ndim, cs, axis, orientation, offs);
    for (int k = 0; k < *n; ++k) {
        dzyx[3 * k] = offs[k].dz;
        dzyx[3 * k + 1] = offs[k].dy;
        dzyx[3 * k + 2] = offs[k].dx;
        rho[k] = offs[k].rho;
    }
    return 0;
}

/* One directional pass, in place.  scan_parallel.cpp:298-318 + run_pass + relax_row. */
static void pass_inplace(const int d[3], const double s[3], int ndim, const float* img,
                         float* dist, int axis, int orientation, double lambda) {
    const int n_sweep = d[axis];
    if (n_sweep < 2) return;
    gdo_off offs[9];
    const int n_offs = pass_offsets(ndim, s, axis, orientation, offs);
    double c0[9];
    for (int k = 0; k < n_offs; ++k) c0[k] = (1.0 - lambda) * offs[k].rho * offs[k].rho;
    const int kind = lambda == 0.0 ? 0 : (lambda == 1.0 ? 1 : 2);
    const ptrdiff_t sy = d[2], sz = (ptrdiff_t)d[1] * d[2];

    for (int step = 1; step < n_sweep; ++step) {
        const int sidx = orientation > 0 ? step : n_sweep - 1 - step;
        int lo[3] = {0, 0, 0}, hi[3] = {d[0], d[1], d[2]};
        lo[axis] = sidx;
        hi[axis] = sidx + 1;
#pragma omp parallel for collapse(2) schedule(static)
        for (int z = lo[0]; z < hi[0]; ++z)
            for (int y = lo[1]; y < hi[1]; ++y)
                for (int x = lo[2]; x < hi[2]; ++x) {
                    const ptrdiff_t p = z * sz + y * sy + x;
                    double best = (double)dist[p];
                    for (int k = 0; k < n_offs; ++k) {
                        const int zz = z + offs[k].dz, yy = y + offs[k].dy, xx = x + offs[k].dx;
                        if (zz < 0 || zz >= d[0] || yy < 0 || yy >= d[1] || xx < 0 || xx >= d[2])
                            continue;
                        const ptrdiff_t q = zz * sz + yy * sy + xx;
                        double cost;
                        if (kind == 0) {
                            cost = offs[k].rho;
                        } else {
                            const double di = (double)img[p] - (double)img[q];
                            cost = kind == 1 ? fabs(di) : sqrt(fma(lambda * di, di, c0[k]));
                        }
                        const double cand = (double)dist[q] + cost;
                        if (cand < best) best = cand;
                    }
                    dist[p] = (float)best;
                }
    }
}

static int seq3[6][2] = {{0, 1}, {0, -1}, {1, 1}, {1, -1}, {2, 1}, {2, -1}};
static int seq2[4][2] = {{1, 1}, {1, -1}, {2, 1}, {2, -1}};

static int params_ok(double lambda, double nu, int iterations) {
    return lambda >= 0.0 && lambda <= 1.0 && nu >= 0.0 && iterations >= 1;
}

static void scan_inplace(const int d[3], const double s[3], int ndim, const float* img,
                         float* dist, double lambda, int iterations) {
    const int n_dir = ndim == 3 ? 6 : 4;
    for (int it = 0; it < iterations; ++it)
        for (int i = 0; i < n_dir; ++i) {
            const int* dir = ndim == 3 ? seq3[i] : seq2[i];
            pass_inplace(d, s, ndim, img, dist, dir[0], dir[1], lambda);
        }
}

int gdo_directional_pass(int ndim, const int* dims, const double* spacing, const float* image,
                         float* dist, int axis, int orientation, double lambda) {
    int cd[3];
    double cs[3];
    if (canon(ndim, dims, spacing, cd, cs)) return 1;
    if (!params_ok(lambda, 0.0, 1) || !direction_valid(axis, orientation, ndim)) return 1;
    pass_inplace(cd, cs, ndim, image, dist, axis, orientation, lambda);
    return 0;
}

int gdo_parallel_scan(int ndim, const int* dims, const double* spacing, const float* image,
                      float* dist, double lambda, int iterations) {
    int cd[3];
    double cs[3];
    if (canon(ndim, dims, spacing, cd, cs) || !params_ok(lambda, 0.0, iterations)) return 1;
    scan_inplace(cd, cs, ndim, image, dist, lambda, iterations);
    return 0;
}

static size_t volume(const int d[3]) { return (size_t)d[0] * d[1] * d[2]; }

/* transforms.cpp:143-158 */
int gdo_generalized_geodesic(int ndim, const int* dims, const double* spacing,
                             const float* image, const float* mask, double lambda, double nu,
                             int iterations, float* out) {
    int cd[3];
    double cs[3];
    if (canon(ndim, dims, spacing, cd, cs) || !params_ok(lambda, nu, iterations)) return 1;
    const size_t n = volume(cd);
    for (size_t i = 0; i < n; ++i)
        if (!(mask[i] >= 0.0f && mask[i] <= 1.0f)) return 1;
    for (size_t i = 0; i < n; ++i) {
        const double v = nu * (double)mask[i];
        out[i] = (float)(v < (double)GDO_INF_SENTINEL ? v : (double)GDO_INF_SENTINEL);
    }
    scan_inplace(cd, cs, ndim, image, out, lambda, iterations);
    return 0;
}

/* transforms.cpp:30-63, 185-238: gsf = erode(dilate(M, theta), theta). */
int gdo_gsf(int ndim, const int* dims, const double* spacing, const float* image,
            const float* mask, double lambda, double nu, int iterations, double theta,
            float* out, int* rounds, int* complement_empty) {
    int cd[3];
    double cs[3];
    if (canon(ndim, dims, spacing, cd, cs) || !params_ok(lambda, nu, iterations)) return 1;
    if (!(theta >= 0.0)) return 1;
    const size_t n = volume(cd);
    float* src = (float*)malloc(n * sizeof(float));
    float* dist = (float*)malloc(n * sizeof(float));
    int r = 0;
    *complement_empty = 0;
    /* dilate: sources S = [M >= 0.5]; soft mask for the transform = complement(S). */
    for (size_t i = 0; i < n; ++i) src[i] = mask[i] >= 0.5f ? 0.0f : 1.0f;
    gdo_generalized_geodesic(ndim, dims, spacing, image, src, lambda, nu, iterations, dist);
    r += iterations;
    for (size_t i = 0; i < n; ++i) out[i] = (double)dist[i] <= theta ? 1.0f : 0.0f;
    /* erode: kept K = [dil >= 0.5]; sources = complement(K); transform mask = K. */
    size_t n_src = 0;
    for (size_t i = 0; i < n; ++i) n_src += out[i] >= 0.5f ? 0 : 1;
    if (n_src == 0) {
        *complement_empty = 1;
    } else {
        for (size_t i = 0; i < n; ++i) src[i] = out[i] >= 0.5f ? 1.0f : 0.0f;
        gdo_generalized_geodesic(ndim, dims, spacing, image, src, lambda, nu, iterations, dist);
        r += iterations;
        for (size_t i = 0; i < n; ++i) out[i] = (double)dist[i] > theta ? 1.0f : 0.0f;
    }
    free(src);
    free(dist);
    if (rounds) *rounds = r;
    return 0;
}

/* scan_parallel.cpp:357-397 (parallel engine only). */
int gdo_scan_to_fixpoint(int ndim, const int* dims, const double* spacing, const float* image,
                         float* dist, double lambda, int max_rounds, double tol,
                         int* rounds_used, int* converged, double* last_change) {
    int cd[3];
    double cs[3];
    if (canon(ndim, dims, spacing, cd, cs) || !params_ok(lambda, 0.0, 1)) return 1;
    if (max_rounds < 1 || !(tol >= 0.0)) return 1;
    const size_t n = volume(cd);
    float* before = (float*)malloc(n * sizeof(float));
    *rounds_used = 0;
    *converged = 0;
    *last_change = 0.0;
    while (*rounds_used < max_rounds) {
        memcpy(before, dist, n * sizeof(float));
        scan_inplace(cd, cs, ndim, image, dist, lambda, 1);
        ++*rounds_used;
        double change = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const double c = (double)before[i] - (double)dist[i];
            if (c > change) change = c;
        }
        *last_change = change;
        if (change <= tol) {
            *converged = 1;
            break;
        }
    }
    free(before);
    return 0;
}

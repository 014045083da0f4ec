// extern "C" boundary (include/geodist_b200.h) over the device engine.
// Host-memory calls stage through cached device buffers and synchronise, the
// way the reference's calls block; device-memory calls enqueue on the caller's
// stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/geodist_b200.h"
#include "aux_kernels.cuh"
#include "engine.cuh"

namespace gdb {
int sweep_max_coresident(int R, bool tb, int nwv, int kind, bool f64, int cs);  // sweep.cu
}

namespace {

thread_local std::string t_err;

int fail(const gdb::Status& s) {
    t_err = s.msg;
    return s.code;
}

int fail(int code, const std::string& m) {
    t_err = m;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    t_err = std::string(what) + ": " + cudaGetErrorString(e);
    return GD_CUDA_ERROR;
}

struct HostStage {
    std::mutex mu;
    void* p[3] = {nullptr, nullptr, nullptr};
    size_t n[3] = {0, 0, 0};
    bool ensure(int i, size_t bytes) {
        if (bytes <= n[i]) return true;
        if (p[i]) cudaFree(p[i]);
        p[i] = nullptr;
        n[i] = 0;
        if (cudaMalloc(&p[i], bytes) != cudaSuccess) return false;
        n[i] = bytes;
        return true;
    }
};

HostStage& stage() {
    static HostStage st[64];
    int dev = 0;
    cudaGetDevice(&dev);
    return st[dev & 63];
}

int check_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(GD_CUDA_ERROR, "no CUDA device available (geodist_b200 has no CPU fallback)");
    return GD_OK;
}

void fill_stats(gd_stats* out, const gdb::ScanStats& st) {
    if (!out) return;
    out->rounds = st.rounds;
    out->converged = st.converged ? 1 : 0;
    out->complement_empty = st.complement_empty ? 1 : 0;
    out->last_change = st.last_change;
    out->kernel_launches = st.kernel_launches;
}

int grid_of(const gd_grid* g, gdb::GridDesc* d) {
    if (!g) return fail(GD_INVALID_ARGUMENT, "null grid");
    gdb::Status s = gdb::make_grid_desc(g->ndim, g->dims, g->spacing, d);
    return s.ok() ? GD_OK : fail(s);
}

// Runs `fn(img, aux, io, stream)` on device pointers, staging host buffers.
// n_in_img/n_in_aux/n_io are element counts; io_in: copy io in before the call.
template <class F>
int run(int mem, void* stream, long long n, const float* img, const float* aux, float* io,
        bool io_in, F&& fn) {
    if (int rc = check_device()) return rc;
    if (mem == GD_MEM_DEVICE) {
        // asynchronous: a deferred error of earlier work on this device (halo
        // watchdog, soft mask out of range) is reported here, before enqueuing more
        gdb::Status w = gdb::take_deferred();
        if (!w.ok()) return fail(w);
        gdb::Status s = fn(img, aux, io, static_cast<cudaStream_t>(stream));
        return s.ok() ? GD_OK : fail(s);
    }
    if (mem != GD_MEM_HOST) return fail(GD_INVALID_ARGUMENT, "mem must be GD_MEM_HOST or GD_MEM_DEVICE");
    HostStage& hs = stage();
    std::lock_guard<std::mutex> lk(hs.mu);
    const size_t bytes = static_cast<size_t>(n) * sizeof(float);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!hs.ensure(0, bytes) || !hs.ensure(1, bytes) || !hs.ensure(2, bytes))
        return fail(GD_CUDA_ERROR, "device allocation failed");
    float* d_img = static_cast<float*>(hs.p[0]);
    float* d_aux = static_cast<float*>(hs.p[1]);
    float* d_io = static_cast<float*>(hs.p[2]);
    cudaError_t e;
    if (img && (e = cudaMemcpyAsync(d_img, img, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return cuda_fail(e, "H2D image");
    if (aux && (e = cudaMemcpyAsync(d_aux, aux, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return cuda_fail(e, "H2D mask");
    if (io_in && (e = cudaMemcpyAsync(d_io, io, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return cuda_fail(e, "H2D dist");
    gdb::Status st = fn(img ? d_img : nullptr, aux ? d_aux : nullptr, d_io, s);
    if (!st.ok()) {
        cudaStreamSynchronize(s);
        return fail(st);
    }
    // The reference validates before computing and leaves the caller's output
    // untouched on error: check the device's deferred-error word before the D2H.
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "stream sync");
    gdb::Status w = gdb::take_deferred();
    if (!w.ok()) return fail(w);
    if ((e = cudaMemcpyAsync(io, d_io, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e, "D2H result");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "stream sync");
    return GD_OK;
}

// Batched host-memory calls pipeline over chunks of volumes (volumes are
// independent): chunk k's H2D on a copy-in stream, its transform on the compute
// stream, its D2H on a copy-out stream, each ordered by events, with three
// device staging slots -- so PCIe in, PCIe out (full duplex) and compute overlap.
// The transforms are enqueued without host synchronisation (the device-side
// gates), so the whole pipeline is issued up front.  On a deferred error the
// caller's output may hold partial results (the single-volume path leaves it
// untouched).
struct Pipeline {
    std::mutex mu;
    cudaStream_t in = nullptr, comp = nullptr, out = nullptr;
    void* p[3][3] = {};
    size_t n[3] = {0, 0, 0};
    cudaEvent_t ev_in[3] = {}, ev_comp[3] = {}, ev_out[3] = {};
    bool ready = false;
    bool init() {
        if (ready) return true;
        if (cudaStreamCreateWithFlags(&in, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking) != cudaSuccess)
            return false;
        for (int k = 0; k < 3; ++k)
            if (cudaEventCreateWithFlags(&ev_in[k], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_comp[k], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_out[k], cudaEventDisableTiming) != cudaSuccess)
                return false;
        ready = true;
        return true;
    }
    bool ensure(int slot, size_t bytes) {
        if (bytes <= n[slot]) return true;
        for (int a = 0; a < 3; ++a) {
            if (p[slot][a]) cudaFree(p[slot][a]);
            p[slot][a] = nullptr;
        }
        n[slot] = 0;
        for (int a = 0; a < 3; ++a)
            if (cudaMalloc(&p[slot][a], bytes) != cudaSuccess) return false;
        n[slot] = bytes;
        return true;
    }
};

Pipeline& pipeline() {
    static Pipeline pl[64];
    int dev = 0;
    cudaGetDevice(&dev);
    return pl[dev & 63];
}

// fn(img, mask, out, nvol, stream) transforms nvol volumes on device pointers.
template <class F>
int run_batched_host(long long vol_elems, int batch, const float* img, const float* mask,
                     float* out, void* user_stream, F&& fn) {
    if (int rc = check_device()) return rc;
    Pipeline& pl = pipeline();
    std::lock_guard<std::mutex> lk(pl.mu);
    if (!pl.init()) return fail(GD_CUDA_ERROR, "pipeline streams");
    // ~8 chunks of at least 64 MB per array: enough to overlap, few enough to
    // keep launch groups full
    const long long vol_bytes = vol_elems * static_cast<long long>(sizeof(float));
    int per = std::max(1, (batch + 7) / 8);
    while (per < batch && static_cast<long long>(per) * vol_bytes < (64ll << 20)) ++per;
    const int chunks = (batch + per - 1) / per;
    cudaError_t e;
    cudaStream_t us = static_cast<cudaStream_t>(user_stream);
    // the caller's stream ordering: start after its pending work
    if ((e = cudaEventRecord(pl.ev_out[2], us)) != cudaSuccess) return cuda_fail(e, "event");
    if ((e = cudaStreamWaitEvent(pl.in, pl.ev_out[2], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    for (int c = 0; c < chunks; ++c) {
        const int slot = c % 3;
        const int b0 = c * per, nv = std::min(per, batch - b0);
        const size_t bytes = static_cast<size_t>(nv) * vol_bytes;
        if (c >= 3) {  // the slot's previous chunk must have left it
            if ((e = cudaStreamWaitEvent(pl.in, pl.ev_comp[slot], 0)) != cudaSuccess ||
                (e = cudaStreamWaitEvent(pl.in, pl.ev_out[slot], 0)) != cudaSuccess)
                return cuda_fail(e, "pipeline wait");
        }
        if (!pl.ensure(slot, static_cast<size_t>(per) * vol_bytes))
            return fail(GD_CUDA_ERROR, "device allocation failed");
        float* di = static_cast<float*>(pl.p[slot][0]);
        float* dm = static_cast<float*>(pl.p[slot][1]);
        float* dout = static_cast<float*>(pl.p[slot][2]);
        const size_t off = static_cast<size_t>(b0) * vol_elems;
        if ((e = cudaMemcpyAsync(di, img + off, bytes, cudaMemcpyHostToDevice, pl.in)) != cudaSuccess ||
            (e = cudaMemcpyAsync(dm, mask + off, bytes, cudaMemcpyHostToDevice, pl.in)) != cudaSuccess ||
            (e = cudaEventRecord(pl.ev_in[slot], pl.in)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(pl.comp, pl.ev_in[slot], 0)) != cudaSuccess)
            return cuda_fail(e, "pipeline H2D");
        gdb::Status st = fn(di, dm, dout, nv, pl.comp);
        if (!st.ok()) {
            cudaDeviceSynchronize();
            return fail(st);
        }
        if ((e = cudaEventRecord(pl.ev_comp[slot], pl.comp)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(pl.out, pl.ev_comp[slot], 0)) != cudaSuccess ||
            (e = cudaMemcpyAsync(out + off, dout, bytes, cudaMemcpyDeviceToHost, pl.out)) != cudaSuccess ||
            (e = cudaEventRecord(pl.ev_out[slot], pl.out)) != cudaSuccess)
            return cuda_fail(e, "pipeline D2H");
    }
    if ((e = cudaStreamSynchronize(pl.out)) != cudaSuccess ||
        (e = cudaStreamSynchronize(pl.comp)) != cudaSuccess)
        return cuda_fail(e, "stream sync");
    gdb::Status w = gdb::take_deferred();
    return w.ok() ? GD_OK : fail(w);
}

int policy_of(const gd_policy* p, gdb::Policy* out) {
    *out = gdb::Policy{};
    if (!p || !p->to_fixpoint) return GD_OK;
    if (p->max_rounds < 1)
        return fail(GD_INVALID_ARGUMENT, "max_rounds must be >= 1, got " + std::to_string(p->max_rounds));
    if (!(p->tol >= 0.0)) return fail(GD_INVALID_ARGUMENT, "tol must be >= 0");
    out->fixpoint = true;
    out->max_rounds = p->max_rounds;
    out->tol = p->tol;
    return GD_OK;
}

}  // namespace

extern "C" {

const char* gd_last_error(void) { return t_err.c_str(); }
int gd_version(void) { return GD_VERSION; }
long long gd_kernel_launches(void) { return gdb::kernel_launch_count(); }

int gd_set_layout_plan(int on) {
    gdb::set_layout_plan(on != 0);
    return GD_OK;
}

int gd_set_exact_blend(int on) {
    gdb::set_exact_blend(on != 0);
    return GD_OK;
}

int gd_generalized_geodesic_batched(const gd_grid* grid, int batch, const float* images,
                                    const float* soft_masks, double lambda, double nu,
                                    int iterations, float* out, int mem, void* stream,
                                    gd_stats* stats) {
    return gd_generalized_geodesic_ex(grid, batch, images, soft_masks, lambda, nu, iterations,
                                      nullptr, out, mem, stream, stats);
}

int gd_generalized_geodesic_ex(const gd_grid* grid, int batch, const float* images,
                               const float* soft_masks, double lambda, double nu, int iterations,
                               const gd_policy* policy, float* out, int mem, void* stream,
                               gd_stats* stats) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    gdb::Policy pol;
    if (int rc = policy_of(policy, &pol)) return rc;
    if (batch < 1) return fail(GD_INVALID_ARGUMENT, "batch must be >= 1");
    if (!images || !soft_masks || !out) return fail(GD_INVALID_ARGUMENT, "null buffer");
    gdb::ScanStats st;
    int rc;
    if (mem == GD_MEM_HOST && batch >= 2 && !pol.fixpoint) {
        // validate before anything is enqueued (the engine repeats it per chunk)
        // (TransformParams::validate, grid.cpp:67-78)
        if (!(lambda >= 0.0 && lambda <= 1.0))
            return fail(GD_INVALID_ARGUMENT, "lambda must lie in [0, 1], got " + std::to_string(lambda));
        if (!(nu >= 0.0)) return fail(GD_INVALID_ARGUMENT, "nu must be >= 0, got " + std::to_string(nu));
        if (iterations < 1)
            return fail(GD_INVALID_ARGUMENT, "iterations must be >= 1, got " + std::to_string(iterations));
        rc = run_batched_host(g.voxels(), batch, images, soft_masks, out, stream,
                              [&](const float* i, const float* m, float* o, int nv,
                                  cudaStream_t s) {
                                  gdb::ScanStats cs;
                                  gdb::Status r = gdb::generalized_geodesic(
                                      g, nv, i, m, o, lambda, nu, iterations, s, &cs, pol);
                                  st.rounds = cs.rounds;
                                  st.kernel_launches += cs.kernel_launches;
                                  return r;
                              });
    } else {
        rc = run(mem, stream, g.voxels() * batch, images, soft_masks, out, false,
                 [&](const float* i, const float* m, float* o, cudaStream_t s) {
                     return gdb::generalized_geodesic(g, batch, i, m, o, lambda, nu, iterations,
                                                      s, &st, pol);
                 });
    }
    fill_stats(stats, st);
    return rc;
}

int gd_geodesic_distance(const gd_grid* grid, const float* image, const float* seed_mask,
                         double lambda, int iterations, const gd_policy* policy, float* out,
                         int mem, void* stream, gd_stats* stats) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    gdb::Policy pol;
    if (int rc = policy_of(policy, &pol)) return rc;
    if (!image || !seed_mask || !out) return fail(GD_INVALID_ARGUMENT, "null buffer");
    gdb::ScanStats st;
    int rc = run(mem, stream, g.voxels(), image, seed_mask, out, false,
                 [&](const float* i, const float* m, float* o, cudaStream_t s) {
                     return gdb::geodesic_distance(g, i, m, o, lambda, iterations, pol, s, &st);
                 });
    fill_stats(stats, st);
    return rc;
}

int gd_euclidean_distance(const gd_grid* grid, const float* seed_mask, int iterations,
                          const gd_policy* policy, float* out, int mem, void* stream,
                          gd_stats* stats) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    gdb::Policy pol;
    if (int rc = policy_of(policy, &pol)) return rc;
    if (!seed_mask || !out) return fail(GD_INVALID_ARGUMENT, "null buffer");
    gdb::ScanStats st;
    int rc = run(mem, stream, g.voxels(), nullptr, seed_mask, out, false,
                 [&](const float*, const float* m, float* o, cudaStream_t s) {
                     return gdb::euclidean_distance(g, m, o, iterations, pol, s, &st);
                 });
    fill_stats(stats, st);
    return rc;
}

int gd_signed_geodesic(const gd_grid* grid, const float* image, const float* mask, double lambda,
                       int iterations, const gd_policy* policy, float* out, int mem,
                       void* stream, gd_stats* stats) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    gdb::Policy pol;
    if (int rc = policy_of(policy, &pol)) return rc;
    if (!image || !mask || !out) return fail(GD_INVALID_ARGUMENT, "null buffer");
    gdb::ScanStats st;
    int rc = run(mem, stream, g.voxels(), image, mask, out, false,
                 [&](const float* i, const float* m, float* o, cudaStream_t s) {
                     return gdb::signed_geodesic(g, i, m, o, lambda, iterations, pol, s, &st);
                 });
    fill_stats(stats, st);
    return rc;
}

int gd_geodesic_dilate(const gd_grid* grid, const float* image, const float* mask, double theta,
                       double lambda, double nu, int iterations, const gd_policy* policy,
                       float* out, int mem, void* stream, gd_stats* stats) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    gdb::Policy pol;
    if (int rc = policy_of(policy, &pol)) return rc;
    if (!image || !mask || !out) return fail(GD_INVALID_ARGUMENT, "null buffer");
    gdb::ScanStats st;
    int rc = run(mem, stream, g.voxels(), image, mask, out, false,
                 [&](const float* i, const float* m, float* o, cudaStream_t s) {
                     return gdb::geodesic_dilate(g, i, m, o, lambda, nu, iterations, theta, pol, s,
                                                 &st);
                 });
    fill_stats(stats, st);
    return rc;
}

int gd_geodesic_erode(const gd_grid* grid, const float* image, const float* mask, double theta,
                      double lambda, double nu, int iterations, const gd_policy* policy,
                      float* out, int mem, void* stream, gd_stats* stats) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    gdb::Policy pol;
    if (int rc = policy_of(policy, &pol)) return rc;
    if (!image || !mask || !out) return fail(GD_INVALID_ARGUMENT, "null buffer");
    gdb::ScanStats st;
    const bool sync_stats = mem != GD_MEM_DEVICE || stats != nullptr;
    int rc = run(mem, stream, g.voxels(), image, mask, out, false,
                 [&](const float* i, const float* m, float* o, cudaStream_t s) {
                     return gdb::geodesic_erode(g, i, m, o, lambda, nu, iterations, theta, pol, s,
                                                &st, sync_stats);
                 });
    fill_stats(stats, st);
    return rc;
}

int gd_gsf_ex(const gd_grid* grid, const float* image, const float* soft_mask, double lambda,
              double nu, int iterations, double theta, const gd_policy* policy, float* out,
              int mem, void* stream, gd_stats* stats) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    gdb::Policy pol;
    if (int rc = policy_of(policy, &pol)) return rc;
    if (!image || !soft_mask || !out) return fail(GD_INVALID_ARGUMENT, "null buffer");
    gdb::ScanStats st;
    const bool sync_stats = mem != GD_MEM_DEVICE || stats != nullptr;
    int rc = run(mem, stream, g.voxels(), image, soft_mask, out, false,
                 [&](const float* i, const float* m, float* o, cudaStream_t s) {
                     return gdb::gsf(g, i, m, o, lambda, nu, iterations, theta, s, &st,
                                     sync_stats, pol);
                 });
    fill_stats(stats, st);
    return rc;
}

int gd_gsf_symmetric(const gd_grid* grid, const float* image, const float* soft_mask,
                     double lambda, double nu, int iterations, double theta,
                     const gd_policy* policy, float* out, int mem, void* stream, gd_stats* stats) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    gdb::Policy pol;
    if (int rc = policy_of(policy, &pol)) return rc;
    if (!image || !soft_mask || !out) return fail(GD_INVALID_ARGUMENT, "null buffer");
    gdb::ScanStats st;
    const bool sync_stats = mem != GD_MEM_DEVICE || stats != nullptr;
    int rc = run(mem, stream, g.voxels(), image, soft_mask, out, false,
                 [&](const float* i, const float* m, float* o, cudaStream_t s) {
                     return gdb::gsf_symmetric(g, i, m, o, lambda, nu, iterations, theta, pol, s,
                                               &st, sync_stats);
                 });
    fill_stats(stats, st);
    return rc;
}

int gd_generalized_geodesic(const gd_grid* grid, const float* image, const float* soft_mask,
                            double lambda, double nu, int iterations, float* out, int mem,
                            void* stream, gd_stats* stats) {
    return gd_generalized_geodesic_batched(grid, 1, image, soft_mask, lambda, nu, iterations, out,
                                           mem, stream, stats);
}

int gd_gsf(const gd_grid* grid, const float* image, const float* soft_mask, double lambda,
           double nu, int iterations, double theta, float* out, int mem, void* stream,
           gd_stats* stats) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    if (!image || !soft_mask || !out) return fail(GD_INVALID_ARGUMENT, "null buffer");
    gdb::ScanStats st;
    // complement_empty / rounds need the device's count: a device-memory call
    // synchronises only when the caller asks for stats
    const bool sync_stats = mem != GD_MEM_DEVICE || stats != nullptr;
    int rc = run(mem, stream, g.voxels(), image, soft_mask, out, false,
                 [&](const float* i, const float* m, float* o, cudaStream_t s) {
                     return gdb::gsf(g, i, m, o, lambda, nu, iterations, theta, s, &st,
                                     sync_stats);
                 });
    fill_stats(stats, st);
    return rc;
}

int gd_directional_pass(const gd_grid* grid, const float* image, float* dist, int axis,
                        int orientation, double lambda, int mem, void* stream) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    if (!image || !dist) return fail(GD_INVALID_ARGUMENT, "null buffer");
    return run(mem, stream, g.voxels(), image, nullptr, dist, true,
               [&](const float* i, const float*, float* d, cudaStream_t s) {
                   return gdb::directional_pass(g, 1, i, d, axis, orientation, lambda, s, nullptr);
               });
}

int gd_parallel_scan(const gd_grid* grid, const float* image, float* dist, double lambda,
                     int iterations, int mem, void* stream) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    if (!image || !dist) return fail(GD_INVALID_ARGUMENT, "null buffer");
    return run(mem, stream, g.voxels(), image, nullptr, dist, true,
               [&](const float* i, const float*, float* d, cudaStream_t s) {
                   return gdb::parallel_scan(g, 1, i, d, lambda, iterations, s, nullptr);
               });
}

int gd_scan_to_fixpoint(const gd_grid* grid, const float* image, float* dist, double lambda,
                        int max_rounds, double tol, int mem, void* stream, gd_stats* stats) {
    gdb::GridDesc g;
    if (int rc = grid_of(grid, &g)) return rc;
    if (!image || !dist) return fail(GD_INVALID_ARGUMENT, "null buffer");
    gdb::ScanStats st;
    int rc = run(mem, stream, g.voxels(), image, nullptr, dist, true,
                 [&](const float* i, const float*, float* d, cudaStream_t s) {
                     return gdb::scan_to_fixpoint(g, i, d, lambda, max_rounds, tol, s, &st);
                 });
    fill_stats(stats, st);
    return rc;
}

int gd_synchronize(void* stream) {
    if (int rc = check_device()) return rc;
    cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "stream sync");
    gdb::Status w = gdb::take_deferred();
    return w.ok() ? GD_OK : fail(w);
}

int gd_set_device(int device) {
    if (int rc = check_device()) return rc;
    cudaError_t e = cudaSetDevice(device);
    return e == cudaSuccess ? GD_OK : cuda_fail(e, "cudaSetDevice");
}

int gd_profile_enable(int on) {
    gdb::profile_enable(on != 0);
    return GD_OK;
}

int gd_profile_read(double* ms5, long long* count5, double* bytes5, int reset) {
    gdb::profile_read(ms5, count5, bytes5, reset != 0);
    return GD_OK;
}

int gd_profile_log(int* kinds, float* ms, int max) { return gdb::profile_log(kinds, ms, max); }

static_assert(sizeof(gd_launch_rec) == sizeof(gdb::LaunchRec), "launch record layout");
int gd_debug_launch_log(gd_launch_rec* out, int max, int reset) {
    return gdb::launch_log(reinterpret_cast<gdb::LaunchRec*>(out), out ? max : 0, reset != 0);
}

int gd_fill_splitmix(float* device_out, long long n, unsigned long long seed, void* stream) {
    if (int rc = check_device()) return rc;
    gdb::Status s = gdb::fill_splitmix(device_out, n, seed, static_cast<cudaStream_t>(stream));
    return s.ok() ? GD_OK : fail(s);
}

}  // extern "C"

// Experiment: background HBM copy traffic on `stream` from `ctas` CTAs that each
// request `smem_bytes` of shared memory (placement on SMs the sweep leaves free).
extern "C" int gd_debug_background_copy(const float* src, float* dst, long long n, int ctas,
                                        int smem_bytes, int reps, void* stream) {
    cudaError_t e = gdb::launch_background_copy(src, dst, n, ctas, smem_bytes, reps,
                                                static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? GD_OK : cuda_fail(e, "background copy");
}

// Diagnostics: co-resident CTA capacity of one sweep configuration.
extern "C" int gd_debug_coresident(int R, int nwv, int kind, int f64) {
    return gdb::sweep_max_coresident(R, false, nwv, kind, f64 != 0, 1);
}

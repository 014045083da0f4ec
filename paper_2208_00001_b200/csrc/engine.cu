// Host engine: per-(device, stream) scratch, TMA descriptors, the pass
// scheduler and the transforms.  See engine.cuh.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "aux_kernels.cuh"
#include "engine.cuh"
#include "metric_host.hpp"
#include "rowchain.cuh"
#include "sweep.cuh"

namespace gdb {

namespace {

std::atomic<long long> g_launches{0};
// Blend arithmetic mode; GEODIST_EXACT_BLEND=1 selects the f64 replica at load.
std::atomic<bool> g_exact_blend{std::getenv("GEODIST_EXACT_BLEND") != nullptr &&
                                std::atoi(std::getenv("GEODIST_EXACT_BLEND")) == 1};

// Layout planner on (default) / the fixed plan (C for z and y, T for x):
// GEODIST_LAYOUT_PLAN=0 at load, gd_set_layout_plan at run time.
std::atomic<bool> g_layout_plan{!(std::getenv("GEODIST_LAYOUT_PLAN") &&
                                  std::atoi(std::getenv("GEODIST_LAYOUT_PLAN")) == 0)};

std::mutex g_log_mu;
std::vector<LaunchRec> g_log;
void log_launch(const LaunchRec& r) {
    std::lock_guard<std::mutex> lk(g_log_mu);
    if (g_log.size() < static_cast<size_t>(kLaunchLogMax)) g_log.push_back(r);
}

// Optional per-launch CUDA-event timing, recorded on the launching stream
// (bench.py's roofline numbers).  Off by default.
struct Profiler {
    std::mutex mu;
    bool on = false;
    struct Rec {
        cudaEvent_t a, b;
        int kind;
        double bytes;
    };
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    double ms[kProfKinds] = {};
    std::vector<std::pair<int, float>> log;  // (kind, ms) per launch, in launch order
    long long count[kProfKinds] = {};
    double bytes[kProfKinds] = {};
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};
Profiler g_prof;

// RAII bracket around one launch.
struct ProfScope {
    bool active = false;
    cudaEvent_t a{}, b{};
    int kind;
    double bytes;
    cudaStream_t s;
    ProfScope(int k, double by, cudaStream_t st) : kind(k), bytes(by), s(st) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        if (!g_prof.on) return;
        active = true;
        a = g_prof.get();
        b = g_prof.get();
        cudaEventRecord(a, s);
    }
    ~ProfScope() {
        if (!active) return;
        cudaEventRecord(b, s);
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.pending.push_back({a, b, kind, bytes});
    }
};

Status cuda_status(cudaError_t e, const char* what) {
    return {kCudaError, std::string(what) + ": " + cudaGetErrorString(e)};
}

#define GD_CK(x)                                              \
    do {                                                      \
        cudaError_t e_ = (x);                                 \
        if (e_ != cudaSuccess) return cuda_status(e_, #x);    \
    } while (0)
#define GD_ST(x)                     \
    do {                             \
        Status s_ = (x);             \
        if (!s_.ok()) return s_;     \
    } while (0)

struct Buf {
    void* p = nullptr;
    size_t n = 0;
    Status ensure(size_t bytes) {
        if (bytes <= n) return Status::Ok();
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        GD_CK(cudaMalloc(&p, bytes));
        n = bytes;
        return Status::Ok();
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct StreamCtx {
    Buf halo;
    size_t halo_bytes_zeroed = 0;
    uint32_t tag = 1;  // 0 never matches: freshly zeroed halo words are stale
    Buf dT, iT, dU, iU, padI, padD, tmp, prev, small, trace, ghost;
};

struct DeviceCtx {
    std::mutex mu;
    std::map<cudaStream_t, StreamCtx> streams;
    // Halo watchdog word in mapped pinned host memory: the sweep kernel sets it
    // when a neighbour wait exceeds the spin limit; the host reads it without a
    // stream synchronisation.
    unsigned int* err_h = nullptr;
    unsigned int* err_d = nullptr;
};

DeviceCtx& device_ctx() {
    static DeviceCtx ctx[64];
    int dev = 0;
    cudaGetDevice(&dev);
    return ctx[dev & 63];
}

// Device pointer of this device's watchdog word (allocated on first use; null if
// mapped host memory is unavailable, which only disables the report).
unsigned int* watchdog_word(DeviceCtx& dc) {
    if (!dc.err_d) {
        void* h = nullptr;
        if (cudaHostAlloc(&h, sizeof(unsigned int), cudaHostAllocMapped) == cudaSuccess) {
            *static_cast<volatile unsigned int*>(h) = 0u;
            void* d = nullptr;
            if (cudaHostGetDevicePointer(&d, h, 0) == cudaSuccess) {
                dc.err_h = static_cast<unsigned int*>(h);
                dc.err_d = static_cast<unsigned int*>(d);
            } else {
                cudaFreeHost(h);
            }
        }
        (void)cudaGetLastError();
    }
    return dc.err_d;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

Status make_map(CUtensorMap* m, const float* base, const uint64_t dims[4],
                const uint64_t strides_bytes[3], const uint32_t box[4]) {
    auto fn = encode_fn();
    if (!fn) return {kCudaError, "cuTensorMapEncodeTiled unavailable"};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    cuuint64_t gd[4] = {dims[0], dims[1], dims[2], dims[3]};
    cuuint64_t gs[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
    cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), gd, gs, bx,
                    es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return {kCudaError, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")"};
    return Status::Ok();
}

int round4(int x) { return (x + 3) & ~3; }

// The volumes a scan works on, in up to three storage layouts, each a rotation
// of the canonical one (outer, middle, inner axis; rows of the inner axis
// pitched to a multiple of 4 floats, as TMA strides need 16-byte multiples):
//   C = [b][z][y][x]  (the caller's layout)
//   T = [b][x][z][y]
//   U = [b][y][x][z]
// A pass along an axis runs in any layout where that axis is outer (z-form
// TMA boxes) or middle (y-form); the plane's rows are the other free axis and
// its contiguous columns the inner one.  The planner (scan_work) picks, per
// pass, the layout that minimises sequential plane steps plus the rotations
// between layouts.  Rotating C -> T -> U -> C is one 2D tile transpose per
// outer slice (aux_kernels.cu transpose_kernel, forward; the inverse backward).
enum LayoutId : int { kLC = 0, kLT = 1, kLU = 2 };

struct Geo {
    int ext[3];  // extents (outer, middle, inner)
    int ax[3];   // canonical axis (0 z, 1 y, 2 x) of each
};

Geo layout_geo(int L, const GridDesc& g) {
    if (L == kLC) return {{g.D, g.H, g.W}, {0, 1, 2}};
    if (L == kLT) return {{g.W, g.D, g.H}, {2, 0, 1}};
    return {{g.H, g.W, g.D}, {1, 2, 0}};
}

struct LayoutBuf {
    float* d = nullptr;
    const float* i = nullptr;
    int P = 0;             // row pitch (floats)
    long long vol = 0;     // volume stride (floats)
    bool img_ready = false;
};

struct Work {
    GridDesc g;
    int B = 1;
    const float* img = nullptr;
    float* dist = nullptr;
    int Wp = 0;
    long long zs = 0, vol = 0;
    LayoutBuf lay[3];

    VolView canon() const { return view(kLC); }
    VolView view(int L) const {
        const Geo q = layout_geo(L, g);
        VolView v;
        v.B = B; v.D = q.ext[0]; v.H = q.ext[1]; v.W = q.ext[2];
        const LayoutBuf& b = lay[L];
        v.ys = b.P; v.zs = static_cast<long long>(q.ext[1]) * b.P; v.vol = b.vol;
        return v;
    }
};

int cost_kind(double lambda) {
    // scan_common.hpp:17-21: exact compare
    if (lambda == 0.0) return kSpatial;
    if (lambda == 1.0) return kIntensity;
    return kBlend;
}

// Device-side decision for one transform (the asynchronous path): the gate
// word the transform's kernels test, written by decide_kernel after the fused
// init/check (or the image check) -- no host synchronisation.
struct Gate {
    const int* word = nullptr;  // null: ungated (nothing to decide)
    bool dual = false;          // lambda = 1: launch the f32 and the f64 sweep, each gated
};

int* gate_word(StreamCtx& sc) { return reinterpret_cast<int*>(sc.small.as<char>() + 64); }

// Image-exactness check (lambda = 1 scans that do not start from a soft mask:
// directional_pass, parallel_scan, scan_to_fixpoint) -> gate word.
Status check_inputs(StreamCtx& sc, const Work& w, cudaStream_t s, Gate* gate) {
    GD_ST(sc.small.ensure(256));
    ImageCheck* dev = sc.small.as<ImageCheck>();
    VolView v = w.canon();
    {
        ProfScope ps(kProfOther, 4.0 * w.B * w.g.voxels(), s);
        GD_CK(launch_image_check(v, w.img, nullptr, dev, s));
    }
    GD_CK(launch_decide(dev, true, nullptr, 0u, gate_word(sc), watchdog_word(device_ctx()), s));
    g_launches += 3;
    gate->word = gate_word(sc);
    gate->dual = true;
    return Status::Ok();
}

Buf& layout_dist_buf(StreamCtx& sc, int L) { return L == kLT ? sc.dT : sc.dU; }
Buf& layout_img_buf(StreamCtx& sc, int L) { return L == kLT ? sc.iT : sc.iU; }

// Allocates layout L's distance buffer and, when the kind reads intensities,
// rotates the image into it once per scan (cached in w.lay[L].i).
Status ensure_layout(StreamCtx& sc, Work& w, int L, bool need_img, cudaStream_t s);

// Strip shape of one sweep (rows per strip, co-residency, launch groups).
struct Shape {
    int R = 0;             // rows per strip (0: plane-step fallback)
    int maxc = 0;          // co-resident CTAs of the shape
    long long per_vol = 0; // strips per volume
    bool tb = false;
    int nwv = 0;
    long long groups = 0;  // sequential launch groups for B volumes
    double rel = 1.0;      // per-step cost relative to R = 4
};

// Rows per strip.  Every strip of a volume must be co-resident (the halo chain
// spins); volumes beyond what fits run in sequential launch groups.  Cost =
// groups x relative per-step cost of the strip shape (taller strips do more
// work per step; measured on B200).  A single large volume keeps R = 4 (enough
// rows to cover the halo latency, strips on every SM); batches of small
// volumes take taller strips so fewer groups run.
Shape choose_shape(int nu, int nv, int B, int kind, bool f64) {
    Shape sh;
    sh.nwv = (nv + kWV - 1) / kWV;
    static const bool force_fallback =
        std::getenv("GEODIST_SWEEP_FALLBACK") && std::atoi(std::getenv("GEODIST_SWEEP_FALLBACK")) == 1;
    static const int r_env =
        std::getenv("GEODIST_SWEEP_R") ? std::atoi(std::getenv("GEODIST_SWEEP_R")) : 0;
    static const int rw_env = [] {
        const char* e = std::getenv("GEODIST_SWEEP_RW");
        const int v = e ? std::atoi(e) : -1;
        sweep_set_rows_per_warp(v);
        return v;
    }();
    (void)rw_env;
    // Temporal blocking over plane pairs (halo every two planes): GEODIST_SWEEP_TB=1.
    // Off by default: measured 16.2 vs 13.3 ms per 512^3 transform -- the B step
    // (no halo wait) still costs ~2300 cycles, so the saved wait does not pay for
    // the ghost rows.
    static const bool tb_env =
        std::getenv("GEODIST_SWEEP_TB") && std::atoi(std::getenv("GEODIST_SWEEP_TB")) == 1;
    double best = 0.0;
    for (int cand : {4, 8, 16, 2, 1}) {
        if (sh.nwv > kMaxWarps || force_fallback) break;
        if ((nu == 1) != (cand == 1)) continue;
        if (sweep_warp_rows(cand, sh.nwv, kind, f64) == 0) continue;
        const bool tbc = tb_env && sweep_has_tb(cand, sh.nwv, kind) && nu > cand;
        const int mc = sweep_max_coresident(cand, tbc, sh.nwv, kind, f64);
        const long long pv = (nu + cand - 1) / cand;
        if (mc <= 0 || pv > mc) continue;
        const long long groups = (B + mc / pv - 1) / (mc / pv);
        // measured per-step cost relative to R = 4 (B200, 64 x 256x256x160 batch)
        const double rel = cand <= 4 ? 1.0 : (cand == 8 ? 2.0 : 3.8);
        double cost = static_cast<double>(groups) * rel;
        if (cand == r_env) cost = -1.0;  // tuning override (experiments)
        if (sh.R == 0 || cost < best) {
            sh.R = cand;
            sh.maxc = mc;
            sh.per_vol = pv;
            sh.tb = tbc;
            sh.groups = groups;
            sh.rel = rel;
            best = cost;
        }
    }
    return sh;
}

// Pass geometry of canonical `axis` in layout L (axis outer: z-form, middle: y-form).
struct PassGeo {
    bool ok = false;
    int ns = 0, nu = 0, nv = 0, sweep_dim = 2;
    long long ss = 0, su = 0;
    int u_axis = 0, v_axis = 0;
};

PassGeo pass_geo(const GridDesc& g, int L, int axis, int P) {
    const Geo q = layout_geo(L, g);
    PassGeo pg;
    if (q.ax[0] == axis) {
        pg.ok = true;
        pg.ns = q.ext[0]; pg.nu = q.ext[1]; pg.nv = q.ext[2]; pg.sweep_dim = 2;
        pg.ss = static_cast<long long>(q.ext[1]) * P; pg.su = P;
        pg.u_axis = q.ax[1];
    } else if (q.ax[1] == axis) {
        pg.ok = true;
        pg.ns = q.ext[1]; pg.nu = q.ext[0]; pg.nv = q.ext[2]; pg.sweep_dim = 1;
        pg.ss = P; pg.su = static_cast<long long>(q.ext[1]) * P;
        pg.u_axis = q.ax[0];
    }
    pg.v_axis = q.ax[2];
    return pg;
}

// One launch group of the persistent sweep kernel: `npass` passes along
// canonical `axis` on layout L's buffers.
Status run_sweep(StreamCtx& sc, const Work& w, int L, int axis, int first_orient, int npass,
                 double lambda, bool f64, const int* gate, int gate_want, cudaStream_t s,
                 ScanStats* st) {
    const GridDesc& g = w.g;
    const LayoutBuf& lb = w.lay[L];
    const PassGeo pg = pass_geo(g, L, axis, lb.P);
    if (!pg.ok) return {kCudaError, "internal: pass axis not outer/middle of its layout"};
    const Geo q = layout_geo(L, g);
    const int ns = pg.ns, nu = pg.nu, nv = pg.nv, sweep_dim = pg.sweep_dim;
    const long long ss = pg.ss, su = pg.su, vol = lb.vol;
    const float* ibase = lb.i;
    float* dbase = lb.d;
    uint64_t dims[4], strides[3];
    dims[0] = q.ext[2]; dims[1] = q.ext[1]; dims[2] = q.ext[0];
    strides[0] = lb.P * 4ull;
    strides[1] = static_cast<uint64_t>(q.ext[1]) * lb.P * 4ull;
    strides[2] = vol * 4ull;
    if (ns < 2) return Status::Ok();  // scan_parallel.cpp:308-310
    const int kind = cost_kind(lambda);
    if (kind == kSpatial) ibase = dbase;  // intensities never read; any valid map will do
    static const bool force_fallback =
        std::getenv("GEODIST_SWEEP_FALLBACK") && std::atoi(std::getenv("GEODIST_SWEEP_FALLBACK")) == 1;
    const Shape sh = choose_shape(nu, nv, w.B, kind, f64);
    const int nwv = sh.nwv, R = sh.R, maxc = sh.maxc;
    const long long per_vol = sh.per_vol;
    const bool tb = sh.tb;
    // R == 0: the plane is wider than kMaxWarps * 128 columns or has more row
    // strips than co-resident CTAs -> the plane-step fallback below.
    const int ntu = static_cast<int>(per_vol);
    const int group = R ? static_cast<int>(std::min<long long>(w.B, maxc / per_vol)) : 0;
    // Thread-block clusters for the halo (GEODIST_SWEEP_CLUSTER=<cs>): strips of one
    // cluster exchange rows through DSMEM.  Needs the launch group to tile into
    // co-resident clusters; otherwise every link uses the tagged L2 words.
    // Default (measured on B200): clusters of 4 (else 2) for the intensity kind on
    // wide planes with many strips -- 512^3 lambda=1: 11.8 vs 13.5 ms of sweep, the
    // fewer L2 halo words shortening the remaining L2 links' round trip.  Blend
    // (16-warp shape), small planes and batches measured slower clustered; clusters
    // of 8 / 16 do not tile 128 CTAs co-resident.
    static const int cs_env =
        std::getenv("GEODIST_SWEEP_CLUSTER") ? std::atoi(std::getenv("GEODIST_SWEEP_CLUSTER")) : -1;
    int cs = 1;
    // Spatial (lambda = 0) prefers pairs: 512^3 13.32 (cs 2) / 13.56 (cs 4) / 13.64 ms (L2 only).
    // Blend measured slower clustered in both its shapes (512^3 lambda = 0.5, sweep:
    // two rows per warp 19.4 ms in clusters of 4, 18.4 of 2, 15.2 L2-only; one row
    // per warp 21.3 / 20.6 / 17.7 total; profiles/r02_variants.txt):
    // opt-in only (GEODIST_BLEND_CLUSTER=1).
    static const bool blend_cl = std::getenv("GEODIST_BLEND_CLUSTER") &&
                                 std::atoi(std::getenv("GEODIST_BLEND_CLUSTER")) == 1;
    const bool cs_default =
        (kind == kIntensity || kind == kSpatial || (kind == kBlend && blend_cl)) && nwv >= 4 &&
        ntu >= 64;
    if (R && !tb && ntu > 1 && (cs_env >= 0 || cs_default) && sweep_has_cluster(R, nwv, kind)) {
        const long long ctas = static_cast<long long>(group) * ntu;
        const int first = cs_env >= 0 ? cs_env : (kind == kSpatial ? 2 : 4);
        const int tries[3] = {first, cs_env >= 0 ? 0 : 2, 0};
        for (int cand : tries) {
            if (cand < 2 || cand > 16) continue;
            if (ctas % cand == 0 && sweep_max_coresident(R, false, nwv, kind, f64, cand) >= ctas) {
                cs = cand;
                break;
            }
        }
    }
    const int hrows = tb ? 2 : 1, doff = tb ? 1 : 0, ioff = tb ? 2 : 1;
    const long long strip_words = 2ll * 2 * hrows * nwv * kWV;
    const int J = npass * (ns - 1);

    SweepParams p{};
    p.ss = ss; p.su = su; p.vol_stride = vol;
    p.ns = ns; p.nu = nu; p.nv = nv; p.ntu = ntu; p.nwv = nwv;
    p.tma_sweep_dim = sweep_dim;
    p.first_orient = first_orient;
    p.npass = npass;
    p.fence_turn = npass == 2 ? 1 : 0;
    p.cs = cs;
    p.lambda = lambda;
    p.lambda_f = static_cast<float>(lambda);
    p.sqrt_lambda_f = static_cast<float>(std::sqrt(lambda));
    p.gate = gate;
    p.gate_mask = kGateMaskBad | kGateF64 | kGateSkip;
    p.gate_want = gate_want;
    for (int du = -1; du <= 1; ++du)
        for (int dv = -1; dv <= 1; ++dv) {
            int d[3];
            d[axis] = -first_orient;
            d[pg.u_axis] = du;
            d[pg.v_axis] = dv;
            const double rho = offset_rho(d[0], d[1], d[2], g.sz, g.sy, g.sx);
            const int k = (du + 1) * 3 + (dv + 1);
            p.rho[k] = rho;
            p.c0[k] = blend_c0(lambda, rho);
            p.c0_f[k] = static_cast<float>(p.c0[k]);
            p.c0l_f[k] = lambda > 0.0 ? static_cast<float>(p.c0[k] / lambda) : 0.0f;
        }

    // Single-row planes (2D images): the row-chain kernel, one CTA per image
    // (GEODIST_ROWCHAIN=0 selects the strip kernel's R = 1 shape instead).
    static const bool rowchain_env =
        !(std::getenv("GEODIST_ROWCHAIN") && std::atoi(std::getenv("GEODIST_ROWCHAIN")) == 0);
    if (nu == 1 && nv <= kRowChainMaxWidth && rowchain_env && !force_fallback) {
        p.ntu = 1;
        p.image = ibase;
        for (int b0 = 0; b0 < w.B; b0 += 65535) {
            p.nvol = std::min(65535, w.B - b0);
            p.dist = dbase + b0 * vol;
            p.image = ibase + b0 * vol;
            const double bytes = static_cast<double>(p.nvol) * g.voxels() * npass *
                                 (kind == kSpatial ? 8.0 : 12.0);
            ProfScope ps(gate_want == kGateF64 ? kProfSweepTwin : kProfSweep, bytes, s);
            GD_CK(launch_row_chain(kind, f64, p, s));
            log_launch({axis, npass, kind, f64 ? 1 : 0, 1, 0, 0, 0, 1, 1, p.nvol, p.nvol, 0, L});
            g_launches += 1;
            if (st) st->kernel_launches += 1;
        }
        return Status::Ok();
    }

    if (R == 0) {
        // One launch per plane step (plane_step_kernel), every volume at once.
        const int n1 = ns - 1;
        auto plane = [&](int j) {
            if (j <= n1) return first_orient > 0 ? j : n1 - j;
            const int k = j - n1;
            return first_orient > 0 ? n1 - k : k;
        };
        for (int b0 = 0; b0 < w.B; b0 += 65535) {
            p.nvol = std::min(65535, w.B - b0);
            p.dist = dbase + b0 * vol;
            p.image = ibase + b0 * vol;
            const double bytes = static_cast<double>(p.nvol) * g.voxels() * npass *
                                 (kind == kSpatial ? 8.0 : 12.0);
            ProfScope ps(gate_want == kGateF64 ? kProfSweepTwin : kProfSweep, bytes, s);
            for (int j = 1; j <= J; ++j) GD_CK(launch_plane_step(kind, f64, p, plane(j), plane(j - 1), s));
            log_launch({axis, npass, kind, f64 ? 1 : 0, 2, 0, 0, 0, 1, 0, p.nvol, 0, 0, L});
            g_launches += J;
            if (st) st->kernel_launches += J;
        }
        return Status::Ok();
    }

    uint32_t box_d[4], box_i[4];
    const uint32_t drows = R + 2 * doff, irows = R + 2 * ioff;
    if (sweep_dim == 2) {
        box_d[0] = kWV; box_d[1] = drows; box_d[2] = 1; box_d[3] = 1;
        box_i[0] = kIW; box_i[1] = irows; box_i[2] = 1; box_i[3] = 1;
    } else {
        box_d[0] = kWV; box_d[1] = 1; box_d[2] = drows; box_d[3] = 1;
        box_i[0] = kIW; box_i[1] = 1; box_i[2] = irows; box_i[3] = 1;
    }

    for (int b0 = 0; b0 < w.B; b0 += group) {
        const int nvol = std::min(group, w.B - b0);
        dims[3] = static_cast<uint64_t>(nvol);
        CUtensorMap tm_d, tm_i;
        GD_ST(make_map(&tm_d, dbase + b0 * vol, dims, strides, box_d));
        GD_ST(make_map(&tm_i, ibase + b0 * vol, dims, strides, box_i));
        const size_t words = static_cast<size_t>(nvol) * per_vol * strip_words;
        GD_ST(sc.halo.ensure(words * 8));
        if (sc.halo_bytes_zeroed < sc.halo.n) {
            GD_CK(cudaMemsetAsync(sc.halo.p, 0, sc.halo.n, s));
            sc.halo_bytes_zeroed = sc.halo.n;
            sc.tag = 1;
        }
        if (static_cast<uint64_t>(sc.tag) + J + 2 >= 0xffffffffull) {
            GD_CK(cudaMemsetAsync(sc.halo.p, 0, sc.halo.n, s));
            sc.tag = 1;
        }
        p.dist = dbase + b0 * vol;
        p.nvol = nvol;
        p.cs = (static_cast<long long>(nvol) * ntu) % cs == 0 ? cs : 1;  // last group may be short
        p.halo = sc.halo.as<unsigned long long>();
        p.ghost = nullptr;
        if (tb && npass == 2) {
            const size_t gfloats = static_cast<size_t>(nvol) * per_vol * 2 *
                                   static_cast<size_t>((ns - 1) / 2 + 1) * nwv * kWV;
            GD_ST(sc.ghost.ensure(gfloats * 4));
            p.ghost = sc.ghost.as<float>();
        }
        p.tag_base = sc.tag;
        p.err = watchdog_word(device_ctx());
        sc.tag += static_cast<uint32_t>(J + 1);
        // Diagnostic cycle counters: only a -DGD_SWEEP_TRACE build writes them.
        static const bool trace_on = std::getenv("GEODIST_SWEEP_TRACE") != nullptr;
        const size_t trace_n = static_cast<size_t>(nvol) * per_vol * 64 * 12;
        if (trace_on) {
            GD_ST(sc.trace.ensure(trace_n * sizeof(long long)));
            GD_CK(cudaMemsetAsync(sc.trace.p, 0, trace_n * sizeof(long long), s));
            p.trace = sc.trace.as<long long>();
            static const int dbg = std::getenv("GEODIST_SWEEP_DEBUG") ? std::atoi(std::getenv("GEODIST_SWEEP_DEBUG")) : 0;
            p.debug_flags = dbg;
        }
        {
            const double bytes = static_cast<double>(nvol) * g.voxels() * npass *
                                 (kind == kSpatial ? 8.0 : 12.0);
            ProfScope ps(gate_want == kGateF64 ? kProfSweepTwin : kProfSweep, bytes, s);
            GD_CK(launch_sweep(kind, f64, R, tb, tm_d, tm_i, p, s));
        }
        log_launch({axis, npass, kind, f64 ? 1 : 0, 0, R, nwv, sweep_warp_rows(R, nwv, kind, f64), p.cs,
                    ntu, nvol, nvol * ntu, tb ? 1 : 0, L});
        if (trace_on) {
            std::vector<long long> h(trace_n);
            GD_CK(cudaMemcpyAsync(h.data(), sc.trace.p, trace_n * sizeof(long long),
                                  cudaMemcpyDeviceToHost, s));
            GD_CK(cudaStreamSynchronize(s));
            const int nw = nwv * sweep_warp_rows(R, nwv, kind, f64);
            for (int w = 0; w < nw; ++w) {
                double acc[12] = {};
                long long n = 0;
                for (long long cta = 0; cta < nvol * per_vol; ++cta) {
                    const long long* o = &h[(cta * 64 + w) * 12];
                    if (o[5] == 0) continue;
                    for (int k = 0; k < 12; ++k) acc[k] += o[k];
                    ++n;
                }
                if (!n) continue;
                const double steps = acc[5] / n;
                auto a = [&](int k) { return acc[k] / n / steps; };
                std::fprintf(stderr,
                             "trace axis=%d R=%d maxc=%d warp=%d: cycles/step total %.0f pre %.0f tma %.0f "
                             "phaseA %.0f spin %.0f crit %.0f tail %.0f barrier %.0f post %.0f "
                             "reloads/step %.2f (ctas %lld)\n",
                             axis, R, maxc, w, a(4), a(8), a(0), a(6), a(1), a(9), a(7), a(2), a(10),
                             a(3), n);
            }
        }
        ++g_launches;
        if (st) ++st->kernel_launches;
    }
    return Status::Ok();
}

// One launch group per pair, or -- lambda = 1 under a device-side gate -- the
// f32 and the f64 instance back to back, each leaving at once unless the gate
// selects it (a skipped launch costs a few microseconds; no host sync).
Status sweep_gated(StreamCtx& sc, const Work& w, int L, int axis, int first_orient, int npass,
                   double lambda, bool f64, const Gate& gate, cudaStream_t s, ScanStats* st) {
    if (!gate.word)
        return run_sweep(sc, w, L, axis, first_orient, npass, lambda, f64, nullptr, 0, s, st);
    if (!gate.dual)
        return run_sweep(sc, w, L, axis, first_orient, npass, lambda, f64, gate.word, 0, s, st);
    GD_ST(run_sweep(sc, w, L, axis, first_orient, npass, lambda, false, gate.word, 0, s, st));
    return run_sweep(sc, w, L, axis, first_orient, npass, lambda, true, gate.word, kGateF64, s,
                     st);
}

Status ensure_layout(StreamCtx& sc, Work& w, int L, bool need_img, cudaStream_t s) {
    if (L == kLC) return Status::Ok();
    const Geo q = layout_geo(L, w.g);
    LayoutBuf& lb = w.lay[L];
    lb.P = round4(q.ext[2]);
    lb.vol = static_cast<long long>(q.ext[0]) * q.ext[1] * lb.P;
    const size_t bytes = static_cast<size_t>(w.B) * lb.vol * sizeof(float);
    Buf& db = layout_dist_buf(sc, L);
    GD_ST(db.ensure(bytes));
    lb.d = db.as<float>();
    if (need_img && !lb.img_ready) {
        Buf& ib = layout_img_buf(sc, L);
        GD_ST(ib.ensure(bytes));
        // C -> T is one forward rotation, C -> U one inverse rotation
        ProfScope ps(kProfTranspose, 8.0 * w.B * w.g.voxels(), s);
        if (L == kLT) GD_CK(launch_transpose(w.view(kLC), w.view(kLT), w.img, ib.as<float>(), true, s));
        else GD_CK(launch_transpose(w.view(kLC), w.view(kLU), w.img, ib.as<float>(), false, s));
        ++g_launches;
        lb.i = ib.as<float>();
        lb.img_ready = true;
    }
    return Status::Ok();
}

// Moves the working distance from layout `from` to `to` (one rotation: forward
// C->T->U->C or its inverse).
Status move_dist(StreamCtx& sc, Work& w, int from, int to, bool need_img, cudaStream_t s) {
    if (from == to) return Status::Ok();
    GD_ST(ensure_layout(sc, w, to, need_img, s));
    ProfScope ps(kProfTranspose, 8.0 * w.B * w.g.voxels(), s);
    // launch_transpose(src view, dst view, src, dst, forward): forward takes
    // [a][b][c] to [c][a][b]; backward is its inverse (src the rotated side)
    GD_CK(launch_transpose(w.view(from), w.view(to), w.lay[from].d, w.lay[to].d,
                           to == (from + 1) % 3, s));
    ++g_launches;
    return Status::Ok();
}

// f64 arithmetic for blend (exact mode); lambda = 1 decides on the device.
// The f32 blend form sqrt(lambda) * sqrt(di^2 + c0 / lambda) needs c0 / lambda
// to stay far from f32 overflow: lambda below 1e-20 takes the f64 replica.
bool blend_f64(int kind, double lambda) {
    return kind == kBlend && (g_exact_blend.load() || lambda < 1e-20);
}

// --- layout planner ------------------------------------------------------------
// Estimated device time (us) of one pass group on layout L: sequential plane
// steps (launch groups x relative step cost x steps) at ~1.1 us per step for
// the persistent kernel, ~0.3 us per row-chain step, one launch per step for
// the plane-step fallback; a rotation moves 8 B per voxel at ~5.5 TB/s.
constexpr double kStepUs = 1.1, kRowChainStepUs = 0.3, kRotateGBs = 5500.0;

double pass_cost_us(const Work& w, int L, int axis, int npass, int kind, bool f64) {
    const PassGeo pg = pass_geo(w.g, L, axis, round4(layout_geo(L, w.g).ext[2]));
    if (!pg.ok) return -1.0;
    if (pg.ns < 2) return 0.0;
    const double steps = static_cast<double>(npass) * (pg.ns - 1);
    if (pg.nu == 1) return steps * kRowChainStepUs;
    const Shape sh = choose_shape(pg.nu, pg.nv, w.B, kind, f64);
    if (sh.R == 0) return steps * (4.0 + 12.0 * w.B * pg.nu * pg.nv / (kRotateGBs * 1e3) * 1e0);
    return static_cast<double>(sh.groups) * sh.rel * steps * kStepUs;
}

double rotate_cost_us(const Work& w) { return 8.0 * w.B * w.g.voxels() / (kRotateGBs * 1e3); }

struct PassSpec {
    int axis, orient, npass;
};

// Cheapest layout per pass (dynamic program over (layout, image copies made)):
// the distance starts and ends in C; entering a layout costs a rotation of the
// distance, and the first use of T / U also a rotation of the image (when the
// kind reads intensities).  2D grids keep C for y and T for x (their U rows are
// a single column).  Ties keep the earlier (lower-numbered) layout.
std::vector<int> plan_layouts(const Work& w, const std::vector<PassSpec>& passes, int kind,
                              bool f64) {
    const int n = static_cast<int>(passes.size());
    std::vector<int> plan(n, kLC);
    if (w.g.ndim == 2 || !g_layout_plan.load()) {  // the fixed plan: C for z / y, T for x
        for (int i = 0; i < n; ++i) plan[i] = passes[i].axis == 2 ? kLT : kLC;
        return plan;
    }
    const bool img = kind != kSpatial;
    const double rot = rotate_cost_us(w);
    constexpr double kInf = 1e300;
    // state: layout L (3) x image-copies mask (bit 0: T, bit 1: U)
    std::vector<double> cost(12, kInf), next(12);
    std::vector<std::vector<int>> from(n, std::vector<int>(12, -1));
    cost[kLC * 4 + 0] = 0.0;
    for (int i = 0; i < n; ++i) {
        std::fill(next.begin(), next.end(), kInf);
        for (int st = 0; st < 12; ++st) {
            if (cost[st] >= kInf) continue;
            const int L0 = st / 4, m0 = st % 4;
            for (int L = 0; L < 3; ++L) {
                const double pc = pass_cost_us(w, L, passes[i].axis, passes[i].npass, kind, f64);
                if (pc < 0.0) continue;
                int m = m0;
                double c = cost[st] + pc + (L != L0 ? rot : 0.0);
                if (img && L != kLC && !(m & (1 << (L - 1)))) {
                    m |= 1 << (L - 1);
                    c += rot;
                }
                const int ns = L * 4 + m;
                if (c < next[ns] - 1e-9) {
                    next[ns] = c;
                    from[i][ns] = st;
                }
            }
        }
        cost.swap(next);
    }
    int best = -1;
    double bc = kInf;
    for (int st = 0; st < 12; ++st) {
        const double c = cost[st] + (st / 4 != kLC ? rot : 0.0);
        if (c < bc - 1e-9) {
            bc = c;
            best = st;
        }
    }
    for (int i = n - 1; i >= 0; --i) {
        plan[i] = best / 4;
        best = from[i][best];
    }
    static const bool dbg = std::getenv("GEODIST_LAYOUT_DEBUG") != nullptr;
    if (dbg) {
        std::fprintf(stderr, "layout plan B=%d D=%d H=%d W=%d kind=%d rot=%.1fus total=%.1fus:", w.B,
                     w.g.D, w.g.H, w.g.W, kind, rot, bc);
        for (int i = 0; i < n; ++i) {
            std::fprintf(stderr, " [axis %d -> L%d (", passes[i].axis, plan[i]);
            for (int L = 0; L < 3; ++L)
                std::fprintf(stderr, "%s%.0f", L ? "/" : "",
                             pass_cost_us(w, L, passes[i].axis, passes[i].npass, kind, f64));
            std::fprintf(stderr, ")]");
        }
        std::fprintf(stderr, "\n");
    }
    return plan;
}

// Runs `passes` on the working distance (bound in C) with the planned layouts,
// rotating between them, and leaves the result in C.
Status run_passes(StreamCtx& sc, Work& w, const std::vector<PassSpec>& passes, double lambda,
                  const Gate& gate, cudaStream_t s, ScanStats* st) {
    const int kind = cost_kind(lambda);
    const bool f64 = blend_f64(kind, lambda);
    const bool img = kind != kSpatial;
    const std::vector<int> plan = plan_layouts(w, passes, kind, f64);
    int cur = kLC;
    for (size_t i = 0; i < passes.size(); ++i) {
        const int L = plan[i];
        if (L != cur) {
            GD_ST(move_dist(sc, w, cur, L, img, s));
            cur = L;
        }
        GD_ST(sweep_gated(sc, w, L, passes[i].axis, passes[i].orient, passes[i].npass, lambda,
                          f64, gate, s, st));
    }
    return move_dist(sc, w, cur, kLC, img, s);
}

// parallel_scan_inplace: for it: FB BF (3D) TB BT LR RL  (metric.cpp:35-44);
// each forward / backward pair of one axis is one persistent launch.
Status scan_work(StreamCtx& sc, Work& w, double lambda, int iterations, const Gate& gate,
                 cudaStream_t s, ScanStats* st) {
    std::vector<PassSpec> passes;
    for (int it = 0; it < iterations; ++it) {
        if (w.g.ndim == 3) passes.push_back({0, +1, 2});
        passes.push_back({1, +1, 2});
        if (w.g.W >= 2) passes.push_back({2, +1, 2});
    }
    GD_ST(run_passes(sc, w, passes, lambda, gate, s, st));
    if (st) st->rounds += iterations;
    return Status::Ok();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Sets up w.img / w.dist: the caller's buffers when the layout is TMA-legal
// (W % 4 == 0, 16-byte aligned), else padded copies (copy_in: dist content).
Status bind(StreamCtx& sc, Work& w, const GridDesc& g, int B, const float* img, float* dist,
            bool copy_dist_in, cudaStream_t s, bool* padded) {
    w.g = g;
    w.B = B;
    const bool direct = (g.W % 4 == 0) && aligned16(img) && aligned16(dist);
    w.Wp = direct ? g.W : round4(g.W);
    w.zs = static_cast<long long>(g.H) * w.Wp;
    w.vol = static_cast<long long>(g.D) * w.zs;
    *padded = !direct;
    if (direct) {
        w.img = img;
        w.dist = dist;
        w.lay[kLC] = {dist, img, w.Wp, w.vol, true};
        return Status::Ok();
    }
    const size_t bytes = static_cast<size_t>(B) * w.vol * sizeof(float);
    GD_ST(sc.padI.ensure(bytes));
    GD_ST(sc.padD.ensure(bytes));
    const size_t rows = static_cast<size_t>(B) * g.D * g.H;
    if (img) {
        GD_CK(cudaMemcpy2DAsync(sc.padI.p, w.Wp * 4, img, g.W * 4, g.W * 4, rows,
                                cudaMemcpyDeviceToDevice, s));
    }
    if (copy_dist_in) {
        GD_CK(cudaMemcpy2DAsync(sc.padD.p, w.Wp * 4, dist, g.W * 4, g.W * 4, rows,
                                cudaMemcpyDeviceToDevice, s));
    }
    w.img = img ? sc.padI.as<float>() : nullptr;
    w.dist = sc.padD.as<float>();
    w.lay[kLC] = {w.dist, w.img, w.Wp, w.vol, true};
    return Status::Ok();
}

Status unbind(const Work& w, float* dist, cudaStream_t s) {
    const size_t rows = static_cast<size_t>(w.B) * w.g.D * w.g.H;
    GD_CK(cudaMemcpy2DAsync(dist, w.g.W * 4, w.dist, w.Wp * 4, w.g.W * 4, rows,
                            cudaMemcpyDeviceToDevice, s));
    return Status::Ok();
}

Status validate_params(double lambda, double nu, int iterations) {
    // TransformParams::validate (grid.cpp:67-78)
    if (!(lambda >= 0.0 && lambda <= 1.0))
        return Status::Invalid("lambda must lie in [0, 1], got " + std::to_string(lambda));
    if (!(nu >= 0.0)) return Status::Invalid("nu must be >= 0, got " + std::to_string(nu));
    if (iterations < 1)
        return Status::Invalid("iterations must be >= 1, got " + std::to_string(iterations));
    return Status::Ok();
}

// scan_to_fixpoint's round loop (scan_parallel.cpp:357-397) on bound work:
// one iteration of the pass sequence per round, then the device max-change
// reduction; the convergence test is a host decision, one sync per round.
Status fixpoint_work(StreamCtx& sc, Work& w, double lambda, const Policy& pol, const Gate& gate,
                     cudaStream_t s, ScanStats* st) {
    const size_t bytes = static_cast<size_t>(w.B) * w.vol * sizeof(float);
    GD_ST(sc.prev.ensure(bytes));
    GD_ST(sc.small.ensure(256));
    unsigned long long* chg = reinterpret_cast<unsigned long long*>(sc.small.as<char>() + 192);
    int rounds = 0;
    double last = 0.0;
    bool converged = false;
    while (rounds < pol.max_rounds) {
        GD_CK(cudaMemcpyAsync(sc.prev.p, w.dist, bytes, cudaMemcpyDeviceToDevice, s));
        GD_ST(scan_work(sc, w, lambda, 1, gate, s, nullptr));
        ++rounds;
        GD_CK(cudaMemsetAsync(chg, 0, sizeof(unsigned long long), s));
        GD_CK(launch_max_change(w.canon(), sc.prev.as<float>(), w.dist, chg, s));
        ++g_launches;
        unsigned long long bits = 0;
        GD_CK(cudaMemcpyAsync(&bits, chg, sizeof(bits), cudaMemcpyDeviceToHost, s));
        GD_CK(cudaStreamSynchronize(s));
        std::memcpy(&last, &bits, sizeof(last));
        if (last <= pol.tol) {
            converged = true;
            break;
        }
    }
    if (st) {
        st->rounds += rounds;
        st->converged = st->converged && converged;
        st->last_change = last;
    }
    return Status::Ok();
}

// run_scan (transforms.cpp:91-125) for the parallel engine on bound work.
Status run_scan_w(StreamCtx& sc, Work& w, double lambda, int iterations, const Policy& pol,
                  const Gate& gate, cudaStream_t s, ScanStats* st) {
    if (pol.fixpoint) return fixpoint_work(sc, w, lambda, pol, gate, s, st);
    return scan_work(sc, w, lambda, iterations, gate, s, st);
}

// A gate closed for the whole transform (kGateSkip, e.g. the GSF erode with an
// empty complement) is also a host fact in fixpoint mode, which synchronises
// anyway: read it so a skipped transform adds no rounds (transforms.cpp:213-219).
bool skipped_on_host(StreamCtx& sc, cudaStream_t s) {
    int g = 0;
    if (cudaMemcpyAsync(&g, gate_word(sc), sizeof(g), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return false;
    return (g & (kGateSkip | kGateMaskBad)) != 0;
}

// generalized_geodesic on bound device buffers, asynchronous in iterations
// mode: the fused init/check kernel and decide_kernel set the gate word; a bad
// mask closes it (nothing runs; the error is reported through the device's
// status word).  skip_if_zero (GSF / geodesic_erode): the whole transform is
// gated off when *skip_if_zero == 0.
Status generalized_locked(StreamCtx& sc, const GridDesc& g, int B, const float* img,
                          const float* mask, float* out, double lambda, double nu, int iterations,
                          const Policy& pol, cudaStream_t s, ScanStats* st,
                          const unsigned long long* skip_if_zero = nullptr) {
    GD_ST(validate_params(lambda, nu, iterations));
    if (pol.fixpoint && B != 1) return Status::Invalid("fixpoint mode takes one grid at a time");
    Work w;
    bool padded = false;
    GD_ST(bind(sc, w, g, B, img, out, false, s, &padded));
    const int kind = cost_kind(lambda);
    // One pass over the caller's (dense) image + mask: soft-mask init into the
    // working distance, mask-range check, image-exactness statistics.
    VolView mv;
    mv.B = B; mv.D = g.D; mv.H = g.H; mv.W = g.W;
    mv.zs = static_cast<long long>(g.H) * g.W; mv.ys = g.W; mv.vol = g.D * mv.zs;
    GD_ST(sc.small.ensure(256));
    ImageCheck* chk = sc.small.as<ImageCheck>();
    const bool want_img = kind == kIntensity;
    {
        ProfScope ps(kProfInit, (want_img ? 12.0 : 8.0) * B * g.voxels(), s);
        GD_CK(launch_init_generalized(mv, w.canon(), mask, w.dist, nu, chk,
                                      want_img ? img : nullptr, s));
    }
    GD_CK(launch_decide(chk, want_img, skip_if_zero, 0u, gate_word(sc), watchdog_word(device_ctx()),
                        s));
    g_launches += 3;
    Gate gate;
    gate.word = gate_word(sc);
    gate.dual = want_img;
    if (!(pol.fixpoint && skipped_on_host(sc, s)))
        GD_ST(run_scan_w(sc, w, lambda, iterations, pol, gate, s, st));
    if (padded) GD_ST(unbind(w, out, s));
    return Status::Ok();
}

// init_hard_seeds + run_scan on the device (geodesic_distance,
// euclidean_distance and signed_geodesic's two halves, transforms.cpp:74-89,
// 127-141, 160-183).  Seeds where M >= 0.5 (invert: where not); no seed ->
// every kernel of the transform is gated off and EmptySeedsError is deferred.
// img may be null for lambda = 0 (never read).
Status hard_seeds_locked(StreamCtx& sc, const GridDesc& g, const float* img, const float* seeds,
                         bool invert, float* out, double lambda, int iterations,
                         const Policy& pol, cudaStream_t s, ScanStats* st) {
    GD_ST(validate_params(lambda, 0.0, iterations));
    Work w;
    bool padded = false;
    GD_ST(bind(sc, w, g, 1, img, out, false, s, &padded));
    GD_ST(sc.small.ensure(256));
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(sc.small.as<char>() + 136);
    VolView mv;
    mv.D = g.D; mv.H = g.H; mv.W = g.W;
    mv.zs = static_cast<long long>(g.H) * g.W; mv.ys = g.W; mv.vol = g.D * mv.zs;
    GD_CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
    {
        ProfScope ps(kProfInit, 8.0 * g.voxels(), s);
        GD_CK(launch_hard_seeds(mv, seeds, w.canon(), w.dist, invert, cnt, s));
    }
    const bool want_img = cost_kind(lambda) == kIntensity;
    ImageCheck* chk = nullptr;
    if (want_img) {
        chk = sc.small.as<ImageCheck>();
        GD_CK(launch_image_check(w.canon(), w.img, nullptr, chk, s));
        g_launches += 2;
    }
    GD_CK(launch_decide(chk, want_img, cnt, kStatusEmptySeeds, gate_word(sc),
                        watchdog_word(device_ctx()), s));
    g_launches += 2;
    Gate gate;
    gate.word = gate_word(sc);
    gate.dual = want_img;
    if (!(pol.fixpoint && skipped_on_host(sc, s)))
        GD_ST(run_scan_w(sc, w, lambda, iterations, pol, gate, s, st));
    if (padded) GD_ST(unbind(w, out, s));
    return Status::Ok();
}

VolView dense_view(const GridDesc& g) {
    VolView v;
    v.D = g.D; v.H = g.H; v.W = g.W; v.ys = g.W; v.zs = static_cast<long long>(g.H) * g.W;
    v.vol = g.D * v.zs;
    return v;
}

// geodesic_dilate (transforms.cpp:185-202): out = [GG(I, complement([M >= 0.5])) <= theta],
// fused with the erode prologue: *n_complement = |{out == 0}|.
Status dilate_locked(StreamCtx& sc, const GridDesc& g, const float* img, const float* mask,
                     float* out, double lambda, double nu, int iterations, double theta,
                     const Policy& pol, cudaStream_t s, ScanStats* st,
                     unsigned long long* n_complement) {
    const VolView v = dense_view(g);
    GD_ST(sc.tmp.ensure(static_cast<size_t>(g.voxels()) * sizeof(float)));
    float* tmp = sc.tmp.as<float>();
    GD_CK(launch_gsf_sources(v, mask, v, tmp, s));
    ++g_launches;
    GD_ST(generalized_locked(sc, g, 1, img, tmp, out, lambda, nu, iterations, pol, s, st));
    GD_CK(cudaMemsetAsync(n_complement, 0, sizeof(unsigned long long), s));
    GD_CK(launch_gsf_dilate(v, out, out, theta, n_complement, s));
    ++g_launches;
    return Status::Ok();
}

// geodesic_erode (transforms.cpp:204-229) with `out` already holding
// kept = [M >= 0.5] and *n_complement its complement count: out = [GG(I, kept) > theta],
// or kept unchanged when the complement is empty (device-side gate).
Status erode_from_kept(StreamCtx& sc, const GridDesc& g, const float* img, float* out,
                       double lambda, double nu, int iterations, double theta, const Policy& pol,
                       cudaStream_t s, ScanStats* st, const unsigned long long* n_complement) {
    const VolView v = dense_view(g);
    GD_ST(sc.tmp.ensure(static_cast<size_t>(g.voxels()) * sizeof(float)));
    float* tmp = sc.tmp.as<float>();
    GD_ST(generalized_locked(sc, g, 1, img, out, tmp, lambda, nu, iterations, pol, s, st,
                             n_complement));
    GD_CK(launch_gsf_erode(v, tmp, v, out, theta, gate_word(sc), s));
    ++g_launches;
    return Status::Ok();
}

// complement_empty / rounds of a possibly skipped erode need the device count.
Status erode_stats(StreamCtx& sc, const unsigned long long* cnt, int iterations,
                   const Policy& pol, cudaStream_t s, ScanStats* st) {
    (void)sc;
    unsigned long long n_src = 0;
    GD_CK(cudaMemcpyAsync(&n_src, cnt, sizeof(n_src), cudaMemcpyDeviceToHost, s));
    GD_CK(cudaStreamSynchronize(s));
    if (n_src == 0) {
        st->complement_empty = true;
        if (!pol.fixpoint) st->rounds -= iterations;  // the gated transform added them
    }
    return Status::Ok();
}

}  // namespace

Status make_grid_desc(int ndim, const int* dims, const double* spacing, GridDesc* out) {
    if (ndim != 2 && ndim != 3)
        return Status::Invalid("grid rank must be 2 or 3, got " + std::to_string(ndim));
    GridDesc g;
    g.ndim = ndim;
    int cd[3] = {1, 1, 1};
    double cs[3] = {1.0, 1.0, 1.0};
    for (int a = 0; a < ndim; ++a) {
        if (dims[a] < 1)
            return Status::Invalid("grid extent must be >= 1, got " + std::to_string(dims[a]));
        if (!(spacing[a] > 0.0) || !std::isfinite(spacing[a]))
            return Status::Invalid("grid spacing must be finite and > 0, got " +
                                   std::to_string(spacing[a]));
        cd[a + 3 - ndim] = dims[a];
        cs[a + 3 - ndim] = spacing[a];
    }
    g.D = cd[0]; g.H = cd[1]; g.W = cd[2];
    g.sz = cs[0]; g.sy = cs[1]; g.sx = cs[2];
    *out = g;
    return Status::Ok();
}

void set_exact_blend(bool on) { g_exact_blend.store(on); }
void set_layout_plan(bool on) { g_layout_plan.store(on); }
bool exact_blend() { return g_exact_blend.load(); }
long long kernel_launch_count() { return g_launches.load(); }

void profile_enable(bool on) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = on;
}

void profile_read(double* ms, long long* count, double* bytes, bool reset) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (auto& r : g_prof.pending) {
        cudaEventSynchronize(r.b);
        float t = 0.0f;
        cudaEventElapsedTime(&t, r.a, r.b);
        g_prof.ms[r.kind] += t;
        g_prof.log.emplace_back(r.kind, t);
        g_prof.count[r.kind] += 1;
        g_prof.bytes[r.kind] += r.bytes;
        g_prof.pool.push_back(r.a);
        g_prof.pool.push_back(r.b);
    }
    g_prof.pending.clear();
    for (int k = 0; k < kProfKinds; ++k) {
        if (ms) ms[k] = g_prof.ms[k];
        if (count) count[k] = g_prof.count[k];
        if (bytes) bytes[k] = g_prof.bytes[k];
        if (reset) {
            if (k == 0) g_prof.log.clear();
            g_prof.ms[k] = 0.0;
            g_prof.count[k] = 0;
            g_prof.bytes[k] = 0.0;
        }
    }
}

Status directional_pass(const GridDesc& g, int B, const float* img, float* dist, int axis,
                        int orientation, double lambda, cudaStream_t s, ScanStats* st) {
    GD_ST(validate_params(lambda, 0.0, 1));
    const bool dir_ok = (orientation == 1 || orientation == -1) &&
                        (g.ndim == 2 ? (axis == 1 || axis == 2) : (axis >= 0 && axis <= 2));
    if (!dir_ok) return Status::Invalid("invalid pass direction for rank " + std::to_string(g.ndim));
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    Work w;
    bool padded = false;
    GD_ST(bind(sc, w, g, B, img, dist, true, s, &padded));
    const int kind = cost_kind(lambda);
    Gate gate;
    if (kind == kIntensity) GD_ST(check_inputs(sc, w, s, &gate));
    // scan_parallel.cpp:308-311: a single-plane sweep axis is a no-op (and a 3D
    // x pass with W < 2 never leaves the caller's layout)
    const int ext[3] = {g.D, g.H, g.W};
    if (ext[axis] >= 2) GD_ST(run_passes(sc, w, {{axis, orientation, 1}}, lambda, gate, s, st));
    if (padded) GD_ST(unbind(w, dist, s));
    return Status::Ok();
}

Status parallel_scan(const GridDesc& g, int B, const float* img, float* dist, double lambda,
                     int iterations, cudaStream_t s, ScanStats* st) {
    GD_ST(validate_params(lambda, 0.0, iterations));
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    Work w;
    bool padded = false;
    GD_ST(bind(sc, w, g, B, img, dist, true, s, &padded));
    Gate gate;
    if (cost_kind(lambda) == kIntensity) GD_ST(check_inputs(sc, w, s, &gate));
    GD_ST(scan_work(sc, w, lambda, iterations, gate, s, st));
    if (padded) GD_ST(unbind(w, dist, s));
    return Status::Ok();
}

Status generalized_geodesic(const GridDesc& g, int B, const float* img, const float* mask,
                            float* out, double lambda, double nu, int iterations, cudaStream_t s,
                            ScanStats* st, const Policy& pol) {
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    return generalized_locked(sc, g, B, img, mask, out, lambda, nu, iterations, pol, s, st);
}

Status geodesic_distance(const GridDesc& g, const float* img, const float* seeds, float* out,
                         double lambda, int iterations, const Policy& pol, cudaStream_t s,
                         ScanStats* st) {
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    return hard_seeds_locked(sc, g, img, seeds, false, out, lambda, iterations, pol, s, st);
}

Status euclidean_distance(const GridDesc& g, const float* seeds, float* out, int iterations,
                          const Policy& pol, cudaStream_t s, ScanStats* st) {
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    // lambda = 0 over a uniform image (transforms.cpp:134-141): the spatial
    // kind never reads intensities, so no image is needed
    return hard_seeds_locked(sc, g, nullptr, seeds, false, out, 0.0, iterations, pol, s, st);
}

Status signed_geodesic(const GridDesc& g, const float* img, const float* mask, float* out,
                       double lambda, int iterations, const Policy& pol, cudaStream_t s,
                       ScanStats* st) {
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    const long long n = g.voxels();
    GD_ST(sc.tmp.ensure(static_cast<size_t>(n) * sizeof(float)));
    float* d_out = sc.tmp.as<float>();
    // d_in from the inside seeds [M >= 0.5], d_out from the outside ones
    GD_ST(hard_seeds_locked(sc, g, img, mask, false, out, lambda, iterations, pol, s, st));
    GD_ST(hard_seeds_locked(sc, g, img, mask, true, d_out, lambda, iterations, pol, s, st));
    GD_CK(launch_subtract(out, d_out, out, n, s));
    ++g_launches;
    return Status::Ok();
}

Status geodesic_dilate(const GridDesc& g, const float* img, const float* mask, float* out,
                       double lambda, double nu, int iterations, double theta, const Policy& pol,
                       cudaStream_t s, ScanStats* st) {
    if (!(theta >= 0.0)) return Status::Invalid("theta must be >= 0");
    GD_ST(validate_params(lambda, nu, iterations));
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    GD_ST(sc.small.ensure(256));
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(sc.small.as<char>() + 128);
    return dilate_locked(sc, g, img, mask, out, lambda, nu, iterations, theta, pol, s, st, cnt);
}

Status geodesic_erode(const GridDesc& g, const float* img, const float* mask, float* out,
                      double lambda, double nu, int iterations, double theta, const Policy& pol,
                      cudaStream_t s, ScanStats* st, bool sync_stats) {
    if (!(theta >= 0.0)) return Status::Invalid("theta must be >= 0");
    GD_ST(validate_params(lambda, nu, iterations));
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    GD_ST(sc.small.ensure(256));
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(sc.small.as<char>() + 128);
    const VolView v = dense_view(g);
    GD_CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
    GD_CK(launch_threshold_count(v, mask, out, cnt, s));
    ++g_launches;
    GD_ST(erode_from_kept(sc, g, img, out, lambda, nu, iterations, theta, pol, s, st, cnt));
    if ((sync_stats || pol.fixpoint) && st) GD_ST(erode_stats(sc, cnt, iterations, pol, s, st));
    return Status::Ok();
}

Status gsf(const GridDesc& g, const float* img, const float* mask, float* out, double lambda,
           double nu, int iterations, double theta, cudaStream_t s, ScanStats* st,
           bool sync_stats, const Policy& pol) {
    GD_ST(validate_params(lambda, nu, iterations));
    if (!(theta >= 0.0)) return Status::Invalid("theta must be >= 0, got " + std::to_string(theta));
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    GD_ST(sc.small.ensure(256));
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(sc.small.as<char>() + 128);
    // gsf = geodesic_erode(geodesic_dilate(M, theta), theta) (transforms.cpp:231-238):
    // the dilate epilogue writes K = [dilated >= 0.5] = dilated and counts its
    // complement; the erode is gated on the device by that count -- when it is 0
    // every erode kernel leaves at once and out keeps K, as the reference
    // returns `kept`.
    GD_ST(dilate_locked(sc, g, img, mask, out, lambda, nu, iterations, theta, pol, s, st, cnt));
    GD_ST(erode_from_kept(sc, g, img, out, lambda, nu, iterations, theta, pol, s, st, cnt));
    if ((sync_stats || pol.fixpoint) && st) GD_ST(erode_stats(sc, cnt, iterations, pol, s, st));
    return Status::Ok();
}

// Upstream-FastGeodis-style symmetric filter in four chained transforms
// (BASELINE.json config 4; PAPER.md:143-153 names GSF without a formula): the
// reference's closing gsf = erode(dilate(M)) (transforms.cpp:231-238)
// followed by the opening dilate(erode(.)), each step the reference's
// geodesic_dilate / geodesic_erode semantics (transforms.cpp:185-229) with the
// erode's empty-complement skip gated on the device.
Status gsf_symmetric(const GridDesc& g, const float* img, const float* mask, float* out,
                     double lambda, double nu, int iterations, double theta, const Policy& pol,
                     cudaStream_t s, ScanStats* st, bool sync_stats) {
    GD_ST(validate_params(lambda, nu, iterations));
    if (!(theta >= 0.0)) return Status::Invalid("theta must be >= 0, got " + std::to_string(theta));
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    GD_ST(sc.small.ensure(256));
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(sc.small.as<char>() + 128);
    unsigned long long* cnt2 = reinterpret_cast<unsigned long long*>(sc.small.as<char>() + 144);
    const VolView v = dense_view(g);
    ScanStats s1, s2;
    // closing: erode(dilate(M))
    GD_ST(dilate_locked(sc, g, img, mask, out, lambda, nu, iterations, theta, pol, s, &s1, cnt));
    GD_ST(erode_from_kept(sc, g, img, out, lambda, nu, iterations, theta, pol, s, &s1, cnt));
    // opening: dilate(erode(closed))
    GD_CK(cudaMemsetAsync(cnt2, 0, sizeof(unsigned long long), s));
    GD_CK(launch_threshold_count(v, out, out, cnt2, s));
    ++g_launches;
    GD_ST(erode_from_kept(sc, g, img, out, lambda, nu, iterations, theta, pol, s, &s2, cnt2));
    GD_ST(dilate_locked(sc, g, img, out, out, lambda, nu, iterations, theta, pol, s, &s2, cnt2));
    if ((sync_stats || pol.fixpoint) && st) {
        GD_ST(erode_stats(sc, cnt, iterations, pol, s, &s1));
        GD_ST(erode_stats(sc, cnt2, iterations, pol, s, &s2));
    }
    if (st) {
        st->rounds += s1.rounds + s2.rounds;
        st->converged = st->converged && s1.converged && s2.converged;
        st->complement_empty = s1.complement_empty || s2.complement_empty;
    }
    return Status::Ok();
}

Status scan_to_fixpoint(const GridDesc& g, const float* img, float* dist, double lambda,
                        int max_rounds, double tol, cudaStream_t s, ScanStats* st) {
    GD_ST(validate_params(lambda, 0.0, 1));
    if (max_rounds < 1)
        return Status::Invalid("max_rounds must be >= 1, got " + std::to_string(max_rounds));
    if (!(tol >= 0.0)) return Status::Invalid("tol must be >= 0");
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    StreamCtx& sc = dc.streams[s];
    Work w;
    bool padded = false;
    GD_ST(bind(sc, w, g, 1, img, dist, true, s, &padded));
    Gate gate;
    if (cost_kind(lambda) == kIntensity) GD_ST(check_inputs(sc, w, s, &gate));
    ScanStats local;
    ScanStats* stp = st ? st : &local;
    stp->converged = true;
    Policy pol;
    pol.fixpoint = true;
    pol.max_rounds = max_rounds;
    pol.tol = tol;
    GD_ST(fixpoint_work(sc, w, lambda, pol, gate, s, stp));
    if (padded) GD_ST(unbind(w, dist, s));
    return Status::Ok();
}

Status fill_splitmix(float* out, long long n, unsigned long long seed, cudaStream_t s) {
    GD_CK(launch_splitmix(out, n, seed, s));
    ++g_launches;
    return Status::Ok();
}

Status take_deferred() {
    DeviceCtx& dc = device_ctx();
    std::lock_guard<std::mutex> lk(dc.mu);
    if (!dc.err_h) return Status::Ok();
    volatile unsigned int* w = dc.err_h;
    const unsigned int v = *w;
    if (v == 0u) return Status::Ok();
    *w = 0u;
    if (v & kStatusWatchdog)
        return {kCudaError,
                "halo watchdog: a strip of the directional-pass kernel waited past the spin "
                "limit for its neighbour; the results of the work enqueued since the last check "
                "are invalid"};
    if (v & kStatusMaskBad)
        return Status::Invalid("generalized_geodesic: mask values must lie in [0, 1]");
    return {kEmptySeeds, "no seed cell at or above the 0.5 mask threshold (or, for "
                         "signed_geodesic, the mask or its complement is empty)"};
}

int launch_log(LaunchRec* out, int max, bool reset) {
    std::lock_guard<std::mutex> lk(g_log_mu);
    const int n = static_cast<int>(g_log.size());
    for (int i = 0; i < n && i < max; ++i) out[i] = g_log[i];
    if (reset) g_log.clear();
    return n;
}

int profile_log(int* kinds, float* ms, int max) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    const int n = static_cast<int>(std::min<size_t>(g_prof.log.size(), static_cast<size_t>(max)));
    for (int i = 0; i < n; ++i) {
        kinds[i] = g_prof.log[i].first;
        ms[i] = g_prof.log[i].second;
    }
    return static_cast<int>(g_prof.log.size());
}

}  // namespace gdb

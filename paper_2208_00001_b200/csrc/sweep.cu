// Sweep dispatch: strip-shape selection helpers, the plane-step fallback and
// the switch over the per-(kind, f64) instantiation units.
#include "sweep_impl.cuh"

namespace gdb {

// Instantiation units (sweep_k*.cu): the persistent kernel for one (kind, f64).
#define GD_SWEEP_INST_DECL(sfx)                                                              \
    cudaError_t sweep_launch_##sfx(int R, bool tb, const CUtensorMap& tm_d,                  \
                                   const CUtensorMap& tm_i, const SweepParams& p,            \
                                   cudaStream_t stream);                                     \
    int sweep_cores_##sfx(int R, bool tb, int nwv, int cs);
GD_SWEEP_INST_DECL(k0)
GD_SWEEP_INST_DECL(k1)
GD_SWEEP_INST_DECL(k1d)
GD_SWEEP_INST_DECL(k2)
GD_SWEEP_INST_DECL(k2d)
#undef GD_SWEEP_INST_DECL

int g_sweep_rw = -1;

cudaError_t launch_sweep(int kind, bool f64, int R, bool tb, const CUtensorMap& tm_d,
                         const CUtensorMap& tm_i, const SweepParams& p, cudaStream_t stream) {
    switch (kind) {
        case kSpatial: return sweep_launch_k0(R, tb, tm_d, tm_i, p, stream);
        case kIntensity:
            return f64 ? sweep_launch_k1d(R, tb, tm_d, tm_i, p, stream)
                       : sweep_launch_k1(R, tb, tm_d, tm_i, p, stream);
        default:
            return f64 ? sweep_launch_k2d(R, tb, tm_d, tm_i, p, stream)
                       : sweep_launch_k2(R, tb, tm_d, tm_i, p, stream);
    }
}

cudaError_t launch_plane_step(int kind, bool f64, const SweepParams& p, int s, int sp,
                              cudaStream_t stream) {
    switch (kind) {
        case kSpatial: return plane_step_one<kSpatial, false>(p, s, sp, stream);
        case kIntensity:
            return f64 ? plane_step_one<kIntensity, true>(p, s, sp, stream)
                       : plane_step_one<kIntensity, false>(p, s, sp, stream);
        default:
            return f64 ? plane_step_one<kBlend, true>(p, s, sp, stream)
                       : plane_step_one<kBlend, false>(p, s, sp, stream);
    }
}

void sweep_set_rows_per_warp(int rw) { g_sweep_rw = rw; }

int sweep_warp_rows(int R, int nwv, int kind, bool f64) {
    const int mw = width_class(nwv);
    RwSel sel(R, mw, false, preferred_rw(kind, f64));
#define GD_CASE(RWW, NW, MM, NS, T, C) \
    if (R == RWW * NW && mw == MM && !T && !C && sel.ok(RWW)) return NW;
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
    return 0;
}

bool sweep_has_tb(int R, int nwv, int kind) {
    const int mw = width_class(nwv);
    RwSel sel(R, mw, true, preferred_rw(kind));
#define GD_CASE(RWW, NW, MM, NS, T, C) \
    if (R == RWW * NW && mw == MM && T && !C && sel.ok(RWW)) return true;
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
    return false;
}

bool sweep_has_cluster(int R, int nwv, int kind) {
    const int mw = width_class(nwv);
    RwSel sel(R, mw, false, preferred_rw(kind));
#define GD_CASE(RWW, NW, MM, NS, T, C) \
    if (R == RWW * NW && mw == MM && !T && C && sel.ok(RWW)) return true;
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
    return false;
}

int sweep_max_coresident(int R, bool tb, int nwv, int kind, bool f64, int cs) {
    switch (kind) {
        case kSpatial: return sweep_cores_k0(R, tb, nwv, cs);
        case kIntensity:
            return f64 ? sweep_cores_k1d(R, tb, nwv, cs) : sweep_cores_k1(R, tb, nwv, cs);
        default:
            return f64 ? sweep_cores_k2d(R, tb, nwv, cs) : sweep_cores_k2(R, tb, nwv, cs);
    }
}

}  // namespace gdb

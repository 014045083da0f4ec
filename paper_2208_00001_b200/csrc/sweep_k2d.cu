// Instantiation unit: the persistent sweep kernel for cost kind kBlend, f64 = true
// (sweep_impl.cuh).  One unit per (kind, f64) so the instances compile in parallel.
#include "sweep_impl.cuh"

namespace gdb {

cudaError_t sweep_launch_k2d(int R, bool tb, const CUtensorMap& tm_d, const CUtensorMap& tm_i,
                              const SweepParams& p, cudaStream_t stream) {
    return dispatch_r<kBlend, true>(R, tb, tm_d, tm_i, p, stream);
}

int sweep_cores_k2d(int R, bool tb, int nwv, int cs) { return dispatch_cores<kBlend, true>(R, tb, nwv, cs); }

}  // namespace gdb

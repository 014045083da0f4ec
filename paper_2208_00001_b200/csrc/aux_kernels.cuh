#pragma once

#include <cuda_runtime.h>

namespace gdb {

// A batch of B volumes of logical extent (D, H, W) in a pitched layout:
// element (b, a0, a1, a2) lives at b*vol + a0*zs + a1*ys + a2, where
// (a0, a1, a2) = (z, y, x) for the canonical layout and (x, z, y) for the
// x-sweep layout.  Element kernels always enumerate canonical (z, y, x).
struct VolView {
    int B = 1, D = 1, H = 1, W = 1;
    long long vol = 0, zs = 0, ys = 0;
    __host__ __device__ long long count() const {
        return static_cast<long long>(B) * D * H * W;
    }
};

struct ImageCheck {
    int emax, tmin, pos, neg, bad_mask, nonfinite;
};

// Soft-mask init (transforms.cpp:150-156) fused with the mask-range and
// image-exactness reduction into `check` (reset here); `img`/`check` may be null.
cudaError_t launch_init_generalized(const VolView& m, const VolView& d, const float* mask,
                                    float* dist, double nu, ImageCheck* check, const float* img,
                                    cudaStream_t s);
cudaError_t launch_transpose(const VolView& src_v, const VolView& dst_v, const float* src,
                             float* dst, bool forward, cudaStream_t s);
cudaError_t launch_image_check(const VolView& v, const float* img, const float* mask,
                               ImageCheck* out, cudaStream_t s);
cudaError_t launch_gsf_sources(const VolView& v, const float* mask, const VolView& o, float* out,
                               cudaStream_t s);
cudaError_t launch_gsf_dilate(const VolView& v, const float* dist, float* out, double theta,
                              unsigned long long* n_complement, cudaStream_t s);
cudaError_t launch_gsf_erode(const VolView& v, const float* dist, const VolView& o, float* out,
                             double theta, const int* gate, cudaStream_t s);
// Deferred-error bits of the per-device status word (mapped host memory).
constexpr unsigned int kStatusWatchdog = 1u;  // a halo wait hit the spin limit
constexpr unsigned int kStatusMaskBad = 2u;   // a soft mask outside [0, 1]
constexpr unsigned int kStatusEmptySeeds = 4u;  // a hard-seed transform without seeds
// One thread: ImageCheck (nullable) + optional count -> gate word (sweep.cuh
// GateBits); a zero count closes the gate (kGateSkip) and raises status_if_skip.
cudaError_t launch_decide(const ImageCheck* chk, bool check_exact,
                          const unsigned long long* skip_if_zero, unsigned int status_if_skip,
                          int* gate, unsigned int* status, cudaStream_t s);
// init_hard_seeds on the device (transforms.cpp:74-89), counting the seeds.
cudaError_t launch_hard_seeds(const VolView& mv, const float* mask, const VolView& dv, float* dist,
                              bool invert, unsigned long long* n_seeds, cudaStream_t s);
// out = [M >= 0.5] and the count of its complement (geodesic_erode prologue).
cudaError_t launch_threshold_count(const VolView& v, const float* mask, float* out,
                                   unsigned long long* n_complement, cudaStream_t s);
cudaError_t launch_background_copy(const float* src, float* dst, long long n, int ctas,
                                   int smem_bytes, int reps, cudaStream_t s);
cudaError_t launch_subtract(const float* a, const float* b, float* out, long long n,
                            cudaStream_t s);
cudaError_t launch_max_change(const VolView& v, const float* before, const float* after,
                              unsigned long long* out, cudaStream_t s);
cudaError_t launch_splitmix(float* out, long long n, unsigned long long seed, cudaStream_t s);

}  // namespace gdb

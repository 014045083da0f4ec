// Element-wise and layout kernels around the sweep: soft-mask init (fused with
// the mask-range / image-exactness check), the x-axis layout transposes, GSF
// thresholds, fixpoint change reduction, and the SplitMix64 synthetic-input
// generator.  All are HBM-bound streams: 16-byte accesses wherever the layout
// allows, grid-stride loops, grids sized as a multiple of the SM count.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "aux_kernels.cuh"
#include "sweep.cuh"

namespace gdb {

namespace {

__device__ __forceinline__ bool dense(const VolView& v) {
    return v.ys == v.W && v.zs == static_cast<long long>(v.H) * v.W &&
           v.vol == static_cast<long long>(v.D) * v.zs;
}

// i enumerates logical voxels (b, z, y, x) densely.
__device__ __forceinline__ long long vox_offset(const VolView& v, long long i) {
    if (dense(v)) return i;
    const long long x = i % v.W;
    long long t = i / v.W;
    const long long y = t % v.H;
    t /= v.H;
    const long long z = t % v.D;
    const long long b = t / v.D;
    return b * v.vol + z * v.zs + y * v.ys + x;
}

// Exponent statistics for the exactness test (see ImageCheck).
struct ExpStats {
    int emax = -1000, tmin = 1000, pos = 0, neg = 0, nonfinite = 0;
    __device__ __forceinline__ void add(float x) {
        const uint32_t u = __float_as_uint(x);
        const int ebits = (u >> 23) & 0xff;
        const uint32_t man = u & 0x7fffffu;
        if (ebits == 0xff) {
            nonfinite = 1;
        } else if (ebits != 0 || man != 0) {
            int e, t;
            if (ebits == 0) {  // subnormal: value = man * 2^-149
                e = -149 + (31 - __clz(man));
                t = -149 + (__ffs(man) - 1);
            } else {
                e = ebits - 127;
                t = ebits - 150 + (__ffs(man | 0x800000u) - 1);
            }
            emax = max(emax, e);
            tmin = min(tmin, t);
            if (u >> 31) neg = 1; else pos = 1;
        }
    }
};

__device__ __forceinline__ void flush_check(const ExpStats& s, int bad_mask, ImageCheck* out) {
    int emax = s.emax, tmin = s.tmin, pos = s.pos, neg = s.neg, nf = s.nonfinite, bm = bad_mask;
    for (int o = 16; o > 0; o >>= 1) {
        emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
        tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
        pos |= __shfl_xor_sync(0xffffffffu, pos, o);
        neg |= __shfl_xor_sync(0xffffffffu, neg, o);
        nf |= __shfl_xor_sync(0xffffffffu, nf, o);
        bm |= __shfl_xor_sync(0xffffffffu, bm, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out->emax, emax);
        atomicMin(&out->tmin, tmin);
        if (pos) atomicOr(&out->pos, 1);
        if (neg) atomicOr(&out->neg, 1);
        if (bm) atomicOr(&out->bad_mask, 1);
        if (nf) atomicOr(&out->nonfinite, 1);
    }
}

__device__ __forceinline__ float init_value(float m, double nu) {
    // transforms.cpp:150-156: f32(min(nu * f64(M), f64(1e10)))
    const double v = nu * static_cast<double>(m);
    return static_cast<float>(v < 1.0e10 ? v : 1.0e10);
}

// Soft-mask init fused with the input checks: one pass over image + mask.
// `img` may be null (no exactness check wanted).  `m` and `d` views may differ
// (the distance may live in a padded working layout).
// `vec`: the host found every pointer 16-byte aligned (float4 path allowed).
__global__ void init_check_kernel(VolView mv, VolView dv, const float* img, const float* mask,
                                  float* dist, double nu, ImageCheck* out, long long n, bool vec) {
    ExpStats st;
    int bad = 0;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    const long long t0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (vec && dense(mv) && dense(dv) && (n & 3) == 0) {
        const long long n4 = n >> 2;
        // Two float4 per stream in flight per thread (all loads issued first):
        // 0.37 ms at 512^3 with one, a 3-stream read/read/write copy.
        auto one = [&](const float4 m, const float4 a, long long i) {
            bad |= !(m.x >= 0.0f && m.x <= 1.0f) | !(m.y >= 0.0f && m.y <= 1.0f) |
                   !(m.z >= 0.0f && m.z <= 1.0f) | !(m.w >= 0.0f && m.w <= 1.0f);
            reinterpret_cast<float4*>(dist)[i] = make_float4(
                init_value(m.x, nu), init_value(m.y, nu), init_value(m.z, nu), init_value(m.w, nu));
            if (img) {
                st.add(a.x); st.add(a.y); st.add(a.z); st.add(a.w);
            }
        };
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        long long i = t0;
        for (; i + stride < n4; i += 2 * stride) {
            const float4 m0 = __ldcs(reinterpret_cast<const float4*>(mask) + i);
            const float4 m1 = __ldcs(reinterpret_cast<const float4*>(mask) + i + stride);
            const float4 a0 = img ? reinterpret_cast<const float4*>(img)[i] : z4;
            const float4 a1 = img ? reinterpret_cast<const float4*>(img)[i + stride] : z4;
            one(m0, a0, i);
            one(m1, a1, i + stride);
        }
        if (i < n4)
            one(__ldcs(reinterpret_cast<const float4*>(mask) + i),
                img ? reinterpret_cast<const float4*>(img)[i] : z4, i);
    } else {
        for (long long i = t0; i < n; i += stride) {
            const long long om = vox_offset(mv, i);
            const float m = mask[om];
            bad |= !(m >= 0.0f && m <= 1.0f);
            dist[vox_offset(dv, i)] = init_value(m, nu);
            if (img) st.add(img[om]);
        }
    }
    flush_check(st, bad, out);
}

// Exactness / mask-range check alone (scans that are not generalized_geodesic).
__global__ void image_check_kernel(VolView v, const float* img, const float* mask,
                                   ImageCheck* out, long long n, bool vec) {
    ExpStats st;
    int bad = 0;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    const long long t0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (vec && dense(v) && (n & 3) == 0) {
        const long long n4 = n >> 2;
        for (long long i = t0; i < n4; i += stride) {
            if (img) {
                const float4 a = reinterpret_cast<const float4*>(img)[i];
                st.add(a.x); st.add(a.y); st.add(a.z); st.add(a.w);
            }
            if (mask) {
                const float4 m = reinterpret_cast<const float4*>(mask)[i];
                bad |= !(m.x >= 0.0f && m.x <= 1.0f) | !(m.y >= 0.0f && m.y <= 1.0f) |
                       !(m.z >= 0.0f && m.z <= 1.0f) | !(m.w >= 0.0f && m.w <= 1.0f);
            }
        }
    } else {
        for (long long i = t0; i < n; i += stride) {
            const long long o = vox_offset(v, i);
            if (img) st.add(img[o]);
            if (mask) {
                const float m = mask[o];
                bad |= !(m >= 0.0f && m <= 1.0f);
            }
        }
    }
    flush_check(st, bad, out);
}

// 64x64-tile transpose of every (b, z) slice between the canonical layout
// [b][z][y][x] (row pitch c.ys, slice pitch c.zs) and the x-sweep layout
// [b][x][z][y] (x pitch t.zs, z pitch t.ys).  FWD: canonical -> x-layout.
// Loads and stores are float4 along the contiguous axis of each side; the
// 64x65 shared tile keeps the column reads to 2-way bank conflicts.
template <bool FWD>
__global__ void __launch_bounds__(256) transpose_kernel(VolView cv, VolView tv, const float* src,
                                                        float* dst, int tiles_a, int tiles_b,
                                                        long long ntiles) {
    __shared__ float tile[64][65];
    const int D = cv.D, H = cv.H, W = cv.W;
    // FWD: tile rows = y (input rows), cols = x.  BWD: tile rows = x, cols = y.
    const int RA = FWD ? H : W;   // extent of the input row axis
    const int CA = FWD ? W : H;   // extent of the input contiguous axis
    const int tid = threadIdx.x;
    const int lr = tid >> 4;          // 0..15
    const int lc = (tid & 15) * 4;    // 0..60
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int ta = static_cast<int>(t % tiles_a);
        const long long rest = t / tiles_a;
        const int tb = static_cast<int>(rest % tiles_b);
        const long long bz = rest / tiles_b;
        const int z = static_cast<int>(bz % D);
        const long long b = bz / D;
        const int r0 = tb * 64, c0 = ta * 64;
        const float* sbase;
        long long s_row;
        if (FWD) {
            sbase = src + b * cv.vol + z * cv.zs;
            s_row = cv.ys;
        } else {
            sbase = src + b * tv.vol + z * tv.ys;
            s_row = tv.zs;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = r0 + i * 16 + lr, cc = c0 + lc;
            float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
            if (r < RA) {
                const float* q = sbase + r * s_row + cc;
                if (cc + 3 < CA) {
                    const float4 a = *reinterpret_cast<const float4*>(q);
                    v0 = a.x; v1 = a.y; v2 = a.z; v3 = a.w;
                } else {
                    if (cc < CA) v0 = q[0];
                    if (cc + 1 < CA) v1 = q[1];
                    if (cc + 2 < CA) v2 = q[2];
                }
            }
            float* trow = tile[i * 16 + lr];
            trow[lc] = v0; trow[lc + 1] = v1; trow[lc + 2] = v2; trow[lc + 3] = v3;
        }
        __syncthreads();
        float* dbase;
        long long d_row;
        if (FWD) {
            dbase = dst + b * tv.vol + z * tv.ys;
            d_row = tv.zs;
        } else {
            dbase = dst + b * cv.vol + z * cv.zs;
            d_row = cv.ys;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int oc = i * 16 + lr;     // output row = input column
            const int orow = c0 + oc;
            const int ocol = r0 + lc;       // output contiguous = input row axis
            if (orow < CA) {
                const float v0 = tile[lc][oc], v1 = tile[lc + 1][oc], v2 = tile[lc + 2][oc],
                            v3 = tile[lc + 3][oc];
                float* q = dbase + orow * d_row + ocol;
                if (ocol + 3 < RA) {
                    *reinterpret_cast<float4*>(q) = make_float4(v0, v1, v2, v3);
                } else {
                    if (ocol < RA) q[0] = v0;
                    if (ocol + 1 < RA) q[1] = v1;
                    if (ocol + 2 < RA) q[2] = v2;
                }
            }
        }
        __syncthreads();
    }
}

// out = [M >= 0.5] ? 0 : 1   (complement_mask(threshold_mask(M)), transforms.cpp:30-48)
__global__ void gsf_sources_kernel(VolView v, const float* mask, VolView o, float* out,
                                   long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float m = mask[vox_offset(v, i)];
        out[vox_offset(o, i)] = m >= 0.5f ? 0.0f : 1.0f;
    }
}

// dilate epilogue fused with the erode prologue (transforms.cpp:195-201, 211-219):
//   dil = [f64(D) <= theta];  K = threshold(dil) = dil;  count(complement(K)).
__global__ void gsf_dilate_kernel(VolView v, const float* dist, float* out, double theta,
                                  unsigned long long* n_complement, long long n) {
    unsigned long long cnt = 0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long o = vox_offset(v, i);
        const float dil = static_cast<double>(dist[o]) <= theta ? 1.0f : 0.0f;
        out[o] = dil;
        cnt += dil >= 0.5f ? 0 : 1;
    }
    for (int s = 16; s > 0; s >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_complement, cnt);
}

// erode epilogue: out = [f64(D) > theta]
__global__ void gsf_erode_kernel(VolView v, const float* dist, VolView o, float* out, double theta,
                                 long long n, const int* gate) {
    if (gate && (*gate & kGateSkip)) return;  // empty complement: out keeps K
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float d = dist[vox_offset(v, i)];
        out[vox_offset(o, i)] = static_cast<double>(d) > theta ? 1.0f : 0.0f;
    }
}

// Hard seeds (init_hard_seeds, transforms.cpp:74-89): dist = 0 where the seed
// test holds, kInfSentinel elsewhere; counts the seeds.  invert: seeds where
// NOT (m >= 0.5) -- the complement mask's seeds (signed_geodesic's outside).
__global__ void hard_seed_kernel(VolView mv, const float* mask, VolView dv, float* dist, int invert,
                                 unsigned long long* n_seeds, long long n) {
    unsigned long long cnt = 0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const bool seed = (mask[vox_offset(mv, i)] >= 0.5f) != (invert != 0);
        dist[vox_offset(dv, i)] = seed ? 0.0f : 1.0e10f;
        cnt += seed ? 1 : 0;
    }
    for (int s = 16; s > 0; s >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_seeds, cnt);
}

// kept = threshold_mask(M) = [M >= 0.5]; counts its complement
// (geodesic_erode's prologue, transforms.cpp:211-219).
__global__ void threshold_count_kernel(VolView v, const float* mask, float* out,
                                       unsigned long long* n_complement, long long n) {
    unsigned long long cnt = 0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long o = vox_offset(v, i);
        const bool k = mask[o] >= 0.5f;
        out[o] = k ? 1.0f : 0.0f;
        cnt += k ? 0 : 1;
    }
    for (int s = 16; s > 0; s >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_complement, cnt);
}

// signed_geodesic epilogue (transforms.cpp:176-182): out = d_in - d_out in f32.
__global__ void subtract_kernel(const float* a, const float* b, float* out, long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = a[i] - b[i];
}

// Experiment only (gd_debug_background_copy): a float4 copy loop run on a few
// CTAs with a large dynamic shared-memory request, so they can only occupy SMs
// the persistent sweep leaves free -- background HBM traffic to measure how
// much the sweep's halo latency suffers from it.
__global__ void background_copy_kernel(const float4* src, float4* dst, long long n4, int reps) {
    extern __shared__ float4 pad[];
    if (threadIdx.x == 0 && n4 < 0) pad[0] = src[0];  // keep the allocation
    for (int r = 0; r < reps; ++r)
        for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
             i += static_cast<long long>(gridDim.x) * blockDim.x)
            dst[i] = __ldcs(src + i);
}

__global__ void reset_check_kernel(ImageCheck* c) {
    *c = ImageCheck{-1000, 1000, 0, 0, 0, 0};
}

// Turns the fused init/check statistics into the gate word the transform's
// kernels test (sweep.cuh GateBits): mask range, the f32/f64 choice for
// lambda = 1 (every I_p - I_q exact in f32 when all values are multiples of
// 2^tmin below 2^(emax+1) with emax - tmin <= 23, 22 with mixed signs), GSF's
// empty-complement skip.  A bad mask also raises the deferred-error bit of the
// device's status word (mapped host memory).
__global__ void decide_kernel(const ImageCheck* chk, int check_exact,
                              const unsigned long long* skip_if_zero, unsigned int status_if_skip,
                              int* gate, unsigned int* status) {
    const ImageCheck h = chk ? *chk : ImageCheck{-1000, 1000, 0, 0, 0, 0};
    int g = 0;
    if (h.bad_mask) g |= kGateMaskBad;
    if (check_exact) {
        bool exact;
        if (h.nonfinite) exact = false;
        else if (h.emax < -999) exact = true;  // all zeros
        else exact = (h.emax - h.tmin) <= ((h.pos && h.neg) ? 22 : 23);
        if (!exact) g |= kGateF64;
    }
    if (skip_if_zero && *skip_if_zero == 0ull) g |= kGateSkip;
    *gate = g;
    if ((g & kGateMaskBad) && status) atomicOr_system(status, kStatusMaskBad);
    if ((g & kGateSkip) && status && status_if_skip) atomicOr_system(status, status_if_skip);
}

// Fixpoint change: max over voxels of f64(before) - f64(after) (scan_parallel.cpp:386-392).
// Only non-negative values matter (change starts at 0), so the f64 bit pattern
// orders like an unsigned integer.
__global__ void max_change_kernel(VolView v, const float* before, const float* after,
                                  unsigned long long* out, long long n) {
    double m = 0.0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long o = vox_offset(v, i);
        const double c = static_cast<double>(before[o]) - static_cast<double>(after[o]);
        m = c > m ? c : m;
    }
    for (int s = 16; s > 0; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
    if ((threadIdx.x & 31) == 0 && m > 0.0)
        atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// SplitMix64 benchmark image (tools/main.cpp:67-81): value i (0-based) is
// f32((mix(seed + (i+1)*gamma) >> 40) * 2^-24), written densely.
__global__ void splitmix_kernel(float* out, long long n, unsigned long long seed) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        unsigned long long z = seed + static_cast<unsigned long long>(i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z = z ^ (z >> 31);
        out[i] = static_cast<float>(static_cast<double>(z >> 40) * 0x1.0p-24);
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

int grid_for(long long n, int threads) {
    const long long need = (n + threads - 1) / threads;
    const long long cap = static_cast<long long>(sm_count()) * 8;
    return static_cast<int>(need < cap ? (need > 0 ? need : 1) : cap);
}

}  // namespace

cudaError_t launch_init_generalized(const VolView& m, const VolView& d, const float* mask,
                                    float* dist, double nu, ImageCheck* check, const float* img,
                                    cudaStream_t s) {
    const long long n = m.count();
    if (check) {
        reset_check_kernel<<<1, 1, 0, s>>>(check);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    // a scratch check target when the caller does not want one
    static ImageCheck* dummy = nullptr;
    if (!check) {
        if (!dummy && cudaMalloc(&dummy, sizeof(ImageCheck)) != cudaSuccess) return cudaErrorMemoryAllocation;
        check = dummy;
        img = nullptr;
    }
    const bool vec = aligned16(mask) && aligned16(dist) && (!img || aligned16(img));
    init_check_kernel<<<grid_for((n + 3) / 4, 256), 256, 0, s>>>(m, d, img, mask, dist, nu, check, n,
                                                                 vec);
    return cudaGetLastError();
}

cudaError_t launch_transpose(const VolView& src_v, const VolView& dst_v, const float* src,
                             float* dst, bool forward, cudaStream_t s) {
    // forward: src canonical -> dst x-layout; backward: src x-layout -> dst canonical.
    const VolView& cv = forward ? src_v : dst_v;
    const VolView& tv = forward ? dst_v : src_v;
    const int RA = forward ? cv.H : cv.W, CA = forward ? cv.W : cv.H;
    const int tiles_a = (CA + 63) / 64, tiles_b = (RA + 63) / 64;
    const long long ntiles = static_cast<long long>(tiles_a) * tiles_b * cv.D * cv.B;
    const long long cap = static_cast<long long>(sm_count()) * 8;
    const int grid = static_cast<int>(ntiles < cap ? ntiles : cap);
    if (forward)
        transpose_kernel<true><<<grid, 256, 0, s>>>(cv, tv, src, dst, tiles_a, tiles_b, ntiles);
    else
        transpose_kernel<false><<<grid, 256, 0, s>>>(cv, tv, src, dst, tiles_a, tiles_b, ntiles);
    return cudaGetLastError();
}

cudaError_t launch_image_check(const VolView& v, const float* img, const float* mask,
                               ImageCheck* out, cudaStream_t s) {
    const long long n = v.count();
    reset_check_kernel<<<1, 1, 0, s>>>(out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const bool vec = (!img || aligned16(img)) && (!mask || aligned16(mask));
    image_check_kernel<<<grid_for((n + 3) / 4, 256), 256, 0, s>>>(v, img, mask, out, n, vec);
    return cudaGetLastError();
}

cudaError_t launch_gsf_sources(const VolView& v, const float* mask, const VolView& o, float* out,
                               cudaStream_t s) {
    const long long n = v.count();
    gsf_sources_kernel<<<grid_for(n, 256), 256, 0, s>>>(v, mask, o, out, n);
    return cudaGetLastError();
}

cudaError_t launch_gsf_dilate(const VolView& v, const float* dist, float* out, double theta,
                              unsigned long long* n_complement, cudaStream_t s) {
    const long long n = v.count();
    gsf_dilate_kernel<<<grid_for(n, 256), 256, 0, s>>>(v, dist, out, theta, n_complement, n);
    return cudaGetLastError();
}

cudaError_t launch_gsf_erode(const VolView& v, const float* dist, const VolView& o, float* out,
                             double theta, const int* gate, cudaStream_t s) {
    const long long n = v.count();
    gsf_erode_kernel<<<grid_for(n, 256), 256, 0, s>>>(v, dist, o, out, theta, n, gate);
    return cudaGetLastError();
}

cudaError_t launch_decide(const ImageCheck* chk, bool check_exact,
                          const unsigned long long* skip_if_zero, unsigned int status_if_skip,
                          int* gate, unsigned int* status, cudaStream_t s) {
    decide_kernel<<<1, 1, 0, s>>>(chk, check_exact ? 1 : 0, skip_if_zero, status_if_skip, gate,
                                  status);
    return cudaGetLastError();
}

cudaError_t launch_hard_seeds(const VolView& mv, const float* mask, const VolView& dv, float* dist,
                              bool invert, unsigned long long* n_seeds, cudaStream_t s) {
    const long long n = mv.count();
    hard_seed_kernel<<<grid_for(n, 256), 256, 0, s>>>(mv, mask, dv, dist, invert ? 1 : 0, n_seeds, n);
    return cudaGetLastError();
}

cudaError_t launch_threshold_count(const VolView& v, const float* mask, float* out,
                                   unsigned long long* n_complement, cudaStream_t s) {
    const long long n = v.count();
    threshold_count_kernel<<<grid_for(n, 256), 256, 0, s>>>(v, mask, out, n_complement, n);
    return cudaGetLastError();
}

cudaError_t launch_background_copy(const float* src, float* dst, long long n, int ctas,
                                   int smem_bytes, int reps, cudaStream_t s) {
    cudaFuncSetAttribute(background_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem_bytes);
    background_copy_kernel<<<ctas, 512, smem_bytes, s>>>(reinterpret_cast<const float4*>(src),
                                                          reinterpret_cast<float4*>(dst), n / 4,
                                                          reps);
    return cudaGetLastError();
}

cudaError_t launch_subtract(const float* a, const float* b, float* out, long long n,
                            cudaStream_t s) {
    subtract_kernel<<<grid_for(n, 256), 256, 0, s>>>(a, b, out, n);
    return cudaGetLastError();
}

cudaError_t launch_max_change(const VolView& v, const float* before, const float* after,
                              unsigned long long* out, cudaStream_t s) {
    const long long n = v.count();
    max_change_kernel<<<grid_for(n, 256), 256, 0, s>>>(v, before, after, out, n);
    return cudaGetLastError();
}

cudaError_t launch_splitmix(float* out, long long n, unsigned long long seed, cudaStream_t s) {
    splitmix_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, n, seed);
    return cudaGetLastError();
}

}  // namespace gdb

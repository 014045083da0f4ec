// Element-wise and layout kernels around the sweep: soft-mask init, the
// x-axis layout transposes, the per-image exactness check, GSF thresholds,
// fixpoint change reduction, and the SplitMix64 synthetic-input generator.
// All are HBM-bound streaming kernels: grid-stride loops, 16-byte accesses
// where the layout allows, grid sized as a multiple of the SM count.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "aux_kernels.cuh"

namespace gdb {

namespace {

__device__ __forceinline__ long long vox_offset(const VolView& v, long long i, int& ok) {
    // i enumerates logical voxels (b, z, y, x) densely.
    ok = 1;
    if (v.ys == v.W && v.zs == static_cast<long long>(v.H) * v.W &&
        v.vol == static_cast<long long>(v.D) * v.zs)
        return i;  // dense canonical layout
    const long long x = i % v.W;
    long long t = i / v.W;
    const long long y = t % v.H;
    t /= v.H;
    const long long z = t % v.D;
    const long long b = t / v.D;
    ok = 1;
    return b * v.vol + z * v.zs + y * v.ys + x;
}

__global__ void init_generalized_kernel(VolView m, VolView d, const float* mask, float* dist,
                                        double nu, long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int ok;
        const long long om = vox_offset(m, i, ok);
        const long long od = vox_offset(d, i, ok);
        // transforms.cpp:150-156: f32(min(nu * f64(M), f64(1e10)))
        const double v = nu * static_cast<double>(mask[om]);
        dist[od] = static_cast<float>(v < 1.0e10 ? v : 1.0e10);
    }
}

// Transpose [b][z][y][x] (src view) -> [b][x][z][y] (dst view) or back.
// 32x32 tiles over (y, x) per (b, z); reads and writes both coalesced.
template <bool FWD>
__global__ void transpose_kernel(VolView src_v, VolView dst_v, const float* src, float* dst) {
    __shared__ float tile[32][33];
    const int D = src_v.D, H = src_v.H, W = src_v.W;
    for (int bz = blockIdx.z; bz < D * src_v.B; bz += gridDim.z) {
    const int z = bz % D, b = bz / D;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    if (FWD) {
        // src [b][z][y][x] row pitch ys; dst [b][x][z][y]: element (x,z,y) at x*dst.zs + z*dst.ys + y
        for (int k = ty; k < 32; k += 8) {
            const int y = y0 + k, x = x0 + tx;
            if (y < H && x < W)
                tile[k][tx] = src[b * src_v.vol + z * src_v.zs + static_cast<long long>(y) * src_v.ys + x];
        }
        __syncthreads();
        for (int k = ty; k < 32; k += 8) {
            const int x = x0 + k, y = y0 + tx;
            if (y < H && x < W)
                dst[b * dst_v.vol + static_cast<long long>(x) * dst_v.zs + z * dst_v.ys + y] = tile[tx][k];
        }
    } else {
        // src [b][x][z][y] -> dst [b][z][y][x]
        for (int k = ty; k < 32; k += 8) {
            const int x = x0 + k, y = y0 + tx;
            if (y < H && x < W)
                tile[k][tx] = src[b * src_v.vol + static_cast<long long>(x) * src_v.zs + z * src_v.ys + y];
        }
        __syncthreads();
        for (int k = ty; k < 32; k += 8) {
            const int y = y0 + k, x = x0 + tx;
            if (y < H && x < W)
                dst[b * dst_v.vol + z * dst_v.zs + static_cast<long long>(y) * dst_v.ys + x] = tile[tx][k];
        }
    }
    __syncthreads();
    }
}

// Image exactness: with x = m * 2^t (m odd), all pairwise differences are
// exact in f32 when (max exponent) - (min t) <= 23 (same sign) / 22 (mixed).
// Also flags masks outside [0, 1] (transforms.cpp:22-28).
__global__ void image_check_kernel(VolView v, const float* img, const float* mask,
                                   ImageCheck* out, long long n) {
    int emax = -1000, tmin = 1000, pos = 0, neg = 0, bad_mask = 0, nonfinite = 0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int ok;
        const long long o = vox_offset(v, i, ok);
        if (img) {
            const float x = img[o];
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
                    const uint32_t full = man | 0x800000u;
                    e = ebits - 127;
                    t = ebits - 150 + (__ffs(full) - 1);
                }
                emax = max(emax, e);
                tmin = min(tmin, t);
                if (u >> 31) neg = 1; else pos = 1;
            }
        }
        if (mask) {
            const float m = mask[o];
            if (!(m >= 0.0f && m <= 1.0f)) bad_mask = 1;
        }
    }
    for (int s = 16; s > 0; s >>= 1) {
        emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, s));
        tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, s));
        pos |= __shfl_xor_sync(0xffffffffu, pos, s);
        neg |= __shfl_xor_sync(0xffffffffu, neg, s);
        bad_mask |= __shfl_xor_sync(0xffffffffu, bad_mask, s);
        nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out->emax, emax);
        atomicMin(&out->tmin, tmin);
        if (pos) atomicOr(&out->pos, 1);
        if (neg) atomicOr(&out->neg, 1);
        if (bad_mask) atomicOr(&out->bad_mask, 1);
        if (nonfinite) atomicOr(&out->nonfinite, 1);
    }
}

// out = [M >= 0.5] ? 0 : 1   (complement_mask(threshold_mask(M)), transforms.cpp:30-48)
__global__ void gsf_sources_kernel(VolView v, const float* mask, VolView o, float* out,
                                   long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int ok;
        const float m = mask[vox_offset(v, i, ok)];
        out[vox_offset(o, i, ok)] = m >= 0.5f ? 0.0f : 1.0f;
    }
}

// dilate epilogue fused with the erode prologue (transforms.cpp:195-201, 211-219):
//   dil = [f64(D) <= theta];  K = threshold(dil) = dil;  count(complement(K)).
__global__ void gsf_dilate_kernel(VolView v, const float* dist, float* out, double theta,
                                  unsigned long long* n_complement, long long n) {
    unsigned long long cnt = 0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int ok;
        const long long o = vox_offset(v, i, ok);
        const float dil = static_cast<double>(dist[o]) <= theta ? 1.0f : 0.0f;
        out[o] = dil;
        cnt += dil >= 0.5f ? 0 : 1;
    }
    for (int s = 16; s > 0; s >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_complement, cnt);
}

// erode epilogue: out = [f64(D) > theta]
__global__ void gsf_erode_kernel(VolView v, const float* dist, VolView o, float* out, double theta,
                                 long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int ok;
        const float d = dist[vox_offset(v, i, ok)];
        out[vox_offset(o, i, ok)] = static_cast<double>(d) > theta ? 1.0f : 0.0f;
    }
}

// Fixpoint change: max over voxels of f64(before) - f64(after) (scan_parallel.cpp:386-392).
// Non-negative values only matter (change starts at 0), so the f64 bit pattern
// orders like an unsigned integer.
__global__ void max_change_kernel(VolView v, const float* before, const float* after,
                                  unsigned long long* out, long long n) {
    double m = 0.0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int ok;
        const long long o = vox_offset(v, i, ok);
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

int grid_for(long long n, int threads) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const long long need = (n + threads - 1) / threads;
    const long long cap = static_cast<long long>(sms) * 8;
    return static_cast<int>(need < cap ? (need > 0 ? need : 1) : cap);
}

}  // namespace

cudaError_t launch_init_generalized(const VolView& m, const VolView& d, const float* mask,
                                    float* dist, double nu, cudaStream_t s) {
    const long long n = m.count();
    init_generalized_kernel<<<grid_for(n, 256), 256, 0, s>>>(m, d, mask, dist, nu, n);
    return cudaGetLastError();
}

cudaError_t launch_transpose(const VolView& src_v, const VolView& dst_v, const float* src,
                             float* dst, bool forward, cudaStream_t s) {
    // src_v / dst_v carry the logical (D, H, W) of the [z][y][x] volume in both
    // directions; zs/ys/vol are the respective layouts' strides.
    const VolView& lv = forward ? src_v : dst_v;
    dim3 grid((lv.W + 31) / 32, (lv.H + 31) / 32, std::min(lv.D * lv.B, 65535));
    dim3 block(32, 8);
    VolView a = src_v, b = dst_v;
    a.D = b.D = lv.D;
    a.H = b.H = lv.H;
    a.W = b.W = lv.W;
    if (forward)
        transpose_kernel<true><<<grid, block, 0, s>>>(a, b, src, dst);
    else
        transpose_kernel<false><<<grid, block, 0, s>>>(a, b, src, dst);
    return cudaGetLastError();
}

cudaError_t launch_image_check(const VolView& v, const float* img, const float* mask,
                               ImageCheck* out, cudaStream_t s) {
    const long long n = v.count();
    ImageCheck init{-1000, 1000, 0, 0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(out, &init, sizeof(init), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    image_check_kernel<<<grid_for(n, 256), 256, 0, s>>>(v, img, mask, out, n);
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
                             double theta, cudaStream_t s) {
    const long long n = v.count();
    gsf_erode_kernel<<<grid_for(n, 256), 256, 0, s>>>(v, dist, o, out, theta, n);
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

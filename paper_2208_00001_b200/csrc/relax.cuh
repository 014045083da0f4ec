// Relaxation arithmetic shared by the sweep kernels (sweep.cu, rowchain.cu):
// one candidate d_q + cost(p, q) per neighbour, per-voxel accumulators and the
// 3-column row window.  The bit-exactness argument is in sweep.cuh.
// Reference: relax_row<K,Contig> /root/reference/proj/src/scan_parallel.cpp:44-87,
// relax_cost / classify_cost scan_common.hpp:15-21,52-68.
#pragma once

#include "sweep.cuh"

namespace gdb {
namespace {

__device__ __forceinline__ float finf() { return __int_as_float(0x7f800000); }

__device__ __forceinline__ unsigned long long f2_bits(float2 v) {
    return (static_cast<unsigned long long>(__float_as_uint(v.y)) << 32) | __float_as_uint(v.x);
}
__device__ __forceinline__ float2 bits_f2(unsigned long long b) {
    return make_float2(__uint_as_float(static_cast<uint32_t>(b)),
                       __uint_as_float(static_cast<uint32_t>(b >> 32)));
}
// Packed sm_100 f32x2 arithmetic (SASS FADD2); |x| folds into the operand.
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(r);
}
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(r);
}

// MUFU.SQRT alone: .ftz drops the denormal-range rescaling (FSETP + 2 FMUL per
// candidate).  x = lambda di^2 + c0 is denormal only when both terms are below
// 1.2e-38, far inside the 1e-6 absolute tolerance.
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// One relaxation candidate d_q + cost(p, q) rounded to f32 (see sweep.cuh for
// why per-candidate rounding is exact).  k = (du+1)*3 + (dv+1).
template <int KIND, bool F64>
__device__ __forceinline__ float candidate(float pq, float iq, float ip, int k,
                                           const SweepParams& p) {
    if constexpr (KIND == kSpatial) {
        return static_cast<float>(static_cast<double>(pq) + p.rho[k]);
    } else if constexpr (KIND == kIntensity) {
        if constexpr (F64) {
            const double di = static_cast<double>(ip) - static_cast<double>(iq);
            return static_cast<float>(static_cast<double>(pq) + fabs(di));
        } else {
            return pq + fabsf(ip - iq);
        }
    } else {
        if constexpr (F64) {
            const double di = static_cast<double>(ip) - static_cast<double>(iq);
            // relax_cost<Blend> as compiled by the reference: sqrt(fma(lambda*di, di, c0))
            return static_cast<float>(static_cast<double>(pq) +
                                      sqrt(fma(p.lambda * di, di, p.c0[k])));
        } else {
            // MUFU.SQRT (about 1 ulp): the IEEE sqrtf adds a slow-path CALL per
            // candidate that serialises the 9-candidate min (3x slower step).
            // sqrt(lambda di^2 + c0) as sqrt(lambda) * sqrt(di^2 + c0 / lambda):
            // FADD, FFMA, MUFU.SQRT, FFMA per candidate instead of FADD, FMUL,
            // FFMA, MUFU.SQRT, FADD (within the tolerance like the f32 form).
            const float di = ip - iq;
            return fmaf(p.sqrt_lambda_f, sqrt_approx(fmaf(di, di, p.c0l_f[k])), pq);
        }
    }
}

// Per-voxel accumulator.  Spatial keeps one f32 minimum per rho class
// (class = (du != 0) + 2 (dv != 0)) and adds rho once per class at the end.
template <int KIND, bool F64>
struct Acc {
    float best;
    __device__ __forceinline__ void init(float dold) { best = dold; }
    __device__ __forceinline__ void add(float pq, float iq, float ip, int k, const SweepParams& p) {
        best = fminf(best, candidate<KIND, F64>(pq, iq, ip, k, p));
    }
    __device__ __forceinline__ float final(const SweepParams&) const { return best; }
};

template <bool F64>
struct Acc<kSpatial, F64> {
    float best;
    float m[4];
    __device__ __forceinline__ void init(float dold) {
        best = dold;
        m[0] = m[1] = m[2] = m[3] = finf();
    }
    __device__ __forceinline__ void add(float pq, float, float, int k, const SweepParams&) {
        const int du = k / 3 - 1, dv = k % 3 - 1;
        const int c = (du != 0 ? 1 : 0) + (dv != 0 ? 2 : 0);
        m[c] = fminf(m[c], pq);
    }
    __device__ __forceinline__ float final(const SweepParams& p) const {
        // class representatives (du,dv) = (0,0),(1,0),(0,1),(1,1) -> k = 4,7,5,8
        // Rounding to f32 is monotone, so the min of the f64 sums rounds to the
        // min of the rounded sums: one F2F down instead of four (conversions
        // run at a quarter of the FP32 rate).  No NaNs reach here.
        const double s0 = static_cast<double>(m[0]) + p.rho[4];
        const double s1 = static_cast<double>(m[1]) + p.rho[7];
        const double s2 = static_cast<double>(m[2]) + p.rho[5];
        const double s3 = static_cast<double>(m[3]) + p.rho[8];
        const double a = s0 < s1 ? s0 : s1, b = s2 < s3 ? s2 : s3;
        return fminf(best, static_cast<float>(a < b ? a : b));
    }
};

// FADD2 packing of column pairs: off — ptxas cannot fold |d| into the packed
// add and the odd-aligned pairs cost register moves (measured: 86 vs 68
// instructions per voxel); the scalar FADD with an |operand| is cheaper.
constexpr bool kPackedIntensity = false;

// The 3-column windows of one previous-plane row for a lane's 4 columns:
// pw/iw[0] = column v-1, [1..4] = own columns, [5] = column v+4.
template <int KIND, bool F64>
__device__ __forceinline__ void relax_row(Acc<KIND, F64> (&acc)[kC], const float (&pw)[6],
                                          const float (&iw)[6], const float (&ip)[kC], int du,
                                          const SweepParams& p) {
    if constexpr (KIND == kIntensity && !F64 && kPackedIntensity) {
        // Packed column pairs: two FADD2 per candidate pair instead of four FADD.
#pragma unroll
        for (int q = 0; q < kC / 2; ++q) {
            const int c0 = 2 * q;
            const float2 ip2 = make_float2(ip[c0], ip[c0 + 1]);
#pragma unroll
            for (int dv = -1; dv <= 1; ++dv) {
                const float2 pq = make_float2(pw[c0 + dv + 1], pw[c0 + dv + 2]);
                const float2 iq = make_float2(iw[c0 + dv + 1], iw[c0 + dv + 2]);
                float2 d = f2_sub(ip2, iq);
                d.x = fabsf(d.x);
                d.y = fabsf(d.y);
                const float2 cand = f2_add(pq, d);
                acc[c0].best = fminf(acc[c0].best, cand.x);
                acc[c0 + 1].best = fminf(acc[c0 + 1].best, cand.y);
            }
        }
    } else {
#pragma unroll
        for (int c = 0; c < kC; ++c)
#pragma unroll
            for (int dv = -1; dv <= 1; ++dv)
                acc[c].add(pw[c + dv + 1], iw[c + dv + 1], ip[c], (du + 1) * 3 + (dv + 1), p);
    }
}

}  // namespace
}  // namespace gdb

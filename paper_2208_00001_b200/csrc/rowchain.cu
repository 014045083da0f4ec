// Row-chain kernel: directional passes whose plane is a single row (2D images,
// nu == 1).  Replaces run_pass<K>'s 2D branch (/root/reference/proj/src/
// scan_parallel.cpp:119-139: v chunked by thread, `omp barrier` per row) for a
// forward+backward pair on one axis.
//
// One CTA per image owns the whole row for the whole pair: each thread keeps 4
// consecutive columns of the previous row (distance and intensity) in
// registers, v +- 1 comes from warp shuffles and the warp-edge columns from a
// double-buffered shared-memory slot, so a plane step is one relax of 4 voxels
// plus ONE barrier -- no inter-CTA hand-off at all (the persistent strip kernel
// pays a TMA ring round trip and a producer warp per step for a row that is
// only 2 KB).  Rows ahead are prefetched into a register ring PF steps deep.
// The backward pass reads the forward pass's output, written by the same
// thread: loads of it are issued after the store (program order), and the PF
// planes nearest the turn -- not yet written when their prefetch would issue --
// come from a shared-memory turn buffer filled by the last forward steps.
// Arithmetic is relax_row / Acc (relax.cuh), identical to the strip kernel.
#include <cuda_runtime.h>

#include "relax.cuh"
#include "rowchain.cuh"

namespace gdb {
namespace {

constexpr int kPF = 8;  // prefetch depth (steps)

template <int KIND, bool F64>
__global__ void __launch_bounds__(512, 1) row_chain_kernel(const __grid_constant__ SweepParams p) {
    constexpr bool kI = KIND != kSpatial;
    extern __shared__ float4 smem4[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nw = blockDim.x >> 5, nvp = blockDim.x * kC;
    float4* edges = smem4;                                       // [2 parities][nw]: {P0, I0, P3, I3}
    float* tbuf = reinterpret_cast<float*>(smem4 + 2 * nw);      // [kPF][nvp] turn buffer
    const float INF = finf();
    const int v0 = tid * kC;
    bool colv[kC];
#pragma unroll
    for (int q = 0; q < kC; ++q) colv[q] = v0 + q < p.nv;
    const bool any = colv[0];
    float* const dist = p.dist + static_cast<long long>(blockIdx.x) * p.vol_stride + v0;
    const float* const img = p.image + static_cast<long long>(blockIdx.x) * p.vol_stride + v0;
    const int n1 = p.ns - 1, J = p.npass * n1;
    auto plane = [&](int j) {
        if (j <= n1) return p.first_orient > 0 ? j : n1 - j;
        const int k = j - n1;
        return p.first_orient > 0 ? n1 - k : k;
    };
    // Distances of step j come from the turn buffer when the forward pass wrote
    // that plane fewer than kPF steps before step j.
    auto in_turn = [&](int j) { return j > n1 && j <= n1 + kPF; };
    auto ld4 = [&](const float* base, int j) -> float4 {
        if (!any) return make_float4(INF, INF, INF, INF);
        return *reinterpret_cast<const float4*>(base + static_cast<long long>(plane(j)) * p.ss);
    };
    auto to_arr = [&](float4 v, float (&a)[kC], float fill) {
        a[0] = colv[0] ? v.x : fill;
        a[1] = colv[1] ? v.y : fill;
        a[2] = colv[2] ? v.z : fill;
        a[3] = colv[3] ? v.w : fill;
    };
    auto save_turn = [&](int j, const float (&N)[kC]) {
        const int t = n1 - j - 1;  // backward step n1 + t + 1 reads this plane
        if (p.npass == 2 && t >= 0 && t < kPF)
            *reinterpret_cast<float4*>(tbuf + t * nvp + v0) = make_float4(N[0], N[1], N[2], N[3]);
    };
    auto put_edges = [&](int j, const float (&N)[kC], const float (&I)[kC]) {
        float4* e = edges + (j & 1) * nw + warp;
        if (lane == 0) { e->x = N[0]; e->y = I[0]; }
        if (lane == kWarpLast) { e->z = N[kC - 1]; e->w = I[kC - 1]; }
    };

    float P[kC], PI[kC];
    float4 Rd[kPF], Ri[kPF];
    // step 0: the first plane is final as loaded
    {
        float4 d0 = ld4(dist, 0), i0 = kI ? ld4(img, 0) : make_float4(0.f, 0.f, 0.f, 0.f);
        to_arr(d0, P, INF);
        to_arr(i0, PI, 0.0f);
        save_turn(0, P);
        put_edges(0, P, PI);
    }
#pragma unroll
    for (int u = 0; u < kPF; ++u) {
        const int j = 1 + u;
        if (j <= J) {
            if (!in_turn(j)) Rd[u] = ld4(dist, j);
            if (kI) Ri[u] = ld4(img, j);
        }
    }
    __syncthreads();

    for (int j0 = 1; j0 <= J; j0 += kPF) {
#pragma unroll
        for (int u = 0; u < kPF; ++u) {
            const int j = j0 + u;
            if (j > J) break;
            // previous row's neighbours v-1 / v+4
            const float4* e = edges + ((j - 1) & 1) * nw;
            float lP = __shfl_up_sync(kFullMask, P[kC - 1], 1);
            float lI = __shfl_up_sync(kFullMask, PI[kC - 1], 1);
            float rP = __shfl_down_sync(kFullMask, P[0], 1);
            float rI = __shfl_down_sync(kFullMask, PI[0], 1);
            if (lane == 0) {
                const float4 w = warp > 0 ? e[warp - 1] : make_float4(0.f, 0.f, INF, 0.f);
                lP = w.z;
                lI = w.w;
            }
            if (lane == kWarpLast) {
                const float4 w = warp + 1 < nw ? e[warp + 1] : make_float4(INF, 0.f, 0.f, 0.f);
                rP = w.x;
                rI = w.y;
            }
            const float pw[6] = {lP, P[0], P[1], P[2], P[3], rP};
            const float iw[6] = {lI, PI[0], PI[1], PI[2], PI[3], rI};
            float dold[kC], ic[kC];
            if (in_turn(j)) {
                const float4 t = *reinterpret_cast<const float4*>(tbuf + (j - n1 - 1) * nvp + v0);
                to_arr(t, dold, INF);
            } else {
                to_arr(Rd[u], dold, INF);
            }
            if (kI) to_arr(Ri[u], ic, 0.0f);
            else
#pragma unroll
                for (int q = 0; q < kC; ++q) ic[q] = 0.0f;
            Acc<KIND, F64> acc[kC];
#pragma unroll
            for (int q = 0; q < kC; ++q) acc[q].init(dold[q]);
            relax_row<KIND, F64>(acc, pw, iw, ic, 0, p);
            float N[kC];
#pragma unroll
            for (int q = 0; q < kC; ++q) N[q] = colv[q] ? acc[q].final(p) : INF;
            if (any) {
                float* o = dist + static_cast<long long>(plane(j)) * p.ss;
                if (colv[kC - 1]) {
                    *reinterpret_cast<float4*>(o) = make_float4(N[0], N[1], N[2], N[3]);
                } else {
#pragma unroll
                    for (int q = 0; q < kC; ++q)
                        if (colv[q]) o[q] = N[q];
                }
            }
            save_turn(j, N);
            put_edges(j, N, ic);
            // prefetch step j + kPF into the slot just consumed (after the store:
            // a backward plane outside the turn window was written at a step <= j)
            const int jn = j + kPF;
            if (jn <= J) {
                if (!in_turn(jn)) Rd[u] = ld4(dist, jn);
                if (kI) Ri[u] = ld4(img, jn);
            }
#pragma unroll
            for (int q = 0; q < kC; ++q) {
                P[q] = N[q];
                PI[q] = ic[q];
            }
            __syncthreads();
        }
    }
}

template <int KIND, bool F64>
cudaError_t launch_one(const SweepParams& p, cudaStream_t s) {
    const int threads = ((p.nv + kC - 1) / kC + 31) / 32 * 32;
    const int nw = threads / 32;
    const size_t smem = 2 * nw * sizeof(float4) + static_cast<size_t>(kPF) * threads * kC * 4;
    if (smem > 48 * 1024) {  // per device: set on every wide launch (cheap)
        const cudaError_t e = cudaFuncSetAttribute(
            row_chain_kernel<KIND, F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
            static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    row_chain_kernel<KIND, F64><<<p.nvol, threads, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_row_chain(int kind, bool f64, const SweepParams& p, cudaStream_t s) {
    if (p.nv > kRowChainMaxWidth || p.nu != 1) return cudaErrorInvalidValue;
    switch (kind) {
        case kSpatial: return launch_one<kSpatial, false>(p, s);
        case kIntensity: return f64 ? launch_one<kIntensity, true>(p, s) : launch_one<kIntensity, false>(p, s);
        default: return f64 ? launch_one<kBlend, true>(p, s) : launch_one<kBlend, false>(p, s);
    }
}

}  // namespace gdb
